# SPDX-License-Identifier: Apache-2.0
"""In-GEMM panel pipelining (north_star subsystem 3): gathered bands land
block by block -- (m-chunk | n-chunk) x k-panel -- while the tcgen05 GEMM
runs, its producer warp polling each block's ready flag before loading it.
Results must be bitwise identical to the unpipelined path (GEMM waits for
whole bands) and to one worker, including a dependent chain whose every
operand is the previous GEMM's output, and with a ready-flag ring so small
that regions are reused every few ops."""
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle as O
from conftest import ROOT

pytestmark = pytest.mark.gpu


def _run(tmp_path, tag, cfg, steps=40):
    out = os.path.join(tmp_path, f"{tag}.npz")
    env = dict(os.environ)
    env["GM_DEBUG_CONFIG"] = cfg
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "pipeline_check.py"), out, str(steps)],
                       capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    return dict(np.load(out)), r.stderr


@pytest.mark.timeout(900)
def test_panel_pipelining_bitwise_equals_whole_band_path(tmp_path):
    # panel_min_gflop=0: pipeline these test-sized GEMMs too (the product
    # default pipelines GEMMs of >= 1 TFLOP per worker)
    on, log = _run(tmp_path, "on", "verbose=1,panel_min_gflop=0")
    off, _ = _run(tmp_path, "off", "panel_flags=0")
    small, _ = _run(tmp_path, "ring", "ready_slots=48,panel_min_gflop=0", steps=120)
    # the pipelined launches really polled flags
    assert "panels=" in log and any(f"panels={p}" in log for p in range(1, 64)), log[-2000:]
    assert any(ln.split("panels=")[1].strip() != "0" for ln in log.splitlines() if "panels=" in ln)
    # the replica-polling forward ran (a 1-panel B flag set per launch)
    assert "replica_fwd" in on
    for k in off:
        if k.startswith("chain"):
            continue
        assert np.array_equal(on[k].view(np.uint8), off[k].view(np.uint8)), k
        assert np.array_equal(small[k].view(np.uint8), off[k].view(np.uint8)), k
    assert np.array_equal(on["chain"].view(np.uint8), on["chain_1worker"].view(np.uint8))
    assert np.array_equal(on["chain"].view(np.uint8), off["chain"].view(np.uint8))
    assert np.array_equal(small["chain"].view(np.uint8), small["chain_1worker"].view(np.uint8))
    vals = (on["chain"].view(np.uint16).astype(np.uint32) << 16).view(np.float32)
    assert np.isfinite(vals).all() and np.abs(vals).max() > 0


@pytest.mark.timeout(600)
def test_panel_pipelining_matches_oracle(tmp_path):
    on, _ = _run(tmp_path, "o", "panel_min_gflop=0", steps=2)
    from paper_1611_07819_b200 import gridmath as G
    m, n, k = 1536, 1280, 4608
    a = O.fill_uniform(m, k, 3, 7)
    b = O.fill_uniform(k, n, 3, 8)
    rows = (700, 716)
    want = O.gemm_c(m, n, k, a, 3, b, 3, np.zeros((m, n), np.float32), 1, 1.0, 0.0, 0, 0, rows)
    assert O.rel_fro(on["grid_bf16"][rows[0]:rows[1]], want[rows[0]:rows[1]]) <= 1e-5
    del G
