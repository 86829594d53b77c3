# SPDX-License-Identifier: Apache-2.0
"""One process per worker (the benchmark's mode): torchrun runs
tools/spmd_check.py -- both data planes, SUMMA panel exchange, replication,
reshape, RAW/WAR chains, record/replay, host streaming, checkpoint -- and
requires bitwise equality with the single-GPU result.

* one rank per GPU (>= 2 GPUs): NCCL control channel, IPC and NCCL planes;
* two ranks per GPU (any box, including a 1-GPU one): the gloo control
  channel and the IPC copy-engine plane (NCCL cannot put two ranks on one
  GPU), with in-GEMM panel pipelining forced on for every 16-bit GEMM.
  On a 4-GPU box this runs the 2x4 grid's 8 ranks."""
import os
import socket
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def _gpus():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


def _run(nproc, debug_config=None):
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "tools", "spmd_check.py")]
    env = dict(os.environ)
    if debug_config:
        env["GM_DEBUG_CONFIG"] = debug_config
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=840, env=env)
    assert out.returncode == 0 and "SPMD_CHECK PASS" in out.stdout, out.stdout[-3000:] + out.stderr[-3000:]
    return out.stdout


@pytest.mark.timeout(900)
def test_spmd_one_rank_per_gpu_matches_single_gpu():
    n = _gpus()
    if n < 2:
        pytest.skip("needs >= 2 GPUs (the two-ranks-per-GPU test covers 1-GPU boxes)")
    _run(4 if n >= 4 else 2)


@pytest.mark.timeout(900)
def test_spmd_two_ranks_per_gpu_gloo_control_matches_single_gpu():
    n = _gpus()
    world = 8 if n >= 4 else (4 if n >= 2 else 2)
    # panel_min_gflop=0: the (small) check GEMMs take the in-GEMM panel
    # pipelining path across ranks too; graph_replay=1: the FC step's replays
    # run as one CUDA graph per rank (IPC flag waits / writes captured),
    # checked against op-by-op replay in one process
    out = _run(world, "panel_min_gflop=0,graph_replay=1")
    assert f"SPMD_CHECK world={world}" in out and "control=gloo" in out, out[-2000:]
    assert "graph_launches=2 bitwise_vs_1process=True" in out, out[-2000:]


@pytest.mark.timeout(1200)
def test_spmd_headline_size_on_the_bench_grid_matches_single_gpu():
    """bf16 32768^3 on the bench's grid (2 ranks on a 1-GPU box, 1x2; 8 ranks
    = the 2x4 grid on a 4-GPU box) plus a dependent GEMM on its output, every
    rank's tiles bitwise equal to one GPU."""
    n = _gpus()
    world = 8 if n >= 4 else 2
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "tools", "spmd_fullsize.py")]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=1100)
    assert out.returncode == 0 and "SPMD_FULLSIZE PASS" in out.stdout, out.stdout[-3000:] + out.stderr[-3000:]
