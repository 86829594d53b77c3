# SPDX-License-Identifier: Apache-2.0
"""One process per GPU (the benchmark's mode): torchrun over the GPUs present
runs tools/spmd_check.py -- NCCL data plane, SUMMA pipelining, replication --
and requires bitwise equality with the single-GPU result. Skips with < 2 GPUs."""
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


@pytest.mark.timeout(600)
def test_spmd_nccl_path_matches_single_gpu():
    n = _gpus()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    n = 4 if n >= 4 else 2
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "tools", "spmd_check.py")]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=540)
    assert out.returncode == 0 and "SPMD_CHECK PASS" in out.stdout, out.stdout[-3000:] + out.stderr[-3000:]
