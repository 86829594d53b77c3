# SPDX-License-Identifier: Apache-2.0
"""Single-process multi-GPU run of the bench workload with the copy-engine
transport (one worker per visible GPU). Dev tool: shows whether copy-engine
panel pulls overlap the persistent GEMM (they use no SMs)."""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_1611_07819_b200 import gridmath as G  # noqa: E402


def main():
    w = torch.cuda.device_count()
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
    transport = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    pr, pc = {1: (1, 1), 2: (1, 2), 4: (2, 2), 8: (2, 4)}[w]
    s = G.Session(workers=w, devices=list(range(w)), transport=transport, panel_cache_bytes=1)
    lay = G.makeGridLayout(n, n, pr, pc, G.makeWorkerGroup(w))
    A = s.createMatrix(n, n, G.Precision.BF16, lay)
    B = s.createMatrix(n, n, G.Precision.BF16, lay)
    C = s.createMatrix(n, n, G.Precision.BF16, lay)
    s.fillUniform(A, 1)
    s.fillUniform(B, 2)
    for _ in range(3):
        s.gemmAsync(A, B, C)
    s.synchronize()
    steps = 10
    s.timerStart()
    for _ in range(steps):
        s.gemmAsync(A, B, C)
    ms = s.timerStop()
    kms = max(s.lastOpKernelMs())
    tf = 2.0 * n ** 3 * steps / (ms / 1e3) / 1e12
    s.synchronize()
    s.gemmAsync(A, B, C)
    s.synchronize()
    print(f"workers={w} transport={transport} n={n}: {tf:.1f} TFLOP/s, {ms / steps:.3f} ms/step, "
          f"kernel {kms:.3f} ms, isolated comm {max(s.lastOpCommMs()):.3f} ms", flush=True)
    s.close()


if __name__ == "__main__":
    main()
