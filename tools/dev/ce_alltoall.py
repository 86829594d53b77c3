# SPDX-License-Identifier: Apache-2.0
"""Copy-engine all-to-all probe (one process, all GPUs): every GPU pulls
`mb` MB from every peer (the FC step's W re-replication / X gather shape),
each peer's piece split into `split` row ranges on separate streams of the
puller. Prints per-GPU ingress GB/s (wall time of the slowest GPU)."""
import sys
import time

import torch

n = torch.cuda.device_count()
mb = float(sys.argv[1]) if len(sys.argv) > 1 else 18.9
nbytes = int(mb * 2**20) // 16 * 16
src = [torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{d}") for d in range(n)]
dst = [[torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{d}") for _ in range(n)] for d in range(n)]
for split in (1, 2, 4, 8):
    streams = [[torch.cuda.Stream(device=d) for _ in range(n * split)] for d in range(n)]

    def run():
        for d in range(n):
            with torch.cuda.device(d):
                for k in range(1, n):
                    p = (d + k) % n
                    step = nbytes // split // 16 * 16
                    for h in range(split):
                        lo = h * step
                        hi = nbytes if h == split - 1 else lo + step
                        with torch.cuda.stream(streams[d][p * split + h]):
                            dst[d][p][lo:hi].copy_(src[p][lo:hi], non_blocking=True)

    for _ in range(3):
        run()
    for d in range(n):
        torch.cuda.synchronize(d)
    t0 = time.perf_counter()
    reps = 10
    for _ in range(reps):
        run()
    for d in range(n):
        torch.cuda.synchronize(d)
    dt = (time.perf_counter() - t0) / reps
    print(f"gpus={n} per-peer {mb} MB split={split}: {dt * 1e6:.0f} us per all-to-all, "
          f"ingress {(n - 1) * nbytes / dt / 1e9:.0f} GB/s per GPU", flush=True)
