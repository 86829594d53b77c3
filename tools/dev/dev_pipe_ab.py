# SPDX-License-Identifier: Apache-2.0
"""A/B of in-GEMM panel pipelining in ONE process per rank (same clocks):
alternates pipelining on/off for the C3 loop (independent and dependent
chain) and for the FC dW GEMM, several rounds; prints medians (max over
ranks). torchrun --nproc-per-node N tools/dev/dev_pipe_ab.py [n]"""
import math
import os
import statistics
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
from paper_1611_07819_b200 import gridmath as G  # noqa: E402

rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
obj = [G.nccl_unique_id() if rank == 0 else None]
dist.broadcast_object_list(obj, src=0)
s = G.Session(workers=world, spmd_rank=rank, devices=[local], nccl_id=obj[0], panel_cache_bytes=1)
g = G.makeWorkerGroup(world)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
pr, pc = {2: (1, 2), 4: (2, 2), 8: (2, 4)}[world]
lay = G.makeGridLayout(n, n, pr, pc, g)
A, B, C = (s.createMatrix(n, n, G.Precision.BF16, lay) for _ in range(3))
s.fillUniform(A, 1)
s.fillUniform(B, 2)
alpha = 1.0 / (math.sqrt(1.0 / 3.0) * math.sqrt(n))


def timed(fn, steps):
    s.synchronize()
    dist.barrier()
    s.timerStart()
    for i in range(steps):
        fn(i)
    ms = s.timerStop() / steps
    t = torch.tensor([ms], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.item()


pair = [A, C]
loops = {
    "indep": lambda i: s.gemmAsync(A, B, C),
    "dep": lambda i: s.gemmAsync(pair[i % 2], B, pair[(i + 1) % 2], alpha, 0.0),
}
res = {(m, k): [] for m in (1, 0) for k in loops}
for rnd in range(int(os.environ.get("AB_ROUNDS", "5"))):
    for mode in (1, 0):
        s.setPanelPipelining(bool(mode))
        for k, fn in loops.items():
            timed(fn, 2)  # warm
            res[(mode, k)].append(timed(fn, 6))
s.setPanelPipelining(True)
# FC dW GEMM: dW = X^T . delta (X gathered), X refreshed each time
batch, fi, fo = 4096, 9216, 4096
X = s.createMatrix(batch, fi, G.Precision.BF16, G.makeRowBlockLayout(batch, fi, g))
DL = s.createMatrix(batch, fo, G.Precision.BF16, G.makeRowBlockLayout(batch, fo, g))
dW = s.createMatrix(fi, fo, G.Precision.BF16, G.makeColBlockLayout(fi, fo, g))
s.fillUniform(DL, 4)
fc = {1: [], 0: []}
for rnd in range(int(os.environ.get("AB_ROUNDS", "5"))):
    for mode in (1, 0):
        s.setPanelPipelining(bool(mode))
        fc[mode].append(timed(lambda i: (s.fillUniform(X, 100 + i), s.gemmAsync(X, DL, dW, 1.0, 0.0, True, False)), 10))
if rank == 0:
    for (mode, k), v in sorted(res.items()):
        print(f"C3 {n}^3 N={world} pipelining={'on ' if mode else 'off'} {k:5s} median {statistics.median(v):8.3f} ms  "
              f"{2 * n ** 3 / statistics.median(v) / 1e9:8.1f} TFLOP/s  runs {['%.3f' % x for x in v]}")
    for mode in (1, 0):
        print(f"FC fill X + dW gemm N={world} pipelining={'on ' if mode else 'off'} median {statistics.median(fc[mode]) * 1e3:7.1f} us")
s.close()
dist.destroy_process_group()
