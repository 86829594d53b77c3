# SPDX-License-Identifier: Apache-2.0
"""Per-op device time of the FC train step (bench --config fc) under torchrun:
each op timed alone (timerStart/timerStop, max over ranks), then the whole
step replayed back to back. Shows where a step's time goes at N > 1."""
import math
import os
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
s = G.Session(workers=world, spmd_rank=rank, devices=[local], nccl_id=obj[0])
g = G.makeWorkerGroup(world)
batch, fi, fo = 4096, 9216, 4096
P = G.Precision.BF16
X = s.createMatrix(batch, fi, P, G.makeRowBlockLayout(batch, fi, g))
W = s.createMatrix(fi, fo, P, G.makeColBlockLayout(fi, fo, g))
Bv = s.createMatrix(1, fo, P, G.makeColBlockLayout(1, fo, g))
Z = s.createMatrix(batch, fo, P, G.makeRowBlockLayout(batch, fo, g))
ACT = s.createMatrix(batch, fo, P, G.makeRowBlockLayout(batch, fo, g))
DL = s.createMatrix(batch, fo, P, G.makeRowBlockLayout(batch, fo, g))
dW = s.createMatrix(fi, fo, P, G.makeColBlockLayout(fi, fo, g))
dB = s.createMatrix(1, fo, P, G.makeColBlockLayout(1, fo, g))
ROW = s.createMatrix(batch, 1, P, G.makeRowBlockLayout(batch, 1, g))
dX = s.createMatrix(batch, fi, P, G.makeRowBlockLayout(batch, fi, g))
s.fillUniform(X, 1)
s.fillUniform(W, 2, -1 / math.sqrt(fi), 1 / math.sqrt(fi))
s.fillUniform(Bv, 3)
s.fillUniform(DL, 4)
s.replicateSync(W)
s.replicateSync(Bv)
SC, EU, EB, RCS = 5, 8, 9, 7
seed = [100]


def refill():
    seed[0] += 2
    s.fillUniform(X, seed[0])
    s.fillUniform(DL, seed[0] + 1)


ops = [
    ("fillUniform X + dAct (new batch)", refill),
    ("fwd gemm (W replica)", lambda: s.gemmAsync(X, W, Z)),
    ("biasAdd", lambda: s.opIssue(EB, [Z.id, Bv.id, Z.id], flags=(5,))),
    ("relu", lambda: s.opIssue(EU, [Z.id, ACT.id], flags=(0,))),
    ("reluGrad", lambda: s.opIssue(EB, [Z.id, DL.id, DL.id], flags=(3,))),
    ("dW gemm (gathers X^T, delta band)", lambda: s.gemmAsync(X, DL, dW, 1.0, 0.0, True, False)),
    ("setConst x2", lambda: (s.opIssue(SC, [ROW.id], 0.0), s.opIssue(SC, [dB.id], 0.0))),
    ("addRowColSum", lambda: s.opIssue(RCS, [DL.id, ROW.id, dB.id], 1.0, flags=(1,))),
    ("dX gemm (W replica)", lambda: s.gemmAsync(DL, W, dX, 1.0, 0.0, False, True)),
    ("axpy W", lambda: s.opIssue(EB, [dW.id, W.id, W.id], -1e-3, flags=(2,))),
    ("axpy b", lambda: s.opIssue(EB, [dB.id, Bv.id, Bv.id], -1e-3, flags=(2,))),
    ("replicate W + b", lambda: (s.replicateAsync(W), s.replicateAsync(Bv))),
]


def timed(fn):
    s.synchronize()
    dist.barrier()
    s.timerStart()
    fn()
    ms = s.timerStop()
    t = torch.tensor([ms], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.item()


for _ in range(3):
    for _, fn in ops:
        fn()
s.synchronize()
res = {name: 0.0 for name, _ in ops}
for _ in range(5):
    for name, fn in ops:
        res[name] += timed(fn) / 5
st = s.queryWorkerStats()[0]
if rank == 0:
    tot = sum(res.values())
    for name, ms in res.items():
        print(f"{name:38s} {ms * 1e3:8.1f} us")
    print(f"{'sum (serialised)':38s} {tot * 1e3:8.1f} us")
# whole step, back to back
def step():
    for _, fn in ops:
        fn()
ms = timed(lambda: [step() for _ in range(10)]) / 10
import time
s.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    step()
host = (time.perf_counter() - t0) / 10
s.synchronize()
if rank == 0:
    print(f"{'host issue per step':38s} {host * 1e6:8.1f} us")
    print(f"{'step (async, back to back)':38s} {ms * 1e3:8.1f} us   cache hits/misses {st['cache_hits']}/{st['cache_misses']}")
s.close()
dist.destroy_process_group()
