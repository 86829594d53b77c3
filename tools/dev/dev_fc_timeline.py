# SPDX-License-Identifier: Apache-2.0
"""Per-op device timeline of the replayed FC train step (bench --config fc)
under torchrun: every rank prints, for the last of several back-to-back
replays, the time (us from the replay's start) at which its compute and comm
streams passed the end of each op. Shows which op the step waits on."""
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
pid = s.beginRecord()
s.gemmAsync(X, W, Z)
s.opIssue(EB, [Z.id, Bv.id, Z.id], flags=(5,))
s.opIssue(EU, [Z.id, ACT.id], flags=(0,))
s.opIssue(EB, [Z.id, DL.id, DL.id], flags=(3,))
s.gemmAsync(X, DL, dW, 1.0, 0.0, True, False)
s.opIssue(SC, [ROW.id], 0.0)
s.opIssue(SC, [dB.id], 0.0)
s.opIssue(RCS, [DL.id, ROW.id, dB.id], 1.0, flags=(1,))
s.gemmAsync(DL, W, dX, 1.0, 0.0, False, True)
s.opIssue(EB, [dW.id, W.id, W.id], -1e-3, flags=(2,))
s.opIssue(EB, [dB.id, Bv.id, Bv.id], -1e-3, flags=(2,))
s.replicateAsync(W)
s.replicateAsync(Bv)
s.endRecord()
for i in range(5):
    s.fillUniform(X, 100 + i)
    s.fillUniform(DL, 200 + i)
    s.replay(pid, sync=False)
s.synchronize()
s.setOpTimeline(True)
for i in range(6):
    s.fillUniform(X, 300 + i)
    s.fillUniform(DL, 400 + i)
    s.replay(pid, sync=False)
s.synchronize()
tl = s.opTimeline()
lines = [f"rank {rank}: " + "  ".join(f"{lab}={c * 1e3:.0f}/{m * 1e3:.0f}" for lab, c, m in tl)]
out = [None] * world
dist.all_gather_object(out, lines)
if rank == 0:
    print("per op: compute/comm stream passed its end, us from the replay start (last of 6 back-to-back replays)")
    for l in out:
        print(l[0])
s.close()
dist.destroy_process_group()
