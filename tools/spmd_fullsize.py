# SPDX-License-Identifier: Apache-2.0
"""The headline workload across ranks (torchrun, one process per worker; with
more ranks than GPUs they share GPUs through the gloo control channel):
bf16 32768^3 (or --n) on the bench's 2D grid (1x2, 2x2, 2x4 for 2/4/8 ranks),
then a dependent second GEMM C2 = a C B (its A panels are the first GEMM's
output, so the in-GEMM panel pipelining carries it). Every rank compares its
own C and C2 tiles bitwise with the same two GEMMs on one GPU (single tile).

    torchrun --nproc-per-node 8 tools/spmd_fullsize.py [n]"""
import math
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)
from paper_1611_07819_b200 import gridmath as G  # noqa: E402

rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
SHARED = world > torch.cuda.device_count()
local = local % torch.cuda.device_count()
torch.cuda.set_device(local)
if SHARED:
    dist.init_process_group("gloo")
else:
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
pr, pc = {1: (1, 1), 2: (1, 2), 4: (2, 2), 8: (2, 4)}[world]
alpha = 1.0 / (math.sqrt(1.0 / 3.0) * math.sqrt(n))

obj = [G.nccl_unique_id() if rank == 0 else None]
dist.broadcast_object_list(obj, src=0)
g = G.makeWorkerGroup(world)
lay = G.makeGridLayout(n, n, pr, pc, g)
mine = [e for e, w in lay.tiles if int(w) == rank]  # local tiles in layout order (packed I/O order)
with G.Session(workers=world, spmd_rank=rank, devices=[local], nccl_id=obj[0], panel_cache_bytes=1,
               control="gloo" if SHARED else None) as s:
    A, B, C, C2 = (s.createMatrix(n, n, G.Precision.BF16, lay) for _ in range(4))
    s.fillUniform(A, 1)
    s.fillUniform(B, 2)
    G.gemm(s, A, B, C, 1.0, 0.0)
    G.gemm(s, C, B, C2, alpha, 0.0)
    got = []
    for M in (C, C2):
        buf = np.empty(s.localBytes(M), np.uint8)
        s.getLocalPacked(M, buf.ctypes.data, buf.nbytes)
        got.append(buf)
    plane = s.transport()
one = G.makeSingleTileLayout(n, n, 0)
with G.Session(workers=1, devices=[local]) as s1:
    A1, B1, C1, D1 = (s1.createMatrix(n, n, G.Precision.BF16, one) for _ in range(4))
    s1.fillUniform(A1, 1)
    s1.fillUniform(B1, 2)
    G.gemm(s1, A1, B1, C1, 1.0, 0.0)
    G.gemm(s1, C1, B1, D1, alpha, 0.0)
    want = []
    for M in (C1, D1):
        full = s1.getDataRaw(M).view(np.uint16).reshape(n, n)
        want.append(np.concatenate([full[e.rowStart:e.rowStart + e.rowCount,
                                         e.colStart:e.colStart + e.colCount].ravel() for e in mine]))
ok = all(np.array_equal(g_.view(np.uint16), w_) for g_, w_ in zip(got, want))
vals = (want[1].astype(np.uint32) << 16).view(np.float32)
ok = ok and bool(np.isfinite(vals).all()) and float(np.abs(vals).max()) > 0
t = torch.tensor([1 if ok else 0], device="cpu" if SHARED else "cuda")
dist.all_reduce(t, op=dist.ReduceOp.MIN)
if rank == 0:
    print(f"SPMD_FULLSIZE n={n} world={world} grid={pr}x{pc} plane={plane} control={'gloo' if SHARED else 'nccl'} "
          f"C and dependent C2 bitwise == 1 GPU on every rank: {t.item() == 1}", flush=True)
    print("SPMD_FULLSIZE " + ("PASS" if t.item() == 1 else "FAIL"), flush=True)
dist.destroy_process_group()
sys.exit(0 if t.item() == 1 else 1)
