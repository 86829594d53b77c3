"""SPMD (one process per GPU) correctness check, launched by torchrun:
    torchrun --nproc-per-node N tools/spmd_check.py
Runs distributed GEMMs through both SPMD data planes -- copy-engine pulls
over CUDA IPC (the default) and NCCL point-to-point (transport=1) -- on
several layouts and compares the gathered C with the single-process result
of the same library (bitwise: deterministic mode is layout/P invariant) and
with the CPU oracle on sampled rows. Also exercises replication, reshape,
and an async GEMM chain whose ops read what the previous op just wrote and
overwrite what it just read (cross-rank RAW/WAR ordering)."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
from paper_1611_07819_b200 import gridmath as G  # noqa: E402
import oracle as O  # noqa: E402

rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
# More ranks than GPUs (e.g. the 2x4 grid's 8 ranks on a 4-GPU box, or 2
# ranks on a 1-GPU box): ranks share devices round-robin. NCCL refuses two
# ranks on one GPU, so the sessions then take the gloo control channel
# (Session(control="gloo")) and the IPC copy-engine data plane only (the
# IPC plane maps same-device peers too); the script's own collectives run
# on the gloo group with CPU tensors.
SHARED = world > torch.cuda.device_count()
local = local % torch.cuda.device_count()
torch.cuda.set_device(local)
if SHARED:
    dist.init_process_group("gloo")
else:
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
CONTROL = "gloo" if SHARED else None
TDEV = "cpu" if SHARED else "cuda"
pr, pc = {1: (1, 1), 2: (1, 2), 4: (2, 2), 8: (2, 4)}[world]
g = G.makeWorkerGroup(world)


def say(msg):
    if rank == 0:
        print(msg, flush=True)


def one_gpu_gemm(m, n, k, prec, pc_out, a, b):
    with G.Session(workers=1, devices=[local]) as s1:
        one = G.makeSingleTileLayout
        A1 = s1.createMatrix(m, k, prec, one(m, k, 0))
        B1 = s1.createMatrix(k, n, prec, one(k, n, 0))
        C1 = s1.createMatrix(m, n, pc_out, one(m, n, 0))
        s1.setDataRaw(A1, a)
        s1.setDataRaw(B1, b)
        G.gemm(s1, A1, B1, C1, 1.0, 0.0)
        return s1.getDataRaw(C1)


def chain(s, lay, n, steps):
    """C = A B / 32; A = C B / 32; B <- fresh values; all async, no syncs.
    Every op reads what the previous op wrote (RAW) and overwrites what the
    previous op read (WAR)."""
    A = s.createMatrix(n, n, G.Precision.BF16, lay)
    B = s.createMatrix(n, n, G.Precision.BF16, lay)
    C = s.createMatrix(n, n, G.Precision.BF16, lay)
    s.fillUniform(A, 11)
    s.fillUniform(B, 12)
    for i in range(steps):
        s.gemmAsync(A, B, C, 1.0 / 32, 0.0)
        s.gemmAsync(C, B, A, 1.0 / 32, 0.0)
        s.fillUniform(B, 100 + i)
    s.gemmAsync(A, B, C, 1.0 / 32, 0.0)
    return s.getDataRaw(C)


def run(transport, nccl_id):
    ok = True
    with G.Session(workers=world, spmd_rank=rank, devices=[local], nccl_id=nccl_id, panel_cache_bytes=1,
                   transport=transport, control=CONTROL) as s:
        plane = s.transport()
        want_plane = "nccl" if transport == 1 else "ipc"
        if plane != want_plane:
            print(f"[rank{rank}] transport={transport}: plane {plane} != {want_plane}", flush=True)
            ok = False
        cases = [
            ("grid bf16", 2048, 1536, 3072, G.Precision.BF16, lambda r, c: G.makeGridLayout(r, c, pr, pc, g)),
            ("rowcol f32", 768, 640, 1024, G.Precision.Single, None),
            ("grid f64", 512, 384, 640, G.Precision.Double, lambda r, c: G.makeGridLayout(r, c, pr, pc, g)),
        ]
        for name, m, n, k, prec, lay in cases:
            if lay is None:
                la, lb, lc = G.makeRowBlockLayout(m, k, g), G.makeColBlockLayout(k, n, g), G.makeColBlockLayout(m, n, g)
            else:
                la, lb, lc = lay(m, k), lay(k, n), lay(m, n)
            pc_out = G.Precision.Single if prec == G.Precision.BF16 else prec
            A = s.createMatrix(m, k, prec, la)
            B = s.createMatrix(k, n, prec, lb)
            C = s.createMatrix(m, n, pc_out, lc)
            s.fillUniform(A, 1)
            s.fillUniform(B, 2)
            G.gemm(s, A, B, C, 1.0, 0.0)
            c = s.getDataRaw(C)
            a = s.getDataRaw(A)
            b = s.getDataRaw(B)
            rows = (m // 3, m // 3 + 16)
            want = O.gemm_c(m, n, k, a, int(prec), b, int(prec), np.zeros((m, n), c.dtype), int(pc_out), 1.0, 0.0,
                            0, 0, rows)
            err = O.rel_fro(c[rows[0]:rows[1]], want[rows[0]:rows[1]])
            tol = 1e-12 if prec == G.Precision.Double else 1e-5
            good = err <= tol
            if rank == 0:
                bit = np.array_equal(c.view(np.uint8), one_gpu_gemm(m, n, k, prec, pc_out, a, b).view(np.uint8))
                say(f"[rank0 {plane}] {name} world={world} rel_fro={err:.3e} bitwise_vs_1gpu={bit}")
                good = good and bit
            ok = ok and good
        # replication + gemm via replica, and the panel cache path
        X = s.createMatrix(512, 768, G.Precision.BF16, G.makeRowBlockLayout(512, 768, g))
        W = s.createMatrix(768, 640, G.Precision.BF16, G.makeColBlockLayout(768, 640, g))
        Z = s.createMatrix(512, 640, G.Precision.Single, G.makeRowBlockLayout(512, 640, g))
        s.fillUniform(X, 5)
        s.fillUniform(W, 6)
        st0 = s.queryWorkerStats()[0]
        h = s.replicateAsync(W)
        ok = ok and s.wait(h) == G.ReplState.Done
        st1 = s.queryWorkerStats()[0]
        G.gemm(s, X, W, Z, 1.0, 0.0)
        st2 = s.queryWorkerStats()[0]
        z = s.getDataRaw(Z)
        x = s.getDataRaw(X)
        w = s.getDataRaw(W)
        want = O.gemm_c(512, 640, 768, x, 3, w, 3, np.zeros((512, 640), np.float32), 1, 1.0, 0.0, 0, 0)
        e = O.rel_fro(z, want)
        recv_repl = st1["bytes_received"] - st0["bytes_received"]
        expect = 768 * 640 * 2 - 768 * (640 // world) * 2 if 640 % world == 0 else None
        good = e <= 1e-5 and st2["bytes_received"] == st1["bytes_received"] and (expect is None or recv_repl == expect)
        say(f"[rank0 {plane}] replication: rel_fro={e:.3e} repl_bytes={recv_repl} expect={expect} "
            f"gemm_bytes={st2['bytes_received'] - st1['bytes_received']}")
        ok = ok and good
        # reshape across ranks: grid -> row-block, Single -> BF16, then back
        R = s.createMatrix(1000, 776, G.Precision.Single, G.makeGridLayout(1000, 776, pr, pc, g))
        s.fillUniform(R, 9)
        r0 = s.getDataRaw(R)
        s.reshape(R, G.makeRowBlockLayout(1000, 776, g), G.Precision.BF16)
        r1 = s.getDataRaw(R)
        u = r0.view(np.uint32).astype(np.uint64)
        want = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
        s.reshape(R, G.makeColBlockLayout(1000, 776, g), G.Precision.Single)
        r2 = s.getDataRaw(R)
        good = np.array_equal(r1.view(np.uint16), want) and np.array_equal(
            r2, (want.astype(np.uint32) << 16).view(np.float32))
        say(f"[rank0 {plane}] reshape grid->row/bf16->col/f32 ok={good}")
        ok = ok and good
        # async RAW/WAR chain vs the same chain on one GPU
        n = 1536
        got = chain(s, G.makeGridLayout(n, n, pr, pc, g), n, 3)
        if rank == 0:
            with G.Session(workers=1, devices=[local]) as s1:
                ref = chain(s1, G.makeSingleTileLayout(n, n, 0), n, 3)
            vals = (got.view(np.uint16).astype(np.uint32) << 16).view(np.float32)
            good = np.array_equal(got.view(np.uint8), ref.view(np.uint8)) and np.isfinite(vals).all() and \
                np.abs(vals).max() > 0
            say(f"[rank0 {plane}] async RAW/WAR chain bitwise_vs_1gpu={good} max|C|={np.abs(vals).max():.3g}")
            ok = ok and good
        # FC train step (reference Trainer order) recorded once and replayed,
        # vs the same pipeline on one process with `world` workers on one GPU
        # (bf16: the replay runs gemm -> biasAdd -> relu as one fused GEMM on every rank)
        for fprec in (G.Precision.Single, G.Precision.BF16):
            g0 = s.graphStats()["launches"]
            fc = fc_steps(s, 4, fprec)
            graphs = s.graphStats()["launches"] - g0  # replays run as CUDA graphs (GM_DEBUG_CONFIG graph_replay=1)
            if rank == 0:
                with G.Session(workers=world, devices=[local]) as s1:
                    s1.setGraphReplay(False)
                    ref = fc_steps(s1, 4, fprec)
                good = all(np.array_equal(fc[k].view(np.uint8), ref[k].view(np.uint8)) for k in fc)
                say(f"[rank0 {plane}] FC step {fprec.name} record/replay (gemm, biasAdd, relu, reluGrad, rowcolsum, "
                    f"axpy, replication) graph_launches={graphs} bitwise_vs_1process={good}")
                ok = ok and good
        # chunked async host streaming: upload A/B, gemm, download C
        n = 1024
        lay = G.makeGridLayout(n, n, pr, pc, g)
        A = s.createMatrix(n, n, G.Precision.BF16, lay)
        B = s.createMatrix(n, n, G.Precision.BF16, lay)
        C = s.createMatrix(n, n, G.Precision.BF16, lay)
        s.fillUniform(A, 21)
        s.fillUniform(B, 22)
        G.gemm(s, A, B, C, 1.0, 0.0)
        want_c = np.zeros(s.localBytes(C), np.uint8)
        s.getLocalPacked(C, want_c.ctypes.data, want_c.nbytes)
        ha = np.zeros(s.localBytes(A), np.uint8)
        hb = np.zeros(s.localBytes(B), np.uint8)
        s.getLocalPacked(A, ha.ctypes.data, ha.nbytes)
        s.getLocalPacked(B, hb.ctypes.data, hb.nbytes)
        s.fillUniform(A, 23)
        s.fillUniform(B, 24)  # overwritten again by the uploads below
        hc = np.zeros_like(want_c)
        for _ in range(2):
            s.setLocalPackedAsync(B, hb.ctypes.data, hb.nbytes, 64 * 1024)
            s.setLocalPackedAsync(A, ha.ctypes.data, ha.nbytes, 64 * 1024)
            s.gemmAsync(A, B, C)
            s.getLocalPackedAsync(C, hc.ctypes.data, hc.nbytes)
        s.synchronize()
        good = bool(np.array_equal(hc, want_c))
        t = torch.tensor([1 if good else 0], device=TDEV)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        good = t.item() == 1
        say(f"[rank0 {plane}] async chunked upload/gemm/download == sync path on every rank: {good}")
        ok = ok and good
        # checkpoint (rank 0 writes the DMCK file) and collective restore
        path = f"/tmp/spmd_ckpt_{os.getpid() if rank == 0 else 0}.dmck"
        obj = [path]
        dist.broadcast_object_list(obj, src=0)
        path = obj[0]
        before = s.getDataRaw(C)
        s.checkpoint(path)
        dist.barrier()
    with G.Session.restore(path, workers=world, spmd_rank=rank, devices=[local], nccl_id=_fresh_id(),
                           transport=transport, control=CONTROL) as s2:
        after = s2.getDataRaw(s2.matrix(C.id))
        good = bool(np.array_equal(after, before))
        say(f"[rank0 {plane}] checkpoint/restore across ranks ok={good}")
        ok = ok and good
    dist.barrier()
    if rank == 0:
        os.remove(path)
    return ok


def _fresh_id():
    obj = [G.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


def fc_steps(s, steps, S=G.Precision.Single):
    batch, fin, fout = 256, 384, 192
    M = dict(X=(batch, fin, G.makeRowBlockLayout), W=(fin, fout, G.makeColBlockLayout),
             B=(1, fout, G.makeColBlockLayout), Z=(batch, fout, G.makeRowBlockLayout),
             A=(batch, fout, G.makeRowBlockLayout), D=(batch, fout, G.makeRowBlockLayout),
             DW=(fin, fout, G.makeColBlockLayout), DB=(1, fout, G.makeColBlockLayout),
             R=(batch, 1, G.makeRowBlockLayout), DX=(batch, fin, G.makeRowBlockLayout))
    m = {k: s.createMatrix(r, c, S, lay(r, c, g)) for k, (r, c, lay) in M.items()}
    s.fillUniform(m["X"], 1)
    s.fillUniform(m["W"], 2, -0.05, 0.05)
    s.fillUniform(m["B"], 3, -0.1, 0.1)
    s.replicateSync(m["W"])
    s.replicateSync(m["B"])
    for i in range(steps):
        s.fillUniform(m["D"], 40 + i)
        if i == 0:
            pid = s.beginRecord()
        if i == 0:
            G.gemm(s, m["X"], m["W"], m["Z"], 1.0, 0.0)
            G.biasAdd(s, m["Z"], m["B"])
            G.relu(s, m["Z"], m["A"])
            G.reluGrad(s, m["Z"], m["D"])
            G.gemm(s, m["X"], m["D"], m["DW"], 1.0, 0.0, True, False)
            G.setConst(s, m["R"], 0.0)
            G.setConst(s, m["DB"], 0.0)
            G.addRowColSum(s, m["D"], m["R"], m["DB"], 1.0, True)
            G.gemm(s, m["D"], m["W"], m["DX"], 1.0, 0.0, False, True)
            G.axpy(s, -0.01, m["DW"], m["W"])
            G.axpy(s, -0.01, m["DB"], m["B"])
            s.replicateAsync(m["W"])
            s.replicateAsync(m["B"])
            s.endRecord()
        else:
            s.replay(pid)
    return {k: s.getDataRaw(m[k]) for k in ("W", "B", "DX", "DB", "A")}


ok = True
for transport in ((0,) if SHARED else (0, 1)):
    obj = [G.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    ok = run(transport, obj[0]) and ok
say(f"SPMD_CHECK world={world} gpus={torch.cuda.device_count()} control={'gloo' if SHARED else 'nccl'}")
t = torch.tensor([1 if ok else 0], device=TDEV)
dist.all_reduce(t, op=dist.ReduceOp.MIN)
say("SPMD_CHECK " + ("PASS" if t.item() == 1 else "FAIL"))
dist.destroy_process_group()
sys.exit(0 if t.item() == 1 else 1)
