# SPDX-License-Identifier: Apache-2.0
"""Runs a fixed set of multi-worker GEMMs (one process, workers on one GPU)
and saves every result to an .npz; tests run it under different
GM_DEBUG_CONFIG settings (in-GEMM panel pipelining on / off, a tiny ready
flag ring) and require the results to be bitwise identical.

    python tools/pipeline_check.py OUT.npz [chain_steps]
"""
import os
import sys

import numpy as np

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)
from paper_1611_07819_b200 import gridmath as G  # noqa: E402


def cases(s, out):
    P = s.workers
    g = G.makeWorkerGroup(P)
    specs = [
        # name, m, n, k, prec, layout kind, transA, transB
        ("grid_bf16", 1536, 1280, 4608, G.Precision.BF16, "grid", False, False),
        ("grid_bf16_ragged", 1000, 1100, 3000, G.Precision.BF16, "grid", False, False),
        ("rowcol_f16_tA", 768, 640, 2304, G.Precision.Half, "rowcol", True, False),
        ("grid_bf16_tB", 1024, 768, 2048, G.Precision.BF16, "grid", False, True),
        ("grid_bf16_tAtB", 512, 1024, 1536, G.Precision.BF16, "grid", True, True),
    ]
    for name, m, n, k, prec, kind, ta, tb in specs:
        ar, ac = (k, m) if ta else (m, k)
        br, bc = (n, k) if tb else (k, n)
        if kind == "grid":
            la = G.makeGridLayout(ar, ac, 2, P // 2, g)
            lb = G.makeGridLayout(br, bc, 2, P // 2, g)
            lc = G.makeGridLayout(m, n, 2, P // 2, g)
        else:
            la, lb, lc = G.makeRowBlockLayout(ar, ac, g), G.makeColBlockLayout(br, bc, g), G.makeColBlockLayout(m, n, g)
        A = s.createMatrix(ar, ac, prec, la)
        B = s.createMatrix(br, bc, prec, lb)
        C = s.createMatrix(m, n, G.Precision.Single, lc)
        s.fillUniform(A, 7)
        s.fillUniform(B, 8)
        G.gemm(s, A, B, C, 1.0, 0.0, ta, tb)
        out[name] = s.getDataRaw(C)
        for M in (A, B, C):
            s.destroy(M)


def chain(s, steps, out):
    """X_{i+1} = a X_i B (bf16, 2x2 grid, all async): every op's A panels
    are the previous op's output (RAW across ops and ranks), and every op
    overwrites the matrix the op before it read (WAR). a = 0.5 / (sigma_B
    sqrt(n)) keeps the values bounded (the chain converges to B's top
    singular direction without overflow)."""
    P = s.workers
    n = 1024
    lay = G.makeGridLayout(n, n, 2, P // 2, G.makeWorkerGroup(P)) if P > 1 else G.makeSingleTileLayout(n, n, 0)
    X = [s.createMatrix(n, n, G.Precision.BF16, lay) for _ in range(2)]
    B = s.createMatrix(n, n, G.Precision.BF16, lay)
    s.fillUniform(X[0], 3)
    s.fillUniform(B, 4)
    alpha = 0.5 / ((1.0 / 3.0) ** 0.5 * n ** 0.5)
    for i in range(steps):
        s.gemmAsync(X[i % 2], B, X[(i + 1) % 2], alpha, 0.0)
    out["chain"] = s.getDataRaw(X[steps % 2])


def replica_forward(s, out):
    """The FC forward behind W's re-replication: W column-block, every step
    mutates W, replicates it asynchronously and immediately multiplies by
    it, so the GEMM reads a replica whose pieces are still landing (it polls
    the per-piece flags when pipelining is on)."""
    P = s.workers
    g = G.makeWorkerGroup(P)
    batch, fi, fo = 512, 768, 1024
    X = s.createMatrix(batch, fi, G.Precision.BF16, G.makeRowBlockLayout(batch, fi, g))
    W = s.createMatrix(fi, fo, G.Precision.BF16, G.makeColBlockLayout(fi, fo, g))
    Z = s.createMatrix(batch, fo, G.Precision.Single, G.makeRowBlockLayout(batch, fo, g))
    s.fillUniform(X, 5)
    s.fillUniform(W, 6, -0.05, 0.05)
    zs = []
    for i in range(4):
        G.mulScalar(s, W, 1.25)
        s.replicateAsync(W)
        s.gemmAsync(X, W, Z)
        zs.append(s.getDataRaw(Z))
    out["replica_fwd"] = np.stack(zs)


def main():
    path = sys.argv[1]
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    out = {}
    with G.Session(workers=4, devices=[0], panel_cache_bytes=1) as s:
        cases(s, out)
        chain(s, steps, out)
        replica_forward(s, out)
    ref = {}
    with G.Session(workers=1, devices=[0]) as s1:  # single worker: no exchange at all
        chain(s1, steps, ref)
    out["chain_1worker"] = ref["chain"]
    np.savez(path, **out)
    print("PIPELINE_CHECK wrote", path, sorted(out))


if __name__ == "__main__":
    main()
