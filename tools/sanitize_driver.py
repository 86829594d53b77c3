# SPDX-License-Identifier: Apache-2.0
"""Small run of every kernel family, for compute-sanitizer:

    compute-sanitizer --tool memcheck  python tools/sanitize_driver.py
    compute-sanitizer --tool racecheck python tools/sanitize_driver.py
    compute-sanitizer --tool synccheck python tools/sanitize_driver.py

tcgen05 GEMM (bf16 wide / narrow tiles, fp16, transposes, the in-GEMM
panel-flag path, 3xTF32 fold, 1xTF32), DMMA fp64, the generator, convert /
reshape, elementwise ops, setConst, the line sums (TMA and cp.async
paths), replication and the fused bias/relu replay epilogue. Results are
checked against the CPU oracle so a sanitizer run is also a parity run."""
import os
import sys

import numpy as np

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
os.environ.setdefault("GM_DEBUG_CONFIG", "panel_min_gflop=0")
import oracle as O  # noqa: E402  (checker only)
from paper_1611_07819_b200 import gridmath as G  # noqa: E402


def check(name, got, want, tol):
    err = O.rel_fro(got, want)
    print(f"{name:40s} rel_fro {err:.2e}", flush=True)
    assert err <= tol, name


def main():
    P = 4
    g = G.makeWorkerGroup(P)
    with G.Session(workers=P, devices=[0], panel_cache_bytes=1) as s:
        for (m, n, k, prec, ta, tb) in [(512, 1024, 4096, G.Precision.BF16, False, False),
                                        (384, 256, 640, G.Precision.BF16, True, False),
                                        (256, 384, 512, G.Precision.Half, False, True),
                                        (320, 288, 352, G.Precision.Single, False, False),
                                        (192, 160, 224, G.Precision.Double, True, True)]:
            ar, ac = (k, m) if ta else (m, k)
            br, bc = (n, k) if tb else (k, n)
            A = s.createMatrix(ar, ac, prec, G.makeGridLayout(ar, ac, 2, 2, g))
            B = s.createMatrix(br, bc, prec, G.makeGridLayout(br, bc, 2, 2, g))
            cprec = G.Precision.Double if prec == G.Precision.Double else G.Precision.Single
            C = s.createMatrix(m, n, cprec, G.makeGridLayout(m, n, 2, 2, g))
            s.fillUniform(A, 1)
            s.fillUniform(B, 2)
            G.gemm(s, A, B, C, 1.0, 0.0, ta, tb)
            a, b, c = s.getDataRaw(A), s.getDataRaw(B), s.getDataRaw(C)
            want = O.gemm_c(m, n, k, a, int(prec), b, int(prec), np.zeros((m, n), c.dtype), int(cprec), 1.0, 0.0,
                            int(ta), int(tb))
            check(f"gemm {prec.name} {m}x{n}x{k} tA={ta} tB={tb}", c, want,
                  1e-12 if prec == G.Precision.Double else 1e-5)
            for M in (A, B, C):
                s.destroy(M)
        # FC layer: replication, fused epilogue through replay, neighbours, line sums
        batch, fi, fo = 256, 384, 192
        X = s.createMatrix(batch, fi, G.Precision.BF16, G.makeRowBlockLayout(batch, fi, g))
        W = s.createMatrix(fi, fo, G.Precision.BF16, G.makeColBlockLayout(fi, fo, g))
        Bv = s.createMatrix(1, fo, G.Precision.BF16, G.makeColBlockLayout(1, fo, g))
        Z = s.createMatrix(batch, fo, G.Precision.BF16, G.makeRowBlockLayout(batch, fo, g))
        ACT = s.createMatrix(batch, fo, G.Precision.BF16, G.makeRowBlockLayout(batch, fo, g))
        R = s.createMatrix(batch, 1, G.Precision.Single, G.makeRowBlockLayout(batch, 1, g))
        CS = s.createMatrix(1, fo, G.Precision.Single, G.makeColBlockLayout(1, fo, g))
        s.fillUniform(X, 3)
        s.fillUniform(W, 4, -0.05, 0.05)
        s.fillUniform(Bv, 5, -0.1, 0.1)
        s.replicateSync(W)
        s.replicateSync(Bv)
        pid = s.beginRecord()
        G.gemm(s, X, W, Z, 1.0, 0.0)
        G.biasAdd(s, Z, Bv)
        G.relu(s, Z, ACT)
        G.setConst(s, R, 0.0)
        G.setConst(s, CS, 0.0)
        G.addRowColSum(s, ACT, R, CS, 1.0, True)
        s.endRecord()
        s.replay(pid)
        act = s.getDataRaw(ACT).view(np.uint16)
        actf = (act.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
        check("addRowColSum rows (TMA path)", s.getDataRaw(R).ravel(), actf.sum(axis=1), 1e-5)
        check("addRowColSum cols (TMA path)", s.getDataRaw(CS).ravel(), actf.sum(axis=0), 1e-5)
        # reshape + convert
        s.reshape(Z, G.makeColBlockLayout(batch, fo, g), G.Precision.Single)
        z = s.getDataRaw(Z)
        assert np.isfinite(z).all()
        print("sanitize driver: all kernel families ran", flush=True)


if __name__ == "__main__":
    main()
