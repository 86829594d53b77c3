# SPDX-License-Identifier: Apache-2.0
"""GPU parity of the FC-layer neighbours of the GEMM:
setConst, relu / mulScalar / add / sub / axpy / reluGrad / copy / biasAdd and
addRowColSum, through the C ABI, against

  * the golden outputs of the UNMODIFIED reference (tests/golden/fc_*.npz,
    oracle/make_golden.py) -- bit-for-bit, except outputs that depend on a
    subnormal Half input (the reference widens those to half their IEEE
    value; the device is IEEE) and fast-mode sums
    (arrival-order partials in the reference);
  * the C restatement (oracle/gemm_oracle.c) on identical inputs for BF16
    storage (not a reference type) and for larger, multi-tile layouts;
  * a composed FC-layer train step (gemm + biasAdd + relu + reluGrad + gemm +
    setConst + addRowColSum + gemm + axpy), reference Trainer order
    (dnn.cpp:140-190).
"""
import numpy as np
import pytest

import oracle as O
from conftest import load_case
from paper_1611_07819_b200 import gridmath as G

pytestmark = pytest.mark.gpu


def layout_of(tiles):
    return G.Layout([(G.TileExtent(*map(int, t[:4])), int(t[4])) for t in tiles])


def half_subnormal(img, prec):
    if prec != 0:
        return np.zeros(img.shape, dtype=bool)
    u = img.view(np.uint16)
    return ((u & 0x7C00) == 0) & ((u & 0x03FF) != 0)


def _uint_view(a):
    a = np.ascontiguousarray(a).reshape(-1)
    return a.view({2: np.uint16, 4: np.uint32, 8: np.uint64}[a.dtype.itemsize])


def same_bits(got, want, prec, mask=None):
    """Bitwise equality of two storage images of precision `prec` (any NaN
    equals any NaN: x86 keeps NaN payloads, the GPU returns the canonical
    NaN), outside `mask`."""
    g, w = _uint_view(got), _uint_view(want)
    if g.shape != w.shape:
        return False
    keep = np.ones(g.shape, dtype=bool) if mask is None else ~np.asarray(mask).reshape(-1)
    stor = {0: np.uint16, 1: np.float32, 2: np.float64, 3: np.uint16}[prec]
    keep &= ~(np.isnan(O.to_f64(g.view(stor), prec)) & np.isnan(O.to_f64(w.view(stor), prec)))
    return np.array_equal(g[keep], w[keep])


def out_precs(c):
    op, sub = c["op"], c["sub"]
    if op == 0:
        return (c["dp"] if sub == 0 else c["xp"]), None
    if op == 1:
        return {2: c["yp"], 3: c["yp"], 5: c["xp"]}.get(sub, c["dp"]), None
    if op == 2:
        return c["yp"], c["dp"]
    return c["xp"], None


def run_fc(c, d, det=True):
    """The reference harness's dispatch (oracle/ref_harness.cpp gmref_fcop) on the device path."""
    with G.Session(workers=c["p"], deterministic=det) as s:
        def mk(img, prec, tiles):
            m = s.createMatrix(img.shape[0], img.shape[1], G.Precision(prec), layout_of(tiles))
            s.setDataRaw(m, np.ascontiguousarray(img))
            return m

        X = mk(d["x"], c["xp"], d["xt"])
        Y = mk(d["y"], c["yp"], d["yt"]) if "y" in d else None
        D = mk(d["d"], c["dp"], d["dt"]) if "d" in d else None
        if c["repl"] & 1:
            s.replicateSync(X)
        if c["repl"] & 2 and Y is not None:
            s.replicateSync(Y)
        op, sub, alpha = c["op"], c["sub"], c["alpha"]
        out, out2 = X, None
        if op == 0:
            if sub == 0:
                G.relu(s, X, D)
                out = D
            else:
                G.mulScalar(s, X, alpha)
        elif op == 1:
            if sub == 0:
                G.addMatrices(s, X, Y, D); out = D
            elif sub == 1:
                G.subMatrices(s, X, Y, D); out = D
            elif sub == 2:
                G.axpy(s, alpha, X, Y); out = Y
            elif sub == 3:
                G.reluGrad(s, X, Y); out = Y
            elif sub == 4:
                G.copyMatrix(s, X, D); out = D
            else:
                G.biasAdd(s, X, Y); out = X
        elif op == 2:
            G.addRowColSum(s, X, Y, D, alpha, sub != 0)
            out, out2 = Y, D
        else:
            G.setConst(s, X, alpha)
        s.verifyMetadataConsistency()
        r0 = s.getDataRaw(out)
        r1 = s.getDataRaw(out2) if out2 is not None else None
        return r0, r1


def fc_masks(c, d):
    """Outputs that depend on a subnormal Half input."""
    op, sub = c["op"], c["sub"]
    xs = half_subnormal(d["x"], c["xp"])
    ys = half_subnormal(d["y"], c["yp"]) if "y" in d else None
    ds = half_subnormal(d["d"], c["dp"]) if "d" in d else None
    if op == 0:
        return xs, None
    if op == 1:
        if sub == 5:
            return xs | ys.reshape(1, -1), None
        if sub == 4:
            return xs, None
        return xs | ys, None
    if op == 2:
        rows = xs.any(axis=1, keepdims=True) | ys
        cols = xs.any(axis=0, keepdims=True) | ds
        return rows, cols
    return None, None


def test_fc_golden_cases_match_reference(golden_index):
    failures = []
    masked = 0
    for c in golden_index["fc_cases"]:
        d = load_case("fc_" + c["name"])
        got0, got1 = run_fc(c, d)
        m0, m1 = fc_masks(c, d)
        masked += int(m0.sum()) if m0 is not None else 0
        want0 = d["out0"].reshape(got0.shape)
        if c["op"] == 2 and c["sub"] == 0:  # fast mode: per-tile partials folded in arrival order
            want1 = d["out1"].reshape(got1.shape)
            ok = all(np.allclose(O.to_f64(_uint_view(g).view(w.dtype), p), O.to_f64(w.reshape(-1), p),
                                 rtol=1e-5, atol=1e-5)
                     for g, w, p in ((got0, want0, c["yp"]), (got1, want1, c["dp"])))
        else:
            p0, p1 = out_precs(c)
            ok = same_bits(got0, want0, p0, m0)
            if got1 is not None:
                ok = ok and same_bits(got1, d["out1"].reshape(got1.shape), p1, m1)
        if not ok:
            failures.append(c["name"])
    assert not failures, failures
    assert len(golden_index["fc_cases"]) >= 20


def flush_half_subnormals(img, prec):
    if prec != 0:
        return img
    out = img.copy()
    out[half_subnormal(out, 0)] &= np.uint16(0x8000)
    return out


LAYOUTS = {
    "row": lambda r, c, p: O.row_block_tiles(r, c, p),
    "col": lambda r, c, p: O.col_block_tiles(r, c, p),
    "grid": lambda r, c, p: O.grid_tiles(r, c, {1: 1, 2: 1, 3: 1, 4: 2, 8: 2}[p], p // {1: 1, 2: 1, 3: 1, 4: 2, 8: 2}[p]),
}


@pytest.mark.parametrize("prec", [3, 0, 1, 2])
@pytest.mark.parametrize("kind", [("relu", True, 0), ("mul", True, 1), ("add", False, 0), ("sub", False, 1),
                                  ("axpy", False, 2), ("relugrad", False, 3), ("copy", False, 4),
                                  ("bias", False, 5)])
def test_elementwise_vs_c_restatement_multi_tile(prec, kind):
    """Larger images, mixed layouts (x grid, y row, dst col on 4 workers):
    device == C restatement bit-for-bit (Half inputs without subnormals)."""
    name, unary, k = kind
    rows, cols, p = 301, 515, 4
    x = flush_half_subnormals(O.fill_uniform(rows, cols, prec, 21).reshape(rows, cols), prec)
    y = flush_half_subnormals(O.fill_uniform(1 if k == 5 else rows, cols, prec, 22), prec)
    y = y.reshape(1 if k == 5 else rows, cols)
    dst = O.fill_uniform(rows, cols, prec, 23).reshape(rows, cols)
    alpha = -0.37
    with G.Session(workers=p) as s:
        X = s.createMatrix(rows, cols, G.Precision(prec), layout_of(LAYOUTS["grid"](rows, cols, p)))
        Y = s.createMatrix(y.shape[0], cols, G.Precision(prec), layout_of(LAYOUTS["row"](y.shape[0], cols, p)))
        D = s.createMatrix(rows, cols, G.Precision(prec), layout_of(LAYOUTS["col"](rows, cols, p)))
        for M, img in ((X, x), (Y, y), (D, dst)):
            s.setDataRaw(M, img)
        if unary:
            if k == 0:
                G.relu(s, X, D); out, want = D, O.ew_c(True, 0, 0.0, x, prec, None, 1, dst, prec)
            else:
                G.mulScalar(s, X, alpha); out, want = X, O.ew_c(True, 1, alpha, x, prec, None, 1, x, prec)
        elif k in (2, 3):
            (G.axpy(s, alpha, X, Y) if k == 2 else G.reluGrad(s, X, Y))
            out, want = Y, O.ew_c(False, k, alpha, x, prec, y, prec, y, prec)
        elif k == 5:
            G.biasAdd(s, X, Y)
            out, want = X, O.ew_c(False, 5, 0.0, x, prec, y, prec, x, prec)
        elif k == 4:
            G.copyMatrix(s, X, D)
            out, want = D, O.ew_c(False, 4, 0.0, x, prec, dst, prec, dst, prec)
        else:
            (G.addMatrices if k == 0 else G.subMatrices)(s, X, Y, D)
            out, want = D, O.ew_c(False, k, 0.0, x, prec, y, prec, dst, prec)
        got = s.getDataRaw(out).reshape(want.shape)
    assert same_bits(got, want, prec), (name, prec)


@pytest.mark.parametrize("prec", [3, 1, 2])
@pytest.mark.parametrize("lay", [("row", "row", "col"), ("grid", "col", "row"), ("col", "grid", "grid")])
def test_row_col_sums_vs_c_restatement(prec, lay):
    """Deterministic addRowColSum: every output is one ascending-index chain,
    bit-for-bit the reference's regardless of layout (kernels.cpp:572-617)."""
    rows, cols, p = 777, 1031, 4
    a = O.fill_uniform(rows, cols, prec, 31).reshape(rows, cols)
    r = O.fill_uniform(rows, 1, prec, 32).reshape(rows, 1)
    c = O.fill_uniform(1, cols, prec, 33).reshape(1, cols)
    alpha = 0.625
    want_r, want_c = O.rowcolsum_c(alpha, a, prec, r, prec, c, prec)
    for det in (True, False):
        with G.Session(workers=p, deterministic=det) as s:
            A = s.createMatrix(rows, cols, G.Precision(prec), layout_of(LAYOUTS[lay[0]](rows, cols, p)))
            R = s.createMatrix(rows, 1, G.Precision(prec), layout_of(LAYOUTS[lay[1]](rows, 1, p)))
            C = s.createMatrix(1, cols, G.Precision(prec), layout_of(LAYOUTS[lay[2]](1, cols, p)))
            for M, img in ((A, a), (R, r), (C, c)):
                s.setDataRaw(M, img)
            G.addRowColSum(s, A, R, C, alpha, det)
            got_r = s.getDataRaw(R).reshape(rows, 1)
            got_c = s.getDataRaw(C).reshape(1, cols)
        assert same_bits(got_r, want_r, prec) and same_bits(got_c, want_c, prec), (prec, lay, det)


@pytest.mark.parametrize("prec", [3, 1, 0])
@pytest.mark.parametrize("shape", [(600, 1000), (4096, 264), (33, 4104), (4096, 4096), (129, 4160)])
def test_row_col_sums_aligned_rows_vs_c_restatement(prec, shape):
    """16-byte aligned rows take the TMA-fed kernel for 16-bit storage
    (256-element stages, mixed-precision FHADD chain steps) and the cp.async
    ring for Single: chains that end mid-stage and output counts that are not
    multiples of 32, bit-for-bit. Half inputs stay clear of subnormals
    (the reference decodes those to half their IEEE value)."""
    rows, cols = shape
    lo = 0.125 if prec == 0 else -1.0
    a = O.fill_uniform(rows, cols, prec, 41, lo, 1.0).reshape(rows, cols)
    r = O.fill_uniform(rows, 1, prec, 42, lo, 1.0).reshape(rows, 1)
    c = O.fill_uniform(1, cols, prec, 43, lo, 1.0).reshape(1, cols)
    want_r, want_c = O.rowcolsum_c(1.0, a, prec, r, prec, c, prec)
    with G.Session(workers=1) as s:
        one = lambda rr, cc: G.makeSingleTileLayout(rr, cc, 0)
        A = s.createMatrix(rows, cols, G.Precision(prec), one(rows, cols))
        R = s.createMatrix(rows, 1, G.Precision(prec), one(rows, 1))
        C = s.createMatrix(1, cols, G.Precision(prec), one(1, cols))
        for M, img in ((A, a), (R, r), (C, c)):
            s.setDataRaw(M, img)
        G.addRowColSum(s, A, R, C, 1.0, True)
        got_r = s.getDataRaw(R).reshape(rows, 1)
        got_c = s.getDataRaw(C).reshape(1, cols)
    assert same_bits(got_r, want_r, prec) and same_bits(got_c, want_c, prec), (prec, shape)


@pytest.mark.parametrize("prec,value", [(0, 65520.0), (1, 1.0 / 3.0), (2, np.pi), (3, -1.0 / 3.0), (3, 1e39)])
def test_set_const(prec, value):
    rows, cols, p = 130, 77, 3
    with G.Session(workers=p) as s:
        M = s.createMatrix(rows, cols, G.Precision(prec), layout_of(LAYOUTS["grid"](rows, cols, p)))
        G.setConst(s, M, value)
        got = s.getDataRaw(M)
    assert same_bits(got, O.set_const_c((rows * cols,), prec, value), prec)


def test_fc_layer_train_step_matches_composed_oracle():
    """One hidden FC layer, reference Trainer order and layouts (dnn.cpp:87-190):
    z = x.W; z += b; act = relu(z); delta = reluGrad(z, dAct);
    dW = x^T.delta; db = colsum(delta); dX = delta.W^T; W -= lr dW; b -= lr db.
    Single storage, 4 workers; W and b replicated (forward reads the replica)."""
    batch, fin, fout, p = 256, 384, 320, 4
    lr = 0.05
    x = O.fill_uniform(batch, fin, 1, 41).reshape(batch, fin)
    w = O.fill_uniform(fin, fout, 1, 42, -0.05, 0.05).reshape(fin, fout)
    b = O.fill_uniform(1, fout, 1, 43, -0.1, 0.1).reshape(1, fout)
    dact = O.fill_uniform(batch, fout, 1, 44).reshape(batch, fout)
    grp = list(range(p))
    with G.Session(workers=p) as s:
        def mk(r, c, lay, img=None):
            m = s.createMatrix(r, c, G.Precision.Single, lay(r, c, grp))
            if img is not None:
                s.setDataRaw(m, img)
            return m
        X = mk(batch, fin, G.makeRowBlockLayout, x)
        W = mk(fin, fout, G.makeColBlockLayout, w)
        Bv = mk(1, fout, G.makeColBlockLayout, b)
        Z = mk(batch, fout, G.makeRowBlockLayout)
        ACT = mk(batch, fout, G.makeRowBlockLayout)
        DEL = mk(batch, fout, G.makeRowBlockLayout, dact)
        DW = mk(fin, fout, G.makeColBlockLayout)
        DB = mk(1, fout, G.makeColBlockLayout)
        ROW = mk(batch, 1, G.makeRowBlockLayout)
        DX = mk(batch, fin, G.makeRowBlockLayout)
        s.replicateSync(W)
        s.replicateSync(Bv)
        G.gemm(s, X, W, Z, 1.0, 0.0)
        G.biasAdd(s, Z, Bv)
        G.relu(s, Z, ACT)
        G.reluGrad(s, Z, DEL)
        G.gemm(s, X, DEL, DW, 1.0, 0.0, True, False)
        G.setConst(s, ROW, 0.0)
        G.setConst(s, DB, 0.0)
        G.addRowColSum(s, DEL, ROW, DB, 1.0, True)
        G.gemm(s, DEL, W, DX, 1.0, 0.0, False, True)
        G.axpy(s, -lr, DW, W)
        G.axpy(s, -lr, DB, Bv)
        s.verifyMetadataConsistency()
        got = {k: s.getDataRaw(M)
               for k, M in dict(z=Z, act=ACT, dl=DEL, dw=DW, db=DB, dx=DX, w=W, b=Bv).items()}
    # Composed oracle (C restatements).
    z = O.gemm_c(batch, fout, fin, x, 1, w, 1, np.zeros((batch, fout), np.float32), 1, 1.0, 0.0, 0, 0)
    # GEMM outputs agree within the fp32 tolerance; the neighbours are then
    # checked bit-for-bit on the device's own GEMM outputs.
    z = O.ew_c(False, 5, 0.0, z, 1, b, 1, z, 1)  # biasAdd in place
    assert O.rel_fro(got["z"], z) <= 1e-5
    assert same_bits(got["act"], O.ew_c(True, 0, 0.0, got["z"], 1, None, 1, got["z"], 1), 1)
    dl = O.ew_c(False, 3, 0.0, got["z"], 1, dact, 1, dact, 1)
    assert same_bits(got["dl"], dl, 1)
    dw = O.gemm_c(fin, fout, batch, x, 1, dl, 1, np.zeros((fin, fout), np.float32), 1, 1.0, 0.0, 1, 0)
    assert O.rel_fro(got["dw"], dw) <= 1e-5
    _, db = O.rowcolsum_c(1.0, dl, 1, np.zeros((batch, 1), np.float32), 1, np.zeros((1, fout), np.float32), 1)
    assert same_bits(got["db"], db, 1)
    dx = O.gemm_c(batch, fin, fout, dl, 1, w, 1, np.zeros((batch, fin), np.float32), 1, 1.0, 0.0, 0, 1)
    assert O.rel_fro(got["dx"], dx) <= 1e-5
    assert same_bits(got["w"], O.ew_c(False, 2, -lr, got["dw"], 1, w, 1, w, 1), 1)
    assert same_bits(got["b"], O.ew_c(False, 2, -lr, got["db"], 1, b, 1, b, 1), 1)


def test_colsum_reuses_gemm_panel():
    """Keep what you've seen: dW = X^T.delta gathers delta's column band for
    each dW owner; addRowColSum's db need is the same band, so it is served
    from the panel cache with no new bytes on the data plane."""
    batch, fin, fout, p = 512, 256, 384, 4
    grp = list(range(p))
    with G.Session(workers=p) as s:
        X = s.createMatrix(batch, fin, G.Precision.Single, G.makeRowBlockLayout(batch, fin, grp))
        DL = s.createMatrix(batch, fout, G.Precision.Single, G.makeRowBlockLayout(batch, fout, grp))
        DW = s.createMatrix(fin, fout, G.Precision.Single, G.makeColBlockLayout(fin, fout, grp))
        DB = s.createMatrix(1, fout, G.Precision.Single, G.makeColBlockLayout(1, fout, grp))
        ROW = s.createMatrix(batch, 1, G.Precision.Single, G.makeRowBlockLayout(batch, 1, grp))
        s.fillUniform(X, 1)
        s.fillUniform(DL, 2)
        G.gemm(s, X, DL, DW, 1.0, 0.0, True, False)
        before = s.queryWorkerStats()
        G.addRowColSum(s, DL, ROW, DB, 1.0, True)
        after = s.queryWorkerStats()
        dl = s.getDataRaw(DL)
        got = s.getDataRaw(DB)
    assert sum(a["bytes_received"] for a in after) == sum(b["bytes_received"] for b in before)
    assert sum(a["cache_hits"] for a in after) >= sum(b["cache_hits"] for b in before) + p
    _, want = O.rowcolsum_c(1.0, dl, 1, np.zeros((batch, 1), np.float32), 1, np.zeros((1, fout), np.float32), 1)
    assert same_bits(got, want, 1)


def test_validation_errors_before_issue():
    with G.Session(workers=2) as s:
        grp = [0, 1]
        A = s.createMatrix(8, 6, G.Precision.Single, G.makeRowBlockLayout(8, 6, grp))
        B = s.createMatrix(8, 5, G.Precision.Single, G.makeRowBlockLayout(8, 5, grp))
        R = s.createMatrix(8, 1, G.Precision.Single, G.makeRowBlockLayout(8, 1, grp))
        C = s.createMatrix(1, 6, G.Precision.Single, G.makeColBlockLayout(1, 6, grp))
        v = A.version()
        with pytest.raises(G.GmError, match="shape mismatch"):
            G.addMatrices(s, A, B, A)
        with pytest.raises(G.GmError, match="bias must be 1 x cols"):
            G.biasAdd(s, A, R)
        with pytest.raises(G.GmError, match="rowAcc must be rows x 1"):
            G.addRowColSum(s, A, C, R, 1.0, True)
        with pytest.raises(G.GmError, match="distinct"):
            G.addRowColSum(s, A, R, R, 1.0, True)
        assert A.version() == v
        s.verifyMetadataConsistency()
