# SPDX-License-Identifier: Apache-2.0
"""GPU parity of the distributed GEMM path against the reference.

Every case runs through the C ABI (Session / createMatrix / setDataRaw /
gemm / getDataRaw, include/gridmath_b200.h) with P virtual workers on the
GPU(s) present, and is compared with the golden outputs of the UNMODIFIED
reference library (tests/golden/, oracle/make_golden.py) or with the C
restatement of its runGemm (oracle/gemm_oracle.c) on identical inputs.

Tolerances (BASELINE.json north_star), relative Frobenius error:
  fp64 <= 1e-12, fp32 / tf32 <= 1e-5, fp16 / bf16 with fp32 accumulation <= 1e-2.
"""
import numpy as np
import pytest

import oracle as O
from conftest import load_case
from paper_1611_07819_b200 import gridmath as G

pytestmark = pytest.mark.gpu

TOL = {0: 1e-2, 1: 1e-5, 2: 1e-12, 3: 1e-2}


def layout_of(tiles):
    return G.Layout([(G.TileExtent(*map(int, t[:4])), int(t[4])) for t in tiles])


def run_session_gemm(p, a, pa, at, b, pb, bt, c, pc, ct, alpha, beta, ta, tb, repl=0, math=0,
                     det=True):
    with G.Session(workers=p, deterministic=det) as s:
        A = s.createMatrix(a.shape[0], a.shape[1], G.Precision(pa), layout_of(at))
        B = s.createMatrix(b.shape[0], b.shape[1], G.Precision(pb), layout_of(bt))
        C = s.createMatrix(c.shape[0], c.shape[1], G.Precision(pc), layout_of(ct))
        s.setDataRaw(A, a)
        s.setDataRaw(B, b)
        s.setDataRaw(C, c)
        if repl & 1:
            s.replicateSync(A)
        if repl & 2:
            s.replicateSync(B)
        G.gemm(s, A, B, C, alpha, beta, bool(ta), bool(tb), math=math)
        s.verifyMetadataConsistency()
        return s.getDataRaw(C)


def err_tol(c):
    # Output precision bounds the achievable error; Half outputs also absorb
    # the reference's subnormal-half widening bug.
    tol = TOL[c["pc"]] if c["pc"] != 1 else 1e-5
    if 2 in (c["pa"], c["pb"], c["pc"]):
        tol = 1e-12 if c["pc"] == 2 else TOL[c["pc"]]
    if c["pc"] == 0:
        tol = 1e-3
    return tol


def test_golden_cases_match_reference(golden_index):
    failures = []
    for c in golden_index["cases"]:
        d = load_case(c["name"])
        got = run_session_gemm(c["p"], d["a"], c["pa"], d["at"], d["b"], c["pb"], d["bt"], d["c"], c["pc"],
                               d["ct"], c["alpha"], c["beta"], c["ta"], c["tb"], c["repl"], det=c["det"])
        if c["special"] == "nan_ab":
            ok = np.array_equal(got, d["out"])  # alpha = 0: C = beta*C exactly, A/B never read
        else:
            e = O.rel_fro(O.to_f64(got, c["pc"]), O.to_f64(d["out"], c["pc"]))
            ok = e <= err_tol(c) and np.isfinite(O.to_f64(got, c["pc"])).all()
            c["err"] = e
        if not ok:
            failures.append((c["name"], c.get("err")))
    assert not failures, failures


def test_bf16_storage_matches_reference_single_compute(golden_index):
    # Same bf16-representable values: reference stores them as Single; the
    # B200 path stores BF16 and runs tcgen05 kind::f16 (bf16) with fp32
    # accumulation -- products exact, so agreement is at fp32 level.
    for name in ("bf16_as_single", "bf16_as_single_p1"):
        c = [x for x in golden_index["cases"] if x["name"] == name][0]
        d = load_case(name)
        a16 = (d["a"].view(np.uint32) >> 16).astype(np.uint16)
        b16 = (d["b"].view(np.uint32) >> 16).astype(np.uint16)
        got = run_session_gemm(c["p"], a16, 3, d["at"], b16, 3, d["bt"], d["c"], 1, d["ct"], c["alpha"],
                               c["beta"], 0, 0)
        assert O.rel_fro(got, d["out"]) <= 1e-5, name


def test_layout_invariance_bitwise():
    # Deterministic mode: one ascending-k chain per element in the kernel,
    # so the result is bitwise independent of layouts and P (reference
    # kernels.hpp:19-22, survey probe).
    from make_golden import irregular_tiles
    m, n, k = 640, 384, 576
    a = O.fill_uniform(m, k, 3, 11)
    b = O.fill_uniform(k, n, 3, 12)
    c = np.zeros((m, n), dtype=np.float32)
    cfgs = [
        (1, [(0, m, 0, k, 0)], [(0, k, 0, n, 0)], [(0, m, 0, n, 0)]),
        (2, O.row_block_tiles(m, k, 2), O.col_block_tiles(k, n, 2), O.grid_tiles(m, n, 1, 2)),
        (4, O.grid_tiles(m, k, 2, 2), O.grid_tiles(k, n, 2, 2), O.grid_tiles(m, n, 2, 2)),
        (3, irregular_tiles(m, k, 3), irregular_tiles(k, n, 3), irregular_tiles(m, n, 3)),
        (8, O.row_block_tiles(m, k, 8), O.col_block_tiles(k, n, 8), O.col_block_tiles(m, n, 8)),
    ]
    outs = [run_session_gemm(p, a, 3, at, b, 3, bt, c, 1, ct, 1.0, 0.0, 0, 0) for p, at, bt, ct in cfgs]
    for o in outs[1:]:
        assert np.array_equal(o.view(np.uint32), outs[0].view(np.uint32))
    ref = O.gemm_c(m, n, k, a, 3, b, 3, c, 1, 1.0, 0.0, 0, 0)
    assert O.rel_fro(outs[0], ref) < 1e-5


def test_config1_fp32_2048_grid_2x2_vs_reference():
    # BASELINE config 1: fp32 2048^3 on a 2x2 block-distributed layout, 4 workers.
    n = 2048
    a = O.fill_uniform(n, n, 1, 1)
    b = O.fill_uniform(n, n, 1, 2)
    c = np.zeros((n, n), dtype=np.float32)
    t = O.grid_tiles(n, n, 2, 2)
    got = run_session_gemm(4, a, 1, t, b, 1, t, c, 1, t, 1.0, 0.0, 0, 0)
    if O.ref_available():
        want, _ = O.gemm_ref(4, a, 1, t, b, 1, t, c, 1, t, 1.0, 0.0, 0, 0)
    else:
        rows = (0, 64)
        want = O.gemm_c(n, n, n, a, 1, b, 1, c, 1, 1.0, 0.0, 0, 0, rows)[: rows[1]]
        got = got[: rows[1]]
    assert O.rel_fro(got, want) <= 1e-5


def test_fp32_tf32_opt_in_mode():
    m, n, k = 384, 320, 448
    a = O.fill_uniform(m, k, 1, 5)
    b = O.fill_uniform(k, n, 1, 6)
    c = np.zeros((m, n), dtype=np.float32)
    t = lambda r, cc: O.grid_tiles(r, cc, 2, 2)
    want = O.gemm_c(m, n, k, a, 1, b, 1, c, 1, 1.0, 0.0, 0, 0)
    got3 = run_session_gemm(4, a, 1, t(m, k), b, 1, t(k, n), c, 1, t(m, n), 1.0, 0.0, 0, 0, math=0)
    got1 = run_session_gemm(4, a, 1, t(m, k), b, 1, t(k, n), c, 1, t(m, n), 1.0, 0.0, 0, 0, math=1)
    assert O.rel_fro(got3, want) <= 1e-5        # 3xTF32 default: fp32-accurate
    assert 1e-5 < O.rel_fro(got1, want) <= 2e-3  # 1xTF32: opt-in, tf32 input rounding
    # on tf32-representable inputs the opt-in mode meets the fp32 bar too
    a_t = (a.view(np.uint32) & 0xFFFFE000).view(np.float32)
    b_t = (b.view(np.uint32) & 0xFFFFE000).view(np.float32)
    want_t = O.gemm_c(m, n, k, a_t, 1, b_t, 1, c, 1, 1.0, 0.0, 0, 0)
    got_t = run_session_gemm(4, a_t, 1, t(m, k), b_t, 1, t(k, n), c, 1, t(m, n), 1.0, 0.0, 0, 0, math=1)
    assert O.rel_fro(got_t, want_t) <= 1e-5


def test_fp64_dmma_vs_oracle():
    m, n, k = 520, 392, 456
    for ta, tb in ((0, 0), (1, 0), (0, 1), (1, 1)):
        a = O.fill_uniform(k if ta else m, m if ta else k, 2, 21)
        b = O.fill_uniform(n if tb else k, k if tb else n, 2, 22)
        c = O.fill_uniform(m, n, 2, 23)
        want = O.gemm_c(m, n, k, a, 2, b, 2, c, 2, 0.75, 0.5, ta, tb)
        got = run_session_gemm(2, a, 2, O.row_block_tiles(*a.shape, 2), b, 2, O.col_block_tiles(*b.shape, 2), c, 2,
                               O.grid_tiles(m, n, 1, 2), 0.75, 0.5, ta, tb)
        assert O.rel_fro(got, want) <= 1e-12, (ta, tb)


def test_mixed_precision_mode():
    # Half operands with Single C (Single compute, fp32 accumulate) and a
    # Double C (Double compute): reference computePrecision, kernels.cpp:136-140.
    m, n, k = 256, 192, 320
    a = O.fill_uniform(m, k, 0, 31)
    b = O.fill_uniform(k, n, 0, 32)
    # Flush subnormal halves: the reference widens them to half their IEEE
    # value (precision.hpp:87 off-by-one); the product is IEEE.
    for x in (a, b):
        x[(x & 0x7C00) == 0] = 0
    for pc, tol in ((1, 1e-5), (2, 1e-12)):
        c = np.zeros((m, n), dtype=O.NP_DTYPE[pc])
        want = O.gemm_c(m, n, k, a, 0, b, 0, c, pc, 1.0, 0.0, 0, 0)
        got = run_session_gemm(4, a, 0, O.grid_tiles(m, k, 2, 2), b, 0, O.grid_tiles(k, n, 2, 2), c, pc,
                               O.grid_tiles(m, n, 2, 2), 1.0, 0.0, 0, 0)
        assert O.rel_fro(got, want) <= tol, pc


def test_config2_bf16_8192_single_gpu_sampled_rows():
    # BASELINE config 2 (bf16 8192^3, one B200), checked on sampled rows
    # against the C restatement (full CPU check would take minutes).
    n = 8192
    with G.Session(workers=1) as s:
        lay = G.makeSingleTileLayout(n, n, 0)
        A = s.createMatrix(n, n, G.Precision.BF16, lay)
        B = s.createMatrix(n, n, G.Precision.BF16, lay)
        C = s.createMatrix(n, n, G.Precision.Single, lay)
        s.fillUniform(A, 1)
        s.fillUniform(B, 2)
        G.gemm(s, A, B, C, 1.0, 0.0)
        got = s.getDataRaw(C)
        a = s.getDataRaw(A)
        b = s.getDataRaw(B)
    assert np.array_equal(a[:4], O.fill_uniform(4, n, 3, 1))  # device generator == oracle generator
    rows = (4096, 4104)
    want = O.gemm_c(n, n, n, a, 3, b, 3, np.zeros((n, n), np.float32), 1, 1.0, 0.0, 0, 0, rows)
    assert O.rel_fro(got[rows[0]:rows[1]], want[rows[0]:rows[1]]) <= 1e-5


def test_dimension_mismatch_and_aliasing_errors():
    with G.Session(workers=2) as s:
        A = s.createMatrix(8, 6, G.Precision.Single, G.makeRowBlockLayout(8, 6, [0, 1]))
        B = s.createMatrix(5, 4, G.Precision.Single, G.makeRowBlockLayout(5, 4, [0, 1]))
        C = s.createMatrix(8, 4, G.Precision.Single, G.makeRowBlockLayout(8, 4, [0, 1]))
        with pytest.raises(G.GmError, match="dimension mismatch"):
            G.gemm(s, A, B, C, 1.0, 0.0)
        with pytest.raises(G.GmError, match="distinct"):
            G.gemm(s, C, C, C, 1.0, 0.0)
        bad = G.Layout([(G.TileExtent(0, 4, 0, 4), 0)])
        with pytest.raises(G.GmError, match="invalid layout"):
            s.createMatrix(8, 4, G.Precision.Single, bad)


def test_kernel_numerics_vs_torch_fp32():
    # Direct kernel check (gm_gemm_local) against a plain PyTorch fp32 reference.
    import ctypes
    import torch
    from paper_1611_07819_b200 import _lib
    lib = _lib.load()
    dt = {3: torch.bfloat16, 0: torch.float16, 1: torch.float32}
    for (m, n, k, ta, tb, p) in [(300, 520, 260, 0, 0, 3), (1024, 768, 512, 1, 1, 0), (256, 384, 512, 1, 0, 1),
                                 (2048, 2048, 2048, 0, 1, 3)]:
        g = torch.Generator(device="cuda").manual_seed(m + n + k)
        A = torch.rand((k, m) if ta else (m, k), device="cuda", generator=g).mul(2).sub(1).to(dt[p])
        B = torch.rand((n, k) if tb else (k, n), device="cuda", generator=g).mul(2).sub(1).to(dt[p])
        C = torch.empty(m, n, device="cuda", dtype=torch.float32)
        d = _lib.gm_gemm_desc(m=m, n=n, k=k, lda=A.shape[1], ldb=B.shape[1], ldc=n, trans_a=ta, trans_b=tb,
                              prec_a=p, prec_b=p, prec_c=1, math=0, cta_group=0, max_ctas=0, alpha=1.0, beta=0.0)
        ws = ctypes.c_uint64()
        _lib.check(lib.gm_gemm_workspace_size(ctypes.byref(d), ctypes.byref(ws)))
        W = torch.empty(max(ws.value, 16), dtype=torch.uint8, device="cuda")
        _lib.check(lib.gm_gemm_local(ctypes.byref(d), A.data_ptr(), B.data_ptr(), C.data_ptr(), W.data_ptr(),
                                     ws.value, torch.cuda.current_stream().cuda_stream))
        torch.cuda.synchronize()
        ref = (A.float().T if ta else A.float()) @ (B.float().T if tb else B.float())
        assert ((C - ref).norm() / ref.norm()).item() <= 1e-5


def test_layout_invariance_bitwise_wide_tiles():
    # k >= 4096 selects the 256x512 (two-UMMA) tile for C tiles wider than 256
    # columns and the 256x256 tile otherwise; both give the same bits.
    m, n, k = 1024, 768, 4608
    a = O.fill_uniform(m, k, 3, 41)
    b = O.fill_uniform(k, n, 3, 42)
    c = np.zeros((m, n), dtype=np.float32)
    outs = [
        run_session_gemm(1, a, 3, [(0, m, 0, k, 0)], b, 3, [(0, k, 0, n, 0)], c, 1, [(0, m, 0, n, 0)], 1.0, 0.0, 0, 0),
        run_session_gemm(4, a, 3, O.grid_tiles(m, k, 2, 2), b, 3, O.grid_tiles(k, n, 2, 2), c, 1,
                         O.grid_tiles(m, n, 2, 2), 1.0, 0.0, 0, 0),
        run_session_gemm(8, a, 3, O.row_block_tiles(m, k, 8), b, 3, O.col_block_tiles(k, n, 8), c, 1,
                         O.col_block_tiles(m, n, 8), 1.0, 0.0, 0, 0),
    ]
    for o in outs[1:]:
        assert np.array_equal(o.view(np.uint32), outs[0].view(np.uint32))
    rows = (100, 116)
    want = O.gemm_c(m, n, k, a, 3, b, 3, c, 1, 1.0, 0.0, 0, 0, rows)
    assert O.rel_fro(outs[0][rows[0]:rows[1]], want[rows[0]:rows[1]]) < 1e-5


RAGGED_SHAPES = [(1, 1, 1), (3, 5, 7), (37, 53, 29), (1, 300, 1), (300, 1, 300), (129, 257, 65), (17, 9, 1031)]
RAGGED_PRECS = [(3, 3, 1), (0, 0, 0), (1, 1, 1), (2, 2, 2), (3, 1, 2), (0, 0, 3)]


@pytest.mark.parametrize("m,n,k", RAGGED_SHAPES)
def test_ragged_shapes_vs_oracle(m, n, k):
    # Edge shapes (single elements, odd sizes, rows/cols below 16 bytes so
    # tiles need padded pitches, k = 1, long thin k): every precision mix
    # and transpose, on 1 worker and on 4 workers with idle owners where a
    # dimension is smaller than the worker count.
    def tiles(rows, cols, kind, p):
        if p == 1:
            return [(0, rows, 0, cols, 0)]
        if kind == "row" and rows >= p:
            return O.row_block_tiles(rows, cols, p)
        if kind == "col" and cols >= p:
            return O.col_block_tiles(rows, cols, p)
        if kind == "grid" and rows >= 2 and cols >= 2:
            return O.grid_tiles(rows, cols, 2, 2)
        return [(0, rows, 0, cols, p - 1)]  # one owner, the others idle

    for (pa, pb, pc) in RAGGED_PRECS:
        for ta, tb in [(0, 0), (1, 1), (1, 0)]:
            seed = m * 7 + n * 11 + k * 13 + pa + 4 * pb + 16 * pc + 64 * ta + 128 * tb
            a = O.fill_uniform(k if ta else m, m if ta else k, pa, seed)
            b = O.fill_uniform(n if tb else k, k if tb else n, pb, seed + 1)
            c = O.fill_uniform(m, n, pc, seed + 2)
            want = O.gemm_c(m, n, k, a, pa, b, pb, c, pc, 0.75, 0.5, ta, tb)
            tol = 1e-12 if 2 in (pa, pb, pc) and pc == 2 else (1e-3 if pc == 0 else TOL[pc])
            for p in (1, 4):
                got = run_session_gemm(p, a, pa, tiles(a.shape[0], a.shape[1], "row", p), b, pb,
                                       tiles(b.shape[0], b.shape[1], "col", p), c, pc, tiles(m, n, "grid", p),
                                       0.75, 0.5, ta, tb)
                err = O.rel_fro(O.to_f64(got, pc), O.to_f64(want, pc))
                assert err <= tol, (m, n, k, pa, pb, pc, ta, tb, p, err)


@pytest.mark.parametrize("tb", [0, 1])
def test_bf16_fold_mode_matches_reference_serial_sum(tb):
    """GM_MATH_FOLD: bf16 operands, Single C, long k -- the accumulation is
    folded into a round-to-nearest fp32 sum every 256 of k, so the result
    tracks the reference's serial fp32 chain (runGemm<float>) far closer than
    the default whole-k tensor-core accumulation; layout-invariant bitwise."""
    m, n, k = 512, 384, 16384
    a = O.fill_uniform(m, k, 3, 41)
    b = O.fill_uniform(n, k, 3, 42) if tb else O.fill_uniform(k, n, 3, 42)
    c = np.zeros((m, n), dtype=np.float32)
    rows = (100, 132)
    want = O.gemm_c(m, n, k, a, 3, b, 3, c, 1, 1.0, 0.0, 0, tb, rows)[rows[0]:rows[1]]
    grid = lambda r, cc: O.grid_tiles(r, cc, 2, 2)
    bt = grid(n, k) if tb else grid(k, n)
    fold = run_session_gemm(4, a, 3, grid(m, k), b, 3, bt, c, 1, grid(m, n), 1.0, 0.0, 0, tb, math=2)
    plain = run_session_gemm(4, a, 3, grid(m, k), b, 3, bt, c, 1, grid(m, n), 1.0, 0.0, 0, tb, math=0)
    e_fold = O.rel_fro(fold[rows[0]:rows[1]], want)
    e_plain = O.rel_fro(plain[rows[0]:rows[1]], want)
    assert e_fold <= 1e-5 and e_fold < e_plain / 2, (e_fold, e_plain)
    one = run_session_gemm(1, a, 3, O.grid_tiles(m, k, 1, 1), b, 3, O.grid_tiles(*b.shape, 1, 1), c, 1,
                           O.grid_tiles(m, n, 1, 1), 1.0, 0.0, 0, tb, math=2)
    assert np.array_equal(fold.view(np.uint8), one.view(np.uint8))
