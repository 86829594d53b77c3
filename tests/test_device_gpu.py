# SPDX-License-Identifier: Apache-2.0
"""Device-layer checks through the C ABI: storage conversions (device vs the
host convertBuffer restatement, bitwise, with edge values), the SplitMix64
generator (device vs oracle, every precision), the pooled arena, and
stream-ordered gemm_async chains with beta accumulation."""
import ctypes

import numpy as np
import pytest

import oracle as O
from paper_1611_07819_b200 import _lib
from paper_1611_07819_b200 import gridmath as G

pytestmark = pytest.mark.gpu

DT = {0: np.uint16, 1: np.float32, 2: np.float64, 3: np.uint16}


def _edge_values():
    v = [0.0, -0.0, 1.0, -1.0, 65504.0, 65519.99, 65520.0, -70000.0, 1e30, -1e-30, 6.0e-5, 5.96e-8,
         2.98e-8, 1e-45, 3.4e38, float("inf"), float("-inf"), 1.0 / 3.0, 2.0 ** -24, 2.0 ** -25]
    rng = np.random.default_rng(3)
    v += list(rng.standard_normal(4000) * 100) + list(rng.uniform(-1e-4, 1e-4, 2000))
    return np.array(v, dtype=np.float64)


def _to_prec(x64, p):
    out = np.empty(x64.size, dtype=DT[p])
    _lib.check(_lib.load().gm_convert_host(x64.ctypes.data, 2, out.ctypes.data, p, x64.size))
    return out


def test_device_convert_matches_host_bitwise():
    import torch
    lib = _lib.load()
    x64 = _edge_values()
    for sp in (0, 1, 2, 3):
        src = _to_prec(x64, sp)
        for dp in (0, 1, 2, 3):
            want = np.empty(src.size, dtype=DT[dp])
            _lib.check(lib.gm_convert_host(src.ctypes.data, sp, want.ctypes.data, dp, src.size))
            d_src = torch.from_numpy(src.view(np.uint8).copy()).cuda()
            d_dst = torch.empty(want.nbytes, dtype=torch.uint8, device="cuda")
            _lib.check(lib.gm_convert(d_src.data_ptr(), sp, d_dst.data_ptr(), dp, src.size, None))
            torch.cuda.synchronize()
            got = d_dst.cpu().numpy().view(DT[dp])
            assert np.array_equal(got.view(np.uint8), want.view(np.uint8)), (sp, dp)


def test_device_generator_matches_oracle_every_precision():
    with G.Session(workers=3) as s:
        for p in (0, 1, 2, 3):
            M = s.createMatrix(37, 53, G.Precision(p), G.makeGridLayout(37, 53, 1, 3, G.makeWorkerGroup(3)))
            s.fillUniform(M, 17, -2.0, 3.0)
            got = s.getDataRaw(M)
            want = O.fill_uniform(37, 53, p, 17, -2.0, 3.0)
            assert np.array_equal(got.view(np.uint8), want.view(np.uint8)), p


@pytest.mark.gpu
@pytest.mark.parametrize("rows,cols,pr,pc", [(40, 96, 1, 3), (41, 180, 2, 2), (33, 184, 1, 2), (300, 1024, 2, 2)])
def test_device_generator_vector_path_matches_oracle(rows, cols, pr, pc):
    # Tiles with 16-byte aligned rows take the 8-columns-per-thread generator;
    # 90- and 92-wide tiles leave a scalar tail (fp64 / fp32) or fall back
    # (16-bit rows not 16-byte aligned).
    with G.Session(workers=pr * pc) as s:
        for p in (0, 1, 2, 3):
            M = s.createMatrix(rows, cols, G.Precision(p),
                               G.makeGridLayout(rows, cols, pr, pc, G.makeWorkerGroup(pr * pc)))
            s.fillUniform(M, 23, -1.0, 1.0)
            got = s.getDataRaw(M)
            want = O.fill_uniform(rows, cols, p, 23, -1.0, 1.0)
            assert np.array_equal(got.view(np.uint8), want.view(np.uint8)), p


def test_arena_reuse_and_counters():
    lib = _lib.load()
    a = ctypes.c_void_p()
    _lib.check(lib.gm_arena_create(0, 0, ctypes.byref(a)))
    ptrs = []
    for sz in (1000, 5000, 1 << 20, 3 << 20):
        p = ctypes.c_void_p()
        _lib.check(lib.gm_arena_alloc(a, sz, ctypes.byref(p)))
        ptrs.append(p.value)
    for p in ptrs:
        _lib.check(lib.gm_arena_free(a, p))
    for sz in (1000, 5000, 1 << 20, 3 << 20):
        p = ctypes.c_void_p()
        _lib.check(lib.gm_arena_alloc(a, sz, ctypes.byref(p)))
        assert p.value in ptrs
    st = _lib.gm_arena_stats()
    _lib.check(lib.gm_arena_get_stats(a, ctypes.byref(st)))
    assert st.allocations_from_os == 4 and st.reuses == 4 and st.frees == 4
    with pytest.raises(_lib.GmError):
        _lib.check(lib.gm_arena_free(a, 12345))
    _lib.check(lib.gm_arena_destroy(a))


def test_async_chain_with_beta_accumulation():
    # C <- A B + C three times through the stream-ordered API (one sync at the end).
    m, n, k, p = 640, 512, 768, 4
    a = O.fill_uniform(m, k, 3, 61)
    b = O.fill_uniform(k, n, 3, 62)
    c0 = O.fill_uniform(m, n, 1, 63)
    with G.Session(workers=p) as s:
        A = s.createMatrix(m, k, G.Precision.BF16, G.makeGridLayout(m, k, 2, 2, G.makeWorkerGroup(p)))
        B = s.createMatrix(k, n, G.Precision.BF16, G.makeRowBlockLayout(k, n, G.makeWorkerGroup(p)))
        C = s.createMatrix(m, n, G.Precision.Single, G.makeColBlockLayout(m, n, G.makeWorkerGroup(p)))
        s.setDataRaw(A, a)
        s.setDataRaw(B, b)
        s.setDataRaw(C, c0)
        for _ in range(3):
            s.gemmAsync(A, B, C, 1.0, 1.0)
        s.synchronize()
        got = s.getDataRaw(C)
        assert C.version() == 4  # setData + 3 gemms
    want = c0
    for _ in range(3):
        want = O.gemm_c(m, n, k, a, 3, b, 3, want, 1, 1.0, 1.0, 0, 0)
    assert O.rel_fro(got, want) <= 1e-5


def test_get_data_roundtrip_all_layouts():
    rng = np.random.default_rng(9)
    img = rng.standard_normal((97, 61)).astype(np.float32)
    with G.Session(workers=4) as s:
        for lay in (G.makeRowBlockLayout(97, 61, G.makeWorkerGroup(4)), G.makeColBlockLayout(97, 61, G.makeWorkerGroup(4)),
                    G.makeGridLayout(97, 61, 2, 2, G.makeWorkerGroup(4)), G.makeSingleTileLayout(97, 61, 3)):
            M = s.createMatrix(97, 61, G.Precision.Single, lay)
            s.setDataRaw(M, img)
            assert np.array_equal(s.getDataRaw(M), img)
            s.setData(M, img.astype(np.float64) * 2)
            assert np.array_equal(s.getData(M), (img * 2).astype(np.float64))
            s.destroy(M)


def test_worker_errors_aggregate_and_session_survives():
    # Reference behaviour: worker failures become one Error ("op failed: worker r: ...",
    # session.cpp:149-154); createMatrix rolls back (session.cpp:208-216).
    with G.Session(workers=2) as s:
        huge = 1 << 22  # 2^22 x 2^22 doubles = 128 TiB
        with pytest.raises(G.GmError, match="op failed: worker"):
            s.createMatrix(huge, huge, G.Precision.Double, G.makeRowBlockLayout(huge, huge, [0, 1]))
        M = s.createMatrix(64, 64, G.Precision.Single, G.makeRowBlockLayout(64, 64, [0, 1]))
        s.fillUniform(M, 1)
        assert s.getDataRaw(M).shape == (64, 64)
        s.verifyMetadataConsistency()
        s.destroy(M)
        with pytest.raises(G.GmError, match="unknown matrix id"):
            s.getDataRaw(M)
        with pytest.raises(G.GmError):
            s.setDataRaw(s.createMatrix(4, 4, G.Precision.Single, G.makeSingleTileLayout(4, 4, 0)),
                         np.zeros(3, dtype=np.float32))


def test_reshape_layouts_and_precisions():
    # reference execReshape (kernels.cpp:1083-1127): pieces from old tiles (or
    # the fresh replica) to the new owners, then convertBuffer to the new precision.
    m, n, p = 150, 94, 4
    g = G.makeWorkerGroup(p)
    img = O.fill_uniform(m, n, 1, 77, -3.0, 3.0)
    with G.Session(workers=p) as s:
        M = s.createMatrix(m, n, G.Precision.Single, G.makeRowBlockLayout(m, n, g))
        s.setDataRaw(M, img)
        v0 = M.version()
        s.reshape(M, G.makeColBlockLayout(m, n, g), G.Precision.Half)
        assert M.version() == v0 + 1 and M.precision() == G.Precision.Half
        want_h = _to_prec(img.astype(np.float64).ravel(), 0).reshape(m, n)  # Single -> Half (RNE)
        assert np.array_equal(s.getDataRaw(M).view(np.uint16), want_h)
        s.reshape(M, G.makeGridLayout(m, n, 2, 2, g), G.Precision.Single)
        back = s.getDataRaw(M)
        assert np.array_equal(back, want_h.view(np.float16).astype(np.float32))
        # via the replica path, then a gemm on the reshaped operand
        h = s.replicateAsync(M)
        assert s.wait(h) == G.ReplState.Done
        s.reshape(M, G.makeSingleTileLayout(m, n, 3), G.Precision.BF16)
        assert M.info()[4] == 2 ** 64 - 1  # replicatedVersion reset with the new descriptor
        want_b = _to_prec(back.astype(np.float64).ravel(), 3).reshape(m, n)
        assert np.array_equal(s.getDataRaw(M).view(np.uint16), want_b)
        B = s.createMatrix(n, 64, G.Precision.BF16, G.makeRowBlockLayout(n, 64, g))
        C = s.createMatrix(m, 64, G.Precision.Single, G.makeGridLayout(m, 64, 2, 2, g))
        s.fillUniform(B, 5)
        G.gemm(s, M, B, C, 1.0, 0.0)
        b = s.getDataRaw(B)
        got = s.getDataRaw(C)
    want = O.gemm_c(m, 64, n, want_b, 3, b, 3, np.zeros((m, 64), np.float32), 1, 1.0, 0.0, 0, 0)
    assert O.rel_fro(got, want) <= 1e-5
