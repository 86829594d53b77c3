# SPDX-License-Identifier: Apache-2.0
"""CPU tests of the drop-in's host logic through the C ABI (no GPU needed):
ABI surface, layouts (ported from reference tests/test_core.cpp:29-127),
descriptor wire bytes (test_core.cpp:129-153), storage conversions, and the
GEMM data-movement plan against the reference planGemm byte oracle."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

import oracle as O
from conftest import ROOT
from paper_1611_07819_b200 import _lib
from paper_1611_07819_b200 import gridmath as G

HEADER = os.path.join(ROOT, "include", "gridmath_b200.h")


def header_symbols():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|void|const char\*)\s+(gm_\w+)\s*\(", txt, re.M)))


def test_library_exports_every_header_symbol():
    syms = header_symbols()
    assert len(syms) >= 40
    out = subprocess.check_output(["nm", "-D", "--defined-only", _lib.LIB_PATH]).decode()
    exported = set(re.findall(r" T (gm_\w+)", out))
    missing = [s for s in syms if s not in exported]
    assert not missing, missing
    assert set(syms) <= set(_lib.EXPORTED) | {"gm_last_error"}
    lib = _lib.load()
    for s in syms:
        getattr(lib, s)


def test_layouts_match_reference_golden(golden_index):
    for L in golden_index["layouts"]:
        if L["kind"] == 0:
            got = G.makeRowBlockLayout(L["rows"], L["cols"], G.makeWorkerGroup(L["pr"]))
        elif L["kind"] == 1:
            got = G.makeColBlockLayout(L["rows"], L["cols"], G.makeWorkerGroup(L["pr"]))
        else:
            got = G.makeGridLayout(L["rows"], L["cols"], L["pr"], L["pc"], G.makeWorkerGroup(L["pr"] * L["pc"]))
        assert [list(t) for t in got.as_tuples()] == L["tiles"], L


def _cover(rows, cols, layout):
    owners = np.zeros((rows, cols), dtype=np.int32)
    for e, _ in layout.tiles:
        owners[e.rowStart:e.rowStart + e.rowCount, e.colStart:e.colStart + e.colCount] += 1
    return owners


def test_generated_layouts_cover_exactly_once():
    # test_core.cpp:107-127
    for p in range(1, 9):
        for rows in range(1, 17, 3):
            for cols in range(1, 17, 5):
                for lay in (G.makeRowBlockLayout(rows, cols, G.makeWorkerGroup(p)),
                            G.makeColBlockLayout(rows, cols, G.makeWorkerGroup(p))):
                    assert (_cover(rows, cols, lay) == 1).all()
                if p == 4:
                    assert (_cover(rows, cols, G.makeGridLayout(rows, cols, 2, 2, G.makeWorkerGroup(4))) == 1).all()
                if p == 8:
                    assert (_cover(rows, cols, G.makeGridLayout(rows, cols, 2, 4, G.makeWorkerGroup(8))) == 1).all()


def test_row_block_remainder_and_errors():
    # test_core.cpp:29-49
    l = G.makeRowBlockLayout(5, 3, G.makeWorkerGroup(2))
    assert [e.rowCount for e, _ in l.tiles] == [3, 2]
    with pytest.raises(G.GmError):
        G.makeRowBlockLayout(4, 4, [])
    with pytest.raises(G.GmError):
        G.makeGridLayout(4, 4, 2, 2, G.makeWorkerGroup(3))


def test_validate_layout_reports_first_violation():
    # test_core.cpp:63-93
    T = G.TileExtent
    assert G.validateLayout(3, 3, G.makeSingleTileLayout(3, 3, 0)) == 0
    assert G.validateLayout(2, 3, G.Layout([(T(0, 1, 0, 3), 0), (T(0, 2, 0, 3), 1)])) == 1
    assert G.validateLayout(4, 3, G.Layout([(T(0, 2, 0, 3), 0)])) == 2
    assert G.validateLayout(4, 3, G.Layout([(T(0, 5, 0, 3), 0)])) == 3
    assert G.validateLayout(2, 2, G.makeSingleTileLayout(2, 2, 7), 4) == 4
    assert G.validateLayout(2, 2, G.makeSingleTileLayout(2, 2, 7)) == 0


def test_descriptor_encoding_matches_reference_bytes(golden_index):
    lib = _lib.load()
    for d in golden_index["descriptors"]:
        lay = G.Layout([(G.TileExtent(*t[:4]), t[4]) for t in d["tiles"]])
        buf = (ctypes.c_uint8 * 4096)()
        n = ctypes.c_uint32()
        _lib.check(lib.gm_descriptor_encode(d["id"], d["rows"], d["cols"], d["prec"], d["version"],
                                            lay.as_c(), len(lay.tiles), buf, 4096, ctypes.byref(n)))
        assert bytes(buf[: n.value]).hex() == d["hex"]


def _convert_host(arr, sp, dp, out_dtype):
    out = np.empty(arr.size, dtype=out_dtype)
    a = np.ascontiguousarray(arr)
    _lib.check(_lib.load().gm_convert_host(a.ctypes.data, sp, out.ctypes.data, dp, a.size))
    return out


def test_host_fp16_rounding_matches_reference():
    d = np.load(os.path.join(ROOT, "tests", "golden", "fp16_codec.npz"))
    got = _convert_host(d["f"], 1, 0, np.uint16)
    assert np.array_equal(got, d["h"])
    # Widening is IEEE-exact (differs from the reference only on subnormals,
    # where the reference is off by a factor of two: DESIGN.md).
    back = _convert_host(d["all_h"], 0, 1, np.float32)
    ieee = d["all_h"].view(np.float16).astype(np.float32)
    fin = np.isfinite(ieee)
    assert np.array_equal(back[fin], ieee[fin])


def test_host_bf16_rounding_is_rne():
    rng = np.random.default_rng(5)
    f = rng.standard_normal(20000).astype(np.float32) * 100
    got = _convert_host(f, 1, 3, np.uint16)
    u = f.view(np.uint32).astype(np.uint64)
    want = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
    assert np.array_equal(got, want)


def plan(workers, a, b, c, ta=0, tb=0, a_repl=0, b_repl=0, prec=(1, 1, 1)):
    """a/b/c: (rows, cols, layout)."""
    lib = _lib.load()
    cap = 1 << 16
    out = (_lib.gm_plan_piece * cap)()
    n = ctypes.c_uint32()
    rb = (ctypes.c_uint64 * workers)()
    _lib.check(lib.gm_plan_gemm(workers, a[0], a[1], prec[0], a[2].as_c(), len(a[2].tiles),
                                b[0], b[1], prec[1], b[2].as_c(), len(b[2].tiles),
                                c[0], c[1], prec[2], c[2].as_c(), len(c[2].tiles),
                                ta, tb, a_repl, b_repl, out, cap, ctypes.byref(n), rb))
    return [(p.src, p.dst, p.operand, p.r0, p.r1, p.c0, p.c1) for p in out[: n.value]], list(rb)


@pytest.mark.parametrize("p,pr,pc", [(1, 1, 1), (2, 1, 2), (4, 2, 2), (8, 2, 4)])
def test_plan_remote_bytes_equal_reference_plan(p, pr, pc):
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    n = 2048
    lay = lambda: G.makeGridLayout(n, n, pr, pc, G.makeWorkerGroup(p))
    pieces, rb = plan(p, (n, n, lay()), (n, n, lay()), (n, n, lay()), prec=(3, 3, 3))
    t = lay().as_tuples()
    ref = O.plan_remote_bytes(p, (n, n), 0, t, (n, n), 0, t, (n, n), 0, t)  # Half = 2 bytes like bf16
    assert rb == ref
    if p > 1:
        # SUMMA closed form: e * [(m/pr) k (pc-1)/pc + k (n/pc) (pr-1)/pr]
        assert rb[0] == 2 * ((n // pr) * n * (pc - 1) // pc + n * (n // pc) * (pr - 1) // pr)


def test_plan_irregular_layouts_match_reference_and_cover_needs():
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    from make_golden import irregular_tiles
    m, n, k, p = 96, 80, 72, 3
    A = G.Layout([(G.TileExtent(*t[:4]), t[4]) for t in irregular_tiles(m, k, p)])
    B = G.makeColBlockLayout(k, n, G.makeWorkerGroup(p))
    C = G.makeRowBlockLayout(m, n, G.makeWorkerGroup(p))
    for ta, tb in ((0, 0),):
        pieces, rb = plan(p, (m, k, A), (k, n, B), (m, n, C), ta, tb)
        ref = O.plan_remote_bytes(p, (m, k), 1, A.as_tuples(), (k, n), 1, B.as_tuples(), (m, n), 1, C.as_tuples())
        assert rb == ref
        # every element of each consumer's A band arrives exactly once
        for w in range(p):
            cov = np.zeros((m, k), dtype=np.int32)
            for (src, dst, op, r0, r1, c0, c1) in pieces:
                if dst == w and op == 0:
                    cov[r0:r1, c0:c1] += 1
            rows = [e for e, o in C.tiles if o == w]
            for e in rows:
                assert (cov[e.rowStart:e.rowStart + e.rowCount, :] == 1).all()


def test_plan_with_replicas_moves_nothing():
    n, p = 512, 4
    lay = G.makeRowBlockLayout(n, n, G.makeWorkerGroup(p))
    W = G.makeColBlockLayout(n, n, G.makeWorkerGroup(p))
    pieces, rb = plan(p, (n, n, lay), (n, n, W), (n, n, lay), b_repl=1)
    assert rb == [0] * p
    assert all(op == 0 for (_, _, op, *_r) in pieces)  # only local A slices (none here: A rows are local)


def test_session_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(G.GmError):
        G.Session(workers=1)


def test_library_then_torch_import_order():
    """The library must not pull an older libnccl.so.2 into the process ahead
    of torch's (same SONAME: the first one loaded wins, and torch then fails
    to import with undefined NCCL symbols)."""
    import subprocess
    import sys
    code = ("import sys; sys.path.insert(0, %r)\n"
            "from paper_1611_07819_b200 import _lib; _lib.load()\n"
            "import torch, torch.distributed\n"
            "print('ok')\n") % ROOT
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-2000:]
