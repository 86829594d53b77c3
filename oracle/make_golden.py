# SPDX-License-Identifier: Apache-2.0
"""TEST INFRASTRUCTURE ONLY: regenerates tests/golden/ by running the
UNMODIFIED reference library (oracle/_ref/libgmref.so, built from
/root/reference/proj by oracle/Makefile) on small seeded cases.

    make -C oracle && python oracle/make_golden.py

The reference's own tests never pin GEMM numerics (tests/test_core.cpp has
no GEMM case and its CMake test target is a placeholder), so the golden
results come from the reference itself, through its public API
(Session/createMatrix/setData/gemm/getDataRaw). Cases mirror the spec's GEMM
examples and the survey's layout-invariance probes.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import oracle as O  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")

H, S, D, B = 0, 1, 2, 3


def irregular_tiles(rows, cols, p):
    """3x3 irregular tiles dealt round-robin over p workers."""
    rcuts = [0, rows // 5, rows // 2, rows]
    ccuts = [0, cols // 3, (3 * cols) // 4, cols]
    tiles, w = [], 0
    for i in range(3):
        for j in range(3):
            tiles.append((rcuts[i], rcuts[i + 1] - rcuts[i], ccuts[j], ccuts[j + 1] - ccuts[j], w % p))
            w += 1
    return tiles


def layouts_for(kind, rows, cols, p):
    if kind == "single":
        return [(0, rows, 0, cols, p - 1)]
    if kind == "row":
        return O.row_block_tiles(rows, cols, p)
    if kind == "col":
        return O.col_block_tiles(rows, cols, p)
    if kind == "grid":
        pr = {1: 1, 2: 1, 3: 1, 4: 2, 8: 2}[p]
        return O.grid_tiles(rows, cols, pr, p // pr)
    if kind == "irregular":
        return irregular_tiles(rows, cols, p)
    raise ValueError(kind)


def bf16_representable(img_f32: np.ndarray) -> np.ndarray:
    """Round a float32 image to bf16 (RNE) but keep it stored as Single."""
    u = img_f32.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


CASES = []


def case(name, m, n, k, pa, pb, pc, p, la, lb, lc, alpha=1.0, beta=0.0, ta=0, tb=0,
         repl=0, det=True, bf16=False, special=None):
    CASES.append(dict(name=name, m=m, n=n, k=k, pa=pa, pb=pb, pc=pc, p=p, la=la, lb=lb, lc=lc,
                      alpha=alpha, beta=beta, ta=ta, tb=tb, repl=repl, det=det, bf16=bf16,
                      special=special))


def build_cases():
    # random 64x48 . 48x32 over P in {1,2,4}, five layout pairs.
    pairs = [("single", "single", "single"), ("row", "col", "grid"), ("grid", "grid", "grid"),
             ("col", "row", "grid"), ("row", "row", "row")]
    for p in (1, 2, 4):
        for (la, lb, lc) in pairs:
            case(f"spec_f32_p{p}_{la}_{lb}_{lc}", 64, 32, 48, S, S, S, p, la, lb, lc)
    # Survey section 4 probes (reduced to 96x80x72): alpha=.75 beta=.5, deterministic.
    for p, (la, lb, lc) in [(1, ("single",) * 3), (2, ("row", "col", "grid")), (4, ("grid",) * 3),
                            (4, ("col", "row", "grid")), (3, ("irregular",) * 3),
                            (8, ("row", "col", "col"))]:
        case(f"probe_f32_p{p}_{la}_{lb}_{lc}", 96, 80, 72, S, S, S, p, la, lb, lc, 0.75, 0.5)
    # Transposes (reference kernels.cpp:209-216, :515-516).
    for ta, tb in [(1, 0), (0, 1), (1, 1)]:
        case(f"trans_f32_{ta}{tb}", 80, 64, 56, S, S, S, 4, "grid", "grid", "row", 1.0, 0.0, ta, tb)
        case(f"trans_f64_{ta}{tb}", 80, 64, 56, D, D, D, 2, "row", "col", "grid", 0.5, 2.0, ta, tb)
    # Precisions / mixed mode (kernels.cpp:136-140; precision.hpp).
    case("half_half_single", 128, 96, 160, H, H, S, 4, "row", "col", "grid")
    case("half_all", 128, 96, 160, H, H, H, 2, "grid", "grid", "grid", 1.0, 0.25)
    case("half_single_double", 96, 64, 80, H, S, D, 4, "row", "col", "grid")
    case("f64_all", 96, 112, 128, D, D, D, 8, "grid", "grid", "grid", 0.75, 0.5)
    case("bf16_as_single", 128, 128, 192, S, S, S, 4, "grid", "grid", "grid", bf16=True)
    case("bf16_as_single_p1", 256, 192, 320, S, S, S, 1, "single", "single", "single", bf16=True)
    # Semantics: A = I -> C = B ; alpha = 0, beta = 1 -> C unchanged.
    case("identity", 48, 40, 48, S, S, S, 4, "grid", "row", "col", special="identity")
    case("alpha0_beta1", 40, 56, 24, S, S, S, 2, "row", "col", "grid", 0.0, 1.0, special="nan_ab")
    case("beta0_nan_c", 40, 56, 24, S, S, S, 2, "row", "col", "grid", 1.0, 0.0, special="nan_c")
    # Replica read path (pieces.cpp:20, worker.cpp:245-448).
    case("replica_b", 64, 96, 80, S, S, S, 4, "row", "col", "row", repl=2)
    case("replica_ab", 64, 96, 80, H, H, S, 4, "col", "col", "row", repl=3)
    # Fast (non-deterministic) mode, numerically close.
    case("fast_mode", 96, 80, 72, S, S, S, 4, "grid", "grid", "grid", det=False)
    # C1 shape class at reduced size (2x2 grid, fp32).
    case("c1_like_256", 256, 256, 256, S, S, S, 4, "grid", "grid", "grid")


FC_CASES = []


def fc_case(name, op, sub, p, shape, xp, lx, yp=None, ly=None, dp=None, ld=None, alpha=0.0, repl=0,
            special=None):
    FC_CASES.append(dict(name=name, op=op, sub=sub, p=p, rows=shape[0], cols=shape[1], xp=xp, lx=lx, yp=yp,
                         ly=ly, dp=dp, ld=ld, alpha=alpha, repl=repl, special=special))


def build_fc_cases():
    # FC-layer neighbours (reference session.cpp:547-609).
    sh = (67, 45)
    fc_case("relu_f32_grid_to_row", 0, 0, 4, sh, S, "grid", dp=S, ld="row", special="specials")
    fc_case("relu_half_p2", 0, 0, 2, sh, H, "row", dp=H, ld="row")
    fc_case("relu_f64_irregular", 0, 0, 3, sh, D, "irregular", dp=D, ld="col")
    fc_case("mulscalar_f32", 0, 1, 4, sh, S, "grid", alpha=0.3)
    fc_case("mulscalar_half", 0, 1, 2, sh, H, "col", alpha=-1.7)
    fc_case("add_f32_mixed_layouts", 1, 0, 4, sh, S, "grid", S, "row", S, "col")
    fc_case("sub_half_single_to_half", 1, 1, 3, sh, H, "irregular", S, "grid", H, "row")
    fc_case("add_f64", 1, 0, 2, sh, D, "row", S, "col", D, "grid")
    fc_case("axpy_f32", 1, 2, 4, sh, S, "grid", S, "grid", alpha=-0.01)
    fc_case("axpy_f64_mixed", 1, 2, 3, sh, S, "row", D, "col", alpha=0.125)
    fc_case("relugrad_f32", 1, 3, 4, sh, S, "grid", S, "grid", special="specials")
    fc_case("relugrad_half", 1, 3, 2, sh, H, "row", H, "col")
    fc_case("copy_single_to_half", 1, 4, 4, sh, S, "grid", dp=H, ld="row")
    fc_case("copy_double_to_single", 1, 4, 2, sh, D, "col", dp=S, ld="grid")
    fc_case("copy_half_to_double", 1, 4, 3, sh, H, "row", dp=D, ld="irregular")
    fc_case("biasadd_f32_row", 1, 5, 4, sh, S, "row", S, "col")
    fc_case("biasadd_f32_replicated", 1, 5, 4, sh, S, "row", S, "col", repl=2)
    fc_case("biasadd_half_bias_grid_x", 1, 5, 4, sh, S, "grid", H, "single")
    fc_case("rowcolsum_det_f32", 2, 1, 4, sh, S, "grid", S, "row", S, "col", alpha=1.0)
    fc_case("rowcolsum_det_f64", 2, 1, 3, sh, D, "irregular", D, "row", S, "col", alpha=-0.5)
    fc_case("rowcolsum_det_half", 2, 1, 2, sh, H, "row", S, "row", H, "col", alpha=0.25)
    fc_case("rowcolsum_fast_f32", 2, 0, 4, sh, S, "grid", S, "row", S, "col", alpha=1.0)
    fc_case("setconst_f32_zero", 3, 0, 4, sh, S, "grid", alpha=0.0)
    fc_case("setconst_half_overflow", 3, 0, 2, sh, H, "row", alpha=65520.0)
    fc_case("setconst_f64_pi", 3, 0, 3, sh, D, "irregular", alpha=3.141592653589793)
    fc_case("setconst_bf16_via_single", 3, 0, 4, sh, S, "col", alpha=1.0 / 3.0)


def run_fc_case(c):
    rows, cols = c["rows"], c["cols"]
    op, sub = c["op"], c["sub"]
    x = O.fill_uniform(rows, cols, c["xp"], 11)
    if c["special"] == "specials":
        flat = x.reshape(-1)
        flat[:6] = np.array([np.nan, np.inf, -np.inf, -0.0, 0.0, -1e-30], dtype=flat.dtype)
    xt = layouts_for(c["lx"], rows, cols, c["p"])
    y = d = None
    yt = dt = []
    if op == 1 and sub == 5:
        y = O.fill_uniform(1, cols, c["yp"], 12)
        yt = layouts_for(c["ly"], 1, cols, c["p"])
    elif op == 2:
        y = O.fill_uniform(rows, 1, c["yp"], 12)
        yt = layouts_for(c["ly"], rows, 1, c["p"])
        d = O.fill_uniform(1, cols, c["dp"], 13)
        dt = layouts_for(c["ld"], 1, cols, c["p"])
    elif c["yp"] is not None:
        y = O.fill_uniform(rows, cols, c["yp"], 12)
        yt = layouts_for(c["ly"], rows, cols, c["p"])
    if op in (0, 1) and c["dp"] is not None:
        d = O.fill_uniform(rows, cols, c["dp"], 13)
        dt = layouts_for(c["ld"], rows, cols, c["p"])
    yp = 1 if c["yp"] is None else c["yp"]
    dp = 1 if c["dp"] is None else c["dp"]
    res = O.fcop_ref(c["p"], op, sub, c["alpha"], x, c["xp"], xt, y, yp, yt, d, dp, dt, c["repl"])
    out0, out1 = res if op == 2 else (res, np.zeros(1))
    arr = dict(x=x, out0=out0, out1=out1, xt=np.array(xt, dtype=np.uint64))
    if y is not None:
        arr.update(y=y, yt=np.array(yt, dtype=np.uint64))
    if d is not None:
        arr.update(d=d, dt=np.array(dt, dtype=np.uint64))
    return arr


def run_case(c):
    m, n, k = c["m"], c["n"], c["k"]
    ar, ac = (k, m) if c["ta"] else (m, k)
    br, bc = (n, k) if c["tb"] else (k, n)
    a = O.fill_uniform(ar, ac, c["pa"], 1)
    b = O.fill_uniform(br, bc, c["pb"], 2)
    cc = O.fill_uniform(m, n, c["pc"], 3)
    if c["bf16"]:
        a = bf16_representable(a)
        b = bf16_representable(b)
    if c["special"] == "identity":
        a = np.eye(m, k, dtype=np.float32)
    if c["special"] == "nan_ab":
        a[:] = np.nan
        b[:] = np.nan
    if c["special"] == "nan_c":
        cc[:] = np.nan
    at = layouts_for(c["la"], ar, ac, c["p"])
    bt = layouts_for(c["lb"], br, bc, c["p"])
    ct = layouts_for(c["lc"], m, n, c["p"])
    out, _ = O.gemm_ref(c["p"], a, c["pa"], at, b, c["pb"], bt, cc, c["pc"], ct, c["alpha"],
                        c["beta"], c["ta"], c["tb"], c["det"], c["repl"])
    return dict(a=a, b=b, c=cc, out=out, at=np.array(at, dtype=np.uint64),
                bt=np.array(bt, dtype=np.uint64), ct=np.array(ct, dtype=np.uint64))


def main():
    os.makedirs(OUT, exist_ok=True)
    build_cases()
    index = []
    for c in CASES:
        arrays = run_case(c)
        np.savez_compressed(os.path.join(OUT, c["name"] + ".npz"), **arrays)
        index.append({k: v for k, v in c.items()})
        print("golden", c["name"])
    build_fc_cases()
    fc_index = []
    for c in FC_CASES:
        np.savez_compressed(os.path.join(OUT, "fc_" + c["name"] + ".npz"), **run_fc_case(c))
        fc_index.append(dict(c))
        print("golden fc", c["name"])
    # Layout vectors from the reference constructors (layout.cpp:13-75).
    lay = []
    for kind in (0, 1):
        for p in (1, 2, 3, 5, 8):
            for rows, cols in ((4, 4), (5, 3), (1, 7), (16, 11), (2, 9)):
                lay.append(dict(kind=kind, rows=rows, cols=cols, pr=p, pc=1,
                                tiles=[list(map(int, t)) for t in O.ref_layout(kind, rows, cols, p)]))
    for pr, pc in ((1, 1), (2, 2), (1, 3), (2, 4), (3, 2)):
        for rows, cols in ((4, 4), (5, 5), (3, 3), (17, 13), (1, 8)):
            lay.append(dict(kind=2, rows=rows, cols=cols, pr=pr, pc=pc,
                            tiles=[list(map(int, t)) for t in O.ref_layout(2, rows, cols, pr, pc)]))
    # Descriptor encodings (descriptor.cpp:6-20).
    import ctypes
    desc = []
    for (mid, rows, cols, prec, ver, p) in ((1, 4, 4, 1, 0, 2), (7, 33, 5, 0, 9, 3),
                                            (2**40 + 3, 1, 17, 2, 123456789, 1)):
        tiles = O.row_block_tiles(rows, cols, p)
        buf = (ctypes.c_uint8 * 4096)()
        ln = ctypes.c_uint32(0)
        O.reflib().gmref_encode_descriptor(mid, rows, cols, prec, ver, O.tiles_array(tiles),
                                           len(tiles), buf, 4096, ctypes.byref(ln))
        desc.append(dict(id=mid, rows=rows, cols=cols, prec=prec, version=ver,
                         tiles=[list(map(int, t)) for t in tiles], hex=bytes(buf[: ln.value]).hex()))
    # fp16 codec vectors (precision.hpp:42-100), like test_core.cpp:155-189.
    rng = np.random.default_rng(13)
    f = np.concatenate([rng.uniform(-70000, 70000, 4000), rng.uniform(-2, 2, 4000),
                        rng.uniform(-1e-4, 1e-4, 4000), rng.uniform(-1e-7, 1e-7, 1000),
                        np.array([0.0, -0.0, 1.0, 65504.0, 65519.99, 65520.0, -65520.0, 1e30,
                                  np.inf, -np.inf, 5.960464477539063e-08, 2.98e-08, 6.1e-05])]
                       ).astype(np.float32)
    h = np.empty(f.shape, dtype=np.uint16)
    O.reflib().gmref_float_to_half(f.ctypes.data, h.ctypes.data, f.size)
    allh = np.arange(65536, dtype=np.uint16)
    back = np.empty(allh.shape, dtype=np.float32)
    O.reflib().gmref_half_to_float(allh.ctypes.data, back.ctypes.data, allh.size)
    np.savez_compressed(os.path.join(OUT, "fp16_codec.npz"), f=f, h=h, all_h=allh, all_f=back)
    with open(os.path.join(OUT, "index.json"), "w") as fh:
        json.dump(dict(cases=index, fc_cases=fc_index, layouts=lay, descriptors=desc,
                       generator="oracle/make_golden.py over oracle/_ref/libgmref.so"), fh, indent=1)
    print("wrote", len(index), "gemm cases,", len(fc_index), "fc cases,", len(lay), "layouts,", len(desc),
          "descriptors")


if __name__ == "__main__":
    main()
