# SPDX-License-Identifier: Apache-2.0
"""TEST INFRASTRUCTURE ONLY -- the parity checker, never the product.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this module.

Two CPU implementations of the reference's GEMM path:

* ``RefLib`` -- the UNMODIFIED reference library (dMath re-creation,
  /root/reference/proj), compiled from its own sources into
  oracle/_ref/libgmref.so by oracle/Makefile and driven through its public
  Session / createMatrix / setData / gemm / getDataRaw API
  (oracle/ref_harness.cpp).
* ``CLib`` -- oracle/gemm_oracle.c, the plain-C restatement of runGemm<T>
  (reference src/kernels.cpp:445-558), of the FC-layer neighbours
  (runElementwise :741-815, runRowColSumDet :570-614, execSetConst :435-443)
  and of the fp16 codec (include/gridmath/precision.hpp:42-100). Pinned
  bit-for-bit against the reference by tests/test_oracle.py and tests/golden/.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_double, c_int32, c_size_t, c_uint16, c_uint32, c_uint64, c_void_p

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libgmref.so")
C_SO = os.path.join(HERE, "_build", "liboracle.so")

NP_DTYPE = {0: np.uint16, 1: np.float32, 2: np.float64, 3: np.uint16}  # storage containers


class HTile(ctypes.Structure):
    _fields_ = [("row_start", c_uint64), ("row_count", c_uint64), ("col_start", c_uint64),
                ("col_count", c_uint64), ("owner", c_uint32)]


def tiles_array(tiles):
    arr = (HTile * max(1, len(tiles)))()
    for i, t in enumerate(tiles):
        arr[i] = HTile(*t)
    return arr


_c = None
_ref = None


def clib():
    global _c
    if _c is None:
        if not os.path.exists(C_SO):
            raise RuntimeError(f"{C_SO} missing: run `make -C {HERE}`")
        lib = ctypes.CDLL(C_SO)
        lib.oracle_float_to_half.argtypes = [ctypes.c_float]
        lib.oracle_float_to_half.restype = c_uint16
        lib.oracle_half_to_float.argtypes = [c_uint16]
        lib.oracle_half_to_float.restype = ctypes.c_float
        lib.oracle_gemm.argtypes = [c_uint64, c_uint64, c_uint64, c_void_p, c_int32, c_void_p,
                                    c_int32, c_void_p, c_int32, c_double, c_double, c_int32,
                                    c_int32, c_uint64, c_uint64]
        lib.oracle_fill_uniform.argtypes = [c_void_p, c_int32, c_uint64, c_uint64, c_uint64,
                                            c_double, c_double]
        lib.oracle_split.argtypes = [c_uint64, c_uint64, POINTER(c_uint64), POINTER(c_uint64)]
        lib.oracle_split.restype = c_uint32
        lib.oracle_elementwise.argtypes = [c_int32, c_int32, c_double, c_uint64, c_uint64, c_void_p,
                                           c_int32, c_void_p, c_int32, c_void_p, c_int32]
        lib.oracle_row_col_sum.argtypes = [c_double, c_uint64, c_uint64, c_void_p, c_int32, c_void_p,
                                           c_int32, c_void_p, c_int32]
        lib.oracle_set_const.argtypes = [c_void_p, c_int32, c_uint64, c_double]
        _c = lib
    return _c


def reflib():
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            raise RuntimeError(f"{REF_SO} missing: run `make -C {HERE}` where /root/reference exists")
        lib = ctypes.CDLL(REF_SO)
        T = POINTER(HTile)
        lib.gmref_gemm.argtypes = [c_uint32, c_int32,
                                   c_uint64, c_uint64, c_int32, T, c_uint32, c_void_p,
                                   c_uint64, c_uint64, c_int32, T, c_uint32, c_void_p,
                                   c_uint64, c_uint64, c_int32, T, c_uint32, c_void_p,
                                   c_double, c_double, c_int32, c_int32, c_int32, c_void_p,
                                   POINTER(c_double), c_char_p, c_size_t]
        lib.gmref_plan_remote_bytes.argtypes = [c_uint32,
                                                c_uint64, c_uint64, c_int32, T, c_uint32,
                                                c_uint64, c_uint64, c_int32, T, c_uint32,
                                                c_uint64, c_uint64, c_int32, T, c_uint32,
                                                c_int32, c_int32, POINTER(c_uint64), c_char_p,
                                                c_size_t]
        lib.gmref_layout.argtypes = [c_int32, c_uint64, c_uint64, c_uint32, c_uint32, T, c_uint32,
                                     POINTER(c_uint32), c_char_p, c_size_t]
        lib.gmref_encode_descriptor.argtypes = [c_uint64, c_uint64, c_uint64, c_int32, c_uint64, T,
                                                c_uint32, POINTER(ctypes.c_uint8), c_uint32,
                                                POINTER(c_uint32)]
        lib.gmref_fcop.argtypes = [c_uint32, c_int32, c_int32, c_double,
                                   c_uint64, c_uint64, c_int32, T, c_uint32, c_void_p,
                                   c_uint64, c_uint64, c_int32, T, c_uint32, c_void_p,
                                   c_uint64, c_uint64, c_int32, T, c_uint32, c_void_p,
                                   c_int32, c_void_p, c_void_p, c_char_p, c_size_t]
        lib.gmref_ckpt_write.argtypes = [c_uint32, c_uint32, POINTER(c_uint64), POINTER(c_uint64), POINTER(c_int32),
                                         POINTER(T), POINTER(c_uint32), POINTER(c_void_p), c_double, c_char_p,
                                         c_char_p, c_size_t]
        lib.gmref_ckpt_read.argtypes = [c_char_p, c_uint32, c_uint32, POINTER(c_uint64), POINTER(c_void_p),
                                        POINTER(c_uint64), c_char_p, c_size_t]
        lib.gmref_float_to_half.argtypes = [c_void_p, c_void_p, c_uint64]
        lib.gmref_half_to_float.argtypes = [c_void_p, c_void_p, c_uint64]
        _ref = lib
    return _ref


def ref_available() -> bool:
    return os.path.exists(REF_SO)


# ---------------------------------------------------------------- helpers

def fill_uniform(rows, cols, prec, seed, lo=-1.0, hi=1.0) -> np.ndarray:
    """SplitMix64(seed) U[lo,hi) rounded to storage `prec` (row-major image)."""
    out = np.empty(rows * cols, dtype=NP_DTYPE[prec])
    clib().oracle_fill_uniform(out.ctypes.data, prec, rows, cols, seed, lo, hi)
    return out.reshape(rows, cols)


def to_f64(img: np.ndarray, prec: int) -> np.ndarray:
    if prec in (1, 2):
        return img.astype(np.float64)
    if prec == 3:
        return (img.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    return img.view(np.float16).astype(np.float64)  # IEEE binary16, exact


def gemm_c(m, n, k, a, pa, b, pb, c, pc, alpha, beta, ta, tb, rows=None) -> np.ndarray:
    """C restatement; returns a new C image (rows [r0, r1) updated if given)."""
    out = np.ascontiguousarray(c).copy()
    r0, r1 = rows if rows is not None else (0, m)
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b)
    clib().oracle_gemm(m, n, k, a.ctypes.data, pa, b.ctypes.data, pb, out.ctypes.data, pc,
                       alpha, beta, ta, tb, r0, r1)
    return out


def gemm_ref(workers, a, pa, a_tiles, b, pb, b_tiles, c, pc, c_tiles, alpha, beta, ta, tb,
             deterministic=True, replicate_mask=0):
    """Runs the unmodified reference Session/gemm. Returns (C image, seconds)."""
    lib = reflib()
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b)
    c = np.ascontiguousarray(c)
    out = np.empty_like(c)
    err = ctypes.create_string_buffer(512)
    secs = c_double(0.0)
    rc = lib.gmref_gemm(workers, 1 if deterministic else 0,
                        a.shape[0], a.shape[1], pa, tiles_array(a_tiles), len(a_tiles), a.ctypes.data,
                        b.shape[0], b.shape[1], pb, tiles_array(b_tiles), len(b_tiles), b.ctypes.data,
                        c.shape[0], c.shape[1], pc, tiles_array(c_tiles), len(c_tiles), c.ctypes.data,
                        alpha, beta, ta, tb, replicate_mask, out.ctypes.data, ctypes.byref(secs),
                        err, 512)
    if rc:
        raise RuntimeError("reference gemm failed: " + err.value.decode())
    return out, secs.value


# ---------------------------------------------------------------- FC-layer neighbours
# op codes shared with oracle/ref_harness.cpp gmref_fcop: 0 EwUnary (kind 0 relu,
# 1 mulScalar), 1 EwBinary (0 add, 1 sub, 2 axpy, 3 reluGrad, 4 copy, 5 biasAdd),
# 2 addRowColSum, 3 setConst.

def ew_c(unary, kind, alpha, x, xp, y, yp, dst, dp):
    """C restatement of one elementwise op; returns the new dst image (dst is
    only used for its shape/precision; aliasing is the caller's choice of x/y)."""
    x = np.ascontiguousarray(x)
    y = np.ascontiguousarray(y) if y is not None else None
    out = np.ascontiguousarray(dst).copy()
    clib().oracle_elementwise(1 if unary else 0, kind, alpha, out.shape[0], out.shape[1], x.ctypes.data, xp,
                              y.ctypes.data if y is not None else None, yp if y is not None else 1,
                              out.ctypes.data, dp)
    return out


def rowcolsum_c(alpha, a, ap, racc, rp, cacc, cp):
    a = np.ascontiguousarray(a)
    r = np.ascontiguousarray(racc).copy()
    c = np.ascontiguousarray(cacc).copy()
    clib().oracle_row_col_sum(alpha, a.shape[0], a.shape[1], a.ctypes.data, ap, r.ctypes.data, rp,
                              c.ctypes.data, cp)
    return r, c


def set_const_c(shape, prec, value):
    out = np.empty(shape, dtype=NP_DTYPE[prec])
    clib().oracle_set_const(out.ctypes.data, prec, out.size, value)
    return out


def fcop_ref(workers, op, sub, alpha, x, xp, x_tiles, y=None, yp=1, y_tiles=(), d=None, dp=1, d_tiles=(),
             replicate_mask=0):
    """Runs one FC-layer neighbour through the unmodified reference Session.
    Returns the result image (op 2: (rowAcc, colAcc))."""
    lib = reflib()
    x = np.ascontiguousarray(x)
    y = np.ascontiguousarray(y) if y is not None else None
    d = np.ascontiguousarray(d) if d is not None else None
    if op == 0:
        out0 = np.empty_like(d if sub == 0 else x)
    elif op == 1:
        out0 = np.empty_like({2: y, 3: y, 5: x}.get(sub, d))
    elif op == 2:
        out0 = np.empty_like(y)
    else:
        out0 = np.empty_like(x)
    out1 = np.empty_like(d) if op == 2 else np.empty(1, np.uint8)
    err = ctypes.create_string_buffer(512)
    yr, yc = (y.shape if y is not None else (0, 0))
    dr, dc = (d.shape if d is not None else (0, 0))
    rc = lib.gmref_fcop(workers, op, sub, alpha,
                        x.shape[0], x.shape[1], xp, tiles_array(x_tiles), len(x_tiles), x.ctypes.data,
                        yr, yc, yp, tiles_array(list(y_tiles)), len(y_tiles), y.ctypes.data if y is not None else None,
                        dr, dc, dp, tiles_array(list(d_tiles)), len(d_tiles), d.ctypes.data if d is not None else None,
                        replicate_mask, out0.ctypes.data, out1.ctypes.data, err, 512)
    if rc:
        raise RuntimeError("reference op failed: " + err.value.decode())
    return (out0, out1) if op == 2 else out0


def plan_remote_bytes(workers, a_shape, pa, a_tiles, b_shape, pb, b_tiles, c_shape, pc, c_tiles,
                      ta=0, tb=0):
    lib = reflib()
    out = (c_uint64 * workers)()
    err = ctypes.create_string_buffer(512)
    rc = lib.gmref_plan_remote_bytes(workers, a_shape[0], a_shape[1], pa, tiles_array(a_tiles),
                                     len(a_tiles), b_shape[0], b_shape[1], pb,
                                     tiles_array(b_tiles), len(b_tiles), c_shape[0], c_shape[1],
                                     pc, tiles_array(c_tiles), len(c_tiles), ta, tb, out, err, 512)
    if rc:
        raise RuntimeError(err.value.decode())
    return list(out)


def ref_layout(kind, rows, cols, pr, pc=1):
    """kind 0 row-block (pr workers), 1 col-block (pr workers), 2 grid pr x pc."""
    lib = reflib()
    cap = 4096
    arr = (HTile * cap)()
    n = c_uint32(0)
    err = ctypes.create_string_buffer(256)
    rc = lib.gmref_layout(kind, rows, cols, pr, pc, arr, cap, ctypes.byref(n), err, 256)
    if rc:
        raise RuntimeError(err.value.decode())
    return [(t.row_start, t.row_count, t.col_start, t.col_count, t.owner) for t in arr[: n.value]]


def split(n, parts):
    starts = (c_uint64 * max(1, parts))()
    lens = (c_uint64 * max(1, parts))()
    cnt = clib().oracle_split(n, parts, starts, lens)
    return [(starts[i], lens[i]) for i in range(cnt)]


def grid_tiles(rows, cols, pr, pc):
    """C restatement of makeGridLayout (layout.cpp:61-75)."""
    rb, cb = split(rows, pr), split(cols, pc)
    return [(r0, rl, c0, cl, r * pc + c) for r, (r0, rl) in enumerate(rb) for c, (c0, cl) in enumerate(cb)]


def row_block_tiles(rows, cols, p):
    return [(r0, rl, 0, cols, i) for i, (r0, rl) in enumerate(split(rows, p))]


def col_block_tiles(rows, cols, p):
    return [(0, rows, c0, cl, i) for i, (c0, cl) in enumerate(split(cols, p))]


def rel_fro(got: np.ndarray, want: np.ndarray) -> float:
    g = np.asarray(got, dtype=np.float64)
    w = np.asarray(want, dtype=np.float64)
    den = np.linalg.norm(w)
    return float(np.linalg.norm(g - w) / (den if den else 1.0))


def ckpt_write_ref(workers, mats, path, alpha=1.0):
    """The reference writes a DMCK checkpoint of `mats` = [(image2d, prec,
    tiles)] (ids 1..n; mulScalar(alpha) on matrix 1 first when alpha != 1)."""
    lib = reflib()
    n = len(mats)
    imgs = [np.ascontiguousarray(m[0]) for m in mats]
    tarrs = [tiles_array(list(m[2])) for m in mats]
    rows = (c_uint64 * n)(*[i.shape[0] for i in imgs])
    cols = (c_uint64 * n)(*[i.shape[1] for i in imgs])
    precs = (c_int32 * n)(*[m[1] for m in mats])
    tp = (POINTER(HTile) * n)(*[ctypes.cast(t, POINTER(HTile)) for t in tarrs])
    nt = (c_uint32 * n)(*[len(m[2]) for m in mats])
    ip = (c_void_p * n)(*[i.ctypes.data for i in imgs])
    err = ctypes.create_string_buffer(512)
    if lib.gmref_ckpt_write(workers, n, rows, cols, precs, tp, nt, ip, alpha, os.fsencode(path), err, 512):
        raise RuntimeError("reference checkpoint failed: " + err.value.decode())


def ckpt_read_ref(path, workers, shapes):
    """The reference restores `path` and returns [(image, version)] for ids
    1..len(shapes); shapes = [(rows, cols, prec)]."""
    lib = reflib()
    n = len(shapes)
    outs = [np.empty((r, c), dtype=NP_DTYPE[p]) for (r, c, p) in shapes]
    ids = (c_uint64 * n)(*range(1, n + 1))
    op = (c_void_p * n)(*[o.ctypes.data for o in outs])
    vers = (c_uint64 * n)()
    err = ctypes.create_string_buffer(512)
    if lib.gmref_ckpt_read(os.fsencode(path), workers, n, ids, op, vers, err, 512):
        raise RuntimeError("reference restore failed: " + err.value.decode())
    return [(outs[i], vers[i]) for i in range(n)]
