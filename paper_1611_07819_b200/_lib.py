# SPDX-License-Identifier: Apache-2.0
"""ctypes binding of the C ABI declared in include/gridmath_b200.h.

The shared library is built in-tree (``make -C paper_1611_07819_b200``) and
is the ONLY execution path: there is no Python or CPU fallback. Loading
fails loudly when the library is missing.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import (POINTER, Structure, c_char_p, c_double, c_int32, c_uint8, c_uint32,
                    c_uint64, c_void_p)

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libgridmath_b200.so")

GM_HALF, GM_SINGLE, GM_DOUBLE, GM_BF16 = 0, 1, 2, 3
GM_MATH_DEFAULT, GM_MATH_TF32, GM_MATH_FOLD = 0, 1, 2
GM_REPL_IN_FLIGHT, GM_REPL_DONE, GM_REPL_FAILED = 0, 1, 2
GM_OP_SET_CONST, GM_OP_GEMM, GM_OP_ADD_ROW_COL_SUM, GM_OP_EW_UNARY, GM_OP_EW_BINARY = 5, 6, 7, 8, 9


class GmError(RuntimeError):
    """Raised for every non-zero status (mirrors gridmath::Error)."""


class gm_tile(Structure):
    _fields_ = [("row_start", c_uint64), ("row_count", c_uint64), ("col_start", c_uint64),
                ("col_count", c_uint64), ("owner", c_uint32)]


class gm_arena_stats(Structure):
    _fields_ = [("allocations_from_os", c_uint64), ("reuses", c_uint64), ("frees", c_uint64),
                ("held_bytes", c_uint64), ("reserved_bytes", c_uint64)]


class gm_gemm_desc(Structure):
    _fields_ = [("m", c_uint64), ("n", c_uint64), ("k", c_uint64), ("lda", c_uint64),
                ("ldb", c_uint64), ("ldc", c_uint64), ("trans_a", c_int32), ("trans_b", c_int32),
                ("prec_a", c_int32), ("prec_b", c_int32), ("prec_c", c_int32), ("math", c_int32),
                ("cta_group", c_int32), ("max_ctas", c_int32), ("alpha", c_double),
                ("beta", c_double)]


class gm_session_options(Structure):
    _fields_ = [("workers", c_uint32), ("deterministic", c_int32),
                ("replication_chunk_bytes", c_uint64), ("root_seed", c_uint64),
                ("check_metadata_every_op", c_int32), ("spmd_rank", c_int32),
                ("num_devices", c_int32), ("devices", c_int32 * 16),
                ("nccl_unique_id", c_uint8 * 128), ("arena_slab_bytes", c_uint64),
                ("gemm_max_ctas", c_int32), ("transport", c_int32), ("panel_cache_bytes", c_uint64),
                ("pipeline_chunks", c_int32), ("control_allreduce_max_u8", c_void_p),
                ("control_user", c_void_p)]


class gm_worker_stats(Structure):
    _fields_ = [("os_allocations", c_uint64), ("reuses", c_uint64), ("frees", c_uint64),
                ("held_bytes", c_uint64), ("resident_bytes", c_uint64), ("cache_hits", c_uint64),
                ("cache_misses", c_uint64), ("cache_bytes", c_uint64), ("bytes_sent", c_uint64),
                ("bytes_received", c_uint64)]


class gm_plan_piece(Structure):
    _fields_ = [("src", c_uint32), ("dst", c_uint32), ("operand", c_uint32), ("pad", c_uint32),
                ("r0", c_uint64), ("r1", c_uint64), ("c0", c_uint64), ("c1", c_uint64)]


_P = POINTER
_SIGNATURES = {
    "gm_last_error": ([], c_char_p),
    "gm_version": ([_P(c_int32), _P(c_int32)], c_int32),
    "gm_device_count": ([_P(c_int32)], c_int32),
    "gm_device_init": ([c_int32], c_int32),
    "gm_device_synchronize": ([c_int32], c_int32),
    "gm_arena_create": ([c_int32, c_uint64, _P(c_void_p)], c_int32),
    "gm_arena_destroy": ([c_void_p], c_int32),
    "gm_arena_alloc": ([c_void_p, c_uint64, _P(c_void_p)], c_int32),
    "gm_arena_free": ([c_void_p, c_void_p], c_int32),
    "gm_arena_get_stats": ([c_void_p, _P(gm_arena_stats)], c_int32),
    "gm_gemm_workspace_size": ([_P(gm_gemm_desc), _P(c_uint64)], c_int32),
    "gm_gemm_local": ([_P(gm_gemm_desc), c_void_p, c_void_p, c_void_p, c_void_p, c_uint64,
                       c_void_p], c_int32),
    "gm_convert": ([c_void_p, c_int32, c_void_p, c_int32, c_uint64, c_void_p], c_int32),
    "gm_copy_rect": ([c_void_p, c_uint64, c_void_p, c_uint64, c_uint64, c_uint64, c_uint32,
                      c_void_p], c_int32),
    "gm_fill_uniform": ([c_void_p, c_int32, c_uint64, c_uint64, c_uint64, c_uint64, c_uint64,
                         c_uint64, c_uint64, c_double, c_double, c_void_p], c_int32),
    "gm_layout_row_block": ([c_uint64, c_uint64, c_uint32, _P(gm_tile), c_uint32, _P(c_uint32)],
                            c_int32),
    "gm_layout_col_block": ([c_uint64, c_uint64, c_uint32, _P(gm_tile), c_uint32, _P(c_uint32)],
                            c_int32),
    "gm_layout_grid": ([c_uint64, c_uint64, c_uint32, c_uint32, _P(gm_tile), c_uint32,
                        _P(c_uint32)], c_int32),
    "gm_layout_validate": ([c_uint64, c_uint64, _P(gm_tile), c_uint32, c_uint32, _P(c_int32)],
                           c_int32),
    "gm_plan_gemm": ([c_uint32, c_uint64, c_uint64, c_int32, _P(gm_tile), c_uint32, c_uint64, c_uint64,
                      c_int32, _P(gm_tile), c_uint32, c_uint64, c_uint64, c_int32, _P(gm_tile), c_uint32,
                      c_int32, c_int32, c_int32, c_int32, _P(gm_plan_piece), c_uint32, _P(c_uint32),
                      _P(c_uint64)], c_int32),
    "gm_descriptor_encode": ([c_uint64, c_uint64, c_uint64, c_int32, c_uint64, _P(gm_tile), c_uint32,
                              _P(c_uint8), c_uint32, _P(c_uint32)], c_int32),
    "gm_convert_host": ([c_void_p, c_int32, c_void_p, c_int32, c_uint64], c_int32),
    "gm_session_options_default": ([_P(gm_session_options)], None),
    "gm_session_create": ([_P(gm_session_options), _P(c_void_p)], c_int32),
    "gm_session_destroy": ([c_void_p], c_int32),
    "gm_session_checkpoint": ([c_void_p, c_char_p], c_int32),
    "gm_session_restore": ([c_char_p, _P(gm_session_options), _P(c_void_p)], c_int32),
    "gm_nccl_unique_id": ([_P(c_uint8 * 128)], c_int32),
    "gm_matrix_create": ([c_void_p, c_uint64, c_uint64, c_int32, _P(gm_tile), c_uint32,
                          _P(c_uint64)], c_int32),
    "gm_matrix_destroy": ([c_void_p, c_uint64], c_int32),
    "gm_matrix_set_raw": ([c_void_p, c_uint64, c_void_p, c_uint64], c_int32),
    "gm_matrix_set_f64": ([c_void_p, c_uint64, c_void_p, c_uint64], c_int32),
    "gm_matrix_set_f32": ([c_void_p, c_uint64, c_void_p, c_uint64], c_int32),
    "gm_matrix_fill_uniform": ([c_void_p, c_uint64, c_uint64, c_double, c_double], c_int32),
    "gm_matrix_get_raw": ([c_void_p, c_uint64, c_void_p, c_uint64], c_int32),
    "gm_matrix_get_local_raw": ([c_void_p, c_uint64, c_void_p, c_uint64], c_int32),
    "gm_matrix_local_bytes": ([c_void_p, c_uint64, _P(c_uint64)], c_int32),
    "gm_matrix_set_local_packed": ([c_void_p, c_uint64, c_void_p, c_uint64], c_int32),
    "gm_matrix_get_local_packed": ([c_void_p, c_uint64, c_void_p, c_uint64], c_int32),
    "gm_matrix_set_local_packed_async": ([c_void_p, c_uint64, c_void_p, c_uint64, c_uint64], c_int32),
    "gm_matrix_get_local_packed_async": ([c_void_p, c_uint64, c_void_p, c_uint64], c_int32),
    "gm_matrix_reshape": ([c_void_p, c_uint64, _P(gm_tile), c_uint32, c_int32], c_int32),
    "gm_matrix_info": ([c_void_p, c_uint64, _P(c_uint64), _P(c_uint64), _P(c_int32),
                        _P(c_uint64), _P(c_uint64)], c_int32),
    "gm_gemm": ([c_void_p, c_uint64, c_uint64, c_uint64, c_double, c_double, c_int32, c_int32],
                c_int32),
    "gm_gemm_ex": ([c_void_p, c_uint64, c_uint64, c_uint64, c_double, c_double, c_int32,
                    c_int32, c_int32], c_int32),
    "gm_gemm_async": ([c_void_p, c_uint64, c_uint64, c_uint64, c_double, c_double, c_int32,
                       c_int32], c_int32),
    "gm_set_const": ([c_void_p, c_uint64, c_double], c_int32),
    "gm_add_row_col_sum": ([c_void_p, c_uint64, c_uint64, c_uint64, c_double, c_int32], c_int32),
    "gm_relu": ([c_void_p, c_uint64, c_uint64], c_int32),
    "gm_mul_scalar": ([c_void_p, c_uint64, c_double], c_int32),
    "gm_add_matrices": ([c_void_p, c_uint64, c_uint64, c_uint64], c_int32),
    "gm_sub_matrices": ([c_void_p, c_uint64, c_uint64, c_uint64], c_int32),
    "gm_axpy": ([c_void_p, c_double, c_uint64, c_uint64], c_int32),
    "gm_relu_grad": ([c_void_p, c_uint64, c_uint64], c_int32),
    "gm_bias_add": ([c_void_p, c_uint64, c_uint64], c_int32),
    "gm_copy_matrix": ([c_void_p, c_uint64, c_uint64], c_int32),
    "gm_cast_precision": ([c_void_p, c_uint64, c_uint64], c_int32),
    "gm_begin_record": ([c_void_p, _P(c_uint64)], c_int32),
    "gm_end_record": ([c_void_p], c_int32),
    "gm_replay": ([c_void_p, c_uint64], c_int32),
    "gm_replay_async": ([c_void_p, c_uint64], c_int32),
    "gm_op_issue": ([c_void_p, c_int32, _P(c_uint64), c_double, c_double, _P(c_uint8), c_int32], c_int32),
    "gm_session_synchronize": ([c_void_p], c_int32),
    "gm_replicate_async": ([c_void_p, c_uint64, _P(c_uint64)], c_int32),
    "gm_replicate_sync": ([c_void_p, c_uint64], c_int32),
    "gm_replicate_wait": ([c_void_p, c_uint64, c_uint64, _P(c_int32)], c_int32),
    "gm_replicate_state": ([c_void_p, c_uint64, c_uint64, _P(c_int32)], c_int32),
    "gm_query_worker_stats": ([c_void_p, _P(gm_worker_stats), c_uint32, _P(c_uint32)], c_int32),
    "gm_verify_metadata": ([c_void_p], c_int32),
    "gm_session_local_workers": ([c_void_p, _P(c_uint32), c_uint32, _P(c_uint32)], c_int32),
    "gm_session_transport": ([c_void_p, _P(c_int32)], c_int32),
    "gm_session_set_panel_pipelining": ([c_void_p, c_int32], c_int32),
    "gm_session_set_graph_replay": ([c_void_p, c_int32], c_int32),
    "gm_session_set_op_timeline": ([c_void_p, c_int32], c_int32),
    "gm_session_op_timeline": ([c_void_p, _P(ctypes.c_float), _P(ctypes.c_float), c_uint32, ctypes.c_char_p, c_uint32,
                                _P(c_uint32)], c_int32),
    "gm_session_graph_stats": ([c_void_p, _P(c_uint64), _P(c_uint64), _P(c_uint64)], c_int32),
    "gm_last_op_kernel_ms": ([c_void_p, _P(ctypes.c_float), c_uint32, _P(c_uint32)], c_int32),
    "gm_last_op_comm_ms": ([c_void_p, _P(ctypes.c_float), c_uint32, _P(c_uint32)], c_int32),
    "gm_timer_kernel_ms": ([c_void_p, _P(ctypes.c_float), _P(c_uint32), c_uint32, _P(c_uint32)], c_int32),
    "gm_timer_start": ([c_void_p], c_int32),
    "gm_timer_stop": ([c_void_p, _P(ctypes.c_float)], c_int32),
    "gm_kernel_launches": ([_P(c_uint64)], c_int32),
    "gm_last_op_device_ms": ([c_void_p, _P(ctypes.c_float), c_uint32, _P(c_uint32)], c_int32),
}

EXPORTED = tuple(_SIGNATURES)

_lib = None


def load() -> ctypes.CDLL:
    """Loads the in-tree library once; raises if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise GmError(f"{LIB_PATH} not built: run `make -C {_HERE}` (or __graft_entry__.build())")
    lib = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
    for name, (argtypes, restype) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = argtypes
        fn.restype = restype
    _lib = lib
    return lib


def check(status: int) -> None:
    if status != 0:
        msg = load().gm_last_error()
        raise GmError(msg.decode() if msg else "gridmath error")
