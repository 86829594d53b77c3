# SPDX-License-Identifier: Apache-2.0
"""Python mirror of the reference's gridmath master API over the C ABI.

Names and argument meaning follow the reference C++ library
(/root/reference/proj/include/gridmath/session.hpp:21-179, layout.hpp:62-85,
precision.hpp:12) so parity tests read like the reference's own usage:

    s = Session(workers=4)
    A = s.createMatrix(m, k, Precision.BF16, makeGridLayout(m, k, 2, 2, makeWorkerGroup(4)))
    s.setDataRaw(A, image)
    gemm(s, A, B, C, 1.0, 0.0)
    out = s.getDataRaw(C)

Every call goes through libgridmath_b200.so (include/gridmath_b200.h); there
is no Python compute path. Errors raise GmError (the reference's
gridmath::Error).
"""
from __future__ import annotations

import ctypes
import os
import enum
from dataclasses import dataclass
from typing import List, Optional, Sequence

import numpy as np

from . import _lib
from ._lib import GmError, check

__all__ = ["Precision", "TileExtent", "Layout", "makeWorkerGroup", "makeRowBlockLayout",
           "makeColBlockLayout", "makeGridLayout", "makeSingleTileLayout", "validateLayout",
           "Session", "DistMatrix", "ReplicationHandle", "ReplState", "gemm", "GmError",
           "nccl_unique_id", "np_storage_dtype", "kernel_launches"]


class Precision(enum.IntEnum):
    Half = _lib.GM_HALF
    Single = _lib.GM_SINGLE
    Double = _lib.GM_DOUBLE
    BF16 = _lib.GM_BF16


def np_storage_dtype(p: Precision):
    """numpy container of a storage precision (bf16 held as raw uint16)."""
    return {Precision.Half: np.float16, Precision.Single: np.float32,
            Precision.Double: np.float64, Precision.BF16: np.uint16}[Precision(p)]


def bytes_of(p: Precision) -> int:
    return {Precision.Half: 2, Precision.Single: 4, Precision.Double: 8, Precision.BF16: 2}[Precision(p)]


class ReplState(enum.IntEnum):
    InFlight = _lib.GM_REPL_IN_FLIGHT
    Done = _lib.GM_REPL_DONE
    Failed = _lib.GM_REPL_FAILED


@dataclass(frozen=True)
class TileExtent:
    rowStart: int
    rowCount: int
    colStart: int
    colCount: int


@dataclass
class Layout:
    tiles: List[tuple]  # [(TileExtent, owner rank)]

    def as_c(self):
        arr = (_lib.gm_tile * max(1, len(self.tiles)))()
        for i, (e, w) in enumerate(self.tiles):
            arr[i] = _lib.gm_tile(e.rowStart, e.rowCount, e.colStart, e.colCount, int(w))
        return arr

    def as_tuples(self):
        return [(e.rowStart, e.rowCount, e.colStart, e.colCount, int(w)) for e, w in self.tiles]


def _from_c(arr, n) -> Layout:
    return Layout([(TileExtent(t.row_start, t.row_count, t.col_start, t.col_count), t.owner)
                   for t in arr[:n]])


def makeWorkerGroup(count: int) -> List[int]:
    return list(range(count))


def _call_layout(fn, *args) -> Layout:
    lib = _lib.load()
    cap = 4096
    arr = (_lib.gm_tile * cap)()
    n = ctypes.c_uint32()
    check(getattr(lib, fn)(*args, arr, cap, ctypes.byref(n)))
    return _from_c(arr, n.value)


def makeRowBlockLayout(rows: int, cols: int, workers: Sequence[int]) -> Layout:
    return _call_layout("gm_layout_row_block", rows, cols, len(workers))


def makeColBlockLayout(rows: int, cols: int, workers: Sequence[int]) -> Layout:
    return _call_layout("gm_layout_col_block", rows, cols, len(workers))


def makeGridLayout(rows: int, cols: int, pr: int, pc: int, workers: Sequence[int]) -> Layout:
    if pr * pc != len(workers):
        raise GmError("makeGridLayout: pr*pc must equal worker count")
    return _call_layout("gm_layout_grid", rows, cols, pr, pc)


def makeSingleTileLayout(rows: int, cols: int, owner: int) -> Layout:
    return Layout([(TileExtent(0, rows, 0, cols), owner)])


def validateLayout(rows: int, cols: int, layout: Layout, workerCount: int = 0) -> int:
    """0 ok, 1 overlap, 2 gap, 3 out of range, 4 unknown worker."""
    v = ctypes.c_int32()
    check(_lib.load().gm_layout_validate(rows, cols, layout.as_c(), len(layout.tiles), workerCount,
                                         ctypes.byref(v)))
    return v.value


def nccl_unique_id() -> bytes:
    buf = (ctypes.c_uint8 * 128)()
    check(_lib.load().gm_nccl_unique_id(ctypes.byref(buf)))
    return bytes(buf)


_CONTROL_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p)


def gloo_control(group=None):
    """SPMD control channel over a torch.distributed gloo group (CPU): the
    session's few blocking control collectives (IPC registration, budget
    agreement, shutdown) run through it instead of an NCCL communicator, so
    several ranks may share one GPU. `group` None: a new gloo group over the
    default world (or the default group itself when it is gloo)."""
    import torch
    import torch.distributed as dist
    if group is None and dist.get_backend() != "gloo":
        group = dist.new_group(backend="gloo")

    def allreduce_max(buf, n, _user):
        try:
            t = torch.frombuffer((ctypes.c_uint8 * n).from_address(buf), dtype=torch.uint8)
            dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
            return 0
        except Exception:  # reported to the library as a failed collective
            return 1

    return allreduce_max


@dataclass(frozen=True)
class DistMatrix:
    session: "Session"
    id: int

    def info(self):
        rows, cols, ver, rv = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
        prec = ctypes.c_int32()
        check(_lib.load().gm_matrix_info(self.session._h, self.id, ctypes.byref(rows), ctypes.byref(cols),
                                         ctypes.byref(prec), ctypes.byref(ver), ctypes.byref(rv)))
        return rows.value, cols.value, Precision(prec.value), ver.value, rv.value

    def rows(self) -> int:
        return self.info()[0]

    def cols(self) -> int:
        return self.info()[1]

    def precision(self) -> Precision:
        return self.info()[2]

    def version(self) -> int:
        return self.info()[3]


@dataclass(frozen=True)
class ReplicationHandle:
    matrixId: int
    version: int


class Session:
    """gridmath::Session. workers = P. spmd_rank >= 0 selects one-process-per-GPU
    mode (this process hosts worker spmd_rank on `devices[0]`)."""

    def __init__(self, workers: int = 1, deterministic: bool = True, devices: Optional[Sequence[int]] = None,
                 spmd_rank: int = -1, nccl_id: Optional[bytes] = None, gemm_max_ctas: int = 0,
                 transport: int = 0, check_metadata_every_op: bool = False, panel_cache_bytes: int = 0,
                 pipeline_chunks: int = 0, control=None, _restore_from: Optional[str] = None):
        """control: None (NCCL control channel under SPMD) or a callable
        (buf_address, nbytes, user) -> int doing an in-place max all-reduce of
        host bytes over the ranks (see gloo_control), or "gloo"."""
        lib = _lib.load()
        o = _lib.gm_session_options()
        lib.gm_session_options_default(ctypes.byref(o))
        o.workers = workers
        o.deterministic = 1 if deterministic else 0
        o.spmd_rank = spmd_rank
        o.check_metadata_every_op = 1 if check_metadata_every_op else 0
        devs = list(devices or [])
        o.num_devices = len(devs)
        for i, d in enumerate(devs[:16]):
            o.devices[i] = d
        if nccl_id is not None:
            ctypes.memmove(o.nccl_unique_id, nccl_id, 128)
        o.gemm_max_ctas = gemm_max_ctas
        o.transport = transport
        o.panel_cache_bytes = panel_cache_bytes
        o.pipeline_chunks = pipeline_chunks
        self._control = None
        if control is not None:
            fn = gloo_control() if control == "gloo" else control
            self._control = _CONTROL_FN(fn)  # kept alive for the session's lifetime
            o.control_allreduce_max_u8 = ctypes.cast(self._control, ctypes.c_void_p)
        self._h = ctypes.c_void_p()
        if _restore_from is None:
            check(lib.gm_session_create(ctypes.byref(o), ctypes.byref(self._h)))
        else:
            check(lib.gm_session_restore(os.fsencode(_restore_from), ctypes.byref(o), ctypes.byref(self._h)))
        self.workers = workers
        self.deterministic = deterministic

    @classmethod
    def restore(cls, path: str, workers: int = 1, **kw) -> "Session":
        """Session::restore (session.cpp:446-480): a new session holding every
        matrix of a DMCK checkpoint (ours or the reference's)."""
        return cls(workers=workers, _restore_from=path, **kw)

    def checkpoint(self, path: str):
        """Session::checkpoint (session.cpp:413-442), DMCK format."""
        check(_lib.load().gm_session_checkpoint(self._h, os.fsencode(path)))

    def matrix(self, mid: int) -> "DistMatrix":
        """Handle of an existing matrix id (e.g. after restore)."""
        return DistMatrix(self, mid)

    def close(self):
        if self._h:
            check(_lib.load().gm_session_destroy(self._h))
            self._h = ctypes.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # --- lifecycle ------------------------------------------------------------
    def createMatrix(self, rows: int, cols: int, prec: Precision, layout: Layout) -> DistMatrix:
        mid = ctypes.c_uint64()
        check(_lib.load().gm_matrix_create(self._h, rows, cols, int(prec), layout.as_c(),
                                           len(layout.tiles), ctypes.byref(mid)))
        return DistMatrix(self, mid.value)

    def destroy(self, m: DistMatrix):
        check(_lib.load().gm_matrix_destroy(self._h, m.id))

    def setDataRaw(self, m: DistMatrix, image: np.ndarray):
        img = np.ascontiguousarray(image)
        check(_lib.load().gm_matrix_set_raw(self._h, m.id, img.ctypes.data, img.nbytes))

    def setDataRawPtr(self, m: DistMatrix, ptr: int, nbytes: int):
        check(_lib.load().gm_matrix_set_raw(self._h, m.id, ptr, nbytes))

    def setData(self, m: DistMatrix, values):
        v = np.ascontiguousarray(values, dtype=np.float64).ravel()
        check(_lib.load().gm_matrix_set_f64(self._h, m.id, v.ctypes.data, v.size))

    def setDataF32(self, m: DistMatrix, values):
        v = np.ascontiguousarray(values, dtype=np.float32).ravel()
        check(_lib.load().gm_matrix_set_f32(self._h, m.id, v.ctypes.data, v.size))

    def fillUniform(self, m: DistMatrix, seed: int, lo: float = -1.0, hi: float = 1.0):
        check(_lib.load().gm_matrix_fill_uniform(self._h, m.id, seed, lo, hi))

    def getDataRaw(self, m: DistMatrix, local_only: bool = False) -> np.ndarray:
        rows, cols, prec, _, _ = m.info()
        out = np.zeros((rows, cols), dtype=np_storage_dtype(prec))
        fn = _lib.load().gm_matrix_get_local_raw if local_only else _lib.load().gm_matrix_get_raw
        check(fn(self._h, m.id, out.ctypes.data, out.nbytes))
        return out

    def getDataRawPtr(self, m: DistMatrix, ptr: int, nbytes: int, local_only: bool = True):
        fn = _lib.load().gm_matrix_get_local_raw if local_only else _lib.load().gm_matrix_get_raw
        check(fn(self._h, m.id, ptr, nbytes))

    def getData(self, m: DistMatrix) -> np.ndarray:
        raw = self.getDataRaw(m)
        if m.precision() == Precision.BF16:
            return (raw.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
        return raw.astype(np.float64)

    def reshape(self, m: DistMatrix, layout: Layout, prec: Optional[Precision] = None):
        """Redistribute to `layout` (and storage `prec`); reference Session::reshape."""
        check(_lib.load().gm_matrix_reshape(self._h, m.id, layout.as_c(), len(layout.tiles),
                                            -1 if prec is None else int(prec)))

    # --- replication -------------------------------------------------------------
    def replicateAsync(self, m: DistMatrix) -> ReplicationHandle:
        v = ctypes.c_uint64()
        check(_lib.load().gm_replicate_async(self._h, m.id, ctypes.byref(v)))
        return ReplicationHandle(m.id, v.value)

    def replicateSync(self, m: DistMatrix):
        check(_lib.load().gm_replicate_sync(self._h, m.id))

    def wait(self, h: ReplicationHandle) -> ReplState:
        st = ctypes.c_int32()
        check(_lib.load().gm_replicate_wait(self._h, h.matrixId, h.version, ctypes.byref(st)))
        return ReplState(st.value)

    def handleState(self, h: ReplicationHandle) -> ReplState:
        st = ctypes.c_int32()
        check(_lib.load().gm_replicate_state(self._h, h.matrixId, h.version, ctypes.byref(st)))
        return ReplState(st.value)

    # --- introspection -----------------------------------------------------------
    def queryWorkerStats(self):
        rows = (_lib.gm_worker_stats * 64)()
        n = ctypes.c_uint32()
        check(_lib.load().gm_query_worker_stats(self._h, rows, 64, ctypes.byref(n)))
        keys = [f[0] for f in _lib.gm_worker_stats._fields_]
        return [{k: getattr(r, k) for k in keys} for r in rows[: n.value]]

    def verifyMetadataConsistency(self):
        check(_lib.load().gm_verify_metadata(self._h))

    def localWorkers(self) -> List[int]:
        arr = (ctypes.c_uint32 * 64)()
        n = ctypes.c_uint32()
        check(_lib.load().gm_session_local_workers(self._h, arr, 64, ctypes.byref(n)))
        return list(arr[: n.value])

    def transport(self) -> str:
        """Data plane in use: "peer_copy" (one process), "nccl", or "ipc"
        (one process per GPU, copy-engine pulls over CUDA IPC)."""
        k = ctypes.c_int32()
        check(_lib.load().gm_session_transport(self._h, ctypes.byref(k)))
        return {0: "peer_copy", 1: "nccl", 2: "ipc"}[k.value]

    def synchronize(self):
        check(_lib.load().gm_session_synchronize(self._h))

    def lastOpDeviceMs(self) -> List[float]:
        arr = (ctypes.c_float * 64)()
        n = ctypes.c_uint32()
        check(_lib.load().gm_last_op_device_ms(self._h, arr, 64, ctypes.byref(n)))
        return list(arr[: n.value])

    def lastOpKernelMs(self) -> List[float]:
        arr = (ctypes.c_float * 64)()
        n = ctypes.c_uint32()
        check(_lib.load().gm_last_op_kernel_ms(self._h, arr, 64, ctypes.byref(n)))
        return list(arr[: n.value])

    def timerKernelMs(self) -> List[tuple]:
        """[(sum of gemm compute-phase ms, gemm count)] per local worker over
        the last timerStart()/timerStop() window."""
        arr = (ctypes.c_float * 64)()
        cnt = (ctypes.c_uint32 * 64)()
        n = ctypes.c_uint32()
        check(_lib.load().gm_timer_kernel_ms(self._h, arr, cnt, 64, ctypes.byref(n)))
        return [(arr[i], cnt[i]) for i in range(n.value)]

    def lastOpCommMs(self) -> List[float]:
        arr = (ctypes.c_float * 64)()
        n = ctypes.c_uint32()
        check(_lib.load().gm_last_op_comm_ms(self._h, arr, 64, ctypes.byref(n)))
        return list(arr[: n.value])

    def localBytes(self, m: DistMatrix) -> int:
        b = ctypes.c_uint64()
        check(_lib.load().gm_matrix_local_bytes(self._h, m.id, ctypes.byref(b)))
        return b.value

    def setLocalPacked(self, m: DistMatrix, ptr: int, nbytes: int):
        check(_lib.load().gm_matrix_set_local_packed(self._h, m.id, ptr, nbytes))

    def getLocalPacked(self, m: DistMatrix, ptr: int, nbytes: int):
        check(_lib.load().gm_matrix_get_local_packed(self._h, m.id, ptr, nbytes))

    def setLocalPackedAsync(self, m: DistMatrix, ptr: int, nbytes: int, chunk_bytes: int = 0):
        check(_lib.load().gm_matrix_set_local_packed_async(self._h, m.id, ptr, nbytes, chunk_bytes))

    def getLocalPackedAsync(self, m: DistMatrix, ptr: int, nbytes: int):
        check(_lib.load().gm_matrix_get_local_packed_async(self._h, m.id, ptr, nbytes))

    def setPanelPipelining(self, on: bool):
        """In-GEMM panel pipelining for later GEMMs (default on)."""
        check(_lib.load().gm_session_set_panel_pipelining(self._h, 1 if on else 0))

    def setGraphReplay(self, on: bool):
        """Replays after a pipeline's first as one CUDA graph (default off)."""
        check(_lib.load().gm_session_set_graph_replay(self._h, 1 if on else 0))

    def graphStats(self) -> dict:
        """{launches, instantiations, nodes} of the captured replays."""
        a, b, c = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
        check(_lib.load().gm_session_graph_stats(self._h, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)))
        return {"launches": a.value, "instantiations": b.value, "nodes": c.value}

    def setOpTimeline(self, on: bool):
        """Developer: record a per-op device timeline of later replays."""
        check(_lib.load().gm_session_set_op_timeline(self._h, 1 if on else 0))

    def opTimeline(self) -> List[tuple]:
        """[(label, compute_ms, comm_ms)] of the last replay (first local worker)."""
        cap = 256
        cm, co = (ctypes.c_float * cap)(), (ctypes.c_float * cap)()
        lab = ctypes.create_string_buffer(8192)
        n = ctypes.c_uint32()
        check(_lib.load().gm_session_op_timeline(self._h, cm, co, cap, lab, 8192, ctypes.byref(n)))
        labels = lab.value.decode().split("\n")
        return [(labels[i], cm[i], co[i]) for i in range(min(n.value, cap))]

    def timerStart(self):
        check(_lib.load().gm_timer_start(self._h))

    def timerStop(self) -> float:
        ms = ctypes.c_float()
        check(_lib.load().gm_timer_stop(self._h, ctypes.byref(ms)))
        return ms.value

    def gemmAsync(self, a: DistMatrix, b: DistMatrix, c: DistMatrix, alpha=1.0, beta=0.0,
                  transA=False, transB=False):
        check(_lib.load().gm_gemm_async(self._h, a.id, b.id, c.id, alpha, beta, int(transA), int(transB)))

    # --- pipeline recording (session.hpp:89-92) ---------------------------------
    def beginRecord(self) -> int:
        pid = ctypes.c_uint64()
        check(_lib.load().gm_begin_record(self._h, ctypes.byref(pid)))
        return pid.value

    def endRecord(self):
        check(_lib.load().gm_end_record(self._h))

    def replay(self, pipeline_id: int, sync: bool = True):
        fn = _lib.load().gm_replay if sync else _lib.load().gm_replay_async
        check(fn(self._h, pipeline_id))

    def opIssue(self, opcode: int, ids, s0: float = 0.0, s1: float = 0.0, flags=(0, 0, 0, 0), sync: bool = False):
        """Issue one wire op (reference OpDescriptor) on the device path."""
        ids4 = (ctypes.c_uint64 * 4)(*(list(ids) + [0] * (4 - len(ids))))
        fl4 = (ctypes.c_uint8 * 4)(*(list(flags) + [0] * (4 - len(flags))))
        check(_lib.load().gm_op_issue(self._h, opcode, ids4, s0, s1, fl4, int(sync)))


def kernel_launches() -> int:
    n = ctypes.c_uint64()
    check(_lib.load().gm_kernel_launches(ctypes.byref(n)))
    return n.value


def gemm(s: Session, a: DistMatrix, b: DistMatrix, c: DistMatrix, alpha: float, beta: float,
         transA: bool = False, transB: bool = False, math: int = _lib.GM_MATH_DEFAULT):
    """gridmath::gemm (session.hpp:161-162): C = alpha*op(A)*op(B) + beta*C."""
    check(_lib.load().gm_gemm_ex(s._h, a.id, b.id, c.id, alpha, beta, int(transA), int(transB), math))


# --- FC-layer neighbours (reference session.hpp:163-174, same names) ----------

def addRowColSum(s: Session, a: DistMatrix, rowAcc: DistMatrix, colAcc: DistMatrix, alpha: float,
                 deterministic: bool):
    check(_lib.load().gm_add_row_col_sum(s._h, a.id, rowAcc.id, colAcc.id, alpha, int(deterministic)))


def relu(s: Session, x: DistMatrix, dst: DistMatrix):
    check(_lib.load().gm_relu(s._h, x.id, dst.id))


def mulScalar(s: Session, x: DistMatrix, alpha: float):
    check(_lib.load().gm_mul_scalar(s._h, x.id, alpha))


def addMatrices(s: Session, x: DistMatrix, y: DistMatrix, dst: DistMatrix):
    check(_lib.load().gm_add_matrices(s._h, x.id, y.id, dst.id))


def subMatrices(s: Session, x: DistMatrix, y: DistMatrix, dst: DistMatrix):
    check(_lib.load().gm_sub_matrices(s._h, x.id, y.id, dst.id))


def axpy(s: Session, alpha: float, x: DistMatrix, y: DistMatrix):
    check(_lib.load().gm_axpy(s._h, alpha, x.id, y.id))


def reluGrad(s: Session, preact: DistMatrix, grad: DistMatrix):
    check(_lib.load().gm_relu_grad(s._h, preact.id, grad.id))


def biasAdd(s: Session, x: DistMatrix, bias: DistMatrix):
    check(_lib.load().gm_bias_add(s._h, x.id, bias.id))


def copyMatrix(s: Session, src: DistMatrix, dst: DistMatrix):
    check(_lib.load().gm_copy_matrix(s._h, src.id, dst.id))


def castPrecision(s: Session, src: DistMatrix, dst: DistMatrix):
    check(_lib.load().gm_cast_precision(s._h, src.id, dst.id))


def setConst(s: Session, m: DistMatrix, value: float):
    check(_lib.load().gm_set_const(s._h, m.id, value))
