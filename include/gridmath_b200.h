/* SPDX-License-Identifier: Apache-2.0
 *
 * gridmath_b200 -- C ABI of the B200-native block-distributed GEMM path.
 *
 * The reference (dMath re-creation, C++20 library `gridmath`, reference
 * proj/) has no FFI; its operator boundary is the C++ master API
 * (proj/include/gridmath/session.hpp:62-179) and the worker op dispatch
 * (proj/src/kernels.cpp:1138-1171). This header is the plain-C surface a
 * binding (ctypes / cgo / JNI) attaches to. Two layers:
 *
 *   gm_session_* / gm_matrix_* / gm_gemm / gm_replicate_*   master API
 *        -> mirrors gridmath::Session + gridmath::gemm  (session.hpp:62-162)
 *   gm_device_* / gm_arena_* / gm_gemm_local / gm_convert / gm_pack_rect
 *        -> the per-worker device layer the worker runtime calls
 *           (replaces runGemm<T>, PoolAllocator, packRect/convertBuffer)
 *
 * Conventions: every function returns 0 on success and non-zero on error;
 * the message is available from gm_last_error() (thread-local), mirroring the
 * reference's gridmath::Error (proj/include/gridmath/common.hpp:11-14).
 * Device pointers and `stream` (a cudaStream_t, NULL = legacy default stream)
 * are plain pointers; there are no torch types anywhere in this ABI.
 */
#ifndef GRIDMATH_B200_H
#define GRIDMATH_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Storage precision tags. 0/1/2 are the reference's gridmath::Precision
 * values (proj/include/gridmath/precision.hpp:12) and keep their descriptor
 * wire bytes; 3 is the new bf16 storage tag. */
enum { GM_HALF = 0, GM_SINGLE = 1, GM_DOUBLE = 2, GM_BF16 = 3 };

/* Math mode for Single-compute GEMMs, carried in OpDescriptor.flags[3]
 * (unused by the reference's Gemm, kernels.cpp:209-211). */
enum { GM_MATH_DEFAULT = 0, /* 3xTF32: fp32-accurate */
       GM_MATH_TF32 = 1,    /* 1xTF32: opt-in, ~1e-4 rel */
       /* 16-bit operands (fp32 accumulate): fold the tensor cores' fp32
        * accumulation into a round-to-nearest fp32 running sum every 256 of
        * k, as the Single path does -- the error of the reference's serial
        * fp32 sum instead of one that grows with k (opt-in; 256-wide tiles). */
       GM_MATH_FOLD = 2 };

/* Replication states (reference gridmath::ReplState, session.hpp:36). */
enum { GM_REPL_IN_FLIGHT = 0, GM_REPL_DONE = 1, GM_REPL_FAILED = 2 };

const char* gm_last_error(void);
int gm_version(int32_t* major, int32_t* minor);

/* ------------------------------------------------------------------------
 * Device layer
 * ---------------------------------------------------------------------- */

int gm_device_count(int32_t* count);
/* Binds the calling thread to `device` and warms the context. */
int gm_device_init(int32_t device);
int gm_device_synchronize(int32_t device);

/* Per-worker pooled device arena (replaces gridmath::PoolAllocator,
 * proj/include/gridmath/pool.hpp:13-67): power-of-two size classes from 256
 * bytes, carved from large cudaMalloc slabs that are never returned until
 * the arena dies, so steady-state ops perform zero cudaMalloc calls. */
typedef struct gm_arena gm_arena;
typedef struct {
  uint64_t allocations_from_os; /* slab cudaMallocs */
  uint64_t reuses;              /* allocations served from a free list */
  uint64_t frees;
  uint64_t held_bytes;          /* bytes parked in free lists */
  uint64_t reserved_bytes;      /* bytes obtained from cudaMalloc */
} gm_arena_stats;

int gm_arena_create(int32_t device, uint64_t slab_bytes, gm_arena** out);
int gm_arena_destroy(gm_arena* arena);
int gm_arena_alloc(gm_arena* arena, uint64_t bytes, void** ptr);
int gm_arena_free(gm_arena* arena, void* ptr);
int gm_arena_get_stats(const gm_arena* arena, gm_arena_stats* out);

/* One local block GEMM:  C = alpha * op(A) * op(B) + beta * C  on the
 * calling thread's current device (replaces runGemm<T>,
 * proj/src/kernels.cpp:445-558). All matrices are row-major with the given
 * pitches (elements). op(A) is m x k (A stored k x m when trans_a), op(B) is
 * k x n (B stored n x k when trans_b). Compute type follows
 * kernels::computePrecision (kernels.cpp:136-140): Double if any operand is
 * Double, else Single; two 16-bit operands of the same kind run natively on
 * tcgen05 kind::f16 with fp32 accumulation. beta == 0 never reads C;
 * alpha == 0 never reads A or B. */
typedef struct {
  uint64_t m, n, k;
  uint64_t lda, ldb, ldc;
  int32_t trans_a, trans_b;
  int32_t prec_a, prec_b, prec_c;
  int32_t math;      /* GM_MATH_* */
  int32_t cta_group; /* 0 = default (2-SM UMMA), 1 = single-SM */
  int32_t max_ctas;  /* 0 = all SMs */
  double alpha, beta;
} gm_gemm_desc;

/* Device scratch bytes gm_gemm_local needs for `d` (operand conversion,
 * 3xTF32 split, alignment staging). */
int gm_gemm_workspace_size(const gm_gemm_desc* d, uint64_t* bytes);
int gm_gemm_local(const gm_gemm_desc* d, const void* a, const void* b, void* c,
                  void* workspace, uint64_t workspace_bytes, void* stream);

/* Elementwise storage conversion (replaces gridmath::convertBuffer,
 * proj/src/precision.cpp:6-28): RNE, Half overflow -> inf, Double->Half via
 * float exactly as the reference. */
int gm_convert(const void* src, int32_t src_prec, void* dst, int32_t dst_prec, uint64_t count,
               void* stream);

/* 2D sub-rectangle copy between row-major buffers (replaces packRect /
 * unpackRect, proj/src/pieces.cpp:45-63). Pitches in elements. */
int gm_copy_rect(const void* src, uint64_t src_ld, void* dst, uint64_t dst_ld, uint64_t rows,
                 uint64_t cols, uint32_t elem_bytes, void* stream);

/* Synthetic input generator: element i of the SplitMix64 stream seeded with
 * `seed` (reference proj/include/gridmath/common.hpp:37-50) mapped to
 * U[lo, hi), rounded RNE to `prec`, written row-major into the rectangle
 * [r0, r0+rows) x [c0, c0+cols) of a `full_cols`-wide matrix held at `dst`
 * with pitch `ld`. Identical values on host (oracle) and device. */
int gm_fill_uniform(void* dst, int32_t prec, uint64_t ld, uint64_t r0, uint64_t rows, uint64_t c0,
                    uint64_t cols, uint64_t full_cols, uint64_t seed, double lo, double hi,
                    void* stream);

/* ------------------------------------------------------------------------
 * Layout helpers (pure host logic; reference proj/src/layout.cpp:13-114)
 * ---------------------------------------------------------------------- */

typedef struct {
  uint64_t row_start, row_count, col_start, col_count;
  uint32_t owner;
} gm_tile;

/* Each writes up to `cap` tiles into `out` and the count into *n. */
int gm_layout_row_block(uint64_t rows, uint64_t cols, uint32_t workers, gm_tile* out,
                        uint32_t cap, uint32_t* n);
int gm_layout_col_block(uint64_t rows, uint64_t cols, uint32_t workers, gm_tile* out,
                        uint32_t cap, uint32_t* n);
int gm_layout_grid(uint64_t rows, uint64_t cols, uint32_t pr, uint32_t pc, gm_tile* out,
                   uint32_t cap, uint32_t* n);
/* 0 = ok, 1 = overlap, 2 = gap, 3 = out of range, 4 = unknown worker
 * (reference LayoutViolation, layout.hpp:56). */
int gm_layout_validate(uint64_t rows, uint64_t cols, const gm_tile* tiles, uint32_t n,
                       uint32_t worker_count, int32_t* violation);

/* GEMM plan (pure host logic, no device needed): every data movement the
 * GEMM C = op(A) op(B) performs for the given layouts, from the same planner
 * the runtime executes (reference planGemm, kernels.cpp:204-251). One entry
 * per piece: `operand` 0 = A / 1 = B, rectangle in the operand's stored
 * coordinates, src == dst for pieces copied from the consumer's own tiles.
 * a_replicated / b_replicated: the operand has a fresh replica (no pieces).
 * remote_bytes[w] (size `workers`): bytes worker w receives from peers. */
typedef struct {
  uint32_t src, dst, operand, pad;
  uint64_t r0, r1, c0, c1;
} gm_plan_piece;

int gm_plan_gemm(uint32_t workers, uint64_t a_rows, uint64_t a_cols, int32_t a_prec,
                 const gm_tile* a_tiles, uint32_t a_n, uint64_t b_rows, uint64_t b_cols,
                 int32_t b_prec, const gm_tile* b_tiles, uint32_t b_n, uint64_t c_rows,
                 uint64_t c_cols, int32_t c_prec, const gm_tile* c_tiles, uint32_t c_n,
                 int32_t trans_a, int32_t trans_b, int32_t a_replicated, int32_t b_replicated,
                 gm_plan_piece* out, uint32_t cap, uint32_t* n, uint64_t* remote_bytes);

/* Descriptor wire encoding (reference descriptor.cpp:6-20): u64 id, u64 rows,
 * u64 cols, u8 precision, u64 version, u32 tiles, per tile 4 x u64 + u32. */
int gm_descriptor_encode(uint64_t id, uint64_t rows, uint64_t cols, int32_t prec,
                         uint64_t version, const gm_tile* tiles, uint32_t n, uint8_t* out,
                         uint32_t cap, uint32_t* len);

/* Host storage conversion (convertBuffer semantics; setData's host path). */
int gm_convert_host(const void* src, int32_t src_prec, void* dst, int32_t dst_prec,
                    uint64_t count);

/* ------------------------------------------------------------------------
 * Master API (reference gridmath::Session, session.hpp:62-179)
 * ---------------------------------------------------------------------- */

typedef struct gm_session gm_session;

typedef struct {
  uint32_t workers;                 /* P, total worker count */
  int32_t deterministic;            /* SessionOptions::deterministic (default 1) */
  uint64_t replication_chunk_bytes; /* kept for wire compatibility */
  uint64_t root_seed;
  int32_t check_metadata_every_op;
  /* B200 placement. Single process (spmd_rank < 0): worker r runs on device
   * devices[r % num_devices] (num_devices == 0: all visible devices).
   * SPMD (one process per GPU, torchrun): this process hosts worker
   * spmd_rank on `devices[0]`; data plane is NCCL, bootstrapped from
   * nccl_unique_id (128 bytes, same on every rank). */
  int32_t spmd_rank;
  int32_t num_devices;
  int32_t devices[16];
  uint8_t nccl_unique_id[128];
  uint64_t arena_slab_bytes;        /* 0 = default */
  int32_t gemm_max_ctas;            /* 0 = all SMs (cap leaves SMs for NCCL) */
  int32_t transport;                /* 0 = auto, 1 = NCCL, 2 = copy engines (IPC pulls under SPMD) */
  uint64_t panel_cache_bytes;       /* per-worker panel cache budget; 0 = 1/4 of HBM, 1 = off */
  int32_t pipeline_chunks;          /* SUMMA overlap chunks per band (0 = auto, 1 = off) */
  /* SPMD control channel. NULL: an NCCL communicator (bootstrapped from
   * nccl_unique_id) carries the few blocking control collectives. Non-NULL:
   * the host calls this instead -- a max-reduce of `bytes` host bytes over
   * every rank, in place, blocking, returning 0 on success (e.g. a gloo
   * all_reduce) -- and no NCCL communicator is created, so several ranks may
   * share one GPU; the data plane is then the copy-engine (IPC) plane. */
  int (*control_allreduce_max_u8)(void* buf, uint64_t bytes, void* user);
  void* control_user;
} gm_session_options;

void gm_session_options_default(gm_session_options* o);
int gm_session_create(const gm_session_options* opts, gm_session** out);
int gm_session_destroy(gm_session* s);
/* Checkpoint-restart (reference Session::checkpoint / restore,
 * session.cpp:413-480) in the reference's DMCK file format: files written by
 * either implementation restore in the other. checkpoint fails while a
 * replication is in flight; under SPMD rank 0 writes (collective). restore
 * creates a session from `opts` (root seed taken from the file) holding every
 * saved matrix with its id and version + 1. */
int gm_session_checkpoint(gm_session* s, const char* path);
int gm_session_restore(const char* path, const gm_session_options* opts, gm_session** out);
/* SPMD only: the NCCL unique id rank 0 must broadcast before create. */
int gm_nccl_unique_id(uint8_t out[128]);

int gm_matrix_create(gm_session* s, uint64_t rows, uint64_t cols, int32_t prec,
                     const gm_tile* tiles, uint32_t ntiles, uint64_t* id);
int gm_matrix_destroy(gm_session* s, uint64_t id);
/* Full row-major image in storage precision. In SPMD mode every rank passes
 * the full image and uploads only its own tiles. */
int gm_matrix_set_raw(gm_session* s, uint64_t id, const void* host, uint64_t bytes);
/* setData (double values, converted like convertBuffer), setDataF32. */
int gm_matrix_set_f64(gm_session* s, uint64_t id, const double* host, uint64_t count);
int gm_matrix_set_f32(gm_session* s, uint64_t id, const float* host, uint64_t count);
/* Device-side generation of the synthetic SplitMix64 inputs (gm_fill_uniform
 * semantics) straight into the owners' tiles; no host image needed. */
int gm_matrix_fill_uniform(gm_session* s, uint64_t id, uint64_t seed, double lo, double hi);
/* getDataRaw: full row-major image (SPMD: tiles not owned locally are
 * gathered from their owners). */
int gm_matrix_get_raw(gm_session* s, uint64_t id, void* host, uint64_t bytes);
/* Copy only the locally owned tiles into `host` (a full-size image); the
 * remaining bytes are left untouched. */
int gm_matrix_get_local_raw(gm_session* s, uint64_t id, void* host, uint64_t bytes);
/* Packed local-tile I/O for one-process-per-GPU use: `host` holds this
 * process's tiles back to back in layout order, each row-major and dense
 * (rowCount x colCount). Bytes must equal the local tiles' total. The
 * matrix version moves exactly like setData. */
int gm_matrix_local_bytes(gm_session* s, uint64_t id, uint64_t* bytes);
int gm_matrix_set_local_packed(gm_session* s, uint64_t id, const void* host, uint64_t bytes);
int gm_matrix_get_local_packed(gm_session* s, uint64_t id, void* host, uint64_t bytes);
/* Asynchronous packed local I/O (stream-ordered; `host` must stay valid and
 * unmodified until gm_session_synchronize; pin it for real overlap).
 * Uploads move in row chunks of ~chunk_bytes (0 = 256 MiB) on a side stream;
 * the next gm_gemm* reading the tile in place starts each of its row chunks
 * as soon as the rows it needs have landed, and a download of its C drains
 * behind the GEMM's row chunks. Version bumps as for the synchronous calls. */
int gm_matrix_set_local_packed_async(gm_session* s, uint64_t id, const void* host, uint64_t bytes,
                                     uint64_t chunk_bytes);
int gm_matrix_get_local_packed_async(gm_session* s, uint64_t id, void* host, uint64_t bytes);
/* Redistribution (reference Session::reshape, session.cpp:310-325): new
 * layout and/or storage precision (new_prec < 0 keeps it); version + 1,
 * replicas reset; values converted like convertBuffer. */
int gm_matrix_reshape(gm_session* s, uint64_t id, const gm_tile* tiles, uint32_t ntiles,
                      int32_t new_prec);
int gm_matrix_info(gm_session* s, uint64_t id, uint64_t* rows, uint64_t* cols, int32_t* prec,
                   uint64_t* version, uint64_t* replicated_version);

/* gridmath::gemm (session.hpp:161-162): synchronous like the reference
 * (returns once every worker finished; errors aggregated). */
int gm_gemm(gm_session* s, uint64_t a, uint64_t b, uint64_t c, double alpha, double beta,
            int32_t trans_a, int32_t trans_b);
/* Same op with the Single-compute math mode in flags[3]. */
int gm_gemm_ex(gm_session* s, uint64_t a, uint64_t b, uint64_t c, double alpha, double beta,
               int32_t trans_a, int32_t trans_b, int32_t math);
/* Asynchronous issue: enqueue on the workers' streams and return; pair
 * with gm_session_synchronize. Used by the benchmark to time on-device. */
int gm_gemm_async(gm_session* s, uint64_t a, uint64_t b, uint64_t c, double alpha, double beta,
                  int32_t trans_a, int32_t trans_b);
int gm_session_synchronize(gm_session* s);

/* FC-layer neighbours of the GEMM (reference session.hpp:163-174; SURVEY
 * 8(f)2), synchronous like gm_gemm. The owner of each destination tile
 * computes it on its GPU; operands in other layouts are gathered like GEMM
 * panels (replica, own tile, panel cache, else copy-engine pulls). Compute
 * type: double iff any operand is Double, else float (kernels.cpp:136-140);
 * results are bit-for-bit the reference's (except subnormal Half inputs,
 * which the device widens IEEE-exactly). */
int gm_set_const(gm_session* s, uint64_t m, double value);                     /* session.cpp:603-608 */
int gm_add_row_col_sum(gm_session* s, uint64_t a, uint64_t row_acc, uint64_t col_acc,
                       double alpha, int32_t deterministic);                   /* session.cpp:547-556 */
int gm_relu(gm_session* s, uint64_t x, uint64_t dst);                          /* session.cpp:580 */
int gm_mul_scalar(gm_session* s, uint64_t x, double alpha);                    /* session.cpp:581-583 */
int gm_add_matrices(gm_session* s, uint64_t x, uint64_t y, uint64_t dst);      /* session.cpp:584-586 */
int gm_sub_matrices(gm_session* s, uint64_t x, uint64_t y, uint64_t dst);      /* session.cpp:587-589 */
int gm_axpy(gm_session* s, double alpha, uint64_t x, uint64_t y);              /* session.cpp:590-592 */
int gm_relu_grad(gm_session* s, uint64_t preact, uint64_t grad);               /* session.cpp:593-595 */
int gm_bias_add(gm_session* s, uint64_t x, uint64_t bias);                     /* session.cpp:596-598 */
int gm_copy_matrix(gm_session* s, uint64_t src, uint64_t dst);                 /* session.cpp:599-601 */
int gm_cast_precision(gm_session* s, uint64_t src, uint64_t dst);              /* session.cpp:602 */
/* Issue one wire op (reference OpDescriptor, ops.hpp:47-60: opcode numbering
 * of OpCode, ids[4], s0, s1, flags[4]) for the device-path opcodes Gemm,
 * SetConst, EwUnary, EwBinary, AddRowColSum. sync = 0: stream-ordered only
 * (pair with gm_session_synchronize). */
#define GM_OP_SET_CONST 5
#define GM_OP_GEMM 6
#define GM_OP_ADD_ROW_COL_SUM 7
#define GM_OP_EW_UNARY 8
#define GM_OP_EW_BINARY 9
int gm_op_issue(gm_session* s, int32_t opcode, const uint64_t ids[4], double s0, double s1,
                const uint8_t flags[4], int32_t sync);

/* Pipeline recording (reference Session::beginRecord / endRecord / replay,
 * session.cpp:385-409). Between begin and end, only recordable ops may be
 * issued (SetConst, Gemm, AddRowColSum, EwUnary, EwBinary, ReplicateStart;
 * anything else fails with "op not recordable inside an open pipeline
 * recording"); they execute normally and are remembered. gm_replay re-issues
 * the steps with fresh exec ids and returns when the device work is done;
 * gm_replay_async only enqueues it. */
int gm_begin_record(gm_session* s, uint64_t* pipeline_id);
int gm_end_record(gm_session* s);
int gm_replay(gm_session* s, uint64_t pipeline_id);
int gm_replay_async(gm_session* s, uint64_t pipeline_id);

/* Replication (session.hpp:81-84). */
int gm_replicate_async(gm_session* s, uint64_t id, uint64_t* version);
int gm_replicate_sync(gm_session* s, uint64_t id);
int gm_replicate_wait(gm_session* s, uint64_t id, uint64_t version, int32_t* state);
int gm_replicate_state(gm_session* s, uint64_t id, uint64_t version, int32_t* state);

/* Introspection (session.hpp:101-112). */
typedef struct {
  uint64_t os_allocations, reuses, frees, held_bytes, resident_bytes;
  uint64_t cache_hits, cache_misses, cache_bytes; /* panel cache */
  uint64_t bytes_sent, bytes_received;            /* data plane */
} gm_worker_stats;
int gm_query_worker_stats(gm_session* s, gm_worker_stats* rows, uint32_t cap, uint32_t* n);
int gm_verify_metadata(gm_session* s);
int gm_session_local_workers(gm_session* s, uint32_t* ranks, uint32_t cap, uint32_t* n);
/* Data plane the session chose: GM_TRANSPORT_PEER_COPY (one process, peer
 * copies), GM_TRANSPORT_NCCL, GM_TRANSPORT_IPC (one process per GPU, copy
 * engines pulling peer tiles over CUDA IPC, ordered by device-side flags). */
#define GM_TRANSPORT_PEER_COPY 0
#define GM_TRANSPORT_NCCL 1
#define GM_TRANSPORT_IPC 2
int gm_session_transport(gm_session* s, int32_t* kind);
/* In-GEMM panel pipelining (default on): gathered bands land block by block
 * while the GEMM runs, its producer polling per-block ready flags. 0 turns
 * it off for later GEMMs of this session (they wait for whole bands). Local
 * to this process (SPMD ranks may differ). */
int gm_session_set_panel_pipelining(gm_session* s, int32_t on);
/* Pipeline replay as one CUDA graph per process (default off, or
 * GM_DEBUG_CONFIG graph_replay=1): the first replay of a pipeline runs op by
 * op, later ones are stream-captured and launched as one graph whose
 * executable is updated in place. The reference's replay is one control
 * message per step (session.cpp:385-409); bitwise the same results either
 * way. Off by default because the graph boundary serialises consecutive
 * steps (measured slower). */
int gm_session_set_graph_replay(gm_session* s, int32_t on);
/* Launches, instantiations (over all pipelines) and node count of the last
 * captured replay graph. */
int gm_session_graph_stats(gm_session* s, uint64_t* launches, uint64_t* instantiations, uint64_t* nodes);
/* Developer timeline of later replays (not in the reference): with on != 0,
 * every replay records device events on the first local worker's compute and
 * comm streams at its start and after each replayed op. gm_session_op_timeline
 * returns, for the last replay, the ms from its start at which each stream
 * passed each op, and the op labels joined by '\n' into `labels`. */
int gm_session_set_op_timeline(gm_session* s, int32_t on);
int gm_session_op_timeline(gm_session* s, float* compute_ms, float* comm_ms, uint32_t cap, char* labels,
                           uint32_t label_bytes, uint32_t* n);
/* Device time of the last gm_gemm/gm_gemm_async per local worker (ms),
 * measured with CUDA events on the worker's compute stream. */
int gm_last_op_device_ms(gm_session* s, float* ms, uint32_t cap, uint32_t* n);
/* Same, restricted to the local GEMM kernels of the last gemm (no exchange). */
int gm_last_op_kernel_ms(gm_session* s, float* ms, uint32_t cap, uint32_t* n);
/* Per local worker: summed duration of the local GEMM kernels (compute
 * phase) of every gemm issued between gm_timer_start and gm_timer_stop, and
 * the number of those gemms (average kernel time = ms_sum / count). */
int gm_timer_kernel_ms(gm_session* s, float* ms_sum, uint32_t* count, uint32_t cap, uint32_t* n);
/* Duration of the last gemm's panel exchange on each local worker's comm
 * stream (0 when nothing moved). */
int gm_last_op_comm_ms(gm_session* s, float* ms, uint32_t cap, uint32_t* n);

/* Device timer over everything enqueued on the local workers' compute
 * streams between start and stop (CUDA events on those streams). stop
 * synchronizes and returns the max over local workers, in ms. */
int gm_timer_start(gm_session* s);
int gm_timer_stop(gm_session* s, float* max_ms);

/* Number of this library's kernels launched by this process so far (GEMM,
 * conversion, staging kernels). */
int gm_kernel_launches(uint64_t* count);

#ifdef __cplusplus
}
#endif

#endif /* GRIDMATH_B200_H */
