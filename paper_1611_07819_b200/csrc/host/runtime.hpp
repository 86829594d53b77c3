// SPDX-License-Identifier: Apache-2.0
// Master / worker runtime of the B200 drop-in (namespace gridmath).
//
// Reference structure kept (proj/include/gridmath/session.hpp:62-179,
// worker.hpp:63-139): a master `Session` owns the descriptor table and issues
// OpDescriptors; every worker mirrors the table via applyOpMetadata and
// executes the op on its own tiles. What changes is where things live:
//   * one worker per GPU slot: tiles, replicas and cached panels are device
//     buffers from a per-worker pooled arena (DeviceArena);
//   * a worker's "thread" is its pair of CUDA streams (compute + comm); the
//     master enqueues async device work instead of waking host threads;
//   * the data plane is copy-engine peer copies (all workers in one
//     process) or NCCL point-to-point / broadcast (one process per GPU,
//     SPMD: every process runs the master logic redundantly -- planning is a
//     pure function of the replicated descriptor table, so all ranks agree on
//     every transfer without negotiation, like the reference's
//     "same pure planning functions on every actor", pieces.hpp:29-31).
#pragma once

#include <cuda_runtime.h>

#include <array>
#include <cstdint>
#include <deque>
#include <functional>
#include <list>
#include <map>
#include <memory>
#include <mutex>
#include <optional>
#include <set>
#include <string>
#include <tuple>
#include <utility>
#include <vector>

#include "../../../include/gridmath_b200.h"
#include "capture.hpp"
#include "core.hpp"
#include "device.hpp"
#include "ops.hpp"

// NCCL's handle type (nccl.h: typedef struct ncclComm* ncclComm_t), so that
// callers of this header do not need NCCL's headers.
typedef struct ncclComm* ncclComm_t;

namespace gridmath {

class Session;

// ---- introspection types of the reference's public Session surface
// (trace.hpp:13-64, fabric.hpp:21-49), filled by the B200 runtime.
enum class EventKind : std::uint8_t {
  PhaseMark,       // master annotation; label carries the phase name
  OpStart,         // a worker's device work for an op is issued (a = execId, b = opcode)
  OpComputeStart,
  OpComputeEnd,
  OpEnd,
  ReplInitiate,    // a = matrixId, b = version
  ReplChunkSent,
  ReplicaValid,    // this worker's full copy became readable (a = matrixId, b = version)
  ReplFailed,
  BatchProduced,
  BatchConsumed,
};

struct TraceEvent {
  std::uint64_t seq = 0;
  std::int64_t actor = 0;  // worker rank, -1 for master
  EventKind kind{};
  std::uint64_t a = 0;
  std::uint64_t b = 0;
  std::string label;
};

// Append-only host event log with a total order (sequence numbers).
class EventTrace {
 public:
  std::uint64_t record(std::int64_t actor, EventKind kind, std::uint64_t a = 0, std::uint64_t b = 0,
                       std::string label = {});
  std::vector<TraceEvent> snapshot() const;
  void clear();

 private:
  mutable std::mutex mu_;
  std::uint64_t seq_ = 0;
  std::vector<TraceEvent> events_;
};

enum class MsgKind : std::uint8_t { Control = 0, Data = 1, Completion = 2 };

struct LinkStats {
  std::uint64_t messageCount = 0;
  std::uint64_t byteCount = 0;  // payload bytes
};

// Per (src, dst) worker pair: Control = ops mirrored to the worker (src =
// master, 0xFFFFFFFF), Data = pieces pulled over the data plane (one
// message per 2D copy), Completion = worker acknowledgements.
struct FabricStats {
  std::map<std::pair<std::uint32_t, std::uint32_t>, std::array<LinkStats, 3>> perLink;
  LinkStats totalByKind(MsgKind k) const;
  LinkStats total() const;
};

inline constexpr std::uint32_t kMasterRank = 0xFFFFFFFFu;

namespace kernels {
// Reference kernels.hpp:68-78 (the conv op is outside the B200 GEMM path;
// declared so reference call sites compile).
struct ConvGeometry {
  std::uint32_t batch = 0;
  std::uint32_t channels = 0, height = 0, width = 0;
  std::uint32_t kernels = 0, kh = 0, kw = 0;
  std::uint32_t stride = 1, pad = 0;
  std::uint32_t outH() const { return (height + 2 * pad - kh) / stride + 1; }
  std::uint32_t outW() const { return (width + 2 * pad - kw) / stride + 1; }
};
}  // namespace kernels

class DistMatrix {
 public:
  DistMatrix() = default;
  DistMatrix(Session* s, std::uint64_t id) : session_(s), id_(id) {}
  std::uint64_t id() const { return id_; }
  std::uint64_t rows() const;
  std::uint64_t cols() const;
  Precision precision() const;
  bool valid() const { return session_ != nullptr; }

 private:
  Session* session_ = nullptr;
  std::uint64_t id_ = 0;
};

enum class ReplState : std::uint8_t { InFlight, Done, Failed };

struct ReplicationHandle {
  std::uint64_t matrixId = 0;
  std::uint64_t version = 0;
};

struct SessionOptions {
  std::uint32_t workers = 1;
  bool deterministic = true;
  std::uint64_t replicationChunkBytes = 1ull << 20;
  std::uint64_t rootSeed = 0;
  bool checkMetadataEveryOp = false;
  // --- B200 placement / data plane ---
  int spmdRank = -1;                  // >= 0: this process hosts only worker spmdRank
  std::vector<int> devices;           // worker r -> devices[r % size]; empty = all visible
  std::array<std::uint8_t, 128> ncclId{};
  int gemmMaxCtas = 0;                // cap the GEMM grid (0 = all SMs)
  std::uint64_t panelCacheBytes = 0;  // per worker; 0 = 1/4 of device memory
  // Data plane. 0 auto: copy engines (single process: peer copies; SPMD:
  // CUDA IPC pulls ordered by device-side flags) when every peer GPU is
  // mappable, else NCCL. 1 forces NCCL point-to-point; 2 requires copy engines.
  int transport = 0;
  int pipelineChunks = 0;             // SUMMA row chunks (0 = auto)
  // SPMD control channel: blocking in-place max-reduce of host bytes over
  // all ranks. Empty: an NCCL communicator carries it. Set: no NCCL at all
  // (ranks may share a GPU); the data plane must be the IPC copy engines.
  std::function<void(void*, std::size_t)> controlAllreduceMax;
};

struct WorkerStatsRow {
  std::uint64_t osAllocations = 0, reuses = 0, frees = 0, heldBytes = 0, residentBytes = 0;
  std::uint64_t cacheHits = 0, cacheMisses = 0, cacheBytes = 0;
  std::uint64_t bytesSent = 0, bytesReceived = 0;
};

struct DeviceTile {
  TileExtent extent;
  void* ptr = nullptr;
  std::uint64_t ld = 0;  // pitch in elements (16-byte multiple when possible)
};

// "Keep what you've seen": operand bands a worker gathered for a GEMM stay
// resident, keyed by (matrix, version, rect), and are reused by later GEMMs
// that need the same region (e.g. W gathered in the forward pass, read again
// transposed by the backward dX GEMM). Entries die when the matrix version
// moves or the matrix is destroyed; LRU eviction keeps the cache within its
// byte budget. The directory is replicated on every SPMD rank (metadata
// only for non-local workers) and updated by the same deterministic rules,
// so every rank knows which transfers a peer will post.
struct CacheEntry {
  std::uint64_t matrixId = 0, version = 0;
  Rect rect;
  std::uint64_t bytes = 0;
  std::uint64_t lastUse = 0;
  void* ptr = nullptr;  // local workers only
  std::uint64_t ld = 0;
  cudaEvent_t ready = nullptr;
};

class PanelCache {
 public:
  CacheEntry* lookup(std::uint64_t id, std::uint64_t version, const Rect& r, std::uint64_t tick);
  bool contains(std::uint64_t id, std::uint64_t version, const Rect& r) const;
  // Returns entries evicted to make room (caller frees their buffers).
  std::vector<CacheEntry> reserve(std::uint64_t bytes, std::uint64_t budget, std::uint64_t protectTick);
  CacheEntry& insert(CacheEntry e);
  std::vector<CacheEntry> dropMatrix(std::uint64_t id, bool keepCurrent, std::uint64_t version);
  std::vector<CacheEntry> dropAll();
  std::uint64_t bytes() const { return bytes_; }
  std::uint64_t hits = 0, misses = 0;

 private:
  std::list<CacheEntry> entries_;
  std::uint64_t bytes_ = 0;
};

enum class ReplicaState : std::uint8_t { Valid = 0, Pending = 1, Stale = 2 };

struct ReplicaEntry {
  void* full = nullptr;  // whole matrix, row-major, pitch `ld`
  std::uint64_t ld = 0;
  // The worker owns the whole matrix as one tile: `full` is that tile (no
  // copy, not owned by the entry). Mutations bump the version, so a replica
  // read only ever sees the version it was made for.
  bool alias = false;
  std::uint64_t version = 0;
  ReplicaState state = ReplicaState::Pending;
  cudaEvent_t ready = nullptr;
  // One u64 per layout tile (source piece) of the matrix: the replication
  // job's pull stream writes pieceReady[t] = version once tile t's copy has
  // landed, so a GEMM reading the replica can start on the pieces already
  // there (e.g. the next step's forward behind W's re-replication).
  std::uint64_t* pieceReady = nullptr;
  std::uint32_t pieces = 0;
};

struct BandView {
  const void* ptr = nullptr;
  std::uint64_t ld = 0;
};

// Per-worker device state (reference WorkerRuntime, worker.hpp:63-139).
class Worker {
 public:
  Worker(std::uint32_t rank, int device, std::uint64_t cacheBudget);
  ~Worker();
  Worker(const Worker&) = delete;
  Worker& operator=(const Worker&) = delete;

  void activate() const;
  cudaEvent_t event();            // from a recycled pool
  void recycle(cudaEvent_t e);
  void* workspace(std::uint64_t bytes);
  // Stream-ordered WAR guard, per matrix: readers of this worker's tiles of
  // a matrix register their completion events; the compute stream waits on
  // them before that matrix is mutated or freed. `owner` is the worker whose
  // pool the event came from (recycled there).
  void addReader(std::uint64_t matrix, cudaEvent_t e, Worker* owner) { readers_[matrix].push_back({e, owner}); }
  void beforeMutation(std::uint64_t matrix, cudaStream_t on = nullptr);  // default: compute
  void releaseReaders();
  // RAW: event on the compute stream after the last op that wrote this
  // worker's tiles of a matrix; readers on other streams wait on it instead
  // of on the whole compute stream (so the next op's panel pulls overlap
  // the current GEMM).
  std::map<std::uint64_t, cudaEvent_t> lastWrite;
  // Event on the compute stream after the last op that used (read or wrote)
  // this worker's tiles of a matrix there: an asynchronous upload into the
  // matrix waits on it instead of on everything the compute stream holds, so
  // it overlaps compute that does not involve the matrix.
  std::map<std::uint64_t, cudaEvent_t> lastTouch;
  // SPMD copy-engine plane: this rank's flag page (device memory, mapped by
  // every peer): written[slot], then readDone[stream][slot].
  std::uint64_t* flags = nullptr;

  // In-GEMM panel pipelining: a ring of u64 ready flags in device memory.
  // The pull streams write a block's flag once its pieces landed; the GEMM
  // producer polls it. Each pipelined GEMM takes a fresh region (values are
  // a per-worker sequence number); a region is handed out again only after
  // the GEMM that polled it has finished (the comm stream waits on its done
  // event), so no kernel ever sees a later op's write.
  std::uint64_t readyCap = 1ull << 16;  // slots (GM_DEBUG_CONFIG ready_slots overrides)
  std::uint64_t* readyFlags = nullptr;
  std::uint64_t readyHead = 0;  // monotonic slot counter (memory slot = head % readyCap)
  std::uint64_t readySeq = 0;   // last published value
  struct ReadyRegion {
    std::uint64_t first = 0, end = 0;
    cudaEvent_t done = nullptr;  // on compute, after the GEMM that polls the region
  };
  std::deque<ReadyRegion> readyInUse;
  // Reserves n contiguous slots; returns the monotonic start. Makes the comm
  // stream wait for every earlier GEMM whose region the new one may reuse.
  std::uint64_t reserveReady(std::uint64_t n);

  // Host<->device streaming (asynchronous packed local I/O): uploads run on
  // `h2d` in row chunks, each with an event, so a GEMM can start on the rows
  // that have landed; downloads run on `d2h` behind the producing op's
  // per-chunk events. Until an op joins it, a matrix's pending upload is
  // the authority for its tiles' contents (flushWritten publishes it from
  // the h2d stream).
  struct UploadChunk {
    std::uint64_t r0 = 0, r1 = 0;  // global rows of the matrix
    cudaEvent_t done = nullptr;
  };
  struct Upload {
    std::vector<UploadChunk> chunks;
    cudaEvent_t done = nullptr;  // after the last chunk
  };
  std::map<std::uint64_t, Upload> uploads;
  // Row-chunk completion events of the last op that wrote a matrix in
  // chunks (the GEMM's S row chunks), for chunked downloads.
  std::map<std::uint64_t, std::vector<UploadChunk>> chunkDone;
  void joinUpload(std::uint64_t matrix);  // compute stream waits; entry dropped
  void dropChunkDone(std::uint64_t matrix);

  std::uint32_t rank;
  int device;
  cudaStream_t compute = nullptr, comm = nullptr, h2d = nullptr, d2h = nullptr;
  // Forked from and joined back into `compute` inside one op (e.g. the
  // column sums of addRowColSum run beside the row sums).
  cudaStream_t aux = nullptr;
  // SPMD copy-engine plane: written[slot] flags are published here, behind
  // the write's event, when a peer first pulls the matrix (not on compute).
  cudaStream_t flagPub = nullptr;
  // ...and peers' readDone flags are awaited here before a mutation (the
  // compute stream then waits on one event instead of one memop per reader).
  cudaStream_t warWait = nullptr;
  // Copy-engine pull streams: one exchange's pieces from different source
  // workers run on different streams (different copy engines), forked from
  // and joined back into the comm or compute stream.
  static constexpr int kPullStreams = 4;
  std::array<cudaStream_t, kPullStreams> pulls{};
  DeviceArena arena;
  DescriptorTable descs;
  std::map<std::uint64_t, std::vector<DeviceTile>> tiles;
  std::map<std::uint64_t, ReplicaEntry> replicas;
  PanelCache cache;
  std::uint64_t cacheBudget;
  std::uint64_t residentBytes = 0, bytesSent = 0, bytesReceived = 0;
  cudaEvent_t tStart = nullptr, tEnd = nullptr, uStart = nullptr, uEnd = nullptr;
  cudaEvent_t kStart = nullptr;  // compute phase of the last gemm (ends at tEnd)
  cudaEvent_t cStart = nullptr, cEnd = nullptr;  // comm-stream exchange of the last gemm
  bool commTimed = false;
  bool timed = false;
  // Compute phase of every gemm between timerStart() and timerStop()
  // (timing-enabled event pairs, drained by timerKernelMs()).
  bool windowOpen = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> kernelWindow;
  ncclComm_t nccl = nullptr;

 private:
  std::vector<cudaEvent_t> pool_;
  std::map<std::uint64_t, std::vector<std::pair<cudaEvent_t, Worker*>>> readers_;
  void* ws_ = nullptr;
  std::uint64_t wsBytes_ = 0;
};

// One movement of a sub-rectangle between workers (reference PieceRoute,
// pieces.hpp:33-40). Pointers are valid only on the side that is local.
struct Xfer {
  std::uint32_t src = 0, dst = 0;
  const void* srcPtr = nullptr;
  std::uint64_t srcLd = 0;
  void* dstPtr = nullptr;
  std::uint64_t dstLd = 0;
  std::uint64_t rows = 0, cols = 0;
  std::uint32_t eb = 0;
  std::uint64_t matrix = 0;  // source matrix id (RAW/WAR tracking)
  // Global origin of the piece in the source matrix (set by planners that
  // can; enables per-chunk waits on a chunked upload of the source).
  bool hasOrigin = false;
  std::uint64_t r0 = 0, c0 = 0;
  // Panel pipelining (consumer side): the copy runs on pull stream
  // `pullStream` (else by source), and when `lastOfBlock` is set that stream
  // then writes *flagAddr = flagValue (the block has landed).
  int pullStream = -1;
  bool lastOfBlock = false;
  std::uint64_t* flagAddr = nullptr;
  std::uint64_t flagValue = 0;
};

// Pure GEMM planning (no device state): merged C row/col intervals per
// worker and one need per interval over the full k range, resolved to the
// replica, a containing local tile, a cached panel (probe callback), or a
// gather from the owners of the intersecting tiles (reference planGemm,
// kernels.cpp:204-251, and NeedPlanner::addNeed, pieces.cpp:14-30).
struct PlannedNeed {
  enum Kind : std::uint8_t { Replica, LocalTile, Cached, Gather } kind = Gather;
  std::uint32_t worker = 0;
  int operand = 0;  // 0 = A, 1 = B
  std::size_t interval = 0;
  Rect rect;
  std::vector<PieceRoute> pieces;  // Gather only (src == worker allowed)
};

struct GemmPlanB200 {
  std::uint64_t m = 0, n = 0, k = 0;
  bool transA = false, transB = false;
  std::vector<std::vector<std::pair<std::uint64_t, std::uint64_t>>> rowsOf, colsOf;
  std::vector<PlannedNeed> needs;  // worker-major: A intervals then B intervals
};

using CacheProbe = std::function<bool(std::uint32_t worker, const MatrixDescriptor&, const Rect&)>;
GemmPlanB200 planGemmB200(const DescriptorTable& t, const OpDescriptor& op, std::uint32_t workers,
                          const CacheProbe& cached);
// Remote bytes each worker receives under `plan` (the panel-traffic figure).
std::vector<std::uint64_t> planRemoteBytes(const GemmPlanB200& plan, const DescriptorTable& t,
                                           std::uint32_t workers);

class Session {
 public:
  explicit Session(SessionOptions opts = {});
  ~Session();
  Session(const Session&) = delete;
  Session& operator=(const Session&) = delete;

  DistMatrix createMatrix(std::uint64_t rows, std::uint64_t cols, Precision p, const Layout& layout);
  // Creates a matrix with a caller-chosen descriptor (id, version, layout);
  // reference Session::createWithDescriptor (session.cpp:200-218).
  DistMatrix createWithDescriptor(const MatrixDescriptor& d);
  void destroy(DistMatrix m);
  void setData(DistMatrix m, const std::vector<double>& rowMajor);
  void setDataF32(DistMatrix m, const std::vector<float>& rowMajor);
  void setDataRaw(DistMatrix m, const void* image, std::uint64_t bytes);
  void fillUniform(DistMatrix m, std::uint64_t seed, double lo, double hi);
  std::vector<double> getData(DistMatrix m);
  std::vector<std::uint8_t> getDataRaw(DistMatrix m);
  void getDataRawInto(DistMatrix m, void* image, std::uint64_t bytes, bool localOnly);
  // Redistribution (reference Session::reshape, session.cpp:310-325, and
  // execReshape, kernels.cpp:1083-1127): new layout and/or storage precision.
  void reshape(DistMatrix m, const Layout& newLayout, std::optional<Precision> newPrecision = std::nullopt);

  // Checkpoint-restart in the reference's DMCK format (session.cpp:413-480):
  // "DMCK", u32 version 1, u64 root seed, u32 count, per matrix (ascending
  // id) its descriptor and full row-major image, then the zlib CRC-32 of
  // everything after the magic. Files are interchangeable with the
  // reference's. Under SPMD every rank gathers, rank 0 writes; restore is
  // collective (every rank reads the file).
  void checkpoint(const std::string& path);
  static std::unique_ptr<Session> restore(const std::string& path, SessionOptions opts);

  // Pipeline recording (reference session.cpp:385-409): recordable ops
  // (SetConst, Gemm, AddRowColSum, EwUnary, EwBinary, ReplicateStart) issued
  // between beginRecord and endRecord execute normally and are remembered;
  // replay re-issues the steps with fresh exec ids (same metadata walk).
  // replay is synchronous like the reference's; sync = false leaves the
  // device work stream-ordered.
  std::uint64_t beginRecord();
  void endRecord();
  void replay(std::uint64_t pipelineId, bool sync = true);
  // Replays after a pipeline's first run as one CUDA graph per process
  // (capture.hpp). Off by default (measured slower);
  // GM_DEBUG_CONFIG graph_replay=1 or setGraphReplay(true) turns it on.
  void setGraphReplay(bool on) { graphReplay_ = on; }
  struct GraphStats {
    std::uint64_t launches = 0, instantiations = 0, nodes = 0;  // nodes: last captured graph
  };
  GraphStats graphStats() const { return graphStats_; }
  // Developer timeline of the next replays: device time (ms, from the
  // replay's start on the first local worker's compute stream) at which its
  // compute and comm streams passed the end of each replayed op.
  void setOpTimeline(bool on) { opTimeline_ = on; }
  struct TimelineEntry {
    std::string label;
    float computeMs = 0.0f, commMs = 0.0f;
  };
  std::vector<TimelineEntry> opTimeline();

  ReplicationHandle replicateAsync(DistMatrix m);
  void replicateSync(DistMatrix m);
  ReplState wait(const ReplicationHandle& h);
  ReplState handleState(const ReplicationHandle& h);

  void verifyMetadataConsistency();
  std::vector<WorkerStatsRow> queryWorkerStats();
  // --- rest of the reference's public surface (session.hpp:86-124)
  // Seeds: every worker's generator seed is deriveSeed(root, rank).
  void distributeSeeds(std::uint64_t rootSeed);
  std::uint64_t rootSeed() const { return rootSeed_; }
  // The master keeps no pooled host buffers here (device arenas are per
  // worker, queryWorkerStats): all-zero row.
  WorkerStatsRow masterPoolStats() const { return {}; }
  FabricStats fabricStats() const;
  EventTrace& trace() { return trace_; }
  void phaseMark(const std::string& label);
  double simulatedElapsed() const { return 0.0; }  // no simulated fabric on the device runtime
  const Worker& workerForTest(std::uint32_t rank) const;
  // Op plumbing: validate, apply metadata and execute any op the runtime
  // executes (Gemm, SetConst, EwUnary, EwBinary, AddRowColSum,
  // ReplicateStart) stream-ordered; awaitAcks waits for the local workers
  // and returns their acknowledgements. extraExecIds is kept for source
  // compatibility (every op takes one exec id here).
  std::uint64_t issueOp(OpDescriptor op, std::uint64_t extraExecIds = 0);
  std::vector<std::pair<std::uint32_t, Completion>> awaitAcks(std::uint64_t execId);
  const MatrixDescriptor& descriptor(std::uint64_t id) const;
  const DescriptorTable& table() const { return table_; }
  std::uint32_t workerCount() const { return opts_.workers; }
  bool deterministic() const { return opts_.deterministic; }
  const SessionOptions& options() const { return opts_; }
  std::vector<std::uint32_t> localRanks() const;
  // 0 = copy engine (one process), 1 = NCCL, 2 = CUDA IPC copy engine (SPMD).
  int transportKind() const { return ipc_ ? 2 : (nccl_ ? 1 : 0); }
  // In-GEMM panel pipelining on/off for later GEMMs (consumer-local).
  void setPanelPipelining(bool on) { panelPipelining_ = on; }

  // Issues a Gemm op (gemm() below wraps it). sync: wait for completion
  // like the reference's acked gemm(); otherwise stream-ordered only.
  void runGemm(const OpDescriptor& op, bool sync);
  // Replay peephole: gemm(C) -> biasAdd(C, b) -> relu(C -> act), all bf16,
  // runs as one GEMM whose epilogue adds the bias and writes act (the three
  // ops' metadata, versions and hazards are applied as if run one by one).
  struct FusedBiasRelu {
    std::uint64_t act = 0;
    std::map<std::tuple<std::uint32_t, std::uint64_t, std::uint64_t>, const void*> bias;  // (rank, row0, col0)
  };
  const FusedBiasRelu* fused_ = nullptr;
  bool fusableBiasRelu(const std::vector<OpDescriptor>& ops, std::size_t i) const;
  void replayOps(const std::vector<OpDescriptor>& ops);
  // Replay peephole: setConst(R, 0) and setConst(C, 0) right before
  // addRowColSum(X, R, C) issue only their metadata; the sums then write
  // 0 + alpha * sum (same bits, two launches fewer).
  bool fusableZeroSums(const std::vector<OpDescriptor>& ops, std::size_t i) const;
  bool zeroSums_ = false;
  void runGemmBiasRelu(const OpDescriptor& g, const OpDescriptor& bo, const OpDescriptor& ro);
  // FC-layer neighbours on device (reference session.cpp:547-609,
  // kernels.cpp:435-815): SetConst, EwUnary, EwBinary, AddRowColSum.
  // Same sync contract as runGemm.
  void runPointwise(const OpDescriptor& op, bool sync);
  void synchronize();
  std::vector<float> lastOpDeviceMs();
  std::vector<float> lastOpKernelMs();
  std::vector<float> lastOpCommMs();
  std::uint64_t localBytes(DistMatrix m) const;
  void setLocalPacked(DistMatrix m, const void* host, std::uint64_t bytes);
  void getLocalPacked(DistMatrix m, void* host, std::uint64_t bytes);
  // Asynchronous variants (stream-ordered; the host buffer must stay valid
  // and unmodified until synchronize()). Uploads move in row chunks of about
  // `chunkBytes` on the workers' h2d streams; a following GEMM that reads
  // the tile in place starts on each row chunk as it lands. Downloads follow
  // the producing GEMM's row chunks on the d2h streams. Pinned host memory
  // makes them truly asynchronous.
  void setLocalPackedAsync(DistMatrix m, const void* host, std::uint64_t bytes, std::uint64_t chunkBytes = 0);
  void getLocalPackedAsync(DistMatrix m, void* host, std::uint64_t bytes);
  void timerStart();
  float timerStop();
  // Per local worker: {sum of gemm compute-phase ms, gemm count} over the
  // last timerStart()/timerStop() window.
  std::vector<std::pair<float, std::uint32_t>> timerKernelMs();

 private:
  std::uint64_t issue(OpDescriptor& op);  // validate + metadata + per-worker mirror
  void requireRecordable(OpCode c) const;
  void joinUploads(const OpDescriptor& op);
  Worker* local(std::uint32_t rank) const;
  bool isLocal(std::uint32_t rank) const;
  void execCreate(const OpDescriptor& op);
  void execDestroy(std::uint64_t id);
  void execGemm(const OpDescriptor& op);
  void execReplicate(std::uint64_t id);
  void execSetConst(const OpDescriptor& op);
  // A read of `rect` of a matrix by `worker` (reference NeedPlanner::addNeed
  // with allowReplica, pieces.cpp:14-30): resolved to the local replica, a
  // containing local tile, a cached panel, or a gather into a dense temp.
  struct ReadNeed {
    std::uint32_t worker = 0;
    std::uint64_t matrix = 0;
    Rect rect;
    BandView view;  // filled for local workers
  };
  void resolveReads(std::vector<ReadNeed>& needs, std::uint64_t mutated, std::vector<Xfer>& xs,
                    std::vector<std::pair<Worker*, void*>>& temps);
  // toH2d: the mutation is an asynchronous upload on the h2d streams -- the
  // WAR waits land there instead of on the compute streams.
  void mutationHook(std::uint64_t id, std::uint64_t oldVersion, bool toH2d = false);
  std::vector<std::uint64_t> pendingTouched_;  // matrices the previous op used
  // maxPull caps the copy-engine pull streams this exchange spreads its
  // sources over (0 = all of Worker::kPullStreams).
  void exchange(std::vector<Xfer>& xs, bool onComm, bool commit = true, int maxPull = 0);
  // --- RAW/WAR bookkeeping shared by the planes
  void flushWritten(std::uint64_t before);  // publish mutations of ops with exec id < before
  void commitReads();    // consumers publish readDone for this op's pulls
  void setupIpc();
  // Blocking max-reduce of a small host byte array over all SPMD ranks
  // (control plane: IPC registration, budgets, shutdown).
  void controlMax(void* host, std::size_t n);
  void registerTiles(std::uint64_t id, const std::string& localError);
  void ipcWait(cudaStream_t s, const std::uint64_t* addr, std::uint64_t value);
  void ipcWrite(cudaStream_t s, std::uint64_t* addr, std::uint64_t value);
  std::uint32_t slotOf(std::uint64_t id) const;
  // Source view of `r` (inside one tile of M owned by `src`): a local tile
  // pointer, or the IPC mapping of a peer's tile. {nullptr, 0} if neither.
  BandView srcView(const MatrixDescriptor& M, std::uint32_t src, const Rect& r);
  void forEachLocal(const std::function<void(Worker&)>& f);
  void checkErrors(std::vector<std::string>& errs);

  SessionOptions opts_;
  DescriptorTable table_;
  std::uint64_t rootSeed_ = 0;
  bool panelPipelining_ = true;
  EventTrace trace_;
  mutable std::mutex statsMu_;
  std::map<std::pair<std::uint32_t, std::uint32_t>, std::array<LinkStats, 3>> links_;
  void countLink(std::uint32_t src, std::uint32_t dst, MsgKind k, std::uint64_t bytes);
  std::vector<std::unique_ptr<Worker>> workers_;  // indexed by rank; null if remote
  std::vector<PanelCache> remoteCaches_;          // directory for non-local workers (SPMD)
  // Per pipeline: the captured replay's executable (declared after workers_,
  // so it is destroyed before them).
  std::map<std::uint64_t, std::unique_ptr<capture::Graph>> graphs_;
  std::optional<bool> graphReplay_;
  struct TimelineMark {
    std::string label;
    cudaEvent_t compute = nullptr, comm = nullptr;
  };
  bool opTimeline_ = false;
  std::vector<TimelineMark> timeline_;
  GraphStats graphStats_;
  std::map<std::pair<std::uint64_t, std::uint64_t>, bool> replFailed_;
  std::uint64_t nextMatrixId_ = 1;
  // Chunked uploads that are the last write of a matrix. The op carries the
  // chunk size, so every rank knows each producer's chunk geometry and the
  // value its upload-chunk flag reaches after each chunk: consumers (peer
  // pulls, local copies) wait per chunk instead of for the whole upload.
  struct ChunkedWrite {
    std::uint64_t execId = 0, chunkBytes = 0;
    std::vector<std::uint64_t> base;  // per rank: its upload-chunk counter before this upload
  };
  std::map<std::uint64_t, ChunkedWrite> chunked_;
  std::map<std::pair<std::uint32_t, std::uint32_t>, std::uint64_t> upCount_;  // (rank, slot) -> chunks so far
  const ChunkedWrite* chunkedSource(std::uint64_t matrix) const;
  // Ordinal of the upload chunk holding global row `row` of tile `tileIdx`
  // among its owner's chunks of matrix M (tiles in layout order), and the
  // chunk's global row range.
  static std::uint32_t chunkOrdinal(const MatrixDescriptor& M, std::size_t tileIdx, std::uint64_t row,
                                    std::uint64_t chunkBytes, std::uint64_t* lo, std::uint64_t* hi);
  std::uint64_t recording_ = 0, nextPipelineId_ = 1;
  std::map<std::uint64_t, std::vector<OpDescriptor>> pipelines_;
  std::set<std::uint64_t> closedPipelines_;
  std::uint64_t nextExec_ = 1;
  std::uint64_t tick_ = 0;
  std::uint64_t gemmEpoch_ = 0;  // arena epoch of band temporaries (one per GEMM)
  bool nccl_ = false;
  bool peerCopies_ = false;
  bool ipc_ = false;
  std::uint64_t curExec_ = 0;                              // exec id of the op being executed
  std::map<std::uint64_t, std::uint64_t> lastMut_;         // matrix -> exec id of its last write
  std::vector<std::pair<std::uint64_t, std::uint64_t>> pendingWritten_;  // (matrix, exec id)
  // Writes of local tiles whose written[slot] flag is not published yet
  // (matrix -> exec id): published on flagPub when a peer pulls the matrix.
  std::map<std::uint64_t, std::uint64_t> unpublished_;
  void publishWritten(Worker& w, std::uint64_t matrix);
  // WAR on the SPMD plane: `ws` waits until every peer that pulled worker w's
  // tiles of `matrix` has published readDone for those pulls.
  void waitRemoteReaders(Worker& w, std::uint64_t matrix, cudaStream_t ws);
  std::map<std::uint64_t, std::uint32_t> slots_;           // matrix -> flag slot (same on all ranks)
  std::vector<std::uint32_t> freeSlots_;
  std::uint32_t nextSlot_ = 0;
  // SPMD IPC plane
  std::vector<std::uint64_t*> peerFlags_;                  // rank -> mapped flag page
  std::map<std::pair<std::uint32_t, std::uint64_t>, void*> ipcOpened_;  // (rank, remote base) -> mapping
  std::map<std::uint64_t, std::vector<void*>> peerTiles_;  // matrix -> per layout tile: mapped ptr
  // producer side: matrix -> (consumer, stream) -> exec id of its last pull
  std::map<std::uint64_t, std::map<std::pair<std::uint32_t, int>, std::uint64_t>> remoteReaders_;
  std::set<std::tuple<std::uint32_t, std::uint64_t, int>> pendingReads_;  // (consumer, matrix, stream)
};

void gemm(Session& s, DistMatrix a, DistMatrix b, DistMatrix c, double alpha, double beta,
          bool transA = false, bool transB = false);
// FC-layer neighbours (reference session.hpp:163-174, same signatures).
void addRowColSum(Session& s, DistMatrix a, DistMatrix rowAcc, DistMatrix colAcc, double alpha,
                  bool deterministic);
void relu(Session& s, DistMatrix x, DistMatrix dst);
void mulScalar(Session& s, DistMatrix x, double alpha);
void addMatrices(Session& s, DistMatrix x, DistMatrix y, DistMatrix dst);
void subMatrices(Session& s, DistMatrix x, DistMatrix y, DistMatrix dst);
void axpy(Session& s, double alpha, DistMatrix x, DistMatrix y);
void reluGrad(Session& s, DistMatrix preact, DistMatrix grad);
void biasAdd(Session& s, DistMatrix x, DistMatrix bias);
void copyMatrix(Session& s, DistMatrix src, DistMatrix dst);
void castPrecision(Session& s, DistMatrix src, DistMatrix dst);
void setConst(Session& s, DistMatrix m, double value);
// Outside the B200 GEMM path (reference session.hpp:175-179): declared so
// reference call sites compile; they throw "op not supported on the B200
// GEMM path" before anything is issued.
void softmaxRows(Session& s, DistMatrix a);
void subtractOneHot(Session& s, DistMatrix probs, DistMatrix labels);
double logLossMean(Session& s, DistMatrix probs, DistMatrix labels);
void conv2dForward(Session& s, DistMatrix input, DistMatrix filters, DistMatrix output,
                   kernels::ConvGeometry g);

}  // namespace gridmath
