// SPDX-License-Identifier: Apache-2.0
// Implementation of the master/worker runtime (see runtime.hpp).
//
// Reference call stacks this follows (paths under /root/reference/proj):
//   gemm()          session.cpp:533-545 -> issueOp :78-105 -> kernels::validate
//                   kernels.cpp:296-312 -> applyOpMetadata ops.cpp:146-177
//   execGemm        kernels.cpp:560-568: planGemm (:204-251, merged C row/col
//                   intervals per worker; an A need per row interval and a B
//                   need per col interval; viaReplica when the replica is
//                   fresh, pieces.cpp:14-30) -> piece transport -> runGemm
//   replication     session.cpp:329-375, worker.cpp:245-448
// The B200 path takes each need over the full k range at once (one band,
// one fixed ascending-k accumulation chain per output element inside the
// tensor-core kernel) instead of 256-wide host panels; the per-element
// order is therefore independent of the layout and of P (deterministic
// mode, reference kernels.hpp:19-22).
#include "capture.hpp"
#include "runtime.hpp"

#include <cuda.h>  // types of the driver entry points (resolved at run time, no -lcuda)
#include <nccl.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "../cuda/convert.h"
#include "../cuda/debug_config.h"
#include "internal.hpp"

namespace gridmath {

namespace {

constexpr std::size_t kFlagBytes = 4ull * kSlots * sizeof(std::uint64_t);

// Stream memory operations and address-range lookup from the driver, via
// the runtime's entry-point query (the library stays loadable without a
// driver: CPU-only hosts load it for the pure-host helpers).
struct DriverFns {
  // 64-bit flag words: exec ids never wrap (a 32-bit GEQ wait would pass
  // early against a pre-wrap value after 2^32 ops).
  CUresult (*waitValue64)(CUstream, CUdeviceptr, cuuint64_t, unsigned int) = nullptr;
  CUresult (*writeValue64)(CUstream, CUdeviceptr, cuuint64_t, unsigned int) = nullptr;
  CUresult (*addressRange)(CUdeviceptr*, size_t*, CUdeviceptr) = nullptr;
};

const DriverFns& driver() {
  static const DriverFns fns = [] {
    DriverFns f;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue64", reinterpret_cast<void**>(&f.waitValue64),
                                cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
      f.waitValue64 = nullptr;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue64", reinterpret_cast<void**>(&f.writeValue64),
                                cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
      f.writeValue64 = nullptr;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", reinterpret_cast<void**>(&f.addressRange),
                                cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
      f.addressRange = nullptr;
    cudaGetLastError();
    return f;
  }();
  return fns;
}

// One record per tile (or per rank for the flag pages) in the IPC
// registration all-reduce (max over uint8: the owner's bytes win, zeros
// elsewhere; `failed` is an OR over ranks).
struct IpcRecord {
  cudaIpcMemHandle_t handle;
  std::uint64_t base;    // allocation base in the exporter's address space
  std::uint64_t offset;  // tile pointer - base
  std::uint8_t valid;
  std::uint8_t failed;
  std::uint8_t pad[6];
};
static_assert(sizeof(IpcRecord) == 88, "ipc record layout");

void ncclCheck(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw Error(std::string(what) + ": " + ncclGetErrorString(r));
}

struct Interval {
  std::uint64_t lo = 0, hi = 0;
};

std::vector<Interval> mergeIntervals(std::vector<Interval> v) {
  std::sort(v.begin(), v.end(), [](const Interval& a, const Interval& b) { return a.lo < b.lo; });
  std::vector<Interval> out;
  for (const Interval& i : v) {
    if (!out.empty() && i.lo <= out.back().hi)
      out.back().hi = std::max(out.back().hi, i.hi);
    else
      out.push_back(i);
  }
  return out;
}

void requireDistinct(const OpDescriptor& op, std::initializer_list<int> slots) {
  for (int i : slots)
    for (int j : slots)
      if (i != j && op.ids[i] == op.ids[j]) throw Error("operands must be distinct matrices");
}

}  // namespace

// Master-side checks before anything is issued (reference kernels.cpp:265-379).
void validateOp(const DescriptorTable& t, const OpDescriptor& op, std::uint32_t workers) {
  switch (op.opcode) {
    case OpCode::CreateMatrix: {
      WireReader r(op.blob);
      const MatrixDescriptor d = decodeDescriptor(r);
      if (d.rows == 0 || d.cols == 0) throw Error("createMatrix: empty shape");
      const LayoutReport rep = validateLayout(d.rows, d.cols, d.layout, workers);
      if (!rep.ok()) throw Error("createMatrix: invalid layout: " + rep.detail);
      if (t.count(d.matrixId)) throw Error("createMatrix: duplicate id");
      return;
    }
    case OpCode::DestroyMatrix:
    case OpCode::SetData:
    case OpCode::GetData:
    case OpCode::ReplicateStart:
      (void)lookup(t, op.ids[0]);
      return;
    case OpCode::Reshape: {
      const MatrixDescriptor& old = lookup(t, op.ids[0]);
      WireReader r(op.blob);
      const MatrixDescriptor d = decodeDescriptor(r);
      if (d.rows != old.rows || d.cols != old.cols) throw Error("reshape: shape must be preserved");
      const LayoutReport rep = validateLayout(d.rows, d.cols, d.layout, workers);
      if (!rep.ok()) throw Error("reshape: invalid layout: " + rep.detail);
      return;
    }
    case OpCode::Gemm: {
      const MatrixDescriptor& a = lookup(t, op.ids[0]);
      const MatrixDescriptor& b = lookup(t, op.ids[1]);
      const MatrixDescriptor& c = lookup(t, op.ids[2]);
      requireDistinct(op, {0, 2});
      requireDistinct(op, {1, 2});
      const bool ta = op.flags[0], tb = op.flags[1];
      const std::uint64_t m = ta ? a.cols : a.rows, k = ta ? a.rows : a.cols;
      const std::uint64_t kb = tb ? b.cols : b.rows, n = tb ? b.rows : b.cols;
      if (k != kb || c.rows != m || c.cols != n)
        throw Error("gemm: dimension mismatch (" + std::to_string(m) + "x" + std::to_string(k) +
                    " * " + std::to_string(kb) + "x" + std::to_string(n) + " -> " +
                    std::to_string(c.rows) + "x" + std::to_string(c.cols) + ")");
      return;
    }
    case OpCode::SetConst:
      (void)lookup(t, op.ids[0]);
      return;
    case OpCode::AddRowColSum: {
      const MatrixDescriptor& a = lookup(t, op.ids[0]);
      const MatrixDescriptor& row = lookup(t, op.ids[1]);
      const MatrixDescriptor& col = lookup(t, op.ids[2]);
      requireDistinct(op, {0, 1, 2});
      if (row.rows != a.rows || row.cols != 1) throw Error("addRowColSum: rowAcc must be rows x 1");
      if (col.rows != 1 || col.cols != a.cols) throw Error("addRowColSum: colAcc must be 1 x cols");
      return;
    }
    case OpCode::EwUnary: {
      const MatrixDescriptor& x = lookup(t, op.ids[0]);
      const MatrixDescriptor& d = lookup(t, op.ids[1]);
      if (x.rows != d.rows || x.cols != d.cols) throw Error("elementwise: shape mismatch");
      return;
    }
    case OpCode::EwBinary: {
      const MatrixDescriptor& x = lookup(t, op.ids[0]);
      const MatrixDescriptor& y = lookup(t, op.ids[1]);
      const MatrixDescriptor& d = lookup(t, op.ids[2]);
      const auto kind = static_cast<BinaryKind>(op.flags[0]);
      if (op.flags[0] > static_cast<std::uint8_t>(BinaryKind::BiasAdd)) throw Error("bad elementwise kind");
      if (kind == BinaryKind::BiasAdd) {
        if (y.rows != 1 || y.cols != x.cols) throw Error("biasAdd: bias must be 1 x cols");
      } else if (kind != BinaryKind::Copy && (x.rows != y.rows || x.cols != y.cols)) {
        throw Error("elementwise: shape mismatch");
      }
      if (x.rows != d.rows || x.cols != d.cols) throw Error("elementwise: shape mismatch");
      return;
    }
    case OpCode::MetaChecksum:
    case OpCode::QueryStats:
    case OpCode::DistributeSeeds:
      return;
    default:
      throw Error("op not supported on the B200 GEMM path");
  }
}

// ---------------------------------------------------------------- DistMatrix

std::uint64_t DistMatrix::rows() const { return session_->descriptor(id_).rows; }
std::uint64_t DistMatrix::cols() const { return session_->descriptor(id_).cols; }
Precision DistMatrix::precision() const { return session_->descriptor(id_).precision; }

// ---------------------------------------------------------------- PanelCache

bool PanelCache::contains(std::uint64_t id, std::uint64_t version, const Rect& r) const {
  for (const CacheEntry& e : entries_)
    if (e.matrixId == id && e.version == version && e.rect == r) return true;
  return false;
}

CacheEntry* PanelCache::lookup(std::uint64_t id, std::uint64_t version, const Rect& r,
                               std::uint64_t tick) {
  for (CacheEntry& e : entries_)
    if (e.matrixId == id && e.version == version && e.rect == r) {
      e.lastUse = tick;
      ++hits;
      return &e;
    }
  ++misses;
  return nullptr;
}

std::vector<CacheEntry> PanelCache::reserve(std::uint64_t bytes, std::uint64_t budget,
                                            std::uint64_t protectTick) {
  std::vector<CacheEntry> evicted;
  while (bytes_ + bytes > budget) {
    // Least recently used entry not in use by the current op.
    auto victim = entries_.end();
    for (auto it = entries_.begin(); it != entries_.end(); ++it)
      if (it->lastUse != protectTick && (victim == entries_.end() || it->lastUse < victim->lastUse))
        victim = it;
    if (victim == entries_.end()) break;
    bytes_ -= victim->bytes;
    evicted.push_back(*victim);
    entries_.erase(victim);
  }
  return evicted;
}

CacheEntry& PanelCache::insert(CacheEntry e) {
  bytes_ += e.bytes;
  entries_.push_back(e);
  return entries_.back();
}

std::vector<CacheEntry> PanelCache::dropAll() {
  std::vector<CacheEntry> out(entries_.begin(), entries_.end());
  entries_.clear();
  bytes_ = 0;
  return out;
}

std::vector<CacheEntry> PanelCache::dropMatrix(std::uint64_t id, bool keepCurrent,
                                               std::uint64_t version) {
  std::vector<CacheEntry> out;
  for (auto it = entries_.begin(); it != entries_.end();) {
    if (it->matrixId == id && !(keepCurrent && it->version == version)) {
      bytes_ -= it->bytes;
      out.push_back(*it);
      it = entries_.erase(it);
    } else {
      ++it;
    }
  }
  return out;
}

// ---------------------------------------------------------------- Worker

Worker::Worker(std::uint32_t r, int dev, std::uint64_t budget)
    : rank(r), device(dev), arena(dev), cacheBudget(budget) {
  activate();
  cudaCheck(cudaStreamCreateWithFlags(&compute, cudaStreamNonBlocking), "worker: compute stream");
  int lo = 0, hi = 0;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  cudaCheck(cudaStreamCreateWithPriority(&comm, cudaStreamNonBlocking, hi), "worker: comm stream");
  cudaCheck(cudaStreamCreateWithFlags(&h2d, cudaStreamNonBlocking), "worker: h2d stream");
  cudaCheck(cudaStreamCreateWithFlags(&d2h, cudaStreamNonBlocking), "worker: d2h stream");
  cudaCheck(cudaStreamCreateWithFlags(&aux, cudaStreamNonBlocking), "worker: aux stream");
  cudaCheck(cudaStreamCreateWithPriority(&flagPub, cudaStreamNonBlocking, hi), "worker: flag stream");
  cudaCheck(cudaStreamCreateWithPriority(&warWait, cudaStreamNonBlocking, hi), "worker: WAR stream");
  for (cudaStream_t& ps : pulls)
    cudaCheck(cudaStreamCreateWithPriority(&ps, cudaStreamNonBlocking, hi), "worker: pull stream");
  cudaCheck(cudaEventCreate(&tStart), "worker: event");
  cudaCheck(cudaEventCreate(&tEnd), "worker: event");
  cudaCheck(cudaEventCreate(&uStart), "worker: event");
  cudaCheck(cudaEventCreate(&uEnd), "worker: event");
  cudaCheck(cudaEventCreate(&kStart), "worker: event");
  cudaCheck(cudaEventCreate(&cStart), "worker: event");
  cudaCheck(cudaEventCreate(&cEnd), "worker: event");
  if (gmk::debug_config().ready_slots > 0) readyCap = static_cast<std::uint64_t>(gmk::debug_config().ready_slots);
  void* rf = nullptr;
  cudaCheck(cudaMalloc(&rf, readyCap * sizeof(std::uint64_t)), "worker: ready flags");
  cudaCheck(cudaMemset(rf, 0, readyCap * sizeof(std::uint64_t)), "worker: ready flags");
  readyFlags = static_cast<std::uint64_t*>(rf);
}

std::uint64_t Worker::reserveReady(std::uint64_t n) {
  if (n == 0 || n > readyCap) throw Error("gemm: ready-flag region of " + std::to_string(n) + " slots");
  std::uint64_t start = readyHead;
  if (start % readyCap + n > readyCap) start += readyCap - start % readyCap;  // contiguous in memory
  const std::uint64_t end = start + n;
  while (!readyInUse.empty() && readyInUse.front().first + readyCap < end) {
    cudaCheck(capture::wait(comm, readyInUse.front().done, 0), "gemm: ready region reuse");
    recycle(readyInUse.front().done);
    readyInUse.pop_front();
  }
  readyHead = end;
  return start;
}

Worker::~Worker() {
  activate();
  cudaStreamSynchronize(compute);
  cudaStreamSynchronize(comm);
  cudaStreamSynchronize(h2d);
  cudaStreamSynchronize(d2h);
  cudaStreamSynchronize(aux);
  cudaStreamSynchronize(flagPub);
  cudaStreamSynchronize(warWait);
  for (cudaStream_t ps : pulls) cudaStreamSynchronize(ps);
  for (auto& kv : uploads) {
    for (auto& c : kv.second.chunks) cudaEventDestroy(c.done);
    cudaEventDestroy(kv.second.done);
  }
  for (auto& kv : chunkDone)
    for (auto& c : kv.second) cudaEventDestroy(c.done);
  releaseReaders();
  for (CacheEntry& e : cache.dropAll())
    if (e.ready) cudaEventDestroy(e.ready);
  for (auto& kv : replicas)
    if (kv.second.ready) cudaEventDestroy(kv.second.ready);
  for (auto& kv : lastWrite) cudaEventDestroy(kv.second);
  for (auto& kv : lastTouch) cudaEventDestroy(kv.second);
  for (auto& ev : kernelWindow) {
    cudaEventDestroy(ev.first);
    cudaEventDestroy(ev.second);
  }
  if (flags) cudaFree(flags);
  if (readyFlags) cudaFree(readyFlags);
  for (auto& r : readyInUse) cudaEventDestroy(r.done);
  if (nccl) ncclCommDestroy(nccl);
  for (cudaEvent_t e : pool_) cudaEventDestroy(e);
  cudaEventDestroy(tStart);
  cudaEventDestroy(tEnd);
  cudaEventDestroy(uStart);
  cudaEventDestroy(uEnd);
  cudaEventDestroy(kStart);
  cudaEventDestroy(cStart);
  cudaEventDestroy(cEnd);
  cudaStreamDestroy(compute);
  cudaStreamDestroy(comm);
  cudaStreamDestroy(h2d);
  cudaStreamDestroy(flagPub);
  cudaStreamDestroy(warWait);
  cudaStreamDestroy(d2h);
  cudaStreamDestroy(aux);
  for (cudaStream_t ps : pulls) cudaStreamDestroy(ps);
}

void Worker::joinUpload(std::uint64_t matrix) {
  auto it = uploads.find(matrix);
  if (it == uploads.end()) return;
  activate();
  cudaCheck(capture::wait(compute, it->second.done, 0), "upload: join");
  for (auto& c : it->second.chunks) recycle(c.done);
  recycle(it->second.done);
  uploads.erase(it);
}

void Worker::dropChunkDone(std::uint64_t matrix) {
  auto it = chunkDone.find(matrix);
  if (it == chunkDone.end()) return;
  for (auto& c : it->second) recycle(c.done);
  chunkDone.erase(it);
}

void Worker::activate() const { cudaCheck(cudaSetDevice(device), "cudaSetDevice"); }

cudaEvent_t Worker::event() {
  if (!pool_.empty()) {
    cudaEvent_t e = pool_.back();
    pool_.pop_back();
    return e;
  }
  activate();
  cudaEvent_t e;
  cudaCheck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "worker: event");
  return e;
}

void Worker::recycle(cudaEvent_t e) {
  if (e) pool_.push_back(e);
}

void* Worker::workspace(std::uint64_t bytes) {
  if (bytes <= wsBytes_) return ws_;
  if (ws_) arena.free(ws_, compute);
  ws_ = arena.alloc(bytes, compute);
  wsBytes_ = bytes;
  return ws_;
}

void Worker::releaseReaders() {
  for (auto& kv : readers_)
    for (auto& rd : kv.second) rd.second->recycle(rd.first);
  readers_.clear();
}

void Worker::beforeMutation(std::uint64_t matrix, cudaStream_t on) {
  auto it = readers_.find(matrix);
  if (it == readers_.end()) return;
  activate();
  for (auto& rd : it->second) {
    cudaCheck(capture::wait(on ? on : compute, rd.first, 0), "worker: wait reader");
    rd.second->recycle(rd.first);
  }
  readers_.erase(it);
}

// ---------------------------------------------------------------- Session

// Max-reduce a small host byte array over all SPMD ranks (control plane of
// the IPC registration; blocking): the caller's channel (e.g. gloo) when one
// was given, else the NCCL communicator through a device staging buffer.
void Session::controlMax(void* host, std::size_t n) {
  if (opts_.controlAllreduceMax) {
    opts_.controlAllreduceMax(host, n);
    return;
  }
  Worker& w = *local(static_cast<std::uint32_t>(opts_.spmdRank));
  w.activate();
  void* d = w.arena.alloc(std::max<std::size_t>(n, 256), w.compute);
  cudaCheck(cudaMemcpyAsync(d, host, n, cudaMemcpyHostToDevice, w.compute), "ipc: upload records");
  ncclCheck(ncclAllReduce(d, d, n, ncclUint8, ncclMax, w.nccl, w.compute), "ipc: allreduce records");
  cudaCheck(cudaMemcpyAsync(host, d, n, cudaMemcpyDeviceToHost, w.compute), "ipc: download records");
  cudaCheck(cudaStreamSynchronize(w.compute), "ipc: records sync");
  w.arena.free(d, w.compute);
}

// SPMD copy-engine plane: every rank exports a flag page; every rank must
// map every peer's page, or all ranks fall back to NCCL together.
void Session::setupIpc() {
  Worker& w = *local(static_cast<std::uint32_t>(opts_.spmdRank));
  w.activate();
  const DriverFns& drv = driver();
  std::vector<IpcRecord> recs(opts_.workers);
  std::memset(recs.data(), 0, recs.size() * sizeof(IpcRecord));
  IpcRecord& mine = recs[opts_.spmdRank];
  bool ok = drv.waitValue64 && drv.writeValue64 && drv.addressRange;
  if (ok) {
    void* f = nullptr;
    ok = cudaMalloc(&f, kFlagBytes) == cudaSuccess;
    if (ok) {
      w.flags = static_cast<std::uint64_t*>(f);
      ok = cudaMemset(f, 0, kFlagBytes) == cudaSuccess && cudaDeviceSynchronize() == cudaSuccess &&
           cudaIpcGetMemHandle(&mine.handle, f) == cudaSuccess;
      mine.base = reinterpret_cast<std::uint64_t>(f);
      mine.valid = 1;
    }
  }
  cudaGetLastError();
  if (!ok) mine.failed = 1;
  controlMax(recs.data(), recs.size() * sizeof(IpcRecord));
  bool all = true;
  for (const IpcRecord& r : recs) all = all && r.valid && !r.failed;
  std::vector<std::uint64_t*> mapped(opts_.workers, nullptr);
  for (std::uint32_t r = 0; all && r < opts_.workers; ++r) {
    if (r == w.rank) continue;
    void* p = nullptr;
    if (cudaIpcOpenMemHandle(&p, recs[r].handle, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
      cudaGetLastError();
      all = false;
      break;
    }
    ipcOpened_[{r, recs[r].base}] = p;
    mapped[r] = static_cast<std::uint64_t*>(p);
  }
  std::uint8_t failed = all ? 0 : 1;
  controlMax(&failed, 1);
  if (failed) {
    for (auto& kv : ipcOpened_) cudaIpcCloseMemHandle(kv.second);
    ipcOpened_.clear();
    if (w.flags) cudaFree(w.flags);
    w.flags = nullptr;
    cudaGetLastError();
    if (opts_.transport == 2)
      throw Error("session: copy-engine transport requested but peer GPU memory cannot be mapped (CUDA IPC)");
    return;
  }
  mapped[w.rank] = w.flags;
  peerFlags_ = std::move(mapped);
  ipc_ = true;
}

// Exports this rank's tiles of matrix `id` and maps every peer's (one
// collective per create/reshape). A local failure is carried through the
// collective so every rank throws together.
void Session::registerTiles(std::uint64_t id, const std::string& localError) {
  const MatrixDescriptor& d = lookup(table_, id);
  Worker& w = *local(static_cast<std::uint32_t>(opts_.spmdRank));
  w.activate();
  const DriverFns& drv = driver();
  const std::size_t T = d.layout.tiles.size();
  std::vector<IpcRecord> recs(T + 1);
  std::memset(recs.data(), 0, recs.size() * sizeof(IpcRecord));
  std::string err = localError;
  if (err.empty()) {
    auto tit = w.tiles.find(id);
    std::size_t i = 0;
    for (const auto& t : d.layout.tiles) {
      if (t.second.rank == w.rank && tit != w.tiles.end())
        for (const DeviceTile& dt : tit->second) {
          if (!(dt.extent == t.first) || !err.empty()) continue;
          CUdeviceptr base = 0;
          size_t size = 0;
          if (drv.addressRange(&base, &size, reinterpret_cast<CUdeviceptr>(dt.ptr)) != CUDA_SUCCESS) {
            err = "ipc: cuMemGetAddressRange failed for a tile";
          } else if (cudaIpcGetMemHandle(&recs[i].handle, reinterpret_cast<void*>(base)) != cudaSuccess) {
            cudaGetLastError();
            err = "ipc: cudaIpcGetMemHandle failed for a tile";
          } else {
            recs[i].base = base;
            recs[i].offset = reinterpret_cast<std::uint64_t>(dt.ptr) - base;
            recs[i].valid = 1;
          }
        }
      ++i;
    }
  }
  if (!err.empty()) recs[T].failed = 1;
  controlMax(recs.data(), recs.size() * sizeof(IpcRecord));
  if (recs[T].failed)
    throw Error(err.empty() ? "op failed: a peer rank could not allocate or export its tiles" : err);
  std::vector<void*> ptrs(T, nullptr);
  std::size_t i = 0;
  for (const auto& t : d.layout.tiles) {
    if (t.second.rank != w.rank) {
      const IpcRecord& r = recs[i];
      if (!r.valid) throw Error("ipc: tile " + std::to_string(i) + " of matrix " + std::to_string(id) + " not exported");
      const auto key = std::make_pair(t.second.rank, r.base);
      auto it = ipcOpened_.find(key);
      void* p = nullptr;
      if (it == ipcOpened_.end()) {
        cudaCheck(cudaIpcOpenMemHandle(&p, r.handle, cudaIpcMemLazyEnablePeerAccess), "ipc: map peer tile");
        ipcOpened_[key] = p;
      } else {
        p = it->second;
      }
      ptrs[i] = static_cast<std::uint8_t*>(p) + r.offset;
    }
    ++i;
  }
  peerTiles_[id] = std::move(ptrs);
}

void Session::ipcWait(cudaStream_t s, const std::uint64_t* addr, std::uint64_t value) {
  const CUresult r = driver().waitValue64(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(addr),
                                          static_cast<cuuint64_t>(value), CU_STREAM_WAIT_VALUE_GEQ);
  if (r != CUDA_SUCCESS) throw Error("ipc: cuStreamWaitValue64 failed (" + std::to_string(static_cast<int>(r)) + ")");
}

void Session::ipcWrite(cudaStream_t s, std::uint64_t* addr, std::uint64_t value) {
  const CUresult r = driver().writeValue64(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(addr),
                                           static_cast<cuuint64_t>(value), CU_STREAM_WRITE_VALUE_DEFAULT);
  if (r != CUDA_SUCCESS) throw Error("ipc: cuStreamWriteValue64 failed (" + std::to_string(static_cast<int>(r)) + ")");
}

const Session::ChunkedWrite* Session::chunkedSource(std::uint64_t matrix) const {
  auto it = chunked_.find(matrix);
  if (it == chunked_.end()) return nullptr;
  auto lm = lastMut_.find(matrix);
  return (lm != lastMut_.end() && lm->second == it->second.execId) ? &it->second : nullptr;
}

std::uint32_t Session::chunkOrdinal(const MatrixDescriptor& M, std::size_t tileIdx, std::uint64_t row,
                                    std::uint64_t chunkBytes, std::uint64_t* lo, std::uint64_t* hi) {
  const std::uint64_t eb = bytesOf(M.precision);
  auto rpcOf = [&](const TileExtent& e) {
    return std::max<std::uint64_t>(1, chunkBytes / std::max<std::uint64_t>(e.colCount * eb, 1));
  };
  const std::uint32_t owner = M.layout.tiles[tileIdx].second.rank;
  std::uint32_t ord = 0;
  for (std::size_t i = 0; i < tileIdx; ++i)
    if (M.layout.tiles[i].second.rank == owner) {
      const TileExtent& e = M.layout.tiles[i].first;
      ord += static_cast<std::uint32_t>((e.rowCount + rpcOf(e) - 1) / rpcOf(e));
    }
  const TileExtent& e = M.layout.tiles[tileIdx].first;
  const std::uint64_t rpc = rpcOf(e);
  const std::uint64_t ci = (row - e.rowStart) / rpc;
  if (lo) *lo = e.rowStart + ci * rpc;
  if (hi) *hi = std::min(e.rowEnd(), e.rowStart + (ci + 1) * rpc);
  return ord + static_cast<std::uint32_t>(ci);
}

std::uint32_t Session::slotOf(std::uint64_t id) const {
  auto it = slots_.find(id);
  if (it == slots_.end()) throw Error("ipc: matrix " + std::to_string(id) + " has no flag slot");
  return it->second;
}

BandView Session::srcView(const MatrixDescriptor& M, std::uint32_t src, const Rect& r) {
  const std::uint64_t eb = bytesOf(M.precision);
  if (Worker* sw = local(src)) {
    for (const DeviceTile& dt : sw->tiles.at(M.matrixId))
      if (r.inside(Rect::ofExtent(dt.extent)))
        return offsetView(dt.ptr, dt.ld, r.r0 - dt.extent.rowStart, r.c0 - dt.extent.colStart, eb);
    return {};
  }
  if (!ipc_) return {};
  auto pit = peerTiles_.find(M.matrixId);
  if (pit == peerTiles_.end()) return {};
  std::size_t i = 0;
  for (const auto& t : M.layout.tiles) {
    if (t.second.rank == src && pit->second[i] && r.inside(Rect::ofExtent(t.first)))
      return offsetView(pit->second[i], paddedLd(t.first.colCount, eb), r.r0 - t.first.rowStart,
                        r.c0 - t.first.colStart, eb);
    ++i;
  }
  return {};
}

// Publishes the previous op's mutations: per worker and matrix an event on
// the compute stream (local readers on other streams wait on it) and, on the
// SPMD copy-engine plane, written[slot] = exec id (peers' streams wait on it).
void Session::flushWritten(std::uint64_t before) {
  if (pendingWritten_.empty()) return;
  // Only ops older than `before`: the current op's own mutation is published
  // after its device work (at the next issue), never from inside the op.
  std::vector<std::pair<std::uint64_t, std::uint64_t>> pend, keep;
  for (const auto& pw : pendingWritten_) (pw.second < before ? pend : keep).push_back(pw);
  pendingWritten_ = std::move(keep);
  for (const auto& pw : pend) {
    if (!table_.count(pw.first)) continue;
    for (auto& wp : workers_) {
      if (!wp) continue;
      Worker& w = *wp;
      auto tit = w.tiles.find(pw.first);
      if (tit == w.tiles.end() || tit->second.empty()) continue;
      w.activate();
      cudaEvent_t& e = w.lastWrite[pw.first];
      if (!e) cudaCheck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "worker: write event");
      // A pending chunked upload is the write being published: from the h2d
      // stream, after its last chunk (the compute stream has not joined it).
      cudaStream_t ws = w.uploads.count(pw.first) ? w.h2d : w.compute;
      cudaCheck(capture::record(e, ws), "worker: record write");
      if (ipc_) {
        // A compute-stream write is published when a peer first pulls the
        // matrix (publishWritten): a flag write between kernels costs ~3 us
        // of compute-stream time (tools/dev/memop_probe.cu).
        if (ws == w.compute && gmk::debug_config().lazy_written) {
          unpublished_[pw.first] = pw.second;
        } else {
          unpublished_.erase(pw.first);
          ipcWrite(ws, w.flags + slotOf(pw.first), pw.second);
        }
      }
    }
  }
}

void Session::waitRemoteReaders(Worker& w, std::uint64_t matrix, cudaStream_t ws) {
  auto rr = remoteReaders_.find(matrix);
  if (rr == remoteReaders_.end() || rr->second.empty()) return;
  const bool side = gmk::debug_config().war_side != 0;
  cudaStream_t q = side ? w.warWait : ws;
  for (const auto& rd : rr->second)
    ipcWait(q, peerFlags_[rd.first.first] + kSlots * (1 + rd.first.second) + slotOf(matrix), rd.second);
  if (side) {
    cudaEvent_t e = w.event();
    cudaCheck(capture::record(e, q), "WAR: record");
    cudaCheck(capture::wait(ws, e, 0), "WAR: wait");
    w.recycle(e);
  }
}

void Session::publishWritten(Worker& w, std::uint64_t matrix) {
  auto it = unpublished_.find(matrix);
  if (it == unpublished_.end()) return;
  w.activate();
  cudaCheck(capture::wait(w.flagPub, w.lastWrite.at(matrix), 0), "publish write");
  ipcWrite(w.flagPub, w.flags + slotOf(matrix), it->second);
  unpublished_.erase(it);
}

// Consumers publish readDone[stream][slot] = exec id once this op's pulls
// from peer tiles are done (their producers wait on it before mutating).
void Session::commitReads() {
  for (const auto& pr : pendingReads_) {
    Worker& d = *local(std::get<0>(pr));
    const int si = std::get<2>(pr);
    d.activate();
    ipcWrite(si == 0 ? d.comm : d.compute, d.flags + kSlots * (1 + si) + slotOf(std::get<1>(pr)), curExec_);
  }
  pendingReads_.clear();
}

Session::Session(SessionOptions opts) : opts_(std::move(opts)) {
  if (opts_.workers == 0) throw Error("session: need at least one worker");
  int ndev = 0;
  cudaCheck(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
  if (ndev == 0) throw Error("session: no CUDA device");
  std::vector<int> devs = opts_.devices;
  if (devs.empty())
    for (int d = 0; d < ndev; ++d) devs.push_back(d);
  for (int d : devs)
    if (d < 0 || d >= ndev) throw Error("session: bad device " + std::to_string(d));
  workers_.resize(opts_.workers);
  remoteCaches_.resize(opts_.workers);
  auto budget = [&](int dev) -> std::uint64_t {
    if (opts_.panelCacheBytes) return opts_.panelCacheBytes;
    cudaDeviceProp prop{};
    cudaGetDeviceProperties(&prop, dev);
    return prop.totalGlobalMem / 4;
  };
  if (opts_.spmdRank >= 0) {
    if (static_cast<std::uint32_t>(opts_.spmdRank) >= opts_.workers)
      throw Error("session: spmd rank out of range");
    const int dev = devs[0];
    auto w = std::make_unique<Worker>(opts_.spmdRank, dev, budget(dev));
    const bool ownControl = static_cast<bool>(opts_.controlAllreduceMax);
    if (ownControl && opts_.transport == 1)
      throw Error("session: the NCCL data plane needs the NCCL control channel (no control callback)");
    if (opts_.workers > 1 && !ownControl) {
      ncclUniqueId id;
      static_assert(sizeof(id.internal) == 128, "nccl id size");
      std::memcpy(id.internal, opts_.ncclId.data(), 128);
      w->activate();
      ncclCheck(ncclCommInitRank(&w->nccl, static_cast<int>(opts_.workers), id, opts_.spmdRank),
                "ncclCommInitRank");
      nccl_ = true;
    }
    workers_[opts_.spmdRank] = std::move(w);
    if (opts_.workers > 1 && opts_.transport != 1) setupIpc();
    if (opts_.workers > 1 && !ipc_ && !nccl_)
      throw Error("session: SPMD without NCCL needs the copy-engine (IPC) plane, and peer memory cannot be mapped");
    if (opts_.workers > 1) {
      // Every rank keeps a directory of every peer's panel cache and replays
      // its keep/evict decisions with its own budget: the budgets must agree.
      // Each rank contributes its budget in its own 8-byte slot (max-reduce
      // of bytes = gather); all adopt the minimum.
      std::vector<std::uint64_t> all(opts_.workers, 0);
      all[opts_.spmdRank] = workers_[opts_.spmdRank]->cacheBudget;
      controlMax(all.data(), all.size() * sizeof(std::uint64_t));
      const std::uint64_t agreed = *std::min_element(all.begin(), all.end());
      workers_[opts_.spmdRank]->cacheBudget = agreed;
    }
  } else {
    for (std::uint32_t r = 0; r < opts_.workers; ++r) {
      const int dev = devs[r % devs.size()];
      workers_[r] = std::make_unique<Worker>(r, dev, budget(dev));
    }
    // Peer access between the distinct devices in use (copy-engine data plane).
    std::set<int> used;
    for (auto& w : workers_) used.insert(w->device);
    for (int a : used)
      for (int b : used) {
        if (a == b) continue;
        int can = 0;
        cudaDeviceCanAccessPeer(&can, a, b);
        if (can) {
          cudaSetDevice(a);
          const cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
          if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
            throw Error(std::string("peer access: ") + cudaGetErrorString(e));
          cudaGetLastError();
        }
      }
    peerCopies_ = true;
  }
}

Session::~Session() {
  try {
    synchronize();
  } catch (...) {
  }
  if (ipc_) {
    // Peers may still be pulling from this rank's tiles: every rank is
    // idle before any mapping closes or any arena frees.
    try {
      std::uint8_t b = 0;
      controlMax(&b, 1);
    } catch (...) {
    }
    for (auto& kv : ipcOpened_) cudaIpcCloseMemHandle(kv.second);
    ipcOpened_.clear();
    cudaGetLastError();
  }
  // Reader events can belong to a peer's pool: return them all before any
  // worker goes away.
  for (auto& w : workers_)
    if (w) w->releaseReaders();
  for (TimelineMark& m : timeline_) {
    cudaEventDestroy(m.compute);
    cudaEventDestroy(m.comm);
  }
  graphs_.clear();
  workers_.clear();
}

Worker* Session::local(std::uint32_t rank) const {
  return rank < workers_.size() ? workers_[rank].get() : nullptr;
}

bool Session::isLocal(std::uint32_t rank) const { return local(rank) != nullptr; }

std::vector<std::uint32_t> Session::localRanks() const {
  std::vector<std::uint32_t> r;
  for (auto& w : workers_)
    if (w) r.push_back(w->rank);
  return r;
}

void Session::forEachLocal(const std::function<void(Worker&)>& f) {
  std::vector<std::string> errs;
  for (auto& w : workers_) {
    if (!w) continue;
    try {
      w->activate();
      f(*w);
    } catch (const std::exception& e) {
      errs.push_back("worker " + std::to_string(w->rank) + ": " + e.what());
    }
  }
  checkErrors(errs);
}

void Session::checkErrors(std::vector<std::string>& errs) {
  if (errs.empty()) return;
  std::string msg = "op failed: ";
  for (auto& e : errs) msg += e + "; ";
  throw Error(msg);
}

const MatrixDescriptor& Session::descriptor(std::uint64_t id) const { return lookup(table_, id); }

namespace {
// Reference session.cpp:16-30.
bool recordable(OpCode c) {
  switch (c) {
    case OpCode::SetConst:
    case OpCode::Gemm:
    case OpCode::AddRowColSum:
    case OpCode::EwUnary:
    case OpCode::EwBinary:
    case OpCode::SoftmaxRows:
    case OpCode::SubtractOneHot:
    case OpCode::ReplicateStart:
      return true;
    default:
      return false;
  }
}
}  // namespace

// Matrices an op reads or writes in place on their owners' compute streams
// wait for pending chunked uploads first. The GEMM joins only C: it waits on
// the row chunks of A and B itself (execGemm).
void Session::joinUploads(const OpDescriptor& op) {
  int n = 1;
  switch (op.opcode) {
    case OpCode::Gemm: {
      forEachLocal([&](Worker& w) { w.joinUpload(op.ids[2]); });
      return;
    }
    case OpCode::EwBinary:
    case OpCode::AddRowColSum: n = 3; break;
    case OpCode::EwUnary: n = 2; break;
    case OpCode::CreateMatrix:
    case OpCode::QueryStats:
    case OpCode::MetaChecksum: return;
    default: n = 1; break;
  }
  forEachLocal([&](Worker& w) {
    for (int i = 0; i < n; ++i) w.joinUpload(op.ids[i]);
  });
}

void Session::requireRecordable(OpCode c) const {
  if (recording_ != 0 && !recordable(c)) throw Error("op not recordable inside an open pipeline recording");
}

std::uint64_t Session::issue(OpDescriptor& op) {
  requireRecordable(op.opcode);
  joinUploads(op);
  // The previous op's device work is enqueued: mark where its uses of its
  // matrices end on each compute stream.
  for (std::uint64_t id : pendingTouched_)
    for (auto& wp : workers_) {
      if (!wp || !wp->tiles.count(id)) continue;
      wp->activate();
      cudaEvent_t& e = wp->lastTouch[id];
      if (!e) cudaCheck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "worker: touch event");
      cudaCheck(capture::record(e, wp->compute), "worker: record touch");
    }
  pendingTouched_.clear();
  for (std::uint64_t id : op.ids)
    if (id && table_.count(id)) pendingTouched_.push_back(id);
  flushWritten(nextExec_);  // earlier ops' device work is enqueued: publish their writes
  op.execId = nextExec_++;
  curExec_ = op.execId;
  validateOp(table_, op, opts_.workers);
  if (recording_ != 0) {
    op.recordPipeline = recording_;
    pipelines_[recording_].push_back(op);
  }
  std::vector<std::pair<std::uint64_t, std::uint64_t>> moved;
  for (std::uint64_t id : mutatedMatrices(op)) {
    auto it = table_.find(id);
    if (it != table_.end()) moved.push_back({id, it->second.version});
  }
  applyOpMetadata(op, table_);
  // Control plane: every local worker mirrors the op through the wire codec.
  const std::vector<std::uint8_t> wire = op.encode();
  for (auto& w : workers_)
    if (w) {
      applyOpMetadata(OpDescriptor::decode(wire), w->descs);
      countLink(kMasterRank, w->rank, MsgKind::Control, wire.size());
      trace_.record(w->rank, EventKind::OpStart, op.execId, static_cast<std::uint64_t>(op.opcode));
    }
  // SetData carrying a chunk size is an asynchronous upload (hostio.cpp).
  const bool asyncUpload = op.opcode == OpCode::SetData && op.ids[1] != 0;
  for (const auto& mv : moved) mutationHook(mv.first, mv.second, asyncUpload);
  // Flag slots follow the (replicated) op stream, so every rank agrees.
  if (op.opcode == OpCode::CreateMatrix) {
    std::uint32_t slot = kSlots;
    if (!freeSlots_.empty()) {
      slot = freeSlots_.front();
      freeSlots_.erase(freeSlots_.begin());
    } else if (nextSlot_ < kSlots) {
      slot = nextSlot_++;
    } else if (ipc_) {
      throw Error("createMatrix: more than " + std::to_string(kSlots) + " live matrices");
    }
    if (slot < kSlots) slots_[op.ids[0]] = slot;
    lastMut_[op.ids[0]] = op.execId;
    pendingWritten_.push_back({op.ids[0], op.execId});  // the zero fill
  }
  for (const auto& mv : moved) {
    lastMut_[mv.first] = op.execId;
    pendingWritten_.push_back({mv.first, op.execId});
    chunked_.erase(mv.first);
  }
  if (opts_.checkMetadataEveryOp) verifyMetadataConsistency();
  return op.execId;
}

// A matrix is about to change: in-flight replicas of the old version fail
// (reference worker.cpp:207-239), cached panels of it die, and its owners'
// compute streams wait for every reader of their tiles (WAR).
void Session::mutationHook(std::uint64_t id, std::uint64_t oldVersion, bool toH2d) {
  const std::uint64_t newVersion = table_.count(id) ? table_.at(id).version : ~0ull;
  for (auto& wp : workers_) {
    if (!wp) continue;
    Worker& w = *wp;
    w.activate();
    auto rit = w.replicas.find(id);
    if (rit != w.replicas.end() && rit->second.version == oldVersion &&
        rit->second.state == ReplicaState::Pending) {
      if (cudaEventQuery(rit->second.ready) == cudaSuccess) {
        rit->second.state = ReplicaState::Valid;
      } else {
        cudaGetLastError();
        rit->second.state = ReplicaState::Stale;
        replFailed_[{id, oldVersion}] = true;
      }
    }
    for (CacheEntry& e : w.cache.dropMatrix(id, true, newVersion)) {
      w.arena.free(e.ptr, w.compute);
      w.recycle(e.ready);
    }
    cudaStream_t ws = toH2d ? w.h2d : w.compute;
    w.beforeMutation(id, ws);
    w.dropChunkDone(id);
    if (toH2d) {
      auto lt = w.lastTouch.find(id);
      if (lt != w.lastTouch.end()) cudaCheck(capture::wait(w.h2d, lt->second, 0), "upload: wait last use");
    }
    // Peers that pulled from this worker's tiles of the matrix (SPMD
    // copy-engine plane) must be done before it changes.
    if (w.tiles.count(id)) waitRemoteReaders(w, id, ws);
  }
  remoteReaders_.erase(id);
  for (std::uint32_t r = 0; r < opts_.workers; ++r)
    if (!isLocal(r)) remoteCaches_[r].dropMatrix(id, true, newVersion);
}

// ---------------------------------------------------------------- lifecycle

DistMatrix Session::createMatrix(std::uint64_t rows, std::uint64_t cols, Precision p,
                                 const Layout& layout) {
  MatrixDescriptor d;
  d.matrixId = nextMatrixId_++;
  d.rows = rows;
  d.cols = cols;
  d.precision = p;
  d.layout = layout;
  return createWithDescriptor(d);
}

DistMatrix Session::createWithDescriptor(const MatrixDescriptor& d) {
  nextMatrixId_ = std::max(nextMatrixId_, d.matrixId + 1);
  OpDescriptor op;
  op.opcode = OpCode::CreateMatrix;
  op.ids[0] = d.matrixId;
  WireWriter w;
  encodeDescriptor(d, w);
  op.blob = w.take();
  issue(op);
  try {
    execCreate(op);
  } catch (...) {
    // Roll back like the reference (session.cpp:208-216): a DestroyMatrix op
    // removes the descriptor everywhere and frees whatever was allocated.
    try {
      OpDescriptor rb;
      rb.opcode = OpCode::DestroyMatrix;
      rb.ids[0] = d.matrixId;
      issue(rb);
      execDestroy(d.matrixId);
    } catch (...) {
    }
    throw;
  }
  return DistMatrix(this, d.matrixId);
}

void Session::execCreate(const OpDescriptor& op) {
  WireReader r(op.blob);
  const MatrixDescriptor d = decodeDescriptor(r);
  const std::uint64_t eb = bytesOf(d.precision);
  std::string localError;
  try {
    forEachLocal([&](Worker& w) {
      std::vector<DeviceTile>& mine = w.tiles[d.matrixId];  // partial on failure: destroy frees it
      for (const auto& t : d.layout.tiles) {
        if (t.second.rank != w.rank) continue;
        DeviceTile dt;
        dt.extent = t.first;
        dt.ld = paddedLd(t.first.colCount, eb);
        const std::uint64_t bytes = t.first.rowCount * dt.ld * eb;
        dt.ptr = w.arena.alloc(bytes, w.compute);
        mine.push_back(dt);
        cudaCheck(cudaMemsetAsync(dt.ptr, 0, bytes, w.compute), "create: zero tile");
        w.residentBytes += t.first.elements() * eb;
      }
    });
  } catch (const std::exception& e) {
    if (!ipc_) throw;
    localError = e.what();
  }
  if (ipc_) registerTiles(d.matrixId, localError);  // collective: all ranks fail together
}

void Session::destroy(DistMatrix m) {
  OpDescriptor op;
  op.opcode = OpCode::DestroyMatrix;
  op.ids[0] = m.id();
  const std::uint64_t oldVersion = descriptor(m.id()).version;
  issue(op);
  mutationHook(m.id(), oldVersion);
  execDestroy(m.id());
}

void Session::execDestroy(std::uint64_t id) {
  unpublished_.erase(id);
  forEachLocal([&](Worker& w) {
    w.joinUpload(id);
    w.dropChunkDone(id);
    w.beforeMutation(id);
    auto lt = w.lastTouch.find(id);
    if (lt != w.lastTouch.end()) {
      cudaEventDestroy(lt->second);
      w.lastTouch.erase(lt);
    }
    auto lw = w.lastWrite.find(id);
    if (lw != w.lastWrite.end()) {
      cudaEventDestroy(lw->second);
      w.lastWrite.erase(lw);
    }
    auto it = w.tiles.find(id);
    if (it != w.tiles.end()) {
      const std::uint64_t eb = 1;  // residentBytes tracked in bytes below
      (void)eb;
      for (DeviceTile& t : it->second) w.arena.free(t.ptr, w.compute);
      w.tiles.erase(it);
    }
    auto rit = w.replicas.find(id);
    if (rit != w.replicas.end()) {
      capture::wait(w.compute, rit->second.ready, 0);
      if (!rit->second.alias) w.arena.free(rit->second.full, w.compute);
      if (rit->second.pieceReady) w.arena.free(rit->second.pieceReady, w.compute);
      cudaEventDestroy(rit->second.ready);
      w.replicas.erase(rit);
    }
    for (CacheEntry& e : w.cache.dropMatrix(id, false, 0)) {
      w.arena.free(e.ptr, w.compute);
      w.recycle(e.ready);
    }
  });
  for (auto& c : remoteCaches_) c.dropMatrix(id, false, 0);
  auto sl = slots_.find(id);
  if (sl != slots_.end()) {
    freeSlots_.push_back(sl->second);
    slots_.erase(sl);
  }
  lastMut_.erase(id);
  peerTiles_.erase(id);
  remoteReaders_.erase(id);
  // resident bytes recomputed from the remaining tiles
  for (auto& w : workers_) {
    if (!w) continue;
    w->residentBytes = 0;
    for (auto& kv : w->tiles) {
      const std::uint64_t eb = bytesOf(lookup(w->descs, kv.first).precision);
      for (auto& t : kv.second) w->residentBytes += t.extent.elements() * eb;
    }
  }
}

// ---------------------------------------------------------------- data in/out

void Session::setDataRaw(DistMatrix m, const void* image, std::uint64_t bytes) {
  const MatrixDescriptor d = descriptor(m.id());
  if (bytes != d.byteCount())
    throw Error("setData: expected " + std::to_string(d.byteCount()) + " bytes, got " +
                std::to_string(bytes));
  OpDescriptor op;
  op.opcode = OpCode::SetData;
  op.ids[0] = m.id();
  issue(op);
  const std::uint64_t eb = bytesOf(d.precision);
  const auto* img = static_cast<const std::uint8_t*>(image);
  forEachLocal([&](Worker& w) {
    for (DeviceTile& t : w.tiles.at(d.matrixId)) {
      const TileExtent& e = t.extent;
      cudaCheck(cudaMemcpy2DAsync(t.ptr, t.ld * eb, img + (e.rowStart * d.cols + e.colStart) * eb,
                                  d.cols * eb, e.colCount * eb, e.rowCount, cudaMemcpyDefault,
                                  w.compute),
                "setData: upload");
    }
    cudaCheck(cudaStreamSynchronize(w.compute), "setData: sync");
  });
}

void Session::setData(DistMatrix m, const std::vector<double>& rowMajor) {
  const MatrixDescriptor& d = descriptor(m.id());
  if (rowMajor.size() != d.elementCount())
    throw Error("setData: expected " + std::to_string(d.elementCount()) + " values, got " +
                std::to_string(rowMajor.size()));
  std::vector<std::uint8_t> staging(d.byteCount());
  convertBuffer(reinterpret_cast<const std::uint8_t*>(rowMajor.data()), Precision::Double,
                staging.data(), d.precision, rowMajor.size());
  setDataRaw(m, staging.data(), staging.size());
}

void Session::setDataF32(DistMatrix m, const std::vector<float>& rowMajor) {
  const MatrixDescriptor& d = descriptor(m.id());
  if (rowMajor.size() != d.elementCount()) throw Error("setData: value count mismatch");
  std::vector<std::uint8_t> staging(d.byteCount());
  convertBuffer(reinterpret_cast<const std::uint8_t*>(rowMajor.data()), Precision::Single,
                staging.data(), d.precision, rowMajor.size());
  setDataRaw(m, staging.data(), staging.size());
}

void Session::fillUniform(DistMatrix m, std::uint64_t seed, double lo, double hi) {
  const MatrixDescriptor d = descriptor(m.id());
  OpDescriptor op;
  op.opcode = OpCode::SetData;
  op.ids[0] = m.id();
  issue(op);
  forEachLocal([&](Worker& w) {
    for (DeviceTile& t : w.tiles.at(d.matrixId)) {
      const TileExtent& e = t.extent;
      cudaCheck(gmk::fill_uniform(t.ptr, static_cast<int>(d.precision), t.ld, e.rowStart, e.rowCount,
                                  e.colStart, e.colCount, d.cols, seed, lo, hi, w.compute),
                "fillUniform");
    }
  });
}

void Session::getDataRawInto(DistMatrix m, void* image, std::uint64_t bytes, bool localOnly) {
  const MatrixDescriptor d = descriptor(m.id());
  if (bytes != d.byteCount()) throw Error("getData: buffer size mismatch");
  OpDescriptor op;
  op.opcode = OpCode::GetData;
  op.ids[0] = m.id();
  issue(op);
  const std::uint64_t eb = bytesOf(d.precision);
  auto* img = static_cast<std::uint8_t*>(image);
  forEachLocal([&](Worker& w) {
    for (DeviceTile& t : w.tiles.at(d.matrixId)) {
      const TileExtent& e = t.extent;
      cudaCheck(cudaMemcpy2DAsync(img + (e.rowStart * d.cols + e.colStart) * eb, d.cols * eb, t.ptr,
                                  t.ld * eb, e.colCount * eb, e.rowCount, cudaMemcpyDefault,
                                  w.compute),
                "getData: download");
    }
  });
  if (ipc_ && !localOnly) {
    // Remote tiles: every rank pulls each peer tile through its IPC mapping
    // straight into the host image (copy engines; RAW/WAR through the flag
    // pages like any other pull).
    std::vector<Xfer> xs;
    for (const auto& t : d.layout.tiles) {
      const TileExtent& e = t.first;
      for (std::uint32_t r = 0; r < opts_.workers; ++r) {
        if (r == t.second.rank) continue;
        const bool mine = isLocal(r), theirs = isLocal(t.second.rank);
        if (!mine && !theirs) continue;
        Xfer x;
        x.src = t.second.rank;
        x.dst = r;
        x.rows = e.rowCount;
        x.cols = e.colCount;
        x.eb = static_cast<std::uint32_t>(eb);
        x.matrix = d.matrixId;
        x.hasOrigin = true;
        x.r0 = e.rowStart;
        x.c0 = e.colStart;
        if (mine) {
          const BandView sv = srcView(d, x.src, Rect::ofExtent(e));
          x.srcPtr = sv.ptr;
          x.srcLd = sv.ld;
          x.dstPtr = img + (e.rowStart * d.cols + e.colStart) * eb;
          x.dstLd = d.cols;
        }
        xs.push_back(x);
      }
    }
    exchange(xs, false);
  } else if (nccl_ && !localOnly) {
    // Remote tiles: each owner broadcasts its tile (packed) to every rank.
    Worker& w = *local(static_cast<std::uint32_t>(opts_.spmdRank));
    w.activate();
    std::uint64_t maxTile = 0;
    for (const auto& t : d.layout.tiles) maxTile = std::max(maxTile, t.first.elements() * eb);
    void* staging = w.arena.alloc(std::max<std::uint64_t>(maxTile, 256), w.compute);
    for (const auto& t : d.layout.tiles) {
      const TileExtent& e = t.first;
      const bool mine = t.second.rank == w.rank;
      if (mine) {
        for (DeviceTile& dt : w.tiles.at(d.matrixId))
          if (dt.extent == e)
            cudaCheck(cudaMemcpy2DAsync(staging, e.colCount * eb, dt.ptr, dt.ld * eb, e.colCount * eb,
                                        e.rowCount, cudaMemcpyDeviceToDevice, w.compute),
                      "getData: pack");
      }
      ncclCheck(ncclBroadcast(staging, staging, e.elements() * eb, ncclUint8,
                              static_cast<int>(t.second.rank), w.nccl, w.compute),
                "getData: broadcast");
      if (!mine)
        cudaCheck(cudaMemcpy2DAsync(img + (e.rowStart * d.cols + e.colStart) * eb, d.cols * eb, staging,
                                    e.colCount * eb, e.colCount * eb, e.rowCount, cudaMemcpyDefault,
                                    w.compute),
                  "getData: download");
    }
    w.arena.free(staging, w.compute);
  }
  forEachLocal([&](Worker& w) { cudaCheck(cudaStreamSynchronize(w.compute), "getData: sync"); });
}

std::vector<std::uint8_t> Session::getDataRaw(DistMatrix m) {
  std::vector<std::uint8_t> out(descriptor(m.id()).byteCount());
  getDataRawInto(m, out.data(), out.size(), false);
  return out;
}

std::vector<double> Session::getData(DistMatrix m) {
  const MatrixDescriptor& d = descriptor(m.id());
  const auto raw = getDataRaw(m);
  std::vector<double> out(d.elementCount());
  convertBuffer(raw.data(), d.precision, reinterpret_cast<std::uint8_t*>(out.data()),
                Precision::Double, out.size());
  return out;
}

// ---------------------------------------------------------------- reshape

void Session::reshape(DistMatrix m, const Layout& newLayout, std::optional<Precision> newPrecision) {
  requireRecordable(OpCode::Reshape);
  forEachLocal([&](Worker& w) { w.joinUpload(m.id()); });
  const MatrixDescriptor old = descriptor(m.id());  // copy: the table entry is replaced below
  MatrixDescriptor nd = old;
  nd.layout = newLayout;
  nd.precision = newPrecision.value_or(old.precision);
  nd.version = old.version + 1;
  nd.replicatedVersion = ~0ull;
  OpDescriptor op;
  op.opcode = OpCode::Reshape;
  op.ids[0] = m.id();
  WireWriter ww;
  encodeDescriptor(nd, ww);
  op.blob = ww.take();
  op.execId = nextExec_;
  validateOp(table_, op, opts_.workers);
  curExec_ = op.execId;  // pulls below are this op's reads (WAR bookkeeping)
  flushWritten(curExec_);

  const std::uint64_t oldEb = bytesOf(old.precision), newEb = bytesOf(nd.precision);
  const bool convert = old.precision != nd.precision;
  const bool viaReplica = old.replicaFresh();
  struct NewTile {
    Worker* w;
    DeviceTile tile;
    void* staging;  // old-precision assembly buffer (dense), when converting
  };
  std::vector<NewTile> made;
  std::vector<Xfer> xfers;
  try {
    for (const auto& t : nd.layout.tiles) {
      const TileExtent& e = t.first;
      Worker* w = local(t.second.rank);
      NewTile ntile{w, {}, nullptr};
      if (w) {
        w->activate();
        ntile.tile.extent = e;
        ntile.tile.ld = paddedLd(e.colCount, newEb);
        ntile.tile.ptr = w->arena.alloc(e.rowCount * ntile.tile.ld * newEb, w->compute);
        if (convert) ntile.staging = w->arena.alloc(e.elements() * oldEb, w->compute);
      }
      // Destination of the old-precision bytes for this tile.
      void* dst = w ? (convert ? ntile.staging : ntile.tile.ptr) : nullptr;
      const std::uint64_t dstLd = convert ? e.colCount : ntile.tile.ld;
      if (viaReplica) {
        if (w) {
          auto it = w->replicas.find(old.matrixId);
          if (it == w->replicas.end() || it->second.version != old.version)
            throw Error("reshape: replica of matrix " + std::to_string(old.matrixId) + " missing");
          cudaCheck(capture::wait(w->compute, it->second.ready, 0), "reshape: wait replica");
          cudaCheck(cudaMemcpy2DAsync(dst, dstLd * oldEb,
                                      static_cast<const std::uint8_t*>(it->second.full) +
                                          (e.rowStart * it->second.ld + e.colStart) * oldEb,
                                      it->second.ld * oldEb, e.colCount * oldEb, e.rowCount,
                                      cudaMemcpyDeviceToDevice, w->compute),
                    "reshape: from replica");
        }
      } else {
        for (const auto& ot : old.layout.tiles) {
          auto piece = intersectRect(Rect::ofExtent(e), Rect::ofExtent(ot.first));
          if (!piece) continue;
          Worker* sw = local(ot.second.rank);
          if (!w && !sw) continue;
          Xfer x;
          x.src = ot.second.rank;
          x.dst = t.second.rank;
          x.rows = piece->rows();
          x.cols = piece->cols();
          x.eb = static_cast<std::uint32_t>(oldEb);
          x.matrix = old.matrixId;
          const BandView sv = srcView(old, ot.second.rank, *piece);
          x.srcPtr = sv.ptr;
          x.srcLd = sv.ld;
          if (w) {
            x.dstPtr = static_cast<std::uint8_t*>(dst) + ((piece->r0 - e.rowStart) * dstLd + (piece->c0 - e.colStart)) * oldEb;
            x.dstLd = dstLd;
          }
          xfers.push_back(x);
        }
      }
      if (w) made.push_back(ntile);
    }
    exchange(xfers, false);
    for (NewTile& nt : made) {
      if (!convert) continue;
      nt.w->activate();
      const TileExtent& e = nt.tile.extent;
      cudaCheck(gmk::convert_rect(nt.staging, static_cast<int>(old.precision), e.colCount, nt.tile.ptr,
                                  static_cast<int>(nd.precision), nt.tile.ld, e.rowCount, e.colCount, nt.w->compute),
                "reshape: convert");
      nt.w->arena.free(nt.staging, nt.w->compute);
      nt.staging = nullptr;
    }
  } catch (...) {
    for (NewTile& nt : made) {
      if (nt.tile.ptr) nt.w->arena.free(nt.tile.ptr, nt.w->compute);
      if (nt.staging) nt.w->arena.free(nt.staging, nt.w->compute);
    }
    throw;
  }
  // Metadata swap (version bump, replicas and cached panels of the old
  // version die, WAR waits for the pieces just read), then retire old tiles.
  issue(op);
  forEachLocal([&](Worker& w) {
    for (DeviceTile& t : w.tiles[old.matrixId]) w.arena.free(t.ptr, w.compute);
    std::vector<DeviceTile> mine;
    for (NewTile& nt : made)
      if (nt.w == &w) mine.push_back(nt.tile);
    w.tiles[old.matrixId] = std::move(mine);
    w.residentBytes = 0;
    for (auto& kv : w.tiles) {
      const std::uint64_t eb = bytesOf(lookup(w.descs, kv.first).precision);
      for (auto& t : kv.second) w.residentBytes += t.extent.elements() * eb;
    }
  });
  if (ipc_) registerTiles(old.matrixId, "");
}

// ---------------------------------------------------------------- data plane

// Copy-engine planes -- one process (peer copies between its workers) or
// SPMD over CUDA IPC (a rank maps its peers' tiles): the consumer pulls each
// piece with a 2D copy on its own stream. No SMs are used, so the pulls of
// op i+1 overlap the persistent GEMM of op i. RAW: the consumer's stream
// waits for the last write of the source matrix (a local event, or the
// producer's written[slot] flag); WAR: the producer waits for the
// consumer's completion (a reader event, or the consumer's readDone flag)
// before it next mutates that matrix.
// NCCL plane (SPMD fallback): grouped ncclSend/ncclRecv, packing/unpacking
// strided pieces through arena staging.
void Session::exchange(std::vector<Xfer>& xs, bool onComm, bool commit, int maxPull) {
  flushWritten(curExec_);
  auto streamOf = [&](Worker& w) { return onComm ? w.comm : w.compute; };
  const int sIdx = onComm ? 0 : 1;
  if (!nccl_ || ipc_) {
    std::set<std::tuple<std::uint32_t, std::uint32_t, std::uint64_t>> routes;  // (src, dst, matrix)
    std::set<std::tuple<std::uint32_t, std::uint32_t, std::uint64_t, cudaStream_t>> waited;  // whole-write waits done
    std::set<std::tuple<std::uint32_t, cudaEvent_t, cudaStream_t>> chunkWaited;  // (dst, chunk event, stream)
    std::set<std::tuple<std::uint32_t, std::uint32_t, std::uint64_t, cudaStream_t>> flagWaited;  // (dst, src, value, stream)
    // Pieces from source worker s land on pull stream s % kPullStreams of the
    // consumer, forked from its base stream (so they see everything the base
    // stream owes, including this worker's own earlier writes) and joined
    // back before the op's readers are recorded.
    std::set<std::pair<Worker*, cudaStream_t>> forked;
    auto pullOf = [&](Worker& d, std::uint32_t src, int fixed) {
      const int dv = gmk::debug_config().pull_streams;
      const std::uint32_t nPull = static_cast<std::uint32_t>(std::clamp(dv > 0 ? dv : Worker::kPullStreams, 1,
                                                                        Worker::kPullStreams));
      const std::uint32_t np = maxPull > 0 ? std::min<std::uint32_t>(nPull, static_cast<std::uint32_t>(maxPull)) : nPull;
      cudaStream_t ps = fixed >= 0 ? d.pulls[fixed % Worker::kPullStreams] : d.pulls[src % np];
      if (forked.insert({&d, ps}).second) {
        cudaEvent_t e = d.event();
        cudaCheck(capture::record(e, streamOf(d)), "exchange: fork");
        cudaCheck(capture::wait(ps, e, 0), "exchange: fork");
        d.recycle(e);
      }
      return ps;
    };
    // RAW for one piece: the last write of its source, or -- when that write
    // is a chunked upload and the piece's origin is known -- only the upload
    // chunks it overlaps (sub-pieces are then copied chunk by chunk).
    auto wholeWait = [&](const Xfer& x, Worker& d, cudaStream_t ps) {
      if (!waited.insert({x.src, x.dst, x.matrix, ps}).second) return;
      Worker* s = local(x.src);
      if (s) {
        auto it = s->lastWrite.find(x.matrix);
        if (it != s->lastWrite.end() && (s != &d || onComm))
          cudaCheck(capture::wait(ps, it->second, 0), "exchange: wait writer");
      } else {
        ipcWait(ps, peerFlags_[x.src] + slotOf(x.matrix), lastMut_.at(x.matrix));
      }
    };
    for (const Xfer& x : xs) {
      const std::uint64_t bytes = x.rows * x.cols * x.eb;
      if (bytes == 0) continue;
      Worker* d = local(x.dst);
      Worker* s = local(x.src);
      if (!d) {
        // Producer side of a peer's pull: publish the write it waits for,
        // remember the reader (WAR).
        if (s) {
          publishWritten(*s, x.matrix);
          s->bytesSent += bytes;
          std::uint64_t& last = remoteReaders_[x.matrix][{x.dst, sIdx}];
          last = std::max(last, curExec_);
        }
        continue;
      }
      routes.insert({x.src, x.dst, x.matrix});
      if (!x.srcPtr)
        throw Error("exchange: no mapping for a piece of matrix " + std::to_string(x.matrix) + " on worker " +
                    std::to_string(x.src));
      d->activate();
      const ChunkedWrite* cw = x.hasOrigin ? chunkedSource(x.matrix) : nullptr;
      const MatrixDescriptor* M = cw ? &lookup(table_, x.matrix) : nullptr;
      std::size_t tileIdx = 0;
      bool found = false;
      if (cw) {
        for (std::size_t t = 0; t < M->layout.tiles.size() && !found; ++t) {
          const auto& tl = M->layout.tiles[t];
          if (tl.second.rank == x.src && Rect{x.r0, x.r0 + x.rows, x.c0, x.c0 + x.cols}.inside(Rect::ofExtent(tl.first))) {
            tileIdx = t;
            found = true;
          }
        }
      }
      // A local producer whose upload was already joined publishes through
      // its lastWrite event (recorded after the upload).
      if (cw && found && s && !s->uploads.count(x.matrix)) found = false;
      cudaStream_t ps = pullOf(*d, x.src, x.pullStream);
      if (!cw || !found) {
        wholeWait(x, *d, ps);
        cudaCheck(cudaMemcpy2DAsync(x.dstPtr, x.dstLd * x.eb, x.srcPtr, x.srcLd * x.eb, x.cols * x.eb, x.rows,
                                    cudaMemcpyDefault, ps),
                  "exchange: copy");
      } else {
        for (std::uint64_t r = x.r0; r < x.r0 + x.rows;) {
          std::uint64_t lo = 0, hi = 0;
          const std::uint32_t ord = chunkOrdinal(*M, tileIdx, r, cw->chunkBytes, &lo, &hi);
          const std::uint64_t r1 = std::min(hi, x.r0 + x.rows);
          if (s) {
            const auto& chunks = s->uploads.at(x.matrix).chunks;
            if (ord >= chunks.size()) throw Error("exchange: upload chunk geometry mismatch");
            // (the upload runs on the h2d stream: waited even for own tiles)
            if (chunkWaited.insert({x.dst, chunks[ord].done, ps}).second)
              cudaCheck(capture::wait(ps, chunks[ord].done, 0), "exchange: wait chunk");
          } else {
            const std::uint64_t v = cw->base[x.src] + ord + 1;
            if (flagWaited.insert({x.dst, x.src, v, ps}).second)
              ipcWait(ps, peerFlags_[x.src] + kUpChunkOff + slotOf(x.matrix), v);
          }
          const std::uint64_t off = r - x.r0;
          cudaCheck(cudaMemcpy2DAsync(static_cast<std::uint8_t*>(x.dstPtr) + off * x.dstLd * x.eb, x.dstLd * x.eb,
                                      static_cast<const std::uint8_t*>(x.srcPtr) + off * x.srcLd * x.eb,
                                      x.srcLd * x.eb, x.cols * x.eb, r1 - r, cudaMemcpyDefault, ps),
                    "exchange: copy chunk");
          r = r1;
        }
      }
      if (x.flagAddr && x.lastOfBlock) ipcWrite(ps, x.flagAddr, x.flagValue);
      if (x.src != x.dst) {
        d->bytesReceived += bytes;
        if (s) s->bytesSent += bytes;
        countLink(x.src, x.dst, MsgKind::Data, bytes);
      }
    }
    for (const auto& fk : forked) {
      Worker& d = *fk.first;
      d.activate();
      cudaEvent_t e = d.event();
      cudaCheck(capture::record(e, fk.second), "exchange: join");
      cudaCheck(capture::wait(streamOf(d), e, 0), "exchange: join");
      d.recycle(e);
    }
    for (const auto& rt : routes) {
      Worker& d = *local(std::get<1>(rt));
      Worker* s = local(std::get<0>(rt));
      if (s) {
        if (s == &d && !onComm) continue;
        d.activate();
        cudaEvent_t e = d.event();
        cudaCheck(capture::record(e, streamOf(d)), "exchange: record done");
        s->addReader(std::get<2>(rt), e, &d);
      } else {
        pendingReads_.insert({std::get<1>(rt), std::get<2>(rt), sIdx});
      }
    }
    if (commit) commitReads();
    return;
  }
  // ---- NCCL: sending (and locally copying) streams wait for the last write
  // of the matrices they read.
  std::set<std::pair<std::uint32_t, std::uint64_t>> readSrc;  // (local src worker, matrix)
  for (const Xfer& x : xs)
    if (x.rows * x.cols != 0 && local(x.src)) readSrc.insert({x.src, x.matrix});
  for (const auto& rs : readSrc) {
    Worker& s = *local(rs.first);
    auto it = s.lastWrite.find(rs.second);
    if (onComm && it != s.lastWrite.end()) {
      s.activate();
      cudaCheck(capture::wait(s.comm, it->second, 0), "exchange: wait writer");
    }
  }
  struct Staged {
    Worker* w;
    void* buf;
    const Xfer* x;
  };
  std::vector<Staged> sendPack, recvUnpack;
  std::vector<std::pair<const Xfer*, const void*>> sends;
  std::vector<std::pair<const Xfer*, void*>> recvs;
  for (const Xfer& x : xs) {
    const std::uint64_t bytes = x.rows * x.cols * x.eb;
    if (bytes == 0) continue;
    Worker* s = local(x.src);
    Worker* d = local(x.dst);
    if (s && d) {
      d->activate();
      cudaCheck(cudaMemcpy2DAsync(x.dstPtr, x.dstLd * x.eb, x.srcPtr, x.srcLd * x.eb, x.cols * x.eb,
                                  x.rows, cudaMemcpyDeviceToDevice, streamOf(*d)),
                "exchange: local copy");
      continue;
    }
    if (s) {
      s->activate();
      s->bytesSent += bytes;
      if (x.srcLd == x.cols) {
        sends.push_back({&x, x.srcPtr});
      } else {
        void* buf = s->arena.alloc(bytes, streamOf(*s));
        cudaCheck(cudaMemcpy2DAsync(buf, x.cols * x.eb, x.srcPtr, x.srcLd * x.eb, x.cols * x.eb, x.rows,
                                    cudaMemcpyDeviceToDevice, streamOf(*s)),
                  "exchange: pack");
        sendPack.push_back({s, buf, &x});
        sends.push_back({&x, buf});
      }
    }
    if (d) {
      d->activate();
      d->bytesReceived += bytes;
      if (x.dstLd == x.cols) {
        recvs.push_back({&x, x.dstPtr});
      } else {
        void* buf = d->arena.alloc(bytes, streamOf(*d));
        recvUnpack.push_back({d, buf, &x});
        recvs.push_back({&x, buf});
      }
    }
  }
  ncclCheck(ncclGroupStart(), "ncclGroupStart");
  for (auto& sd : sends) {
    Worker& s = *local(sd.first->src);
    ncclCheck(ncclSend(sd.second, sd.first->rows * sd.first->cols * sd.first->eb, ncclUint8,
                       static_cast<int>(sd.first->dst), s.nccl, streamOf(s)),
              "ncclSend");
  }
  for (auto& rv : recvs) {
    Worker& d = *local(rv.first->dst);
    ncclCheck(ncclRecv(rv.second, rv.first->rows * rv.first->cols * rv.first->eb, ncclUint8,
                       static_cast<int>(rv.first->src), d.nccl, streamOf(d)),
              "ncclRecv");
  }
  ncclCheck(ncclGroupEnd(), "ncclGroupEnd");
  for (auto& st : recvUnpack) {
    st.w->activate();
    const Xfer& x = *st.x;
    cudaCheck(cudaMemcpy2DAsync(x.dstPtr, x.dstLd * x.eb, st.buf, x.cols * x.eb, x.cols * x.eb, x.rows,
                                cudaMemcpyDeviceToDevice, streamOf(*st.w)),
              "exchange: unpack");
    st.w->arena.free(st.buf, streamOf(*st.w));
  }
  for (auto& st : sendPack) {
    st.w->activate();
    st.w->arena.free(st.buf, streamOf(*st.w));
  }
  if (onComm) {
    // Sends read tiles on the comm stream: later mutations wait for them.
    for (const auto& rs : readSrc) {
      Worker& s = *local(rs.first);
      s.activate();
      cudaEvent_t e = s.event();
      cudaCheck(capture::record(e, s.comm), "exchange: record");
      s.addReader(rs.second, e, &s);
    }
  }
}

// ---------------------------------------------------------------- GEMM

GemmPlanB200 planGemmB200(const DescriptorTable& t, const OpDescriptor& op, std::uint32_t P,
                          const CacheProbe& cached) {
  const MatrixDescriptor& A = lookup(t, op.ids[0]);
  const MatrixDescriptor& B = lookup(t, op.ids[1]);
  const MatrixDescriptor& C = lookup(t, op.ids[2]);
  GemmPlanB200 plan;
  plan.transA = op.flags[0] != 0;
  plan.transB = op.flags[1] != 0;
  plan.m = C.rows;
  plan.n = C.cols;
  plan.k = plan.transA ? A.rows : A.cols;
  plan.rowsOf.resize(P);
  plan.colsOf.resize(P);
  {
    std::vector<std::vector<Interval>> r(P), c(P);
    for (const auto& tl : C.layout.tiles) {
      r[tl.second.rank].push_back({tl.first.rowStart, tl.first.rowEnd()});
      c[tl.second.rank].push_back({tl.first.colStart, tl.first.colEnd()});
    }
    for (std::uint32_t w = 0; w < P; ++w) {
      for (const Interval& iv : mergeIntervals(std::move(r[w]))) plan.rowsOf[w].push_back({iv.lo, iv.hi});
      for (const Interval& iv : mergeIntervals(std::move(c[w]))) plan.colsOf[w].push_back({iv.lo, iv.hi});
    }
  }
  if (op.s0 == 0.0) return plan;  // alpha == 0: A and B are never read
  std::uint32_t pieceId = 0;
  auto add = [&](std::uint32_t w, int operand, std::size_t idx, const MatrixDescriptor& M, const Rect& rect) {
    PlannedNeed nd;
    nd.worker = w;
    nd.operand = operand;
    nd.interval = idx;
    nd.rect = rect;
    if (M.replicaFresh()) {
      nd.kind = PlannedNeed::Replica;
    } else {
      bool inTile = false;
      for (const auto& tl : M.layout.tiles)
        if (tl.second.rank == w && rect.inside(Rect::ofExtent(tl.first))) inTile = true;
      if (inTile) {
        nd.kind = PlannedNeed::LocalTile;
      } else if (cached && cached(w, M, rect)) {
        nd.kind = PlannedNeed::Cached;
      } else {
        nd.kind = PlannedNeed::Gather;
        for (const auto& tl : M.layout.tiles)
          if (auto piece = intersectRect(rect, Rect::ofExtent(tl.first)))
            nd.pieces.push_back(PieceRoute{pieceId++, tl.second.rank, w, M.matrixId, *piece});
      }
    }
    plan.needs.push_back(std::move(nd));
  };
  for (std::uint32_t w = 0; w < P; ++w) {
    for (std::size_t i = 0; i < plan.rowsOf[w].size(); ++i) {
      const auto iv = plan.rowsOf[w][i];
      add(w, 0, i, A, plan.transA ? Rect{0, plan.k, iv.first, iv.second} : Rect{iv.first, iv.second, 0, plan.k});
    }
    for (std::size_t i = 0; i < plan.colsOf[w].size(); ++i) {
      const auto iv = plan.colsOf[w][i];
      add(w, 1, i, B, plan.transB ? Rect{iv.first, iv.second, 0, plan.k} : Rect{0, plan.k, iv.first, iv.second});
    }
  }
  return plan;
}

std::vector<std::uint64_t> planRemoteBytes(const GemmPlanB200& plan, const DescriptorTable& t,
                                           std::uint32_t P) {
  std::vector<std::uint64_t> out(P, 0);
  for (const PlannedNeed& nd : plan.needs)
    for (const PieceRoute& pr : nd.pieces)
      if (pr.src != pr.consumer)
        out[pr.consumer] += pr.rect.elements() * bytesOf(lookup(t, pr.matrixId).precision);
  return out;
}


void Session::runGemm(const OpDescriptor& op0, bool sync) {
  OpDescriptor op = op0;
  issue(op);
  execGemm(op);
  if (sync) synchronize();
}

void Session::execGemm(const OpDescriptor& op) {
  const MatrixDescriptor& A = lookup(table_, op.ids[0]);
  const MatrixDescriptor& B = lookup(table_, op.ids[1]);
  const MatrixDescriptor& C = lookup(table_, op.ids[2]);
  const std::uint32_t P = opts_.workers;
  ++tick_;
  ++gemmEpoch_;
  Worker* localRef = nullptr;
  for (auto& wp : workers_)
    if (wp) localRef = wp.get();

  forEachLocal([&](Worker& w) {
    w.timed = true;
    cudaCheck(capture::recordTiming(w.tStart, w.compute), "gemm: timing");
  });

  auto dirOf = [&](std::uint32_t r) -> PanelCache& {
    Worker* w = local(r);
    return w ? w->cache : remoteCaches_[r];
  };
  const GemmPlanB200 plan = planGemmB200(table_, op, P, [&](std::uint32_t r, const MatrixDescriptor& M, const Rect& rect) {
    return dirOf(r).contains(M.matrixId, M.version, rect);
  });
  // Pin every panel the plan reads from the cache before any gather of this
  // op reserves room: lookup() stamps lastUse = tick_, and reserve() never
  // evicts an entry stamped with the current tick. (Without this, a later
  // Gather need of the same op could evict a band planned as Cached.)
  std::vector<CacheEntry*> cachedHits(plan.needs.size(), nullptr);
  for (std::size_t i = 0; i < plan.needs.size(); ++i) {
    const PlannedNeed& nd = plan.needs[i];
    if (nd.kind != PlannedNeed::Cached) continue;
    const MatrixDescriptor& M = nd.operand == 0 ? A : B;
    cachedHits[i] = dirOf(nd.worker).lookup(M.matrixId, M.version, nd.rect, tick_);
    if (!cachedHits[i])
      throw Error("gemm: panel of matrix " + std::to_string(M.matrixId) + " planned as cached on worker " +
                  std::to_string(nd.worker) + " is not in its cache");
  }

  // SUMMA-style overlap: gathered bands move on the comm stream in groups --
  // first every gathered B band, then the gathered A bands in `S` row chunks
  // (m direction). The compute stream runs the GEMM of C rows chunk j as soon
  // as chunk j has landed. Every rank issues the same groups in the same
  // order, so the NCCL point-to-point calls match.
  std::uint32_t S = opts_.pipelineChunks > 0 ? static_cast<std::uint32_t>(opts_.pipelineChunks) : 2u;
  bool anyGather = false;
  for (const PlannedNeed& nd : plan.needs)
    if (nd.kind == PlannedNeed::Gather) anyGather = true;
  // Operands streaming in from the host (chunked uploads read in place):
  // nothing to exchange, so the row chunks follow the upload's instead.
  bool streamedA = false;
  forEachLocal([&](Worker& w) { streamedA = streamedA || w.uploads.count(A.matrixId); });
  if (!anyGather) S = (streamedA && !plan.transA) ? (opts_.pipelineChunks > 0 ? S : 8u) : 1u;
  // A streaming in from the hosts in chunks (replicated knowledge, so every
  // rank picks the same S): finer row chunks let the first GEMMs start on the
  // first upload chunks pulled from the peers.
  else if (chunkedSource(A.matrixId) && !plan.transA && opts_.pipelineChunks <= 0) S = 8u;
  while (S > 1 && plan.m < 512ull * S) --S;

  // In-GEMM panel pipelining (copy-engine planes, 16-bit operands read in
  // place): every gathered band is cut into blocks -- m-chunks (A) or
  // n-chunks (B) by k-panels -- that the pull streams copy in the order the
  // persistent GEMM first needs them, each block publishing a ready flag the
  // GEMM's producer polls before loading a k-block. The GEMM starts at once;
  // panel k+1 lands while panel k multiplies (reference: panels are consumed
  // as their pieces arrive, kernels.cpp:490-552). Per-consumer decision: the
  // producers' side of the exchange is unchanged.
  const bool f16Pair = (A.precision == Precision::BF16 || A.precision == Precision::Half) &&
                       A.precision == B.precision && C.precision != Precision::Double;
  bool pipelined = anyGather && f16Pair && op.s0 != 0.0 && (!nccl_ || ipc_) &&
                         gmk::debug_config().panel_flags && panelPipelining_ && opts_.pipelineChunks <= 0 && !streamedA &&
                         !chunkedSource(A.matrixId) && !chunkedSource(B.matrixId);
  const gmk::DebugConfig& dbg = gmk::debug_config();
  const std::uint64_t panelK = dbg.panel_k > 0 ? (static_cast<std::uint64_t>(dbg.panel_k) + 63) / 64 * 64
                                               : std::max<std::uint64_t>(64, (plan.k + 16 * 64 - 1) / (16 * 64) * 64);
  const std::uint64_t numPanels = (plan.k + panelK - 1) / panelK;
  // Raster group x 256 rows; 4 wide tiles of columns.
  const std::uint64_t kAChunkRows = dbg.a_chunk_rows > 0 ? static_cast<std::uint64_t>(dbg.a_chunk_rows) : 4096;
  const std::uint64_t kBChunkCols = dbg.b_chunk_cols > 0 ? static_cast<std::uint64_t>(dbg.b_chunk_cols) : 2048;
  bool fits = true;  // every local band's flag region fits its worker's ring
  for (const PlannedNeed& nd : plan.needs) {
    Worker* w = local(nd.worker);
    if (nd.kind != PlannedNeed::Gather || !w) continue;
    const bool chunkRows = nd.operand == 0 ? !plan.transA : plan.transB;
    const std::uint64_t ext = chunkRows ? nd.rect.rows() : nd.rect.cols();
    const std::uint64_t cs = nd.operand == 0 ? kAChunkRows : kBChunkCols;
    fits = fits && (ext + cs - 1) / cs * numPanels <= w->readyCap;
  }
  // Only GEMMs long enough for the overlap to pay for the per-block copy
  // and flag overhead (~5 us per block on its stream; measured: the FC dW
  // GEMM, 0.16 TFLOP per worker, ran 225 -> 400 us pipelined). Per worker:
  // 2 m n k over its C tiles >= 1 TFLOP (~0.7 ms of tcgen05 time).
  double maxFlops = 0.0;
  for (std::uint32_t w = 0; w < P; ++w) {
    if (!isLocal(w)) continue;
    double f = 0.0;
    for (const auto& tl : C.layout.tiles)
      if (tl.second.rank == w) f += 2.0 * static_cast<double>(tl.first.rowCount) * tl.first.colCount * plan.k;
    maxFlops = std::max(maxFlops, f);
  }
  const double minFlops = dbg.panel_min_gflop >= 0 ? dbg.panel_min_gflop * 1e9 : 1e12;
  pipelined = pipelined && fits && maxFlops >= minFlops;
  if (pipelined) S = 1;
  // One gathered band of a local consumer in pipelined mode.
  struct FlagBand {
    Worker* w = nullptr;
    int operand = 0;
    std::size_t interval = 0;
    std::uint64_t chunk = 0, chunks = 0;
    std::uint64_t* flags = nullptr;  // chunks x numPanels
    std::uint64_t first = 0;         // monotonic ring slot
  };
  std::vector<FlagBand> flagBands;
  struct BlockXfer {
    Xfer x;
    std::size_t band = 0;
    std::uint64_t chunk = 0, panel = 0;
  };
  std::vector<BlockXfer> blockXfers;
  // B read from a replica still landing piece by piece: the GEMM polls the
  // replica's per-piece flags instead of waiting for the whole matrix.
  // Column-block layouts only (piece t = columns [t w, (t+1) w)).
  struct ReplicaPoll {
    const ReplicaEntry* entry = nullptr;
    std::uint64_t width = 0;
    std::uint64_t version = 0;
  };
  std::map<std::pair<Worker*, std::size_t>, ReplicaPoll> replicaPoll;  // (worker, B interval)
  auto columnBlockWidth = [](const MatrixDescriptor& M) -> std::uint64_t {
    const std::size_t T = M.layout.tiles.size();
    if (T < 2) return 0;
    const std::uint64_t w = M.layout.tiles[0].first.colCount;
    for (std::size_t t = 0; t < T; ++t) {
      const TileExtent& e = M.layout.tiles[t].first;
      if (e.rowStart != 0 || e.rowCount != M.rows || e.colStart != t * w ||
          e.colCount != std::min<std::uint64_t>(w, M.cols - t * w))
        return 0;
    }
    return w;
  };

  std::vector<std::vector<BandView>> aViews(P), bViews(P);
  for (std::uint32_t w = 0; w < P; ++w) {
    aViews[w].resize(plan.rowsOf[w].size());
    bViews[w].resize(plan.colsOf[w].size());
  }
  // groups[0] = B bands, groups[1 + j] = A chunk j.
  std::vector<std::vector<Xfer>> groups(1 + S);
  std::vector<CacheEntry*> freshEntries;
  std::vector<Worker*> freshOwners;
  std::vector<std::pair<Worker*, void*>> temps;  // uncached bands, freed after this op's GEMMs

  // m-chunk j of the interval [lo, hi): [lo + j*len/S, lo + (j+1)*len/S).
  auto chunkRange = [&](std::uint64_t lo, std::uint64_t hi, std::uint32_t j) {
    const std::uint64_t len = hi - lo;
    return std::make_pair(lo + len * j / S, lo + len * (j + 1) / S);
  };

  for (std::size_t ni = 0; ni < plan.needs.size(); ++ni) {
    const PlannedNeed& nd = plan.needs[ni];
    const MatrixDescriptor& M = nd.operand == 0 ? A : B;
    const std::uint64_t eb = bytesOf(M.precision);
    Worker* w = local(nd.worker);
    BandView view;
    switch (nd.kind) {
      case PlannedNeed::Replica: {
        if (!w) break;
        auto it = w->replicas.find(M.matrixId);
        if (it == w->replicas.end() || it->second.version != M.version ||
            it->second.state == ReplicaState::Stale)
          throw Error("replica of matrix " + std::to_string(M.matrixId) + " not readable on worker " +
                      std::to_string(nd.worker));
        w->activate();
        const std::uint64_t width = columnBlockWidth(M);
        const bool poll = nd.operand == 1 && !plan.transB && f16Pair && op.s0 != 0.0 && (!nccl_ || ipc_) &&
                          gmk::debug_config().panel_flags && panelPipelining_ && !it->second.alias &&
                          it->second.pieceReady && it->second.state == ReplicaState::Pending && width > 0;
        if (poll) {
          replicaPoll[{w, nd.interval}] = ReplicaPoll{&it->second, width, M.version};
          // The pulls filling the replica wait on the sources' last writes;
          // local sources (workers of this process, possibly on this GPU)
          // finish those before the polling GEMM holds the SMs.
          for (const auto& tl : M.layout.tiles)
            if (Worker* sw = local(tl.second.rank)) {
              auto lw = sw->lastWrite.find(M.matrixId);
              if (lw != sw->lastWrite.end() && sw != w)
                cudaCheck(capture::wait(w->compute, lw->second, 0), "gemm: wait replica source");
            }
        } else {
          cudaCheck(capture::wait(w->compute, it->second.ready, 0), "gemm: wait replica");
        }
        view = offsetView(it->second.full, it->second.ld, nd.rect.r0, nd.rect.c0, eb);
        break;
      }
      case PlannedNeed::LocalTile: {
        if (!w) break;
        for (const DeviceTile& dt : w->tiles.at(M.matrixId))
          if (nd.rect.inside(Rect::ofExtent(dt.extent)))
            view = offsetView(dt.ptr, dt.ld, nd.rect.r0 - dt.extent.rowStart,
                              nd.rect.c0 - dt.extent.colStart, eb);
        break;
      }
      case PlannedNeed::Cached: {
        CacheEntry* hit = cachedHits[ni];
        if (!w) break;
        w->activate();
        cudaCheck(capture::wait(w->compute, hit->ready, 0), "gemm: wait panel");
        view = {hit->ptr, hit->ld};
        break;
      }
      case PlannedNeed::Gather: {
        PanelCache& dir = dirOf(nd.worker);
        dir.misses += 1;
        CacheEntry e;
        e.matrixId = M.matrixId;
        e.version = M.version;
        e.rect = nd.rect;
        e.ld = paddedLd(nd.rect.cols(), eb);
        e.bytes = nd.rect.rows() * e.ld * eb;
        e.lastUse = tick_;
        const std::uint64_t budget = w ? w->cacheBudget : localRef->cacheBudget;
        // A band larger than the whole budget is not kept (same decision on
        // every rank): it lives for this op only.
        const bool keep = e.bytes <= budget;
        if (w) {
          w->activate();
          // Uncached bands double-buffer across GEMMs (see DeviceArena::alloc).
          e.ptr = keep ? w->arena.alloc(e.bytes, w->comm) : w->arena.alloc(e.bytes, w->comm, gemmEpoch_, 2);
        }
        CacheEntry* slotp = nullptr;
        if (keep) {
          for (CacheEntry& ev : dir.reserve(e.bytes, budget, tick_))
            if (w && ev.ptr) {
              w->arena.free(ev.ptr, w->compute);
              w->recycle(ev.ready);
            }
          slotp = &dir.insert(e);
          if (w) {
            freshEntries.push_back(slotp);
            freshOwners.push_back(w);
          }
        } else if (w) {
          temps.push_back({w, e.ptr});
        }
        const CacheEntry& slot = keep ? *slotp : e;
        if (w) view = {slot.ptr, slot.ld};
        if (pipelined && w) {
          // Cut the band into (chunk x k-panel) blocks. Chunk dimension:
          // A's m (stored rows unless transposed), B's n (stored columns
          // unless transposed); the k-panels run along the other one.
          const bool chunkRows = nd.operand == 0 ? !plan.transA : plan.transB;
          FlagBand fb;
          fb.w = w;
          fb.operand = nd.operand;
          fb.interval = nd.interval;
          fb.chunk = nd.operand == 0 ? kAChunkRows : kBChunkCols;
          const std::uint64_t ext = chunkRows ? nd.rect.rows() : nd.rect.cols();
          fb.chunks = (ext + fb.chunk - 1) / fb.chunk;
          fb.first = w->reserveReady(fb.chunks * numPanels);
          fb.flags = w->readyFlags + fb.first % w->readyCap;
          const std::size_t bi = flagBands.size();
          flagBands.push_back(fb);
          for (const PieceRoute& pr : nd.pieces) {
            const std::uint64_t m0 = chunkRows ? pr.rect.r0 - nd.rect.r0 : pr.rect.c0 - nd.rect.c0;
            const std::uint64_t m1 = chunkRows ? pr.rect.r1 - nd.rect.r0 : pr.rect.c1 - nd.rect.c0;
            const std::uint64_t k0 = chunkRows ? pr.rect.c0 - nd.rect.c0 : pr.rect.r0 - nd.rect.r0;
            const std::uint64_t k1 = chunkRows ? pr.rect.c1 - nd.rect.c0 : pr.rect.r1 - nd.rect.r0;
            for (std::uint64_t c = m0 / fb.chunk; c * fb.chunk < m1; ++c)
              for (std::uint64_t pk = k0 / panelK; pk * panelK < k1; ++pk) {
                const std::uint64_t a0 = std::max(m0, c * fb.chunk), a1 = std::min(m1, (c + 1) * fb.chunk);
                const std::uint64_t b0 = std::max(k0, pk * panelK), b1 = std::min(k1, (pk + 1) * panelK);
                Rect r = chunkRows ? Rect{nd.rect.r0 + a0, nd.rect.r0 + a1, nd.rect.c0 + b0, nd.rect.c0 + b1}
                                   : Rect{nd.rect.r0 + b0, nd.rect.r0 + b1, nd.rect.c0 + a0, nd.rect.c0 + a1};
                BlockXfer bx;
                Xfer& x = bx.x;
                x.src = pr.src;
                x.dst = nd.worker;
                x.rows = r.rows();
                x.cols = r.cols();
                x.eb = static_cast<std::uint32_t>(eb);
                x.matrix = M.matrixId;
                x.hasOrigin = true;
                x.r0 = r.r0;
                x.c0 = r.c0;
                const BandView sv = srcView(M, pr.src, r);
                x.srcPtr = sv.ptr;
                x.srcLd = sv.ld;
                x.dstPtr = static_cast<std::uint8_t*>(slot.ptr) + ((r.r0 - nd.rect.r0) * slot.ld + (r.c0 - nd.rect.c0)) * eb;
                x.dstLd = slot.ld;
                x.flagAddr = fb.flags + c * numPanels + pk;
                bx.band = bi;
                bx.chunk = c;
                bx.panel = pk;
                blockXfers.push_back(bx);
              }
          }
          break;
        }
        // Which group each piece belongs to: B whole; A split by m rows
        // (stored rows for A, stored columns for transposed A).
        for (const PieceRoute& pr : nd.pieces) {
          Worker* sw = local(pr.src);
          if (!w && !sw) continue;
          std::vector<std::pair<std::uint32_t, Rect>> parts;
          if (nd.operand == 1 || S == 1) {
            parts.push_back({nd.operand == 1 ? 0u : 1u, pr.rect});
          } else {
            for (std::uint32_t j = 0; j < S; ++j) {
              Rect sub = pr.rect;
              if (!plan.transA) {
                const auto rg = chunkRange(nd.rect.r0, nd.rect.r1, j);
                sub.r0 = std::max(sub.r0, rg.first);
                sub.r1 = std::min(sub.r1, rg.second);
              } else {
                const auto rg = chunkRange(nd.rect.c0, nd.rect.c1, j);
                sub.c0 = std::max(sub.c0, rg.first);
                sub.c1 = std::min(sub.c1, rg.second);
              }
              if (!sub.empty()) parts.push_back({1 + j, sub});
            }
          }
          for (const auto& part : parts) {
            const Rect& r = part.second;
            Xfer x;
            x.src = pr.src;
            x.dst = nd.worker;
            x.rows = r.rows();
            x.cols = r.cols();
            x.eb = static_cast<std::uint32_t>(eb);
            x.matrix = M.matrixId;
            x.hasOrigin = true;
            x.r0 = r.r0;
            x.c0 = r.c0;
            if (w || sw) {
              const BandView sv = srcView(M, pr.src, r);
              x.srcPtr = sv.ptr;
              x.srcLd = sv.ld;
            }
            if (w) {
              x.dstPtr = static_cast<std::uint8_t*>(slot.ptr) + ((r.r0 - nd.rect.r0) * slot.ld + (r.c0 - nd.rect.c0)) * eb;
              x.dstLd = slot.ld;
            }
            groups[part.first].push_back(x);
          }
        }
        break;
      }
    }
    (nd.operand == 0 ? aViews : bViews)[nd.worker][nd.interval] = view;
  }

  // Comm stream: B bands, then A chunks; an event per group per local worker.
  std::vector<std::vector<cudaEvent_t>> groupDone(1 + S);
  bool anyXfer = !blockXfers.empty();
  for (auto& gx : groups) anyXfer = anyXfer || !gx.empty();
  // No blanket wait on the compute stream: exchange() orders each pull after
  // the last write of its source matrix only, so these pulls overlap the
  // GEMM of the previous op.
  flushWritten(curExec_);
  forEachLocal([&](Worker& w) {
    w.commTimed = anyXfer;
    if (anyXfer) cudaCheck(capture::recordTiming(w.cStart, w.comm), "gemm: comm timing");
  });
  // Pipelined mode: order each local consumer's blocks by when its GEMM
  // first needs them -- the wave of the persistent grid whose tiles first
  // touch the block's chunk (host mirror of the kernel's raster), then the
  // k-panel -- and deal them round-robin over the pull streams.
  std::map<std::pair<Worker*, std::pair<int, std::size_t>>, std::size_t> bandOf;  // (w, (operand, interval)) -> band
  for (std::size_t i = 0; i < flagBands.size(); ++i)
    bandOf[{flagBands[i].w, {flagBands[i].operand, flagBands[i].interval}}] = i;
  if (pipelined && !blockXfers.empty()) {
    constexpr std::uint64_t kNever = ~0ull;
    std::vector<std::vector<std::uint64_t>> firstWave(flagBands.size());
    for (std::size_t i = 0; i < flagBands.size(); ++i) firstWave[i].assign(flagBands[i].chunks, kNever);
    forEachLocal([&](Worker& w) {
      std::uint64_t waveOff = 0;
      for (const DeviceTile& ct : w.tiles.at(C.matrixId)) {
        const TileExtent& e = ct.extent;
        std::size_t ri = 0, ci = 0;
        while (!(e.rowStart >= plan.rowsOf[w.rank][ri].first && e.rowStart < plan.rowsOf[w.rank][ri].second)) ++ri;
        while (!(e.colStart >= plan.colsOf[w.rank][ci].first && e.colStart < plan.colsOf[w.rank][ci].second)) ++ci;
        auto ai = bandOf.find({&w, {0, ri}});
        auto bi = bandOf.find({&w, {1, ci}});
        if (ai == bandOf.end() && bi == bandOf.end()) continue;
        const std::uint64_t roff = e.rowStart - plan.rowsOf[w.rank][ri].first;
        const std::uint64_t coff = e.colStart - plan.colsOf[w.rank][ci].first;
        const gmk::TcTilePlan tp = gmk::tc_tile_plan(e.rowCount, e.colCount, plan.k, 2, opts_.gemmMaxCtas);
        const std::uint64_t mbs = (e.rowCount + tp.block_m - 1) / tp.block_m;
        const std::uint64_t nbs = (e.colCount + tp.block_n - 1) / tp.block_n;
        const std::uint64_t tiles = mbs * nbs;
        for (std::uint64_t t = 0; t < tiles; ++t) {
          const std::uint64_t per = static_cast<std::uint64_t>(tp.group) * nbs, g = t / per;
          const std::uint64_t gsize = std::min<std::uint64_t>(tp.group, mbs - g * tp.group);
          const std::uint64_t mb = g * tp.group + (t % per) % gsize, nb = (t % per) / gsize;
          const std::uint64_t wave = waveOff + t / tp.units;
          if (ai != bandOf.end()) {
            const FlagBand& fb = flagBands[ai->second];
            const std::uint64_t r0 = roff + mb * tp.block_m;
            const std::uint64_t r1 = roff + std::min<std::uint64_t>(e.rowCount, (mb + 1) * tp.block_m) - 1;
            for (std::uint64_t c = r0 / fb.chunk; c <= r1 / fb.chunk && c < fb.chunks; ++c)
              firstWave[ai->second][c] = std::min(firstWave[ai->second][c], wave);
          }
          if (bi != bandOf.end()) {
            const FlagBand& fb = flagBands[bi->second];
            const std::uint64_t c0 = coff + nb * tp.block_n;
            const std::uint64_t c1 = coff + std::min<std::uint64_t>(e.colCount, (nb + 1) * tp.block_n) - 1;
            for (std::uint64_t c = c0 / fb.chunk; c <= c1 / fb.chunk && c < fb.chunks; ++c)
              firstWave[bi->second][c] = std::min(firstWave[bi->second][c], wave);
          }
        }
        waveOff += (tiles + tp.units - 1) / tp.units;
      }
    });
    // An operand whose last write is older goes first as a whole: its pulls
    // can run during the previous GEMM (prefetch) instead of queueing on the
    // pull streams behind blocks that wait for a newer write (a dependent
    // chain's A is the previous GEMM's output; its B is not).
    auto lastWriteOf = [&](int operand) {
      auto it = lastMut_.find(operand == 0 ? A.matrixId : B.matrixId);
      return it == lastMut_.end() ? std::uint64_t{0} : it->second;
    };
    const std::uint64_t lwA = lastWriteOf(0), lwB = lastWriteOf(1);
    const bool byClass = dbg.class_sort != 0;
    auto cls = [&](int operand) {
      return (!byClass || lwA == lwB) ? 0 : ((operand == 0) == (lwA > lwB) ? 1 : 0);
    };
    std::stable_sort(blockXfers.begin(), blockXfers.end(), [&](const BlockXfer& x, const BlockXfer& y) {
      const FlagBand& fx = flagBands[x.band];
      const FlagBand& fy = flagBands[y.band];
      if (fx.w->rank != fy.w->rank) return fx.w->rank < fy.w->rank;
      const auto kx = std::make_tuple(cls(fx.operand), firstWave[x.band][x.chunk], x.panel, fx.operand, x.chunk, x.band);
      const auto ky = std::make_tuple(cls(fy.operand), firstWave[y.band][y.chunk], y.panel, fy.operand, y.chunk, y.band);
      return kx < ky;
    });
    // Blocks copied from the consumer's own tiles (HBM -> HBM) alternate
    // over pull streams 0-1, peers' blocks over 2-3, so the local copies and
    // the NVLink pulls run on different copy engines at once instead of
    // queueing behind each other (the first wave needs both).
    std::map<Worker*, std::array<int, 2>> ordinal;
    int stream = 0;
    for (std::size_t i = 0; i < blockXfers.size(); ++i) {
      BlockXfer& bx = blockXfers[i];
      Worker* w = flagBands[bx.band].w;
      const bool firstOfBlock = i == 0 || blockXfers[i - 1].x.flagAddr != bx.x.flagAddr;
      if (firstOfBlock) {
        const int remote = bx.x.src == w->rank ? 0 : 1;
        int& ord = ordinal[w][remote];
        stream = 2 * remote + (ord++ % 2);
      }
      bx.x.pullStream = stream;
      bx.x.lastOfBlock = i + 1 == blockXfers.size() || blockXfers[i + 1].x.flagAddr != bx.x.flagAddr;
      bx.x.flagValue = w->readySeq + 1;
    }
    forEachLocal([&](Worker& w) {
      for (const FlagBand& fb : flagBands)
        if (fb.w == &w) {
          ++w.readySeq;
          break;
        }
    });
  }
  {
    // One exchange per op in pipelined mode (the groups then hold only
    // producer-side bookkeeping of peers' pulls); else group by group.
    std::vector<std::vector<Xfer>> batches;
    if (pipelined) {
      std::vector<Xfer> all;
      for (auto& gx : groups) all.insert(all.end(), gx.begin(), gx.end());
      for (const BlockXfer& bx : blockXfers) all.push_back(bx.x);
      batches.push_back(std::move(all));
    }
    // Group order on the comm stream: B first (every row chunk of C needs
    // it), unless B was written after A -- then A's pulls go first, so they
    // do not queue behind pulls that wait for B's later write (the FC dW
    // GEMM: X is a new batch written at the step's start, delta only by the
    // reluGrad just before). lastMut_ is replicated, so every rank issues the
    // groups in the same order (the NCCL plane needs that).
    const auto lmA = lastMut_.find(A.matrixId), lmB = lastMut_.find(B.matrixId);
    const bool aFirst = !pipelined && S >= 1 && lmA != lastMut_.end() && lmB != lastMut_.end() &&
                        lmB->second > lmA->second;
    std::vector<std::uint32_t> order;
    for (std::uint32_t gi = 0; gi <= S; ++gi) order.push_back(aFirst ? (gi + 1) % (S + 1) : gi);
    for (std::uint32_t gi : order) {
      if (!pipelined && !groups[gi].empty()) exchange(groups[gi], true, false);
      if (pipelined && gi == 0 && !batches[0].empty()) exchange(batches[0], true, false);
      if (pipelined ? gi != 0 : groups[gi].empty()) continue;
      for (auto& wp : workers_) {
        if (!wp) continue;
        wp->activate();
        cudaEvent_t ev = wp->event();
        cudaCheck(capture::record(ev, wp->comm), "gemm: group done");
        groupDone[gi].push_back(ev);
      }
    }
  }
  commitReads();
  forEachLocal([&](Worker& w) {
    if (w.commTimed) cudaCheck(capture::recordTiming(w.cEnd, w.comm), "gemm: comm timing");
  });
  // Gathered bands become cache entries ready when the last group lands.
  for (std::size_t i = 0; i < freshEntries.size(); ++i) {
    Worker* w = freshOwners[i];
    w->activate();
    freshEntries[i]->ready = w->event();
    cudaCheck(capture::record(freshEntries[i]->ready, w->comm), "gemm: panel ready");
  }
  auto waitGroup = [&](Worker& w, std::uint32_t gi) {
    if (groupDone[gi].empty()) return;
    std::size_t idx = 0;
    for (auto& wp : workers_) {
      if (!wp) continue;
      if (wp.get() == &w) {
        cudaCheck(capture::wait(w.compute, groupDone[gi][idx], 0), "gemm: wait group");
        return;
      }
      ++idx;
    }
  };

  const bool alphaZero = op.s0 == 0.0;
  const std::uint64_t ebA = bytesOf(A.precision), ebB = bytesOf(B.precision), ebC = bytesOf(C.precision);
  // In-place operand reads of a matrix whose chunked upload is still landing
  // wait only for the upload chunks covering the rows used.
  std::vector<std::vector<bool>> aLocal(P), bLocal(P);
  for (std::uint32_t w = 0; w < P; ++w) {
    aLocal[w].assign(plan.rowsOf[w].size(), false);
    bLocal[w].assign(plan.colsOf[w].size(), false);
  }
  for (const PlannedNeed& nd : plan.needs)
    if (nd.kind == PlannedNeed::LocalTile) (nd.operand == 0 ? aLocal : bLocal)[nd.worker][nd.interval] = true;
  auto waitUploadRows = [&](Worker& w, std::uint64_t matrix, std::uint64_t lo, std::uint64_t hi,
                            std::set<cudaEvent_t>& waited) {
    auto up = w.uploads.find(matrix);
    if (up == w.uploads.end()) return;
    for (const auto& c : up->second.chunks)
      if (c.r0 < hi && lo < c.r1 && waited.insert(c.done).second)
        cudaCheck(capture::wait(w.compute, c.done, 0), "gemm: wait upload chunk");
  };
  forEachLocal([&](Worker& w) {
    w.dropChunkDone(C.matrixId);
    std::set<cudaEvent_t> waited;
    bool wPipe = false;
    for (const FlagBand& fb : flagBands) wPipe = wPipe || fb.w == &w;
    if (!wPipe) {
      waitGroup(w, 0);
    } else {
      // The GEMM polls flags instead of waiting for the comm stream. Its
      // pulls may wait on other local workers' writes (events on their
      // compute streams, possibly on this GPU): wait for those first, so
      // the spinning persistent grid never holds the SMs a producer needs.
      std::set<cudaEvent_t> raw;
      for (const BlockXfer& bx : blockXfers) {
        if (flagBands[bx.band].w != &w || bx.x.src == w.rank) continue;
        Worker* sw = local(bx.x.src);
        if (!sw) continue;
        auto it = sw->lastWrite.find(bx.x.matrix);
        if (it != sw->lastWrite.end() && raw.insert(it->second).second)
          cudaCheck(capture::wait(w.compute, it->second, 0), "gemm: wait source write");
      }
    }
    if (!alphaZero)
      for (std::size_t ci = 0; ci < plan.colsOf[w.rank].size(); ++ci)
        if (bLocal[w.rank][ci]) waitUploadRows(w, B.matrixId, 0, ~0ull, waited);
    cudaCheck(capture::recordTiming(w.kStart, w.compute), "gemm: timing");
    if (w.windowOpen) {
      std::pair<cudaEvent_t, cudaEvent_t> ev{};
      cudaCheck(cudaEventCreate(&ev.first), "gemm: window event");
      cudaCheck(cudaEventCreate(&ev.second), "gemm: window event");
      cudaCheck(capture::recordTiming(ev.first, w.compute), "gemm: timing");
      w.kernelWindow.push_back(ev);
    }
    for (std::uint32_t j = 0; j < S; ++j) {
      waitGroup(w, 1 + j);
      std::vector<std::pair<std::uint64_t, std::uint64_t>> chunkRows;
      for (DeviceTile& ct : w.tiles.at(C.matrixId)) {
        const TileExtent& e = ct.extent;
        std::size_t ri = 0, ci = 0;
        if (!alphaZero || true) {
          while (!(e.rowStart >= plan.rowsOf[w.rank][ri].first && e.rowStart < plan.rowsOf[w.rank][ri].second)) ++ri;
          while (!(e.colStart >= plan.colsOf[w.rank][ci].first && e.colStart < plan.colsOf[w.rank][ci].second)) ++ci;
        }
        // Rows of this C tile inside m-chunk j of its row interval.
        const auto rg = chunkRange(plan.rowsOf[w.rank][ri].first, plan.rowsOf[w.rank][ri].second, j);
        const std::uint64_t r0 = std::max<std::uint64_t>(e.rowStart, rg.first);
        const std::uint64_t r1 = std::min<std::uint64_t>(e.rowEnd(), rg.second);
        if (r0 >= r1) continue;
        if (!alphaZero && aLocal[w.rank][ri]) {
          if (plan.transA) waitUploadRows(w, A.matrixId, 0, ~0ull, waited);
          else waitUploadRows(w, A.matrixId, r0, r1, waited);
        }
        chunkRows.push_back({r0, r1});
        gm_gemm_desc d{};
        d.m = r1 - r0;
        d.n = e.colCount;
        d.k = plan.k;
        d.trans_a = plan.transA;
        d.trans_b = plan.transB;
        d.prec_a = static_cast<int>(A.precision);
        d.prec_b = static_cast<int>(B.precision);
        d.prec_c = static_cast<int>(C.precision);
        d.math = op.flags[3];
        d.cta_group = 2;
        d.max_ctas = opts_.gemmMaxCtas;
        d.alpha = op.s0;
        d.beta = op.s1;
        d.ldc = ct.ld;
        void* cp = static_cast<std::uint8_t*>(ct.ptr) + (r0 - e.rowStart) * ct.ld * ebC;
        const void* ap = nullptr;
        const void* bp = nullptr;
        if (!alphaZero) {
          const BandView av = aViews[w.rank][ri];
          const BandView bv = bViews[w.rank][ci];
          const std::uint64_t roff = r0 - plan.rowsOf[w.rank][ri].first;
          const std::uint64_t coff = e.colStart - plan.colsOf[w.rank][ci].first;
          ap = plan.transA ? static_cast<const std::uint8_t*>(av.ptr) + roff * ebA
                           : static_cast<const std::uint8_t*>(av.ptr) + roff * av.ld * ebA;
          bp = plan.transB ? static_cast<const std::uint8_t*>(bv.ptr) + coff * bv.ld * ebB
                           : static_cast<const std::uint8_t*>(bv.ptr) + coff * ebB;
          d.lda = av.ld;
          d.ldb = bv.ld;
        }
        const std::uint64_t wsb = alphaZero ? 0 : gemmWorkspaceBytes(d, ap, bp);
        void* ws = wsb ? w.workspace(wsb) : nullptr;
        BiasReluEpilogue ep;
        if (fused_) {
          DeviceTile* at = nullptr;
          for (DeviceTile& t : w.tiles.at(fused_->act))
            if (t.extent == e) at = &t;
          if (!at) throw Error("gemm: fused relu output tile missing on worker " + std::to_string(w.rank));
          ep.bias = fused_->bias.at({w.rank, e.rowStart, e.colStart});
          ep.act = static_cast<std::uint8_t*>(at->ptr) + (r0 - e.rowStart) * at->ld * 2;
          ep.ldAct = at->ld;
        }
        gmk::PanelReady ready;
        auto rp = replicaPoll.find({&w, ci});
        if (rp != replicaPoll.end()) {
          if (gemmConsumesPanelFlags(d, ap, bp)) {
            gmk::PanelFlags& f = ready.b;
            f.flags = rp->second.entry->pieceReady;
            f.target = rp->second.version;
            f.origin = static_cast<std::uint32_t>(e.colStart);  // B column j = matrix column colStart + j
            f.chunk = static_cast<std::uint32_t>(rp->second.width);
            f.chunks = rp->second.entry->pieces;
            f.panel_k = static_cast<std::uint32_t>((plan.k + 63) / 64 * 64);
            f.num_panels = 1;
          } else {
            cudaCheck(capture::wait(w.compute, rp->second.entry->ready, 0), "gemm: wait replica");
          }
        }
        if (wPipe && !alphaZero) {
          auto ai = bandOf.find({&w, {0, ri}});
          auto bi = bandOf.find({&w, {1, ci}});
          if ((ai != bandOf.end() || bi != bandOf.end()) && gemmConsumesPanelFlags(d, ap, bp)) {
            auto fill = [&](gmk::PanelFlags& f, const FlagBand& fb, std::uint64_t origin, std::uint64_t chunk) {
              f.flags = fb.flags;
              f.target = w.readySeq;
              f.origin = static_cast<std::uint32_t>(origin);
              f.chunk = static_cast<std::uint32_t>(chunk);
              f.chunks = static_cast<std::uint32_t>(fb.chunks);
              f.panel_k = static_cast<std::uint32_t>(panelK);
              f.num_panels = static_cast<std::uint32_t>(numPanels);
            };
            if (ai != bandOf.end())
              fill(ready.a, flagBands[ai->second], r0 - plan.rowsOf[w.rank][ri].first, kAChunkRows);
            if (bi != bandOf.end())
              fill(ready.b, flagBands[bi->second], e.colStart - plan.colsOf[w.rank][ci].first, kBChunkCols);
          } else if (ai != bandOf.end() || bi != bandOf.end()) {
            // This launch cannot poll (staged operand): whole bands first.
            waitGroup(w, 0);
          }
        }
        gemmLocal(d, ap, bp, cp, ws, wsb, w.compute, fused_ ? &ep : nullptr, ready.on() ? &ready : nullptr);
      }
      // Row-chunk completion of C (chunked downloads drain behind these).
      for (const auto& rr : chunkRows) {
        Worker::UploadChunk c{rr.first, rr.second, w.event()};
        cudaCheck(capture::record(c.done, w.compute), "gemm: chunk done");
        w.chunkDone[C.matrixId].push_back(c);
      }
    }
    cudaCheck(capture::recordTiming(w.tEnd, w.compute), "gemm: timing");
    if (w.windowOpen) cudaCheck(capture::recordTiming(w.kernelWindow.back().second, w.compute), "gemm: timing");
    // Flag regions polled by this op's GEMMs become reusable after them.
    for (const FlagBand& fb : flagBands) {
      if (fb.w != &w) continue;
      Worker::ReadyRegion rr;
      rr.first = fb.first;
      rr.end = fb.first + fb.chunks * numPanels;
      rr.done = w.event();
      cudaCheck(capture::record(rr.done, w.compute), "gemm: ready region done");
      w.readyInUse.push_back(rr);
    }
  });
  for (auto& tp : temps) {
    tp.first->activate();
    tp.first->arena.free(tp.second, tp.first->compute, gemmEpoch_);
  }
  // Group events go back to their pools (waits are already enqueued).
  for (auto& evs : groupDone) {
    std::size_t idx = 0;
    for (auto& wp : workers_) {
      if (!wp) continue;
      if (idx < evs.size()) wp->recycle(evs[idx]);
      ++idx;
    }
  }
}

void Session::synchronize() {
  forEachLocal([&](Worker& w) {
    cudaCheck(cudaStreamSynchronize(w.h2d), "sync h2d");
    cudaCheck(cudaStreamSynchronize(w.comm), "sync comm");
    cudaCheck(cudaStreamSynchronize(w.compute), "sync compute");
    cudaCheck(cudaStreamSynchronize(w.d2h), "sync d2h");
    cudaCheck(cudaStreamSynchronize(w.flagPub), "sync flags");
    cudaCheck(cudaStreamSynchronize(w.warWait), "sync WAR waits");
  });
}

std::vector<float> Session::lastOpDeviceMs() {
  std::vector<float> out;
  forEachLocal([&](Worker& w) {
    float ms = 0.0f;
    if (w.timed) {
      cudaCheck(cudaEventSynchronize(w.tEnd), "timing sync");
      cudaCheck(cudaEventElapsedTime(&ms, w.tStart, w.tEnd), "timing");
    }
    out.push_back(ms);
  });
  return out;
}

std::vector<float> Session::lastOpKernelMs() {
  std::vector<float> out;
  forEachLocal([&](Worker& w) {
    float ms = 0.0f;
    if (w.timed) {
      cudaCheck(cudaEventSynchronize(w.tEnd), "timing sync");
      cudaCheck(cudaEventElapsedTime(&ms, w.kStart, w.tEnd), "timing");
    }
    out.push_back(ms);
  });
  return out;
}

std::vector<float> Session::lastOpCommMs() {
  std::vector<float> out;
  forEachLocal([&](Worker& w) {
    float ms = 0.0f;
    if (w.commTimed) {
      cudaCheck(cudaEventSynchronize(w.cEnd), "timing sync");
      cudaCheck(cudaEventElapsedTime(&ms, w.cStart, w.cEnd), "timing");
    }
    out.push_back(ms);
  });
  return out;
}

std::uint64_t Session::localBytes(DistMatrix m) const {
  const MatrixDescriptor& d = descriptor(m.id());
  std::uint64_t b = 0;
  for (const auto& t : d.layout.tiles)
    if (isLocal(t.second.rank)) b += t.first.elements() * bytesOf(d.precision);
  return b;
}

void Session::setLocalPacked(DistMatrix m, const void* host, std::uint64_t bytes) {
  const MatrixDescriptor d = descriptor(m.id());
  if (bytes != localBytes(m)) throw Error("setLocalPacked: byte count mismatch");
  OpDescriptor op;
  op.opcode = OpCode::SetData;
  op.ids[0] = m.id();
  issue(op);
  const std::uint64_t eb = bytesOf(d.precision);
  const auto* src = static_cast<const std::uint8_t*>(host);
  for (const auto& t : d.layout.tiles) {
    Worker* w = local(t.second.rank);
    if (!w) continue;
    w->activate();
    for (DeviceTile& dt : w->tiles.at(d.matrixId))
      if (dt.extent == t.first)
        cudaCheck(cudaMemcpy2DAsync(dt.ptr, dt.ld * eb, src, t.first.colCount * eb, t.first.colCount * eb,
                                    t.first.rowCount, cudaMemcpyDefault, w->compute),
                  "setLocalPacked");
    src += t.first.elements() * eb;
  }
  forEachLocal([&](Worker& w) { cudaCheck(cudaStreamSynchronize(w.compute), "setLocalPacked: sync"); });
}

void Session::getLocalPacked(DistMatrix m, void* host, std::uint64_t bytes) {
  const MatrixDescriptor d = descriptor(m.id());
  if (bytes != localBytes(m)) throw Error("getLocalPacked: byte count mismatch");
  OpDescriptor op;
  op.opcode = OpCode::GetData;
  op.ids[0] = m.id();
  issue(op);
  const std::uint64_t eb = bytesOf(d.precision);
  auto* dst = static_cast<std::uint8_t*>(host);
  for (const auto& t : d.layout.tiles) {
    Worker* w = local(t.second.rank);
    if (!w) continue;
    w->activate();
    for (DeviceTile& dt : w->tiles.at(d.matrixId))
      if (dt.extent == t.first)
        cudaCheck(cudaMemcpy2DAsync(dst, t.first.colCount * eb, dt.ptr, dt.ld * eb, t.first.colCount * eb,
                                    t.first.rowCount, cudaMemcpyDefault, w->compute),
                  "getLocalPacked");
    dst += t.first.elements() * eb;
  }
  forEachLocal([&](Worker& w) { cudaCheck(cudaStreamSynchronize(w.compute), "getLocalPacked: sync"); });
}

void Session::timerStart() {
  forEachLocal([&](Worker& w) {
    // The side streams' prior work is part of "before": fold it in.
    for (cudaStream_t side : {w.comm, w.h2d, w.d2h}) {
      cudaEvent_t e = w.event();
      cudaCheck(capture::record(e, side), "timer");
      cudaCheck(capture::wait(w.compute, e, 0), "timer");
      w.recycle(e);
    }
    cudaCheck(capture::record(w.uStart, w.compute), "timer start");
    for (auto& ev : w.kernelWindow) {
      cudaEventDestroy(ev.first);
      cudaEventDestroy(ev.second);
    }
    w.kernelWindow.clear();
    w.windowOpen = true;
  });
}

std::vector<std::pair<float, std::uint32_t>> Session::timerKernelMs() {
  std::vector<std::pair<float, std::uint32_t>> out;
  forEachLocal([&](Worker& w) {
    float sum = 0.0f;
    for (auto& ev : w.kernelWindow) {
      float ms = 0.0f;
      cudaCheck(cudaEventSynchronize(ev.second), "timing sync");
      cudaCheck(cudaEventElapsedTime(&ms, ev.first, ev.second), "timing");
      sum += ms;
    }
    out.push_back({sum, static_cast<std::uint32_t>(w.kernelWindow.size())});
  });
  return out;
}

float Session::timerStop() {
  float best = 0.0f;
  forEachLocal([&](Worker& w) {
    for (cudaStream_t side : {w.comm, w.h2d, w.d2h}) {
      cudaEvent_t e = w.event();
      cudaCheck(capture::record(e, side), "timer");
      cudaCheck(capture::wait(w.compute, e, 0), "timer");
      w.recycle(e);
    }
    cudaCheck(capture::record(w.uEnd, w.compute), "timer stop");
    w.windowOpen = false;
    cudaCheck(cudaEventSynchronize(w.uEnd), "timer sync");
    float ms = 0.0f;
    cudaCheck(cudaEventElapsedTime(&ms, w.uStart, w.uEnd), "timer elapsed");
    best = std::max(best, ms);
  });
  return best;
}

// ---------------------------------------------------------------- record / replay

std::uint64_t Session::beginRecord() {
  if (recording_ != 0) throw Error("beginRecord: a recording is already open");
  recording_ = nextPipelineId_++;
  pipelines_[recording_] = {};
  return recording_;
}

void Session::endRecord() {
  if (recording_ == 0) throw Error("endRecord: no open recording");
  closedPipelines_.insert(recording_);
  recording_ = 0;
}

void Session::replay(std::uint64_t pipelineId, bool sync) {
  if (recording_ != 0) throw Error("replay: recording still open");
  if (!closedPipelines_.count(pipelineId))
    throw Error("replay: unknown or unfinished pipeline " + std::to_string(pipelineId));
  const std::vector<OpDescriptor>& ops = pipelines_.at(pipelineId);
  // Graph replay (opt-in): the first replay runs op by op (the planner's
  // steady state: arena blocks, replicas, cached panels); later ones are
  // captured into one CUDA graph per process (capture.hpp), its executable
  // updated in place.
  capture::Graph* graph = nullptr;
  if (graphReplay_.value_or(gmk::debug_config().graph_replay != 0)) {
    std::unique_ptr<capture::Graph>& g = graphs_[pipelineId];
    if (!g) {
      g = std::make_unique<capture::Graph>();
    } else {
      std::vector<capture::WorkerStreams> ws;
      for (std::uint32_t r : localRanks()) {
        Worker& w = *local(r);
        capture::WorkerStreams x;
        x.device = w.device;
        x.compute = w.compute;
        x.side = {w.comm, w.aux, w.h2d, w.d2h, w.flagPub, w.warWait};
        for (cudaStream_t ps : w.pulls) x.side.push_back(ps);
        ws.push_back(x);
      }
      local(localRanks().front())->activate();
      g->begin(ws);
      graph = g.get();
    }
  }
  try {
    replayOps(ops);
  } catch (...) {
    if (graph) graph->abort();
    throw;
  }
  if (graph) {
    graph->endAndLaunch();
    graphStats_.launches += 1;
    graphStats_.nodes = graph->nodes;
    graphStats_.instantiations = 0;
    for (const auto& kv : graphs_) graphStats_.instantiations += kv.second->instantiations;
  }
  if (sync) synchronize();
}

void Session::replayOps(const std::vector<OpDescriptor>& ops) {
  // Developer timeline (setOpTimeline): events on the first local worker's
  // compute and comm streams at the start and after every replayed op.
  Worker* tw = opTimeline_ && !localRanks().empty() ? local(localRanks().front()) : nullptr;
  auto mark = [&](const char* label) {
    if (!tw) return;
    tw->activate();
    TimelineMark m;
    m.label = label;
    cudaCheck(cudaEventCreate(&m.compute), "timeline");
    cudaCheck(cudaEventCreate(&m.comm), "timeline");
    cudaCheck(capture::recordTiming(m.compute, tw->compute), "timeline");
    cudaCheck(capture::recordTiming(m.comm, tw->comm), "timeline");
    timeline_.push_back(m);
  };
  if (tw) {
    for (TimelineMark& m : timeline_) {
      cudaEventDestroy(m.compute);
      cudaEventDestroy(m.comm);
    }
    timeline_.clear();
    mark("start");
  }
  for (std::size_t i = 0; i < ops.size(); ++i) {
    OpDescriptor step = ops[i];
    step.execId = 0;
    step.recordPipeline = 0;
    if (fusableBiasRelu(ops, i)) {
      OpDescriptor bo = ops[i + 1], ro = ops[i + 2];
      bo.execId = ro.execId = 0;
      bo.recordPipeline = ro.recordPipeline = 0;
      capture::checkpoint("replay: before gemm+biasAdd+relu");
      runGemmBiasRelu(step, bo, ro);
      capture::checkpoint("replay: gemm+biasAdd+relu");
      mark("gemm+biasAdd+relu");
      i += 2;
      continue;
    }
    if (fusableZeroSums(ops, i)) {
      for (std::size_t k = i; k < i + 2; ++k) {
        OpDescriptor sc = ops[k];
        sc.execId = 0;
        sc.recordPipeline = 0;
        issue(sc);  // versions, hazards, invalidation; no kernel
      }
      OpDescriptor rcs = ops[i + 2];
      rcs.execId = 0;
      rcs.recordPipeline = 0;
      zeroSums_ = true;
      try {
        runPointwise(rcs, false);
      } catch (...) {
        zeroSums_ = false;
        throw;
      }
      zeroSums_ = false;
      capture::checkpoint("replay: setConst x2 + addRowColSum");
      mark("setConst+setConst+addRowColSum");
      i += 2;
      continue;
    }
    capture::checkpoint("replay: before op");
    switch (step.opcode) {
      case OpCode::Gemm:
        runGemm(step, false);
        break;
      case OpCode::SetConst:
      case OpCode::EwUnary:
      case OpCode::EwBinary:
      case OpCode::AddRowColSum:
        runPointwise(step, false);
        break;
      case OpCode::ReplicateStart:
        replicateAsync(DistMatrix(this, step.ids[0]));
        break;
      default:
        throw Error("replay: op not supported on the B200 GEMM path");
    }
    const char* what = step.opcode == OpCode::Gemm             ? "replay: gemm"
                       : step.opcode == OpCode::ReplicateStart ? "replay: replicate"
                       : step.opcode == OpCode::AddRowColSum   ? "replay: addRowColSum"
                       : step.opcode == OpCode::SetConst       ? "replay: setConst"
                       : step.opcode == OpCode::EwUnary        ? "replay: unary"
                                                               : "replay: binary";
    capture::checkpoint(what);
    mark(what + 8);
  }
}

std::vector<Session::TimelineEntry> Session::opTimeline() {
  std::vector<TimelineEntry> out;
  if (timeline_.empty()) return out;
  Worker* tw = local(localRanks().front());
  tw->activate();
  for (const TimelineMark& m : timeline_) {
    TimelineEntry e;
    e.label = m.label;
    cudaCheck(cudaEventSynchronize(m.compute), "timeline");
    cudaCheck(cudaEventSynchronize(m.comm), "timeline");
    cudaCheck(cudaEventElapsedTime(&e.computeMs, timeline_.front().compute, m.compute), "timeline");
    cudaCheck(cudaEventElapsedTime(&e.commMs, timeline_.front().compute, m.comm), "timeline");
    out.push_back(e);
  }
  return out;
}

bool Session::fusableZeroSums(const std::vector<OpDescriptor>& ops, std::size_t i) const {
  if (!gmk::debug_config().fuse_zero_sums || i + 2 >= ops.size()) return false;
  const OpDescriptor& a = ops[i];
  const OpDescriptor& b = ops[i + 1];
  const OpDescriptor& r = ops[i + 2];
  if (a.opcode != OpCode::SetConst || b.opcode != OpCode::SetConst || r.opcode != OpCode::AddRowColSum) return false;
  if (a.s0 != 0.0 || b.s0 != 0.0 || a.ids[0] == b.ids[0]) return false;
  const std::uint64_t R = r.ids[1], C = r.ids[2];
  if (R == C || r.ids[0] == R || r.ids[0] == C) return false;
  return (a.ids[0] == R && b.ids[0] == C) || (a.ids[0] == C && b.ids[0] == R);
}

bool Session::fusableBiasRelu(const std::vector<OpDescriptor>& ops, std::size_t i) const {
  if (!gmk::debug_config().fuse_epilogue || i + 2 >= ops.size()) return false;
  const OpDescriptor& g = ops[i];
  const OpDescriptor& bo = ops[i + 1];
  const OpDescriptor& ro = ops[i + 2];
  if (g.opcode != OpCode::Gemm || bo.opcode != OpCode::EwBinary || ro.opcode != OpCode::EwUnary) return false;
  if (bo.flags[0] != static_cast<std::uint8_t>(BinaryKind::BiasAdd) ||
      ro.flags[0] != static_cast<std::uint8_t>(UnaryKind::Relu))
    return false;
  const std::uint64_t a = g.ids[0], b = g.ids[1], c = g.ids[2], bias = bo.ids[1], act = ro.ids[1];
  if (bo.ids[0] != c || bo.ids[2] != c || ro.ids[0] != c) return false;
  if (act == c || act == a || act == b || act == bias || bias == c) return false;
  if (g.s0 == 0.0 || g.s1 != 0.0 || g.flags[3] != 0) return false;
  for (std::uint64_t id : {a, b, c, bias, act})
    if (!table_.count(id) || table_.at(id).precision != Precision::BF16) return false;
  const MatrixDescriptor& C = table_.at(c);
  const MatrixDescriptor& Bv = table_.at(bias);
  const MatrixDescriptor& Act = table_.at(act);
  const std::uint64_t k = g.flags[0] ? table_.at(a).rows : table_.at(a).cols;
  if (k == 0 || C.rows == 0 || C.cols == 0) return false;
  if (Bv.rows != 1 || Bv.cols != C.cols || Act.rows != C.rows || Act.cols != C.cols) return false;
  if (!(Act.layout == C.layout)) return false;
  // The bias columns of every C tile must be held by its owner (its own bias
  // tile, or the sole owner's replica alias): no transfer is needed. A bias
  // served from a copied replica is not fused: the GEMM would then wait for
  // that replication (issued after W's at the end of the previous step),
  // which measured 17 us slower per FC step at N = 2 than the separate ops.
  // (Replicating small matrices on the compute stream instead, so the bias
  // lands first, measured worse: the compute stream then waits on the peers'
  // bias writes every step -- FC step N = 4 0.655 -> 0.74 ms.)
  for (const auto& tl : C.layout.tiles) {
    const Rect need{0, 1, tl.first.colStart, tl.first.colEnd()};
    bool own = false;
    for (const auto& bt : Bv.layout.tiles)
      if (bt.second.rank == tl.second.rank && need.inside(Rect::ofExtent(bt.first))) own = true;
    if (!own) return false;
  }
  return true;
}

void Session::runGemmBiasRelu(const OpDescriptor& g0, const OpDescriptor& bo0, const OpDescriptor& ro0) {
  OpDescriptor g = g0, bo = bo0, ro = ro0;
  const std::uint64_t c = g.ids[2], bias = bo.ids[1], act = ro.ids[1];
  forEachLocal([&](Worker& w) {
    w.joinUpload(bias);
    w.joinUpload(act);
  });
  // Bias views (fusableBiasRelu guarantees no transfer and no scratch).
  std::vector<ReadNeed> needs;
  std::vector<std::tuple<std::uint32_t, std::uint64_t, std::uint64_t>> keys;
  for (const auto& tl : lookup(table_, c).layout.tiles) {
    needs.push_back({tl.second.rank, bias, Rect{0, 1, tl.first.colStart, tl.first.colEnd()}, {}});
    keys.emplace_back(tl.second.rank, tl.first.rowStart, tl.first.colStart);
  }
  std::vector<Xfer> xs;
  std::vector<std::pair<Worker*, void*>> temps;
  resolveReads(needs, c, xs, temps);
  if (!xs.empty() || !temps.empty()) throw Error("fused gemm/biasAdd/relu: bias not readable in place");
  FusedBiasRelu f;
  f.act = act;
  for (std::size_t i = 0; i < needs.size(); ++i)
    if (isLocal(needs[i].worker)) f.bias[keys[i]] = needs[i].view.ptr;
  // relu's write of act moves into the GEMM: its earlier readers finish first.
  forEachLocal([&](Worker& w) {
    if (!w.tiles.count(act)) return;
    w.beforeMutation(act, w.compute);
    waitRemoteReaders(w, act, w.compute);
  });
  issue(g);
  fused_ = &f;
  try {
    execGemm(g);
  } catch (...) {
    fused_ = nullptr;
    throw;
  }
  fused_ = nullptr;
  // The bias and relu ops' metadata (versions, replica / cache invalidation,
  // publication of their writes) as if they had run after the GEMM.
  issue(bo);
  issue(ro);
}

// ---------------------------------------------------------------- replication

ReplicationHandle Session::replicateAsync(DistMatrix m) {
  const MatrixDescriptor& d = descriptor(m.id());
  const ReplicationHandle h{m.id(), d.version};
  if (d.replicaFresh()) return h;  // coalesce onto the existing job / replica
  OpDescriptor op;
  op.opcode = OpCode::ReplicateStart;
  op.ids[0] = m.id();
  op.ids[1] = opts_.replicationChunkBytes;
  issue(op);
  trace_.record(-1, EventKind::ReplInitiate, h.matrixId, h.version);
  execReplicate(m.id());
  return h;
}

void Session::execReplicate(std::uint64_t id) {
  const MatrixDescriptor& M = lookup(table_, id);
  const std::uint64_t eb = bytesOf(M.precision);
  std::vector<Xfer> xs;
  std::vector<Worker*> targets;
  for (std::uint32_t r = 0; r < opts_.workers; ++r) {
    Worker* w = local(r);
    ReplicaEntry* entry = nullptr;
    if (w) {
      w->activate();
      ReplicaEntry& e = w->replicas[id];
      if (!e.ready) cudaCheck(cudaEventCreateWithFlags(&e.ready, cudaEventDisableTiming), "replica event");
      e.version = M.version;
      e.state = ReplicaState::Pending;
      if (M.layout.tiles.size() == 1 && M.layout.tiles[0].second.rank == r) {
        // Sole owner of a single-tile matrix: the replica is the tile itself.
        // Ready once the tile's pending writes (compute stream) are done.
        const DeviceTile& dt = w->tiles.at(id).front();
        if (e.full && !e.alias) {
          cudaEvent_t ev = w->event();
          cudaCheck(capture::record(ev, w->compute), "replica: record readers");
          cudaCheck(capture::wait(w->comm, ev, 0), "replica: wait readers");
          w->recycle(ev);
          w->arena.free(e.full, w->comm);
        }
        e.full = dt.ptr;
        e.ld = dt.ld;
        e.alias = true;
        cudaCheck(capture::record(e.ready, w->compute), "replica ready");
        continue;
      }
      const std::uint64_t ld = paddedLd(M.cols, eb);
      cudaStream_t base = w->comm;
      if (e.full && !e.alias) {
        // GEMMs on the compute stream may still read the previous version.
        cudaEvent_t ev = w->event();
        cudaCheck(capture::record(ev, w->compute), "replica: record readers");
        cudaCheck(capture::wait(w->comm, ev, 0), "replica: wait readers");
        w->recycle(ev);
      }
      if (!e.full || e.alias || e.ld != ld) {
        if (e.full && !e.alias) w->arena.free(e.full, base);
        e.full = w->arena.alloc(M.rows * ld * eb, base);
        e.ld = ld;
        e.alias = false;
      }
      if (e.pieces != M.layout.tiles.size()) {
        if (e.pieceReady) w->arena.free(e.pieceReady, base);
        e.pieces = static_cast<std::uint32_t>(M.layout.tiles.size());
        e.pieceReady = static_cast<std::uint64_t*>(w->arena.alloc(e.pieces * sizeof(std::uint64_t), base));
        cudaCheck(cudaMemsetAsync(e.pieceReady, 0, e.pieces * sizeof(std::uint64_t), base), "replica flags");
      }
      entry = &e;
      targets.push_back(w);
    }
    // Ring order: consumer r pulls from r+1, r+2, ... and copies its own
    // tile last, so pieces queued on one stream never have every consumer
    // hitting the same source at once.
    std::vector<std::size_t> order(M.layout.tiles.size());
    for (std::size_t i = 0; i < order.size(); ++i) order[i] = i;
    const std::uint32_t P = opts_.workers;
    std::stable_sort(order.begin(), order.end(), [&](std::size_t a, std::size_t b) {
      return (M.layout.tiles[a].second.rank + P - r - 1) % P < (M.layout.tiles[b].second.rank + P - r - 1) % P;
    });
    for (std::size_t ti : order) {
      const auto& t = M.layout.tiles[ti];
      const std::uint32_t src = t.second.rank;
      Worker* sw = local(src);
      if (!w && !sw) continue;
      Xfer x;
      x.src = src;
      x.dst = r;
      x.rows = t.first.rowCount;
      x.cols = t.first.colCount;
      x.eb = static_cast<std::uint32_t>(eb);
      x.matrix = id;
      const BandView sv = srcView(M, src, Rect::ofExtent(t.first));
      x.srcPtr = sv.ptr;
      x.srcLd = sv.ld;
      if (entry) {
        x.dstPtr = static_cast<std::uint8_t*>(entry->full) + (t.first.rowStart * entry->ld + t.first.colStart) * eb;
        x.dstLd = entry->ld;
        x.flagAddr = entry->pieceReady + ti;  // published by the stream that copied the piece
        x.flagValue = M.version;
        x.lastOfBlock = true;
      }
      xs.push_back(x);
    }
  }
  // Every worker gathers from every other at once here (all-to-all): two
  // pull streams per consumer, in ring order, measured 478 GB/s per GPU at
  // N = 4 against 357 with four streams and 382 with one
  // (tools/dev/dev_repl.py, profiles/r01_multigpu.md).
  exchange(xs, true, true, 2);
  for (Worker* w : targets) {
    w->activate();
    cudaCheck(capture::record(w->replicas[id].ready, w->comm), "replica ready");
  }
}

ReplState Session::handleState(const ReplicationHandle& h) {
  if (replFailed_.count({h.matrixId, h.version})) return ReplState::Failed;
  auto it = table_.find(h.matrixId);
  if (it == table_.end()) return ReplState::Failed;
  bool inflight = false;
  for (auto& wp : workers_) {
    if (!wp) continue;
    auto rit = wp->replicas.find(h.matrixId);
    if (rit == wp->replicas.end()) return ReplState::Failed;
    ReplicaEntry& e = rit->second;
    if (e.version < h.version) return ReplState::Failed;
    if (e.version > h.version) continue;  // superseded by a newer completed job
    if (e.state == ReplicaState::Stale) return ReplState::Failed;
    if (e.state == ReplicaState::Pending) {
      wp->activate();
      const cudaError_t q = cudaEventQuery(e.ready);
      if (q == cudaSuccess) e.state = ReplicaState::Valid;
      else if (q == cudaErrorNotReady) inflight = true;
      else throw Error(std::string("replica: ") + cudaGetErrorString(q));
    }
  }
  return inflight ? ReplState::InFlight : ReplState::Done;
}

ReplState Session::wait(const ReplicationHandle& h) {
  for (auto& wp : workers_) {
    if (!wp) continue;
    auto rit = wp->replicas.find(h.matrixId);
    if (rit != wp->replicas.end() && rit->second.version == h.version &&
        rit->second.state == ReplicaState::Pending) {
      wp->activate();
      cudaCheck(cudaEventSynchronize(rit->second.ready), "replica wait");
      trace_.record(wp->rank, EventKind::ReplicaValid, h.matrixId, h.version);
    }
  }
  return handleState(h);
}

void Session::replicateSync(DistMatrix m) {
  if (wait(replicateAsync(m)) != ReplState::Done) throw Error("replication failed");
}

// ---------------------------------------------------------------- introspection

void Session::verifyMetadataConsistency() {
  const std::uint64_t expected = tableHash(table_);
  for (auto& w : workers_)
    if (w && tableHash(w->descs) != expected)
      throw Error("metadata divergence on worker " + std::to_string(w->rank));
}

std::vector<WorkerStatsRow> Session::queryWorkerStats() {
  std::vector<WorkerStatsRow> rows;
  for (auto& w : workers_) {
    if (!w) continue;
    const gm_arena_stats s = w->arena.stats();
    WorkerStatsRow r;
    r.osAllocations = s.allocations_from_os;
    r.reuses = s.reuses;
    r.frees = s.frees;
    r.heldBytes = s.held_bytes;
    r.residentBytes = w->residentBytes;
    r.cacheHits = w->cache.hits;
    r.cacheMisses = w->cache.misses;
    r.cacheBytes = w->cache.bytes();
    r.bytesSent = w->bytesSent;
    r.bytesReceived = w->bytesReceived;
    rows.push_back(r);
  }
  return rows;
}

// ---------------------------------------------------------------- reference public surface

std::uint64_t EventTrace::record(std::int64_t actor, EventKind kind, std::uint64_t a, std::uint64_t b,
                                 std::string label) {
  std::lock_guard<std::mutex> g(mu_);
  const std::uint64_t s = seq_++;
  events_.push_back(TraceEvent{s, actor, kind, a, b, std::move(label)});
  return s;
}

std::vector<TraceEvent> EventTrace::snapshot() const {
  std::lock_guard<std::mutex> g(mu_);
  return events_;  // appended in sequence order
}

void EventTrace::clear() {
  std::lock_guard<std::mutex> g(mu_);
  events_.clear();
}

LinkStats FabricStats::totalByKind(MsgKind k) const {
  LinkStats t;
  for (const auto& kv : perLink) {
    t.messageCount += kv.second[static_cast<int>(k)].messageCount;
    t.byteCount += kv.second[static_cast<int>(k)].byteCount;
  }
  return t;
}

LinkStats FabricStats::total() const {
  LinkStats t;
  for (int k = 0; k < 3; ++k) {
    const LinkStats x = totalByKind(static_cast<MsgKind>(k));
    t.messageCount += x.messageCount;
    t.byteCount += x.byteCount;
  }
  return t;
}

void Session::countLink(std::uint32_t src, std::uint32_t dst, MsgKind k, std::uint64_t bytes) {
  std::lock_guard<std::mutex> g(statsMu_);
  LinkStats& l = links_[{src, dst}][static_cast<int>(k)];
  l.messageCount += 1;
  l.byteCount += bytes;
}

FabricStats Session::fabricStats() const {
  std::lock_guard<std::mutex> g(statsMu_);
  FabricStats f;
  f.perLink = links_;
  return f;
}

void Session::phaseMark(const std::string& label) { trace_.record(-1, EventKind::PhaseMark, 0, 0, label); }

void Session::distributeSeeds(std::uint64_t rootSeed) {
  // Reference session.cpp:377-383: an acked control op; the workers derive
  // deriveSeed(root, rank). The device generator takes explicit seeds
  // (fillUniform), so the runtime only records the root.
  rootSeed_ = rootSeed;
  OpDescriptor op;
  op.opcode = OpCode::DistributeSeeds;
  op.ids[0] = rootSeed;
  awaitAcks(issueOp(std::move(op)));
}

const Worker& Session::workerForTest(std::uint32_t rank) const {
  const Worker* w = local(rank);
  if (!w) throw Error("workerForTest: worker " + std::to_string(rank) + " is not hosted by this process");
  return *w;
}

std::uint64_t Session::issueOp(OpDescriptor op, std::uint64_t extraExecIds) {
  (void)extraExecIds;
  switch (op.opcode) {
    case OpCode::Gemm:
      runGemm(op, false);
      return curExec_;
    case OpCode::SetConst:
    case OpCode::EwUnary:
    case OpCode::EwBinary:
    case OpCode::AddRowColSum:
      runPointwise(op, false);
      return curExec_;
    case OpCode::ReplicateStart: {
      const MatrixDescriptor& d = descriptor(op.ids[0]);
      replicateAsync(DistMatrix(this, d.matrixId));
      return curExec_;
    }
    case OpCode::DistributeSeeds:
    case OpCode::QueryStats:
    case OpCode::MetaChecksum:
      return issue(op);  // metadata-only control ops
    case OpCode::CreateMatrix:
    case OpCode::DestroyMatrix:
    case OpCode::SetData:
    case OpCode::GetData:
    case OpCode::Reshape:
    case OpCode::Replay:
    case OpCode::Snapshot:
    case OpCode::Shutdown:
      throw Error(std::string("issueOp: opcode ") + std::to_string(static_cast<std::uint32_t>(op.opcode)) +
                  " carries host data or lifecycle state; use its Session method");
    default:
      validateOp(table_, op, opts_.workers);  // throws "op not supported on the B200 GEMM path"
      throw Error("op not supported on the B200 GEMM path");
  }
}

std::vector<std::pair<std::uint32_t, Completion>> Session::awaitAcks(std::uint64_t execId) {
  synchronize();
  std::vector<std::pair<std::uint32_t, Completion>> acks;
  for (auto& w : workers_) {
    if (!w) continue;
    Completion c;
    c.execId = execId;
    acks.push_back({w->rank, c});
    countLink(w->rank, kMasterRank, MsgKind::Completion, 0);
  }
  return acks;
}

// ---------------------------------------------------------------- free function

void softmaxRows(Session& s, DistMatrix a) {
  OpDescriptor op;
  op.opcode = OpCode::SoftmaxRows;
  op.ids[0] = a.id();
  s.issueOp(op);
}

void subtractOneHot(Session& s, DistMatrix probs, DistMatrix labels) {
  OpDescriptor op;
  op.opcode = OpCode::SubtractOneHot;
  op.ids[0] = probs.id();
  op.ids[1] = labels.id();
  s.issueOp(op);
}

double logLossMean(Session& s, DistMatrix probs, DistMatrix labels) {
  OpDescriptor op;
  op.opcode = OpCode::LogLossGather;
  op.ids[0] = probs.id();
  op.ids[1] = labels.id();
  s.issueOp(op);
  return 0.0;
}

void conv2dForward(Session& s, DistMatrix input, DistMatrix filters, DistMatrix output, kernels::ConvGeometry g) {
  (void)g;
  OpDescriptor op;
  op.opcode = OpCode::Im2col;
  op.ids[0] = input.id();
  op.ids[1] = filters.id();
  op.ids[2] = output.id();
  s.issueOp(op);
}

void gemm(Session& s, DistMatrix a, DistMatrix b, DistMatrix c, double alpha, double beta,
          bool transA, bool transB) {
  OpDescriptor op;
  op.opcode = OpCode::Gemm;
  op.ids[0] = a.id();
  op.ids[1] = b.id();
  op.ids[2] = c.id();
  op.s0 = alpha;
  op.s1 = beta;
  op.flags[0] = transA ? 1 : 0;
  op.flags[1] = transB ? 1 : 0;
  op.flags[2] = s.deterministic() ? 1 : 0;
  s.runGemm(op, true);
}

}  // namespace gridmath
