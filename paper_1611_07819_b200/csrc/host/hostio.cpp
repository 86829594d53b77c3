// SPDX-License-Identifier: Apache-2.0
// Host <-> device streaming of a worker's own tiles (packed local I/O), the
// operand path of a caller that keeps its matrices in host memory: the
// reference's setData / getData (session.cpp:240-308) restated for one
// process per GPU, made asynchronous and chunked so PCIe traffic overlaps
// the tensor-core work:
//   * uploads move in row chunks on the worker's h2d stream, one event per
//     chunk; the next GEMM that reads the tile in place waits only for the
//     rows each of its row chunks needs (execGemm), everything else joins the
//     whole upload first (Session::joinUploads);
//   * downloads wait per row chunk for the producing GEMM's chunk events
//     (Worker::chunkDone) and run on the d2h stream, so C drains while later
//     chunks are still being computed.
#include <cuda_runtime.h>

#include <algorithm>

#include "capture.hpp"
#include "internal.hpp"
#include "runtime.hpp"

namespace gridmath {

void Session::setLocalPackedAsync(DistMatrix m, const void* host, std::uint64_t bytes, std::uint64_t chunkBytes) {
  const MatrixDescriptor d = descriptor(m.id());
  if (bytes != localBytes(m)) throw Error("setLocalPacked: byte count mismatch");
  const std::uint64_t chunk = chunkBytes ? chunkBytes : (256ull << 20);
  OpDescriptor op;
  op.opcode = OpCode::SetData;
  op.ids[0] = m.id();
  op.ids[1] = chunk;  // the chunk geometry travels with the op: every rank can follow the chunks
  issue(op);  // joins an earlier upload of m (WAW); WAR waits land on the compute stream
  const std::uint64_t eb = bytesOf(d.precision);
  // Replicated chunk bookkeeping: each owner's upload-chunk counter for the
  // matrix's flag slot advances by its number of chunks.
  if (ipc_) {
    ChunkedWrite cw;
    cw.execId = op.execId;
    cw.chunkBytes = chunk;
    cw.base.assign(opts_.workers, 0);
    const std::uint32_t slot = slotOf(m.id());
    std::vector<std::uint32_t> n(opts_.workers, 0);
    for (const auto& t : d.layout.tiles) {
      const std::uint64_t rpc = std::max<std::uint64_t>(1, chunk / std::max<std::uint64_t>(t.first.colCount * eb, 1));
      n[t.second.rank] += static_cast<std::uint32_t>((t.first.rowCount + rpc - 1) / rpc);
    }
    for (std::uint32_t r = 0; r < opts_.workers; ++r) {
      std::uint64_t& cnt = upCount_[{r, slot}];
      cw.base[r] = cnt;
      cnt += n[r];
    }
    chunked_[m.id()] = std::move(cw);
  } else {
    ChunkedWrite cw;
    cw.execId = op.execId;
    cw.chunkBytes = chunk;
    chunked_[m.id()] = std::move(cw);
  }
  const auto* src = static_cast<const std::uint8_t*>(host);
  std::set<Worker*> started;
  for (const auto& t : d.layout.tiles) {
    Worker* w = local(t.second.rank);
    if (!w) continue;
    w->activate();
    if (started.insert(w).second) {
      // WAR: issue() made the h2d stream wait for the old contents' last use
      // on the compute stream, their readers on other streams and the peers'
      // pulls -- not for unrelated compute, which the upload overlaps.
      w->dropChunkDone(m.id());
    }
    Worker::Upload& up = w->uploads[m.id()];
    const TileExtent& e = t.first;
    for (DeviceTile& dt : w->tiles.at(d.matrixId)) {
      if (!(dt.extent == e)) continue;
      const std::uint64_t rowBytes = e.colCount * eb;
      const std::uint64_t rpc = std::max<std::uint64_t>(1, chunk / std::max<std::uint64_t>(rowBytes, 1));
      for (std::uint64_t r = 0; r < e.rowCount; r += rpc) {
        const std::uint64_t n = std::min(rpc, e.rowCount - r);
        cudaCheck(cudaMemcpy2DAsync(static_cast<std::uint8_t*>(dt.ptr) + r * dt.ld * eb, dt.ld * eb,
                                    src + r * rowBytes, rowBytes, rowBytes, n, cudaMemcpyDefault, w->h2d),
                  "upload: chunk");
        Worker::UploadChunk c{e.rowStart + r, e.rowStart + r + n, w->event()};
        cudaCheck(capture::record(c.done, w->h2d), "upload: chunk event");
        if (ipc_)  // peers pulling these rows wait for this value (ChunkedWrite::base)
          ipcWrite(w->h2d, w->flags + kUpChunkOff + slotOf(m.id()),
                   chunked_.at(m.id()).base[w->rank] + static_cast<std::uint64_t>(up.chunks.size()) + 1);
        up.chunks.push_back(c);
      }
    }
    src += e.elements() * eb;
  }
  for (Worker* w : started) {
    Worker::Upload& up = w->uploads[m.id()];
    up.done = w->event();
    cudaCheck(capture::record(up.done, w->h2d), "upload: done");
  }
}

void Session::getLocalPackedAsync(DistMatrix m, void* host, std::uint64_t bytes) {
  const MatrixDescriptor d = descriptor(m.id());
  if (bytes != localBytes(m)) throw Error("getLocalPacked: byte count mismatch");
  OpDescriptor op;
  op.opcode = OpCode::GetData;
  op.ids[0] = m.id();
  issue(op);
  const std::uint64_t eb = bytesOf(d.precision);
  auto* dst = static_cast<std::uint8_t*>(host);
  std::set<Worker*> used;
  for (const auto& t : d.layout.tiles) {
    Worker* w = local(t.second.rank);
    if (!w) continue;
    w->activate();
    used.insert(w);
    const TileExtent& e = t.first;
    const std::uint64_t rowBytes = e.colCount * eb;
    for (DeviceTile& dt : w->tiles.at(d.matrixId)) {
      if (!(dt.extent == e)) continue;
      // Row ranges covered by the last writer's chunk events; the rest (or
      // everything, if the last writer did not work in chunks) follows the
      // compute stream as a whole.
      std::vector<Worker::UploadChunk> parts;
      auto cd = w->chunkDone.find(m.id());
      if (cd != w->chunkDone.end())
        for (const auto& c : cd->second) {
          const std::uint64_t lo = std::max(c.r0, e.rowStart), hi = std::min(c.r1, e.rowEnd());
          if (lo < hi) parts.push_back({lo, hi, c.done});
        }
      std::sort(parts.begin(), parts.end(), [](const auto& a, const auto& b) { return a.r0 < b.r0; });
      std::uint64_t covered = e.rowStart;
      bool contiguous = true;
      for (const auto& p : parts) {
        if (p.r0 != covered) contiguous = false;
        covered = std::max(covered, p.r1);
      }
      if (parts.empty() || !contiguous || covered != e.rowEnd()) {
        cudaEvent_t ev = w->event();
        cudaCheck(capture::record(ev, w->compute), "download: order");
        parts.assign(1, Worker::UploadChunk{e.rowStart, e.rowEnd(), ev});
        cudaCheck(capture::wait(w->d2h, ev, 0), "download: wait");
        w->recycle(ev);
        parts[0].done = nullptr;
      }
      for (const auto& p : parts) {
        if (p.done) cudaCheck(capture::wait(w->d2h, p.done, 0), "download: wait chunk");
        const std::uint64_t r = p.r0 - e.rowStart;
        cudaCheck(cudaMemcpy2DAsync(dst + r * rowBytes, rowBytes, static_cast<const std::uint8_t*>(dt.ptr) + r * dt.ld * eb,
                                    dt.ld * eb, rowBytes, p.r1 - p.r0, cudaMemcpyDefault, w->d2h),
                  "download: chunk");
      }
    }
    dst += e.elements() * eb;
  }
  // WAR: the next mutation of m waits for these reads.
  for (Worker* w : used) {
    cudaEvent_t e = w->event();
    cudaCheck(capture::record(e, w->d2h), "download: done");
    w->addReader(m.id(), e, w);
  }
}

}  // namespace gridmath
