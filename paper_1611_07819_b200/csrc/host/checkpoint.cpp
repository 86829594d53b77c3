// SPDX-License-Identifier: Apache-2.0
// Checkpoint-restart of device-resident matrices, in the
// reference's DMCK file format so checkpoints move freely between the two
// implementations (reference Session::checkpoint / restore,
// proj/src/session.cpp:413-480):
//   "DMCK" | u32 version = 1 | u64 root seed | u32 matrix count |
//   per matrix in ascending id: descriptor (descriptor.cpp encoding) + full
//   row-major image in storage precision | u32 CRC-32 (zlib) of everything
//   between the magic and the CRC.
// Images come off the GPUs through getDataRaw (2D copies per tile; SPMD:
// every rank gathers, rank 0 writes) and are streamed to the file with an
// incremental CRC, one matrix in host memory at a time. Restore creates each
// matrix with its saved id and version (layouts that do not fit the new
// worker count fall back to a row-block layout, like the reference), then
// uploads it with a SetData op (version + 1, as in the reference).
#include <zlib.h>

#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "internal.hpp"
#include "runtime.hpp"

namespace gridmath {

namespace {
constexpr char kCheckpointMagic[4] = {'D', 'M', 'C', 'K'};
constexpr std::uint32_t kCheckpointVersion = 1;

struct FileCloser {
  void operator()(std::FILE* f) const {
    if (f) std::fclose(f);
  }
};
}  // namespace

void Session::checkpoint(const std::string& path) {
  // Reference: refuse while a replication job is still moving bytes.
  for (auto& wp : workers_) {
    if (!wp) continue;
    wp->activate();
    for (auto& [id, e] : wp->replicas) {
      if (e.state != ReplicaState::Pending) continue;
      const cudaError_t q = cudaEventQuery(e.ready);
      if (q == cudaSuccess) {
        e.state = ReplicaState::Valid;
      } else if (q == cudaErrorNotReady) {
        throw Error("checkpoint: replication of matrix " + std::to_string(id) + " still in flight");
      } else {
        throw Error(std::string("checkpoint: ") + cudaGetErrorString(q));
      }
    }
  }
  const bool writer = opts_.spmdRank <= 0;
  std::unique_ptr<std::FILE, FileCloser> f;
  if (writer) {
    f.reset(std::fopen(path.c_str(), "wb"));
    if (!f) throw Error("checkpoint: cannot open " + path);
  }
  uLong crc = ::crc32(0L, Z_NULL, 0);
  auto emit = [&](const void* p, std::size_t n) {
    const auto* b = static_cast<const Bytef*>(p);
    for (std::size_t off = 0; off < n;) {  // zlib takes uInt lengths
      const std::size_t len = std::min<std::size_t>(n - off, 1u << 30);
      crc = ::crc32(crc, b + off, static_cast<uInt>(len));
      off += len;
    }
    if (f && n && std::fwrite(p, 1, n, f.get()) != n) throw Error("checkpoint: write failed");
  };
  if (f && std::fwrite(kCheckpointMagic, 1, 4, f.get()) != 4) throw Error("checkpoint: write failed");
  {
    WireWriter h;
    h.u32(kCheckpointVersion);
    h.u64(opts_.rootSeed);
    h.u32(static_cast<std::uint32_t>(table_.size()));
    emit(h.view().data(), h.view().size());
  }
  std::vector<std::uint64_t> ids;
  for (const auto& kv : table_) ids.push_back(kv.first);
  std::vector<std::uint8_t> image;
  for (std::uint64_t id : ids) {
    WireWriter w;
    encodeDescriptor(table_.at(id), w);
    emit(w.view().data(), w.view().size());
    image.resize(table_.at(id).byteCount());
    getDataRawInto(DistMatrix(this, id), image.data(), image.size(), false);
    emit(image.data(), image.size());
  }
  WireWriter tail;
  tail.u32(static_cast<std::uint32_t>(crc));
  if (f) {
    if (std::fwrite(tail.view().data(), 1, 4, f.get()) != 4 || std::fflush(f.get()) != 0)
      throw Error("checkpoint: write failed");
  }
}

std::unique_ptr<Session> Session::restore(const std::string& path, SessionOptions opts) {
  std::vector<std::uint8_t> bytes;
  {
    std::unique_ptr<std::FILE, FileCloser> f(std::fopen(path.c_str(), "rb"));
    if (!f) throw Error("restore: cannot open " + path);
    std::fseek(f.get(), 0, SEEK_END);
    const long len = std::ftell(f.get());
    std::fseek(f.get(), 0, SEEK_SET);
    bytes.resize(len > 0 ? static_cast<std::size_t>(len) : 0);
    if (!bytes.empty() && std::fread(bytes.data(), 1, bytes.size(), f.get()) != bytes.size())
      throw Error("restore: read failed");
  }
  if (bytes.size() < 4 + 4 + 8 + 4 + 4 || std::memcmp(bytes.data(), kCheckpointMagic, 4) != 0)
    throw Error("restore: corrupt file (bad magic or truncated)");
  const std::size_t bodyLen = bytes.size() - 4 - 4;
  uLong crc = ::crc32(0L, Z_NULL, 0);
  for (std::size_t off = 0; off < bodyLen;) {
    const std::size_t len = std::min<std::size_t>(bodyLen - off, 1u << 30);
    crc = ::crc32(crc, bytes.data() + 4 + off, static_cast<uInt>(len));
    off += len;
  }
  WireReader tail(bytes.data() + 4 + bodyLen, 4);
  if (tail.u32() != static_cast<std::uint32_t>(crc)) throw Error("restore: corrupt file (CRC mismatch)");

  WireReader r(bytes.data() + 4, bodyLen);
  if (r.u32() != kCheckpointVersion) throw Error("restore: unsupported format version");
  opts.rootSeed = r.u64();
  const std::uint32_t count = r.u32();
  auto session = std::make_unique<Session>(opts);
  for (std::uint32_t i = 0; i < count; ++i) {
    MatrixDescriptor d = decodeDescriptor(r);
    const std::uint64_t payloadBytes = d.byteCount();
    const std::uint8_t* payload = r.raw(payloadBytes);
    if (!validateLayout(d.rows, d.cols, d.layout, opts.workers).ok())
      d.layout = makeRowBlockLayout(d.rows, d.cols, makeWorkerGroup(opts.workers));
    const DistMatrix m = session->createWithDescriptor(d);
    session->setDataRaw(m, payload, payloadBytes);
  }
  if (!r.done()) throw Error("restore: trailing bytes");
  return session;
}

}  // namespace gridmath
