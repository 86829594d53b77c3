// SPDX-License-Identifier: Apache-2.0
// Core value types of the gridmath drop-in: errors, the counter-based
// generator, the little-endian wire codec, tile layouts, storage precisions,
// matrix descriptors and piece geometry.
//
// Semantics and byte encodings are those of the reference library so that
// descriptors, layouts and op payloads are bit-for-bit compatible:
//   Error / SplitMix64 / fnv1a ........ proj/include/gridmath/common.hpp:11-65
//   WireWriter / WireReader ........... proj/include/gridmath/wire.hpp:14-91
//   Layout + constructors + validate .. proj/include/gridmath/layout.hpp:13-85,
//                                       proj/src/layout.cpp:13-114
//   Precision + fp16 codec ............ proj/include/gridmath/precision.hpp:12-153
//   MatrixDescriptor + codec .......... proj/include/gridmath/descriptor.hpp:15-44
//   Rect / PieceRoute / NeedPlanner ... proj/include/gridmath/pieces.hpp:13-97
// One addition: Precision::BF16 = 3 (bf16 storage). Tags 0..2 are unchanged,
// so descriptors of existing precisions encode to identical bytes.
#pragma once

#include <cstddef>
#include <cstdint>
#include <cstring>
#include <map>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace gridmath {

class Error : public std::runtime_error {
 public:
  explicit Error(const std::string& what) : std::runtime_error(what) {}
};

// ---------------------------------------------------------------- generator
inline constexpr std::uint64_t kSeedSalt = 0x9E3779B97F4A7C15ull;

inline std::uint64_t avalanche64(std::uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

inline std::uint64_t deriveSeed(std::uint64_t rootSeed, std::uint32_t rank) {
  return avalanche64(rootSeed ^ (static_cast<std::uint64_t>(rank) + 1) * kSeedSalt);
}

// Counter-based stream: draw i (0-based) = avalanche64(seed + (i+1)*salt).
class SplitMix64 {
 public:
  explicit SplitMix64(std::uint64_t seed) : state_(seed) {}
  std::uint64_t next() { return avalanche64(state_ += kSeedSalt); }
  double nextUnit() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
  double nextUniform(double lo, double hi) { return lo + (hi - lo) * nextUnit(); }
  std::uint64_t nextBelow(std::uint64_t bound) { return bound ? next() % bound : 0; }

 private:
  std::uint64_t state_;
};

inline std::uint64_t fnv1a(const void* data, std::size_t n,
                           std::uint64_t h = 0xcbf29ce484222325ull) {
  const auto* p = static_cast<const unsigned char*>(data);
  for (std::size_t i = 0; i < n; ++i) h = (h ^ p[i]) * 0x100000001b3ull;
  return h;
}

// ---------------------------------------------------------------- wire codec
class WireWriter {
 public:
  void u8(std::uint8_t v) { buf_.push_back(v); }
  void u32(std::uint32_t v) { put(v, 4); }
  void u64(std::uint64_t v) { put(v, 8); }
  void f64(double v) {
    std::uint64_t b;
    std::memcpy(&b, &v, 8);
    u64(b);
  }
  void bytes(const void* p, std::size_t n) {
    const auto* b = static_cast<const std::uint8_t*>(p);
    buf_.insert(buf_.end(), b, b + n);
  }
  std::vector<std::uint8_t> take() { return std::move(buf_); }
  const std::vector<std::uint8_t>& view() const { return buf_; }

 private:
  void put(std::uint64_t v, int n) {
    for (int i = 0; i < n; ++i) buf_.push_back(static_cast<std::uint8_t>(v >> (8 * i)));
  }
  std::vector<std::uint8_t> buf_;
};

class WireReader {
 public:
  WireReader(const std::uint8_t* p, std::size_t n) : p_(p), n_(n) {}
  explicit WireReader(const std::vector<std::uint8_t>& v) : p_(v.data()), n_(v.size()) {}
  std::uint8_t u8() { return static_cast<std::uint8_t>(get(1)); }
  std::uint32_t u32() { return static_cast<std::uint32_t>(get(4)); }
  std::uint64_t u64() { return get(8); }
  double f64() {
    const std::uint64_t b = u64();
    double v;
    std::memcpy(&v, &b, 8);
    return v;
  }
  void bytes(void* dst, std::size_t n) {
    need(n);
    if (n) std::memcpy(dst, p_ + pos_, n);
    pos_ += n;
  }
  // Borrow the next n bytes (valid while the underlying buffer lives).
  const std::uint8_t* raw(std::size_t n) {
    need(n);
    const std::uint8_t* p = p_ + pos_;
    pos_ += n;
    return p;
  }
  std::size_t remaining() const { return n_ - pos_; }
  bool done() const { return pos_ == n_; }

 private:
  std::uint64_t get(int n) {
    need(static_cast<std::size_t>(n));
    std::uint64_t v = 0;
    for (int i = 0; i < n; ++i) v |= static_cast<std::uint64_t>(p_[pos_ + i]) << (8 * i);
    pos_ += static_cast<std::size_t>(n);
    return v;
  }
  void need(std::size_t n) const {
    if (pos_ + n > n_) throw Error("wire: truncated buffer");
  }
  const std::uint8_t* p_;
  std::size_t n_;
  std::size_t pos_ = 0;
};

// ---------------------------------------------------------------- precision
enum class Precision : std::uint8_t { Half = 0, Single = 1, Double = 2, BF16 = 3 };

std::size_t bytesOf(Precision p);
const char* precisionName(Precision p);
Precision precisionFromTag(std::uint8_t t);

// IEEE binary16: RNE, >= 65520 -> inf, NaN stays NaN (payload >> 13 or 1).
std::uint16_t floatToHalf(float f);
float halfToFloat(std::uint16_t h);  // exact
// bfloat16: RNE from float (NaN -> quiet NaN), exact widening.
std::uint16_t floatToBf16(float f);
float bf16ToFloat(std::uint16_t b);

double loadScalarD(const std::uint8_t* base, Precision p, std::size_t idx);
void storeScalarD(std::uint8_t* base, Precision p, std::size_t idx, double v);
// Elementwise storage conversion (reference convertBuffer semantics).
void convertBuffer(const std::uint8_t* src, Precision srcPrec, std::uint8_t* dst,
                   Precision dstPrec, std::size_t count);

// ---------------------------------------------------------------- layout
struct WorkerId {
  std::uint32_t rank = 0;
  friend bool operator==(WorkerId a, WorkerId b) { return a.rank == b.rank; }
  friend bool operator<(WorkerId a, WorkerId b) { return a.rank < b.rank; }
};

struct TileExtent {
  std::uint64_t rowStart = 0, rowCount = 0, colStart = 0, colCount = 0;
  std::uint64_t rowEnd() const { return rowStart + rowCount; }
  std::uint64_t colEnd() const { return colStart + colCount; }
  std::uint64_t elements() const { return rowCount * colCount; }
  bool contains(std::uint64_t i, std::uint64_t j) const {
    return i >= rowStart && i < rowEnd() && j >= colStart && j < colEnd();
  }
  bool overlaps(const TileExtent& o) const {
    return rowStart < o.rowEnd() && o.rowStart < rowEnd() && colStart < o.colEnd() &&
           o.colStart < colEnd();
  }
  friend bool operator==(const TileExtent& a, const TileExtent& b) {
    return a.rowStart == b.rowStart && a.rowCount == b.rowCount && a.colStart == b.colStart &&
           a.colCount == b.colCount;
  }
};

struct Layout {
  std::vector<std::pair<TileExtent, WorkerId>> tiles;
  friend bool operator==(const Layout& a, const Layout& b) {
    if (a.tiles.size() != b.tiles.size()) return false;
    for (std::size_t i = 0; i < a.tiles.size(); ++i)
      if (!(a.tiles[i].first == b.tiles[i].first) || !(a.tiles[i].second == b.tiles[i].second))
        return false;
    return true;
  }
};

enum class LayoutViolation { Ok, Overlap, Gap, OutOfRange, UnknownWorker };

struct LayoutReport {
  LayoutViolation kind = LayoutViolation::Ok;
  std::string detail;
  bool ok() const { return kind == LayoutViolation::Ok; }
};

std::vector<WorkerId> makeWorkerGroup(std::uint32_t count);
Layout makeRowBlockLayout(std::uint64_t rows, std::uint64_t cols,
                          const std::vector<WorkerId>& workers);
Layout makeColBlockLayout(std::uint64_t rows, std::uint64_t cols,
                          const std::vector<WorkerId>& workers);
Layout makeGridLayout(std::uint64_t rows, std::uint64_t cols, std::uint32_t pr, std::uint32_t pc,
                      const std::vector<WorkerId>& workers);
Layout makeSingleTileLayout(std::uint64_t rows, std::uint64_t cols, WorkerId owner);
LayoutReport validateLayout(std::uint64_t rows, std::uint64_t cols, const Layout& layout,
                            std::uint32_t workerCount = 0);
WorkerId tileOwner(const Layout& layout, std::uint64_t i, std::uint64_t j);

// ---------------------------------------------------------------- descriptor
struct MatrixDescriptor {
  std::uint64_t matrixId = 0;
  std::uint64_t rows = 0;
  std::uint64_t cols = 0;
  Precision precision = Precision::Single;
  Layout layout;
  std::uint64_t version = 0;
  // Not on the wire: set by ReplicateStart at issue time; kernels read the
  // local replica while it equals `version`.
  std::uint64_t replicatedVersion = ~0ull;

  std::uint64_t elementCount() const { return rows * cols; }
  std::uint64_t byteCount() const { return elementCount() * bytesOf(precision); }
  bool replicaFresh() const { return replicatedVersion == version; }
};

// u64 id, u64 rows, u64 cols, u8 precision, u64 version, u32 tiles,
// per tile 4 x u64 extent + u32 rank.
void encodeDescriptor(const MatrixDescriptor& d, WireWriter& w);
MatrixDescriptor decodeDescriptor(WireReader& r);
std::uint64_t descriptorHash(const MatrixDescriptor& d);
using DescriptorTable = std::map<std::uint64_t, MatrixDescriptor>;
std::uint64_t tableHash(const DescriptorTable& t);

// ---------------------------------------------------------------- pieces
struct Rect {
  std::uint64_t r0 = 0, r1 = 0, c0 = 0, c1 = 0;
  std::uint64_t rows() const { return r1 - r0; }
  std::uint64_t cols() const { return c1 - c0; }
  std::uint64_t elements() const { return rows() * cols(); }
  bool empty() const { return r0 >= r1 || c0 >= c1; }
  bool inside(const Rect& o) const { return r0 >= o.r0 && r1 <= o.r1 && c0 >= o.c0 && c1 <= o.c1; }
  static Rect ofExtent(const TileExtent& e) { return {e.rowStart, e.rowEnd(), e.colStart, e.colEnd()}; }
  static Rect full(const MatrixDescriptor& d) { return {0, d.rows, 0, d.cols}; }
  friend bool operator==(const Rect& a, const Rect& b) {
    return a.r0 == b.r0 && a.r1 == b.r1 && a.c0 == b.c0 && a.c1 == b.c1;
  }
  friend bool operator<(const Rect& a, const Rect& b) {
    if (a.r0 != b.r0) return a.r0 < b.r0;
    if (a.r1 != b.r1) return a.r1 < b.r1;
    if (a.c0 != b.c0) return a.c0 < b.c0;
    return a.c1 < b.c1;
  }
};

std::optional<Rect> intersectRect(const Rect& a, const Rect& b);

struct PieceRoute {
  std::uint32_t pieceId = 0;
  std::uint32_t src = 0;
  std::uint32_t consumer = 0;
  std::uint64_t matrixId = 0;
  Rect rect;
};

struct RegionNeed {
  std::uint64_t matrixId = 0;
  std::uint32_t consumer = 0;
  Rect rect;
  bool viaReplica = false;
  std::vector<PieceRoute> pieces;  // empty when viaReplica
};

class NeedPlanner {
 public:
  RegionNeed& addNeed(const MatrixDescriptor& d, const Rect& rect, std::uint32_t consumer,
                      bool allowReplica);
  const std::vector<RegionNeed>& needs() const { return needs_; }
  std::vector<RegionNeed>& needs() { return needs_; }
  std::uint32_t pieceCount() const { return nextPieceId_; }

 private:
  std::uint32_t nextPieceId_ = 0;
  std::vector<RegionNeed> needs_;
};

struct ByteRun {
  std::uint64_t offset = 0, length = 0;
};
std::vector<ByteRun> tileByteRuns(const MatrixDescriptor& d, const TileExtent& e);

// Host row-major rectangle pack/unpack (tile buffer row-major over `extent`).
void packRect(const std::uint8_t* tileData, const TileExtent& extent, const Rect& rect,
              std::size_t elemBytes, std::uint8_t* out);
void unpackRect(std::uint8_t* tileData, const TileExtent& extent, const Rect& rect,
                std::size_t elemBytes, const std::uint8_t* in);

}  // namespace gridmath
