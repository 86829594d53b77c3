// SPDX-License-Identifier: Apache-2.0
// Implementation of the core value types (see core.hpp for the reference
// file:line each one follows).
#include "core.hpp"

#include <algorithm>
#include <bit>
#include <cmath>

namespace gridmath {

// ---------------------------------------------------------------- precision

std::size_t bytesOf(Precision p) {
  switch (p) {
    case Precision::Half: return 2;
    case Precision::Single: return 4;
    case Precision::Double: return 8;
    case Precision::BF16: return 2;
  }
  throw Error("bad precision tag");
}

const char* precisionName(Precision p) {
  switch (p) {
    case Precision::Half: return "half";
    case Precision::Single: return "single";
    case Precision::Double: return "double";
    case Precision::BF16: return "bf16";
  }
  return "?";
}

Precision precisionFromTag(std::uint8_t t) {
  if (t > 3) throw Error("bad precision tag");
  return static_cast<Precision>(t);
}

std::uint16_t floatToHalf(float f) {
  const std::uint32_t x = std::bit_cast<std::uint32_t>(f);
  const std::uint16_t sign = static_cast<std::uint16_t>((x >> 16) & 0x8000u);
  const std::uint32_t ax = x & 0x7FFFFFFFu;
  if (ax > 0x7F800000u) {  // NaN keeps a nonzero payload
    const std::uint32_t pay = (ax & 0x007FFFFFu) >> 13;
    return static_cast<std::uint16_t>(sign | 0x7C00u | (pay ? pay : 1u));
  }
  if (ax >= 0x477FF000u) return static_cast<std::uint16_t>(sign | 0x7C00u);  // >= 65520 or inf
  if (ax < 0x38800000u) {
    // Below 2^-14: binary16 subnormal step is 2^-24; the scaled value is
    // exact in double and nearbyint rounds half to even.
    const double scaled = static_cast<double>(std::bit_cast<float>(ax)) * 16777216.0;
    return static_cast<std::uint16_t>(sign | static_cast<std::uint16_t>(std::nearbyint(scaled)));
  }
  const std::uint32_t e = ax >> 23;
  const std::uint32_t m = ax & 0x007FFFFFu;
  std::uint32_t h = ((e - 112u) << 10) | (m >> 13);
  const std::uint32_t rem = m & 0x1FFFu;
  if (rem > 0x1000u || (rem == 0x1000u && (h & 1u))) ++h;  // carry may reach the exponent
  return static_cast<std::uint16_t>(sign | h);
}

float halfToFloat(std::uint16_t h) {
  const std::uint32_t sign = static_cast<std::uint32_t>(h & 0x8000u) << 16;
  const std::uint32_t e = (h >> 10) & 0x1Fu;
  const std::uint32_t m = h & 0x3FFu;
  if (e == 31) return std::bit_cast<float>(sign | 0x7F800000u | (m << 13));
  const float mag = e == 0 ? std::ldexp(static_cast<float>(m), -24)
                           : std::ldexp(static_cast<float>(m | 0x400u), static_cast<int>(e) - 25);
  return sign ? -mag : mag;
}

std::uint16_t floatToBf16(float f) {
  std::uint32_t u = std::bit_cast<std::uint32_t>(f);
  if ((u & 0x7FFFFFFFu) > 0x7F800000u) return 0x7FFFu;  // same canonical NaN as cuda_bf16
  u += 0x7FFFu + ((u >> 16) & 1u);
  return static_cast<std::uint16_t>(u >> 16);
}

float bf16ToFloat(std::uint16_t b) { return std::bit_cast<float>(static_cast<std::uint32_t>(b) << 16); }

double loadScalarD(const std::uint8_t* base, Precision p, std::size_t idx) {
  switch (p) {
    case Precision::Half: {
      std::uint16_t h;
      std::memcpy(&h, base + idx * 2, 2);
      return halfToFloat(h);
    }
    case Precision::Single: {
      float f;
      std::memcpy(&f, base + idx * 4, 4);
      return f;
    }
    case Precision::Double: {
      double d;
      std::memcpy(&d, base + idx * 8, 8);
      return d;
    }
    case Precision::BF16: {
      std::uint16_t b;
      std::memcpy(&b, base + idx * 2, 2);
      return bf16ToFloat(b);
    }
  }
  throw Error("bad precision tag");
}

void storeScalarD(std::uint8_t* base, Precision p, std::size_t idx, double v) {
  switch (p) {
    case Precision::Half: {
      const std::uint16_t h = floatToHalf(static_cast<float>(v));
      std::memcpy(base + idx * 2, &h, 2);
      return;
    }
    case Precision::Single: {
      const float f = static_cast<float>(v);
      std::memcpy(base + idx * 4, &f, 4);
      return;
    }
    case Precision::Double:
      std::memcpy(base + idx * 8, &v, 8);
      return;
    case Precision::BF16: {
      const std::uint16_t b = floatToBf16(static_cast<float>(v));
      std::memcpy(base + idx * 2, &b, 2);
      return;
    }
  }
  throw Error("bad precision tag");
}

void convertBuffer(const std::uint8_t* src, Precision srcPrec, std::uint8_t* dst,
                   Precision dstPrec, std::size_t count) {
  if (srcPrec == dstPrec) {
    std::memcpy(dst, src, count * bytesOf(srcPrec));
    return;
  }
  for (std::size_t i = 0; i < count; ++i) storeScalarD(dst, dstPrec, i, loadScalarD(src, srcPrec, i));
}

// ---------------------------------------------------------------- layout

namespace {
// Near-equal split of n into `parts` (earliest parts take the remainder);
// empty parts are dropped.
std::vector<std::pair<std::uint64_t, std::uint64_t>> evenSplit(std::uint64_t n,
                                                              std::uint64_t parts) {
  std::vector<std::pair<std::uint64_t, std::uint64_t>> out;
  std::uint64_t at = 0;
  for (std::uint64_t p = 0; p < parts; ++p) {
    const std::uint64_t len = n / parts + (p < n % parts ? 1 : 0);
    if (len == 0) continue;
    out.emplace_back(at, len);
    at += len;
  }
  return out;
}
}  // namespace

std::vector<WorkerId> makeWorkerGroup(std::uint32_t count) {
  std::vector<WorkerId> g(count);
  for (std::uint32_t i = 0; i < count; ++i) g[i].rank = i;
  return g;
}

Layout makeRowBlockLayout(std::uint64_t rows, std::uint64_t cols,
                          const std::vector<WorkerId>& workers) {
  if (workers.empty()) throw Error("makeRowBlockLayout: empty worker list");
  if (rows == 0 || cols == 0) throw Error("makeRowBlockLayout: zero-sized matrix");
  Layout l;
  const auto bands = evenSplit(rows, workers.size());
  for (std::size_t i = 0; i < bands.size(); ++i)
    l.tiles.push_back({TileExtent{bands[i].first, bands[i].second, 0, cols}, workers[i]});
  return l;
}

Layout makeColBlockLayout(std::uint64_t rows, std::uint64_t cols,
                          const std::vector<WorkerId>& workers) {
  if (workers.empty()) throw Error("makeColBlockLayout: empty worker list");
  if (rows == 0 || cols == 0) throw Error("makeColBlockLayout: zero-sized matrix");
  Layout l;
  const auto bands = evenSplit(cols, workers.size());
  for (std::size_t i = 0; i < bands.size(); ++i)
    l.tiles.push_back({TileExtent{0, rows, bands[i].first, bands[i].second}, workers[i]});
  return l;
}

Layout makeGridLayout(std::uint64_t rows, std::uint64_t cols, std::uint32_t pr, std::uint32_t pc,
                      const std::vector<WorkerId>& workers) {
  if (static_cast<std::uint64_t>(pr) * pc != workers.size())
    throw Error("makeGridLayout: pr*pc must equal worker count");
  if (rows == 0 || cols == 0) throw Error("makeGridLayout: zero-sized matrix");
  Layout l;
  const auto rb = evenSplit(rows, pr);
  const auto cb = evenSplit(cols, pc);
  for (std::size_t r = 0; r < rb.size(); ++r)
    for (std::size_t c = 0; c < cb.size(); ++c)
      l.tiles.push_back({TileExtent{rb[r].first, rb[r].second, cb[c].first, cb[c].second},
                         workers[r * pc + c]});
  return l;
}

Layout makeSingleTileLayout(std::uint64_t rows, std::uint64_t cols, WorkerId owner) {
  Layout l;
  l.tiles.push_back({TileExtent{0, rows, 0, cols}, owner});
  return l;
}

LayoutReport validateLayout(std::uint64_t rows, std::uint64_t cols, const Layout& layout,
                            std::uint32_t workerCount) {
  std::uint64_t covered = 0;
  for (std::size_t i = 0; i < layout.tiles.size(); ++i) {
    const TileExtent& e = layout.tiles[i].first;
    const WorkerId w = layout.tiles[i].second;
    const std::string tag = "tile " + std::to_string(i);
    if (e.rowCount == 0 || e.colCount == 0) return {LayoutViolation::OutOfRange, tag + " is empty"};
    if (e.rowEnd() > rows || e.colEnd() > cols)
      return {LayoutViolation::OutOfRange, tag + " exceeds matrix bounds"};
    if (workerCount != 0 && w.rank >= workerCount)
      return {LayoutViolation::UnknownWorker, tag + " owned by rank " + std::to_string(w.rank)};
    for (std::size_t j = 0; j < i; ++j)
      if (e.overlaps(layout.tiles[j].first))
        return {LayoutViolation::Overlap,
                "tiles " + std::to_string(j) + " and " + std::to_string(i) + " overlap"};
    covered += e.elements();
  }
  if (covered != rows * cols)
    return {LayoutViolation::Gap, "tiles cover " + std::to_string(covered) + " of " +
                                      std::to_string(rows * cols) + " elements"};
  return {};
}

WorkerId tileOwner(const Layout& layout, std::uint64_t i, std::uint64_t j) {
  for (const auto& t : layout.tiles)
    if (t.first.contains(i, j)) return t.second;
  throw Error("tileOwner: index (" + std::to_string(i) + "," + std::to_string(j) +
              ") not covered by layout");
}

// ---------------------------------------------------------------- descriptor

void encodeDescriptor(const MatrixDescriptor& d, WireWriter& w) {
  w.u64(d.matrixId);
  w.u64(d.rows);
  w.u64(d.cols);
  w.u8(static_cast<std::uint8_t>(d.precision));
  w.u64(d.version);
  w.u32(static_cast<std::uint32_t>(d.layout.tiles.size()));
  for (const auto& t : d.layout.tiles) {
    w.u64(t.first.rowStart);
    w.u64(t.first.rowCount);
    w.u64(t.first.colStart);
    w.u64(t.first.colCount);
    w.u32(t.second.rank);
  }
}

MatrixDescriptor decodeDescriptor(WireReader& r) {
  MatrixDescriptor d;
  d.matrixId = r.u64();
  d.rows = r.u64();
  d.cols = r.u64();
  d.precision = precisionFromTag(r.u8());
  d.version = r.u64();
  const std::uint32_t n = r.u32();
  d.layout.tiles.reserve(n);
  for (std::uint32_t i = 0; i < n; ++i) {
    TileExtent e;
    e.rowStart = r.u64();
    e.rowCount = r.u64();
    e.colStart = r.u64();
    e.colCount = r.u64();
    d.layout.tiles.push_back({e, WorkerId{r.u32()}});
  }
  return d;
}

std::uint64_t descriptorHash(const MatrixDescriptor& d) {
  WireWriter w;
  encodeDescriptor(d, w);
  return fnv1a(w.view().data(), w.view().size());
}

std::uint64_t tableHash(const DescriptorTable& t) {
  std::uint64_t h = 0xcbf29ce484222325ull;
  for (const auto& kv : t) {
    const std::uint64_t dh = descriptorHash(kv.second);
    h = fnv1a(&dh, sizeof dh, h);
  }
  return h;
}

// ---------------------------------------------------------------- pieces

std::optional<Rect> intersectRect(const Rect& a, const Rect& b) {
  const Rect r{std::max(a.r0, b.r0), std::min(a.r1, b.r1), std::max(a.c0, b.c0),
               std::min(a.c1, b.c1)};
  if (r.empty()) return std::nullopt;
  return r;
}

RegionNeed& NeedPlanner::addNeed(const MatrixDescriptor& d, const Rect& rect,
                                 std::uint32_t consumer, bool allowReplica) {
  RegionNeed need;
  need.matrixId = d.matrixId;
  need.consumer = consumer;
  need.rect = rect;
  need.viaReplica = allowReplica && d.replicaFresh();
  if (!need.viaReplica) {
    for (const auto& t : d.layout.tiles) {
      if (auto piece = intersectRect(rect, Rect::ofExtent(t.first)))
        need.pieces.push_back(PieceRoute{nextPieceId_++, t.second.rank, consumer, d.matrixId, *piece});
    }
  }
  needs_.push_back(std::move(need));
  return needs_.back();
}

std::vector<ByteRun> tileByteRuns(const MatrixDescriptor& d, const TileExtent& e) {
  const std::uint64_t eb = bytesOf(d.precision);
  if (e.colStart == 0 && e.colCount == d.cols) return {{e.rowStart * d.cols * eb, e.rowCount * d.cols * eb}};
  std::vector<ByteRun> runs(e.rowCount);
  for (std::uint64_t i = 0; i < e.rowCount; ++i)
    runs[i] = {((e.rowStart + i) * d.cols + e.colStart) * eb, e.colCount * eb};
  return runs;
}

void packRect(const std::uint8_t* tileData, const TileExtent& extent, const Rect& rect,
              std::size_t elemBytes, std::uint8_t* out) {
  const std::size_t row = rect.cols() * elemBytes;
  for (std::uint64_t r = rect.r0; r < rect.r1; ++r)
    std::memcpy(out + (r - rect.r0) * row,
                tileData + ((r - extent.rowStart) * extent.colCount + (rect.c0 - extent.colStart)) * elemBytes,
                row);
}

void unpackRect(std::uint8_t* tileData, const TileExtent& extent, const Rect& rect,
                std::size_t elemBytes, const std::uint8_t* in) {
  const std::size_t row = rect.cols() * elemBytes;
  for (std::uint64_t r = rect.r0; r < rect.r1; ++r)
    std::memcpy(tileData + ((r - extent.rowStart) * extent.colCount + (rect.c0 - extent.colStart)) * elemBytes,
                in + (r - rect.r0) * row, row);
}

}  // namespace gridmath
