// SPDX-License-Identifier: Apache-2.0
#include "capture.hpp"
#include "device.hpp"

#include <algorithm>
#include <cstdlib>

#include "../cuda/convert.h"
#include "../cuda/debug_config.h"
#include "../cuda/gemm_f64.h"
#include "../cuda/gemm_tc.h"

namespace gridmath {

void cudaCheck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw Error(std::string(what) + ": " + cudaGetErrorString(e));
}

// ---------------------------------------------------------------- arena

DeviceArena::DeviceArena(int device) : device_(device) {}

DeviceArena::~DeviceArena() {
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(device_);
  for (auto& kv : free_)
    for (auto& b : kv.second)
      if (b.released) cudaEventDestroy(b.released);
  for (void* p : owned_) cudaFree(p);
  for (cudaEvent_t e : eventPool_) cudaEventDestroy(e);
  cudaSetDevice(prev);
}

std::uint64_t DeviceArena::sizeClass(std::uint64_t bytes) {
  std::uint64_t c = 256;
  while (c < bytes && c < (1ull << 20)) c <<= 1;
  if (c >= bytes) return c;
  // Above 1 MiB: classes at 1, 1.25, 1.5, 1.75 x 2^k.
  std::uint64_t p = 1ull << 20;
  while (p * 2 <= bytes) p <<= 1;
  for (std::uint64_t q = 1; q <= 4; ++q) {
    const std::uint64_t cand = p + (p / 4) * q;
    if (cand >= bytes) return q == 4 ? p * 2 : cand;
  }
  return p * 2;
}

void* DeviceArena::alloc(std::uint64_t bytes, cudaStream_t stream, std::uint64_t epoch, std::uint64_t minAge) {
  if (bytes == 0) throw Error("arena: zero-byte allocation");
  const std::uint64_t cls = sizeClass(bytes);
  std::lock_guard<std::mutex> lock(mu_);
  auto& list = free_[cls];
  // FIFO: the block released longest ago (its release event has most likely
  // completed); with minAge, skip blocks released too recently.
  auto pick = list.begin();
  while (pick != list.end() && minAge && pick->epoch + minAge > epoch) ++pick;
  if (pick != list.end()) {
    Block b = *pick;
    list.erase(pick);
    if (b.released) {
      cudaCheck(capture::wait(stream, b.released, 0), "arena: wait on release");
      eventPool_.push_back(b.released);
    }
    stats_.reuses += 1;
    stats_.held_bytes -= cls;
    live_[b.ptr] = cls;
    return b.ptr;
  }
  void* p = nullptr;
  const cudaError_t e = cudaMalloc(&p, cls);
  if (e != cudaSuccess) {
    cudaGetLastError();
    throw Error("arena: cudaMalloc of " + std::to_string(cls) + " bytes failed: " +
                cudaGetErrorString(e));
  }
  owned_.push_back(p);
  stats_.allocations_from_os += 1;
  stats_.reserved_bytes += cls;
  live_[p] = cls;
  return p;
}

void DeviceArena::free(void* p, cudaStream_t stream, std::uint64_t epoch) {
  if (!p) return;
  std::lock_guard<std::mutex> lock(mu_);
  auto it = live_.find(p);
  if (it == live_.end()) throw Error("arena: foreign or double free");
  const std::uint64_t cls = it->second;
  live_.erase(it);
  cudaEvent_t ev = nullptr;
  if (!eventPool_.empty()) {
    ev = eventPool_.back();
    eventPool_.pop_back();
  } else {
    cudaCheck(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "arena: event");
  }
  cudaCheck(capture::record(ev, stream), "arena: record release");
  free_[cls].push_back(Block{p, ev, epoch});
  stats_.frees += 1;
  stats_.held_bytes += cls;
}

gm_arena_stats DeviceArena::stats() const {
  std::lock_guard<std::mutex> lock(mu_);
  return stats_;
}

// ---------------------------------------------------------------- local GEMM

namespace {

constexpr std::uint64_t kAlign = 256;

std::uint64_t roundUp(std::uint64_t x, std::uint64_t a) { return (x + a - 1) / a * a; }

bool isF16Kind(int p) { return p == GM_HALF || p == GM_BF16; }

std::uint64_t elemBytes(int p) {
  switch (p) {
    case GM_HALF:
    case GM_BF16: return 2;
    case GM_SINGLE: return 4;
    case GM_DOUBLE: return 8;
  }
  throw Error("gemm: bad precision tag " + std::to_string(p));
}

// Pitch (elements) for a staged buffer: rows padded to 128 bytes.
std::uint64_t stagedLd(std::uint64_t cols, std::uint64_t eb) { return roundUp(cols * eb, 128) / eb; }

std::uint64_t tf32Chunk() {
  const int v = gmk::debug_config().tf32_chunk;
  return v > 0 ? static_cast<std::uint64_t>(v) : std::uint64_t{256};
}

bool tmaOk(const void* p, std::uint64_t ld, std::uint64_t eb) {
  return (reinterpret_cast<std::uintptr_t>(p) % 16) == 0 && (ld * eb) % 16 == 0 &&
         ld * eb < (1ull << 40);
}

struct OperandShape {
  std::uint64_t rows, cols;  // as stored
};

struct Plan {
  enum Path { F64, F16, TF32, TF32X3 } path;
  bool stageA = false, stageB = false;
  int stagePrec = GM_SINGLE;  // storage of staged operands
  std::uint64_t bytes = 0;
};

Plan makePlan(const gm_gemm_desc& d, const void* a, const void* b) {
  Plan pl{};
  const OperandShape sa{d.trans_a ? d.k : d.m, d.trans_a ? d.m : d.k};
  const OperandShape sb{d.trans_b ? d.n : d.k, d.trans_b ? d.k : d.n};
  const bool dbl = d.prec_a == GM_DOUBLE || d.prec_b == GM_DOUBLE || d.prec_c == GM_DOUBLE;
  if (dbl) {
    pl.path = Plan::F64;
    pl.stagePrec = GM_DOUBLE;
    auto ok = [](const void* p, int prec, std::uint64_t ld) {
      return prec == GM_DOUBLE && (reinterpret_cast<std::uintptr_t>(p) % 16) == 0 && ld % 2 == 0;
    };
    pl.stageA = !ok(a, d.prec_a, d.lda);
    pl.stageB = !ok(b, d.prec_b, d.ldb);
    if (pl.stageA) pl.bytes += roundUp(sa.rows * stagedLd(sa.cols, 8) * 8, kAlign);
    if (pl.stageB) pl.bytes += roundUp(sb.rows * stagedLd(sb.cols, 8) * 8, kAlign);
    return pl;
  }
  if (isF16Kind(d.prec_a) && d.prec_a == d.prec_b) {
    pl.path = Plan::F16;
    pl.stagePrec = d.prec_a;
    pl.stageA = !tmaOk(a, d.lda, 2);
    pl.stageB = !tmaOk(b, d.ldb, 2);
    if (pl.stageA) pl.bytes += roundUp(sa.rows * stagedLd(sa.cols, 2) * 2, kAlign);
    if (pl.stageB) pl.bytes += roundUp(sb.rows * stagedLd(sb.cols, 2) * 2, kAlign);
    return pl;
  }
  // tf32 paths run K-major only: MN-major operands are transposed while
  // they are staged (3xTF32 stages everything anyway for the hi/lo split).
  // Staged shapes: A as m x k, B as n x k.
  const std::uint64_t aBytes = roundUp(d.m * stagedLd(d.k, 4) * 4, kAlign);
  const std::uint64_t bBytes = roundUp(d.n * stagedLd(d.k, 4) * 4, kAlign);
  if (d.math == GM_MATH_TF32) {
    pl.path = Plan::TF32;
    pl.stageA = d.prec_a != GM_SINGLE || d.trans_a || !tmaOk(a, d.lda, 4);
    pl.stageB = d.prec_b != GM_SINGLE || !d.trans_b || !tmaOk(b, d.ldb, 4);
    if (pl.stageA) pl.bytes += aBytes;
    if (pl.stageB) pl.bytes += bBytes;
    return pl;
  }
  pl.path = Plan::TF32X3;  // hi + lo for both operands, always staged
  pl.stageA = pl.stageB = true;
  pl.bytes = 2 * aBytes + 2 * bBytes;
  (void)sa;
  (void)sb;
  return pl;
}

}  // namespace

std::uint64_t gemmWorkspaceBytes(const gm_gemm_desc& d) {
  // Worst case over alignment: assume staging is needed whenever it could be.
  const void* odd = reinterpret_cast<const void*>(static_cast<std::uintptr_t>(2));
  gm_gemm_desc dd = d;
  dd.lda = dd.lda | 1;
  dd.ldb = dd.ldb | 1;
  return makePlan(dd, odd, odd).bytes;
}

std::uint64_t gemmWorkspaceBytes(const gm_gemm_desc& d, const void* a, const void* b) {
  if (d.m == 0 || d.n == 0 || d.alpha == 0.0 || d.k == 0) return 0;
  return makePlan(d, a, b).bytes;
}

bool gemmConsumesPanelFlags(const gm_gemm_desc& d, const void* a, const void* b) {
  if (d.m == 0 || d.n == 0 || d.alpha == 0.0 || d.k == 0) return false;
  if (d.prec_c == GM_DOUBLE) return false;
  const Plan pl = makePlan(d, a, b);
  return pl.path == Plan::F16 && !pl.stageA && !pl.stageB;
}

void gemmLocal(const gm_gemm_desc& d, const void* a, const void* b, void* c, void* workspace,
               std::uint64_t workspaceBytes, cudaStream_t stream, const BiasReluEpilogue* ep,
               const gmk::PanelReady* ready) {
  if (d.m == 0 || d.n == 0) return;
  if (ready && ready->on() && !gemmConsumesPanelFlags(d, a, b))
    throw Error("gemm: panel flags need the 16-bit tcgen05 path reading both operands in place");
  if (ep && (d.alpha == 0.0 || d.k == 0 || d.prec_c != GM_BF16 || d.prec_a == GM_DOUBLE || d.prec_b == GM_DOUBLE))
    throw Error("gemm: fused bias/relu epilogue needs the tcgen05 path with bf16 C");
  for (int p : {d.prec_a, d.prec_b, d.prec_c}) (void)elemBytes(p);
  if (d.m > 0x7FFFFFFFull || d.n > 0x7FFFFFFFull || d.k > 0x7FFFFFFFull)
    throw Error("gemm: dimension exceeds 2^31");
  if (d.alpha == 0.0 || d.k == 0) {
    // alpha == 0: A and B are never read (reference kernels.cpp:232, :472).
    cudaCheck(gmk::scale_rect(c, d.prec_c, d.ldc, d.m, d.n, d.beta, stream), "gemm: scale C");
    return;
  }
  const Plan pl = makePlan(d, a, b);
  if (pl.bytes > workspaceBytes)
    throw Error("gemm: workspace too small (" + std::to_string(workspaceBytes) + " < " +
                std::to_string(pl.bytes) + ")");
  auto* ws = static_cast<std::uint8_t*>(workspace);
  const std::uint64_t aRows = d.trans_a ? d.k : d.m, aCols = d.trans_a ? d.m : d.k;
  const std::uint64_t bRows = d.trans_b ? d.n : d.k, bCols = d.trans_b ? d.k : d.n;
  const char* err = nullptr;

  if (pl.path == Plan::F64) {
    gmk::F64GemmArgs g;
    g.m = d.m;
    g.n = d.n;
    g.k = d.k;
    g.trans_a = d.trans_a != 0;
    g.trans_b = d.trans_b != 0;
    g.a = a;
    g.lda = d.lda;
    g.b = b;
    g.ldb = d.ldb;
    if (pl.stageA) {
      const std::uint64_t ld = stagedLd(aCols, 8);
      cudaCheck(gmk::convert_rect(a, d.prec_a, d.lda, ws, GM_DOUBLE, ld, aRows, aCols, stream), "gemm: stage A");
      g.a = ws;
      g.lda = ld;
      ws += roundUp(aRows * ld * 8, kAlign);
    }
    if (pl.stageB) {
      const std::uint64_t ld = stagedLd(bCols, 8);
      cudaCheck(gmk::convert_rect(b, d.prec_b, d.ldb, ws, GM_DOUBLE, ld, bRows, bCols, stream), "gemm: stage B");
      g.b = ws;
      g.ldb = ld;
      ws += roundUp(bRows * ld * 8, kAlign);
    }
    g.c = c;
    g.ldc = d.ldc;
    g.c_prec = d.prec_c;
    g.alpha = d.alpha;
    g.beta = d.beta;
    if (gmk::f64_gemm(g, stream, &err)) throw Error(std::string("gemm(f64): ") + err);
    return;
  }

  gmk::TcGemmArgs g;
  g.m = d.m;
  g.n = d.n;
  g.k = d.k;
  g.trans_a = d.trans_a != 0;
  g.trans_b = d.trans_b != 0;
  g.c = c;
  g.ldc = d.ldc;
  g.c_dtype = d.prec_c == GM_SINGLE ? 2 : (d.prec_c == GM_BF16 ? 1 : 0);
  g.alpha = d.alpha;
  g.beta = d.beta;
  g.cta_group = d.cta_group == 1 ? 1 : 2;
  g.max_ctas = d.max_ctas;
  g.a = {a, d.lda};
  g.b = {b, d.ldb};
  if (ready) g.ready = *ready;

  if (pl.path == Plan::F16) {
    const std::uint64_t eb = 2;
    if (pl.stageA) {
      const std::uint64_t ld = stagedLd(aCols, eb);
      cudaCheck(gmk::convert_rect(a, d.prec_a, d.lda, ws, pl.stagePrec, ld, aRows, aCols, stream), "gemm: stage A");
      g.a = {ws, ld};
      ws += roundUp(aRows * ld * eb, kAlign);
    }
    if (pl.stageB) {
      const std::uint64_t ld = stagedLd(bCols, eb);
      cudaCheck(gmk::convert_rect(b, d.prec_b, d.ldb, ws, pl.stagePrec, ld, bRows, bCols, stream), "gemm: stage B");
      g.b = {ws, ld};
      ws += roundUp(bRows * ld * eb, kAlign);
    }
    g.kind = d.prec_a == GM_BF16 ? gmk::TcKind::BF16 : gmk::TcKind::F16;
  } else {
    // Stage A as m x k and B as n x k (K-major), splitting into hi/lo for 3xTF32.
    const bool split = pl.path == Plan::TF32X3;
    const std::uint64_t lda = stagedLd(d.k, 4), ldb = stagedLd(d.k, 4);
    auto stage = [&](const void* src, int prec, std::uint64_t ld, bool kMajor, std::uint64_t rows,
                     std::uint64_t cols, std::uint64_t dld, float** hi, float** lo) {
      // rows x cols as stored; output (kMajor ? rows x cols : cols x rows).
      const std::uint64_t outRows = kMajor ? rows : cols;
      *hi = reinterpret_cast<float*>(ws);
      ws += roundUp(outRows * dld * 4, kAlign);
      *lo = nullptr;
      if (split) {
        *lo = reinterpret_cast<float*>(ws);
        ws += roundUp(outRows * dld * 4, kAlign);
      }
      if (kMajor && split)
        cudaCheck(gmk::split_tf32(src, prec, ld, *hi, *lo, dld, rows, cols, stream), "gemm: split");
      else if (kMajor)
        cudaCheck(gmk::convert_rect(src, prec, ld, *hi, GM_SINGLE, dld, rows, cols, stream), "gemm: stage");
      else
        cudaCheck(gmk::split_tf32_t(src, prec, ld, *hi, *lo, dld, rows, cols, split, stream), "gemm: stage^T");
    };
    float *ahi = nullptr, *alo = nullptr, *bhi = nullptr, *blo = nullptr;
    if (pl.stageA) {
      stage(a, d.prec_a, d.lda, !d.trans_a, aRows, aCols, lda, &ahi, &alo);
      g.a = {ahi, lda};
      g.a_lo = {alo, lda};
    }
    if (pl.stageB) {
      stage(b, d.prec_b, d.ldb, d.trans_b != 0, bRows, bCols, ldb, &bhi, &blo);
      g.b = {bhi, ldb};
      g.b_lo = {blo, ldb};
    }
    g.trans_a = false;
    g.trans_b = true;
    g.kind = split ? gmk::TcKind::TF32X3 : gmk::TcKind::TF32;
  }
  if (g.kind == gmk::TcKind::TF32X3 || g.kind == gmk::TcKind::TF32) {
    // The tensor cores' fp32 accumulation truncates, so its error grows
    // linearly with k. The kernel accumulates fixed global k-chunks of
    // kTf32Chunk in TMEM and folds each into an fp32 running sum with a
    // round-to-nearest FMA (TMEM-resident, inside the one launch); chunk
    // boundaries are fixed multiples, so the result stays layout/P
    // independent.
    const std::uint64_t L = tf32Chunk();
    if (d.k > L) g.fold_k = L;
  }
  if (pl.path == Plan::F16 && d.math == GM_MATH_FOLD && !ep) {
    // Same fixed global k-chunks as the Single path: layout/P independent.
    const std::uint64_t L = tf32Chunk();
    if (d.k > L) g.fold_k = L;
  }
  if (ep) {
    g.bias = ep->bias;
    g.act = ep->act;
    g.ld_act = ep->ldAct;
  }
  if (gmk::tc_gemm(g, stream, &err)) throw Error(std::string("gemm(tcgen05): ") + err);
}

}  // namespace gridmath
