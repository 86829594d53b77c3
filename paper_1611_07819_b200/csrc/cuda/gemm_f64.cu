// SPDX-License-Identifier: Apache-2.0
// Double-compute local block GEMM on the fp64 tensor path (DMMA,
// mma.sync.m8n8k4.f64 -- tcgen05 has no f64 kind).
//
// Device replacement of runGemm<double> (reference proj/src/kernels.cpp:445-558
// with computePrecision == Double, :136-140). Operands arrive as fp64
// (the caller upcasts Half/Single/BF16 exactly, like convertToT, :27-41);
// C is written in its storage precision (double -> float -> half for Half,
// as storeScalar does, precision.hpp:129-149). Each output element is one
// fixed ascending-k FMA chain, independent of tiling and distribution.
//
// Tiling: 64x128 CTA tile, BK=16, 4 warps (2 x 2) of 32x64, two CTAs per SM,
// 3-stage cp.async ring with zero-filled out-of-range chunks; fragments for
// the next k-step are loaded while the current one's DMMAs issue.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "convert.h"
#include "gemm_f64.h"

namespace gmk {

namespace {

constexpr int kBK = 16, kStages = 3;

template <int BM, int BN, int WGM, int WGN>
struct F64Cfg {
  static constexpr int kThreads = WGM * WGN * 32;
  static constexpr int kWM = BM / WGM, kWN = BN / WGN;  // warp tile
  static constexpr int kMI = kWM / 8, kNJ = kWN / 8;     // m8n8 fragments per warp
  // A is [BM][BK+4] (k-contiguous) or [BK][BM+4]; B is [BN][BK+4] or [BK][BN+4].
  static constexpr int kASize = BM * (kBK + 4) > kBK * (BM + 4) ? BM * (kBK + 4) : kBK * (BM + 4);
  static constexpr int kBSize = BN * (kBK + 4) > kBK * (BN + 4) ? BN * (kBK + 4) : kBK * (BN + 4);
  static constexpr int kStage = kASize + kBSize;  // doubles
  static constexpr size_t kSmem = static_cast<size_t>(kStages) * kStage * sizeof(double);
};

struct F64Params {
  const double* a;
  const double* b;
  void* c;
  uint64_t lda, ldb, ldc;
  uint32_t m, n, k;
  int c_prec;
  double alpha, beta;
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(smem))),
               "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N));
}

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
      : "+d"(d[0]), "+d"(d[1])
      : "d"(a), "d"(b));
}

// Loads a (ROWS x 16) slab of a row-major operand whose contiguous axis is k
// ("k-contiguous", dst [mn][BK+4]) or a (16 x ROWS) slab whose contiguous
// axis is mn ("mn-contiguous", dst [k][ROWS+4]). Out-of-range chunks are
// zero-filled.
template <bool kKContig, int ROWS, int THREADS>
__device__ __forceinline__ void load_tile(double* dst, const double* src, uint64_t ld, uint32_t mn0,
                                          uint32_t mn_lim, uint32_t k0, uint32_t k_lim) {
  if constexpr (kKContig) {
    for (int i = threadIdx.x; i < ROWS * (kBK / 2); i += THREADS) {
      const int r = i / (kBK / 2), ch = i % (kBK / 2);
      const uint32_t gr = mn0 + r, gk = k0 + ch * 2;
      uint32_t bytes = 0;
      const double* g = src;
      if (gr < mn_lim && gk < k_lim) {
        bytes = (gk + 1 < k_lim) ? 16 : 8;
        g = src + static_cast<uint64_t>(gr) * ld + gk;
      }
      cp_async16(dst + r * (kBK + 4) + ch * 2, g, bytes);
    }
  } else {
    for (int i = threadIdx.x; i < kBK * (ROWS / 2); i += THREADS) {
      const int r = i / (ROWS / 2), ch = i % (ROWS / 2);
      const uint32_t gk = k0 + r, gm = mn0 + ch * 2;
      uint32_t bytes = 0;
      const double* g = src;
      if (gk < k_lim && gm < mn_lim) {
        bytes = (gm + 1 < mn_lim) ? 16 : 8;
        g = src + static_cast<uint64_t>(gk) * ld + gm;
      }
      cp_async16(dst + r * (ROWS + 4) + ch * 2, g, bytes);
    }
  }
}

__device__ __forceinline__ void store_c(const F64Params& p, uint32_t r, uint32_t c, double v) {
  if (r >= p.m || c >= p.n) return;
  const uint64_t idx = static_cast<uint64_t>(r) * p.ldc + c;
  double out = p.alpha * v;
  switch (p.c_prec) {
    case 2: {
      double* cp = reinterpret_cast<double*>(p.c);
      if (p.beta != 0.0) out += p.beta * cp[idx];
      cp[idx] = out;
      break;
    }
    case 1: {
      float* cp = reinterpret_cast<float*>(p.c);
      if (p.beta != 0.0) out += p.beta * static_cast<double>(cp[idx]);
      cp[idx] = __double2float_rn(out);
      break;
    }
    case 0: {
      __half* cp = reinterpret_cast<__half*>(p.c);
      if (p.beta != 0.0) out += p.beta * static_cast<double>(__half2float(cp[idx]));
      cp[idx] = __float2half_rn(__double2float_rn(out));
      break;
    }
    default: {
      __nv_bfloat16* cp = reinterpret_cast<__nv_bfloat16*>(p.c);
      if (p.beta != 0.0) out += p.beta * static_cast<double>(__bfloat162float(cp[idx]));
      cp[idx] = __float2bfloat16_rn(__double2float_rn(out));
      break;
    }
  }
}

template <int BM, int BN, int WGM, int WGN, int MINB, bool kTA, bool kTB>
__global__ void __launch_bounds__(WGM * WGN * 32, MINB) f64_gemm_kernel(const F64Params p) {
  using Cfg = F64Cfg<BM, BN, WGM, WGN>;
  constexpr int MI = Cfg::kMI, NJ = Cfg::kNJ;
  extern __shared__ __align__(16) double sm[];

  const uint32_t m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int wm = warp / WGN, wn = warp % WGN;
  const int gid = lane / 4, tig = lane % 4;

  double acc[MI][NJ][2];
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const uint32_t nk = (p.k + kBK - 1) / kBK;
  auto issue = [&](uint32_t kb, int slot) {
    double* st = sm + slot * Cfg::kStage;
    // A: op(A) is m x k; stored m x k (k-contiguous) or k x m (transA).
    load_tile<!kTA, BM, Cfg::kThreads>(st, p.a, p.lda, m0, p.m, kb * kBK, p.k);
    // B: op(B) is k x n; stored k x n (n-contiguous) or n x k (transB).
    load_tile<kTB, BN, Cfg::kThreads>(st + Cfg::kASize, p.b, p.ldb, n0, p.n, kb * kBK, p.k);
  };

#pragma unroll
  for (int s = 0; s < kStages - 1; ++s) {
    if (static_cast<uint32_t>(s) < nk) issue(s, s);
    cp_async_commit();
  }

  double af[2][MI], bf[2][NJ];
  auto frags = [&](const double* ta, const double* tb, int kk, int buf) {
#pragma unroll
    for (int i = 0; i < MI; ++i) {
      const int r = wm * Cfg::kWM + i * 8 + gid;
      af[buf][i] = kTA ? ta[(kk + tig) * (BM + 4) + r] : ta[r * (kBK + 4) + kk + tig];
    }
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      const int c = wn * Cfg::kWN + j * 8 + gid;
      bf[buf][j] = kTB ? tb[c * (kBK + 4) + kk + tig] : tb[(kk + tig) * (BN + 4) + c];
    }
  };

  for (uint32_t kb = 0; kb < nk; ++kb) {
    cp_async_wait<kStages - 2>();
    __syncthreads();
    const uint32_t nxt = kb + kStages - 1;
    if (nxt < nk) issue(nxt, nxt % kStages);
    cp_async_commit();

    const double* ta = sm + (kb % kStages) * Cfg::kStage;
    const double* tb = ta + Cfg::kASize;
    frags(ta, tb, 0, 0);
#pragma unroll
    for (int kk = 0; kk < kBK; kk += 4) {
      const int cur = (kk / 4) & 1;
      if (kk + 4 < kBK) frags(ta, tb, kk + 4, cur ^ 1);  // next fragments in flight under the MMAs
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NJ; ++j) dmma(acc[i][j], af[cur][i], bf[cur][j]);
    }
  }
  cp_async_wait<0>();

#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      const uint32_t r = m0 + wm * Cfg::kWM + i * 8 + gid;
      const uint32_t c = n0 + wn * Cfg::kWN + j * 8 + tig * 2;
      store_c(p, r, c, acc[i][j][0]);
      store_c(p, r, c + 1, acc[i][j][1]);
    }
}

template <int BM, int BN, int WGM, int WGN, int MINB>
void launch_f64(const F64Params& p, bool ta, bool tb, cudaStream_t stream) {
  using Cfg = F64Cfg<BM, BN, WGM, WGN>;
  dim3 grid((p.n + BN - 1) / BN, (p.m + BM - 1) / BM);
  auto go = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(Cfg::kSmem));
    kern<<<grid, Cfg::kThreads, Cfg::kSmem, stream>>>(p);
  };
  if (!ta && !tb) go(f64_gemm_kernel<BM, BN, WGM, WGN, MINB, false, false>);
  else if (!ta && tb) go(f64_gemm_kernel<BM, BN, WGM, WGN, MINB, false, true>);
  else if (ta && !tb) go(f64_gemm_kernel<BM, BN, WGM, WGN, MINB, true, false>);
  else go(f64_gemm_kernel<BM, BN, WGM, WGN, MINB, true, true>);
}

}  // namespace

int f64_gemm(const F64GemmArgs& g, cudaStream_t stream, const char** err) {
  F64Params p{};
  p.a = static_cast<const double*>(g.a);
  p.b = static_cast<const double*>(g.b);
  p.c = g.c;
  p.lda = g.lda;
  p.ldb = g.ldb;
  p.ldc = g.ldc;
  p.m = static_cast<uint32_t>(g.m);
  p.n = static_cast<uint32_t>(g.n);
  p.k = static_cast<uint32_t>(g.k);
  p.c_prec = g.c_prec;
  p.alpha = g.alpha;
  p.beta = g.beta;
  // 64x128 CTA tiles, 4 warps of 32x64, two CTAs per SM (their barriers
  // interleave); GM_F64_TILE=128 selects the 128x128 / 8-warp variant.
  static const int variant = [] {
    const char* v = std::getenv("GM_F64_TILE");
    return v ? std::atoi(v) : 64;
  }();
  if (variant == 128) launch_f64<128, 128, 2, 4, 1>(p, g.trans_a, g.trans_b, stream);
  else launch_f64<64, 128, 2, 2, 2>(p, g.trans_a, g.trans_b, stream);
  count_launch();
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    *err = cudaGetErrorString(e);
    return 1;
  }
  return 0;
}

}  // namespace gmk
