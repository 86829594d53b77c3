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
// Tiling: 128x128 CTA tile, BK=16, 8 warps (2 x 4) of 64x32, 3-stage
// cp.async ring with zero-filled out-of-range chunks.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "convert.h"
#include "gemm_f64.h"

namespace gmk {

namespace {

constexpr int kBM = 128, kBN = 128, kBK = 16, kStages = 3, kThreads = 256;
constexpr int kPadK = kBK + 4;    // [mn][k] tiles: 20 doubles per row
constexpr int kPadMN = kBM + 4;   // [k][mn] tiles: 132 doubles per row
constexpr int kTileDoubles = kBM * kPadK > kBK * kPadMN ? kBM * kPadK : kBK * kPadMN;

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

// Loads a (rows x 16) slab of a row-major operand whose contiguous axis is k
// ("k-contiguous", dst [mn][k]) or a (16 x cols) slab whose contiguous axis is
// mn ("mn-contiguous", dst [k][mn]). Out-of-range chunks are zero-filled.
template <bool kKContig>
__device__ __forceinline__ void load_tile(double* dst, const double* src, uint64_t ld,
                                          uint32_t mn0, uint32_t mn_lim, uint32_t k0,
                                          uint32_t k_lim) {
  if constexpr (kKContig) {
    // 128 rows x 8 chunks of 2 doubles.
    for (int i = threadIdx.x; i < kBM * (kBK / 2); i += kThreads) {
      const int r = i / (kBK / 2), ch = i % (kBK / 2);
      const uint32_t gr = mn0 + r, gk = k0 + ch * 2;
      uint32_t bytes = 0;
      const double* g = src;
      if (gr < mn_lim && gk < k_lim) {
        bytes = (gk + 1 < k_lim) ? 16 : 8;
        g = src + static_cast<uint64_t>(gr) * ld + gk;
      }
      cp_async16(dst + r * kPadK + ch * 2, g, bytes);
    }
  } else {
    // 16 rows (k) x 64 chunks.
    for (int i = threadIdx.x; i < kBK * (kBM / 2); i += kThreads) {
      const int r = i / (kBM / 2), ch = i % (kBM / 2);
      const uint32_t gk = k0 + r, gm = mn0 + ch * 2;
      uint32_t bytes = 0;
      const double* g = src;
      if (gk < k_lim && gm < mn_lim) {
        bytes = (gm + 1 < mn_lim) ? 16 : 8;
        g = src + static_cast<uint64_t>(gk) * ld + gm;
      }
      cp_async16(dst + r * kPadMN + ch * 2, g, bytes);
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

template <bool kTA, bool kTB>
__global__ void __launch_bounds__(kThreads, 1) f64_gemm_kernel(const F64Params p) {
  extern __shared__ __align__(16) double sm[];
  double* sa = sm;                              // [kStages][kTileDoubles]
  double* sb = sm + kStages * kTileDoubles;     // [kStages][kTileDoubles]

  const uint32_t m0 = blockIdx.y * kBM, n0 = blockIdx.x * kBN;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int wm = warp / 4, wn = warp % 4;  // 2 x 4 warps, 64 x 32 each
  const int gid = lane / 4, tig = lane % 4;

  double acc[8][4][2];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const uint32_t nk = (p.k + kBK - 1) / kBK;
  auto issue = [&](uint32_t kb, int slot) {
    // A: op(A) is m x k; stored m x k (k-contiguous) or k x m (transA).
    load_tile<!kTA>(sa + slot * kTileDoubles, p.a, p.lda, m0, p.m, kb * kBK, p.k);
    // B: op(B) is k x n; stored k x n (n-contiguous) or n x k (transB).
    load_tile<kTB>(sb + slot * kTileDoubles, p.b, p.ldb, n0, p.n, kb * kBK, p.k);
  };

#pragma unroll
  for (int s = 0; s < kStages - 1; ++s) {
    if (static_cast<uint32_t>(s) < nk) issue(s, s);
    cp_async_commit();
  }

  for (uint32_t kb = 0; kb < nk; ++kb) {
    cp_async_wait<kStages - 2>();
    __syncthreads();
    const uint32_t nxt = kb + kStages - 1;
    if (nxt < nk) issue(nxt, nxt % kStages);
    cp_async_commit();

    const double* ta = sa + (kb % kStages) * kTileDoubles;
    const double* tb = sb + (kb % kStages) * kTileDoubles;
#pragma unroll
    for (int kk = 0; kk < kBK; kk += 4) {
      double af[8], bf[4];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int r = wm * 64 + i * 8 + gid;
        af[i] = kTA ? ta[(kk + tig) * kPadMN + r] : ta[r * kPadK + kk + tig];
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int c = wn * 32 + j * 8 + gid;
        bf[j] = kTB ? tb[c * kPadK + kk + tig] : tb[(kk + tig) * kPadMN + c];
      }
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();

#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t r = m0 + wm * 64 + i * 8 + gid;
      const uint32_t c = n0 + wn * 32 + j * 8 + tig * 2;
      store_c(p, r, c, acc[i][j][0]);
      store_c(p, r, c + 1, acc[i][j][1]);
    }
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
  const size_t smem = 2ull * kStages * kTileDoubles * sizeof(double);
  dim3 grid((p.n + kBN - 1) / kBN, (p.m + kBM - 1) / kBM);
  auto pick = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    kern<<<grid, kThreads, smem, stream>>>(p);
    count_launch();
  };
  if (!g.trans_a && !g.trans_b) pick(f64_gemm_kernel<false, false>);
  else if (!g.trans_a && g.trans_b) pick(f64_gemm_kernel<false, true>);
  else if (g.trans_a && !g.trans_b) pick(f64_gemm_kernel<true, false>);
  else pick(f64_gemm_kernel<true, true>);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    *err = cudaGetErrorString(e);
    return 1;
  }
  return 0;
}

}  // namespace gmk
