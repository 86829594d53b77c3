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

// Paired-fragment variant (64x128 CTA, 4 warps of 32x64, two CTAs per SM):
// every fragment load is one 16-byte LDS serving two MMAs. Along an
// operand's contiguous axis two neighbouring elements go to the same lane:
//   * k-contiguous operands (A, or B^T): lane tig takes k = 2*tig + q of the
//     8-wide k pair p, i.e. MMA k-step 2p + q uses k = 8p + 2*tig + q;
//   * mn-contiguous operands (A^T, or B): m/n tiles come in pairs whose
//     MMA-local row/column g maps to 2g (first) and 2g + 1 (second) of the
//     16-wide pair, which the epilogue undoes.
// Each output element is still one fixed-order FMA chain over k (the k
// order is a fixed global permutation within every 8-wide k group), so the
// result is independent of tiling and distribution. Shared-memory row
// pitches of 24 doubles (k-contiguous, 192 B = 64 mod 128) and BM/BN + 2
// doubles (mn-contiguous: lanes read rows 2*tig + q apart, and 2 x pitch =
// 32 mod 128 B) keep the 16-byte loads conflict-free.
namespace paired {
constexpr int BM = 64, BN = 128, kThreads = 128, kPK = 24;
constexpr int kASize = BM * kPK > kBK * (BM + 2) ? BM * kPK : kBK * (BM + 2);
constexpr int kBSize = BN * kPK > kBK * (BN + 2) ? BN * kPK : kBK * (BN + 2);
constexpr int kStage = kASize + kBSize;
constexpr size_t kSmem = static_cast<size_t>(kStages) * kStage * sizeof(double);

template <bool kKContig, int ROWS>
__device__ __forceinline__ void load(double* dst, const double* src, uint64_t ld, uint32_t mn0, uint32_t mn_lim,
                                     uint32_t k0, uint32_t k_lim) {
  if constexpr (kKContig) {
    for (int i = threadIdx.x; i < ROWS * (kBK / 2); i += kThreads) {
      const int r = i / (kBK / 2), ch = i % (kBK / 2);
      const uint32_t gr = mn0 + r, gk = k0 + ch * 2;
      uint32_t bytes = 0;
      const double* g = src;
      if (gr < mn_lim && gk < k_lim) {
        bytes = (gk + 1 < k_lim) ? 16 : 8;
        g = src + static_cast<uint64_t>(gr) * ld + gk;
      }
      cp_async16(dst + r * kPK + ch * 2, g, bytes);
    }
  } else {
    for (int i = threadIdx.x; i < kBK * (ROWS / 2); i += kThreads) {
      const int r = i / (ROWS / 2), ch = i % (ROWS / 2);
      const uint32_t gk = k0 + r, gm = mn0 + ch * 2;
      uint32_t bytes = 0;
      const double* g = src;
      if (gk < k_lim && gm < mn_lim) {
        bytes = (gm + 1 < mn_lim) ? 16 : 8;
        g = src + static_cast<uint64_t>(gk) * ld + gm;
      }
      cp_async16(dst + r * (ROWS + 2) + ch * 2, g, bytes);
    }
  }
}

__device__ __forceinline__ double2 lds2(const double* p) { return *reinterpret_cast<const double2*>(p); }

template <bool kTA, bool kTB>
__global__ void __launch_bounds__(kThreads, 2) kernel(const F64Params p) {
  extern __shared__ __align__(16) double sm[];
  const uint32_t m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int wm = warp / 2, wn = warp % 2;  // warp tile 32 x 64
  const int gid = lane / 4, tig = lane % 4;
  constexpr int MI = 4, NJ = 8;

  double acc[MI][NJ][2];
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const uint32_t nk = (p.k + kBK - 1) / kBK;
  auto issue = [&](uint32_t kb, int slot) {
    double* st = sm + slot * kStage;
    load<!kTA, BM>(st, p.a, p.lda, m0, p.m, kb * kBK, p.k);
    load<kTB, BN>(st + kASize, p.b, p.ldb, n0, p.n, kb * kBK, p.k);
  };
#pragma unroll
  for (int s = 0; s < kStages - 1; ++s) {
    if (static_cast<uint32_t>(s) < nk) issue(s, s);
    cp_async_commit();
  }

  // Fragment loaders for MMA k-step ks (0..3) of the current block.
  auto fragA = [&](const double* ta, int ks, double (&a)[MI]) {
    const int pp = ks / 2, q = ks % 2;
    if constexpr (!kTA) {  // [m][kPK], k-paired: one LDS per m-tile per k pair
#pragma unroll
      for (int i = 0; i < MI; ++i) {
        const double2 v = lds2(ta + (wm * 32 + i * 8 + gid) * kPK + pp * 8 + 2 * tig);
        a[i] = q ? v.y : v.x;
      }
    } else {  // [k][BM+2], m-paired tiles (2ii, 2ii+1)
#pragma unroll
      for (int ii = 0; ii < MI / 2; ++ii) {
        const double2 v = lds2(ta + (pp * 8 + 2 * tig + q) * (BM + 2) + wm * 32 + ii * 16 + 2 * gid);
        a[2 * ii] = v.x;
        a[2 * ii + 1] = v.y;
      }
    }
  };
  auto fragB = [&](const double* tb, int ks, double (&b)[NJ]) {
    const int pp = ks / 2, q = ks % 2;
    if constexpr (kTB) {  // [n][kPK], k-paired
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        const double2 v = lds2(tb + (wn * 64 + j * 8 + gid) * kPK + pp * 8 + 2 * tig);
        b[j] = q ? v.y : v.x;
      }
    } else {  // [k][BN+2], n-paired tiles (2jj, 2jj+1)
#pragma unroll
      for (int jj = 0; jj < NJ / 2; ++jj) {
        const double2 v = lds2(tb + (pp * 8 + 2 * tig + q) * (BN + 2) + wn * 64 + jj * 16 + 2 * gid);
        b[2 * jj] = v.x;
        b[2 * jj + 1] = v.y;
      }
    }
  };

  // Interior CTAs (the whole 64 x 128 tile inside C) refill full k-blocks
  // through precomputed per-thread source pointers: thread t copies A rows
  // t/8 + 16j (j < 4) at k chunk t%8 and, NN, B k-rows t/64 + 2j (j < 8) at
  // n chunk t%64 -- two base pointers and two strides instead of per-copy
  // index math and bounds checks. Edge CTAs and the last partial k-block use
  // the general loader.
  const bool fast = !kTA && !kTB && m0 + BM <= p.m && n0 + BN <= p.n;
  const double* fa = p.a + static_cast<uint64_t>(m0 + threadIdx.x / 8) * p.lda + 2 * (threadIdx.x % 8);
  const double* fb = p.b + static_cast<uint64_t>(threadIdx.x / 64) * p.ldb + n0 + 2 * (threadIdx.x % 64);
  const uint64_t sa16 = 16 * p.lda, sb2 = 2 * p.ldb;
  const uint32_t da = (threadIdx.x / 8) * kPK + 2 * (threadIdx.x % 8);
  const uint32_t db = (threadIdx.x / 64) * (BN + 2) + 2 * (threadIdx.x % 64);
  auto refill = [&](uint32_t kb, int slot) {
    if (fast && (kb + 1) * kBK <= p.k) {
      double* st = sm + slot * kStage;
      const double* ga = fa + kb * kBK;
#pragma unroll
      for (int j = 0; j < 4; ++j) cp_async16(st + da + j * 16 * kPK, ga + j * sa16, 16);
      const double* gb = fb + static_cast<uint64_t>(kb * kBK) * p.ldb;
#pragma unroll
      for (int j = 0; j < 8; ++j) cp_async16(st + kASize + db + j * 2 * (BN + 2), gb + j * sb2, 16);
    } else {
      issue(kb, slot);
    }
  };

  for (uint32_t kb = 0; kb < nk; ++kb) {
    cp_async_wait<kStages - 2>();
    __syncthreads();
    const uint32_t nxt = kb + kStages - 1;
    const double* ta = sm + (kb % kStages) * kStage;
    const double* tb = ta + kASize;
    double a[2][MI], b[2][NJ];
    fragA(ta, 0, a[0]);
    fragB(tb, 0, b[0]);
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      const int cur = ks & 1;
      if (ks + 1 < 4) {
        fragA(ta, ks + 1, a[cur ^ 1]);
        fragB(tb, ks + 1, b[cur ^ 1]);
      }
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NJ; ++j) dmma(acc[i][j], a[cur][i], b[cur][j]);
      if (ks == 0) {
        // Refill the slot every thread finished reading before the barrier
        // above, once this k-block's first DMMAs are queued.
        if (nxt < nk) refill(nxt, nxt % kStages);
        cp_async_commit();
      }
    }
  }
  cp_async_wait<0>();

#pragma unroll
  for (int i = 0; i < MI; ++i) {
    const uint32_t r = m0 + wm * 32 + (kTA ? (i / 2) * 16 + 2 * gid + (i % 2) : i * 8 + gid);
#pragma unroll
    for (int j = 0; j < NJ; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int cl = 2 * tig + e;  // MMA-local column
        const uint32_t c = n0 + wn * 64 + (kTB ? j * 8 + cl : (j / 2) * 16 + 2 * cl + (j % 2));
        store_c(p, r, c, acc[i][j][e]);
      }
  }
}

void launch(const F64Params& p, bool ta, bool tb, cudaStream_t stream) {
  dim3 grid((p.n + BN - 1) / BN, (p.m + BM - 1) / BM);
  auto go = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kSmem));
    kern<<<grid, kThreads, kSmem, stream>>>(p);
  };
  if (!ta && !tb) go(kernel<false, false>);
  else if (!ta && tb) go(kernel<false, true>);
  else if (ta && !tb) go(kernel<true, false>);
  else go(kernel<true, true>);
}
}  // namespace paired

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
  paired::launch(p, g.trans_a, g.trans_b, stream);
  count_launch();
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    *err = cudaGetErrorString(e);
    return 1;
  }
  return 0;
}

}  // namespace gmk
