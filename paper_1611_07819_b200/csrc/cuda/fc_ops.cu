// SPDX-License-Identifier: Apache-2.0
// FC-layer neighbours of the GEMM on device:
//   elementwise unary / binary ..... reference runElementwise, proj/src/kernels.cpp:741-815
//   setConst ....................... execSetConst, kernels.cpp:435-443
//   deterministic row / col sums ... runRowColSumDet, kernels.cpp:572-617
// All HBM-bound. Per element the arithmetic is the reference's, in its
// compute type (double iff any operand is Double, kernels.cpp:136-140), with
// separately rounded multiplies and adds, so results are bit-for-bit the
// reference's except for subnormal Half inputs.
#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

#include "convert.h"
#include "fc_ops.h"
#include "gemm_tc.h"
#include "prec.cuh"
#include "ptx.cuh"

namespace gmk {

namespace {

template <typename T>
__device__ __forceinline__ T ew_eval(int kind, T xv, const EwView& y, uint64_t yidx, T alpha) {
  switch (kind) {
    case kEwRelu: return xv > T(0) ? xv : T(0);
    case kEwMulScalar: return mul_rn(alpha, xv);
    case kEwAdd: return add_rn(xv, load_as<T>(y.ptr, y.prec, yidx));
    case kEwSub: return sub_rn(xv, load_as<T>(y.ptr, y.prec, yidx));
    case kEwAxpy: return add_rn(mul_rn(alpha, xv), load_as<T>(y.ptr, y.prec, yidx));
    case kEwReluGrad: return xv > T(0) ? load_as<T>(y.ptr, y.prec, yidx) : T(0);
    case kEwBiasAdd: return add_rn(xv, load_as<T>(y.ptr, y.prec, yidx));
    default: return xv;  // kEwCopy
  }
}

// Generic path (operands of different storage precisions): blockIdx.y
// strides rows, threads stride columns, so every warp touches one contiguous
// row segment of each operand; the kind and precision switches are uniform.
// Line-sum output: acc[idx] = acc[idx] + alpha * sum, or 0 + alpha * sum
// when the caller zeroed the outputs by definition (kLineSumsZeroAcc in
// acc_prec: the replay peephole that folds setConst(0) into the sums).
template <typename T>
__device__ __forceinline__ void line_sum_out(void* acc, int acc_prec, uint64_t idx, T alpha, T sum) {
  const int p = acc_prec & 0xFF;
  const T cur = (acc_prec & kLineSumsZeroAcc) ? T(0) : load_as<T>(acc, p, idx);
  store_as(acc, p, idx, add_rn(cur, mul_rn(alpha, sum)));
}

template <typename T>
__global__ void ew_kernel(EwView x, EwView y, int ybc, void* __restrict__ d, uint64_t dld, int dprec,
                          uint64_t rows, uint64_t cols, int kind, T alpha) {
  for (uint64_t r = blockIdx.y; r < rows; r += gridDim.y) {
    const uint64_t xo = r * x.ld, yo = ybc ? 0 : r * y.ld, dof = r * dld;
    for (uint64_t c = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; c < cols;
         c += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
      const T xv = load_as<T>(x.ptr, x.prec, xo + c);
      store_as(d, dprec, dof + c, ew_eval<T>(kind, xv, y, yo + c, alpha));
    }
  }
}

// Storage element of precision tag P and its conversions to / from the
// compute type (same rules as load_elem* / store_elem*).
template <int P> struct Stor { using type = uint16_t; };
template <> struct Stor<1> { using type = float; };
template <> struct Stor<2> { using type = double; };

template <int P, typename T>
__device__ __forceinline__ T widen(typename Stor<P>::type v) {
  if constexpr (P == 0) return static_cast<T>(half_bits_to_f32(v));
  else if constexpr (P == 3) return static_cast<T>(__uint_as_float(static_cast<uint32_t>(v) << 16));
  else return static_cast<T>(v);
}
template <int P, typename T>
__device__ __forceinline__ typename Stor<P>::type narrow(T v) {
  if constexpr (P == 2) return static_cast<double>(v);
  else {
    const float f = static_cast<float>(v);  // T is float unless P == 2
    if constexpr (P == 0) return f32_to_half_bits(f);
    else if constexpr (P == 3) return f32_to_bf16_bits(f);
    else return f;
  }
}

// Same-precision fast path: one 16-byte vector per thread per step (8 half /
// bf16, 4 single or 2 double elements), every operand 16-byte aligned with
// a 16-byte-multiple pitch (checked at launch). HBM-bound.
template <typename T, int P>
__global__ void ew_vec_kernel(EwView x, EwView y, int ybc, void* __restrict__ d, uint64_t dld, uint64_t rows,
                              uint64_t cols, int kind, T alpha) {
  using S = typename Stor<P>::type;
  constexpr int N = 16 / sizeof(S);
  union V {
    uint4 u;
    S e[N];
  };
  const uint64_t nvec = (cols + N - 1) / N;
  const bool useY = kind >= kEwAdd && kind != kEwCopy;
  for (uint64_t r = blockIdx.y; r < rows; r += gridDim.y) {
    const S* xr = static_cast<const S*>(x.ptr) + r * x.ld;
    const S* yr = static_cast<const S*>(y.ptr) + (ybc ? 0 : r * y.ld);
    S* dr = static_cast<S*>(d) + r * dld;
    for (uint64_t v = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; v < nvec;
         v += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
      const uint64_t c0 = v * N;
      if (c0 + N <= cols) {
        V xv, yv, out;
        xv.u = __ldg(reinterpret_cast<const uint4*>(xr + c0));
        if (useY) yv.u = __ldg(reinterpret_cast<const uint4*>(yr + c0));
#pragma unroll
        for (int k = 0; k < N; ++k) {
          const T a = widen<P, T>(xv.e[k]);
          T o;
          switch (kind) {
            case kEwRelu: o = a > T(0) ? a : T(0); break;
            case kEwMulScalar: o = mul_rn(alpha, a); break;
            case kEwAdd:
            case kEwBiasAdd: o = add_rn(a, widen<P, T>(yv.e[k])); break;
            case kEwSub: o = sub_rn(a, widen<P, T>(yv.e[k])); break;
            case kEwAxpy: o = add_rn(mul_rn(alpha, a), widen<P, T>(yv.e[k])); break;
            case kEwReluGrad: o = a > T(0) ? widen<P, T>(yv.e[k]) : T(0); break;
            default: o = a; break;
          }
          out.e[k] = narrow<P, T>(o);
        }
        *reinterpret_cast<uint4*>(dr + c0) = out.u;
      } else {
        for (uint64_t c = c0; c < cols; ++c) {
          const T a = widen<P, T>(xr[c]);
          T o;
          switch (kind) {
            case kEwRelu: o = a > T(0) ? a : T(0); break;
            case kEwMulScalar: o = mul_rn(alpha, a); break;
            case kEwAdd:
            case kEwBiasAdd: o = add_rn(a, widen<P, T>(yr[c])); break;
            case kEwSub: o = sub_rn(a, widen<P, T>(yr[c])); break;
            case kEwAxpy: o = add_rn(mul_rn(alpha, a), widen<P, T>(yr[c])); break;
            case kEwReluGrad: o = a > T(0) ? widen<P, T>(yr[c]) : T(0); break;
            default: o = a; break;
          }
          dr[c] = narrow<P, T>(o);
        }
      }
    }
  }
}

__global__ void set_const_kernel(void* __restrict__ d, uint64_t ld, int prec, uint64_t rows, uint64_t cols,
                                 double v) {
  for (uint64_t r = blockIdx.y; r < rows; r += gridDim.y)
    for (uint64_t c = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; c < cols;
         c += static_cast<uint64_t>(gridDim.x) * blockDim.x)
      store_elem(d, prec, r * ld + c, v);
}

// Line sums with the reference's sequential chain: 32 outputs per CTA. The
// whole CTA streams the band in 32 x 256 chunks (coalesced along rows),
// prefetching chunk i+1 into registers while warp 0 folds chunk i out of
// shared memory (double-buffered); lane o adds its line's values in
// ascending index order. One chain per output, so each sum is bitwise the
// serial ascending-index sum, independent of layout and tiling.
constexpr int kOut = 32, kStep = 256, kLsThreads = 256, kPer = kOut * kStep / kLsThreads;

template <typename T>
__global__ void __launch_bounds__(kLsThreads) line_sums_kernel(EwView a, uint64_t rows, uint64_t cols,
                                                                int by_rows, void* __restrict__ acc,
                                                                uint64_t acc_stride, int acc_prec, T alpha) {
  extern __shared__ __align__(16) unsigned char ls_smem[];
  T(*st)[kOut][kStep + 1] = reinterpret_cast<T(*)[kOut][kStep + 1]>(ls_smem);
  const uint64_t outs = by_rows ? rows : cols;  // number of sums
  const uint64_t len = by_rows ? cols : rows;   // length of each chain
  const uint64_t o0 = static_cast<uint64_t>(blockIdx.x) * kOut;
  const int tid = threadIdx.x;
  T pre[kPer];
  auto coords = [&](int i, uint64_t s0, int& o, int& s, uint64_t& r, uint64_t& c) {
    if (by_rows) {  // consecutive i -> consecutive columns of one row
      o = i / kStep;
      s = i % kStep;
      r = o0 + o;
      c = s0 + s;
    } else {  // consecutive i -> consecutive columns (outputs) of one row
      s = i / kOut;
      o = i % kOut;
      r = s0 + s;
      c = o0 + o;
    }
  };
  auto fetch = [&](uint64_t s0) {
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      int o, s;
      uint64_t r, c;
      coords(tid + j * kLsThreads, s0, o, s, r, c);
      pre[j] = (r < rows && c < cols) ? load_as<T>(a.ptr, a.prec, r * a.ld + c) : T(0);
    }
  };
  T sum = T(0);
  int buf = 0;
  fetch(0);
  for (uint64_t s0 = 0; s0 < len; s0 += kStep, buf ^= 1) {
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      int o, s;
      uint64_t r, c;
      coords(tid + j * kLsThreads, s0, o, s, r, c);
      st[buf][o][s] = pre[j];
    }
    __syncthreads();
    if (s0 + kStep < len) fetch(s0 + kStep);  // in flight while warp 0 sums
    if (tid < kOut) {
      const int n = static_cast<int>(len - s0 < kStep ? len - s0 : kStep);
      for (int s = 0; s < n; ++s) sum = add_rn(sum, st[buf][tid][s]);
    }
    // Buffer buf is rewritten two iterations later, after the barrier that
    // warp 0 reaches only once it has finished here.
  }
  if (tid < kOut && o0 + tid < outs) {
    const uint64_t idx = (o0 + tid) * acc_stride;
    line_sum_out<T>(acc, acc_prec, idx, alpha, sum);
  }
}

// Line sums, aligned fast path: the same ascending chains, fed by a 4-stage
// cp.async ring of raw storage in shared memory (16-byte copies, zero-filled
// past the band's edge), so ~3 stages (384 elements per chain) are in flight
// while warp 0 folds the current one. A CTA owns 32 outputs:
//   by rows: stage = 32 rows x 128 elements, row pitch 128*E + 16 bytes, so
//            lane o's 16-byte LDS of its row are bank-conflict-free;
//   by cols: stage = 128 rows x 32 elements (lane o reads column o).
// Zero padding is exact: a chain that starts at +0 never holds -0, so adding
// +0 leaves it unchanged.
constexpr int kAsThreads = 128;
// Elements per chain per stage: 256 for 16-bit storage (one barrier per 256
// folds; 6 x 16.5 KB ring, two CTAs per SM), 128 for wider elements.
constexpr int as_step(int elem_bytes) { return elem_bytes <= 2 ? 256 : 128; }
// Ring depth: the folding warp eats a chunk in ~512 cycles, so keep ~5 chunks
// in flight to cover HBM latency (4 for 8-byte elements: smem).
constexpr int as_stages(int elem_bytes) { return elem_bytes >= 8 ? 4 : 6; }

__device__ __forceinline__ void cp_async16(uint32_t saddr, const void* g, uint32_t bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(saddr), "l"(g), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// s + widen(v) in one instruction: sm_100's mixed-precision add (PTX
// add.rn.f32.bf16 / .f16, SASS FHADD[.BF16], which also reads the upper half
// of a register directly). The 16-bit value converts to fp32 exactly, so the
// result is the same round-to-nearest fp32 add as add_rn(s, widen(v)), with
// no widen instruction on the ordered chain.
template <int P>
__device__ __forceinline__ float add_mixed(float s, uint16_t v) {
  static_assert(P == 0 || P == 3, "16-bit storage only");
  if constexpr (P == 3)
    asm("add.rn.f32.bf16 %0, %1, %0;" : "+f"(s) : "h"(v));
  else
    asm("add.rn.f32.f16 %0, %1, %0;" : "+f"(s) : "h"(v));
  return s;
}
template <int P>
__device__ __forceinline__ float add_mixed2(float s, uint32_t word) {
  uint16_t lo, hi;
  asm("mov.b32 {%0, %1}, %2;" : "=h"(lo), "=h"(hi) : "r"(word));
  return add_mixed<P>(add_mixed<P>(s, lo), hi);
}
// One step of an ordered line-sum chain: the mixed-precision add when the
// chain is fp32 over 16-bit storage, else widen + add_rn.
template <int P, typename T>
__device__ __forceinline__ T fold_step(T s, typename Stor<P>::type v) {
  if constexpr (std::is_same<T, float>::value && (P == 0 || P == 3))
    return add_mixed<P>(s, static_cast<uint16_t>(v));
  else
    return add_rn(s, widen<P, T>(v));
}

template <typename T, int P>
__global__ void __launch_bounds__(kAsThreads) line_sums_async_kernel(const void* __restrict__ a, uint64_t lda,
                                                                      uint64_t rows, uint64_t cols, int by_rows,
                                                                      void* __restrict__ acc, uint64_t acc_stride,
                                                                      int acc_prec, T alpha) {
  using S = typename Stor<P>::type;
  constexpr int E = sizeof(S), VE = 16 / E;
  constexpr int kAsStages = as_stages(E);
  constexpr int kAsStep = as_step(E);
  constexpr int kPitchR = kAsStep * E + 16, kStageR = 32 * kPitchR;
  constexpr int kPitchC = 32 * E, kStageC = kAsStep * kPitchC;
  constexpr int kStage = kStageR > kStageC ? kStageR : kStageC;
  extern __shared__ __align__(128) unsigned char ring[];
  const uint32_t ring_s = static_cast<uint32_t>(__cvta_generic_to_shared(ring));
  const uint64_t outs = by_rows ? rows : cols;
  const uint64_t len = by_rows ? cols : rows;
  const uint64_t o0 = static_cast<uint64_t>(blockIdx.x) * 32;
  const uint64_t nchunks = (len + kAsStep - 1) / kAsStep;
  const unsigned char* ab = static_cast<const unsigned char*>(a);
  const int tid = threadIdx.x;
  // The folding warp: row-sum CTAs use warp 0, column-sum CTAs warp 2. The
  // two directions run concurrently (two streams) and share SMs, so their
  // folding warps sit on different SM sub-partitions instead of contending
  // for one scheduler's issue slots.
  const int fw = by_rows ? 0 : 2;
  const bool folder = (tid >> 5) == fw;
  const int lane = tid & 31;

  auto issue = [&](uint64_t chunk) {
    const uint32_t st = ring_s + static_cast<uint32_t>((chunk % kAsStages) * kStage);
    const uint64_t s0 = chunk * kAsStep;
    constexpr int kVecs = 32 * kAsStep / VE;  // 16-byte copies per stage
    // The three other warps copy; the folding warp only folds.
    if (folder) return;
    const int ptid = tid - (tid >= fw * 32 ? 32 : 0);
    for (int q = ptid; q < kVecs; q += kAsThreads - 32) {
      uint64_t r, c;
      uint32_t soff;
      if (by_rows) {
        constexpr int per = kAsStep / VE;
        const int o = q / per, v = q % per;
        r = o0 + o;
        c = s0 + static_cast<uint64_t>(v) * VE;
        soff = static_cast<uint32_t>(o * kPitchR + v * 16);
      } else {
        constexpr int per = 32 / VE;
        const int sr = q / per, v = q % per;
        r = s0 + sr;
        c = o0 + static_cast<uint64_t>(v) * VE;
        soff = static_cast<uint32_t>(sr * kPitchC + v * 16);
      }
      uint32_t bytes = 0;
      const unsigned char* g = ab;
      if (r < rows && c < cols) {
        const uint64_t left = (cols - c) * E;
        bytes = left < 16 ? static_cast<uint32_t>(left) : 16u;
        g = ab + (r * lda + c) * E;
      }
      cp_async16(st + soff, g, bytes);
    }
  };

  for (int i = 0; i < kAsStages - 1; ++i) {
    if (static_cast<uint64_t>(i) < nchunks) issue(i);
    cp_async_commit();
  }
  T sum = T(0);
  for (uint64_t i = 0; i < nchunks; ++i) {
    cp_async_wait<kAsStages - 2>();
    __syncthreads();
    if (i + kAsStages - 1 < nchunks) issue(i + kAsStages - 1);
    cp_async_commit();
    if (folder) {
      const unsigned char* st = ring + (i % kAsStages) * kStage;
      if (by_rows) {
        const unsigned char* row = st + lane * kPitchR;
#pragma unroll 16
        for (int v = 0; v < kAsStep / VE; ++v) {
          union {
            uint4 u;
            S e[VE];
          } w;
          w.u = *reinterpret_cast<const uint4*>(row + v * 16);
#pragma unroll
          for (int k = 0; k < VE; ++k) sum = fold_step<P, T>(sum, w.e[k]);
        }
      } else {
        const S* col = reinterpret_cast<const S*>(st) + lane;
#pragma unroll 64
        for (int sr = 0; sr < kAsStep; ++sr) sum = fold_step<P, T>(sum, col[sr * 32]);
      }
    }
  }
  cp_async_wait<0>();
  if (folder && o0 + lane < outs) {
    const uint64_t idx = (o0 + lane) * acc_stride;
    line_sum_out<T>(acc, acc_prec, idx, alpha, sum);
  }
}

// Line sums for 16-bit storage, TMA-fed: the same ascending chains (one
// lane = one output), but the stages arrive by cp.async.bulk.tensor issued
// by one thread, so the folding warp owns its SM sub-partition (no copy
// warps competing for issue slots) and synchronises through mbarriers, not
// a CTA barrier per stage. 64 threads: warp 0 folds, warp 1 lane 0 loads.
//   by rows: a stage is 4 boxes of 32 rows x 64 elements (128-byte rows,
//            128-byte swizzle: lane o's 16-byte chunk j of its row sits at
//            j ^ (o & 7), so the 8 lanes of an LDS.128 phase hit 8 banks);
//   by cols: a stage is one box of 256 rows x 32 elements (lane o reads
//            column o: a warp reads one contiguous 64-byte row).
// The chain step is sm_100's mixed-precision add (add_mixed), one FHADD per
// element with no separate widen.
// Out-of-range box elements are zero-filled by TMA: exact, a chain starting
// at +0 never holds -0.
constexpr int kTsThreads = 64;
constexpr int kTsStep = 256;     // elements per chain per stage
constexpr int kTsStages = 6;
constexpr int kTsStage = 16384;  // bytes per stage (32 x 256 x 2)

template <typename T, int P>
__global__ void __launch_bounds__(kTsThreads) line_sums_tma_kernel(const __grid_constant__ CUtensorMap map,
                                                                   uint64_t rows, uint64_t cols, int by_rows,
                                                                   void* __restrict__ acc, uint64_t acc_stride,
                                                                   int acc_prec, T alpha) {
  using S = typename Stor<P>::type;
  static_assert(sizeof(S) == 2, "16-bit storage only");
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // Offset from the shared array itself (not through an integer cast), so
  // the folds compile to LDS rather than generic loads.
  unsigned char* ring = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + kTsStages * kTsStage);
  uint64_t* empty = full + kTsStages;
  const uint64_t outs = by_rows ? rows : cols;
  const uint64_t len = by_rows ? cols : rows;
  const uint64_t o0 = static_cast<uint64_t>(blockIdx.x) * 32;
  const uint32_t nchunks = static_cast<uint32_t>((len + kTsStep - 1) / kTsStep);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 32) {
    tma_prefetch_desc(&map);
    for (int s = 0; s < kTsStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    fence_barrier_init();
  }
  __syncthreads();
  if (warp == 1) {
    if (lane == 0) {
      for (uint32_t i = 0; i < nchunks; ++i) {
        const uint32_t s = i % kTsStages;
        if (i >= kTsStages) mbar_wait(&empty[s], ((i / kTsStages) - 1) & 1);
        unsigned char* st = ring + s * kTsStage;
        mbar_arrive_expect_tx(&full[s], kTsStage);
        const int32_t k0 = static_cast<int32_t>(i * kTsStep);
        if (by_rows) {
#pragma unroll
          for (int b = 0; b < 4; ++b) tma_load_2d(st + b * 4096, &map, &full[s], k0 + b * 64, static_cast<int32_t>(o0));
        } else {
          tma_load_2d(st, &map, &full[s], static_cast<int32_t>(o0), k0);
        }
      }
    }
    return;
  }
  T sum = T(0);
  for (uint32_t i = 0; i < nchunks; ++i) {
    const uint32_t s = i % kTsStages;
    mbar_wait(&full[s], (i / kTsStages) & 1);
    const unsigned char* st = ring + s * kTsStage;
    if (by_rows) {
      // A box row (64 elements) is loaded ahead of its 64 ordered adds.
      const unsigned char* row = st + lane * 128;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        uint4 w[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) w[j] = *reinterpret_cast<const uint4*>(row + b * 4096 + ((j ^ (lane & 7)) << 4));
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint32_t q[4] = {w[j].x, w[j].y, w[j].z, w[j].w};
#pragma unroll
          for (int k = 0; k < 4; ++k) sum = add_mixed2<P>(sum, q[k]);
        }
      }
    } else {
      // 32 rows of the lane's column are loaded ahead of their adds.
      const S* col = reinterpret_cast<const S*>(st) + lane;
#pragma unroll 1
      for (int r0 = 0; r0 < kTsStep; r0 += 32) {
        S v[32];
#pragma unroll
        for (int r = 0; r < 32; ++r) v[r] = col[(r0 + r) * 32];
#pragma unroll
        for (int r = 0; r < 32; ++r) sum = add_mixed<P>(sum, static_cast<uint16_t>(v[r]));
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
  if (o0 + lane < outs) {
    const uint64_t idx = (o0 + lane) * acc_stride;
    line_sum_out<T>(acc, acc_prec, idx, alpha, sum);
  }
}

template <typename T, int P>
cudaError_t launch_sums_tma(EwView band, uint64_t rows, uint64_t cols, int by_rows, void* acc, uint64_t acc_stride,
                            int acc_prec, T alpha, cudaStream_t s, bool* done) {
  *done = false;
  CUtensorMap map;
  const int enc = by_rows ? encode_map_2d(&map, band.ptr, 2, cols, rows, band.ld, 64, 32, 128)
                          : encode_map_2d(&map, band.ptr, 2, cols, rows, band.ld, 32, kTsStep, 0);
  if (enc) return cudaSuccess;  // not encodable: the cp.async path runs instead
  constexpr size_t smem = kTsStages * kTsStage + 2 * kTsStages * 8 + 1024;
  const cudaError_t attr = cudaFuncSetAttribute(line_sums_tma_kernel<T, P>,
                                                cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (attr != cudaSuccess) return attr;
  const uint64_t outs = by_rows ? rows : cols;
  line_sums_tma_kernel<T, P><<<static_cast<unsigned>((outs + 31) / 32), kTsThreads, smem, s>>>(
      map, rows, cols, by_rows, acc, acc_stride, acc_prec, alpha);
  *done = true;
  return cudaSuccess;
}

template <typename T, int P>
cudaError_t launch_sums_async(EwView band, uint64_t rows, uint64_t cols, int by_rows, void* acc,
                              uint64_t acc_stride, int acc_prec, T alpha, cudaStream_t s) {
  using S = typename Stor<P>::type;
  constexpr int E = sizeof(S);
  constexpr int kAsStep = as_step(E);
  constexpr int kStageR = 32 * (kAsStep * E + 16), kStageC = kAsStep * 32 * E;
  constexpr size_t smem = static_cast<size_t>(as_stages(E)) * (kStageR > kStageC ? kStageR : kStageC);
  // Per device (the attribute lives in each device's context).
  const cudaError_t attr = cudaFuncSetAttribute(line_sums_async_kernel<T, P>,
                                                cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (attr != cudaSuccess) return attr;
  const uint64_t outs = by_rows ? rows : cols;
  line_sums_async_kernel<T, P><<<static_cast<unsigned>((outs + 31) / 32), kAsThreads, smem, s>>>(
      band.ptr, band.ld, rows, cols, by_rows, acc, acc_stride, acc_prec, alpha);
  return cudaSuccess;
}

dim3 rect_grid(uint64_t rows, uint64_t cols, unsigned threads) {
  uint64_t gx = (cols + threads - 1) / threads;
  if (gx > 64) gx = 64;
  if (gx == 0) gx = 1;
  uint64_t gy = (148ull * 8 + gx - 1) / gx;
  if (gy > rows) gy = rows;
  if (gy > 65535) gy = 65535;
  if (gy == 0) gy = 1;
  return dim3(static_cast<unsigned>(gx), static_cast<unsigned>(gy));
}

bool vec_ok(const void* p, uint64_t ld, int eb) {
  return (reinterpret_cast<uintptr_t>(p) % 16 == 0) && ((ld * eb) % 16 == 0);
}

template <typename T, int P>
void launch_vec(EwView x, EwView y, int ybc, void* dst, uint64_t dld, uint64_t rows, uint64_t cols, int kind,
                T alpha, cudaStream_t s) {
  constexpr int N = 16 / sizeof(typename Stor<P>::type);
  const dim3 g = rect_grid(rows, (cols + N - 1) / N, 256);
  ew_vec_kernel<T, P><<<g, 256, 0, s>>>(x, y, ybc, dst, dld, rows, cols, kind, alpha);
}

}  // namespace

cudaError_t ew_apply(EwView x, EwView y, int y_row_bcast, void* dst, uint64_t dld, int dprec, uint64_t rows,
                     uint64_t cols, int kind, double alpha, int double_compute, cudaStream_t s) {
  if (rows == 0 || cols == 0) return cudaSuccess;
  const bool useY = kind >= kEwAdd && kind != kEwCopy;
  const int eb = dprec == 2 ? 8 : (dprec == 1 ? 4 : 2);
  const bool same = x.prec == dprec && (!useY || y.prec == dprec);
  const bool aligned = vec_ok(x.ptr, x.ld, eb) && vec_ok(dst, dld, eb) && (!useY || vec_ok(y.ptr, y.ld, eb));
  if (same && aligned) {
    const float af = static_cast<float>(alpha);
    switch (dprec) {
      case 0: launch_vec<float, 0>(x, y, y_row_bcast, dst, dld, rows, cols, kind, af, s); break;
      case 1: launch_vec<float, 1>(x, y, y_row_bcast, dst, dld, rows, cols, kind, af, s); break;
      case 2: launch_vec<double, 2>(x, y, y_row_bcast, dst, dld, rows, cols, kind, alpha, s); break;
      default: launch_vec<float, 3>(x, y, y_row_bcast, dst, dld, rows, cols, kind, af, s); break;
    }
  } else {
    const dim3 g = rect_grid(rows, cols, 256);
    if (double_compute)
      ew_kernel<double><<<g, 256, 0, s>>>(x, y, y_row_bcast, dst, dld, dprec, rows, cols, kind, alpha);
    else
      ew_kernel<float><<<g, 256, 0, s>>>(x, y, y_row_bcast, dst, dld, dprec, rows, cols, kind,
                                         static_cast<float>(alpha));
  }
  count_launch();
  return cudaGetLastError();
}

cudaError_t set_const(void* dst, uint64_t ld, int prec, uint64_t rows, uint64_t cols, double value,
                      cudaStream_t s) {
  if (rows == 0 || cols == 0) return cudaSuccess;
  set_const_kernel<<<rect_grid(rows, cols, 256), 256, 0, s>>>(dst, ld, prec, rows, cols, value);
  count_launch();
  return cudaGetLastError();
}

cudaError_t line_sums(EwView band, uint64_t rows, uint64_t cols, int by_rows, void* acc, uint64_t acc_stride,
                      int acc_prec, double alpha, int double_compute, cudaStream_t s) {
  const uint64_t outs = by_rows ? rows : cols;
  if (outs == 0) return cudaSuccess;
  const int eb = band.prec == 2 ? 8 : (band.prec == 1 ? 4 : 2);
  // Fast path: 16-byte aligned band rows; the chain type follows the
  // reference (double iff any operand is Double).
  if (vec_ok(band.ptr, band.ld, eb) && (double_compute ? band.prec == 2 : band.prec != 2)) {
    cudaError_t e;
    const float af = static_cast<float>(alpha);
    if (band.prec == 0 || band.prec == 3) {
      bool done = false;
      e = band.prec == 0 ? launch_sums_tma<float, 0>(band, rows, cols, by_rows, acc, acc_stride, acc_prec, af, s, &done)
                         : launch_sums_tma<float, 3>(band, rows, cols, by_rows, acc, acc_stride, acc_prec, af, s, &done);
      if (e != cudaSuccess) return e;
      if (done) {
        count_launch();
        return cudaGetLastError();
      }
    }
    switch (band.prec) {
      case 0: e = launch_sums_async<float, 0>(band, rows, cols, by_rows, acc, acc_stride, acc_prec, af, s); break;
      case 1: e = launch_sums_async<float, 1>(band, rows, cols, by_rows, acc, acc_stride, acc_prec, af, s); break;
      case 2: e = launch_sums_async<double, 2>(band, rows, cols, by_rows, acc, acc_stride, acc_prec, alpha, s); break;
      default: e = launch_sums_async<float, 3>(band, rows, cols, by_rows, acc, acc_stride, acc_prec, af, s); break;
    }
    if (e != cudaSuccess) return e;
    count_launch();
    return cudaGetLastError();
  }
  const unsigned grid = static_cast<unsigned>((outs + kOut - 1) / kOut);
  if (double_compute) {
    const size_t smem = 2 * kOut * (kStep + 1) * sizeof(double);
    const cudaError_t attr =
        cudaFuncSetAttribute(line_sums_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (attr != cudaSuccess) return attr;
    line_sums_kernel<double><<<grid, kLsThreads, smem, s>>>(band, rows, cols, by_rows, acc, acc_stride, acc_prec,
                                                            alpha);
  } else {
    const size_t smem = 2 * kOut * (kStep + 1) * sizeof(float);
    const cudaError_t attr =
        cudaFuncSetAttribute(line_sums_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (attr != cudaSuccess) return attr;
    line_sums_kernel<float><<<grid, kLsThreads, smem, s>>>(band, rows, cols, by_rows, acc, acc_stride, acc_prec,
                                                           static_cast<float>(alpha));
  }
  count_launch();
  return cudaGetLastError();
}

}  // namespace gmk
