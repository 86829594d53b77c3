// SPDX-License-Identifier: Apache-2.0
// Storage-precision conversion, rectangle staging, 3xTF32 operand split and
// the SplitMix64 synthetic-input generator, all as HBM-bound grid-stride
// kernels (one pass, coalesced along rows).
//
// Conversion semantics follow the reference's convertBuffer / storeScalar
// (proj/src/precision.cpp:6-28, proj/include/gridmath/precision.hpp:42-149):
//   * any -> Half rounds through float (double -> float -> half, RNE), values
//     >= 65520 become +-inf, NaN keeps its top payload bits (or 1);
//   * Double -> Single is RNE;  Half/Single/BF16 -> wider is exact;
//   * BF16 (new tag 3) is RNE from float, and from double through float,
//     matching the Half convention.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>

#include "convert.h"
#include "prec.cuh"

namespace gmk {

// Rectangle iteration without a 64-bit division per element: rows go over
// blockIdx.x (grid-stride), columns over blockIdx.y * blockDim.x + threadIdx.x
// (stride gridDim.y * blockDim.x). rect_grid() sizes the grid.
#define GM_FOR_RECT(rows, cols, r, c)                                                   \
  for (uint64_t r = blockIdx.x; r < (rows); r += gridDim.x)                            \
    for (uint64_t c = static_cast<uint64_t>(blockIdx.y) * blockDim.x + threadIdx.x; c < (cols); \
         c += static_cast<uint64_t>(gridDim.y) * blockDim.x)

// Elementwise rectangle conversion. Single->Half takes the float fast path
// (the reference's convertBuffer does the same; the results are identical).
__global__ void convert_rect_kernel(const void* __restrict__ src, int sp, uint64_t sld,
                                    void* __restrict__ dst, int dp, uint64_t dld, uint64_t rows,
                                    uint64_t cols) {
  const bool via_f32 = (sp != 2 && dp != 2);
  GM_FOR_RECT(rows, cols, r, c) {
    if (via_f32)
      store_elem_f32(dst, dp, r * dld + c, load_elem_f32(src, sp, r * sld + c));
    else
      store_elem(dst, dp, r * dld + c, load_elem(src, sp, r * sld + c));
  }
}

// 3xTF32 split: hi = tf32_rna(x) (low 13 mantissa bits zero), lo = x - hi.
__global__ void split_tf32_kernel(const void* __restrict__ src, int sp, uint64_t sld,
                                  float* __restrict__ hi, float* __restrict__ lo, uint64_t dld,
                                  uint64_t rows, uint64_t cols) {
  GM_FOR_RECT(rows, cols, r, c) {
    const float x = load_elem_f32(src, sp, r * sld + c);
    uint32_t h;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(x));
    const float hf = __uint_as_float(h);
    hi[r * dld + c] = hf;
    lo[r * dld + c] = x - hf;
  }
}

// Transposing variants: src is R x C (pitch sld); dst is C x R (pitch dld).
// 32x32 tiles staged through shared memory so both sides stay coalesced.
__global__ void split_tf32_t_kernel(const void* __restrict__ src, int sp, uint64_t sld,
                                    float* __restrict__ hi, float* __restrict__ lo, uint64_t dld,
                                    uint64_t rows, uint64_t cols, int split) {
  __shared__ float tile[32][33];
  const uint64_t r0 = static_cast<uint64_t>(blockIdx.y) * 32, c0 = static_cast<uint64_t>(blockIdx.x) * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const uint64_t r = r0 + i, c = c0 + threadIdx.x;
    tile[i][threadIdx.x] = (r < rows && c < cols) ? load_elem_f32(src, sp, r * sld + c) : 0.0f;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const uint64_t oc = c0 + i, orow = r0 + threadIdx.x;  // output row = source col
    if (oc < cols && orow < rows) {
      const float x = tile[threadIdx.x][i];
      if (split) {
        uint32_t h;
        asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(x));
        const float hf = __uint_as_float(h);
        hi[oc * dld + orow] = hf;
        lo[oc * dld + orow] = x - hf;
      } else {
        hi[oc * dld + orow] = x;
      }
    }
  }
}

__device__ __forceinline__ uint64_t avalanche64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  return z;
}

// Draw i (0-based) of SplitMix64(seed) is avalanche64(seed + (i+1)*salt)
// (reference common.hpp:37-50); element (r, c) of a full_cols-wide matrix is
// draw r*full_cols + c, mapped to lo + (hi-lo)*u with u in [0,1) on 53 bits,
// then stored like setData (double -> storage, convertBuffer rules).
__global__ void fill_uniform_kernel(void* __restrict__ dst, int prec, uint64_t ld, uint64_t r0,
                                    uint64_t rows, uint64_t c0, uint64_t cols, uint64_t full_cols,
                                    uint64_t seed, double lo, double hi) {
  GM_FOR_RECT(rows, cols, r, c) {
    const uint64_t draw = (r0 + r) * full_cols + (c0 + c);
    const uint64_t x = avalanche64(seed + (draw + 1) * 0x9E3779B97F4A7C15ull);
    const double u = static_cast<double>(x >> 11) * 0x1.0p-53;
    // Separate multiply and add (no FMA contraction), exactly like the
    // reference's nextUniform built without -march.
    store_elem(dst, prec, r * ld + c, __dadd_rn(lo, __dmul_rn(hi - lo, u)));
  }
}

// Same draws, eight consecutive columns per thread and one 16-byte store per
// 16 bytes of output. The generator is issue-bound (three 64-bit multiplies,
// a u64 -> f64 convert and two f64 ops per element), so the per-element hash
// input advances by one add (z += salt) instead of a 64-bit multiply, and
// the index / precision switch is hoisted out of the element loop. Needs
// 16-byte aligned rows (dst and ld * elem); the < 8 trailing columns of a
// row go through the scalar formula.
template <int P>
__device__ __forceinline__ void store8(void* dst, uint64_t idx, const double (&v)[8]) {
  if constexpr (P == 2) {
    double2* d = reinterpret_cast<double2*>(reinterpret_cast<double*>(dst) + idx);
#pragma unroll
    for (int i = 0; i < 4; ++i) d[i] = make_double2(v[2 * i], v[2 * i + 1]);
  } else if constexpr (P == 1) {
    float4* d = reinterpret_cast<float4*>(reinterpret_cast<float*>(dst) + idx);
#pragma unroll
    for (int i = 0; i < 2; ++i)
      d[i] = make_float4(__double2float_rn(v[4 * i]), __double2float_rn(v[4 * i + 1]),
                         __double2float_rn(v[4 * i + 2]), __double2float_rn(v[4 * i + 3]));
  } else {
    uint32_t w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float a = __double2float_rn(v[2 * i]), b = __double2float_rn(v[2 * i + 1]);
      const uint32_t ha = P == 0 ? f32_to_half_bits(a) : f32_to_bf16_bits(a);
      const uint32_t hb = P == 0 ? f32_to_half_bits(b) : f32_to_bf16_bits(b);
      w[i] = ha | (hb << 16);
    }
    *reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(dst) + idx) = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

template <int P>
__global__ void fill_uniform_vec_kernel(void* __restrict__ dst, uint64_t ld, uint64_t r0, uint64_t rows,
                                        uint64_t c0, uint64_t cols, uint64_t full_cols, uint64_t seed,
                                        double lo, double hi) {
  constexpr uint64_t kSalt = 0x9E3779B97F4A7C15ull;
  const uint64_t groups = cols / 8;
  const uint64_t tid = static_cast<uint64_t>(blockIdx.y) * blockDim.x + threadIdx.x;
  const uint64_t stride = static_cast<uint64_t>(gridDim.y) * blockDim.x;
  const double span = hi - lo;
  for (uint64_t r = blockIdx.x; r < rows; r += gridDim.x) {
    // Hash input of column 0 of this row: seed + (draw + 1) * salt.
    const uint64_t z_row = seed + ((r0 + r) * full_cols + c0 + 1) * kSalt;
    for (uint64_t g = tid; g < groups; g += stride) {
      uint64_t z = z_row + (8 * g) * kSalt;
      double v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j, z += kSalt) {
        const double u = static_cast<double>(avalanche64(z) >> 11) * 0x1.0p-53;
        v[j] = __dadd_rn(lo, __dmul_rn(span, u));
      }
      store8<P>(dst, r * ld + 8 * g, v);
    }
    for (uint64_t c = 8 * groups + tid; c < cols; c += stride) {
      const double u = static_cast<double>(avalanche64(z_row + c * kSalt) >> 11) * 0x1.0p-53;
      store_elem(dst, P, r * ld + c, __dadd_rn(lo, __dmul_rn(span, u)));
    }
  }
}

// C = beta * C (alpha == 0 path; beta == 0 writes zeros without reading C).
__global__ void scale_rect_kernel(void* __restrict__ c, int prec, uint64_t ld, uint64_t rows,
                                  uint64_t cols, double beta) {
  GM_FOR_RECT(rows, cols, r, cc) {
    const uint64_t idx = r * ld + cc;
    if (beta == 0.0) {
      store_elem(c, prec, idx, 0.0);
    } else if (prec == 2) {
      store_elem(c, prec, idx, beta * load_elem(c, prec, idx));
    } else {
      // Single compute: beta and C in float, like runGemm<float>.
      store_elem_f32(c, prec, idx, static_cast<float>(beta) * load_elem_f32(c, prec, idx));
    }
  }
}

namespace {
std::atomic<uint64_t> g_launches{0};
}  // namespace

uint64_t kernel_launches() { return g_launches.load(); }
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

namespace {
// ~16 blocks of 256 threads per SM in total: columns get up to
// ceil(cols / 256) blocks (at most 16), rows the rest.
dim3 rect_grid(uint64_t rows, uint64_t cols) {
  uint64_t gy = (cols + 255) / 256;
  if (gy > 16) gy = 16;
  if (gy == 0) gy = 1;
  uint64_t gx = 148ull * 16 / gy;
  if (gx > rows) gx = rows;
  if (gx == 0) gx = 1;
  return dim3(static_cast<unsigned>(gx), static_cast<unsigned>(gy), 1);
}
}  // namespace

cudaError_t convert_rect(const void* src, int sp, uint64_t sld, void* dst, int dp, uint64_t dld,
                         uint64_t rows, uint64_t cols, cudaStream_t s) {
  if (rows == 0 || cols == 0) return cudaSuccess;
  convert_rect_kernel<<<rect_grid(rows, cols), 256, 0, s>>>(src, sp, sld, dst, dp, dld, rows, cols);
  count_launch();
  return cudaGetLastError();
}

cudaError_t split_tf32(const void* src, int sp, uint64_t sld, float* hi, float* lo, uint64_t dld,
                       uint64_t rows, uint64_t cols, cudaStream_t s) {
  if (rows == 0 || cols == 0) return cudaSuccess;
  split_tf32_kernel<<<rect_grid(rows, cols), 256, 0, s>>>(src, sp, sld, hi, lo, dld, rows, cols);
  count_launch();
  return cudaGetLastError();
}

cudaError_t split_tf32_t(const void* src, int sp, uint64_t sld, float* hi, float* lo,
                         uint64_t dld, uint64_t rows, uint64_t cols, bool split, cudaStream_t s) {
  if (rows == 0 || cols == 0) return cudaSuccess;
  dim3 grid(static_cast<unsigned>((cols + 31) / 32), static_cast<unsigned>((rows + 31) / 32));
  split_tf32_t_kernel<<<grid, dim3(32, 8), 0, s>>>(src, sp, sld, hi, lo, dld, rows, cols, split ? 1 : 0);
  count_launch();
  return cudaGetLastError();
}

cudaError_t fill_uniform(void* dst, int prec, uint64_t ld, uint64_t r0, uint64_t rows, uint64_t c0,
                         uint64_t cols, uint64_t full_cols, uint64_t seed, double lo, double hi,
                         cudaStream_t s) {
  if (rows == 0 || cols == 0) return cudaSuccess;
  const uint64_t es = prec == 2 ? 8 : prec == 1 ? 4 : 2;
  if (cols >= 8 && reinterpret_cast<uintptr_t>(dst) % 16 == 0 && (ld * es) % 16 == 0 && prec >= 0 &&
      prec <= 3) {
    const dim3 grid = rect_grid(rows, cols / 8);
    switch (prec) {
      case 0: fill_uniform_vec_kernel<0><<<grid, 256, 0, s>>>(dst, ld, r0, rows, c0, cols, full_cols, seed, lo, hi); break;
      case 1: fill_uniform_vec_kernel<1><<<grid, 256, 0, s>>>(dst, ld, r0, rows, c0, cols, full_cols, seed, lo, hi); break;
      case 2: fill_uniform_vec_kernel<2><<<grid, 256, 0, s>>>(dst, ld, r0, rows, c0, cols, full_cols, seed, lo, hi); break;
      default: fill_uniform_vec_kernel<3><<<grid, 256, 0, s>>>(dst, ld, r0, rows, c0, cols, full_cols, seed, lo, hi); break;
    }
    count_launch();
    return cudaGetLastError();
  }
  fill_uniform_kernel<<<rect_grid(rows, cols), 256, 0, s>>>(dst, prec, ld, r0, rows, c0, cols,
                                                            full_cols, seed, lo, hi);
  count_launch();
  return cudaGetLastError();
}

cudaError_t scale_rect(void* c, int prec, uint64_t ld, uint64_t rows, uint64_t cols, double beta,
                       cudaStream_t s) {
  if (rows == 0 || cols == 0) return cudaSuccess;
  scale_rect_kernel<<<rect_grid(rows, cols), 256, 0, s>>>(c, prec, ld, rows, cols, beta);
  count_launch();
  return cudaGetLastError();
}

}  // namespace gmk
