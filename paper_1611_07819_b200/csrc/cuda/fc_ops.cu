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

#include "convert.h"
#include "fc_ops.h"
#include "prec.cuh"

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

// blockIdx.y strides rows, threads stride columns: every warp touches one
// contiguous row segment of each operand (coalesced); the kind and precision
// switches are uniform across the grid.
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

__global__ void set_const_kernel(void* __restrict__ d, uint64_t ld, int prec, uint64_t rows, uint64_t cols,
                                 double v) {
  for (uint64_t r = blockIdx.y; r < rows; r += gridDim.y)
    for (uint64_t c = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; c < cols;
         c += static_cast<uint64_t>(gridDim.x) * blockDim.x)
      store_elem(d, prec, r * ld + c, v);
}

// Line sums with the reference's sequential chain: 32 outputs per CTA; the
// whole CTA stages 32 x 64 chunks of the band through shared memory
// (coalesced along rows, double-buffered), and warp 0's lane o folds its
// line's 64 values in ascending index order. One chain per output, so the
// sum is bitwise the serial ascending-index sum.
constexpr int kOut = 32, kStep = 64, kLsThreads = 256;

template <typename T>
__global__ void __launch_bounds__(kLsThreads) line_sums_kernel(EwView a, uint64_t rows, uint64_t cols,
                                                                int by_rows, void* __restrict__ acc,
                                                                uint64_t acc_stride, int acc_prec, T alpha) {
  __shared__ T st[2][kOut][kStep + 1];
  const uint64_t outs = by_rows ? rows : cols;  // number of sums
  const uint64_t len = by_rows ? cols : rows;   // length of each chain
  const uint64_t o0 = static_cast<uint64_t>(blockIdx.x) * kOut;
  const int tid = threadIdx.x;
  T sum = T(0);
  int buf = 0;
  for (uint64_t s0 = 0; s0 < len; s0 += kStep, buf ^= 1) {
    for (int i = tid; i < kOut * kStep; i += kLsThreads) {
      int o, s;
      uint64_t r, c;
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
      st[buf][o][s] = (r < rows && c < cols) ? load_as<T>(a.ptr, a.prec, r * a.ld + c) : T(0);
    }
    __syncthreads();
    if (tid < kOut) {
      const int n = static_cast<int>(len - s0 < kStep ? len - s0 : kStep);
      for (int s = 0; s < n; ++s) sum = add_rn(sum, st[buf][tid][s]);
    }
    // The next chunk goes to the other buffer; the one after that reuses this
    // buffer only after the barrier that warp 0 reaches once it is done here.
  }
  if (tid < kOut && o0 + tid < outs) {
    const uint64_t idx = (o0 + tid) * acc_stride;
    const T cur = load_as<T>(acc, acc_prec, idx);
    store_as(acc, acc_prec, idx, add_rn(cur, mul_rn(alpha, sum)));
  }
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

}  // namespace

cudaError_t ew_apply(EwView x, EwView y, int y_row_bcast, void* dst, uint64_t dld, int dprec, uint64_t rows,
                     uint64_t cols, int kind, double alpha, int double_compute, cudaStream_t s) {
  if (rows == 0 || cols == 0) return cudaSuccess;
  const dim3 g = rect_grid(rows, cols, 256);
  if (double_compute)
    ew_kernel<double><<<g, 256, 0, s>>>(x, y, y_row_bcast, dst, dld, dprec, rows, cols, kind, alpha);
  else
    ew_kernel<float><<<g, 256, 0, s>>>(x, y, y_row_bcast, dst, dld, dprec, rows, cols, kind,
                                       static_cast<float>(alpha));
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
  const unsigned grid = static_cast<unsigned>((outs + kOut - 1) / kOut);
  if (double_compute)
    line_sums_kernel<double><<<grid, kLsThreads, 0, s>>>(band, rows, cols, by_rows, acc, acc_stride, acc_prec,
                                                         alpha);
  else
    line_sums_kernel<float><<<grid, kLsThreads, 0, s>>>(band, rows, cols, by_rows, acc, acc_stride, acc_prec,
                                                        static_cast<float>(alpha));
  count_launch();
  return cudaGetLastError();
}

}  // namespace gmk
