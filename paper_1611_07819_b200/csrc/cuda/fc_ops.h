// SPDX-License-Identifier: Apache-2.0
// FC-layer neighbours of the GEMM: elementwise unary and
// binary ops, setConst, and the deterministic row/column sums, per tile.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace gmk {

// One operand view: storage precision tag (0 half, 1 single, 2 double,
// 3 bf16), row pitch in elements.
struct EwView {
  const void* ptr;
  uint64_t ld;
  int prec;
};

// Kinds: reference UnaryKind (ops.hpp:41) as 0..1, BinaryKind (ops.hpp:42)
// as 16 + kind.
enum EwKind : int {
  kEwRelu = 0,
  kEwMulScalar = 1,
  kEwAdd = 16,
  kEwSub = 17,
  kEwAxpy = 18,
  kEwReluGrad = 19,
  kEwCopy = 20,
  kEwBiasAdd = 21,
};

// dst(r, c) = f(x(r, c), y(r, c) or y(0, c) when y_row_bcast), computed in
// double when `double_compute`, else float, stored in dst's precision.
cudaError_t ew_apply(EwView x, EwView y, int y_row_bcast, void* dst, uint64_t dld, int dprec,
                     uint64_t rows, uint64_t cols, int kind, double alpha, int double_compute,
                     cudaStream_t s);
// Every element of the rows x cols rectangle = value (storeScalar<double>).
cudaError_t set_const(void* dst, uint64_t ld, int prec, uint64_t rows, uint64_t cols, double value,
                      cudaStream_t s);
// acc_prec | kLineSumsZeroAcc: the outputs count as zero (acc[o] = 0 + alpha
// * sum, bit-for-bit a setConst(0) followed by the sums).
constexpr int kLineSumsZeroAcc = 0x100;
// acc[o] = acc[o] + alpha * sum, one sum per row (by_rows) or per column of
// the rows x cols band, accumulated in ascending index order in the compute
// type (bit-for-bit the reference's runRowColSumDet chain). acc element o
// lives at acc + o * acc_stride.
cudaError_t line_sums(EwView band, uint64_t rows, uint64_t cols, int by_rows, void* acc,
                      uint64_t acc_stride, int acc_prec, double alpha, int double_compute,
                      cudaStream_t s);

}  // namespace gmk
