// SPDX-License-Identifier: Apache-2.0
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace gmk {
struct F64GemmArgs {
  uint64_t m = 0, n = 0, k = 0;
  bool trans_a = false, trans_b = false;
  const void* a = nullptr;  // fp64, 16B aligned, even pitch
  const void* b = nullptr;
  void* c = nullptr;
  uint64_t lda = 0, ldb = 0, ldc = 0;
  int c_prec = 2;           // storage precision of C (GM_* tag)
  double alpha = 1.0, beta = 0.0;
};
int f64_gemm(const F64GemmArgs& args, cudaStream_t stream, const char** err);
}  // namespace gmk
