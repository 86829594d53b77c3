// SPDX-License-Identifier: Apache-2.0
// Host-side entry for the tcgen05 tile GEMM (gemm_tc.cu).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace gmk {

enum class TcKind : int { F16 = 0, BF16 = 1, TF32 = 2, TF32X3 = 3 };

struct TcOperand {
  const void* ptr = nullptr;  // 16-byte aligned
  uint64_t ld = 0;            // row pitch in elements (pitch bytes % 16 == 0)
};

struct TcGemmArgs {
  uint64_t m = 0, n = 0, k = 0;
  bool trans_a = false, trans_b = false;
  TcKind kind = TcKind::BF16;
  TcOperand a, b, a_lo, b_lo;  // *_lo only for TF32X3
  void* c = nullptr;
  uint64_t ldc = 0;
  uint32_t c_dtype = 1;  // 0 f16, 1 bf16, 2 f32
  double alpha = 1.0, beta = 0.0;
  int cta_group = 2;     // 1 or 2 (2-SM UMMA)
  int max_ctas = 0;      // 0 = all SMs (persistent grid); else cap (leaves SMs for comm)
  // TF32 kinds: fold the tensor-core accumulation into an fp32 running sum
  // every fold_k of k (a multiple of 32; 0 = accumulate all of k in TMEM).
  uint64_t fold_k = 0;
  // Fused `biasAdd + relu` epilogue (bf16 C): C = bf16(bf16(alpha*acc) +
  // bias[col]), act = relu(C). bias holds the local C's n columns.
  const void* bias = nullptr;
  void* act = nullptr;
  uint64_t ld_act = 0;
};

// Launches on `stream`; returns 0 or 1 with *err set (static string).
int tc_gemm(const TcGemmArgs& args, cudaStream_t stream, const char** err);

}  // namespace gmk
