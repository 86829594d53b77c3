// SPDX-License-Identifier: Apache-2.0
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace gmk {
// prec tags: 0 half, 1 single, 2 double, 3 bf16 (gridmath_b200.h GM_*).
cudaError_t convert_rect(const void* src, int sp, uint64_t sld, void* dst, int dp, uint64_t dld,
                         uint64_t rows, uint64_t cols, cudaStream_t s);
cudaError_t split_tf32(const void* src, int sp, uint64_t sld, float* hi, float* lo, uint64_t dld,
                       uint64_t rows, uint64_t cols, cudaStream_t s);
// Transposing split/convert to fp32: src R x C -> dst C x R (hi only when !split).
cudaError_t split_tf32_t(const void* src, int sp, uint64_t sld, float* hi, float* lo,
                         uint64_t dld, uint64_t rows, uint64_t cols, bool split, cudaStream_t s);
cudaError_t fill_uniform(void* dst, int prec, uint64_t ld, uint64_t r0, uint64_t rows, uint64_t c0,
                         uint64_t cols, uint64_t full_cols, uint64_t seed, double lo, double hi,
                         cudaStream_t s);
cudaError_t scale_rect(void* c, int prec, uint64_t ld, uint64_t rows, uint64_t cols, double beta,
                       cudaStream_t s);
// Process-wide count of kernels this library launched.
uint64_t kernel_launches();
void count_launch();
}  // namespace gmk
