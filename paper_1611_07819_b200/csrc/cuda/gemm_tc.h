// SPDX-License-Identifier: Apache-2.0
// Host-side entry for the tcgen05 tile GEMM (gemm_tc.cu).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>

namespace gmk {

enum class TcKind : int { F16 = 0, BF16 = 1, TF32 = 2, TF32X3 = 3 };

struct TcOperand {
  const void* ptr = nullptr;  // 16-byte aligned
  uint64_t ld = 0;            // row pitch in elements (pitch bytes % 16 == 0)
};

// In-GEMM panel pipelining: an operand arrives block by block -- A in
// (m-chunk x k-panel) blocks, B in (n-chunk x k-panel) blocks -- and whoever
// lands a block writes flags[chunk * num_panels + panel] = target (a
// gathered band's pull streams, or a replication job per source piece). The
// GEMM's producer waits for the blocks a k-block reads before loading it, so
// panel k+1 lands while panel k multiplies. Null flags: operand resident.
struct PanelFlags {
  const uint64_t* flags = nullptr;
  uint64_t target = 0;
  uint32_t origin = 0;    // kernel row (A) / column (B) j lies in chunk (origin + j) / chunk
  uint32_t chunk = 0;     // rows (A) / columns (B) per chunk
  uint32_t chunks = 0;    // flag rows (all blocks landed: lockstep rule)
  uint32_t panel_k = 0;   // k elements per panel (multiple of the k-block)
  uint32_t num_panels = 0;
};
struct PanelReady {
  PanelFlags a, b;
#ifdef __CUDACC__
  __host__ __device__
#endif
  bool on() const { return a.flags || b.flags; }
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
  PanelReady ready;  // 16-bit kinds only
};

// The 16-bit kernel's tile raster for a launch of this shape on the current
// device (host mirror, for ordering panel transfers by when the persistent
// grid first needs them): tile = block_m x block_n, tiles in groups of
// `group` M-blocks (m fastest inside a group), `units` CTA pairs.
struct TcTilePlan {
  uint32_t block_m = 256, block_n = 512, group = 16, units = 74;
};
TcTilePlan tc_tile_plan(uint64_t m, uint64_t n, uint64_t k, int cta_group, int max_ctas);

// 2D tensor map (cuTensorMapEncodeTiled through the runtime's driver entry
// point) of a row-major matrix: inner = columns, outer = rows, pitch in
// elements, box in elements, swizzle 0/32/64/128 bytes. 0 on success.
int encode_map_2d(CUtensorMap* map, const void* ptr, int elem_bytes, uint64_t inner, uint64_t outer,
                  uint64_t pitch_elems, uint32_t box_inner, uint32_t box_outer, int swizzle_bytes);

// Launches on `stream`; returns 0 or 1 with *err set (static string).
int tc_gemm(const TcGemmArgs& args, cudaStream_t stream, const char** err);

}  // namespace gmk
