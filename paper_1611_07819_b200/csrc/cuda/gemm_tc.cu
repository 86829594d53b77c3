// SPDX-License-Identifier: Apache-2.0
// Local block GEMM on the 5th-generation tensor cores (sm_100a).
//
//   C[m,n] = alpha * sum_k op(A)[m,k] * op(B)[k,n]  (+ beta * C[m,n])
//
// This is the device replacement of the reference's scalar panel loop
// runGemm<T> (reference proj/src/kernels.cpp:445-558, hot loop :506-519).
// Semantics kept: beta == 0 never reads C (kernels.cpp:463); accumulation
// per output element is one ascending-k chain (kernels.cpp:527-528), here in
// fp32 TMEM with a fixed K=16 MMA step, so results do not depend on how C is
// tiled or distributed (deterministic mode).
//
// Structure (persistent, warp-specialised, one CTA or CTA pair per SM/TPC):
//   warp 0      TMA producer: k-blocks of A and B into a kStages smem ring
//   warp 1      MMA issuer (leader CTA only): tcgen05.mma kind::f16/tf32,
//               fp32 accumulators double-buffered in TMEM (2 x 256 columns)
//   warps 2..5  epilogue: tcgen05.ld TMEM -> registers -> alpha/beta ->
//               convert -> global stores
// A may be K-major (row-major A) or MN-major (transA); B may be MN-major
// (row-major B) or K-major (transB) -- both majors are native to tcgen05 for
// 16-bit and tf32 inputs, so no transpose pass is needed.
// For Single-precision storage the 3xTF32 variant splits A and B into
// hi/lo tf32 pairs (split kernel in convert.cu) and issues hi*lo + lo*hi +
// hi*hi per k-step, which reproduces fp32 GEMM accuracy (~1e-7 rel).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <algorithm>
#include <cstdio>
#include <map>
#include <mutex>
#include <utility>

#include "convert.h"
#include "debug_config.h"
#include "gemm_tc.h"
#include "ptx.cuh"

namespace gmk {

constexpr uint32_t kBlockMcta = 128;  // accumulator rows per CTA (TMEM lanes)
constexpr uint32_t kMmaN = 256;       // N of one tcgen05.mma (TMEM columns per chunk)
constexpr uint32_t kSwizzleBytes = 128;

// Operand element = 2 bytes (kind::f16) or 4 bytes (kind::tf32). A k-block
// is one 128-byte swizzle row: 64 x 16-bit or 32 x 32-bit elements.
// kChunks = UMMAs (N = 256 each) per k-step: the CTA(-pair) tile is
// (128 * kCG) x (256 * kChunks). kChunks = 2 fills all 512 TMEM columns with
// one accumulator (no accumulator double-buffering); kChunks = 1 keeps two
// accumulators so the epilogue of tile t overlaps the MMAs of tile t+1.
template <int kCG, int kElemBytes, int kSplit, int kChunks>
struct TcCfg {
  static constexpr uint32_t kBlockK = kSwizzleBytes / kElemBytes;
  static constexpr uint32_t kMmaK = 32 / kElemBytes;  // 16 (f16) or 8 (tf32)
  static constexpr uint32_t kBlockN = kMmaN * kChunks;  // tile N of the CTA pair
  static constexpr uint32_t kChunkNcta = kMmaN / kCG;   // B columns per CTA per chunk
  static constexpr uint32_t kAccStages = 2 / kChunks;
  static constexpr uint32_t kBytesA = kBlockMcta * kSwizzleBytes;  // per operand part
  static constexpr uint32_t kBytesBChunk = kChunkNcta * kSwizzleBytes;
  static constexpr uint32_t kBytesB = kBytesBChunk * kChunks;
  static constexpr uint32_t kParts = kSplit ? 2 : 1;               // hi (+ lo)
  static constexpr uint32_t kStageBytes = kParts * (kBytesA + kBytesB);
  static constexpr uint32_t kStages = (192u * 1024u) / kStageBytes;
  // Epilogue warps: 8 for the 16-bit kinds (two per TMEM lane quarter, each
  // draining half of the accumulator columns), so the single-buffered wide
  // accumulator -- and a folded k-chunk -- is released twice as fast; 4 (one
  // per quarter) for the tf32 kinds, whose register count leaves no room.
  static constexpr uint32_t kEpiWarps = kElemBytes == 2 ? 8 : 4;
  static constexpr uint32_t kThreads = (2 + kEpiWarps) * 32;
  // Epilogue staging for TMA stores: 32 KB over the epilogue warps.
  static constexpr uint32_t kStagingBytes = 4u * 2u * 4096u;
  static constexpr uint32_t kWarpStaging = kStagingBytes / kEpiWarps;
  static constexpr uint32_t kSmemBytes = kStages * kStageBytes + kStagingBytes + 1024 + 256;
  static constexpr uint32_t kClusterCtas = kCG;
  static_assert(kAccStages * kChunks * kMmaN <= 512, "TMEM columns");
};

struct TcParams {
  uint32_t m, n, k;
  uint32_t a_mn_major, b_mn_major;
  uint32_t idesc;
  float alpha, beta;
  void* c;
  uint64_t ldc;
  uint32_t c_dtype;  // 0 f16, 1 bf16, 2 f32
  uint32_t c_vec;    // 16B vector stores legal
  uint32_t num_m_blocks, num_n_blocks;  // in units of the CTA(-pair) tile
  uint32_t group;                       // raster group (M-blocks)
  uint32_t hint_a, hint_b;              // L2 policy for A / B loads (0 normal, 1 evict_last, 2 evict_first)
  uint32_t* sync_ctr;                   // lockstep counter (a zeroed ring slot) or null
  uint32_t sync_every;                  // k-blocks per lockstep checkpoint
  uint32_t tma_store;                   // C written by TMA stores (beta == 0, aligned C)
  uint32_t fold_kb;                     // k-blocks per folded k-chunk (Single compute), 0 = off
  uint32_t lockstep_data;               // wait at lockstep checkpoints before all panels landed
  // Fused FC forward epilogue (bf16 C only; null = off): bias[col] of the
  // local C columns, act = relu output with pitch ld_act.
  const uint16_t* bias;
  uint16_t* act;
  uint64_t ld_act;
  uint32_t bias_vec, act_vec;           // 16-byte loads / stores legal
  uint32_t act_tma;                     // act written by TMA stores beside C's
  // In-GEMM panel pipelining (the SUMMA exchange lands while the GEMM runs):
  // ready.a[(chunk * num_panels + panel) * streams + s] >= ready.target once
  // pull stream s has copied its pieces of A's (m-chunk, k-panel) block (B:
  // n-chunks). The producer checks the blocks a k-block reads before it
  // loads them. Null flag array: that operand is resident.
  PanelReady ready;
};

// Lockstep: persistent CTA pairs run ~100 tiles back to back and drift apart,
// after which pairs that share a panel no longer read it while it is in L2.
// Every `sync_every` k-blocks the pair leader's producer checks in (always)
// and, while waiting is enabled, waits until all pairs reached the previous
// checkpoint. The wait is bounded (~40 us): a pair whose wait times out
// stops waiting for the rest of its tile, and for the rest of the launch
// after kMaxLockstepTimeouts timeouts -- so a pair that is not resident (SMs
// held by another kernel), a finished tail, or pairs stalled on panel flags
// delay the others boundedly and never block them. Returns false on timeout.
constexpr uint32_t kMaxLockstepTimeouts = 4;
__device__ __forceinline__ bool lockstep(uint32_t* ctr, uint32_t checkpoint, uint32_t units, bool wait) {
  atomicAdd(ctr, 1u);
  if (!wait) return true;
  const uint32_t target = checkpoint * units;
  uint64_t t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
    if (v >= target) return true;
    uint64_t t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    if (t1 - t0 > 40000) return false;
    __nanosleep(64);
  }
}

__device__ __forceinline__ void tile_coords(uint32_t t, const TcParams& p, uint32_t num_n,
                                            uint32_t& mb, uint32_t& nb) {
  // Rasterize in groups of `group` M-blocks (m-fastest inside a group) so the
  // tiles that run concurrently share A and B k-slabs in L2.
  const uint32_t group = p.group;
  const uint32_t per_group = group * num_n;
  const uint32_t g = t / per_group;
  const uint32_t first_m = g * group;
  const uint32_t gsize = min(group, p.num_m_blocks - first_m);
  const uint32_t r = t % per_group;
  mb = first_m + r % gsize;
  nb = r / gsize;
}

// Waits until blocks [c0, c1] x {panel} of one operand have landed, then
// orders the generic-proxy acquire before the async-proxy (TMA) reads of
// the landed bytes.
__device__ __forceinline__ void wait_ready(const PanelFlags& r, uint32_t c0, uint32_t c1, uint32_t panel) {
  for (uint32_t c = c0; c <= c1; ++c) {
    const uint64_t* f = r.flags + static_cast<uint64_t>(c) * r.num_panels + panel;
    for (;;) {
      uint64_t v;
      asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(f) : "memory");
      if (v >= r.target) break;
      __nanosleep(1024);
    }
  }
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

// True once every block of both operands has landed (non-blocking check).
__device__ __forceinline__ bool all_ready(const PanelReady& r) {
  for (int op = 0; op < 2; ++op) {
    const PanelFlags& p = op ? r.b : r.a;
    if (!p.flags) continue;
    const uint32_t n = p.chunks * p.num_panels;
    for (uint32_t i = 0; i < n; ++i) {
      uint64_t v;
      asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p.flags + i) : "memory");
      if (v < p.target) return false;
    }
  }
  return true;
}

__device__ __forceinline__ float load_c(const TcParams& p, uint64_t off) {
  if (p.c_dtype == 2) return reinterpret_cast<const float*>(p.c)[off];
  if (p.c_dtype == 1) return __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(p.c)[off]);
  return __half2float(reinterpret_cast<const __half*>(p.c)[off]);
}

// Replayed `gemm -> biasAdd -> relu` (bf16, Single compute) in one pass:
// each op of the unfused sequence rounds its result to storage precision, so
// z = bf16(float(bf16(x)) + b) and act = z > 0 ? z : 0 exactly as the
// separate ops compute them (reference kernels.cpp:741-815; biasAdd adds in
// float without FMA, relu maps NaN and -0 to +0). f becomes float(z); act is
// written with direct stores (each thread owns 64 contiguous bytes of a row).
// act_out != null: the relu words are returned (staged for a TMA store)
// instead of stored.
__device__ __forceinline__ void bias_relu32(const TcParams& p, uint32_t row, uint32_t col0, float (&f)[32],
                                            uint32_t* act_out = nullptr) {
  const bool full = col0 + 32 <= p.n;
  const bool vec = full && p.bias_vec && p.act_vec;
  uint16_t* dst = p.act + static_cast<uint64_t>(row) * p.ld_act + col0;
  // Eight columns at a time: one 16-byte bias load and one 16-byte act store.
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    uint32_t bw[4];
    if (vec) {
      const uint4 w = __ldg(reinterpret_cast<const uint4*>(p.bias + col0) + g);
      bw[0] = w.x; bw[1] = w.y; bw[2] = w.z; bw[3] = w.w;
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t c = col0 + 8 * g + 2 * j;
        bw[j] = (c < p.n ? p.bias[c] : 0u) | ((c + 1 < p.n ? p.bias[c + 1] : 0u) << 16);
      }
    }
    uint32_t packed[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int i0 = 8 * g + 2 * j;
      const float b0 = __uint_as_float(bw[j] << 16), b1 = __uint_as_float(bw[j] & 0xFFFF0000u);
      const float h0 = __bfloat162float(__float2bfloat16_rn(f[i0]));
      const float h1 = __bfloat162float(__float2bfloat16_rn(f[i0 + 1]));
      f[i0] = __bfloat162float(__float2bfloat16_rn(__fadd_rn(h0, b0)));
      f[i0 + 1] = __bfloat162float(__float2bfloat16_rn(__fadd_rn(h1, b1)));
      const uint32_t lo = f[i0] > 0.0f ? (__float_as_uint(f[i0]) >> 16) : 0u;
      const uint32_t hi = f[i0 + 1] > 0.0f ? (__float_as_uint(f[i0 + 1]) >> 16) : 0u;
      packed[j] = lo | (hi << 16);
    }
    if (act_out) {
#pragma unroll
      for (int j = 0; j < 4; ++j) act_out[4 * g + j] = packed[j];
    } else if (row < p.m) {
      if (vec) {
        reinterpret_cast<uint4*>(dst)[g] = make_uint4(packed[0], packed[1], packed[2], packed[3]);
      } else {
        for (uint32_t i = 0; i < 8 && col0 + 8 * g + i < p.n; ++i)
          dst[8 * g + i] = static_cast<uint16_t>(i & 1 ? packed[i >> 1] >> 16 : packed[i >> 1] & 0xFFFFu);
      }
    }
  }
}

__device__ __forceinline__ void store_row32(const TcParams& p, uint32_t row, uint32_t col0,
                                            const uint32_t (&v)[32], float alpha) {
  if (row >= p.m || col0 >= p.n) return;
  const uint64_t base = static_cast<uint64_t>(row) * p.ldc + col0;
  float f[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) f[i] = alpha * __uint_as_float(v[i]);
  const bool full = col0 + 32 <= p.n;
  if (p.beta != 0.0f) {
    if (full) {
#pragma unroll
      for (int i = 0; i < 32; ++i) f[i] += p.beta * load_c(p, base + i);
    } else {
      for (uint32_t i = 0; i < 32 && col0 + i < p.n; ++i) f[i] += p.beta * load_c(p, base + i);
    }
  }
  if (p.bias) bias_relu32(p, row, col0, f);
  if (full && p.c_vec) {
    if (p.c_dtype == 2) {
      float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(p.c) + base);
#pragma unroll
      for (int i = 0; i < 8; ++i) dst[i] = make_float4(f[4 * i], f[4 * i + 1], f[4 * i + 2], f[4 * i + 3]);
    } else {
      uint32_t packed[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        if (p.c_dtype == 1) {
          __nv_bfloat162 h = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
          packed[i] = *reinterpret_cast<uint32_t*>(&h);
        } else {
          __half2 h = __floats2half2_rn(f[2 * i], f[2 * i + 1]);
          packed[i] = *reinterpret_cast<uint32_t*>(&h);
        }
      }
      uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(p.c) + base);
#pragma unroll
      for (int i = 0; i < 4; ++i)
        dst[i] = make_uint4(packed[4 * i], packed[4 * i + 1], packed[4 * i + 2], packed[4 * i + 3]);
    }
    return;
  }
  for (uint32_t i = 0; i < 32 && col0 + i < p.n; ++i) {
    if (p.c_dtype == 2)
      reinterpret_cast<float*>(p.c)[base + i] = f[i];
    else if (p.c_dtype == 1)
      reinterpret_cast<__nv_bfloat16*>(p.c)[base + i] = __float2bfloat16_rn(f[i]);
    else
      reinterpret_cast<__half*>(p.c)[base + i] = __float2half_rn(f[i]);
  }
}

// kSplit: 3xTF32 (maps a_hi/a_lo, b_hi/b_lo). Otherwise a single pair.
template <int kCG, int kElemBytes, int kSplit, int kChunks>
__global__ void __launch_bounds__(TcCfg<kCG, kElemBytes, kSplit, kChunks>::kThreads, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b,
                   const __grid_constant__ CUtensorMap tm_a_lo,
                   const __grid_constant__ CUtensorMap tm_b_lo,
                   const __grid_constant__ CUtensorMap tm_c,
                   const __grid_constant__ CUtensorMap tm_act, const TcParams p) {
  using Cfg = TcCfg<kCG, kElemBytes, kSplit, kChunks>;
  constexpr uint32_t kStages = Cfg::kStages;
  constexpr uint32_t kBlockK = Cfg::kBlockK;
  constexpr uint32_t kMmaK = Cfg::kMmaK;
  constexpr uint32_t kChunkNcta = Cfg::kChunkNcta;
  constexpr uint32_t kAcc = Cfg::kAccStages;
  constexpr uint32_t kElems128 = kSwizzleBytes / kElemBytes;  // elements per 128B row

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* staging = smem + kStages * Cfg::kStageBytes;  // 1024-aligned (stage bytes are KB multiples)
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(staging + Cfg::kStagingBytes);
  uint64_t* empty_bar = full_bar + kStages;
  uint64_t* tfull_bar = empty_bar + kStages;  // [kAcc]
  uint64_t* tempty_bar = tfull_bar + 2;       // [kAcc]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const uint32_t warp = warp_id_sync();
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t rank = (kCG == 2) ? cluster_ctarank() : 0;  // rank in the UMMA pair
  const bool leader = rank == 0;
  const uint16_t pair_mask = static_cast<uint16_t>((1u << kCG) - 1);

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_a);
    tma_prefetch_desc(&tm_b);
    if (p.tma_store) tma_prefetch_desc(&tm_c);
    if (p.act_tma) tma_prefetch_desc(&tm_act);
    if (kSplit) {
      tma_prefetch_desc(&tm_a_lo);
      tma_prefetch_desc(&tm_b_lo);
    }
    for (uint32_t s = 0; s < kStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (uint32_t a = 0; a < 2; ++a) {  // wide tiles: [0] / [1] = the two accumulator halves
      mbar_init(&tfull_bar[a], 1);
      mbar_init(&tempty_bar[a], Cfg::kEpiWarps * kCG);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<kCG>(tmem_slot, 512);
  if constexpr (kCG == 2) {
    cluster_sync();
  } else {
    __syncthreads();
  }
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // Programmatic dependent launch: this CTA lets the next kernel on the
  // stream be scheduled onto SMs as they free up, and the prologue above
  // (barriers, TMEM, descriptor prefetch) overlapped the previous kernel's
  // tail; global memory is touched only once the previous grid completed.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");

  const uint32_t num_tiles = p.num_m_blocks * p.num_n_blocks;
  const uint32_t num_kb = (p.k + kBlockK - 1) / kBlockK;
  // Fold mode (tf32 kinds, 256-wide tiles): one chunk accumulator plus a
  // running-sum region in TMEM instead of two tile accumulators.
  const bool fold = kChunks == 1 && p.fold_kb > 0;
  const uint32_t unit = blockIdx.x / Cfg::kClusterCtas, num_units = gridDim.x / Cfg::kClusterCtas;

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      uint32_t stage = 0, phase = 0;
      const uint64_t pol_a = l2_policy(static_cast<int>(p.hint_a));
      const uint64_t pol_b = l2_policy(static_cast<int>(p.hint_b));
      const bool synced = p.sync_ctr != nullptr && rank == 0;
      uint32_t timeouts = 0;
      const uint32_t cps_per_tile = synced ? (num_kb + p.sync_every - 1) / p.sync_every : 0;
      const PanelReady& rd = p.ready;
      const uint32_t a_kbp = rd.a.flags ? rd.a.panel_k / kBlockK : 0;  // k-blocks per panel
      const uint32_t b_kbp = rd.b.flags ? rd.b.panel_k / kBlockK : 0;
      // While panels are still landing, pairs stall on data at different
      // times, so a lockstep timeout then says nothing about residency: it
      // ends the wait for the current tile only, and counts towards the
      // launch-wide cut-off once every block has landed. (Not waiting at all
      // during that phase measured worse: the pairs drift apart and lose
      // their L2 reuse -- dependent chain N = 2 26.41 vs 25.77 ms.)
      bool data_done = !rd.on();
      uint32_t local_tile = 0;
      for (uint32_t t = unit; t < num_tiles; t += num_units, ++local_tile) {
        uint32_t mb, nb;
        tile_coords(t, p, p.num_n_blocks, mb, nb);
        const int32_t m0 = static_cast<int32_t>(mb * kBlockMcta * kCG + rank * kBlockMcta);
        if (!data_done) data_done = all_ready(rd);
        bool wait_sync = synced && (data_done || p.lockstep_data) && timeouts < kMaxLockstepTimeouts;
        // Flag blocks this CTA's loads touch: its own 128 rows of A, the
        // tile's columns of B.
        uint32_t ac0 = 0, ac1 = 0, bc0 = 0, bc1 = 0;
        if (rd.a.flags) {
          const uint32_t r1 = min(static_cast<uint32_t>(m0) + kBlockMcta, p.m) - 1;
          ac0 = (rd.a.origin + static_cast<uint32_t>(m0)) / rd.a.chunk;
          ac1 = (rd.a.origin + r1) / rd.a.chunk;
        }
        if (rd.b.flags) {
          const uint32_t c0 = nb * Cfg::kBlockN, c1 = min(c0 + Cfg::kBlockN, p.n) - 1;
          bc0 = (rd.b.origin + c0) / rd.b.chunk;
          bc1 = (rd.b.origin + c1) / rd.b.chunk;
        }
        for (uint32_t kb = 0; kb < num_kb; ++kb) {
          if (synced && kb % p.sync_every == 0 &&
              !lockstep(p.sync_ctr, local_tile * cps_per_tile + kb / p.sync_every, num_units, wait_sync)) {
            wait_sync = false;  // rest of this tile
            if (data_done) ++timeouts;
          }
          if (a_kbp && kb % a_kbp == 0) wait_ready(rd.a, ac0, ac1, kb / a_kbp);
          if (b_kbp && kb % b_kbp == 0) wait_ready(rd.b, bc0, bc1, kb / b_kbp);
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* sa = smem + stage * Cfg::kStageBytes;
          uint8_t* sb = sa + Cfg::kParts * Cfg::kBytesA;
          const int32_t k0 = static_cast<int32_t>(kb * kBlockK);
          // The leader's barrier tracks both CTAs' bytes; the peer's TMA
          // completions land on it directly (2-SM TMA), no peer arrive needed.
          if (leader) mbar_arrive_expect_tx(&full_bar[stage], Cfg::kStageBytes * kCG);
          for (uint32_t part = 0; part < Cfg::kParts; ++part) {
            const CUtensorMap* ma = part ? &tm_a_lo : &tm_a;
            const CUtensorMap* mbm = part ? &tm_b_lo : &tm_b;
            uint8_t* da = sa + part * Cfg::kBytesA;
            uint8_t* db = sb + part * Cfg::kBytesB;
            if (!p.a_mn_major) {
              if (kCG == 2) tma_load_2d_2sm_hint(da, ma, &full_bar[stage], k0, m0, pol_a);
              else tma_load_2d(da, ma, &full_bar[stage], k0, m0);
            } else {
              // MN-major: boxes of (128 B of M) x kBlockK rows of K.
#pragma unroll
              for (uint32_t j = 0; j < kBlockMcta / kElems128; ++j) {
                if (kCG == 2)
                  tma_load_2d_2sm(da + j * kBlockK * kSwizzleBytes, ma, &full_bar[stage], m0 + j * kElems128, k0);
                else
                  tma_load_2d(da + j * kBlockK * kSwizzleBytes, ma, &full_bar[stage], m0 + j * kElems128, k0);
              }
            }
            // B: chunk c of this CTA covers global columns
            // nb*kBlockN + c*256 + rank*kChunkNcta + [0, kChunkNcta).
#pragma unroll
            for (uint32_t c = 0; c < kChunks; ++c) {
              const int32_t n0 = static_cast<int32_t>(nb * Cfg::kBlockN + c * kMmaN + rank * kChunkNcta);
              uint8_t* dc = db + c * Cfg::kBytesBChunk;
              if (p.b_mn_major) {
#pragma unroll
                for (uint32_t j = 0; j < kChunkNcta / kElems128; ++j) {
                  if (kCG == 2)
                    tma_load_2d_2sm_hint(dc + j * kBlockK * kSwizzleBytes, mbm, &full_bar[stage], n0 + j * kElems128, k0, pol_b);
                  else
                    tma_load_2d(dc + j * kBlockK * kSwizzleBytes, mbm, &full_bar[stage], n0 + j * kElems128, k0);
                }
              } else {
                if (kCG == 2) tma_load_2d_2sm(dc, mbm, &full_bar[stage], k0, n0);
                else tma_load_2d(dc, mbm, &full_bar[stage], k0, n0);
              }
            }
          }
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      if (synced) {
        // Finished: release the others' waits. The last pair to finish
        // (nobody waits any more) zeroes the counter for the next launch on
        // the same stream, so launches need no memset in between.
        const uint32_t old = atomicAdd(p.sync_ctr, 1u << 24);
        if ((old >> 24) + 1 == num_units) atomicExch(p.sync_ctr, 0u);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (leader && lane == 0) {
      uint32_t stage = 0, phase = 0, acc = 0, acc_phase = 0;
      // K-major: advance 32 bytes per MMA-K step inside the 128B swizzle row;
      // MN-major: advance (kMmaK rows x 128B).
      const uint32_t a_lbo = p.a_mn_major ? kBlockK * kSwizzleBytes : 16;
      const uint32_t b_lbo = p.b_mn_major ? kBlockK * kSwizzleBytes : 16;
      const uint32_t a_step = p.a_mn_major ? kMmaK * kSwizzleBytes : 32;
      const uint32_t b_step = p.b_mn_major ? kMmaK * kSwizzleBytes : 32;
      uint32_t fq = 0;  // fold mode: k-chunks issued so far
      // Issues k-block kq's UMMAs of chunks [c0, c1) from `stage`.
      auto issue = [&](uint32_t stage_i, uint32_t kq, uint32_t tmem_acc, uint32_t c0, uint32_t c1) {
        const uint32_t sa = smem_u32(smem + stage_i * Cfg::kStageBytes);
        const uint32_t sb = sa + Cfg::kParts * Cfg::kBytesA;
#pragma unroll
        for (uint32_t kk = 0; kk < kBlockK / kMmaK; ++kk) {
          const uint32_t first = (kq | kk) == 0 ? 0u : 1u;
          const uint64_t ah = sdesc_sw128(sa + kk * a_step, a_lbo, 1024);
#pragma unroll
          for (uint32_t c = 0; c < kChunks; ++c) {
            if (c < c0 || c >= c1) continue;
            const uint32_t tmem_d = tmem_acc + c * kMmaN;
            const uint32_t bc = sb + c * Cfg::kBytesBChunk;
            const uint64_t bh = sdesc_sw128(bc + kk * b_step, b_lbo, 1024);
            if constexpr (kSplit) {
              const uint64_t al = sdesc_sw128(sa + Cfg::kBytesA + kk * a_step, a_lbo, 1024);
              const uint64_t bl = sdesc_sw128(bc + Cfg::kBytesB + kk * b_step, b_lbo, 1024);
              mma_tf32<kCG>(tmem_d, al, bh, p.idesc, first);
              mma_tf32<kCG>(tmem_d, ah, bl, p.idesc, 1u);
              mma_tf32<kCG>(tmem_d, ah, bh, p.idesc, 1u);
            } else if constexpr (kElemBytes == 4) {
              mma_tf32<kCG>(tmem_d, ah, bh, p.idesc, first);
            } else {
              mma_f16<kCG>(tmem_d, ah, bh, p.idesc, first);
            }
          }
        }
      };
      auto commit_stage = [&](uint32_t stage_i) {
        if constexpr (kCG == 2) mma_commit_2sm(&empty_bar[stage_i], pair_mask);
        else mma_commit(&empty_bar[stage_i]);
      };
      for (uint32_t t = unit; t < num_tiles; t += num_units) {
        uint32_t kb0 = 0;  // k-blocks already issued for this tile
        if (kChunks == 2 && !fold) {
          // Wide tile: the epilogue frees the accumulator's low half (chunk
          // 0's columns) before the high half, so chunk 0 of the first
          // staged k-blocks starts while chunk 1 is still being drained;
          // each chunk's k order is unchanged (bitwise identical results).
          mbar_wait(&tempty_bar[0], acc_phase ^ 1);
          tc_fence_after();
          const uint32_t ahead = min(kStages, num_kb);
          const uint32_t s0 = stage, ph0 = phase;
          for (uint32_t j = 0; j < ahead; ++j) {
            mbar_wait(&full_bar[stage], phase);
            tc_fence_after();
            issue(stage, j, tmem_base, 0, 1);
            if (++stage == kStages) {
              stage = 0;
              phase ^= 1;
            }
          }
          mbar_wait(&tempty_bar[1], acc_phase ^ 1);
          tc_fence_after();
          stage = s0;
          phase = ph0;
          for (uint32_t j = 0; j < ahead; ++j) {
            issue(stage, j, tmem_base, 1, 2);
            commit_stage(stage);
            if (j + 1 == num_kb) {
              if constexpr (kCG == 2) mma_commit_2sm(&tfull_bar[0], pair_mask);
              else mma_commit(&tfull_bar[0]);
            }
            if (++stage == kStages) {
              stage = 0;
              phase ^= 1;
            }
          }
          kb0 = ahead;
        } else if (!fold) {
          mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
          tc_fence_after();
        }
        const uint32_t tmem_acc = fold ? tmem_base : tmem_base + acc * kChunks * kMmaN;
        for (uint32_t kb = kb0; kb < num_kb; ++kb) {
          const uint32_t kq = fold ? kb % p.fold_kb : kb;  // k-block within the accumulation
          if (fold && kq == 0) {
            mbar_wait(&tempty_bar[0], (fq & 1) ^ 1);  // chunk buffer folded by the epilogue
            tc_fence_after();
          }
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          issue(stage, kq, tmem_acc, 0, kChunks);
          commit_stage(stage);
          if (fold ? (kq + 1 == p.fold_kb || kb + 1 == num_kb) : kb + 1 == num_kb) {
            if constexpr (kCG == 2) mma_commit_2sm(&tfull_bar[fold ? 0 : acc], pair_mask);
            else mma_commit(&tfull_bar[fold ? 0 : acc]);
            if (fold) ++fq;
          }
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (!fold && ++acc == kAcc) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const uint32_t lane_grp = warp & 3;  // TMEM lanes [32*lane_grp, +32)
    const uint32_t ew = warp - 2;        // epilogue warp 0 .. kEpiWarps-1
    uint8_t* stg = staging + ew * Cfg::kWarpStaging;
    // Columns of the tile this warp drains: all of them, or one half when
    // two warps share a lane quarter.
    constexpr uint32_t kCols = Cfg::kBlockN * 4 / Cfg::kEpiWarps;
    const uint32_t col_begin = (ew / 4) * kCols;
    const uint32_t cbytes = p.c_dtype == 2 ? 4 : 2;
    uint32_t acc = 0, acc_phase = 0, iter = 0;
    uint32_t fq = 0;  // fold mode: k-chunks consumed so far
    // Writes 32 columns (c .. c+31 of the tile) of this thread's row:
    // out = alpha_eff * v (+ beta * C), through swizzled smem + TMA store, or
    // direct stores. The smem buffer is reused two slices later, after its
    // TMA store has finished reading it.
    auto emit = [&](uint32_t nb, uint32_t row0, uint32_t row, uint32_t c, const uint32_t (&v)[32],
                    float alpha_eff) {
      if (!p.tma_store) {
        store_row32(p, row, nb * Cfg::kBlockN + c, v, alpha_eff);
        return;
      }
      // A slot holds one slice: 2 KB for 16-bit C, 4 KB for fp32 C or a
      // fused C + act pair; the warp's staging holds `slots` of them (that
      // many stores in flight while the next slice is staged).
      const uint32_t slot_bytes = (p.act_tma || cbytes == 4) ? 4096u : 2048u;
      const uint32_t slots = Cfg::kWarpStaging / slot_bytes;
      uint8_t* buf = stg + (iter % slots) * slot_bytes;
      if (lane == 0 && iter >= slots) {
        if (slots >= 4) bulk_wait_read<3>();
        else if (slots == 2) bulk_wait_read<1>();
        else bulk_wait_read<0>();
      }
      ++iter;
      __syncwarp();
      if (cbytes == 2) {
        // 32 x 64 B rows, 64-byte swizzle: chunk j of row r at (j ^ ((r >> 1) & 3)).
        uint32_t packed[16];
        float xf[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) xf[i] = alpha_eff * __uint_as_float(v[i]);
        if (p.act_tma) {
          uint32_t ap[16];
          bias_relu32(p, row, nb * Cfg::kBlockN + c, xf, ap);
#pragma unroll
          for (uint32_t j = 0; j < 4; ++j) {
            const uint32_t pj = j ^ ((lane >> 1) & 3);
            *reinterpret_cast<uint4*>(buf + 2048 + lane * 64 + pj * 16) =
                make_uint4(ap[4 * j], ap[4 * j + 1], ap[4 * j + 2], ap[4 * j + 3]);
          }
        } else if (p.bias) {
          bias_relu32(p, row, nb * Cfg::kBlockN + c, xf);
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float x0 = xf[2 * i], x1 = xf[2 * i + 1];
          if (p.c_dtype == 1) {
            __nv_bfloat162 h = __floats2bfloat162_rn(x0, x1);
            packed[i] = *reinterpret_cast<uint32_t*>(&h);
          } else {
            __half2 h = __floats2half2_rn(x0, x1);
            packed[i] = *reinterpret_cast<uint32_t*>(&h);
          }
        }
#pragma unroll
        for (uint32_t j = 0; j < 4; ++j) {
          const uint32_t pj = j ^ ((lane >> 1) & 3);
          *reinterpret_cast<uint4*>(buf + lane * 64 + pj * 16) =
              make_uint4(packed[4 * j], packed[4 * j + 1], packed[4 * j + 2], packed[4 * j + 3]);
        }
      } else {
        // 32 x 128 B rows, 128-byte swizzle: chunk j of row r at (j ^ (r & 7)).
#pragma unroll
        for (uint32_t j = 0; j < 8; ++j) {
          const uint32_t pj = j ^ (lane & 7);
          *reinterpret_cast<float4*>(buf + lane * 128 + pj * 16) =
              make_float4(alpha_eff * __uint_as_float(v[4 * j]), alpha_eff * __uint_as_float(v[4 * j + 1]),
                          alpha_eff * __uint_as_float(v[4 * j + 2]), alpha_eff * __uint_as_float(v[4 * j + 3]));
        }
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        tma_store_2d(&tm_c, buf, static_cast<int32_t>(nb * Cfg::kBlockN + c), static_cast<int32_t>(row0));
        if (p.act_tma)
          tma_store_2d(&tm_act, buf + 2048, static_cast<int32_t>(nb * Cfg::kBlockN + c), static_cast<int32_t>(row0));
        bulk_commit();
      }
    };
    auto release = [&](uint32_t a) {
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (kCG == 2 && !leader) mbar_arrive_cluster(&tempty_bar[a], 0);
        else mbar_arrive(&tempty_bar[a]);
      }
    };
    for (uint32_t t = unit; t < num_tiles; t += num_units) {
      uint32_t mb, nb;
      tile_coords(t, p, p.num_n_blocks, mb, nb);
      const uint32_t row0 = mb * kBlockMcta * kCG + rank * kBlockMcta + lane_grp * 32;
      const uint32_t row = row0 + lane;
      if (fold) {
        // k-chunk folding (Single compute): TMEM columns [0, 256) take chunk
        // q's products, [256, 512) hold the running fp32 sum of this thread's
        // row: s = alpha*P_0, then s = fma(alpha, P_q, s) -- one rounding per
        // fixed 256-wide k-chunk instead of the tensor cores' truncating
        // accumulation over all of k. The last chunk writes C.
        const uint32_t lanes = (lane_grp * 32) << 16;
        const uint32_t tchunk = tmem_base + lanes, tsum = tmem_base + lanes + kMmaN;
        const uint32_t nq = (num_kb + p.fold_kb - 1) / p.fold_kb;
        for (uint32_t q = 0; q < nq; ++q, ++fq) {
          mbar_wait(&tfull_bar[0], fq & 1);
          tc_fence_after();
          const bool last = q + 1 == nq;
#pragma unroll 1
          for (uint32_t c = col_begin; c < col_begin + kCols; c += 32) {
            uint32_t v[32], sum[32];
            __syncwarp();
            tmem_ld_32x32b_x32(tchunk + c, v);
            if (q > 0) tmem_ld_32x32b_x32(tsum + c, sum);
            tmem_wait_ld();
            if (c + 32 == col_begin + kCols) release(0);  // this warp's part of the chunk buffer read
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              const float x = __uint_as_float(v[i]);
              sum[i] = __float_as_uint(q > 0 ? __fmaf_rn(p.alpha, x, __uint_as_float(sum[i])) : __fmul_rn(p.alpha, x));
            }
            if (!last) tmem_st_32x32b_x32(tsum + c, sum);
            else emit(nb, row0, row, c, sum, 1.0f);
          }
          if (!last) tmem_wait_st();
        }
        continue;
      }
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      const uint32_t taddr = tmem_base + ((lane_grp * 32) << 16) + acc * kChunks * kMmaN;
      // Slices of 32 columns, the TMEM load of slice s+1 in flight while
      // slice s is converted and stored. TMA-store path: the accumulator is
      // released as soon as the last slice is in registers; the direct path
      // after all stores.
      // Wide tiles drain chunk 0's columns first (released on tempty[0]),
      // then chunk 1's (tempty[1]): the MMA warp restarts chunk 0 early.
      // Each warp takes a quarter-row slice of each chunk.
      constexpr bool kSplitRelease = kChunks == 2;
      constexpr uint32_t kSegs = kSplitRelease ? 2 : 1;
      constexpr uint32_t kSegCols = kSplitRelease ? kMmaN * 4 / Cfg::kEpiWarps : kCols;
      uint32_t va[32], vb[32];
#pragma unroll 1
      for (uint32_t seg = 0; seg < kSegs; ++seg) {
        const uint32_t c_begin = kSplitRelease ? seg * kMmaN + (ew / 4) * kSegCols : col_begin;
        const uint32_t rel = kSplitRelease ? seg : acc;
        __syncwarp();
        tmem_ld_32x32b_x32(taddr + c_begin, va);
        tmem_wait_ld();
#pragma unroll 1
        for (uint32_t c = c_begin; c < c_begin + kSegCols; c += 64) {
          const bool more = c + 64 < c_begin + kSegCols;
          tmem_ld_32x32b_x32(taddr + c + 32, vb);
          emit(nb, row0, row, c, va, p.alpha);
          tmem_wait_ld();
          if (p.tma_store && !more) release(rel);
          if (more) tmem_ld_32x32b_x32(taddr + c + 64, va);
          emit(nb, row0, row, c + 32, vb, p.alpha);
          if (more) tmem_wait_ld();
        }
        if (!p.tma_store) release(rel);
      }
      if (++acc == kAcc) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
    if (p.tma_store && lane == 0) bulk_wait<0>();  // stores complete before smem goes away
  }

  __syncwarp();
  tc_fence_before();
  if constexpr (kCG == 2) {
    cluster_sync();
  } else {
    __syncthreads();
  }
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<kCG>(tmem_base, 512);
  }
}

// ------------------------------------------------------------------ host side

namespace {

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

int make_map_2d(CUtensorMap* map, const void* ptr, CUtensorMapDataType dt, uint32_t esize,
                uint64_t inner, uint64_t outer, uint64_t pitch_elems, uint32_t box_inner,
                uint32_t box_outer, const char** err,
                CUtensorMapSwizzle swizzle = CU_TENSOR_MAP_SWIZZLE_128B) {
  auto fn = encode_fn();
  if (!fn) {
    *err = "cuTensorMapEncodeTiled unavailable";
    return 1;
  }
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {pitch_elems * esize};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  const int promo = debug_config().l2_promo;
  const CUtensorMapL2promotion pr = promo == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
                                    : promo == 64 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                                    : promo == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                                                   : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  CUresult r = fn(map, dt, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle, pr,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    *err = "cuTensorMapEncodeTiled failed (alignment or stride)";
    return 1;
  }
  return 0;
}

}  // namespace

int encode_map_2d(CUtensorMap* map, const void* ptr, int elem_bytes, uint64_t inner, uint64_t outer,
                  uint64_t pitch_elems, uint32_t box_inner, uint32_t box_outer, int swizzle_bytes) {
  const char* err = nullptr;
  const CUtensorMapDataType dt = elem_bytes == 2 ? CU_TENSOR_MAP_DATA_TYPE_UINT16
                                 : elem_bytes == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                                   : CU_TENSOR_MAP_DATA_TYPE_FLOAT64;
  const CUtensorMapSwizzle sw = swizzle_bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                : swizzle_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                : swizzle_bytes == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                                      : CU_TENSOR_MAP_SWIZZLE_NONE;
  return make_map_2d(map, ptr, dt, static_cast<uint32_t>(elem_bytes), inner, outer, pitch_elems, box_inner,
                     box_outer, &err, sw);
}

namespace {

int sm_count(int dev) {
  static int counts[64] = {0};
  if (dev < 0 || dev >= 64) return 148;
  if (!counts[dev]) cudaDeviceGetAttribute(&counts[dev], cudaDevAttrMultiProcessorCount, dev);
  return counts[dev];
}

// Lockstep counter of a stream: launches on one stream never overlap, and
// the last pair of each launch zeroes the counter, so one zeroed counter per
// (device, stream) serves every launch without aliasing (stream ids are
// unique for the process lifetime, cudaStreamGetId).
// cudaStreamGetId invalidates a stream capture in progress (CUDA-graph
// replay, host/capture.hpp): while capturing, the counter is found by the
// stream handle, as the last uncaptured launch on that handle resolved it
// (none yet: no lockstep for this launch).
uint32_t* lockstep_counter(int dev, cudaStream_t stream) {
  static std::mutex mu;
  static std::map<std::pair<int, unsigned long long>, uint32_t*> ctrs;
  static std::map<std::pair<int, cudaStream_t>, uint32_t*> byHandle;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(stream, &cs) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  if (cs != cudaStreamCaptureStatusNone) {
    std::lock_guard<std::mutex> lock(mu);
    auto h = byHandle.find({dev, stream});
    return h == byHandle.end() ? nullptr : h->second;
  }
  unsigned long long sid = 0;
  if (cudaStreamGetId(stream, &sid) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  std::lock_guard<std::mutex> lock(mu);
  auto it = ctrs.find({dev, sid});
  if (it != ctrs.end()) {
    byHandle[{dev, stream}] = it->second;
    return it->second;
  }
  uint32_t* c = nullptr;
  if (cudaMalloc(&c, sizeof(uint32_t)) != cudaSuccess || cudaMemsetAsync(c, 0, sizeof(uint32_t), stream) != cudaSuccess) {
    cudaGetLastError();
    if (c) cudaFree(c);
    return nullptr;
  }
  ctrs[{dev, sid}] = c;
  byHandle[{dev, stream}] = c;
  return c;
}

// Persistent grid = the number of CTAs (CTA pairs) that are co-resident.
template <int kCG, int kElemBytes, int kSplit, int kChunks>
int resident_ctas(int dev) {
  using Cfg = TcCfg<kCG, kElemBytes, kSplit, kChunks>;
  static int resident[64] = {0};
  if (dev < 0 || dev >= 64) return sm_count(dev);
  if (!resident[dev]) {
    auto kern = tc_gemm_kernel<kCG, kElemBytes, kSplit, kChunks>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmemBytes);
    cudaLaunchConfig_t cfg{};
    cfg.blockDim = dim3(Cfg::kThreads, 1, 1);
    cfg.dynamicSmemBytes = Cfg::kSmemBytes;
    cfg.gridDim = dim3(sm_count(dev), 1, 1);
    cudaLaunchAttribute attrs[1];
    attrs[0].id = cudaLaunchAttributeClusterDimension;
    attrs[0].val.clusterDim.x = Cfg::kClusterCtas;
    attrs[0].val.clusterDim.y = 1;
    attrs[0].val.clusterDim.z = 1;
    cfg.attrs = attrs;
    cfg.numAttrs = 1;
    int clusters = 0;
    if (cudaOccupancyMaxActiveClusters(&clusters, kern, &cfg) != cudaSuccess || clusters <= 0) {
      cudaGetLastError();
      clusters = sm_count(dev) / Cfg::kClusterCtas;
    }
    resident[dev] = clusters * Cfg::kClusterCtas;
  }
  return resident[dev];
}

template <int kCG, int kElemBytes, int kSplit, int kChunks>
int launch(const TcOperand& a, const TcOperand& b, const TcOperand* a_lo, const TcOperand* b_lo,
           const TcParams& p0, int max_ctas, cudaStream_t stream, const char** err) {
  using Cfg = TcCfg<kCG, kElemBytes, kSplit, kChunks>;
  const DebugConfig& dbg = debug_config();
  const CUtensorMapDataType dt = kElemBytes == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                                 : CU_TENSOR_MAP_DATA_TYPE_UINT16;
  constexpr uint32_t kChunk = kSwizzleBytes / kElemBytes;
  TcParams p = p0;
  CUtensorMap ma, mb, mal, mbl;
  auto map_a = [&](CUtensorMap* m, const TcOperand& op) {
    // A logical M x K. K-major: stored M rows x K cols; MN-major: K rows x M cols.
    if (!p.a_mn_major) return make_map_2d(m, op.ptr, dt, kElemBytes, p.k, p.m, op.ld, Cfg::kBlockK, kBlockMcta, err);
    return make_map_2d(m, op.ptr, dt, kElemBytes, p.m, p.k, op.ld, kChunk, Cfg::kBlockK, err);
  };
  auto map_b = [&](CUtensorMap* m, const TcOperand& op) {
    // B logical K x N. MN-major: stored K rows x N cols; K-major: N rows x K cols.
    if (p.b_mn_major) return make_map_2d(m, op.ptr, dt, kElemBytes, p.n, p.k, op.ld, kChunk, Cfg::kBlockK, err);
    return make_map_2d(m, op.ptr, dt, kElemBytes, p.k, p.n, op.ld, Cfg::kBlockK, Cfg::kChunkNcta, err);
  };
  if (map_a(&ma, a) || map_b(&mb, b)) return 1;
  if (kSplit) {
    if (map_a(&mal, *a_lo) || map_b(&mbl, *b_lo)) return 1;
  } else {
    mal = ma;
    mbl = mb;
  }
  for (const PanelFlags* f : {&p.ready.a, &p.ready.b})
    if (f->flags && (!f->panel_k || f->panel_k % Cfg::kBlockK || !f->chunk || !f->num_panels)) {
      *err = "tc_gemm: panel flags need panel_k a multiple of the k-block and non-zero chunk sizes";
      return 1;
    }
  p.num_m_blocks = (p.m + kBlockMcta * kCG - 1) / (kBlockMcta * kCG);
  // Raster group 16: an interleaved sweep at 32768^3 measured 12-16 2% faster
  // than 32 (DRAM 84 -> 67 GB).
  p.group = dbg.raster_group > 0 ? static_cast<uint32_t>(dbg.raster_group) : 16u;
  p.hint_a = static_cast<uint32_t>(dbg.hint_a);
  p.hint_b = static_cast<uint32_t>(dbg.hint_b);
  // Lockstep every 8 k-blocks for long-k launches with wide tiles (32768^3:
  // DRAM 67.7 -> 52.8 GB per launch against 16, SM clock under the power
  // cap +2.4%, throughput +0.7%; profiles/r02_kernel.md).
  const uint32_t kblocks = (p.k + Cfg::kBlockK - 1) / Cfg::kBlockK;
  p.sync_every = dbg.tc_sync >= 0 ? static_cast<uint32_t>(dbg.tc_sync) : (kblocks >= 64 && kChunks == 2 ? 8u : 0u);
  p.sync_ctr = nullptr;
  p.lockstep_data = static_cast<uint32_t>(dbg.lockstep_data);
  if (p.group > p.num_m_blocks) p.group = p.num_m_blocks;
  p.num_n_blocks = (p.n + Cfg::kBlockN - 1) / Cfg::kBlockN;
  int dev = 0;
  cudaGetDevice(&dev);
  auto kern = tc_gemm_kernel<kCG, kElemBytes, kSplit, kChunks>;
  cudaLaunchConfig_t cfg{};
  cfg.blockDim = dim3(Cfg::kThreads, 1, 1);
  cfg.dynamicSmemBytes = Cfg::kSmemBytes;
  cfg.stream = stream;
  cudaLaunchAttribute attrs[2];
  attrs[0].id = cudaLaunchAttributeClusterDimension;
  attrs[0].val.clusterDim.x = Cfg::kClusterCtas;
  attrs[0].val.clusterDim.y = 1;
  attrs[0].val.clusterDim.z = 1;
  attrs[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attrs[1].val.programmaticStreamSerializationAllowed = dbg.pdl ? 1 : 0;
  cfg.attrs = attrs;
  cfg.numAttrs = 2;
  const int res = resident_ctas<kCG, kElemBytes, kSplit, kChunks>(dev);
  int ctas = res;
  if (max_ctas > 0 && max_ctas < ctas) ctas = max_ctas;
  ctas = (ctas / Cfg::kClusterCtas) * Cfg::kClusterCtas;
  const int need = static_cast<int>(p.num_n_blocks * p.num_m_blocks) * Cfg::kClusterCtas;
  if (need < ctas) ctas = need;
  cfg.gridDim = dim3(ctas, 1, 1);
  if (p.sync_every > 0) p.sync_ctr = lockstep_counter(dev, stream);
  if (dbg.verbose)
    std::fprintf(stderr, "[gm] tc_gemm cg=%d elem=%d split=%d chunks=%d m=%u n=%u k=%u grid=%d resident=%d stages=%u smem=%u panels=%u\n",
                 kCG, kElemBytes, kSplit, kChunks, p.m, p.n, p.k, ctas, res,
                 Cfg::kStages, Cfg::kSmemBytes, p.ready.a.num_panels + p.ready.b.num_panels);
  CUtensorMap mc = ma;
  {
    const uint32_t cb = p.c_dtype == 2 ? 4 : 2;
    p.tma_store = 0;
    if (dbg.tma_store && p.beta == 0.0f && (reinterpret_cast<uintptr_t>(p.c) % 16) == 0 && (p.ldc * cb) % 16 == 0) {
      const char* e2 = nullptr;
      if (make_map_2d(&mc, p.c, cb == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_UINT16, cb, p.n,
                      p.m, p.ldc, 32, 32, &e2,
                      cb == 4 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B) == 0)
        p.tma_store = 1;
    }
  }
  CUtensorMap mact = mc;
  p.act_tma = 0;
  if (p.tma_store && p.bias && p.act_vec) {
    const char* e2 = nullptr;
    if (make_map_2d(&mact, p.act, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, p.n, p.m, p.ld_act, 32, 32, &e2,
                    CU_TENSOR_MAP_SWIZZLE_64B) == 0)
      p.act_tma = 1;
  }
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, ma, mb, mal, mbl, mc, mact, p);
  count_launch();
  if (e != cudaSuccess) {
    *err = cudaGetErrorString(e);
    return 1;
  }
  return 0;
}

bool wide_tiles(uint64_t m, uint64_t n, uint64_t k, int cg) {
  const int env_chunks = debug_config().tc_chunks;
  if (env_chunks) return env_chunks == 2;
  // k >= 2048: with 8 epilogue warps draining the single accumulator the
  // wide tile beats 256-wide tiles from k = 2048 on (8192^2: 252 vs 266 us),
  // not at 1024 (166 vs 154).
  if (!(k >= 2048 && n > kMmaN)) return false;
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t units = static_cast<uint64_t>(sm_count(dev)) / cg;
  const uint64_t mrows = kBlockMcta * cg;
  auto fill = [&](uint64_t tiles) {
    const uint64_t waves = (tiles + units - 1) / units;
    return static_cast<double>(tiles) / static_cast<double>(waves * units);
  };
  const uint64_t mb = (m + mrows - 1) / mrows;
  const double f_wide = fill(mb * ((n + 2 * kMmaN - 1) / (2 * kMmaN)));
  const double f_narrow = fill(mb * ((n + kMmaN - 1) / kMmaN));
  return !(f_narrow > f_wide + 0.05);
}

}  // namespace

TcTilePlan tc_tile_plan(uint64_t m, uint64_t n, uint64_t k, int cta_group, int max_ctas) {
  const int cg = cta_group == 1 ? 1 : 2;
  int dev = 0;
  cudaGetDevice(&dev);
  const bool wide = wide_tiles(m, n, k, cg);
  TcTilePlan t;
  t.block_m = kBlockMcta * cg;
  t.block_n = wide ? 2 * kMmaN : kMmaN;
  int ctas = cg == 1 ? (wide ? resident_ctas<1, 2, 0, 2>(dev) : resident_ctas<1, 2, 0, 1>(dev))
                     : (wide ? resident_ctas<2, 2, 0, 2>(dev) : resident_ctas<2, 2, 0, 1>(dev));
  if (max_ctas > 0 && max_ctas < ctas) ctas = max_ctas;
  t.units = std::max(1, ctas / cg);
  const uint32_t mblocks = static_cast<uint32_t>((m + t.block_m - 1) / t.block_m);
  const int rg = debug_config().raster_group;
  t.group = std::min(rg > 0 ? static_cast<uint32_t>(rg) : 16u, std::max(1u, mblocks));
  return t;
}

int tc_gemm(const TcGemmArgs& g, cudaStream_t stream, const char** err) {
  TcParams p{};
  p.m = static_cast<uint32_t>(g.m);
  p.n = static_cast<uint32_t>(g.n);
  p.k = static_cast<uint32_t>(g.k);
  p.a_mn_major = g.trans_a ? 1 : 0;
  p.b_mn_major = g.trans_b ? 0 : 1;
  p.alpha = static_cast<float>(g.alpha);
  p.beta = static_cast<float>(g.beta);
  p.c = g.c;
  p.ldc = g.ldc;
  p.c_dtype = g.c_dtype;
  p.ready = g.ready;
  const uint32_t cb = g.c_dtype == 2 ? 4 : 2;
  p.c_vec = ((reinterpret_cast<uintptr_t>(g.c) % 16) == 0 && (g.ldc * cb) % 16 == 0) ? 1 : 0;
  if (g.bias) {
    if (g.c_dtype != 1 || !g.act) {
      *err = "fused bias/relu epilogue needs bf16 C and an output";
      return 1;
    }
    p.bias = static_cast<const uint16_t*>(g.bias);
    p.act = static_cast<uint16_t*>(g.act);
    p.ld_act = g.ld_act;
    p.bias_vec = (reinterpret_cast<uintptr_t>(g.bias) % 16) == 0 ? 1 : 0;
    p.act_vec = ((reinterpret_cast<uintptr_t>(g.act) % 16) == 0 && (g.ld_act * 2) % 16 == 0) ? 1 : 0;
  }
  const int cg = g.cta_group == 1 ? 1 : 2;
  const uint32_t mrows = kBlockMcta * cg;
  if (g.kind == TcKind::F16 || g.kind == TcKind::BF16) {
    const uint32_t fmt = g.kind == TcKind::BF16 ? 1 : 0;
    p.idesc = make_idesc(fmt, fmt, p.a_mn_major, p.b_mn_major, mrows, kMmaN);
    if (g.fold_k) {
      // k-chunk folding (GM_MATH_FOLD): 256-wide tiles, TMEM split into the
      // chunk accumulator and the running sum.
      if (g.fold_k % 64 || g.bias) {
        *err = "tc_gemm: 16-bit fold_k must be a multiple of 64 (and no fused epilogue)";
        return 1;
      }
      p.fold_kb = static_cast<uint32_t>(g.fold_k / 64);  // 64 16-bit elements per k-block
      return cg == 1 ? launch<1, 2, 0, 1>(g.a, g.b, nullptr, nullptr, p, g.max_ctas, stream, err)
                     : launch<2, 2, 0, 1>(g.a, g.b, nullptr, nullptr, p, g.max_ctas, stream, err);
    }
    // Wide tiles (256 x 512 per CTA pair, two UMMAs per k-step) halve the
    // distinct A panels in flight and cut L2->SMEM traffic by a quarter;
    // their single accumulator leaves the epilogue unoverlapped, which only
    // pays off when the k loop is long. Wide tiles are kept only when they
    // fill the persistent grid's waves as well as 256-wide tiles do (a
    // 1024 x 4096 output is 32 wide tiles for 74 pairs: 43% of the SMs; 64
    // narrow tiles fill 86%). Same bits either way.
    const bool wide = wide_tiles(g.m, g.n, g.k, cg);
    if (cg == 1)
      return wide ? launch<1, 2, 0, 2>(g.a, g.b, nullptr, nullptr, p, g.max_ctas, stream, err)
                  : launch<1, 2, 0, 1>(g.a, g.b, nullptr, nullptr, p, g.max_ctas, stream, err);
    return wide ? launch<2, 2, 0, 2>(g.a, g.b, nullptr, nullptr, p, g.max_ctas, stream, err)
                : launch<2, 2, 0, 1>(g.a, g.b, nullptr, nullptr, p, g.max_ctas, stream, err);
  }
  if (g.ready.on()) {
    *err = "tc_gemm: panel flags are consumed by the 16-bit kinds only";
    return 1;
  }
  p.idesc = make_idesc(2, 2, p.a_mn_major, p.b_mn_major, mrows, kMmaN);
  if (g.fold_k) {
    if (g.fold_k % 32) {
      *err = "tc_gemm: fold_k must be a multiple of 32";
      return 1;
    }
    p.fold_kb = static_cast<uint32_t>(g.fold_k / 32);  // 32 tf32 elements per k-block
  }
  if (g.kind == TcKind::TF32)
    return cg == 1 ? launch<1, 4, 0, 1>(g.a, g.b, nullptr, nullptr, p, g.max_ctas, stream, err)
                   : launch<2, 4, 0, 1>(g.a, g.b, nullptr, nullptr, p, g.max_ctas, stream, err);
  return cg == 1 ? launch<1, 4, 1, 1>(g.a, g.b, &g.a_lo, &g.b_lo, p, g.max_ctas, stream, err)
                 : launch<2, 4, 1, 1>(g.a, g.b, &g.a_lo, &g.b_lo, p, g.max_ctas, stream, err);
}

}  // namespace gmk
