// SPDX-License-Identifier: Apache-2.0
// Developer overrides, all in one place: read once from the environment
// variable GM_DEBUG_CONFIG, a comma-separated list of key=value pairs, e.g.
//   GM_DEBUG_CONFIG="raster_group=12,tc_chunks=1,verbose=1"
// Unknown keys are an error (reported on stderr once, then ignored). Every
// default is the product setting; nothing on a launch path reads getenv.
#pragma once
#include <cstdint>

namespace gmk {

struct DebugConfig {
  int raster_group = 0;    // tcgen05 GEMM raster group in M-blocks (0 = product default 16)
  int tc_chunks = 0;       // 1 = force 256-wide tiles, 2 = force 256x512 tiles (0 = auto)
  int tc_sync = -1;        // lockstep checkpoint every N k-blocks (0 = off, -1 = auto)
  int tma_store = 1;       // 0 = epilogue writes C with direct stores
  int l2_promo = 128;      // TMA L2 promotion bytes (0, 64, 128, 256)
  int hint_a = 0, hint_b = 0;  // TMA L2 cache hints (0 normal, 1 evict_last, 2 evict_first)
  int panel_flags = 1;     // 0 = GEMM waits for whole bands (no in-kernel panel pipelining)
  int pdl = 1;             // 0 = no programmatic dependent launch between GEMM kernels
  int lockstep_data = 1;   // 0 = pairs do not wait at lockstep checkpoints while panels are landing
  int class_sort = 1;      // 0 = pipelined blocks purely in need order (no older-operand-first)
  int panel_min_gflop = -1;  // pipeline GEMMs of at least this many GFLOP per worker (-1 = 1000)
  int panel_k = 0;         // k elements per pipelined panel (0 = auto)
  int a_chunk_rows = 0;    // pipelined A block rows (0 = auto)
  int b_chunk_cols = 0;    // pipelined B block columns (0 = auto)
  int ready_slots = 0;     // ready-flag ring slots per worker (0 = 65536; small values test reuse)
  int pull_streams = 0;    // copy-engine pull streams per exchange (0 = all)
  int fuse_zero_sums = 1;  // 0 = replay runs setConst(0) x2 before addRowColSum as kernels
  int fuse_epilogue = 1;   // 0 = replay does not fuse gemm -> biasAdd -> relu
  int tf32_chunk = 256;    // Single-compute k-chunk folded into the fp32 running sum
  int lazy_written = 1;
  int war_side = 1;        // 0 = peers' readDone waits go straight onto the mutating stream    // 0 = publish written[slot] flags on the compute stream after every write
  int graph_replay = 0;    // 1 = replays after the first run as one captured CUDA graph
  int verbose = 0;         // 1 = log every GEMM launch configuration to stderr
};

const DebugConfig& debug_config();

}  // namespace gmk
