// SPDX-License-Identifier: Apache-2.0
// C ABI: device layer and layout helpers (include/gridmath_b200.h).
#include <cuda_runtime.h>

#include <string>

#include "../host/core.hpp"
#include "../host/device.hpp"
#include "../cuda/convert.h"
#include "abi_util.hpp"

struct gm_arena {
  explicit gm_arena(int dev) : arena(dev) {}
  gridmath::DeviceArena arena;
};

namespace gridmath::abi {

namespace {
thread_local std::string g_last_error;
}

void setLastError(const std::string& msg) { g_last_error = msg; }
const char* lastErrorCStr() { return g_last_error.c_str(); }

}  // namespace gridmath::abi

using gridmath::abi::guard;

namespace {

cudaStream_t asStream(void* s) { return static_cast<cudaStream_t>(s); }

int fillTiles(const gridmath::Layout& l, gm_tile* out, uint32_t cap, uint32_t* n) {
  if (n) *n = static_cast<uint32_t>(l.tiles.size());
  if (l.tiles.size() > cap) throw gridmath::Error("layout: output capacity too small");
  for (std::size_t i = 0; i < l.tiles.size(); ++i) {
    const auto& e = l.tiles[i].first;
    out[i] = gm_tile{e.rowStart, e.rowCount, e.colStart, e.colCount, l.tiles[i].second.rank};
  }
  return 0;
}

}  // namespace

extern "C" {

const char* gm_last_error(void) { return gridmath::abi::lastErrorCStr(); }

int gm_version(int32_t* major, int32_t* minor) {
  if (major) *major = 0;
  if (minor) *minor = 1;
  return 0;
}

int gm_device_count(int32_t* count) {
  return guard([&] {
    int n = 0;
    gridmath::cudaCheck(cudaGetDeviceCount(&n), "cudaGetDeviceCount");
    *count = n;
  });
}

int gm_device_init(int32_t device) {
  return guard([&] {
    gridmath::cudaCheck(cudaSetDevice(device), "cudaSetDevice");
    gridmath::cudaCheck(cudaFree(nullptr), "context init");
  });
}

int gm_device_synchronize(int32_t device) {
  return guard([&] {
    gridmath::cudaCheck(cudaSetDevice(device), "cudaSetDevice");
    gridmath::cudaCheck(cudaDeviceSynchronize(), "cudaDeviceSynchronize");
  });
}

int gm_arena_create(int32_t device, uint64_t /*slab_bytes*/, gm_arena** out) {
  return guard([&] { *out = new gm_arena(device); });
}

int gm_arena_destroy(gm_arena* arena) {
  return guard([&] { delete arena; });
}

int gm_arena_alloc(gm_arena* arena, uint64_t bytes, void** ptr) {
  return guard([&] { *ptr = arena->arena.alloc(bytes, nullptr); });
}

int gm_arena_free(gm_arena* arena, void* ptr) {
  return guard([&] { arena->arena.free(ptr, nullptr); });
}

int gm_arena_get_stats(const gm_arena* arena, gm_arena_stats* out) {
  return guard([&] { *out = arena->arena.stats(); });
}

int gm_gemm_workspace_size(const gm_gemm_desc* d, uint64_t* bytes) {
  return guard([&] { *bytes = gridmath::gemmWorkspaceBytes(*d); });
}

int gm_gemm_local(const gm_gemm_desc* d, const void* a, const void* b, void* c, void* workspace,
                  uint64_t workspace_bytes, void* stream) {
  return guard([&] { gridmath::gemmLocal(*d, a, b, c, workspace, workspace_bytes, asStream(stream)); });
}

int gm_convert(const void* src, int32_t src_prec, void* dst, int32_t dst_prec, uint64_t count,
               void* stream) {
  return guard([&] {
    gridmath::precisionFromTag(static_cast<uint8_t>(src_prec));
    gridmath::precisionFromTag(static_cast<uint8_t>(dst_prec));
    gridmath::cudaCheck(gmk::convert_rect(src, src_prec, count, dst, dst_prec, count, 1, count,
                                          asStream(stream)),
                        "gm_convert");
  });
}

int gm_copy_rect(const void* src, uint64_t src_ld, void* dst, uint64_t dst_ld, uint64_t rows,
                 uint64_t cols, uint32_t elem_bytes, void* stream) {
  return guard([&] {
    gridmath::cudaCheck(cudaMemcpy2DAsync(dst, dst_ld * elem_bytes, src, src_ld * elem_bytes,
                                          cols * elem_bytes, rows, cudaMemcpyDefault,
                                          asStream(stream)),
                        "gm_copy_rect");
  });
}

int gm_fill_uniform(void* dst, int32_t prec, uint64_t ld, uint64_t r0, uint64_t rows, uint64_t c0,
                    uint64_t cols, uint64_t full_cols, uint64_t seed, double lo, double hi,
                    void* stream) {
  return guard([&] {
    gridmath::precisionFromTag(static_cast<uint8_t>(prec));
    gridmath::cudaCheck(gmk::fill_uniform(dst, prec, ld, r0, rows, c0, cols, full_cols, seed, lo,
                                          hi, asStream(stream)),
                        "gm_fill_uniform");
  });
}

int gm_layout_row_block(uint64_t rows, uint64_t cols, uint32_t workers, gm_tile* out,
                        uint32_t cap, uint32_t* n) {
  return guard([&] {
    fillTiles(gridmath::makeRowBlockLayout(rows, cols, gridmath::makeWorkerGroup(workers)), out, cap, n);
  });
}

int gm_layout_col_block(uint64_t rows, uint64_t cols, uint32_t workers, gm_tile* out,
                        uint32_t cap, uint32_t* n) {
  return guard([&] {
    fillTiles(gridmath::makeColBlockLayout(rows, cols, gridmath::makeWorkerGroup(workers)), out, cap, n);
  });
}

int gm_layout_grid(uint64_t rows, uint64_t cols, uint32_t pr, uint32_t pc, gm_tile* out,
                   uint32_t cap, uint32_t* n) {
  return guard([&] {
    fillTiles(gridmath::makeGridLayout(rows, cols, pr, pc, gridmath::makeWorkerGroup(pr * pc)), out,
              cap, n);
  });
}

int gm_layout_validate(uint64_t rows, uint64_t cols, const gm_tile* tiles, uint32_t n,
                       uint32_t worker_count, int32_t* violation) {
  return guard([&] {
    gridmath::Layout l;
    for (uint32_t i = 0; i < n; ++i)
      l.tiles.push_back({gridmath::TileExtent{tiles[i].row_start, tiles[i].row_count,
                                              tiles[i].col_start, tiles[i].col_count},
                         gridmath::WorkerId{tiles[i].owner}});
    *violation = static_cast<int32_t>(gridmath::validateLayout(rows, cols, l, worker_count).kind);
  });
}

}  // extern "C"
