// SPDX-License-Identifier: Apache-2.0
// Per-worker device layer: the pooled HBM arena and the local block GEMM
// driver that picks the tensor-core kernel for a precision combination.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <mutex>
#include <vector>

#include "../../../include/gridmath_b200.h"
#include "core.hpp"
#include "../cuda/gemm_tc.h"

namespace gridmath {

// Throws gridmath::Error with the CUDA message.
void cudaCheck(cudaError_t e, const char* what);

// Pooled device allocator; device twin of PoolAllocator (reference
// proj/include/gridmath/pool.hpp:13-67, proj/src/pool.cpp:29-63): size
// classes (powers of two from 256 B, quarter steps above 1 MiB to bound
// waste on multi-GiB tiles), free lists that are never returned to the
// driver while the arena lives. Frees are stream-ordered: a freed block
// carries an event and the next user of the block waits on it, so a block
// still being read by an in-flight kernel is never overwritten.
class DeviceArena {
 public:
  explicit DeviceArena(int device);
  ~DeviceArena();
  DeviceArena(const DeviceArena&) = delete;
  DeviceArena& operator=(const DeviceArena&) = delete;

  // `stream`: the stream that will first touch the block (waits on the
  // block's release event if it was recycled). With minAge > 0 only blocks
  // freed at least `minAge` epochs before `epoch` are reused (else a new
  // block is allocated): per-op temporaries double-buffer, so the next op
  // can fill its buffer while the current op still reads its own.
  void* alloc(std::uint64_t bytes, cudaStream_t stream, std::uint64_t epoch = 0, std::uint64_t minAge = 0);
  // `stream`: the stream whose pending work last used the block.
  void free(void* p, cudaStream_t stream, std::uint64_t epoch = 0);
  gm_arena_stats stats() const;
  static std::uint64_t sizeClass(std::uint64_t bytes);
  int device() const { return device_; }

 private:
  struct Block {
    void* ptr;
    cudaEvent_t released;
    std::uint64_t epoch;
  };
  int device_;
  mutable std::mutex mu_;
  std::map<std::uint64_t, std::vector<Block>> free_;
  std::map<void*, std::uint64_t> live_;   // ptr -> class
  std::vector<void*> owned_;
  std::vector<cudaEvent_t> eventPool_;
  gm_arena_stats stats_{};
};

// Local GEMM on the current device. Returns the staging workspace it needs.
std::uint64_t gemmWorkspaceBytes(const gm_gemm_desc& d);  // worst case over alignment
std::uint64_t gemmWorkspaceBytes(const gm_gemm_desc& d, const void* a, const void* b);
// Throws gridmath::Error on failure.
// Optional fused epilogue (replayed gemm -> biasAdd -> relu, bf16 C on the
// tcgen05 path): bias = the C tile's n bias columns, act = relu output.
struct BiasReluEpilogue {
  const void* bias = nullptr;
  void* act = nullptr;
  std::uint64_t ldAct = 0;
};
// `ready`: in-GEMM panel pipelining flags (see gmk::PanelReady); only the
// 16-bit tcgen05 path reading both operands in place consumes them
// (gemmConsumesPanelFlags).
bool gemmConsumesPanelFlags(const gm_gemm_desc& d, const void* a, const void* b);
void gemmLocal(const gm_gemm_desc& d, const void* a, const void* b, void* c, void* workspace,
               std::uint64_t workspaceBytes, cudaStream_t stream, const BiasReluEpilogue* ep = nullptr,
               const gmk::PanelReady* ready = nullptr);

}  // namespace gridmath
