// SPDX-License-Identifier: Apache-2.0
// All-to-all replication probe (single process, every GPU a source and a
// destination at once, as replicateAsync of a block-distributed matrix at
// N = ngpu): each GPU owns a contiguous `piece` bytes and gathers all pieces
// into a full replica. Modes: CE pull (per-source streams), CE push, SM pull
// kernel (16-byte loads from peer memory over NVLink).
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

struct Srcs { const uint4* p[8]; };

__global__ void sm_pull(Srcs s, int n, uint4* dst, size_t piece16) {
  for (int src = 0; src < n; ++src)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < piece16; i += (size_t)gridDim.x * blockDim.x)
      dst[src * piece16 + i] = s.p[src][i];
}

int main(int argc, char** argv) {
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  if (n < 2) { printf("need >= 2 GPUs\n"); return 0; }
  const size_t piece = (argc > 1 ? atol(argv[1]) : 18874368);  // 9216 x 1024 bf16
  for (int a = 0; a < n; ++a) { cudaSetDevice(a); for (int b = 0; b < n; ++b) if (a != b) cudaDeviceEnablePeerAccess(b, 0); }
  cudaGetLastError();
  std::vector<void*> src(n), dst(n);
  std::vector<std::vector<cudaStream_t>> st(n, std::vector<cudaStream_t>(n));
  std::vector<cudaEvent_t> e0(n), e1(n);
  for (int d = 0; d < n; ++d) {
    cudaSetDevice(d);
    CK(cudaMalloc(&src[d], piece));
    CK(cudaMalloc(&dst[d], piece * n));
    cudaMemset(src[d], d, piece);
    for (auto& s : st[d]) cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaEventCreate(&e0[d]); cudaEventCreate(&e1[d]);
  }
  for (int mode = 0; mode < 3; ++mode) {
    for (int rep = 0; rep < 3; ++rep) {
      for (int d = 0; d < n; ++d) { cudaSetDevice(d); cudaDeviceSynchronize(); }
      for (int d = 0; d < n; ++d) { cudaSetDevice(d); cudaEventRecord(e0[d], st[d][0]); }
      for (int d = 0; d < n; ++d) {
        cudaSetDevice(d);
        for (int i = 1; i < n; ++i) cudaStreamWaitEvent(st[d][i], e0[d], 0);
        if (mode == 0) {  // pull: GPU d's streams copy every source's piece into d's replica
          for (int s = 0; s < n; ++s)
            cudaMemcpyAsync((char*)dst[d] + s * piece, src[s], piece, cudaMemcpyDefault, st[d][s]);
        } else if (mode == 1) {  // push: GPU d's streams copy its piece into every replica
          for (int t = 0; t < n; ++t)
            cudaMemcpyAsync((char*)dst[t] + d * piece, src[d], piece, cudaMemcpyDefault, st[d][t]);
        } else {
          Srcs s{};
          for (int k = 0; k < n; ++k) s.p[k] = (const uint4*)src[k];
          sm_pull<<<148 * 4, 512, 0, st[d][0]>>>(s, n, (uint4*)dst[d], piece / 16);
        }
        for (int i = 1; i < n; ++i) { cudaEvent_t j; cudaEventCreateWithFlags(&j, cudaEventDisableTiming); cudaEventRecord(j, st[d][i]); cudaStreamWaitEvent(st[d][0], j, 0); }
        cudaEventRecord(e1[d], st[d][0]);
      }
      float worst = 0;
      for (int d = 0; d < n; ++d) { cudaSetDevice(d); cudaEventSynchronize(e1[d]); float ms; cudaEventElapsedTime(&ms, e0[d], e1[d]); worst = ms > worst ? ms : worst; }
      if (rep == 2)
        printf("n=%d piece %.1f MB %-8s: %.1f us, %.0f GB/s per GPU in (remote bytes)\n", n, piece / 1e6,
               mode == 0 ? "CE pull" : mode == 1 ? "CE push" : "SM pull", worst * 1e3, piece * (n - 1) / (worst * 1e-3) / 1e9);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
