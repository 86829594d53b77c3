// SPDX-License-Identifier: Apache-2.0
// Copy-engine probe: peer 2D pulls (GPU1 -> GPU0) of `rows` x `width` bytes
// into a destination with a wider pitch, on 1..4 streams at once (one piece
// per stream), as the replication of a column-block matrix does.
#include <cstdio>
#include <cuda_runtime.h>
#include <vector>

int main() {
  int n = 0;
  cudaGetDeviceCount(&n);
  if (n < 2) { printf("need 2 GPUs\n"); return 0; }
  cudaSetDevice(0);
  cudaDeviceEnablePeerAccess(1, 0);
  cudaSetDevice(1);
  cudaDeviceEnablePeerAccess(0, 0);
  const size_t rows = 9216;
  for (size_t width : {2048, 4096, 8192, 32768}) {
    const int pieces = 4;
    cudaSetDevice(1);
    std::vector<void*> src(pieces);
    for (auto& p : src) cudaMalloc(&p, rows * width);
    cudaSetDevice(0);
    void* dst;
    cudaMalloc(&dst, rows * width * pieces);
    std::vector<cudaStream_t> st(pieces);
    for (auto& s : st) cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int ns : {1, 2, 4}) {
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0, st[0]);
        for (int i = 1; i < ns; ++i) cudaStreamWaitEvent(st[i], e0, 0);
        for (int i = 0; i < pieces; ++i)
          cudaMemcpy2DAsync(static_cast<char*>(dst) + i * width, width * pieces, src[i], width, width, rows,
                            cudaMemcpyDefault, st[i % ns]);
        for (int i = 1; i < ns; ++i) {
          cudaEvent_t j;
          cudaEventCreateWithFlags(&j, cudaEventDisableTiming);
          cudaEventRecord(j, st[i]);
          cudaStreamWaitEvent(st[0], j, 0);
        }
        cudaEventRecord(e1, st[0]);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep) printf("row %6zu B x %zu rows, %d pieces on %d stream(s): %.1f GB/s\n", width, rows, pieces, ns,
                        rows * width * pieces / (ms * 1e-3) / 1e9);
      }
    }
    cudaFree(dst);
    cudaSetDevice(1);
    for (auto& p : src) cudaFree(p);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
