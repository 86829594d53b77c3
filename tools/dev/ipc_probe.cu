// SPDX-License-Identifier: Apache-2.0
// Dev probe (2 GPUs, 2 processes via fork): CUDA IPC mapping of a peer
// allocation, cross-process ordering with stream memory operations on
// peer-mapped flags (wait on a remote flag; write a remote flag), and
// copy-engine pull bandwidth of strided 2D copies, alone and while a
// persistent kernel occupies every SM of the pulling GPU.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o ipc_probe ipc_probe.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <sys/wait.h>
#include <unistd.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e_ = (x);                                                              \
    if (e_ != cudaSuccess) {                                                           \
      std::fprintf(stderr, "rank %d: %s failed: %s\n", rank, #x, cudaGetErrorString(e_)); \
      std::exit(1);                                                                    \
    }                                                                                  \
  } while (0)

typedef CUresult (*WaitFn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*WriteFn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

__global__ void spin_fill(unsigned* p, size_t n, unsigned v, long long cycles) {
  long long t0 = clock64();
  while (clock64() - t0 < cycles) {
  }
  for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) p[i] = v;
}

__global__ void hog(long long cycles) {
  long long t0 = clock64();
  while (clock64() - t0 < cycles) {
  }
}

struct Msg {
  cudaIpcMemHandle_t data, flags;
};

int main() {
  int p01[2], p10[2];
  if (pipe(p01) || pipe(p10)) return 1;
  const pid_t pid = fork();
  const int rank = pid == 0 ? 1 : 0;
  CK(cudaSetDevice(rank));
  WaitFn waitv = nullptr;
  WriteFn writev = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuStreamWaitValue32", (void**)&waitv, cudaEnableDefault, &q));
  CK(cudaGetDriverEntryPoint("cuStreamWriteValue32", (void**)&writev, cudaEnableDefault, &q));
  int nsm = 0;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, rank));

  const size_t rows = 16384, rowBytes = 32768, pitch = 65536;  // 512 MiB piece of a 1 GiB tile
  const size_t bytes = rows * pitch;
  unsigned *data = nullptr, *flags = nullptr, *dst = nullptr;
  CK(cudaMalloc(&data, bytes));
  CK(cudaMalloc(&flags, 4096));
  CK(cudaMalloc(&dst, rows * rowBytes));
  CK(cudaMemset(data, 0, bytes));
  CK(cudaMemset(flags, 0, 4096));
  CK(cudaDeviceSynchronize());
  Msg mine{}, peer{};
  CK(cudaIpcGetMemHandle(&mine.data, data));
  CK(cudaIpcGetMemHandle(&mine.flags, flags));
  int wfd = rank == 0 ? p01[1] : p10[1], rfd = rank == 0 ? p10[0] : p01[0];
  if (write(wfd, &mine, sizeof mine) != sizeof mine || read(rfd, &peer, sizeof peer) != sizeof peer) return 1;
  unsigned *pdata = nullptr, *pflags = nullptr;
  CK(cudaIpcOpenMemHandle((void**)&pdata, peer.data, cudaIpcMemLazyEnablePeerAccess));
  CK(cudaIpcOpenMemHandle((void**)&pflags, peer.flags, cudaIpcMemLazyEnablePeerAccess));
  cudaStream_t s;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const long long spin = 2000LL * 1000 * 100;  // ~100 ms at ~2 GHz

  // Test 1: producer (rank 0) fills its data after a long spin, then writes
  // its LOCAL flag; consumer (rank 1) waits on the REMOTE flag, then pulls.
  if (rank == 0) {
    spin_fill<<<nsm, 256, 0, s>>>(data, bytes / 4, 0xA5A5A5A5u, spin);
    CK(cudaGetLastError());
    if (writev(s, (CUdeviceptr)flags, 1, 0) != CUDA_SUCCESS) std::printf("rank0 write local flag FAILED\n");
  } else {
    CUresult r = waitv(s, (CUdeviceptr)pflags, 1, CU_STREAM_WAIT_VALUE_GEQ);
    if (r != CUDA_SUCCESS) std::printf("rank1 wait on remote flag FAILED (%d)\n", (int)r);
    CK(cudaMemcpy2DAsync(dst, rowBytes, pdata, pitch, rowBytes, rows, cudaMemcpyDefault, s));
  }
  CK(cudaStreamSynchronize(s));
  if (rank == 1) {
    std::vector<unsigned> h(1024);
    CK(cudaMemcpy(h.data(), dst + (rows * rowBytes / 4) - 1024, 4096, cudaMemcpyDeviceToHost));
    bool ok = true;
    for (unsigned v : h) ok = ok && v == 0xA5A5A5A5u;
    std::printf("test1 wait-on-remote-flag: %s\n", ok ? "PASS" : "FAIL (read stale data)");
  }
  // Test 2: producer writes the consumer's flag REMOTELY; consumer waits locally.
  if (rank == 0) {
    spin_fill<<<nsm, 256, 0, s>>>(data, bytes / 4, 0x5A5A5A5Au, spin);
    if (writev(s, (CUdeviceptr)(pflags + 1), 2, 0) != CUDA_SUCCESS) std::printf("rank0 write remote flag FAILED\n");
  } else {
    if (waitv(s, (CUdeviceptr)(flags + 1), 2, CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
      std::printf("rank1 wait local FAILED\n");
    CK(cudaMemcpy2DAsync(dst, rowBytes, pdata, pitch, rowBytes, rows, cudaMemcpyDefault, s));
  }
  CK(cudaStreamSynchronize(s));
  if (rank == 1) {
    std::vector<unsigned> h(1024);
    CK(cudaMemcpy(h.data(), dst + (rows * rowBytes / 4) - 1024, 4096, cudaMemcpyDeviceToHost));
    bool ok = true;
    for (unsigned v : h) ok = ok && v == 0x5A5A5A5Au;
    std::printf("test2 remote-write/local-wait: %s\n", ok ? "PASS" : "FAIL (read stale data)");
  }
  // Test 3: pull bandwidth, 2D strided (512 MiB), alone and under an SM hog.
  if (rank == 1) {
    for (int it = 0; it < 2; ++it)
      CK(cudaMemcpy2DAsync(dst, rowBytes, pdata, pitch, rowBytes, rows, cudaMemcpyDefault, s));
    CK(cudaEventRecord(e0, s));
    for (int it = 0; it < 5; ++it)
      CK(cudaMemcpy2DAsync(dst, rowBytes, pdata, pitch, rowBytes, rows, cudaMemcpyDefault, s));
    CK(cudaEventRecord(e1, s));
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    std::printf("test3 2D pull alone: %.1f GB/s\n", 5.0 * rows * rowBytes / (ms / 1e3) / 1e9);
    // contiguous
    CK(cudaEventRecord(e0, s));
    for (int it = 0; it < 5; ++it) CK(cudaMemcpyAsync(dst, pdata, rows * rowBytes, cudaMemcpyDefault, s));
    CK(cudaEventRecord(e1, s));
    CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
    std::printf("test3 1D pull alone: %.1f GB/s\n", 5.0 * rows * rowBytes / (ms / 1e3) / 1e9);
    cudaStream_t hs;
    CK(cudaStreamCreateWithFlags(&hs, cudaStreamNonBlocking));
    CK(cudaFuncSetAttribute(hog, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    hog<<<nsm, 128, 200 * 1024, hs>>>(spin * 3);
    CK(cudaGetLastError());
    CK(cudaEventRecord(e0, s));
    for (int it = 0; it < 5; ++it)
      CK(cudaMemcpy2DAsync(dst, rowBytes, pdata, pitch, rowBytes, rows, cudaMemcpyDefault, s));
    CK(cudaEventRecord(e1, s));
    CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
    const bool hogRunning = cudaStreamQuery(hs) == cudaErrorNotReady;
    std::printf("test3 2D pull under SM hog: %.1f GB/s (hog still running: %d)\n",
                5.0 * rows * rowBytes / (ms / 1e3) / 1e9, hogRunning);
    CK(cudaStreamSynchronize(hs));
  }
  // Both sides done before unmapping.
  char c = 0;
  if (write(wfd, &c, 1) != 1 || read(rfd, &c, 1) != 1) return 1;
  CK(cudaIpcCloseMemHandle(pdata));
  CK(cudaIpcCloseMemHandle(pflags));
  if (rank == 0) {
    int st = 0;
    waitpid(pid, &st, 0);
    std::printf("probe done (child status %d)\n", st);
  }
  return 0;
}
