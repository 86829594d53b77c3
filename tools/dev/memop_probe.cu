// Probe: device-side cost of publishing a flag on a stream, between small
// kernels: cuStreamWriteValue64 (default memory barrier) vs a one-thread
// flag kernel (st.release.sys) vs an 8-byte cudaMemcpyAsync, and the cost of
// a 2D copy followed by each.  nvcc -gencode arch=compute_100a,code=sm_100a -O2 memop_probe.cu -o memop_probe
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__global__ void empty_kernel(int* p) {
  if (threadIdx.x == 0 && p) p[0] += 1;
}

__global__ void flag_kernel(unsigned long long* f, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(f), "l"(v) : "memory");
}

typedef CUresult (*WriteFn)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);

int main() {
  cudaSetDevice(0);
  WriteFn w64 = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuStreamWriteValue64", reinterpret_cast<void**>(&w64), cudaEnableDefault, &q);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  int* scratch;
  unsigned long long* flag;
  cudaMalloc(&scratch, 4096);
  cudaMalloc(&flag, 4096);
  void *src, *dst;
  const size_t rows = 256, cols = 8192;  // 2 MiB block, 8 KB rows
  cudaMalloc(&src, rows * cols * 2);
  cudaMalloc(&dst, rows * cols * 2);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int N = 2000;
  auto run = [&](const char* name, auto body) {
    for (int i = 0; i < 50; ++i) body(i);
    cudaStreamSynchronize(s);
    cudaEventRecord(e0, s);
    for (int i = 0; i < N; ++i) body(i);
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%-44s %8.3f us per iteration\n", name, ms * 1000.0f / N);
  };
  unsigned long long v = 1;
  run("kernel", [&](int) { empty_kernel<<<1, 32, 0, s>>>(scratch); });
  run("kernel + writeValue64 (default)", [&](int) {
    empty_kernel<<<1, 32, 0, s>>>(scratch);
    w64(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(flag), ++v, CU_STREAM_WRITE_VALUE_DEFAULT);
  });
  run("kernel + flag kernel (st.release.sys)", [&](int) {
    empty_kernel<<<1, 32, 0, s>>>(scratch);
    flag_kernel<<<1, 1, 0, s>>>(flag, ++v);
  });
  run("kernel + 8-byte D2D memcpy", [&](int) {
    empty_kernel<<<1, 32, 0, s>>>(scratch);
    cudaMemcpyAsync(flag + 1, flag, 8, cudaMemcpyDeviceToDevice, s);
  });
  run("2D copy 2 MiB (8 KB rows)", [&](int) {
    cudaMemcpy2DAsync(dst, cols * 2, src, cols * 2, cols * 2, rows, cudaMemcpyDeviceToDevice, s);
  });
  run("2D copy + writeValue64 (default)", [&](int) {
    cudaMemcpy2DAsync(dst, cols * 2, src, cols * 2, cols * 2, rows, cudaMemcpyDeviceToDevice, s);
    w64(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(flag), ++v, CU_STREAM_WRITE_VALUE_DEFAULT);
  });
  run("2D copy + flag kernel", [&](int) {
    cudaMemcpy2DAsync(dst, cols * 2, src, cols * 2, cols * 2, rows, cudaMemcpyDeviceToDevice, s);
    flag_kernel<<<1, 1, 0, s>>>(flag, ++v);
  });
  run("2D copy + 8-byte D2D memcpy", [&](int) {
    cudaMemcpy2DAsync(dst, cols * 2, src, cols * 2, cols * 2, rows, cudaMemcpyDeviceToDevice, s);
    cudaMemcpyAsync(flag + 1, flag, 8, cudaMemcpyDeviceToDevice, s);
  });
  printf("done\n");
  return 0;
}
