// Micro-probe: cycles per element of an ordered fp32 add chain, one warp
// per SM sub-partition, (a) register operands, (b) LDS.32 operands.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void chain_reg(float* out, long long* cyc, float a, int n) {
  float s = 0.f, v = a;
  long long t0 = clock64();
  for (int i = 0; i < n; i += 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) { s = __fadd_rn(s, v); v = v * 1.0000001f; }
  }
  long long t1 = clock64();
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void chain_pure(float* out, long long* cyc, float a, int n) {
  float s = 0.f;
  long long t0 = clock64();
  for (int i = 0; i < n; i += 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) s = __fadd_rn(s, a + j);
  }
  long long t1 = clock64();
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void chain_lds(float* out, long long* cyc, int n) {
  __shared__ float F[128 * 32];
  for (int i = threadIdx.x; i < 128 * 32; i += blockDim.x) F[i] = 1.0f + i * 1e-3f;
  __syncthreads();
  float s = 0.f;
  long long t0 = clock64();
  for (int r = 0; r < n / 128; ++r) {
#pragma unroll
    for (int k = 0; k < 128; ++k) s = __fadd_rn(s, F[k * 32 + threadIdx.x]);
  }
  long long t1 = clock64();
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  float* out; long long* cyc; long long h;
  cudaMalloc(&out, 4096); cudaMalloc(&cyc, 8);
  const int n = 4096;
  for (int rep = 0; rep < 2; ++rep) {
    chain_pure<<<1, 32>>>(out, cyc, 1.0f, n); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("pure reg chain: %.2f cycles/element\n", double(h) / n);
    chain_reg<<<1, 32>>>(out, cyc, 1.0f, n); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("reg chain + fmul: %.2f cycles/element\n", double(h) / n);
    chain_lds<<<1, 32>>>(out, cyc, n); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("lds chain: %.2f cycles/element\n", double(h) / n);
  }
  return 0;
}
