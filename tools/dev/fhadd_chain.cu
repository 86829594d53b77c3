// Micro-probe: cycles per element of an ordered fp32 chain over bf16 values
// in shared memory, one warp: (a) LDS.U16 + FHADD.BF16, (b) LDS.32 + two
// FHADD.BF16 (lo, hi) into one chain, (c) LDS.128 + eight FHADD.BF16.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ float addbf(float s, uint16_t v) {
  asm("add.rn.f32.bf16 %0, %1, %0;" : "+f"(s) : "h"(v));
  return s;
}
__device__ __forceinline__ float addbf2(float s, uint32_t w) {
  uint16_t lo, hi;
  asm("mov.b32 {%0, %1}, %2;" : "=h"(lo), "=h"(hi) : "r"(w));
  return addbf(addbf(s, lo), hi);
}
__global__ void chain_u16(float* out, long long* cyc, int n) {
  __shared__ uint16_t F[256 * 32];
  for (int i = threadIdx.x; i < 256 * 32; i += blockDim.x) F[i] = 0x3f80 + (i & 7);
  __syncthreads();
  float s = 0.f;
  long long t0 = clock64();
  for (int r = 0; r < n / 256; ++r) {
#pragma unroll 1
    for (int r0 = 0; r0 < 256; r0 += 32) {
      uint16_t v[32];
#pragma unroll
      for (int k = 0; k < 32; ++k) v[k] = F[(r0 + k) * 32 + threadIdx.x];
#pragma unroll
      for (int k = 0; k < 32; ++k) s = addbf(s, v[k]);
    }
  }
  long long t1 = clock64();
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void chain_u32(float* out, long long* cyc, int n) {
  __shared__ uint32_t F[128 * 32];
  for (int i = threadIdx.x; i < 128 * 32; i += blockDim.x) F[i] = 0x3f803f80u + (i & 7);
  __syncthreads();
  float s = 0.f;
  long long t0 = clock64();
  for (int r = 0; r < n / 256; ++r) {
#pragma unroll
    for (int k = 0; k < 128; ++k) s = addbf2(s, F[k * 32 + threadIdx.x]);
  }
  long long t1 = clock64();
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void chain_v4(float* out, long long* cyc, int n) {
  __shared__ uint4 F[32 * 32];
  for (int i = threadIdx.x; i < 32 * 32; i += blockDim.x) F[i] = make_uint4(0x3f803f80u, 0x3f813f81u, 0x3f823f82u, i);
  __syncthreads();
  float s = 0.f;
  long long t0 = clock64();
  for (int r = 0; r < n / 256; ++r) {
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      const uint4 w = F[threadIdx.x * 32 + (k ^ (threadIdx.x & 7))];
      s = addbf2(s, w.x); s = addbf2(s, w.y); s = addbf2(s, w.z); s = addbf2(s, w.w);
    }
  }
  long long t1 = clock64();
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
// Event-timed: 128 CTAs (one per SM, like the line-sum kernels), us per launch.
template <typename K>
float timed(K kern, float* out, long long* cyc, int n) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  kern<<<128, 32>>>(out, cyc, n);
  cudaEventRecord(a);
  for (int i = 0; i < 10; ++i) kern<<<128, 32>>>(out, cyc, n);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  return ms * 100.0f;  // us per launch
}
int main() {
  float* out; long long* cyc; long long h;
  cudaMalloc(&out, 4096); cudaMalloc(&cyc, 8);
  const int n = 4096;
  for (int rep = 0; rep < 2; ++rep) {
    chain_u16<<<1, 32>>>(out, cyc, n); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("LDS.U16 + FHADD.BF16: %.2f cycles/element\n", double(h) / n);
    chain_u32<<<1, 32>>>(out, cyc, n); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("LDS.32 + 2 FHADD.BF16: %.2f cycles/element\n", double(h) / n);
    chain_v4<<<1, 32>>>(out, cyc, n); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("LDS.128 + 8 FHADD.BF16: %.2f cycles/element\n", double(h) / n);
  }
  long long h2 = 0;
  float us = timed(chain_v4, out, cyc, n);
  cudaMemcpy(&h2, cyc, 8, cudaMemcpyDeviceToHost);
  printf("128 CTAs LDS.128 chain: %.2f us per launch, %.2f cycles/element by clock64 -> %.2f GHz\n", us,
         double(h2) / n, double(h2) / (us * 1e3));
  us = timed(chain_u16, out, cyc, n);
  cudaMemcpy(&h2, cyc, 8, cudaMemcpyDeviceToHost);
  printf("128 CTAs LDS.U16 chain: %.2f us per launch, %.2f cycles/element by clock64 -> %.2f GHz\n", us,
         double(h2) / n, double(h2) / (us * 1e3));
  return 0;
}
