// SPDX-License-Identifier: Apache-2.0
// DMMA issue-rate probe: FP64 mma.sync shapes m8n8k4 / m16n8k4 / m16n8k8 /
// m16n8k16 from registers (no memory traffic), 148 x k CTAs, to size the fp64
// GEMM's inner loop. Prints TFLOP/s per shape.
#include <cstdio>
#include <cuda_runtime.h>

template <int SHAPE>
__global__ void probe(double* out, int iters) {
  double a[8], b[4], c[8][4];
  for (int i = 0; i < 8; ++i) a[i] = 1.0 + threadIdx.x * 1e-9 + i;
  for (int i = 0; i < 4; ++i) b[i] = 1.0 - threadIdx.x * 1e-9 + i;
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 4; ++j) c[i][j] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      if constexpr (SHAPE == 0) {  // m8n8k4: a 1, b 1, c 2
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a[t]), "d"(b[t % 4]));
      } else if constexpr (SHAPE == 1) {  // m16n8k4: a 2, b 1, c 4
        asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                     : "+d"(c[t][0]), "+d"(c[t][1]), "+d"(c[t][2]), "+d"(c[t][3]) : "d"(a[t]), "d"(a[(t + 1) % 8]), "d"(b[t % 4]));
      } else if constexpr (SHAPE == 2) {  // m16n8k8: a 4, b 2, c 4
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+d"(c[t][0]), "+d"(c[t][1]), "+d"(c[t][2]), "+d"(c[t][3])
                     : "d"(a[t]), "d"(a[(t + 1) % 8]), "d"(a[(t + 2) % 8]), "d"(a[(t + 3) % 8]), "d"(b[t % 4]), "d"(b[(t + 1) % 4]));
      } else {  // m16n8k16: a 8, b 4, c 4
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                     : "+d"(c[t][0]), "+d"(c[t][1]), "+d"(c[t][2]), "+d"(c[t][3])
                     : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                       "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
      }
    }
  }
  double s = 0;
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 4; ++j) s += c[i][j];
  if (s == 12345.0) out[threadIdx.x] = s;
}

template <int SHAPE>
void run(const char* name, double flop_per_mma, int warps_per_cta) {
  double* out;
  cudaMalloc(&out, 1 << 20);
  const int iters = 20000, ctas = 148 * 2;
  probe<SHAPE><<<ctas, warps_per_cta * 32>>>(out, 10);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  probe<SHAPE><<<ctas, warps_per_cta * 32>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double flops = flop_per_mma * 8.0 * iters * ctas * warps_per_cta;
  printf("%-10s warps/cta=%2d  %.2f TFLOP/s  (%s)\n", name, warps_per_cta, flops / (ms * 1e-3) / 1e12,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(out);
}

int main() {
  for (int w : {4, 8, 16}) {
    run<0>("m8n8k4", 8 * 8 * 4 * 2, w);
    run<1>("m16n8k4", 16 * 8 * 4 * 2, w);
    run<2>("m16n8k8", 16 * 8 * 8 * 2, w);
    run<3>("m16n8k16", 16 * 8 * 16 * 2, w);
  }
  return 0;
}
