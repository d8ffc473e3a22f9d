// FP64 throughput probe on sm_100a: DMMA (mma.sync f64) shapes vs scalar DFMA.
// Register-only loops with independent accumulator chains; reports TFLOP/s.
#include <cstdio>
#include <cuda_runtime.h>

#define ITERS 4096
#define CHAINS 4

__global__ void k_m8n8k4(double* out, double seed) {
  double a = seed + threadIdx.x, b = seed * 0.5;
  double c[CHAINS][2] = {};
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int j = 0; j < CHAINS; ++j)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
  }
  double s = 0; for (int j = 0; j < CHAINS; ++j) s += c[j][0] + c[j][1];
  if (s == 1.2345) out[0] = s;
}
__global__ void k_m16n8k4(double* out, double seed) {
  double a0 = seed + threadIdx.x, a1 = seed, b = seed * 0.5;
  double c[CHAINS][4] = {};
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int j = 0; j < CHAINS; ++j)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                   : "+d"(c[j][0]), "+d"(c[j][1]), "+d"(c[j][2]), "+d"(c[j][3]) : "d"(a0), "d"(a1), "d"(b));
  }
  double s = 0; for (int j = 0; j < CHAINS; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  if (s == 1.2345) out[0] = s;
}
__global__ void k_m16n8k8(double* out, double seed) {
  double a0 = seed + threadIdx.x, a1 = seed, a2 = seed * 3, a3 = seed * 4, b0 = seed * 0.5, b1 = seed * 0.25;
  double c[CHAINS][4] = {};
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int j = 0; j < CHAINS; ++j)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+d"(c[j][0]), "+d"(c[j][1]), "+d"(c[j][2]), "+d"(c[j][3])
                   : "d"(a0), "d"(a1), "d"(a2), "d"(a3), "d"(b0), "d"(b1));
  }
  double s = 0; for (int j = 0; j < CHAINS; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  if (s == 1.2345) out[0] = s;
}
__global__ void k_m16n8k16(double* out, double seed) {
  double a[8], b[4];
  for (int i = 0; i < 8; ++i) a[i] = seed * (i + 1) + threadIdx.x;
  for (int i = 0; i < 4; ++i) b[i] = seed * (i + 2);
  double c[CHAINS][4] = {};
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int j = 0; j < CHAINS; ++j)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                   : "+d"(c[j][0]), "+d"(c[j][1]), "+d"(c[j][2]), "+d"(c[j][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0; for (int j = 0; j < CHAINS; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  if (s == 1.2345) out[0] = s;
}
__global__ void k_dfma(double* out, double seed) {
  double x[8];
  for (int i = 0; i < 8; ++i) x[i] = seed + i + threadIdx.x;
  double m = 1.0000001, a = 1e-9;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int j = 0; j < 8; ++j) x[j] = fma(x[j], m, a);
  }
  double s = 0; for (int j = 0; j < 8; ++j) s += x[j];
  if (s == 1.2345) out[0] = s;
}

template <typename K>
void run(const char* name, K kern, double flops_per_warp_iter, int warps_per_block) {
  double* d; cudaMalloc(&d, 8);
  int blocks = 148 * 4;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int w = 0; w < 2; ++w) kern<<<blocks, 32 * warps_per_block>>>(d, 1.0);
  cudaEventRecord(e0);
  const int reps = 5;
  for (int r = 0; r < reps; ++r) kern<<<blocks, 32 * warps_per_block>>>(d, 1.0);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double flops = flops_per_warp_iter * ITERS * (double)blocks * warps_per_block * reps;
  printf("%-10s warps/blk=%2d  %8.2f TFLOP/s  (%s)\n", name, warps_per_block, flops / (ms * 1e-3) / 1e12,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  for (int w : {4, 8, 16}) {
    run("m8n8k4", k_m8n8k4, 2.0 * 8 * 8 * 4 * CHAINS, w);
    run("m16n8k4", k_m16n8k4, 2.0 * 16 * 8 * 4 * CHAINS, w);
    run("m16n8k8", k_m16n8k8, 2.0 * 16 * 8 * 8 * CHAINS, w);
    run("m16n8k16", k_m16n8k16, 2.0 * 16 * 8 * 16 * CHAINS, w);
    run("dfma", k_dfma, 2.0 * 32 * 32, w);
  }
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("clock attr %d kHz\n", clk);
  return 0;
}
