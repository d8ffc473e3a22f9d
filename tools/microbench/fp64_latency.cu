// FP64 dependent-chain latency on one warp (cycles per op): DFMA, DMUL, sqrt, division, rsqrt,
// shared-memory load, shuffle, __syncthreads (256 threads).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lat(double* out, long long* cyc, double x0, int n) {
  __shared__ double sm[1024];
  __shared__ long long c[8];
  double x = x0 + threadIdx.x * 1e-9;
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = 1.0 + i * 1e-12;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, 0.999999999, 1e-9);
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) x = x * 1.0000000001;
  long long t2 = clock64();
  for (int i = 0; i < n; ++i) x = sqrt(x) + 0.5;
  long long t3 = clock64();
  for (int i = 0; i < n; ++i) x = 1.0 / x + 0.5;
  long long t4 = clock64();
  for (int i = 0; i < n; ++i) x = rsqrt(x) + 0.5;
  long long t5 = clock64();
  int idx = threadIdx.x & 7;
  for (int i = 0; i < n; ++i) { x += sm[idx]; idx = (int)(x * 1e-30) + (threadIdx.x & 7); }
  long long t6 = clock64();
  for (int i = 0; i < n; ++i) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31) + 1e-9;
  long long t7 = clock64();
  for (int i = 0; i < n; ++i) { __syncthreads(); x += 1e-9; }
  long long t8 = clock64();
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4;
    cyc[5] = t6 - t5; cyc[6] = t7 - t6; cyc[7] = t8 - t7;
  }
  out[threadIdx.x] = x;
}

int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 1024 * 8); cudaMallocManaged(&cyc, 8 * 8);
  const int n = 1000;
  const char* names[8] = {"DFMA", "DMUL", "sqrt(f64)", "1/x (f64)", "rsqrt(f64)", "LDS dep", "SHFL", "bar.sync(256)"};
  for (int threads : {32, 256}) {
    lat<<<1, threads>>>(out, cyc, 1.5, n);
    cudaDeviceSynchronize();
    lat<<<1, threads>>>(out, cyc, 1.5, n);
    cudaDeviceSynchronize();
    printf("threads=%d\n", threads);
    for (int k = 0; k < 8; ++k) printf("  %-14s %7.1f cycles/op\n", names[k], (double)cyc[k] / n);
  }
  return 0;
}
