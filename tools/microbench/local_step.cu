// Where do the cycles of one local Jacobi rotation step go?  A copy of the step loop of
// hp_jacobi.cu's local_solve (one-barrier form, NT threads) on a random symmetric 64x64
// matrix, with clock64() stamps per phase on warp 0 / lane 0 and on the last warp.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cuda_runtime.h>

constexpr int PS = 64, LS = PS + 1;

__device__ __forceinline__ void circle_pair(int nplayers, int r, int k, int& a, int& b) {
  const int m = nplayers - 1;
  if (k == 0) { a = m; b = r; } else { a = r + k; if (a >= m) a -= m; b = r - k + m; if (b >= m) b -= m; }
}

template <int NT>
__global__ void __launch_bounds__(NT) step_bench(const double* A0, double* out, long long* stamps, int variant) {
  constexpr int NW = NT / 32;
  extern __shared__ double dsm[];
  double* sA[2] = {dsm, dsm + PS * LS};
  double* sW = dsm + 2 * PS * LS;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int e = tid; e < PS * PS; e += NT) {
    const int j = e / PS, i = e % PS;
    sA[0][i * LS + j] = A0[j * PS + i];
    sW[j * LS + i] = (i == j) ? 1.0 : 0.0;
  }
  __syncthreads();
  double* Acur = sA[0];
  double* Anx = sA[1];
  double* Wl = sW;
  long long acc[5] = {0, 0, 0, 0, 0};
  for (int step = 0; step < PS - 1; ++step) {
    long long c0 = clock64();
    int a, b;
    circle_pair(PS, step, lane, a, b);
    const double aii = Acur[a * LS + a], ajj = Acur[b * LS + b], aij = Acur[a * LS + b];
    int r;
    if (variant == 0 || variant == 2 || variant == 4)
      r = fabs(aij) > 1e-300 && fabs(aij) > 1e-16 * sqrt(fabs(aii) * fabs(ajj));
    else
      r = fabs(aij) > 1e-300 && aij * aij > 1e-32 * fabs(aii * ajj);
    double c = 1.0, s = 0.0, t = 0.0;
    if (variant >= 4) {
      const double dd = ajj - aii, a2 = 2.0 * aij;
      const double tt = (dd >= 0.0 ? a2 : -a2) / (fabs(dd) + sqrt(fma(dd, dd, a2 * a2)));
      const double cc = rsqrt(fma(tt, tt, 1.0));
      t = r ? tt : 0.0;
      c = r ? cc : 1.0;
      s = r ? tt * cc : 0.0;
    } else if (r) {
      const double dd = ajj - aii, a2 = 2.0 * aij;
      t = (dd >= 0.0 ? a2 : -a2) / (fabs(dd) + sqrt(fma(dd, dd, a2 * a2)));
      c = rsqrt(fma(t, t, 1.0));
      s = t * c;
    }
    long long c1 = clock64();
    if (variant >= 4) {
      constexpr int NH = 32 / NW;
      int i1s[NH], j1s[NH];
      double cps[NH], sps[NH], v[NH][4];
#pragma unroll
      for (int h = 0; h < NH; ++h) {
        const int P = warp + NW * h;
        cps[h] = __shfl_sync(0xffffffffu, c, P);
        sps[h] = __shfl_sync(0xffffffffu, s, P);
        i1s[h] = __shfl_sync(0xffffffffu, a, P);
        j1s[h] = __shfl_sync(0xffffffffu, b, P);
      }
#pragma unroll
      for (int h = 0; h < NH; ++h) {
        v[h][0] = Acur[i1s[h] * LS + a];
        v[h][1] = Acur[i1s[h] * LS + b];
        v[h][2] = Acur[j1s[h] * LS + a];
        v[h][3] = Acur[j1s[h] * LS + b];
      }
#pragma unroll
      for (int h = 0; h < NH; ++h) {
        const bool dg = (warp + NW * h) == lane;
        const double cp = cps[h], sp = sps[h];
        const double b00 = v[h][0], b01 = v[h][1], b10 = v[h][2], b11 = v[h][3];
        const double m00 = cp * b00 - sp * b10, m01 = cp * b01 - sp * b11;
        const double m10 = sp * b00 + cp * b10, m11 = sp * b01 + cp * b11;
        const double n00 = c * m00 - s * m01, n01 = s * m00 + c * m01;
        const double n10 = c * m10 - s * m11, n11 = s * m10 + c * m11;
        // the pair's own 2x2 block: exact annihilation (b00 = a_ii, b01 = b10 = a_ij, b11 = a_jj)
        const double d00 = b00 - t * b01, d11 = b11 + t * b01, od = r ? 0.0 : b01;
        const int i1 = i1s[h], j1 = j1s[h];
        Anx[i1 * LS + a] = dg ? d00 : n00;
        Anx[i1 * LS + b] = dg ? od : n01;
        Anx[j1 * LS + a] = dg ? od : n10;
        Anx[j1 * LS + b] = dg ? d11 : n11;
      }
    } else if (variant >= 2) {
      constexpr int NH = 32 / NW;
      int i1s[NH], j1s[NH], rps[NH];
      double cps[NH], sps[NH], v[NH][4];
#pragma unroll
      for (int h = 0; h < NH; ++h) {
        const int P = warp + NW * h;
        rps[h] = __shfl_sync(0xffffffffu, r, P);
        cps[h] = __shfl_sync(0xffffffffu, c, P);
        sps[h] = __shfl_sync(0xffffffffu, s, P);
        i1s[h] = __shfl_sync(0xffffffffu, a, P);
        j1s[h] = __shfl_sync(0xffffffffu, b, P);
      }
#pragma unroll
      for (int h = 0; h < NH; ++h) {
        const int P = warp + NW * h;
        const bool dg = (P == lane);
        const int cc0 = dg ? i1s[h] : a, cc1 = dg ? j1s[h] : b;
        v[h][0] = Acur[i1s[h] * LS + cc0];
        v[h][1] = Acur[i1s[h] * LS + cc1];
        v[h][2] = Acur[j1s[h] * LS + cc0];
        v[h][3] = Acur[j1s[h] * LS + cc1];
      }
#pragma unroll
      for (int h = 0; h < NH; ++h) {
        const int P = warp + NW * h;
        const int i1 = i1s[h], j1 = j1s[h];
        double b00 = v[h][0], b01 = v[h][1], b10 = v[h][2], b11 = v[h][3];
        if (P == lane) {
          if (r) {
            Anx[i1 * LS + i1] = b00 - t * b01; Anx[j1 * LS + j1] = b11 + t * b01;
            Anx[i1 * LS + j1] = 0.0; Anx[j1 * LS + i1] = 0.0;
          } else {
            Anx[i1 * LS + i1] = b00; Anx[j1 * LS + j1] = b11; Anx[i1 * LS + j1] = b01; Anx[j1 * LS + i1] = b01;
          }
          continue;
        }
        if (rps[h]) {
          const double cp = cps[h], sp = sps[h];
          const double n00 = cp * b00 - sp * b10, n01 = cp * b01 - sp * b11;
          const double n10 = sp * b00 + cp * b10, n11 = sp * b01 + cp * b11;
          b00 = n00; b01 = n01; b10 = n10; b11 = n11;
        }
        if (r) {
          const double n00 = c * b00 - s * b01, n01 = s * b00 + c * b01;
          const double n10 = c * b10 - s * b11, n11 = s * b10 + c * b11;
          b00 = n00; b01 = n01; b10 = n10; b11 = n11;
        }
        Anx[i1 * LS + a] = b00; Anx[i1 * LS + b] = b01; Anx[j1 * LS + a] = b10; Anx[j1 * LS + b] = b11;
      }
    } else
#pragma unroll
    for (int h = 0; h < 32 / NW; ++h) {
      const int P = warp + NW * h;
      const int rp = __shfl_sync(0xffffffffu, r, P);
      const double cp = __shfl_sync(0xffffffffu, c, P), sp = __shfl_sync(0xffffffffu, s, P);
      const int i1 = __shfl_sync(0xffffffffu, a, P), j1 = __shfl_sync(0xffffffffu, b, P);
      if (P == lane) {
        const double x00 = Acur[i1 * LS + i1], x11 = Acur[j1 * LS + j1], x01 = Acur[i1 * LS + j1];
        if (r) {
          Anx[i1 * LS + i1] = x00 - t * x01; Anx[j1 * LS + j1] = x11 + t * x01;
          Anx[i1 * LS + j1] = 0.0; Anx[j1 * LS + i1] = 0.0;
        } else {
          Anx[i1 * LS + i1] = x00; Anx[j1 * LS + j1] = x11; Anx[i1 * LS + j1] = x01; Anx[j1 * LS + i1] = x01;
        }
        continue;
      }
      double b00 = Acur[i1 * LS + a], b01 = Acur[i1 * LS + b], b10 = Acur[j1 * LS + a], b11 = Acur[j1 * LS + b];
      if (rp) {
        const double n00 = cp * b00 - sp * b10, n01 = cp * b01 - sp * b11;
        const double n10 = sp * b00 + cp * b10, n11 = sp * b01 + cp * b11;
        b00 = n00; b01 = n01; b10 = n10; b11 = n11;
      }
      if (r) {
        const double n00 = c * b00 - s * b01, n01 = s * b00 + c * b01;
        const double n10 = c * b10 - s * b11, n11 = s * b10 + c * b11;
        b00 = n00; b01 = n01; b10 = n10; b11 = n11;
      }
      Anx[i1 * LS + a] = b00; Anx[i1 * LS + b] = b01; Anx[j1 * LS + a] = b10; Anx[j1 * LS + b] = b11;
    }
    long long c2 = clock64();
    if (variant >= 4) {
      constexpr int NR = 64 / NW;
      double wi[NR], wj[NR];
#pragma unroll
      for (int h = 0; h < NR; ++h) {
        wi[h] = Wl[a * LS + warp + NW * h];
        wj[h] = Wl[b * LS + warp + NW * h];
      }
#pragma unroll
      for (int h = 0; h < NR; ++h) {
        Wl[a * LS + warp + NW * h] = c * wi[h] - s * wj[h];
        Wl[b * LS + warp + NW * h] = s * wi[h] + c * wj[h];
      }
    } else if (variant >= 2) {
      if (r) {
        constexpr int NR = 64 / NW;
        double wi[NR], wj[NR];
#pragma unroll
        for (int h = 0; h < NR; ++h) {
          wi[h] = Wl[a * LS + warp + NW * h];
          wj[h] = Wl[b * LS + warp + NW * h];
        }
#pragma unroll
        for (int h = 0; h < NR; ++h) {
          Wl[a * LS + warp + NW * h] = c * wi[h] - s * wj[h];
          Wl[b * LS + warp + NW * h] = s * wi[h] + c * wj[h];
        }
      }
    } else if (r) {
#pragma unroll
      for (int h = 0; h < 64 / NW; ++h) {
        const int row = warp + NW * h;
        const double wi = Wl[a * LS + row], wj = Wl[b * LS + row];
        Wl[a * LS + row] = c * wi - s * wj;
        Wl[b * LS + row] = s * wi + c * wj;
      }
    }
    __syncwarp();
    long long c3 = clock64();
    double* tmp = Acur; Acur = Anx; Anx = tmp;
    __syncthreads();
    long long c4 = clock64();
    acc[0] += c1 - c0; acc[1] += c2 - c1; acc[2] += c3 - c2; acc[3] += c4 - c3; acc[4] += c4 - c0;
  }
  if (lane == 0 && (warp == 0 || warp == NW - 1))
    for (int k = 0; k < 5; ++k) stamps[(warp == 0 ? 0 : 5) + k] = acc[k];
  for (int e = tid; e < PS * PS; e += NT) out[e] = Acur[(e / PS) * LS + e % PS] + Wl[(e / PS) * LS + e % PS];
}


// variant 6: indices computed directly (no shuffles); operands of A and W loaded by every warp
// while warp 0 computes the 32 rotations into a shared table; barrier; update; barrier
template <int NT>
__global__ void __launch_bounds__(NT) step_bench6(const double* A0, double* out, long long* stamps) {
  constexpr int NW = NT / 32, NH = 32 / NW, NR = 64 / NW;
  extern __shared__ double dsm[];
  __shared__ double4 rot[32];   // c, s, t, r
  double* Acur = dsm;
  double* Anx = dsm + PS * LS;
  double* Wl = dsm + 2 * PS * LS;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int e = tid; e < PS * PS; e += NT) {
    const int j = e / PS, i = e % PS;
    Acur[i * LS + j] = A0[j * PS + i];
    Wl[j * LS + i] = (i == j) ? 1.0 : 0.0;
  }
  __syncthreads();
  long long acc[5] = {0, 0, 0, 0, 0};
  for (int step = 0; step < PS - 1; ++step) {
    long long c0 = clock64();
    int a, b;
    circle_pair(PS, step, lane, a, b);
    int i1s[NH], j1s[NH];
    double v[NH][4], wi[NR], wj[NR];
#pragma unroll
    for (int h = 0; h < NH; ++h) circle_pair(PS, step, warp + NW * h, i1s[h], j1s[h]);
#pragma unroll
    for (int h = 0; h < NH; ++h) {
      v[h][0] = Acur[i1s[h] * LS + a];
      v[h][1] = Acur[i1s[h] * LS + b];
      v[h][2] = Acur[j1s[h] * LS + a];
      v[h][3] = Acur[j1s[h] * LS + b];
    }
#pragma unroll
    for (int h = 0; h < NR; ++h) {
      wi[h] = Wl[a * LS + warp + NW * h];
      wj[h] = Wl[b * LS + warp + NW * h];
    }
    if (warp == 0) {
      const double aii = Acur[a * LS + a], ajj = Acur[b * LS + b], aij = Acur[a * LS + b];
      const int r = fabs(aij) > 1e-300 && aij * aij > 1e-32 * fabs(aii * ajj);
      const double dd = ajj - aii, a2 = 2.0 * aij;
      const double tt = (dd >= 0.0 ? a2 : -a2) / (fabs(dd) + sqrt(fma(dd, dd, a2 * a2)));
      const double cc = rsqrt(fma(tt, tt, 1.0));
      rot[lane] = make_double4(r ? cc : 1.0, r ? tt * cc : 0.0, r ? tt : 0.0, r ? 1.0 : 0.0);
    }
    long long c1 = clock64();
    __syncthreads();
    const double4 mine = rot[lane];
    const double c = mine.x, s = mine.y, t = mine.z;
    const bool r = mine.w != 0.0;
    long long c2 = clock64();
#pragma unroll
    for (int h = 0; h < NH; ++h) {
      const bool dg = (warp + NW * h) == lane;
      const double4 rp = rot[warp + NW * h];
      const double cp = rp.x, sp = rp.y;
      const double b00 = v[h][0], b01 = v[h][1], b10 = v[h][2], b11 = v[h][3];
      const double m00 = cp * b00 - sp * b10, m01 = cp * b01 - sp * b11;
      const double m10 = sp * b00 + cp * b10, m11 = sp * b01 + cp * b11;
      const double n00 = c * m00 - s * m01, n01 = s * m00 + c * m01;
      const double n10 = c * m10 - s * m11, n11 = s * m10 + c * m11;
      const double d00 = b00 - t * b01, d11 = b11 + t * b01, od = r ? 0.0 : b01;
      const int i1 = i1s[h], j1 = j1s[h];
      Anx[i1 * LS + a] = dg ? d00 : n00;
      Anx[i1 * LS + b] = dg ? od : n01;
      Anx[j1 * LS + a] = dg ? od : n10;
      Anx[j1 * LS + b] = dg ? d11 : n11;
    }
#pragma unroll
    for (int h = 0; h < NR; ++h) {
      Wl[a * LS + warp + NW * h] = c * wi[h] - s * wj[h];
      Wl[b * LS + warp + NW * h] = s * wi[h] + c * wj[h];
    }
    long long c3 = clock64();
    double* tmp = Acur; Acur = Anx; Anx = tmp;
    __syncthreads();
    long long c4 = clock64();
    acc[0] += c1 - c0; acc[1] += c2 - c1; acc[2] += c3 - c2; acc[3] += c4 - c3; acc[4] += c4 - c0;
  }
  if (lane == 0 && (warp == 0 || warp == NW - 1))
    for (int k = 0; k < 5; ++k) stamps[(warp == 0 ? 0 : 5) + k] = acc[k];
  for (int e = tid; e < PS * PS; e += NT) out[e] = Acur[(e / PS) * LS + e % PS] + Wl[(e / PS) * LS + e % PS];
}

int main() {
  double h[PS * PS];
  srand(1);
  for (int i = 0; i < PS; ++i)
    for (int j = 0; j <= i; ++j) { double v = (double)rand() / RAND_MAX - 0.5; if (i == j) v += 10.0 * (PS - i); h[i * PS + j] = h[j * PS + i] = v; }
  double *dA, *dout; long long* st;
  cudaMalloc(&dA, sizeof(h)); cudaMalloc(&dout, sizeof(h)); cudaMallocManaged(&st, 10 * 8);
  cudaMemcpy(dA, h, sizeof(h), cudaMemcpyHostToDevice);
  const int smem = 3 * PS * LS * 8;
  cudaFuncSetAttribute(step_bench<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(step_bench<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char* nm[5] = {"rotation", "2x2 blocks", "W update", "barrier", "step total"};
  for (int variant = 4; variant < 6; ++variant) {
    for (int rep = 0; rep < 2; ++rep) {
      step_bench<256><<<1, 256, smem>>>(dA, dout, st, variant);
      cudaDeviceSynchronize();
    }
    printf("NT=256 variant %d (cycles per step, warp 0 | last warp)\n", variant);
    for (int k = 0; k < 5; ++k) printf("  %-12s %8.1f | %8.1f\n", nm[k], st[k] / 63.0, st[5 + k] / 63.0);
    for (int rep = 0; rep < 2; ++rep) {
      step_bench<512><<<1, 512, smem>>>(dA, dout, st, variant);
      cudaDeviceSynchronize();
    }
    printf("NT=512 variant %d\n", variant);
    for (int k = 0; k < 5; ++k) printf("  %-12s %8.1f | %8.1f\n", nm[k], st[k] / 63.0, st[5 + k] / 63.0);
  }
  cudaFuncSetAttribute(step_bench6<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(step_bench6<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char* nm6[5] = {"loads+rot", "barrier 1", "update", "barrier 2", "step total"};
  for (int rep = 0; rep < 2; ++rep) { step_bench6<256><<<1, 256, smem>>>(dA, dout, st); cudaDeviceSynchronize(); }
  printf("NT=256 variant 6\n");
  for (int k = 0; k < 5; ++k) printf("  %-12s %8.1f | %8.1f\n", nm6[k], st[k] / 63.0, st[5 + k] / 63.0);
  for (int rep = 0; rep < 2; ++rep) { step_bench6<512><<<1, 512, smem>>>(dA, dout, st); cudaDeviceSynchronize(); }
  printf("NT=512 variant 6\n");
  for (int k = 0; k < 5; ++k) printf("  %-12s %8.1f | %8.1f\n", nm6[k], st[k] / 63.0, st[5 + k] / 63.0);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
