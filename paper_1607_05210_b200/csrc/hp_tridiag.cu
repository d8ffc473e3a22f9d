// K2t -- the leading eigenpairs of a symmetric positive (semi)definite matrix by Householder
// tridiagonalisation, for the large preconditioned eigenproblems H = L^T L of a node POD
// (replaces scipy.linalg.eigh, pod.py:329-331, where the block-Jacobi solve of hp_jacobi.cu needs
// ~11 sweeps x 8 n^3 flops).  Three stages, every one deterministic (no floating-point atomics,
// fixed reduction orders):
//
//   1. sytrd_panel  : H = Q T Q^T.  One cooperative launch per 64-column panel; a column step is
//                     three grid-wide phases -- (P1) the deferred rank-2 corrections give the
//                     current column x, (P2) every column dot A[:, c] . x of the trailing matrix
//                     (HBM/L2-bound: the matrix is symmetric, so the matrix-vector product is a
//                     set of contiguous column dots, each owned by one CTA -- no cross-CTA
//                     partial sums), together with the panel dots V^T x, W^T x, (P3) the
//                     Householder scalars, v, and w = tau (A v - V W^T v - W V^T v).  The
//                     reflector is applied unscaled (v = s x + t e_1), so its norm needs no
//                     phase of its own.  The trailing update A -= V W^T + W V^T is one DMMA
//                     GEMM per panel ([V|W] [W|V]^T, exactly symmetric output).
//   2. tri_*        : eigenvalues >= floor and their eigenvectors of T without any
//                     re-orthogonalisation (MRRR with a single root representation): T - sigma I
//                     = L D L^T with sigma just below lambda_min, so every eigenvalue is defined
//                     to high RELATIVE accuracy by (L, D); differential-qds Sturm counts
//                     (warp-wide multisection), then one twisted factorisation per eigenvalue
//                     with Rayleigh-quotient correction.  Orthogonality is O(u / relgap): the
//                     caller gets the smallest relative gap and falls back to block Jacobi for
//                     clustered spectra.
//   3. back-transform: W = Q Z by compact-WY blocks, T^-1 = striu(V^T V) + diag(1/tau)
//                     (two GEMMs and a 64 x 64 triangular solve per panel).
#include <cooperative_groups.h>

#include <algorithm>
#include <cfloat>
#include <cmath>

#include "hp_common.cuh"

namespace cg = cooperative_groups;

namespace hp {

int gemm_run(bool a_kmajor, bool b_kmajor, int64_t M, int64_t N, int64_t K, VecSet A, VecSet B, bool aligned16,
             double alpha, double beta, double* C, int64_t ldc, const double* row_scale, const double* col_scale,
             const double* col_div, int sym, int b_upper, void* ws, size_t ws_bytes, cudaStream_t st);
size_t gemm_workspace_bytes(int64_t M, int64_t N, int64_t K, int sym, int b_upper);

namespace trd {

constexpr int NB = 64;    // panel width
constexpr int TT = 512;   // threads per CTA of the panel kernel
constexpr int NW = TT / 32;
constexpr unsigned FULL = 0xffffffffu;
constexpr double UNIT = 2.220446049250313e-16;

struct Panel {
  double* A;
  int64_t lda;
  int n;
  double* P;  // [V | W]  (n x 2 NB)
  double* Q;  // [W | V]
  int64_t ldp;
  double* Vall;  // all reflectors (n x n, zero above the unit entries)
  int64_t ldv;
  double* x;
  double* y;
  double* wt;
  double* pxv;
  double* pxw;
  double* red;
  double* d;
  double* e;
  double* tau;
  int j0, j1;
  int per_max;
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}

// block sum in a fixed order; every thread receives it (buf: NW + 1 doubles)
__device__ __forceinline__ double block_sum(double v, double* buf) {
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) buf[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < NW; ++w) s += buf[w];
    buf[NW] = s;
  }
  __syncthreads();
  const double r = buf[NW];
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(TT, 1) sytrd_panel(Panel p) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) unsigned char smraw[];
  const int n = p.n;
  const int nev = (n + 1) & ~1;
  double* xs = reinterpret_cast<double*>(smraw);  // nev + 2
  double* rowV = xs + nev + 2;
  double* rowW = rowV + NB;
  double* cV = rowW + NB;
  double* cW = cV + NB;
  double* scal = cW + NB;    // 16
  double* rbuf = scal + 16;  // 32
  double* part = rbuf + 32;  // NW * per_max
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int G = gridDim.x, cta = blockIdx.x;
  const int sub = lane & 3;
  const int wbase = ((cta * TT + tid) >> 5) * 8;  // first row group of this warp (8 groups of 4 lanes)
  const int wstride = (G * TT) >> 2;
  const int64_t ldp = p.ldp;
  double* Pv = p.P;
  double* Pw = p.P + (int64_t)NB * ldp;
  double* Qw = p.Q;
  double* Qv = p.Q + (int64_t)NB * ldp;
  double tau_prev = 0.0;

  for (int j = p.j0; j <= p.j1; ++j) {
    const int i = j - p.j0;
    // ------------------------------------------------------------------ P1: finish w_{i-1}, column x
    double alpha_p = 0.0;
    if (i > 0) {
      if (warp == 0) {
        double s = 0.0;
        for (int c = lane; c < G; c += 32) s += __ldcg(p.red + c);
        s = warp_sum(s);
        if (lane == 0) scal[5] = -0.5 * tau_prev * s;
      }
      __syncthreads();
      alpha_p = scal[5];
    }
    const bool stop_here = (j == p.j1) && (p.j1 < n - 1);  // panel end: only finish the last w
    if (tid < i) {
      const double vv = __ldcg(Pv + j + (int64_t)tid * ldp);
      double wv;
      if (tid == i - 1)
        wv = __ldcg(p.wt + j) + alpha_p * vv;
      else
        wv = __ldcg(Pw + j + (int64_t)tid * ldp);
      rowV[tid] = vv;
      rowW[tid] = wv;
    }
    __syncthreads();
    for (int rb = j + wbase; rb < n; rb += wstride) {
      const int r = rb + (lane >> 2);
      const bool valid = r < n;
      double acc = 0.0, wfin = 0.0;
      const bool fin = valid && i > 0 && sub == ((i - 1) & 3);
      if (fin) wfin = __ldcg(p.wt + r) + alpha_p * __ldcg(Pv + r + (int64_t)(i - 1) * ldp);
      if (valid && !stop_here) {
        for (int c = sub; c < i; c += 4) {
          const double vv = __ldcg(Pv + r + (int64_t)c * ldp);
          const double ww = (c == i - 1) ? wfin : __ldcg(Pw + r + (int64_t)c * ldp);
          acc = fma(vv, rowW[c], acc);
          acc = fma(ww, rowV[c], acc);
        }
      }
      if (fin) {
        Pw[r + (int64_t)(i - 1) * ldp] = wfin;
        Qw[r + (int64_t)(i - 1) * ldp] = wfin;
      }
      acc += __shfl_xor_sync(FULL, acc, 1);
      acc += __shfl_xor_sync(FULL, acc, 2);
      if (valid && !stop_here && sub == 0) {
        const double a = p.A[r + (int64_t)j * p.lda] - acc;
        if (r == j)
          p.d[j] = a;
        else
          p.x[r] = a;
      }
    }
    if (j == p.j1) break;
    grid.sync();
    // ------------------------------------------------------------------ P2: column dots with x
    const int r0 = (j + 1) & ~1;
    const int len = nev - r0;
    const int nr = n - 1 - j;
    for (int q = tid; q < len; q += TT) {
      const int r = r0 + q;
      xs[q] = (r > j && r < n) ? __ldcg(p.x + r) : 0.0;
    }
    __syncthreads();
    double ss = 0.0;
    for (int q = tid; q < len; q += TT)
      if (r0 + q >= j + 2) ss = fma(xs[q], xs[q], ss);
    const double ssq = block_sum(ss, rbuf);
    const double alpha = xs[j + 1 - r0];
    {
      const int ntask = nr + 2 * i;
      const int per = (ntask + G - 1) / G;
      const int t0 = min(ntask, cta * per), t1 = min(ntask, t0 + per);
      const int len2 = len >> 1;
      const double2* xs2 = reinterpret_cast<const double2*>(xs);
      auto task_ptr = [&](int tk) -> const double2* {
        tk = min(tk, t1 - 1);
        const double* ptr;
        if (tk < nr)
          ptr = p.A + (int64_t)(j + 1 + tk) * p.lda + r0;
        else if (tk < nr + i)
          ptr = Pv + (int64_t)(tk - nr) * ldp + r0;
        else
          ptr = Pw + (int64_t)(tk - nr - i) * ldp + r0;
        return reinterpret_cast<const double2*>(ptr);
      };
      for (int tb = t0; tb < t1; tb += 4) {
        const double2* q0 = task_ptr(tb);
        const double2* q1 = task_ptr(tb + 1);
        const double2* q2 = task_ptr(tb + 2);
        const double2* q3 = task_ptr(tb + 3);
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll 2
        for (int q = tid; q < len2; q += TT) {
          const double2 xv = xs2[q];
          const double2 v0 = __ldcg(q0 + q);
          const double2 v1 = __ldcg(q1 + q);
          const double2 v2 = __ldcg(q2 + q);
          const double2 v3 = __ldcg(q3 + q);
          a0 = fma(v0.x, xv.x, a0);
          a0 = fma(v0.y, xv.y, a0);
          a1 = fma(v1.x, xv.x, a1);
          a1 = fma(v1.y, xv.y, a1);
          a2 = fma(v2.x, xv.x, a2);
          a2 = fma(v2.y, xv.y, a2);
          a3 = fma(v3.x, xv.x, a3);
          a3 = fma(v3.y, xv.y, a3);
        }
        a0 = warp_sum(a0);
        a1 = warp_sum(a1);
        a2 = warp_sum(a2);
        a3 = warp_sum(a3);
        if (lane == 0) {
          double* dst = part + warp * p.per_max + (tb - t0);
          dst[0] = a0;
          if (tb + 1 < t1) dst[1] = a1;
          if (tb + 2 < t1) dst[2] = a2;
          if (tb + 3 < t1) dst[3] = a3;
        }
      }
      __syncthreads();
      for (int k = tid; k < t1 - t0; k += TT) {
        double s = 0.0;
        for (int w = 0; w < NW; ++w) s += part[w * p.per_max + k];
        const int tk = t0 + k;
        if (tk < nr)
          p.y[j + 1 + tk] = s;
        else if (tk < nr + i)
          p.pxv[tk - nr] = s;
        else
          p.pxw[tk - nr - i] = s;
      }
    }
    grid.sync();
    // ------------------------------------------------------------------ P3: reflector, w
    double tau, beta, s, t;
    {
      const double xnorm = sqrt(ssq);
      if (xnorm == 0.0) {
        tau = 0.0;
        beta = alpha;
        s = 0.0;
        t = 0.0;
      } else {
        beta = -copysign(hypot(alpha, xnorm), alpha);
        tau = (beta - alpha) / beta;
        s = 1.0 / (alpha - beta);
        t = -beta * s;
      }
    }
    if (cta == 0 && tid == 0) {
      p.e[j] = beta;
      p.tau[j] = tau;
    }
    if (tid < i) {
      cV[tid] = s * __ldcg(p.pxv + tid) + t * __ldcg(Pv + (j + 1) + (int64_t)tid * ldp);
      cW[tid] = s * __ldcg(p.pxw + tid) + t * __ldcg(Pw + (j + 1) + (int64_t)tid * ldp);
    }
    __syncthreads();
    double pwv = 0.0;
    for (int rb = j + 1 + wbase; rb < n; rb += wstride) {
      const int r = rb + (lane >> 2);
      const bool valid = r < n;
      double acc = 0.0;
      if (valid) {
        for (int c = sub; c < i; c += 4) {
          acc = fma(__ldcg(Pv + r + (int64_t)c * ldp), cW[c], acc);
          acc = fma(__ldcg(Pw + r + (int64_t)c * ldp), cV[c], acc);
        }
      }
      acc += __shfl_xor_sync(FULL, acc, 1);
      acc += __shfl_xor_sync(FULL, acc, 2);
      if (valid && sub == 0) {
        const double v = (tau == 0.0) ? 0.0 : ((r == j + 1) ? 1.0 : s * xs[r - r0]);
        const double av = s * __ldcg(p.y + r) + t * p.A[r + (int64_t)(j + 1) * p.lda];
        const double wtil = tau * (av - acc);
        Pv[r + (int64_t)i * ldp] = v;
        Qv[r + (int64_t)i * ldp] = v;
        p.Vall[r + (int64_t)j * p.ldv] = v;
        p.wt[r] = wtil;
        pwv = fma(wtil, v, pwv);
      }
    }
    const double tot = block_sum(pwv, rbuf);
    if (tid == 0) p.red[cta] = tot;
    tau_prev = tau;
    grid.sync();
  }
}

// ------------------------------------------------------------------------------- tridiagonal stage
// #eigenvalues of L D L^T below x (differential stationary qds transform)
__device__ __forceinline__ int negcount(const double* __restrict__ d, const double* __restrict__ lld, int n, double x,
                                        double pivmin) {
  double t = -x;
  int neg = 0;
  for (int i = 0; i < n - 1; ++i) {
    double dp = d[i] + t;
    if (fabs(dp) < pivmin) dp = -pivmin;
    neg += dp < 0.0;
    t = (t / dp) * lld[i] - x;
  }
  double dp = d[n - 1] + t;
  if (fabs(dp) < pivmin) dp = -pivmin;
  neg += dp < 0.0;
  return neg;
}

// T - shift I = L D L^T, sequential; returns whether every pivot is positive and finite
__device__ bool ldl_factor(const double* a, const double* b, int n, double shift, double* d, double* l, double* ld,
                           double* lld) {
  bool ok = true;
  double di = a[0] - shift;
  for (int i = 0; i < n - 1; ++i) {
    d[i] = di;
    ok = ok && (di > 0.0) && isfinite(di);
    const double li = b[i] / di;
    if (l) l[i] = li;
    if (ld) ld[i] = b[i];
    lld[i] = li * b[i];
    di = (a[i + 1] - shift) - li * b[i];
  }
  d[n - 1] = di;
  ok = ok && (di > 0.0) && isfinite(di);
  return ok;
}

enum { I_SIGMA = 0, I_LMAX, I_LMIN, I_K, I_OK, I_TNORM, I_PIVMIN, I_HI, I_LO, I_MINGAP, I_MAXRES, I_BAD, I_COUNT };

// One CTA of 1024 threads: spectrum bounds, lambda_max / lambda_min by 1025-way multisection on a
// safely definite representation, the count K of eigenvalues >= floor_rel * lambda_max, and the root
// representation T - sigma I = L D L^T with sigma just below lambda_min.
__global__ void __launch_bounds__(1024, 1) tri_prepare(const double* a, const double* b, int n, double floor_rel,
                                                        double* d0, double* lld0, double* d1, double* l1, double* ld1,
                                                        double* lld1, double* info) {
  __shared__ double sh[40];
  __shared__ double bounds[2];
  const int tid = threadIdx.x;
  double gl = DBL_MAX, gu = -DBL_MAX, em = 0.0, tn = 0.0;
  for (int i = tid; i < n; i += 1024) {
    const double el = i > 0 ? fabs(b[i - 1]) : 0.0, er = i < n - 1 ? fabs(b[i]) : 0.0;
    gl = fmin(gl, a[i] - el - er);
    gu = fmax(gu, a[i] + el + er);
    em = fmax(em, er);
    tn = fmax(tn, fmax(fabs(a[i]), er));
  }
  for (int o = 16; o; o >>= 1) {
    gl = fmin(gl, __shfl_xor_sync(FULL, gl, o));
    gu = fmax(gu, __shfl_xor_sync(FULL, gu, o));
    em = fmax(em, __shfl_xor_sync(FULL, em, o));
    tn = fmax(tn, __shfl_xor_sync(FULL, tn, o));
  }
  __shared__ double red[4][32];
  if ((tid & 31) == 0) {
    red[0][tid >> 5] = gl;
    red[1][tid >> 5] = gu;
    red[2][tid >> 5] = em;
    red[3][tid >> 5] = tn;
  }
  __syncthreads();
  if (tid == 0) {
    for (int w = 1; w < 32; ++w) {
      gl = fmin(gl, red[0][w]);
      gu = fmax(gu, red[1][w]);
      em = fmax(em, red[2][w]);
      tn = fmax(tn, red[3][w]);
    }
    const double width = fmax(gu - gl, DBL_MIN);
    const double sigma0 = gl - 0.01 * width - 16.0 * UNIT * tn;
    const double pivmin = DBL_MIN * fmax(1.0, em * em);
    ldl_factor(a, b, n, sigma0, d0, nullptr, nullptr, lld0);
    sh[0] = sigma0;
    sh[1] = pivmin;
    sh[2] = tn;
    sh[3] = (gu - sigma0) * (1.0 + 1e-10) + 16.0 * UNIT * tn;  // upper bound of the shifted spectrum
  }
  __syncthreads();
  const double sigma0 = sh[0], pivmin = sh[1], tnorm = sh[2], top = sh[3];
  double ext[2];
  for (int which = 0; which < 2; ++which) {  // 0: lambda_max (ascending index n-1), 1: lambda_min (index 0)
    const int want = which == 0 ? n - 1 : 0;
    if (tid == 0) {
      bounds[0] = 0.0;
      bounds[1] = top;
    }
    __syncthreads();
    for (int round = 0; round < 7; ++round) {
      const double lo = bounds[0], hi = bounds[1];
      const double step = (hi - lo) / 1025.0;
      const double xq = lo + step * (double)(tid + 1);
      const int c = negcount(d0, lld0, n, xq, pivmin);
      const int cnt = __syncthreads_count(c <= want);  // points at or below the wanted eigenvalue
      if (tid == 0) {
        if (cnt > 0) bounds[0] = lo + step * (double)cnt;
        if (cnt < 1024) bounds[1] = lo + step * (double)(cnt + 1);
      }
      __syncthreads();
    }
    ext[which] = 0.5 * (bounds[0] + bounds[1]) + sigma0;
    __syncthreads();
  }
  const double lam_max = ext[0], lam_min = ext[1];
  const double floor_abs = floor_rel * lam_max;
  if (tid == 0) {
    int K = n;
    if (floor_abs - sigma0 > 0.0) K = n - negcount(d0, lld0, n, floor_abs - sigma0, pivmin);
    double delta = 256.0 * UNIT * tnorm;
    bool ok = false;
    double sigma = 0.0;
    for (int attempt = 0; attempt < 4 && !ok; ++attempt) {
      sigma = lam_min - delta;
      ok = ldl_factor(a, b, n, sigma, d1, l1, ld1, lld1);
      if (!ok) delta *= 8.0;
    }
    info[I_SIGMA] = sigma;
    info[I_LMAX] = lam_max;
    info[I_LMIN] = lam_min;
    info[I_K] = (double)K;
    info[I_OK] = (ok && isfinite(lam_max) && lam_max > 0.0) ? 1.0 : 0.0;
    info[I_TNORM] = tnorm;
    info[I_PIVMIN] = pivmin;
    info[I_HI] = (lam_max - sigma) * (1.0 + 1e-8) + 64.0 * UNIT * tnorm;
    info[I_LO] = 0.25 * delta;
  }
}

// One warp per wanted eigenvalue (descending index k): 32-way multisection on a geometric grid, so
// small eigenvalues are located to the same RELATIVE accuracy as large ones.
__global__ void __launch_bounds__(256) tri_bisect(const double* d, const double* lld, int n, int K, const double* info,
                                                  double* lam_s, double* blo, double* bhi) {
  const int k = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (k >= K) return;
  const int want = n - 1 - k;
  const double pivmin = info[I_PIVMIN];
  double lo = info[I_LO], hi = info[I_HI];
  for (int round = 0; round < 14; ++round) {
    const double lr = log2(hi / lo);
    if (!(lr > 8.0 * UNIT)) break;
    double xq = lo * exp2(lr * (double)(lane + 1) / 33.0);
    xq = fmin(fmax(xq, lo), hi);
    const int c = negcount(d, lld, n, xq, pivmin);
    const unsigned okm = __ballot_sync(FULL, c <= want);
    const int cnt = __popc(okm);
    const double nlo = __shfl_sync(FULL, xq, max(cnt - 1, 0));
    const double nhi = __shfl_sync(FULL, xq, min(cnt, 31));
    if (cnt > 0) lo = nlo;
    if (cnt < 32) hi = nhi;
  }
  if (lane == 0) {
    lam_s[k] = sqrt(lo) * sqrt(hi);
    blo[k] = lo * (1.0 - 64.0 * UNIT);
    bhi[k] = hi * (1.0 + 64.0 * UNIT);
  }
}

// One thread per wanted eigenvalue: twisted factorisation (stationary qds from the top, progressive
// qds from the bottom, twist where |gamma| is smallest), Rayleigh-quotient correction of the
// eigenvalue (at most 3 passes), eigenvector written normalised to column k of Z.
__global__ void __launch_bounds__(32) tri_getvec(const double* __restrict__ d, const double* __restrict__ l,
                                                  const double* __restrict__ ld, const double* __restrict__ lld,
                                                  int n, int K, int64_t kp, const double* info, double* lam_s,
                                                  const double* blo, const double* bhi, double* __restrict__ LP,
                                                  double* __restrict__ UM, double* __restrict__ PP,
                                                  double* __restrict__ Z, int64_t ldz, double* lam_out,
                                                  double* resid) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= K) return;
  const double pivmin = info[I_PIVMIN], sigma = info[I_SIGMA];
  double lam = lam_s[k];
  const double lo = blo[k], hi = bhi[k];
  double* lp = LP + k;
  double* um = UM + k;
  double* pp = PP + k;
  int r = 0;
  double gam = 0.0, ztz = 1.0;
  for (int it = 0; it < 3; ++it) {
    double pcur = d[n - 1] - lam;
    pp[(int64_t)(n - 1) * kp] = pcur;
    for (int i = n - 2; i >= 0; --i) {
      double dm = lld[i] + pcur;
      if (fabs(dm) < pivmin) dm = -pivmin;
      const double tmp = d[i] / dm;
      um[(int64_t)i * kp] = l[i] * tmp;
      pcur = pcur * tmp - lam;
      pp[(int64_t)i * kp] = pcur;
    }
    double s = -lam, sarr = 0.0;
    gam = sarr + pp[0];
    double best = fabs(gam);
    r = 0;
    for (int i = 0; i < n - 1; ++i) {
      double dp = d[i] + s;
      if (fabs(dp) < pivmin) dp = -pivmin;
      const double lpi = ld[i] / dp;
      lp[(int64_t)i * kp] = lpi;
      sarr = s * lpi * l[i];
      s = sarr - lam;
      const double g = sarr + pp[(int64_t)(i + 1) * kp];
      if (fabs(g) < best) {
        best = fabs(g);
        gam = g;
        r = i + 1;
      }
    }
    ztz = 1.0;
    double z = 1.0;
    for (int i = r - 1; i >= 0; --i) {
      z = -lp[(int64_t)i * kp] * z;
      ztz = fma(z, z, ztz);
    }
    z = 1.0;
    for (int i = r; i < n - 1; ++i) {
      z = -um[(int64_t)i * kp] * z;
      ztz = fma(z, z, ztz);
    }
    const double rq = gam / ztz;
    if (it == 2 || !(fabs(rq) > 4.0 * UNIT * fabs(lam))) break;
    const double nl = lam + rq;
    if (!(nl > lo && nl < hi)) break;
    lam = nl;
  }
  const double scale = rsqrt(ztz);
  double* zc = Z + (int64_t)k * ldz;
  zc[r] = scale;
  double z = 1.0;
  for (int i = r - 1; i >= 0; --i) {
    z = -lp[(int64_t)i * kp] * z;
    zc[i] = z * scale;
  }
  z = 1.0;
  for (int i = r; i < n - 1; ++i) {
    z = -um[(int64_t)i * kp] * z;
    zc[i + 1] = z * scale;
  }
  lam_s[k] = lam;
  lam_out[k] = lam + sigma;
  const double res = fabs(gam) * scale / fabs(lam);
  resid[k] = (isfinite(res) && isfinite(scale) && scale > 0.0) ? res : DBL_MAX;
}

// smallest relative gap between consecutive computed eigenvalues, largest relative residual
__global__ void __launch_bounds__(1024, 1) tri_check(const double* lam_s, const double* resid, int K, int n,
                                                     double* lam_out, double* info) {
  __shared__ double r0[32], r1[32];
  const int tid = threadIdx.x;
  double mg = DBL_MAX, mr = 0.0;
  for (int k = tid; k < K; k += 1024) {
    if (k + 1 < K) mg = fmin(mg, fabs(lam_s[k] - lam_s[k + 1]) / fabs(lam_s[k]));
    mr = fmax(mr, resid[k]);
  }
  for (int k = K + tid; k < n; k += 1024) lam_out[k] = 0.0;
  for (int o = 16; o; o >>= 1) {
    mg = fmin(mg, __shfl_xor_sync(FULL, mg, o));
    mr = fmax(mr, __shfl_xor_sync(FULL, mr, o));
  }
  if ((tid & 31) == 0) {
    r0[tid >> 5] = mg;
    r1[tid >> 5] = mr;
  }
  __syncthreads();
  if (tid == 0) {
    for (int w = 1; w < 32; ++w) {
      mg = fmin(mg, r0[w]);
      mr = fmax(mr, r1[w]);
    }
    info[I_MINGAP] = mg;
    info[I_MAXRES] = mr;
    info[I_BAD] = (mr == DBL_MAX || !(mg == mg)) ? 1.0 : 0.0;
  }
}

// ------------------------------------------------------------------------------- back-transform
// S = V_b^T V_b  ->  T^-1 = striu(S) + diag(1 / tau)   (tau = 0: the reflector is the identity)
__global__ void tinv_build(double* S, int lds, const double* tau, int nb) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nb * nb) return;
  const int i = e % nb, c = e / nb;
  if (i > c)
    S[i + c * lds] = 0.0;
  else if (i == c)
    S[i + c * lds] = tau[i] != 0.0 ? 1.0 / tau[i] : 1.0;
}

// Y <- T Y, i.e. solve the upper-triangular T^-1 Y' = Y; one thread per column of Y
__global__ void __launch_bounds__(128) trsm_tinv(const double* Tinv, int ldt, int nb, double* Y, int ldy, int K) {
  __shared__ double ts[NB * NB];
  for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) ts[e] = Tinv[(e % nb) + (e / nb) * ldt];
  __syncthreads();
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= K) return;
  double* y = Y + (int64_t)k * ldy;
  for (int i = nb - 1; i >= 0; --i) {
    double s = y[i];
    for (int c = i + 1; c < nb; ++c) s = fma(-ts[i + c * nb], y[c], s);
    y[i] = s / ts[i + i * nb];
  }
}

__global__ void copy_in(const double* H, int64_t ldh, int n, double* A, int64_t lda) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= lda * (int64_t)n) return;
  const int64_t r = e % lda, c = e / lda;
  A[e] = r < n ? H[r + c * ldh] : 0.0;
}

}  // namespace trd

static size_t al256(size_t x) { return (x + 255) & ~size_t(255); }

int64_t syev_tri_max_order() { return 24000; }

size_t syev_tri_workspace_bytes(int64_t n) {
  using namespace trd;
  if (n <= 0) return 256;
  const int64_t lda = (n + 1) & ~int64_t(1);
  size_t o = 0;
  o += 2 * al256((size_t)lda * n * 8);        // A, Vall
  o += 2 * al256((size_t)lda * 2 * NB * 8);   // P, Q
  o += 20 * al256((size_t)(n + 2) * 8);       // vectors
  o += 4 * al256(1024 * 8);                   // pxv, pxw, red, info
  o += 3 * al256((size_t)lda * n * 8);        // LP, UM, PP
  o += al256((size_t)NB * n * 8) + al256((size_t)NB * NB * 8);  // Y, S
  size_t g = gemm_workspace_bytes(n, n, 2 * NB, 1, 0);
  g = std::max(g, gemm_workspace_bytes(NB, n, n, 0, 0));
  g = std::max(g, gemm_workspace_bytes(n, n, NB, 0, 0));
  g = std::max(g, gemm_workspace_bytes(NB, NB, n, 0, 0));
  o += al256(g) + 256;
  return o;
}

// Eigenpairs of the symmetric positive semidefinite H (n x n) with lambda >= floor_rel * lambda_max:
// lam_desc[0..K) descending (the rest zeroed), eigenvectors in the first K columns of W (n x n).
// status_out: 0 = done; 1 = declined (clustered spectrum, relative gap below relgap_min, or no
// definite root representation) -- W / lam_desc are then not meaningful and the caller falls back
// to hp_syev.  diag (nullable, host, 4 doubles): min relative gap, max relative residual, sigma, K.
int syev_tri_run(const double* H, int64_t ldh, int64_t n64, double floor_rel, double relgap_min, double* lam_desc,
                 double* W, int64_t ldw, int64_t* k_out, int* status_out, double* diag, void* ws, size_t ws_bytes,
                 cudaStream_t st) {
  using namespace trd;
  HP_REQUIRE(n64 >= 2 && n64 <= syev_tri_max_order(), "syev_tri: order out of range");
  HP_REQUIRE(ws_bytes >= syev_tri_workspace_bytes(n64), "syev_tri: workspace too small");
  HP_REQUIRE(ldw >= n64 && ldw % 2 == 0, "syev_tri: ldw must be even and >= n");
  const int n = (int)n64;
  const int64_t lda = (n64 + 1) & ~int64_t(1);
  *k_out = 0;
  *status_out = 1;
  char* base = static_cast<char*>(ws);
  size_t o = 0;
  auto take = [&](size_t bytes) {
    char* ptr = base + o;
    o += al256(bytes);
    return reinterpret_cast<double*>(ptr);
  };
  double* A = take((size_t)lda * n * 8);
  double* Vall = take((size_t)lda * n * 8);
  double* P = take((size_t)lda * 2 * NB * 8);
  double* Q = take((size_t)lda * 2 * NB * 8);
  double* vec[20];
  for (auto& v : vec) v = take((size_t)(n + 2) * 8);
  double *x = vec[0], *y = vec[1], *wt = vec[2], *dT = vec[3], *eT = vec[4], *tau = vec[5], *d0 = vec[6],
         *lld0 = vec[7], *d1 = vec[8], *l1 = vec[9], *ld1 = vec[10], *lld1 = vec[11], *lam_s = vec[12],
         *blo = vec[13], *bhi = vec[14], *resid = vec[15];
  double* pxv = take(1024 * 8);
  double* pxw = take(1024 * 8);
  double* red = take(1024 * 8);
  double* info = take(1024 * 8);
  double* LP = take((size_t)lda * n * 8);
  double* UM = take((size_t)lda * n * 8);
  double* PP = take((size_t)lda * n * 8);
  double* Y = take((size_t)NB * n * 8);
  double* S = take((size_t)NB * NB * 8);
  void* gws = base + o;
  const size_t gwsb = ws_bytes - o;

  copy_in<<<(unsigned)ceil_div(lda * n, 256), 256, 0, st>>>(H, ldh, n, A, lda);
  HP_CHECK_LAUNCH("tri copy_in");
  HP_CHECK_CUDA(zero_async(Vall, (size_t)lda * n * 8, st));
  HP_CHECK_CUDA(zero_async(P, (size_t)lda * 2 * NB * 8, st));
  HP_CHECK_CUDA(zero_async(Q, (size_t)lda * 2 * NB * 8, st));
  HP_CHECK_CUDA(zero_async(x, (size_t)(n + 2) * 8, st));
  HP_CHECK_CUDA(zero_async(y, (size_t)(n + 2) * 8, st));
  HP_CHECK_CUDA(zero_async(wt, (size_t)(n + 2) * 8, st));
  count_launches(6);

  int nsm = num_sms();
  const int G = std::max(1, std::min(nsm, 1024));
  const int per_max = (int)ceil_div((int64_t)n + 2 * NB, G) + 4;
  const int nev = (n + 1) & ~1;
  const size_t smem = (size_t)(nev + 2 + 4 * NB + 16 + 32 + (size_t)NW * per_max) * 8;
  HP_REQUIRE(smem <= 220 * 1024, "syev_tri: order too large for the panel kernel");
  static std::atomic<unsigned long long> configured{0};
  const int rc0 = once_per_device(configured, []() -> int {
    HP_CHECK_CUDA(cudaFuncSetAttribute(sytrd_panel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    return (int)HP_OK;
  });
  if (rc0 != HP_OK) return rc0;
  int per_sm = 0;
  HP_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void*)sytrd_panel, TT, smem));
  HP_REQUIRE(per_sm >= 1, "syev_tri: the panel kernel does not fit on an SM");

  Panel p{};
  p.A = A;
  p.lda = lda;
  p.n = n;
  p.P = P;
  p.Q = Q;
  p.ldp = lda;
  p.Vall = Vall;
  p.ldv = lda;
  p.x = x;
  p.y = y;
  p.wt = wt;
  p.pxv = pxv;
  p.pxw = pxw;
  p.red = red;
  p.d = dT;
  p.e = eT;
  p.tau = tau;
  p.per_max = per_max;
  for (int j0 = 0; j0 < n - 1;) {
    const int j1 = std::min(j0 + NB, n - 1);
    p.j0 = j0;
    p.j1 = j1;
    void* args[] = {&p};
    HP_CHECK_CUDA(cudaLaunchCooperativeKernel((void*)sytrd_panel, G, TT, args, smem, st));
    count_launches(1);
    if (j1 < n - 1) {
      // trailing update A[j1:, j1:] -= [V | W] [W | V]^T  (lower tiles computed, mirrored)
      const int64_t n1 = n - j1;
      VecSet pa{P + j1, lda, nullptr};
      VecSet qb{Q + j1, lda, nullptr};
      const int rc = gemm_run(false, false, n1, n1, 2 * NB, pa, qb, true, -1.0, 1.0, A + j1 + (int64_t)j1 * lda, lda,
                              nullptr, nullptr, nullptr, 1, 0, gws, gwsb, st);
      if (rc) return rc;
    }
    j0 = j1;
  }

  tri_prepare<<<1, 1024, 0, st>>>(dT, eT, n, floor_rel, d0, lld0, d1, l1, ld1, lld1, info);
  HP_CHECK_LAUNCH("tri_prepare");
  char* pin = pinned_scratch();
  HP_REQUIRE(pin != nullptr, "syev_tri: pinned host scratch unavailable");
  double* hinfo = reinterpret_cast<double*>(pin + 160);  // 12 doubles: [160, 256)
  HP_CHECK_CUDA(d2h_small(hinfo, info, 12 * sizeof(double), st));
  count_launches(1);
  HP_CHECK_CUDA(cudaStreamSynchronize(st));
  const bool ok = hinfo[I_OK] != 0.0;
  const int K = (int)hinfo[I_K];
  if (diag) {
    diag[0] = 0.0;
    diag[1] = 0.0;
    diag[2] = hinfo[I_SIGMA];
    diag[3] = (double)K;
  }
  if (!ok) return HP_OK;  // declined
  if (K <= 0) {
    HP_CHECK_CUDA(zero_async(lam_desc, (size_t)n * 8, st));
    count_launches(1);
    *status_out = 0;
    return HP_OK;
  }
  tri_bisect<<<(unsigned)ceil_div((int64_t)K * 32, 256), 256, 0, st>>>(d1, lld1, n, K, info, lam_s, blo, bhi);
  HP_CHECK_LAUNCH("tri_bisect");
  tri_getvec<<<(unsigned)ceil_div(K, 32), 32, 0, st>>>(d1, l1, ld1, lld1, n, K, lda, info, lam_s, blo, bhi, LP, UM,
                                                         PP, W, ldw, lam_desc, resid);
  HP_CHECK_LAUNCH("tri_getvec");
  tri_check<<<1, 1024, 0, st>>>(lam_s, resid, K, n, lam_desc, info);
  HP_CHECK_LAUNCH("tri_check");
  HP_CHECK_CUDA(d2h_small(hinfo, info, 12 * sizeof(double), st));
  count_launches(1);
  HP_CHECK_CUDA(cudaStreamSynchronize(st));
  if (diag) {
    diag[0] = hinfo[I_MINGAP];
    diag[1] = hinfo[I_MAXRES];
  }
  if (hinfo[I_BAD] != 0.0 || !(hinfo[I_MINGAP] >= relgap_min) || !(hinfo[I_MAXRES] <= 1e-6)) return HP_OK;  // declined

  // W = Q Z: panels in reverse order, rows [j0, n) (row j0 of V_b is zero: keeps 16-byte alignment)
  const int npanel = (int)ceil_div(n - 1, NB);
  for (int b = npanel - 1; b >= 0; --b) {
    const int j0 = b * NB;
    const int j1 = std::min(j0 + NB, n - 1);
    const int nbe = j1 - j0;
    const int64_t rows = n - j0;
    VecSet vb{Vall + j0 + (int64_t)j0 * lda, lda, nullptr};
    VecSet zb{W + j0, ldw, nullptr};
    int rc = gemm_run(true, true, nbe, nbe, rows, vb, vb, true, 1.0, 0.0, S, NB, nullptr, nullptr, nullptr, 0, 0, gws,
                      gwsb, st);
    if (rc) return rc;
    tinv_build<<<(unsigned)ceil_div(nbe * nbe, 256), 256, 0, st>>>(S, NB, tau + j0, nbe);
    HP_CHECK_LAUNCH("tinv_build");
    rc = gemm_run(true, true, nbe, K, rows, vb, zb, true, 1.0, 0.0, Y, NB, nullptr, nullptr, nullptr, 0, 0, gws, gwsb,
                  st);
    if (rc) return rc;
    trsm_tinv<<<(unsigned)ceil_div(K, 128), 128, 0, st>>>(S, NB, nbe, Y, NB, K);
    HP_CHECK_LAUNCH("trsm_tinv");
    VecSet yb{Y, NB, nullptr};
    rc = gemm_run(false, true, rows, K, nbe, vb, yb, true, -1.0, 1.0, W + j0, ldw, nullptr, nullptr, nullptr, 0, 0, gws,
                  gwsb, st);
    if (rc) return rc;
  }
  *k_out = K;
  *status_out = 0;
  return HP_OK;
}

}  // namespace hp
