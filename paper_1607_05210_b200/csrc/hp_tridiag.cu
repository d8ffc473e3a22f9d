// K2t -- the leading eigenpairs of a symmetric positive (semi)definite matrix by Householder
// tridiagonalisation, for the large preconditioned eigenproblems H = L^T L of a node POD
// (replaces scipy.linalg.eigh, pod.py:329-331, where the block-Jacobi solve of hp_jacobi.cu needs
// ~11 sweeps x 8 n^3 flops).  Three stages, every one deterministic (no floating-point atomics,
// fixed reduction orders):
//
//   1. sytrd_panel  : H = Q T Q^T.  One cooperative launch per 64-column panel; a column step is
//                     two grid-wide phases -- (P2) every column dot A[:, c] . x of the trailing
//                     matrix with the current column x (HBM/L2-bound: the matrix is symmetric, so
//                     the matrix-vector product is a set of contiguous column dots, each owned by
//                     one CTA -- no cross-CTA partial sums), together with the panel dots V^T x,
//                     W^T x and x^T A x; (P3) the Householder scalars, v, w = tau (A v - V W^T v
//                     - W V^T v) + alpha' v and the NEXT column x in one pass over the panel rows.
//                     The reflector is applied unscaled (v = s x + t e_1) and w^T v is obtained
//                     from v^T A v - 2 (V^T v).(W^T v), so neither the norm nor alpha' needs a
//                     grid-wide phase of its own.  The trailing update A -= V W^T + W V^T is one
//                     DMMA GEMM per panel ([V|W] [W|V]^T, exactly symmetric output).
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
#include <cstdio>

#include "hp_common.cuh"

namespace cg = cooperative_groups;

namespace hp {

int gemm_run(bool a_kmajor, bool b_kmajor, int64_t M, int64_t N, int64_t K, VecSet A, VecSet B, bool aligned16,
             double alpha, double beta, double* C, int64_t ldc, const double* row_scale, const double* col_scale,
             const double* col_div, int sym, int b_upper, void* ws, size_t ws_bytes, cudaStream_t st);
size_t gemm_workspace_bytes(int64_t M, int64_t N, int64_t K, int sym, int b_upper);

namespace trd {

constexpr int NB = 64;    // panel width
constexpr int BT = 256;   // reflectors per compact-WY block of the back-transformation
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
  double* pxv;
  double* pxw;
  double* red;
  double* d;
  double* e;
  double* tau;
  int j0, j1;
  int per_max;
  unsigned long long* prof;  // optional phase timing (8 size buckets x 6 phases, ns), CTA 0 thread 0
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

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// w_r = tau (A v - V W^T v - W V^T v)_r + alpha' v_r: one expression shared by the row owners and by
// the CTA-local copy of row j+1, so both produce the same bits
__device__ __forceinline__ double w_entry(double tau, double av, double acc, double alpha_p, double v) {
  return fma(alpha_p, v, tau * (av - acc));
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
  const int sub8 = lane & 7;
  const int wbase8 = ((cta * TT + tid) >> 5) * 4;  // first row of this warp (4 rows of 8 lanes)
  const int wstride8 = (G * TT) >> 3;
  const int64_t ldp = p.ldp;
  double* Pv = p.P;
  double* Pw = p.P + (int64_t)NB * ldp;
  double* Qw = p.Q;
  double* Qv = p.Q + (int64_t)NB * ldp;
  const bool prof = p.prof != nullptr && blockIdx.x == 0 && threadIdx.x == 0;

  // the panel's first column: the trailing matrix is fully updated
  for (int r = p.j0 + cta * TT + tid; r < n; r += G * TT) {
    const double a = p.A[r + (int64_t)p.j0 * p.lda];
    if (r == p.j0)
      p.d[r] = a;
    else
      p.x[r] = a;
  }
  grid.sync();

  for (int j = p.j0; j < p.j1; ++j) {
    const int i = j - p.j0;
    unsigned long long tp[4];
    if (prof) tp[0] = gtime();
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
      const bool wmode = per <= NW;  // few short columns: one warp per column, no cross-warp sums
      if (wmode) {
        if (t0 + warp < t1) {
          const double2* q0 = task_ptr(t0 + warp);
          double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
          int q = lane;
          for (; q + 96 < len2; q += 128) {
            const double2 v0 = __ldcg(q0 + q), v1 = __ldcg(q0 + q + 32), v2 = __ldcg(q0 + q + 64),
                          v3 = __ldcg(q0 + q + 96);
            const double2 x0 = xs2[q], x1 = xs2[q + 32], x2 = xs2[q + 64], x3 = xs2[q + 96];
            a0 = fma(v0.x, x0.x, a0);
            a0 = fma(v0.y, x0.y, a0);
            a1 = fma(v1.x, x1.x, a1);
            a1 = fma(v1.y, x1.y, a1);
            a2 = fma(v2.x, x2.x, a2);
            a2 = fma(v2.y, x2.y, a2);
            a3 = fma(v3.x, x3.x, a3);
            a3 = fma(v3.y, x3.y, a3);
          }
          for (; q < len2; q += 32) {
            const double2 v0 = __ldcg(q0 + q);
            const double2 x0 = xs2[q];
            a0 = fma(v0.x, x0.x, a0);
            a0 = fma(v0.y, x0.y, a0);
          }
          a0 = warp_sum((a0 + a1) + (a2 + a3));
          if (lane == 0) part[warp] = a0;
        }
      } else {
        // serpentine: odd columns walk their chunk backwards, so a sweep starts on the part of the
        // trailing matrix the previous sweep left in L2
        const int ngroup = (t1 - t0 + 3) >> 2;
        for (int g = 0; g < ngroup; ++g) {
          const int tb = t0 + 4 * ((j & 1) ? ngroup - 1 - g : g);
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
      }
      __syncthreads();
      double xa = 0.0;  // this CTA's share of x^T A x
      for (int k = tid; k < t1 - t0; k += TT) {
        double s;
        if (wmode) {
          s = part[k];
        } else {
          s = 0.0;
          for (int w = 0; w < NW; ++w) s += part[w * p.per_max + k];
        }
        const int tk = t0 + k;
        if (tk < nr) {
          p.y[j + 1 + tk] = s;
          xa = fma(s, xs[j + 1 + tk - r0], xa);
        } else if (tk < nr + i) {
          p.pxv[tk - nr] = s;
        } else {
          p.pxw[tk - nr - i] = s;
        }
      }
      xa = block_sum(xa, rbuf);
      if (tid == 0) p.red[cta] = xa;
    }
    // Prefetch for P3: this thread's panel row, row j+1 of the panel and column j+1 of A depend on
    // nothing this column's dots produce, so their L2 round trip overlaps the grid barrier
    auto load_row = [&](int r, bool valid, double (&vv)[8], double (&ww)[8], double& anext) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int c = sub8 + 8 * u;
        const bool on = valid && c < i;
        vv[u] = on ? __ldcg(Pv + r + (int64_t)c * ldp) : 0.0;
        ww[u] = on ? __ldcg(Pw + r + (int64_t)c * ldp) : 0.0;
      }
      anext = valid ? p.A[r + (int64_t)(j + 1) * p.lda] : 0.0;
    };
    double vv[8], ww[8], anext;
    const int r_first = j + 1 + wbase8 + (lane >> 3);
    load_row(r_first, r_first < n, vv, ww, anext);
    double rv = 0.0, rw = 0.0;
    if (tid < i) {
      rv = __ldcg(Pv + (j + 1) + (int64_t)tid * ldp);
      rw = __ldcg(Pw + (j + 1) + (int64_t)tid * ldp);
    }
    const double a11 = p.A[(j + 1) + (int64_t)(j + 1) * p.lda];
    if (prof) tp[1] = gtime();
    grid.sync();
    if (prof) tp[2] = gtime();
    // ------------------------------------------------------------------ P3: reflector, w, next column
    const double y1 = __ldcg(p.y + j + 1);
    double yr = r_first < n ? __ldcg(p.y + r_first) : 0.0;
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
      rowV[tid] = rv;
      rowW[tid] = rw;
      cV[tid] = s * __ldcg(p.pxv + tid) + t * rv;
      cW[tid] = s * __ldcg(p.pxw + tid) + t * rw;
    } else if (tid < NB) {
      rowV[tid] = rowW[tid] = cV[tid] = cW[tid] = 0.0;
    }
    __syncthreads();
    if (warp == 0) {  // x^T A x: the CTA partials in a fixed order
      double a = 0.0;
      for (int c = lane; c < G; c += 32) a += __ldcg(p.red + c);
      a = warp_sum(a);
      if (lane == 0) scal[0] = a;
    } else if (warp == 1) {  // (V^T v) . (W^T v)
      double a = 0.0;
      for (int c = lane; c < i; c += 32) a = fma(cV[c], cW[c], a);
      a = warp_sum(a);
      if (lane == 0) scal[1] = a;
    } else if (warp == 2) {  // row j+1 of V W^T v + W V^T v, in the row owner's summation order
      double a = 0.0;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int c = sub8 + 8 * u;
        a = fma(rowV[c], cW[c], a);
        a = fma(rowW[c], cV[c], a);
      }
#pragma unroll
      for (int o = 1; o < 8; o <<= 1) a += __shfl_xor_sync(FULL, a, o);
      if (lane == 0) scal[2] = a;
    }
    __syncthreads();
    // w^T v = tau (v^T A v - 2 (V^T v).(W^T v)) with v = s x + t e_1: no grid-wide reduction of its own
    const double vAv = s * s * scal[0] + 2.0 * s * t * y1 + t * t * a11;
    const double alpha_p = -0.5 * tau * (tau * (vAv - 2.0 * scal[1]));
    const double vj1 = (tau == 0.0) ? 0.0 : 1.0;
    const double wrow = w_entry(tau, s * y1 + t * a11, scal[2], alpha_p, vj1);  // W[j+1, i]
    const bool do_next = (j + 1 < p.j1) || (p.j1 == n - 1);
    for (int rb = j + 1 + wbase8; rb < n; rb += wstride8) {  // 8 lanes per row (one pass for n <= 9472)
      const int r = rb + (lane >> 3);
      const bool valid = r < n;
      if (rb != j + 1 + wbase8) {
        load_row(r, valid, vv, ww, anext);
        yr = valid ? __ldcg(p.y + r) : 0.0;
      }
      double acc1 = 0.0, acc2 = 0.0;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int c = sub8 + 8 * u;  // c < NB: the coefficient arrays are zero past i
        acc1 = fma(vv[u], cW[c], acc1);
        acc1 = fma(ww[u], cV[c], acc1);
        acc2 = fma(vv[u], rowW[c], acc2);
        acc2 = fma(ww[u], rowV[c], acc2);
      }
#pragma unroll
      for (int o = 1; o < 8; o <<= 1) {
        acc1 += __shfl_xor_sync(FULL, acc1, o);
        acc2 += __shfl_xor_sync(FULL, acc2, o);
      }
      if (valid && sub8 == 0) {
        const double v = (tau == 0.0) ? 0.0 : ((r == j + 1) ? 1.0 : s * xs[r - r0]);
        const double w = w_entry(tau, s * yr + t * anext, acc1, alpha_p, v);
        Pv[r + (int64_t)i * ldp] = v;
        Qv[r + (int64_t)i * ldp] = v;
        p.Vall[r + (int64_t)j * p.ldv] = v;
        Pw[r + (int64_t)i * ldp] = w;
        Qw[r + (int64_t)i * ldp] = w;
        if (do_next) {
          const double xn = anext - acc2 - (v * wrow + w * vj1);
          if (r == j + 1)
            p.d[j + 1] = xn;
          else
            p.x[r] = xn;
        }
      }
    }
    if (prof) tp[3] = gtime();
    grid.sync();
    if (prof) {
      unsigned long long* b = p.prof + 6 * ((int)(((long long)j * 8) / n));
      b[0] += tp[1] - tp[0];  // P2
      b[1] += tp[2] - tp[1];  // sync B
      b[2] += tp[3] - tp[2];  // P3
      b[3] += gtime() - tp[3];  // sync A
    }
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

enum { I_SIGMA = 0, I_LMAX, I_LMIN, I_K, I_OK, I_TNORM, I_PIVMIN, I_HI, I_LO, I_MINGAP, I_MAXRES, I_BAD, I_MAXIT, I_SUMIT, I_COUNT };

// One CTA of 512 threads (16 warps: the Sturm recurrences are division-latency chains, more warps
// on the SM would only queue on its issue slots): spectrum bounds, lambda_max and lambda_min by
// 257-way multisection on a safely definite representation (both at once, one half of the CTA
// each), the count K of eigenvalues >= floor_rel * lambda_max, and the root representation
// T - sigma I = L D L^T with sigma just below lambda_min.
__global__ void __launch_bounds__(512, 1) tri_prepare(const double* a, const double* b, int n, double floor_rel,
                                                       double* d0, double* lld0, double* d1, double* l1, double* ld1,
                                                       double* lld1, double* info) {
  __shared__ double sh[8];
  __shared__ double bounds[2][2];
  __shared__ int cnts[2];
  __shared__ double red[4][16];
  const int tid = threadIdx.x;
  double gl = DBL_MAX, gu = -DBL_MAX, em = 0.0, tn = 0.0;
  for (int i = tid; i < n; i += 512) {
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
  if ((tid & 31) == 0) {
    red[0][tid >> 5] = gl;
    red[1][tid >> 5] = gu;
    red[2][tid >> 5] = em;
    red[3][tid >> 5] = tn;
  }
  __syncthreads();
  if (tid == 0) {
    for (int w = 1; w < 16; ++w) {
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
    const double top = (gu - sigma0) * (1.0 + 1e-10) + 16.0 * UNIT * tn;  // bound of the shifted spectrum
    bounds[0][0] = bounds[1][0] = 0.0;
    bounds[0][1] = bounds[1][1] = top;
  }
  __syncthreads();
  const double sigma0 = sh[0], pivmin = sh[1], tnorm = sh[2];
  const int which = tid >> 8;  // 0: lambda_max (ascending index n-1), 1: lambda_min (index 0)
  const int want = which == 0 ? n - 1 : 0;
  const int t = tid & 255;
  for (int round = 0; round < 8; ++round) {
    if (tid < 2) cnts[tid] = 0;
    __syncthreads();
    const double lo = bounds[which][0], hi = bounds[which][1];
    const double step = (hi - lo) / 257.0;
    const double xq = lo + step * (double)(t + 1);
    const int c = negcount(d0, lld0, n, xq, pivmin);
    const unsigned okm = __ballot_sync(FULL, c <= want);  // points at or below the wanted eigenvalue
    if ((tid & 31) == 0) atomicAdd(&cnts[which], __popc(okm));
    __syncthreads();
    if (t == 0) {
      const int cnt = cnts[which];
      if (cnt > 0) bounds[which][0] = lo + step * (double)cnt;
      if (cnt < 256) bounds[which][1] = lo + step * (double)(cnt + 1);
    }
    __syncthreads();
  }
  if (tid == 0) {
    const double lam_max = 0.5 * (bounds[0][0] + bounds[0][1]) + sigma0;
    const double lam_min = 0.5 * (bounds[1][0] + bounds[1][1]) + sigma0;
    const double floor_abs = floor_rel * lam_max;
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

// Eight lanes per wanted eigenvalue (descending index k; a full warp per eigenvalue was bound by the
// SM's issue slots: 37 warps per SM of division chains): 9-way multisection on a geometric grid (small
// eigenvalues are located to the same RELATIVE accuracy as large ones) until the bracket holds
// exactly this eigenvalue and is narrower than 2^-30 octaves; tri_getvec's Rayleigh-quotient
// iteration converges in one step from there.  A cluster keeps subdividing (at most 24 rounds).
constexpr int BL = 8;  // lanes per eigenvalue in tri_bisect
__global__ void __launch_bounds__(256) tri_bisect(const double* d, const double* lld, int n, int K, const double* info,
                                                  double* lam_s, double* blo, double* bhi) {
  const int k = (blockIdx.x * blockDim.x + threadIdx.x) / BL;
  const int lane = threadIdx.x & 31;
  const int sub = lane & (BL - 1);
  const int gbase = lane & ~(BL - 1);
  const unsigned gmask = ((1u << BL) - 1u) << gbase;  // this eigenvalue's lanes (groups diverge freely)
  if (k >= K) return;
  const int want = n - 1 - k;
  const double pivmin = info[I_PIVMIN];
  double lo = info[I_LO], hi = info[I_HI];
  int clo = 0, chi = n;  // eigenvalues below lo / below hi
  for (int round = 0; round < 24; ++round) {
    const double lr = log2(hi / lo);
    if (!(lr > 8.0 * UNIT)) break;
    if (clo == want && chi == want + 1 && lr <= 0x1p-30) break;
    double xq = lo * exp2(lr * (double)(sub + 1) / (double)(BL + 1));
    xq = fmin(fmax(xq, lo), hi);
    const int c = negcount(d, lld, n, xq, pivmin);
    const unsigned okm = (__ballot_sync(gmask, c <= want) & gmask) >> gbase;
    const int cnt = __popc(okm);
    const double nlo = __shfl_sync(gmask, xq, gbase + max(cnt - 1, 0));
    const int nclo = __shfl_sync(gmask, c, gbase + max(cnt - 1, 0));
    const double nhi = __shfl_sync(gmask, xq, gbase + min(cnt, BL - 1));
    const int nchi = __shfl_sync(gmask, c, gbase + min(cnt, BL - 1));
    if (cnt > 0) {
      lo = nlo;
      clo = nclo;
    }
    if (cnt < BL) {
      hi = nhi;
      chi = nchi;
    }
  }
  if (sub == 0) {
    lam_s[k] = sqrt(lo) * sqrt(hi);
    blo[k] = lo;
    bhi[k] = hi;
  }
}

// z_r = 1, z_i = -lplus_i z_{i+1} (i < r), z_{i+1} = -uminus_i z_i (i >= r): returns z^T z; with
// STORE the entries are written scaled to column zc.  The factor loads run PF steps ahead of the
// multiply chain (they depend on nothing but the index).
constexpr int PF = 8;
template <bool STORE>
__device__ __forceinline__ double twisted_z(const double* __restrict__ lp, const double* __restrict__ um, int64_t kp,
                                            int n, int r, double scale, double* __restrict__ zc) {
  double ztz = 1.0, z = 1.0;
  if (STORE) zc[r] = scale;
  for (int i0 = r - 1; i0 >= 0; i0 -= PF) {
    double f[PF];
#pragma unroll
    for (int u = 0; u < PF; ++u) f[u] = (i0 - u >= 0) ? lp[(int64_t)(i0 - u) * kp] : 0.0;
#pragma unroll
    for (int u = 0; u < PF; ++u) {
      if (i0 - u >= 0) {
        z = -f[u] * z;
        ztz = fma(z, z, ztz);
        if (STORE) zc[i0 - u] = z * scale;
      }
    }
  }
  z = 1.0;
  for (int i0 = r; i0 < n - 1; i0 += PF) {
    double f[PF];
#pragma unroll
    for (int u = 0; u < PF; ++u) f[u] = (i0 + u < n - 1) ? um[(int64_t)(i0 + u) * kp] : 0.0;
#pragma unroll
    for (int u = 0; u < PF; ++u) {
      if (i0 + u < n - 1) {
        z = -f[u] * z;
        ztz = fma(z, z, ztz);
        if (STORE) zc[i0 + u + 1] = z * scale;
      }
    }
  }
  return ztz;
}

// One thread per wanted eigenvalue: twisted factorisation (stationary qds from the top, progressive
// qds from the bottom, twist where |gamma| is smallest), Rayleigh-quotient correction of the
// eigenvalue inside the Sturm bracket (cubic convergence; a step that leaves the bracket becomes a
// bisection), eigenvector written normalised to column k of Z.
__global__ void __launch_bounds__(32) tri_getvec(const double* __restrict__ d, const double* __restrict__ l,
                                                 const double* __restrict__ ld, const double* __restrict__ lld,
                                                 int n, int K, int64_t kp, const double* info, double* lam_s,
                                                 const double* blo, const double* bhi, double* __restrict__ LP,
                                                 double* __restrict__ UM, double* __restrict__ PP,
                                                 double* __restrict__ Z, int64_t ldz, double* lam_out,
                                                 double* resid, int* iters) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= K) return;
  const double pivmin = info[I_PIVMIN], sigma = info[I_SIGMA];
  double lam = lam_s[k];
  double lo = blo[k], hi = bhi[k];
  double* lp = LP + k;
  double* um = UM + k;
  double* pp = PP + k;
  int r = 0;
  double gam = 0.0, ztz = 1.0;
  const int want = n - 1 - k;
  constexpr int MAXIT = 5;
  int its = 0;
  for (int it = 0; it < MAXIT; ++it) {
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
    gam = sarr + pcur;  // pp[0]
    double best = fabs(gam);
    r = 0;
    int neg = 0;  // Sturm count at lam, a by-product of the stationary transform
    for (int i0 = 0; i0 < n - 1; i0 += PF) {
      double pb[PF];
#pragma unroll
      for (int u = 0; u < PF; ++u) pb[u] = (i0 + u < n - 1) ? pp[(int64_t)(i0 + u + 1) * kp] : 0.0;
#pragma unroll
      for (int u = 0; u < PF; ++u) {
        const int i = i0 + u;
        if (i < n - 1) {
          double dp = d[i] + s;
          if (fabs(dp) < pivmin) dp = -pivmin;
          neg += dp < 0.0;
          const double lpi = ld[i] / dp;
          lp[(int64_t)i * kp] = lpi;
          sarr = s * lpi * l[i];
          s = sarr - lam;
          const double g = sarr + pb[u];
          if (fabs(g) < best) {
            best = fabs(g);
            gam = g;
            r = i + 1;
          }
        }
      }
    }
    neg += (d[n - 1] + s) < 0.0;
    ztz = twisted_z<false>(lp, um, kp, n, r, 1.0, nullptr);
    const double rq = gam / ztz;
    if (neg <= want)
      lo = fmax(lo, lam);
    else
      hi = fmin(hi, lam);
    its = it + 1;
    if (it == MAXIT - 1 || !(fabs(rq) > 8.0 * UNIT * fabs(lam))) break;
    double nl = lam + rq;
    // a step that leaves the bracket (beyond rounding slack) is replaced by a geometric bisection
    if (!(nl > lo * (1.0 - 32.0 * UNIT) && nl < hi * (1.0 + 32.0 * UNIT))) nl = sqrt(lo) * sqrt(hi);
    if (nl == lam) break;
    lam = nl;
  }
  const double scale = rsqrt(ztz);
  twisted_z<true>(lp, um, kp, n, r, scale, Z + (int64_t)k * ldz);
  lam_s[k] = lam;
  lam_out[k] = lam + sigma;
  iters[k] = its;
  const double res = fabs(gam) * scale / fabs(lam);
  resid[k] = (isfinite(res) && isfinite(scale) && scale > 0.0) ? res : DBL_MAX;
}

// smallest relative gap between consecutive computed eigenvalues, largest relative residual
__global__ void __launch_bounds__(1024, 1) tri_check(const double* lam_s, const double* resid, const int* iters, int K,
                                                     int n, double* lam_out, double* info) {
  __shared__ double r0[32], r1[32], r2[32], r3[32];
  const int tid = threadIdx.x;
  double mg = DBL_MAX, mr = 0.0, mi = 0.0, si = 0.0;
  for (int k = tid; k < K; k += 1024) {
    if (k + 1 < K) mg = fmin(mg, fabs(lam_s[k] - lam_s[k + 1]) / fabs(lam_s[k]));
    mr = fmax(mr, resid[k]);
    mi = fmax(mi, (double)iters[k]);
    si += (double)iters[k];
  }
  for (int k = K + tid; k < n; k += 1024) lam_out[k] = 0.0;
  for (int o = 16; o; o >>= 1) {
    mg = fmin(mg, __shfl_xor_sync(FULL, mg, o));
    mr = fmax(mr, __shfl_xor_sync(FULL, mr, o));
    mi = fmax(mi, __shfl_xor_sync(FULL, mi, o));
    si += __shfl_xor_sync(FULL, si, o);
  }
  if ((tid & 31) == 0) {
    r0[tid >> 5] = mg;
    r1[tid >> 5] = mr;
    r2[tid >> 5] = mi;
    r3[tid >> 5] = si;
  }
  __syncthreads();
  if (tid == 0) {
    for (int w = 1; w < 32; ++w) {
      mg = fmin(mg, r0[w]);
      mr = fmax(mr, r1[w]);
      mi = fmax(mi, r2[w]);
      si += r3[w];
    }
    info[I_MAXIT] = mi;
    info[I_SUMIT] = si;
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

// Y <- T Y, i.e. solve the upper-triangular T^-1 Y' = Y (a diagonal block of at most NB rows); one
// thread per column of Y with the column in registers (fully unrolled back-substitution, reciprocal
// pivots from shared memory; rows past nb act as an identity block)
__global__ void __launch_bounds__(128) trsm_tinv(const double* Tinv, int ldt, int nb, double* Y, int ldy, int K) {
  __shared__ double ts[NB * NB];
  __shared__ double rd[NB];
  for (int e = threadIdx.x; e < NB * NB; e += blockDim.x) {
    const int i = e % NB, c = e / NB;
    ts[e] = (i < nb && c < nb && i < c) ? Tinv[i + (int64_t)c * ldt] : 0.0;
  }
  if (threadIdx.x < NB) rd[threadIdx.x] = threadIdx.x < nb ? 1.0 / Tinv[threadIdx.x + (int64_t)threadIdx.x * ldt] : 1.0;
  __syncthreads();
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= K) return;
  double* yc = Y + (int64_t)k * ldy;
  double y[NB];
#pragma unroll
  for (int i = 0; i < NB; ++i) y[i] = i < nb ? yc[i] : 0.0;
#pragma unroll
  for (int i = NB - 1; i >= 0; --i) {
    double s = y[i];
#pragma unroll
    for (int c = i + 1; c < NB; ++c) s = fma(-ts[i + c * NB], y[c], s);
    y[i] = s * rd[i];
  }
#pragma unroll
  for (int i = 0; i < NB; ++i)
    if (i < nb) yc[i] = y[i];
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
  o += al256((size_t)BT * n * 8) + al256((size_t)BT * BT * 8);  // Y, S
  size_t g = gemm_workspace_bytes(n, n, 2 * NB, 1, 0);
  for (int64_t mb : {(int64_t)NB, (int64_t)(2 * NB), (int64_t)(3 * NB), (int64_t)BT}) {
    g = std::max(g, gemm_workspace_bytes(mb, n, n, 0, 0));
    g = std::max(g, gemm_workspace_bytes(n, n, mb, 0, 0));
    g = std::max(g, gemm_workspace_bytes(mb, mb, n, 0, 0));
    g = std::max(g, gemm_workspace_bytes(NB, n, mb, 0, 0));
  }
  o += al256(g) + 256;
  return o;
}

// Eigenpairs of the symmetric positive semidefinite H (n x n) with lambda >= floor_rel * lambda_max:
// lam_desc[0..K) descending (the rest zeroed), eigenvectors in the first K columns of W (n x n).
// status_out: 0 = done; 1 = declined (clustered spectrum, relative gap below relgap_min, or no
// definite root representation) -- W / lam_desc are then not meaningful and the caller falls back
// to hp_syev.  diag (nullable, host, 8 doubles): min relative gap, max relative residual, sigma, K,
// sytrd stage ms, tridiagonal stage ms, max Rayleigh-quotient iterations, 0.
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
  double *x = vec[0], *y = vec[1], *dT = vec[3], *eT = vec[4], *tau = vec[5], *d0 = vec[6],
         *lld0 = vec[7], *d1 = vec[8], *l1 = vec[9], *ld1 = vec[10], *lld1 = vec[11], *lam_s = vec[12],
         *blo = vec[13], *bhi = vec[14], *resid = vec[15];
  double* pxv = take(1024 * 8);
  double* pxw = take(1024 * 8);
  double* red = take(1024 * 8);
  double* info = take(1024 * 8);
  double* LP = take((size_t)lda * n * 8);
  double* UM = take((size_t)lda * n * 8);
  double* PP = take((size_t)lda * n * 8);
  double* Y = take((size_t)BT * n * 8);
  double* S = take((size_t)BT * BT * 8);
  void* gws = base + o;
  const size_t gwsb = ws_bytes - o;

  // stage timing: CUDA events on the launching stream (diag receives the sytrd / tridiagonal stage
  // times for the caller's roofline; hp_set_debug bit 3 prints every stage)
  const bool trace = (debug_flags() & DBG_TRI_TRACE) != 0;
  struct Events {
    cudaEvent_t ev[6] = {};
    ~Events() {
      for (auto& e : ev)
        if (e) cudaEventDestroy(e);
    }
  } evs;
  cudaEvent_t* ev = evs.ev;
  auto mark = [&](int i) {
    if (ev[i] || cudaEventCreate(&ev[i]) == cudaSuccess) cudaEventRecord(ev[i], st);
  };
  auto elapsed = [&](int a, int b) -> double {
    float ms = 0.f;
    if (!ev[a] || !ev[b] || cudaEventElapsedTime(&ms, ev[a], ev[b]) != cudaSuccess) return 0.0;
    return (double)ms;
  };
  auto report = [&](int last) {
    if (!trace) return;
    cudaEventSynchronize(ev[last]);
    static const char* names[] = {"sytrd", "prepare", "bisect+getvec", "check", "backtransform"};
    fprintf(stderr, "[hp_syev_tri] n=%d", n);
    for (int i = 0; i < last; ++i) fprintf(stderr, " %s=%.2fms", names[i], elapsed(i, i + 1));
    fprintf(stderr, "\n");
  };
  mark(0);
  copy_in<<<(unsigned)ceil_div(lda * n, 256), 256, 0, st>>>(H, ldh, n, A, lda);
  HP_CHECK_LAUNCH("tri copy_in");
  HP_CHECK_CUDA(zero_async(Vall, (size_t)lda * n * 8, st));
  HP_CHECK_CUDA(zero_async(P, (size_t)lda * 2 * NB * 8, st));
  HP_CHECK_CUDA(zero_async(Q, (size_t)lda * 2 * NB * 8, st));
  HP_CHECK_CUDA(zero_async(x, (size_t)(n + 2) * 8, st));
  HP_CHECK_CUDA(zero_async(y, (size_t)(n + 2) * 8, st));
  count_launches(5);

  int nsm = num_sms();
  const int G = std::max(1, std::min(nsm, 1024));
  const int per_max = std::max((int)ceil_div((int64_t)n + 2 * NB, G) + 4, NW);
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
  p.pxv = pxv;
  p.pxw = pxw;
  p.red = red;
  p.d = dT;
  p.e = eT;
  p.tau = tau;
  p.per_max = per_max;
  p.prof = nullptr;
  if (trace) {
    p.prof = reinterpret_cast<unsigned long long*>(info + 512);
    HP_CHECK_CUDA(zero_async(p.prof, 48 * 8, st));
  }
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

  mark(1);
  if (trace) {
    unsigned long long hp[48];
    if (cudaMemcpyAsync(hp, p.prof, sizeof(hp), cudaMemcpyDeviceToHost, st) == cudaSuccess &&
        cudaStreamSynchronize(st) == cudaSuccess) {
      fprintf(stderr, "[sytrd_panel] per-phase ms by column octile (P2, syncB, P3, syncA)\n");
      for (int b = 0; b < 8; ++b) {
        fprintf(stderr, "  octile %d:", b);
        for (int q = 0; q < 4; ++q) fprintf(stderr, " %7.2f", hp[6 * b + q] * 1e-6);
        fprintf(stderr, "\n");
      }
    }
  }
  tri_prepare<<<1, 512, 0, st>>>(dT, eT, n, floor_rel, d0, lld0, d1, l1, ld1, lld1, info);
  HP_CHECK_LAUNCH("tri_prepare");
  char* pin = pinned_scratch();
  HP_REQUIRE(pin != nullptr, "syev_tri: pinned host scratch unavailable");
  double* hinfo = reinterpret_cast<double*>(pin + 256);  // 16 doubles: [256, 384)
  HP_CHECK_CUDA(d2h_small(hinfo, info, 16 * sizeof(double), st));
  count_launches(1);
  HP_CHECK_CUDA(cudaStreamSynchronize(st));
  const bool ok = hinfo[I_OK] != 0.0;
  const int K = (int)hinfo[I_K];
  if (diag) {
    for (int q = 0; q < 8; ++q) diag[q] = 0.0;
    diag[2] = hinfo[I_SIGMA];
    diag[3] = (double)K;
    diag[4] = elapsed(0, 1);
  }
  mark(2);
  if (!ok || K <= 0) report(2);
  if (!ok) return HP_OK;  // declined
  if (K <= 0) {
    HP_CHECK_CUDA(zero_async(lam_desc, (size_t)n * 8, st));
    count_launches(1);
    *status_out = 0;
    return HP_OK;
  }
  tri_bisect<<<(unsigned)ceil_div((int64_t)K * BL, 256), 256, 0, st>>>(d1, lld1, n, K, info, lam_s, blo, bhi);
  HP_CHECK_LAUNCH("tri_bisect");
  tri_getvec<<<(unsigned)ceil_div(K, 32), 32, 0, st>>>(d1, l1, ld1, lld1, n, K, lda, info, lam_s, blo, bhi, LP, UM,
                                                         PP, W, ldw, lam_desc, resid, reinterpret_cast<int*>(vec[16]));
  HP_CHECK_LAUNCH("tri_getvec");
  mark(3);
  tri_check<<<1, 1024, 0, st>>>(lam_s, resid, reinterpret_cast<const int*>(vec[16]), K, n, lam_desc, info);
  HP_CHECK_LAUNCH("tri_check");
  HP_CHECK_CUDA(d2h_small(hinfo, info, 16 * sizeof(double), st));
  count_launches(1);
  HP_CHECK_CUDA(cudaStreamSynchronize(st));
  if (diag) {
    diag[0] = hinfo[I_MINGAP];
    diag[1] = hinfo[I_MAXRES];
    diag[5] = elapsed(1, 3);
    diag[6] = hinfo[I_MAXIT];
  }
  mark(4);
  if (trace)
    fprintf(stderr, "[hp_syev_tri] K=%d getvec iterations max %.0f mean %.2f, min relgap %.2e, max resid %.2e\n", K,
            hinfo[I_MAXIT], hinfo[I_SUMIT] / std::max(K, 1), hinfo[I_MINGAP], hinfo[I_MAXRES]);
  if (hinfo[I_BAD] != 0.0 || !(hinfo[I_MINGAP] >= relgap_min) || !(hinfo[I_MAXRES] <= 1e-6)) {
    report(4);
    return HP_OK;  // declined
  }

  // W = Q Z: compact-WY blocks of BT reflectors in reverse order, rows [j0, n) (row j0 of V_b is
  // zero: keeps 16-byte alignment).  Y = V_b^T Z; Y <- T Y by blocked back-substitution with the
  // upper-triangular T^-1 (64-row diagonal blocks in shared memory, GEMMs above them); Z -= V_b Y.
  const int nblock = (int)ceil_div(n - 1, BT);
  for (int b = nblock - 1; b >= 0; --b) {
    const int j0 = b * BT;
    const int j1 = std::min(j0 + BT, n - 1);
    const int nbe = j1 - j0;
    const int64_t rows = n - j0;
    VecSet vb{Vall + j0 + (int64_t)j0 * lda, lda, nullptr};
    VecSet zb{W + j0, ldw, nullptr};
    int rc = gemm_run(true, true, nbe, nbe, rows, vb, vb, true, 1.0, 0.0, S, BT, nullptr, nullptr, nullptr, 0, 0, gws,
                      gwsb, st);
    if (rc) return rc;
    tinv_build<<<(unsigned)ceil_div(nbe * nbe, 256), 256, 0, st>>>(S, BT, tau + j0, nbe);
    HP_CHECK_LAUNCH("tinv_build");
    rc = gemm_run(true, true, nbe, K, rows, vb, zb, true, 1.0, 0.0, Y, BT, nullptr, nullptr, nullptr, 0, 0, gws, gwsb,
                  st);
    if (rc) return rc;
    for (int c0 = ((nbe - 1) / NB) * NB; c0 >= 0; c0 -= NB) {
      const int c1 = std::min(c0 + NB, nbe);
      if (c1 < nbe) {
        VecSet ta{S + c0 + (int64_t)c1 * BT, BT, nullptr};
        VecSet yl{Y + c1, BT, nullptr};
        rc = gemm_run(false, true, c1 - c0, K, nbe - c1, ta, yl, true, -1.0, 1.0, Y + c0, BT, nullptr, nullptr,
                      nullptr, 0, 0, gws, gwsb, st);
        if (rc) return rc;
      }
      trsm_tinv<<<(unsigned)ceil_div(K, 128), 128, 0, st>>>(S + c0 + (int64_t)c0 * BT, BT, c1 - c0, Y + c0, BT, K);
      HP_CHECK_LAUNCH("trsm_tinv");
    }
    VecSet yb{Y, BT, nullptr};
    rc = gemm_run(false, true, rows, K, nbe, vb, yb, true, -1.0, 1.0, W + j0, ldw, nullptr, nullptr, nullptr, 0, 0, gws,
                  gwsb, st);
    if (rc) return rc;
  }
  mark(5);
  report(5);
  *k_out = K;
  *status_out = 0;
  return HP_OK;
}

}  // namespace hp
