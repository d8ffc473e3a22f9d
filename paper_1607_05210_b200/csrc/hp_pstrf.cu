// Pivoted Cholesky of the node Gramian: the preconditioner of the eigensolver.
//
// G (m x m, symmetric positive semi-definite up to rounding) is factored as
// G = L L^T + E with complete diagonal pivoting, L (m x r) stored with its
// rows in the ORIGINAL index order -- pivoting is bookkeeping only, nothing
// is swapped.  The factorisation runs until the largest remaining pivot is
// <= tol (E is then rounding noise below the Gramian cutoff of pod.py:284).
//
// Why: the eigenvalues of G are those of H = L^T L (r x r) and its
// eigenvectors are V = L W Lambda^{-1/2} (W = eigenvectors of H).  H is
// strongly graded (column norms of L follow the pivots), so two-sided Jacobi
// on H converges in a handful of sweeps where Jacobi on G stalls at the
// rounding floor -- the QR-preconditioning of Drmac & Veselic, applied to the
// method of snapshots.
//
// Kernel structure, per panel of PB columns:
//   pstrf_panel_sm : cooperative persistent kernel (one CTA per SM).  For each
//                 column j: grid-wide argmax of the running diagonal d
//                 (ties -> smallest index), L[:, j] = (A[:, p] - L_panel L_panel[p]^T)
//                 / sqrt(d_p) over the CTA's row slice, d -= L[:, j]^2.
//                 One grid.sync() per column.
//   trailing    : A -= L_panel L_panel^T (full m x m, symmetric) on the DMMA
//                 GEMM engine.
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>

#include "hp_common.cuh"

namespace cg = cooperative_groups;

namespace hp {

int gemm_run(bool a_kmajor, bool b_kmajor, int64_t M, int64_t N, int64_t K, VecSet A, VecSet B, bool aligned16,
             double alpha, double beta, double* C, int64_t ldc, const double* row_scale, const double* col_scale,
             const double* col_div, int sym, int b_upper, void* ws, size_t ws_bytes, cudaStream_t st);
size_t gemm_workspace_bytes(int64_t M, int64_t N, int64_t K, int sym, int b_upper);

namespace pc {

constexpr int PB = 128;      // panel width
constexpr int PT = 256;      // threads per CTA

struct Params {
  double* A;        // m x m working copy (trailing-updated), ld = lda
  int64_t lda;
  int64_t m;
  double* L;        // m x m (first r columns used), ld = ldl
  int64_t ldl;
  double* d;        // running diagonal, -inf once pivoted
  int* piv;         // piv[j] = original index of the j-th pivot
  double* red_v;    // per-CTA argmax partials
  int* red_i;
  int* rank;        // device: number of columns factored so far (stops growing at tol)
  double* Lrm;      // m x PB row-major copy of the current panel of L (pivot-row fetches)
  double tol;
  int k0, k1;       // panel columns [k0, k1)
};

__device__ __forceinline__ bool better(double v, int i, double bv, int bi) {
  return v > bv || (v == bv && i < bi);
}

// CTA-local argmax of the running diagonal over rows [r0, r1) -> partials[slot][blockIdx.x]
__device__ __forceinline__ void local_argmax(const Params& p, int64_t r0, int64_t r1, int slot, double* sv, int* si) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double bv = -INFINITY;
  int bi = 0x7fffffff;
  for (int64_t i = r0 + tid; i < r1; i += PT) {
    const double v = p.d[i];
    if (better(v, (int)i, bv, bi)) {
      bv = v;
      bi = (int)i;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (better(ov, oi, bv, bi)) {
      bv = ov;
      bi = oi;
    }
  }
  if (lane == 0) {
    sv[warp] = bv;
    si[warp] = bi;
  }
  __syncthreads();
  if (tid == 0) {
    double cv = sv[0];
    int ci = si[0];
    for (int w = 1; w < PT / 32; ++w)
      if (better(sv[w], si[w], cv, ci)) {
        cv = sv[w];
        ci = si[w];
      }
    p.red_v[slot * 1024 + blockIdx.x] = cv;
    p.red_i[slot * 1024 + blockIdx.x] = ci;
  }
}

// One grid-wide barrier per column: the argmax partials for column j+1 are produced in the
// same pass that computes column j (double-buffered by column parity).  Global-memory form,
// used only when a CTA's rows of the panel do not fit in shared memory (pstrf_panel_sm).
__global__ void __launch_bounds__(PT) pstrf_panel(Params p) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double sv[PT / 32];
  __shared__ int si[PT / 32];
  __shared__ double s_dp;
  __shared__ int s_p;
  __shared__ double s_lp[PB];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t nblk = gridDim.x;
  const int64_t per = (p.m + nblk - 1) / nblk;
  const int64_t r0 = blockIdx.x * per, r1 = min(p.m, r0 + per);

  local_argmax(p, r0, r1, p.k0 & 1, sv, si);
  grid.sync();
  for (int j = p.k0; j < p.k1; ++j) {
    const int slot = j & 1;
    // every CTA reduces the partials redundantly (identical result everywhere)
    if (warp == 0) {
      double gv = -INFINITY;
      int gi = 0x7fffffff;
      for (int b = lane; b < (int)nblk; b += 32) {
        const double v = __ldcg(p.red_v + slot * 1024 + b);
        const int ii = __ldcg(p.red_i + slot * 1024 + b);
        if (better(v, ii, gv, gi)) {
          gv = v;
          gi = ii;
        }
      }
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, gv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, gi, o);
        if (better(ov, oi, gv, gi)) {
          gv = ov;
          gi = oi;
        }
      }
      if (lane == 0) {
        s_dp = gv;
        s_p = gi;
      }
    }
    __syncthreads();
    const double dp = s_dp;
    const int pv = s_p;
    // factorisation finished: the remaining pivots are rounding noise.  The test is
    // uniform across the grid (every CTA reduced the same partials); rank stays j.
    if (!(dp > p.tol)) return;
    const double ljj = sqrt(dp);
    for (int t = p.k0 + tid; t < j; t += PT)
      s_lp[t - p.k0] = __ldcg(p.L + (int64_t)t * p.ldl + pv);
    __syncthreads();
    const double* acol = p.A + (int64_t)pv * p.lda;
    const double rl = 1.0 / ljj;
    for (int64_t i = r0 + tid; i < r1; i += PT) {
      double li;
      if (i == pv) {
        li = ljj;
        p.d[i] = -INFINITY;
      } else if (p.d[i] == -INFINITY) {
        li = 0.0;  // already pivoted: L is lower triangular in pivot order
      } else {
        double s = i <= pv ? acol[i] : p.A[i * p.lda + pv];  // only the upper part of A is kept up to date
        for (int t = p.k0; t < j; ++t) s -= p.L[(int64_t)t * p.ldl + i] * s_lp[t - p.k0];
        li = s * rl;
        p.d[i] -= li * li;
      }
      p.L[(int64_t)j * p.ldl + i] = li;
    }
    if (tid == 0 && pv >= r0 && pv < r1) p.piv[j] = pv;
    if (blockIdx.x == 0 && tid == 0) *p.rank = j + 1;
    __syncthreads();
    local_argmax(p, r0, r1, slot ^ 1, sv, si);  // partials for column j+1
    grid.sync();
  }
}

// The shared-memory form of pstrf_panel (the CTA's rows of the panel fit in shared memory):
// per column, the critical path between two grid barriers is
//   reduce the argmax partials -> fetch the pivot row of the panel (and, overlapped with it,
//   this thread's entry of the pivot column of A) -> the update dot products -> the CTA's
//   argmax partial for the next column.
// The running diagonal of the CTA's rows lives in shared memory for the whole panel (written
// back on exit), the dot products are split over RT threads per row (RT independent partial
// sums, combined by shuffles in a fixed order) and the argmax partial is one warp's reduction
// of shared memory.  Same pivots and the same factor up to the summation order of the dots.
constexpr int RT = 4;  // threads per row in the update dot products
__global__ void __launch_bounds__(PT) pstrf_panel_sm(Params p) {
  extern __shared__ double s_rows[];
  cg::grid_group grid = cg::this_grid();
  __shared__ double s_dp;
  __shared__ int s_p;
  __shared__ double s_lp[PB];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t nblk = gridDim.x;
  const int64_t per = (p.m + nblk - 1) / nblk;
  const int64_t r0 = blockIdx.x * per, r1 = min(p.m, r0 + per);
  const int nr = r1 > r0 ? (int)(r1 - r0) : 0;
  double* s_d = s_rows + (int64_t)per * PB;  // running diagonal of rows [r0, r1)
  for (int i = tid; i < nr; i += PT) s_d[i] = p.d[r0 + i];
  __syncthreads();
  // warp 0: argmax of s_d (ties -> smallest index) -> partials[slot][blockIdx.x]
  auto cta_argmax = [&](int slot) {
    if (warp != 0) return;
    double bv = -INFINITY;
    int bi = 0x7fffffff;
    for (int i = lane; i < nr; i += 32) {
      const double v = s_d[i];
      if (better(v, (int)(r0 + i), bv, bi)) {
        bv = v;
        bi = (int)(r0 + i);
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (better(ov, oi, bv, bi)) {
        bv = ov;
        bi = oi;
      }
    }
    if (lane == 0) {
      p.red_v[slot * 1024 + blockIdx.x] = bv;
      p.red_i[slot * 1024 + blockIdx.x] = bi;
    }
  };
  auto write_back = [&]() {
    for (int i = tid; i < nr; i += PT) p.d[r0 + i] = s_d[i];
  };
  cta_argmax(p.k0 & 1);
  grid.sync();
  const int sub = tid % RT;
  for (int j = p.k0; j < p.k1; ++j) {
    const int slot = j & 1;
    if (warp == 0) {
      double gv = -INFINITY;
      int gi = 0x7fffffff;
      for (int b = lane; b < (int)nblk; b += 32) {
        const double v = __ldcg(p.red_v + slot * 1024 + b);
        const int ii = __ldcg(p.red_i + slot * 1024 + b);
        if (better(v, ii, gv, gi)) {
          gv = v;
          gi = ii;
        }
      }
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, gv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, gi, o);
        if (better(ov, oi, gv, gi)) {
          gv = ov;
          gi = oi;
        }
      }
      if (lane == 0) {
        s_dp = gv;
        s_p = gi;
      }
    }
    __syncthreads();
    const double dp = s_dp;
    const int pv = s_p;
    if (!(dp > p.tol)) {  // uniform across the grid: the remaining pivots are rounding noise
      write_back();
      return;
    }
    const double ljj = sqrt(dp);
    const int nj = j - p.k0;
    for (int t = tid; t < nj; t += PT) s_lp[t] = __ldcg(p.Lrm + (int64_t)pv * PB + t);
    // this thread's first row's entry of the pivot column, in flight with the pivot-row fetch
    const double* acol = p.A + (int64_t)pv * p.lda;
    const int row_first = tid / RT;
    double a_first = 0.0;
    // (only the upper part of the working matrix is kept up to date by the trailing updates:
    // entry (i, pv) is read as (min, max))
    if (sub == 0 && row_first < nr) {
      const int64_t i0 = r0 + row_first;
      a_first = i0 <= pv ? acol[i0] : p.A[i0 * p.lda + pv];
    }
    __syncthreads();
    const double rl = 1.0 / ljj;
    for (int rb = 0; rb < nr; rb += PT / RT) {
      const int il = rb + tid / RT;  // local row (uniform within a group of RT lanes)
      const bool live = il < nr;
      const int64_t i = r0 + il;
      const double di = live ? s_d[il] : -INFINITY;
      const bool upd = live && i != pv && di != -INFINITY;
      double part = 0.0;
      if (upd) {
        const double* sr = s_rows + il;
        for (int t = sub; t < nj; t += RT) part = fma(-sr[(int64_t)t * per], s_lp[t], part);
      }
      // fixed-order combination of the RT partial sums (lanes of a group are consecutive)
      part += __shfl_xor_sync(0xffffffffu, part, 1);
      part += __shfl_xor_sync(0xffffffffu, part, 2);
      if (live && sub == 0) {
        double li;
        if (i == pv) {
          li = ljj;
          s_d[il] = -INFINITY;
        } else if (di == -INFINITY) {
          li = 0.0;  // already pivoted: L is lower triangular in pivot order
        } else {
          const double a = rb == 0 ? a_first : (i <= pv ? acol[i] : p.A[i * p.lda + pv]);
          li = (a + part) * rl;
          s_d[il] = di - li * li;
        }
        p.L[(int64_t)j * p.ldl + i] = li;
        s_rows[(int64_t)nj * per + il] = li;
        p.Lrm[i * PB + nj] = li;
      }
    }
    if (tid == 0 && pv >= r0 && pv < r1) p.piv[j] = pv;
    if (blockIdx.x == 0 && tid == 0) *p.rank = j + 1;
    __syncthreads();
    cta_argmax(slot ^ 1);  // partials for column j+1
    grid.sync();
  }
  write_back();
}

__global__ void diag_init(const double* G, int64_t ldg, int64_t m, double* A, int64_t lda, double* d) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= m * m) return;
  const int64_t j = e / m, i = e % m;
  const double v = G[j * ldg + i];
  A[j * lda + i] = v;
  if (i == j) d[i] = v;
}

__global__ void max_diag_kernel(const double* d, int64_t m, double* out) {
  __shared__ double red[256];
  double mx = 0.0;
  for (int64_t i = threadIdx.x; i < m; i += 256) mx = fmax(mx, fabs(d[i]));
  red[threadIdx.x] = mx;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = red[0];
}

// y = G x (G symmetric, column-major): y_j = G[:, j] . x, one warp per column (contiguous reads,
// four independent partial sums per lane, fixed-order combination)
__global__ void __launch_bounds__(256) gemv_sym(const double* __restrict__ G, int64_t ldg, int64_t m,
                                                const double* __restrict__ x, double* __restrict__ y) {
  const int64_t j = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (j >= m) return;
  const double* g = G + j * ldg;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  int64_t i = lane;
  for (; i + 96 < m; i += 128) {
    s0 = fma(g[i], x[i], s0);
    s1 = fma(g[i + 32], x[i + 32], s1);
    s2 = fma(g[i + 64], x[i + 64], s2);
    s3 = fma(g[i + 96], x[i + 96], s3);
  }
  for (; i < m; i += 32) s0 = fma(g[i], x[i], s0);
  double s = (s0 + s1) + (s2 + s3);
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) y[j] = s;
}

// x = y / ||y||, out = ||y|| (single CTA, fixed-order reduction)
__global__ void normalise(const double* y, int64_t m, double* x, double* out) {
  __shared__ double red[256];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < m; i += 256) s += y[i] * y[i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int k = 128; k > 0; k >>= 1) {
    if (threadIdx.x < k) red[threadIdx.x] += red[threadIdx.x + k];
    __syncthreads();
  }
  const double nrm = sqrt(red[0]);
  for (int64_t i = threadIdx.x; i < m; i += 256) x[i] = nrm > 0.0 ? y[i] / nrm : 0.0;
  if (threadIdx.x == 0) out[0] = nrm;
}

__global__ void fill_value(double* x, int64_t m, double v) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m) x[i] = v;
}

}  // namespace pc

size_t pstrf_workspace_bytes(int64_t m) {
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  const int64_t ld = (m + 1) & ~int64_t(1);
  size_t o = al((size_t)ld * m * 8);          // A
  o += al((size_t)m * 8);                       // d
  o += al(2048 * 8) + al(2048 * 4) + al(64);    // partials (2 x 1024) + rank + scal
  o += 2 * al((size_t)m * 8);                   // power-iteration vectors
  o += al((size_t)m * pc::PB * 8);              // row-major panel copy
  o += al(gemm_workspace_bytes(m, m, pc::PB, 1, 0));
  return o;
}

// G (m x m) -> L (m x r, rows in original order), piv (r), rank r (host).
// tol_rel: stop when the largest remaining pivot <= tol_rel * max_i |G_ii|.
int pstrf_run(const double* G, int64_t ldg, int64_t m, double* L, int64_t ldl, int* piv, double tol_rel,
              double tol_lam, int64_t* rank_out, void* ws, size_t ws_bytes, cudaStream_t st) {
  using namespace pc;
  HP_REQUIRE(ws_bytes >= pstrf_workspace_bytes(m), "pstrf: workspace too small");
  *rank_out = 0;
  if (m == 0) return HP_OK;
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  const int64_t lda = (m + 1) & ~int64_t(1);
  char* base = static_cast<char*>(ws);
  size_t o = 0;
  double* A = reinterpret_cast<double*>(base + o);
  o += al((size_t)lda * m * 8);
  double* d = reinterpret_cast<double*>(base + o);
  o += al((size_t)m * 8);
  double* red_v = reinterpret_cast<double*>(base + o);
  o += al(2048 * 8);
  int* red_i = reinterpret_cast<int*>(base + o);
  o += al(2048 * 4);
  int* rank = reinterpret_cast<int*>(base + o);
  double* scal = reinterpret_cast<double*>(base + o + 16);
  double* lam_est = reinterpret_cast<double*>(base + o + 32);
  o += al(64);
  double* px = reinterpret_cast<double*>(base + o);
  o += al((size_t)m * 8);
  double* py = reinterpret_cast<double*>(base + o);
  o += al((size_t)m * 8);
  double* Lrm = reinterpret_cast<double*>(base + o);
  o += al((size_t)m * PB * 8);
  void* gws = base + o;
  const size_t gwsb = ws_bytes - o;

  diag_init<<<(unsigned)ceil_div(m * m, 256), 256, 0, st>>>(G, ldg, m, A, lda, d);
  HP_CHECK_LAUNCH("diag_init");
  max_diag_kernel<<<1, 256, 0, st>>>(d, m, scal);
  HP_CHECK_LAUNCH("max_diag");
  HP_CHECK_CUDA(zero_async(rank, sizeof(int), st));
  // lower bound of lambda_max by power iteration: ||G x|| <= lambda_max for ||x|| = 1
  // host read-backs through this thread's PINNED scratch: a pageable device-to-host copy can
  // queue behind unrelated host-to-device transfers (the e2e leaf uploads on the copy stream)
  char* pin = pinned_scratch();
  HP_REQUIRE(pin != nullptr, "pstrf: pinned host scratch unavailable");
  double* pin_lam = reinterpret_cast<double*>(pin + 128);
  double* pin_scal = reinterpret_cast<double*>(pin + 136);
  int* pin_rank = reinterpret_cast<int*>(pin + 144);
  double host_lam = 0.0;
  if (tol_lam > 0.0) {
    fill_value<<<(unsigned)ceil_div(m, 256), 256, 0, st>>>(px, m, 1.0 / sqrt((double)m));
    HP_CHECK_LAUNCH("fill_value");
    for (int it = 0; it < 8; ++it) {
      gemv_sym<<<(unsigned)ceil_div(m * 32, 256), 256, 0, st>>>(A, lda, m, px, py);
      HP_CHECK_LAUNCH("gemv_sym");
      normalise<<<1, 256, 0, st>>>(py, m, px, lam_est);
      HP_CHECK_LAUNCH("normalise");
    }
    HP_CHECK_CUDA(d2h_small(pin_lam, lam_est, sizeof(double), st));
  }
  double host_scal = 0.0;
  HP_CHECK_CUDA(d2h_small(pin_scal, scal, sizeof(double), st));
  HP_CHECK_CUDA(cudaStreamSynchronize(st));
  if (tol_lam > 0.0) host_lam = *pin_lam;
  host_scal = *pin_scal;
  if (!(host_scal > 0.0)) return HP_OK;  // all-zero Gramian: rank 0

  int dev = 0, nsm = 148, per_sm = 1;
  HP_CHECK_CUDA(cudaGetDevice(&dev));
  HP_CHECK_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  // one CTA per SM (at most one per 64 rows); the CTA's panel rows in shared memory when they fit
  const int rows_per_cta = 64;
  int grid = (int)std::min<int64_t>((int64_t)nsm, ceil_div(m, rows_per_cta));
  grid = std::max(1, std::min(grid, 1024));
  const int64_t per = ceil_div(m, grid);
  const size_t rows_smem = (size_t)per * (PB + 1) * 8;  // panel rows + running diagonal
  const bool srows = rows_smem <= 200 * 1024;
  static std::atomic<unsigned long long> configured{0};
  const int rc0 = once_per_device(configured, []() -> int {
    HP_CHECK_CUDA(cudaFuncSetAttribute(pstrf_panel_sm, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    return (int)HP_OK;
  });
  if (rc0 != HP_OK) return rc0;
  HP_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
      &per_sm, srows ? (const void*)pstrf_panel_sm : (const void*)pstrf_panel, PT, srows ? rows_smem : 0));
  HP_REQUIRE(per_sm >= 1, "pstrf: the panel kernel does not fit on an SM");

  Params p{};
  p.A = A;
  p.lda = lda;
  p.m = m;
  p.L = L;
  p.ldl = ldl;
  p.d = d;
  p.piv = piv;
  p.red_v = red_v;
  p.red_i = red_i;
  p.rank = rank;
  p.Lrm = Lrm;
  p.tol = std::max(tol_rel * host_scal, tol_lam * host_lam);
  int host_rank = 0;
  for (int64_t k0 = 0; k0 < m; k0 += PB) {
    p.k0 = (int)k0;
    p.k1 = (int)std::min<int64_t>(m, k0 + PB);
    void* args[] = {&p};
    if (srows)
      HP_CHECK_CUDA(cudaLaunchCooperativeKernel((void*)pstrf_panel_sm, grid, PT, args, rows_smem, st));
    else
      HP_CHECK_CUDA(cudaLaunchCooperativeKernel((void*)pstrf_panel, grid, PT, args, 0, st));
    count_launches(1);
    HP_CHECK_CUDA(d2h_small(pin_rank, rank, sizeof(int), st));
    HP_CHECK_CUDA(cudaStreamSynchronize(st));
    host_rank = *pin_rank;
    const int64_t done = host_rank;
    if (done < p.k1 || done >= m) break;
    // trailing update of the whole working matrix: A -= L_panel L_panel^T
    VecSet a{L + k0 * ldl, ldl, nullptr};
    // (upper part only, sym = 2: the panel kernels read entry (i, pv) as (min, max), and the mirror
    // was a third of this update's memory traffic, all of it scattered 8-byte stores)
    int rc = gemm_run(false, false, m, m, p.k1 - k0, a, a, (ldl % 2 == 0), -1.0, 1.0, A, lda, nullptr, nullptr,
                      nullptr, 2, 0, gws, gwsb, st);
    if (rc) return rc;
  }
  *rank_out = host_rank;
  return HP_OK;
}

}  // namespace hp
