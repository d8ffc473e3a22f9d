// Per-node POD steps around the contractions:
//   K3 truncation scan   (pod.py:190-205, 278-289)
//   K5 drift reduction   (pod.py:245-247) + CholQR re-orthonormalisation
//      (same span and Gram-Schmidt order as the MGS sweep of pod.py:227-237)
//   K6 sign convention   (pod.py:214-224)
// plus layout helpers (row-major upload transpose, sqrt(w) row scaling for
// weighted spaces pod.py:76-84, column scaling for ModeSet.scaled pod.py:160-162).
#include <algorithm>
#include <cmath>

#include "hp_common.cuh"

namespace hp {

int gemm_run(bool a_kmajor, bool b_kmajor, int64_t M, int64_t N, int64_t K, VecSet A, VecSet B, bool aligned16,
             double alpha, double beta, double* C, int64_t ldc, const double* row_scale, const double* col_scale,
             const double* col_div, int sym, int b_upper, void* ws, size_t ws_bytes, cudaStream_t st);
size_t gemm_workspace_bytes(int64_t M, int64_t N, int64_t K, int sym, int b_upper);
int scale_run(const double* src, int64_t lds, int64_t rows, int64_t cols, const double* rs, const double* rd,
              const double* cs, double* dst, int64_t ldd, cudaStream_t st);

// ------------------------------------------------------------------ K3 truncation
// info[0] = lam_max, info[1] = nkeep, info[2] = N, info[3] = tail_energy
//
// Bit-for-bit the reference's arithmetic (pod.py:198-205, 284-289):
//   keep  = lam >= cutoff * lam_max * m                       (a prefix: lam is descending)
//   sig   = sqrt(lam_keep)
//   tails = reversed sequential cumsum of sig*sig (np.cumsum: one add per entry, smallest first;
//           sig*sig rounded before the add -- no FMA contraction)
//   N     = first index with tails[N] <= eps^2                 (np.argmax of the mask)
//   tail  = np.sum(lam_keep[N:])                              (NumPy's pairwise summation)
// The cumsum is inherently sequential; it runs on one thread from the smallest kept value
// upward and stops as soon as the running tail exceeds eps^2 (rounding is monotone, so no
// later index can satisfy the budget again) -- it only walks the discarded tail.
constexpr int TR_T = 256;

// numpy/_core/src/umath/loops_utils.h.src pairwise_sum (PW_BLOCKSIZE 128, 8-way unroll), the
// summation np.sum applies to a contiguous float64 array.
__device__ double np_pairwise_sum(const double* a, int64_t n) {
  if (n < 8) {
    double res = 0.0;
    for (int64_t i = 0; i < n; ++i) res = __dadd_rn(res, a[i]);
    return res;
  }
  if (n <= 128) {
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    int64_t i = 8;
    for (; i < n - (n % 8); i += 8) {
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], a[i + j]);
    }
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __dadd_rn(res, a[i]);
    return res;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  return __dadd_rn(np_pairwise_sum(a, n2), np_pairwise_sum(a + n2, n - n2));
}

__global__ void __launch_bounds__(TR_T) truncate_kernel(const double* lam, int64_t n, double eps, double cutoff,
                                                        int64_t m, double* sigma, double* info) {
  __shared__ unsigned long long sh_nkeep;
  const int tid = threadIdx.x;
  const double lam_max = n > 0 ? lam[0] : 0.0;
  if (!(lam_max > 0.0)) {
    if (tid == 0) {
      info[0] = lam_max;
      info[1] = 0;
      info[2] = 0;
      info[3] = 0.0;
    }
    return;
  }
  const double thr = __dmul_rn(__dmul_rn(cutoff, lam_max), (double)m);
  if (tid == 0) sh_nkeep = 0;
  __syncthreads();
  unsigned long long local_cnt = 0;
  for (int64_t i = tid; i < n; i += TR_T) local_cnt += (lam[i] >= thr);
  atomicAdd(&sh_nkeep, local_cnt);
  __syncthreads();
  const int64_t nk = (int64_t)sh_nkeep;
  for (int64_t i = tid; i < nk; i += TR_T) sigma[i] = __dsqrt_rn(lam[i]);
  if (tid != 0) return;
  const double eps2 = __dmul_rn(eps, eps);
  int64_t N = nk;  // tails[nk] = 0 always satisfies the budget
  double run = 0.0;
  for (int64_t i = nk - 1; i >= 0; --i) {
    const double si = __dsqrt_rn(lam[i]);
    run = __dadd_rn(run, __dmul_rn(si, si));
    if (run <= eps2)
      N = i;
    else
      break;
  }
  info[0] = lam_max;
  info[1] = (double)nk;
  info[2] = (double)N;
  info[3] = np_pairwise_sum(lam + N, nk - N);
}

int truncate_run(const double* lam, int64_t n, double eps, double cutoff, int64_t m, double* sigma, double* info,
                 cudaStream_t st) {
  truncate_kernel<<<1, TR_T, 0, st>>>(lam, n, eps, cutoff, m, sigma, info);
  HP_CHECK_LAUNCH("truncate_kernel");
  return HP_OK;
}

// ------------------------------------------------------------------ K5 drift
__device__ __forceinline__ void atomic_max_pos(double* addr, double v) {
  // non-negative doubles order like their bit patterns
  atomicMax(reinterpret_cast<unsigned long long*>(addr), (unsigned long long)__double_as_longlong(v));
}

__global__ void drift_kernel(const double* C, int64_t ldc, int64_t n, double* out) {
  __shared__ double red[256];
  double mx = 0.0;
  const int64_t total = n * n;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / n, i = e % n;
    double v = C[j * ldc + i] - (i == j ? 1.0 : 0.0);
    v = fabs(v);
    if (!(v <= mx)) mx = v;  // propagates NaN as +inf-ish below
  }
  if (mx != mx) mx = INFINITY;
  red[threadIdx.x] = mx;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x == 0) atomic_max_pos(out, red[0]);
}

int drift_run(const double* C, int64_t ldc, int64_t n, double* out, cudaStream_t st) {
  HP_CHECK_CUDA(zero_async(out, sizeof(double), st));
  if (n == 0) return HP_OK;
  const int64_t blocks = std::min<int64_t>(ceil_div(n * n, 256), 4 * 148);
  drift_kernel<<<(unsigned)blocks, 256, 0, st>>>(C, ldc, n, out);
  HP_CHECK_LAUNCH("drift_kernel");
  return HP_OK;
}

// ------------------------------------------------------------------ K6 signs
// One CTA per mode: argmax |U[:,k]| (first index on ties), sign -> +1 if 0,
// flip U[:,k] (and R[:,k] when given).  Optionally also writes the signed
// sigma*sign scale the parent consumes.
// One CTA of ST threads per column.  The scan keeps 8 independent loads in flight per thread
// (the former one-load-at-a-time loop was latency bound: ~1.2 ms per config-2 merge for 78
// columns of 500k rows); rows are visited in increasing order per thread and the tree reduction
// prefers the smaller index on ties, so the winner is the first index of the largest |u|.
constexpr int ST = 1024;
__global__ void __launch_bounds__(ST) signs_kernel(double* U, int64_t ldu, int64_t d, double* R, int64_t ldr,
                                                   int64_t mr, double* sign_out) {
  __shared__ double bv[ST];
  __shared__ int64_t bi[ST];
  __shared__ double sgn;
  const int64_t k = blockIdx.x;
  double* col = U + k * ldu;
  double best = -1.0;
  int64_t bidx = 0;
  int64_t i = threadIdx.x;
  for (; i + 7 * (int64_t)ST < d; i += 8 * (int64_t)ST) {
    double a[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) a[u] = fabs(col[i + u * (int64_t)ST]);
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (a[u] > best) {
        best = a[u];
        bidx = i + u * (int64_t)ST;
      }
  }
  for (; i < d; i += ST) {
    const double a = fabs(col[i]);
    if (a > best) {
      best = a;
      bidx = i;
    }
  }
  bv[threadIdx.x] = best;
  bi[threadIdx.x] = bidx;
  __syncthreads();
  for (int s = ST / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      const double ov = bv[threadIdx.x + s];
      const int64_t oi = bi[threadIdx.x + s];
      if (ov > bv[threadIdx.x] || (ov == bv[threadIdx.x] && oi < bi[threadIdx.x])) {
        bv[threadIdx.x] = ov;
        bi[threadIdx.x] = oi;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double v = col[bi[0]];
    sgn = v < 0.0 ? -1.0 : 1.0;
    if (sign_out) sign_out[k] = sgn;
  }
  __syncthreads();
  if (sgn < 0.0) {
    for (int64_t j = threadIdx.x; j < d; j += ST) col[j] = -col[j];
    if (R)
      for (int64_t j = threadIdx.x; j < mr; j += ST) R[k * ldr + j] = -R[k * ldr + j];
  }
}

// per column: largest |u| of the local row block and its global row index (first on ties)
__global__ void col_absmax_kernel(const double* U, int64_t ldu, int64_t rows, int64_t row_offset, double* vals,
                                  int64_t* idx) {
  __shared__ double bv[256];
  __shared__ int64_t bi[256];
  const int64_t k = blockIdx.x;
  const double* col = U + k * ldu;
  double best = -1.0;
  int64_t bidx = 0;
  for (int64_t i = threadIdx.x; i < rows; i += blockDim.x) {
    const double a = fabs(col[i]);
    if (a > best) {
      best = a;
      bidx = i;
    }
  }
  bv[threadIdx.x] = best;
  bi[threadIdx.x] = bidx;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      const double ov = bv[threadIdx.x + s];
      const int64_t oi = bi[threadIdx.x + s];
      if (ov > bv[threadIdx.x] || (ov == bv[threadIdx.x] && oi < bi[threadIdx.x])) {
        bv[threadIdx.x] = ov;
        bi[threadIdx.x] = oi;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    vals[k] = rows > 0 ? bv[0] : -1.0;
    idx[k] = row_offset + bi[0];
  }
}

// per column: sum_i w_i a_i^2 (w nullable = Euclidean), fixed-order block reduction
// (InnerProductSpace.norms_sq, pod.py:93-97)
__global__ void col_norms_sq_kernel(const double* A, int64_t lda, int64_t rows, const double* w, double* out) {
  __shared__ double red[256];
  const double* col = A + (int64_t)blockIdx.x * lda;
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < rows; i += 256) {
    const double a = col[i];
    s += w ? a * (w[i] * a) : a * a;
  }
  red[threadIdx.x] = s;
  __syncthreads();
  for (int st = 128; st > 0; st >>= 1) {
    if (threadIdx.x < st) red[threadIdx.x] += red[threadIdx.x + st];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[blockIdx.x] = red[0];
}

int col_norms_sq_run(const double* A, int64_t lda, int64_t rows, int64_t cols, const double* w, double* out,
                     cudaStream_t st) {
  if (cols == 0) return HP_OK;
  col_norms_sq_kernel<<<(unsigned)cols, 256, 0, st>>>(A, lda, rows, w, out);
  HP_CHECK_LAUNCH("col_norms_sq_kernel");
  return HP_OK;
}

// dst <- dst + src (contiguous; the fixed-tree shard sums of the row-distributed root)
__global__ void add_kernel(double* dst, const double* src, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = __dadd_rn(dst[i], src[i]);
}

int add_run(double* dst, const double* src, int64_t n, cudaStream_t st) {
  if (n <= 0) return HP_OK;
  const unsigned grid = (unsigned)std::min<int64_t>(ceil_div(n, 256), 8 * 148);
  add_kernel<<<grid, 256, 0, st>>>(dst, src, n);
  HP_CHECK_LAUNCH("add_kernel");
  return HP_OK;
}

int col_absmax_run(const double* U, int64_t ldu, int64_t rows, int64_t N, int64_t row_offset, double* vals,
                   int64_t* idx, cudaStream_t st) {
  if (N == 0) return HP_OK;
  col_absmax_kernel<<<(unsigned)N, 256, 0, st>>>(U, ldu, rows, row_offset, vals, idx);
  HP_CHECK_LAUNCH("col_absmax_kernel");
  return HP_OK;
}

int signs_run(double* U, int64_t ldu, int64_t d, int64_t N, double* R, int64_t ldr, int64_t mr, double* sign_out,
              cudaStream_t st) {
  if (N == 0) return HP_OK;
  signs_kernel<<<(unsigned)N, ST, 0, st>>>(U, ldu, d, R, ldr, mr, sign_out);
  HP_CHECK_LAUNCH("signs_kernel");
  return HP_OK;
}

// ------------------------------------------------------------------ Cholesky (CholQR)
constexpr int CB = 64;

// Factor the kb x kb diagonal block at A[k0,k0] (lower, in place), write its inverse into
// Linv[k0.., k0..] (lower) and flag a non-positive pivot.
// Right-looking and fused: step j takes the pivot, scales column j of L and row j of
// X = L^{-1} (X solves L X = I; R holds the running right-hand side), then applies the rank-1
// updates to the trailing block of A and to R -- 64 steps of 3 barriers, no serial loops.
__global__ void __launch_bounds__(256) potrf_diag(double* A, int64_t lda, int64_t k0, int kb, double* Linv, int64_t ldi,
                                                   int* info) {
  extern __shared__ double pd_smem[];
  double (*L)[CB + 1] = reinterpret_cast<double (*)[CB + 1]>(pd_smem);
  double (*X)[CB + 1] = reinterpret_cast<double (*)[CB + 1]>(pd_smem + CB * (CB + 1));
  __shared__ int bad;
  const int tid = threadIdx.x;
  if (tid == 0) bad = 0;
  for (int e = tid; e < CB * CB; e += 256) {
    const int j = e / CB, i = e % CB;
    L[i][j] = (i < kb && j < kb && i >= j) ? A[(k0 + j) * lda + k0 + i] : 0.0;
    X[i][j] = (i == j) ? 1.0 : 0.0;
  }
  // pivot 0; every later pivot is taken by the thread that applied its last update (below)
  if (tid == 0 && kb > 0) {
    const double d0 = L[0][0];
    if (!(d0 > 0.0)) {
      bad = 1;
      L[0][0] = 1.0;
    } else {
      L[0][0] = sqrt(d0);
    }
  }
  __syncthreads();
  // One barrier per column: column j of L and row j of R = L^{-1} are scaled by 1 / L[j][j] on the
  // fly where they are read (in place only at the write-back), so the products are the ones an
  // in-place scaling would form -- same bits, no separate scaling phase.
  for (int j = 0; j < kb; ++j) {
    const double rpiv = 1.0 / L[j][j];
    // trailing A -= l_j l_j^T (lower part) and R[i][c] -= L[i][j] R[j][c] (i > j, c <= j):
    // thread = (column c, row phase), no index division
    {
      const int c = tid & (CB - 1);
      const double xjc = X[j][c] * rpiv, lcj = L[c][j] * rpiv;
      for (int ii = j + 1 + (tid >> 6); ii < kb; ii += 256 / CB) {
        const double lij = L[ii][j] * rpiv;
        if (c <= j)
          X[ii][c] -= lij * xjc;
        else if (c <= ii)
          L[ii][c] -= lij * lcj;
      }
    }
    if (tid == j + 1 && j + 1 < kb) {  // this thread just applied the last update of the next pivot
      const double dn = L[j + 1][j + 1];
      if (!(dn > 0.0)) {
        bad = 1;
        L[j + 1][j + 1] = 1.0;
      } else {
        L[j + 1][j + 1] = sqrt(dn);
      }
    }
    __syncthreads();
  }
  for (int e = tid; e < kb * kb; e += 256) {
    const int j = e / kb, i = e % kb;
    const double li = i == j ? L[i][i] : L[i][j] * (1.0 / L[j][j]);
    A[(k0 + j) * lda + k0 + i] = (i >= j) ? li : 0.0;
    Linv[(k0 + j) * ldi + k0 + i] = (i >= j) ? X[i][j] * (1.0 / L[i][i]) : 0.0;
  }
  if (tid == 0 && bad) atomicOr(info, 1);
}

// Cholesky factor AND its inverse, C = L L^T, Linv = L^{-1}, by recursive halving
// (C = [[C11, .], [C21, C22]]):
//   L11, X11 = chol_inv(C11);  L21 = C21 X11^T;  C22 -= L21 L21^T;  L22, X22 = chol_inv(C22);
//   X21 = -X22 (L21 X11)
// The 64 x 64 leaves are potrf_diag; everything else is DMMA GEMMs whose big instances are
// full-size GEMM shapes (the former block-column loop launched 3 small kernels per 64 columns
// and re-wrote the whole trailing matrix each time).  C's lower part is consumed.  T: scratch
// of ldt x chol_t_cols(n) doubles.
static int chol_inv_rec(double* A, int64_t lda, int64_t o, int64_t n, double* Linv, int64_t ldi, double* T,
                        int64_t ldt, int* info, void* ws, size_t ws_bytes, cudaStream_t st) {
  if (n <= CB) {
    static std::atomic<unsigned long long> configured{0};
    const int pd_smem = 2 * CB * (CB + 1) * 8;
    const int rc0 = once_per_device(configured, [&]() -> int {
      HP_CHECK_CUDA(cudaFuncSetAttribute(potrf_diag, cudaFuncAttributeMaxDynamicSharedMemorySize, pd_smem));
      return (int)HP_OK;
    });
    if (rc0 != HP_OK) return rc0;
    potrf_diag<<<1, 256, pd_smem, st>>>(A, lda, o, (int)n, Linv, ldi, info);
    HP_CHECK_LAUNCH("potrf_diag");
    return HP_OK;
  }
  int64_t h = ceil_div(n / 2, CB) * CB;
  if (h >= n) h = n - CB;
  const int64_t n2 = n - h;
  const bool al = (lda % 2 == 0) && (ldi % 2 == 0) && (ldt % 2 == 0) && (o % 2 == 0) && (h % 2 == 0);
  int rc = chol_inv_rec(A, lda, o, h, Linv, ldi, T, ldt, info, ws, ws_bytes, st);
  if (rc) return rc;
  double* X11 = Linv + o * ldi + o;
  double* X21 = Linv + o * ldi + o + h;
  double* X22 = Linv + (o + h) * ldi + o + h;
  double* C21 = A + o * lda + o + h;
  double* C22 = A + (o + h) * lda + o + h;
  // T = L21 = C21 X11^T   (B(k, j) = X11(j, k): N-major operand)
  rc = gemm_run(false, false, n2, h, h, VecSet{C21, lda, nullptr}, VecSet{X11, ldi, nullptr}, al, 1.0, 0.0, T, ldt,
                nullptr, nullptr, nullptr, 0, 0, ws, ws_bytes, st);
  // C22 -= L21 L21^T
  if (!rc)
    rc = gemm_run(false, false, n2, n2, h, VecSet{T, ldt, nullptr}, VecSet{T, ldt, nullptr}, al, -1.0, 1.0, C22, lda,
                  nullptr, nullptr, nullptr, 1, 0, ws, ws_bytes, st);
  // X21 <- L21 X11 (parked in its final place), then T is free for the recursion
  if (!rc)
    rc = gemm_run(false, true, n2, h, h, VecSet{T, ldt, nullptr}, VecSet{X11, ldi, nullptr}, al, 1.0, 0.0, X21, ldi,
                  nullptr, nullptr, nullptr, 0, 0, ws, ws_bytes, st);
  if (!rc) rc = chol_inv_rec(A, lda, o + h, n2, Linv, ldi, T, ldt, info, ws, ws_bytes, st);
  // X21 = -X22 (L21 X11)
  if (!rc)
    rc = gemm_run(false, true, n2, h, n2, VecSet{X22, ldi, nullptr}, VecSet{X21, ldi, nullptr}, al, -1.0, 0.0, T, ldt,
                  nullptr, nullptr, nullptr, 0, 0, ws, ws_bytes, st);
  if (!rc) rc = scale_run(T, ldt, n2, h, nullptr, nullptr, nullptr, X21, ldi, st);
  return rc;
}

int64_t chol_t_cols(int64_t n) { return std::max<int64_t>(ceil_div(std::max<int64_t>(n, 1) / 2, CB) * CB, CB); }

int chol_inv_run(double* C, int64_t ldc, int64_t n, double* Linv, int64_t ldi, double* T, int* info, void* ws,
                 size_t ws_bytes, cudaStream_t st) {
  HP_CHECK_CUDA(zero_async(info, sizeof(int), st));
  if (n == 0) return HP_OK;
  HP_CHECK_CUDA(zero_2d_async(Linv, ldi, n, n, st));
  return chol_inv_rec(C, ldc, 0, n, Linv, ldi, T, (n + 1) & ~int64_t(1), info, ws, ws_bytes, st);
}

// ------------------------------------------------------------------ layout helpers
__global__ void transpose_rm_to_cm(const double* src, int64_t rows, int64_t cols, double* dst, int64_t ldd) {
  // src row-major rows x cols; dst col-major with leading dimension ldd
  __shared__ double tile[32][33];
  const int64_t c0 = (int64_t)blockIdx.x * 32, r0 = (int64_t)blockIdx.y * 32;
  for (int dy = threadIdx.y; dy < 32; dy += 8) {
    const int64_t r = r0 + dy, c = c0 + threadIdx.x;
    tile[dy][threadIdx.x] = (r < rows && c < cols) ? src[r * cols + c] : 0.0;
  }
  __syncthreads();
  for (int dy = threadIdx.y; dy < 32; dy += 8) {
    const int64_t c = c0 + dy, r = r0 + threadIdx.x;
    if (r < rows && c < cols) dst[c * ldd + r] = tile[threadIdx.x][dy];
  }
}

int transpose_run(const double* src, int64_t rows, int64_t cols, double* dst, int64_t ldd, cudaStream_t st) {
  if (rows == 0 || cols == 0) return HP_OK;
  dim3 grid((unsigned)ceil_div(cols, 32), (unsigned)ceil_div(rows, 32));
  transpose_rm_to_cm<<<grid, dim3(32, 8), 0, st>>>(src, rows, cols, dst, ldd);
  HP_CHECK_LAUNCH("transpose_rm_to_cm");
  return HP_OK;
}

// dst[:, j] = src[:, j] * (rs ? rs[i] : 1) / (rd ? rd[i] : 1) * (cs ? cs[j] : 1)
__global__ void scale_kernel(const double* src, int64_t lds, int64_t rows, int64_t cols, const double* rs,
                             const double* rd, const double* cs, double* dst, int64_t ldd) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= rows * cols) return;
  const int64_t j = e / rows, i = e % rows;
  double v = src[j * lds + i];
  if (rs) v *= rs[i];
  if (rd) v /= rd[i];
  if (cs) v *= cs[j];
  dst[j * ldd + i] = v;
}

int scale_run(const double* src, int64_t lds, int64_t rows, int64_t cols, const double* rs, const double* rd,
              const double* cs, double* dst, int64_t ldd, cudaStream_t st) {
  if (rows == 0 || cols == 0) return HP_OK;
  scale_kernel<<<(unsigned)ceil_div(rows * cols, 256), 256, 0, st>>>(src, lds, rows, cols, rs, rd, cs, dst, ldd);
  HP_CHECK_LAUNCH("scale_kernel");
  return HP_OK;
}

__global__ void finite_kernel(const double* src, int64_t lds, int64_t rows, int64_t cols, int* bad) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= rows * cols) return;
  const int64_t j = e / rows, i = e % rows;
  const double v = src[j * lds + i];
  if (!isfinite(v)) atomicOr(bad, 1);
}

int finite_check_run(const double* src, int64_t lds, int64_t rows, int64_t cols, int* bad, cudaStream_t st) {
  HP_CHECK_CUDA(zero_async(bad, sizeof(int), st));
  if (rows == 0 || cols == 0) return HP_OK;
  finite_kernel<<<(unsigned)ceil_div(rows * cols, 256), 256, 0, st>>>(src, lds, rows, cols, bad);
  HP_CHECK_LAUNCH("finite_kernel");
  return HP_OK;
}

// ------------------------------------------------------------------ sum of squares
// Deterministic two-pass reduction: fixed per-block partials, then one block
// sums them in index order (residual energy of actual_mean_error,
// hierarchy.py:249-253).
constexpr int SQ_BLOCKS = 1024;

__global__ void sumsq_partial(const double* A, int64_t lda, int64_t rows, int64_t cols, double* partial) {
  __shared__ double red[256];
  const int64_t total = rows * cols;
  double s = 0.0;
  for (int64_t e = (int64_t)blockIdx.x * 256 + threadIdx.x; e < total; e += (int64_t)SQ_BLOCKS * 256) {
    const int64_t j = e / rows, i = e % rows;
    const double v = A[j * lda + i];
    s += v * v;
  }
  red[threadIdx.x] = s;
  __syncthreads();
  for (int k = 128; k > 0; k >>= 1) {
    if (threadIdx.x < k) red[threadIdx.x] += red[threadIdx.x + k];
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = red[0];
}

__global__ void sumsq_final(const double* partial, double* out) {
  __shared__ double red[256];
  double s = 0.0;
  for (int i = threadIdx.x; i < SQ_BLOCKS; i += 256) s += partial[i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int k = 128; k > 0; k >>= 1) {
    if (threadIdx.x < k) red[threadIdx.x] += red[threadIdx.x + k];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = red[0];
}

int sumsq_run(const double* A, int64_t lda, int64_t rows, int64_t cols, double* out, double* partial,
              cudaStream_t st) {
  sumsq_partial<<<SQ_BLOCKS, 256, 0, st>>>(A, lda, rows, cols, partial);
  HP_CHECK_LAUNCH("sumsq_partial");
  sumsq_final<<<1, 256, 0, st>>>(partial, out);
  HP_CHECK_LAUNCH("sumsq_final");
  return HP_OK;
}

}  // namespace hp
