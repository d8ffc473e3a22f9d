#include <cstdio>
#include <cstdlib>
// extern "C" boundary of libhapod_b200.so (declared in include/hapod_b200.h).
// Plain pointers and sizes only; every entry returns an hp status code and
// leaves a thread-local message for hp_last_error().
#include <algorithm>
#include <atomic>
#include <cmath>
#include <mutex>
#include <string>

#include "hp_common.cuh"

namespace hp {

static thread_local std::string g_last_error;
static std::atomic<long long> g_launches{0};
void count_launches(long long n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
static std::atomic<int> g_debug{0};
int debug_flags() { return g_debug.load(std::memory_order_relaxed); }
void set_error(const std::string& msg) { g_last_error = msg; }
const char* last_error() { return g_last_error.c_str(); }

char* pinned_scratch() {
  thread_local char* buf = nullptr;
  if (!buf && cudaMallocHost(&buf, 512) != cudaSuccess) buf = nullptr;
  return buf;
}

int num_sms() {
  int dev = 0, n = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

int gemm_run(bool a_kmajor, bool b_kmajor, int64_t M, int64_t N, int64_t K, VecSet A, VecSet B, bool aligned16,
             double alpha, double beta, double* C, int64_t ldc, const double* row_scale, const double* col_scale,
             const double* col_div, int sym, int b_upper, void* ws, size_t ws_bytes, cudaStream_t st);
size_t gemm_workspace_bytes(int64_t M, int64_t N, int64_t K, int sym, int b_upper);
void gemm_set_nosplit(bool on);
void gemm_set_wavesplit(bool on);
bool gemm_plan_is_single_split(int64_t M, int64_t N, int64_t K, int sym);
size_t syev_workspace_bytes(int64_t n);
int64_t syev_padded_order(int64_t n);
int syev_run(const double* G, int64_t ldg, int64_t n, double* lam_desc, double* V, int64_t ldv, int64_t nvec,
             double tol_rel, double tol_abs, double tol_angle, double keep_floor, int max_sweeps, int refine,
             int* sweeps_out, double* flops_out, void* ws, size_t ws_bytes, cudaStream_t st, int64_t vrow0 = 0,
             int64_t vrow1 = -1);
int64_t syev_tri_max_order();
size_t syev_tri_workspace_bytes(int64_t n);
int syev_tri_run(const double* H, int64_t ldh, int64_t n, double floor_rel, double relgap_min, double* lam_desc,
                 double* W, int64_t ldw, int64_t* k_out, int* status_out, double* diag, void* ws, size_t ws_bytes,
                 cudaStream_t st);
int truncate_run(const double* lam, int64_t n, double eps, double cutoff, int64_t m, double* sigma, double* info,
                 cudaStream_t st);
int drift_run(const double* C, int64_t ldc, int64_t n, double* out, cudaStream_t st);
int signs_run(double* U, int64_t ldu, int64_t d, int64_t N, double* R, int64_t ldr, int64_t mr, double* sign_out,
              cudaStream_t st);
int64_t chol_t_cols(int64_t n);
int chol_inv_run(double* C, int64_t ldc, int64_t n, double* Linv, int64_t ldi, double* T, int* info, void* ws,
                 size_t ws_bytes, cudaStream_t st);
int transpose_run(const double* src, int64_t rows, int64_t cols, double* dst, int64_t ldd, cudaStream_t st);
int scale_run(const double* src, int64_t lds, int64_t rows, int64_t cols, const double* rs, const double* rd,
              const double* cs, double* dst, int64_t ldd, cudaStream_t st);
int finite_check_run(const double* src, int64_t lds, int64_t rows, int64_t cols, int* bad, cudaStream_t st);
int sumsq_run(const double* A, int64_t lda, int64_t rows, int64_t cols, double* out, double* partial,
              cudaStream_t st);
int add_run(double* dst, const double* src, int64_t n, cudaStream_t st);
int col_norms_sq_run(const double* A, int64_t lda, int64_t rows, int64_t cols, const double* w, double* out,
                     cudaStream_t st);
int col_absmax_run(const double* U, int64_t ldu, int64_t rows, int64_t N, int64_t row_offset, double* vals,
                   int64_t* idx, cudaStream_t st);
size_t pstrf_workspace_bytes(int64_t m);
int pstrf_run(const double* G, int64_t ldg, int64_t m, double* L, int64_t ldl, int* piv, double tol_rel,
              double tol_lam, int64_t* rank_out, void* ws, size_t ws_bytes, cudaStream_t st);

static inline VecSet vs(const hp_vecset& v) { return VecSet{v.base, v.ld, v.table}; }

// ---------------------------------------------------------------- re-orthonormalisation
// split-K partials of any GEMM the engine plans (splits x tiles <= 2 waves of 148 SMs)
static constexpr size_t kSplitKMax = (size_t)2 * 148 * 128 * 128 * 8;

struct ReorthoLayout {
  size_t off_X, off_A, off_Linv, off_T, off_info, off_gemm, total;
};

static ReorthoLayout reortho_layout(int64_t d, int64_t N, int64_t ldx) {
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  ReorthoLayout L;
  size_t o = 0;
  const int64_t ldn = (N + 1) & ~int64_t(1);
  L.off_X = o;
  o = al(o + (size_t)ldx * N * 8);
  L.off_A = o;
  o = al(o + (size_t)ldn * N * 8);
  L.off_Linv = o;
  o = al(o + (size_t)ldn * N * 8);
  L.off_T = o;
  o = al(o + (size_t)ldn * chol_t_cols(N) * 8);
  L.off_info = o;
  o = al(o + 16);
  L.off_gemm = o;
  // the Cholesky/inverse recursion's mid-size products may split K to fill the chip
  size_t g = std::max(gemm_workspace_bytes(N, N, d, 1, 0), kSplitKMax);
  o = al(o + g);
  L.total = o;
  return L;
}

// One CholQR pass: Y = X * L^{-T} where C = X^T X = L L^T.  C is consumed.
static int cholqr_pass(const double* X, int64_t ldx, int64_t d, int64_t N, double* C, int64_t ldc, double* Y,
                       int64_t ldy, const ReorthoLayout& L, char* base, size_t ws_bytes, cudaStream_t st,
                       int* host_info) {
  double* Linv = reinterpret_cast<double*>(base + L.off_Linv);
  double* T = reinterpret_cast<double*>(base + L.off_T);
  int* info = reinterpret_cast<int*>(base + L.off_info);
  void* gws = base + L.off_gemm;
  const size_t gwsb = ws_bytes - L.off_gemm;
  const int64_t ldn = (N + 1) & ~int64_t(1);
  int rc = chol_inv_run(C, ldc, N, Linv, ldn, T, info, gws, gwsb, st);
  if (rc) return rc;
  HP_CHECK_CUDA(d2h_small(host_info, info, sizeof(int), st));
  // Y = X * Linv^T : B(k, n) = Linv(n, k) -> N-major operand (vector k = column k of Linv), upper triangular
  VecSet a{X, ldx, nullptr};
  VecSet b{Linv, ldn, nullptr};
  rc = gemm_run(false, false, d, N, N, a, b, (ldx % 2 == 0) && (ldn % 2 == 0), 1.0, 0.0, Y, ldy, nullptr, nullptr,
                nullptr, 0, 1, gws, gwsb, st);
  return rc;
}

// drift below which one CholQR pass is already orthonormal to the rounding level
static constexpr double kSinglePassDrift = 1e-1;

static int gram_sym(const double* X, int64_t ldx, int64_t d, int64_t N, double* C, int64_t ldc, void* ws,
                    size_t wsb, cudaStream_t st) {
  VecSet a{X, ldx, nullptr};
  gemm_set_wavesplit(true);  // X^T X only feeds the drift and the Cholesky of CholQR
  const int rc = gemm_run(true, true, N, N, d, a, a, (ldx % 2 == 0), 1.0, 0.0, C, ldc, nullptr, nullptr, nullptr, 1,
                          0, ws, wsb, st);
  gemm_set_wavesplit(false);
  return rc;
}

__global__ void add_diag(double* C, int64_t ldc, int64_t n, double s) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) C[i * ldc + i] += s;
}

__global__ void trace_kernel(const double* C, int64_t ldc, int64_t n, double* out) {
  __shared__ double red[256];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += 256) s += C[i * ldc + i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int k = 128; k > 0; k >>= 1) {
    if (threadIdx.x < k) red[threadIdx.x] += red[threadIdx.x + k];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = red[0];
}

__global__ void block_gram_fill(double* G, int64_t ldg, int64_t n_old, int64_t m, const double* sigma) {
  // top-left diag(sigma^2) (pod.py:377) and the lower-left mirror of the mixed block
  const int64_t total = n_old + m;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < n_old * n_old) {
    const int64_t j = e / n_old, i = e % n_old;
    G[j * ldg + i] = (i == j) ? sigma[i] * sigma[i] : 0.0;
  }
  const int64_t e2 = e - n_old * n_old;
  if (e2 >= 0 && e2 < n_old * m) {
    const int64_t j = e2 / m, i = e2 % m;  // lower-left (n_old + i, j) <- upper-right (j, n_old + i)
    G[j * ldg + n_old + i] = G[(n_old + i) * ldg + j];
  }
  (void)total;
}

}  // namespace hp

using namespace hp;

extern "C" {

int hp_abi_version(void) { return HP_ABI_VERSION; }
long long hp_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }
int hp_set_debug(int flags) { return g_debug.exchange(flags); }
const char* hp_last_error(void) { return hp::last_error(); }

int hp_device_sm_count(int device) {
  int n = 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return -1;
  return n;
}

size_t hp_gemm_workspace_bytes(int64_t M, int64_t N, int64_t K, int sym, int b_upper) {
  return gemm_workspace_bytes(M, N, K, sym, b_upper);
}

int hp_gemm(int a_kmajor, int b_kmajor, int64_t M, int64_t N, int64_t K, hp_vecset A, hp_vecset B, double alpha,
            double beta, double* C, int64_t ldc, const double* row_scale, const double* col_scale,
            const double* col_div, int sym, int b_upper, void* ws, size_t ws_bytes, void* stream) {
  return gemm_run(a_kmajor != 0, b_kmajor != 0, M, N, K, vs(A), vs(B), A.aligned16 && B.aligned16, alpha, beta, C,
                  ldc, row_scale, col_scale, col_div, sym, b_upper, ws, ws_bytes, (cudaStream_t)stream);
}

size_t hp_gram_workspace_bytes(int64_t d, int64_t m) { return gemm_workspace_bytes(m, m, d, 1, 0); }

int hp_gram(hp_vecset S, int64_t d, int64_t m, const double* colscale, double* G, int64_t ldg, void* ws,
            size_t ws_bytes, void* stream) {
  HP_REQUIRE(d >= 0 && m >= 0 && ldg >= m, "hp_gram: bad dimensions");
  return gemm_run(true, true, m, m, d, vs(S), vs(S), S.aligned16 != 0, 1.0, 0.0, G, ldg, colscale, colscale, nullptr,
                  1, 0, ws, ws_bytes, (cudaStream_t)stream);
}

int hp_gram_single_split(int64_t m, int64_t d) { return gemm_plan_is_single_split(m, m, d, 1) ? 1 : 0; }

int hp_gram_pair(hp_vecset Ua, const double* sa, int64_t na, hp_vecset Ub, const double* sb, int64_t nb, int64_t d,
                 int same, double* G, int64_t ldg, void* stream) {
  HP_REQUIRE(na >= 0 && nb >= 0 && d >= 0 && ldg >= na && G, "hp_gram_pair: bad dimensions");
  HP_REQUIRE(!same || na == nb, "hp_gram_pair: a diagonal block is square");
  gemm_set_nosplit(true);
  const int rc = gemm_run(true, true, na, nb, d, vs(Ua), vs(Ub), Ua.aligned16 && Ub.aligned16, 1.0, 0.0, G, ldg, sa, sb,
                          nullptr, same ? 1 : 0, 0, nullptr, 0, (cudaStream_t)stream);
  gemm_set_nosplit(false);
  return rc;
}

__global__ void mirror_upper_kernel(double* G, int64_t ldg, int64_t n) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n * n) return;
  const int64_t i = e % n, j = e / n;
  if (i > j) G[i + j * ldg] = G[j + i * ldg];
}

int hp_mirror_upper(double* G, int64_t ldg, int64_t n, void* stream) {
  HP_REQUIRE(n >= 0 && ldg >= std::max<int64_t>(n, 1), "hp_mirror_upper: bad dimensions");
  if (n == 0) return HP_OK;
  mirror_upper_kernel<<<(unsigned)ceil_div(n * n, 256), 256, 0, (cudaStream_t)stream>>>(G, ldg, n);
  HP_CHECK_LAUNCH("mirror_upper_kernel");
  return HP_OK;
}

size_t hp_block_gram_workspace_bytes(int64_t d, int64_t n_old, int64_t m) {
  return std::max(gemm_workspace_bytes(n_old, m, d, 0, 0), gemm_workspace_bytes(m, m, d, 1, 0));
}

int hp_block_gram(hp_vecset Phi, const double* sigma, int64_t n_old, hp_vecset F, const double* fscale, int64_t m,
                  int64_t d, double* G, int64_t ldg, void* ws, size_t ws_bytes, void* stream) {
  HP_REQUIRE(n_old >= 0 && m >= 0 && d >= 0 && ldg >= n_old + m, "hp_block_gram: bad dimensions");
  cudaStream_t st = (cudaStream_t)stream;
  if (m > 0) {
    // mixed block sigma o (Phi^T F)  (pod.py:379-381)
    int rc = gemm_run(true, true, n_old, m, d, vs(Phi), vs(F), Phi.aligned16 && F.aligned16, 1.0, 0.0,
                      G + n_old * ldg, ldg, sigma, fscale, nullptr, 0, 0, ws, ws_bytes, st);
    if (rc) return rc;
    // fresh block gramian(F)  (pod.py:383)
    rc = gemm_run(true, true, m, m, d, vs(F), vs(F), F.aligned16 != 0, 1.0, 0.0, G + n_old * ldg + n_old, ldg,
                  fscale, fscale, nullptr, 1, 0, ws, ws_bytes, st);
    if (rc) return rc;
  }
  const int64_t work = n_old * n_old + n_old * m;
  if (work > 0) {
    block_gram_fill<<<(unsigned)ceil_div(work, 256), 256, 0, st>>>(G, ldg, n_old, m, sigma);
    HP_CHECK_LAUNCH("block_gram_fill");
  }
  return HP_OK;
}

size_t hp_syev_workspace_bytes(int64_t n) { return syev_workspace_bytes(n); }

int hp_syev(const double* G, int64_t ldg, int64_t n, double* lam_desc, double* V, int64_t ldv, int64_t nvec,
            double tol_rel, double tol_abs, double tol_angle, double keep_floor, int max_sweeps, int refine,
            int* sweeps, double* flops, void* ws, size_t ws_bytes, void* stream) {
  return syev_run(G, ldg, n, lam_desc, V, ldv, nvec, tol_rel, tol_abs, tol_angle, keep_floor, max_sweeps, refine,
                  sweeps, flops, ws, ws_bytes, (cudaStream_t)stream);
}

int64_t hp_syev_padded_order(int64_t n) { return syev_padded_order(n); }

int hp_syev_rows(const double* G, int64_t ldg, int64_t n, double* lam_desc, double* V, int64_t ldv, int64_t nvec,
                 double tol_rel, double tol_abs, double tol_angle, double keep_floor, int max_sweeps, int* sweeps,
                 double* flops, int64_t vrow0, int64_t vrow1, void* ws, size_t ws_bytes, void* stream) {
  return syev_run(G, ldg, n, lam_desc, V, ldv, nvec, tol_rel, tol_abs, tol_angle, keep_floor, max_sweeps, 0, sweeps,
                  flops, ws, ws_bytes, (cudaStream_t)stream, vrow0, vrow1);
}

int64_t hp_syev_tri_max_order(void) { return syev_tri_max_order(); }

size_t hp_syev_tri_workspace_bytes(int64_t n) { return syev_tri_workspace_bytes(n); }

int hp_syev_tri(const double* H, int64_t ldh, int64_t n, double floor_rel, double relgap_min, double* lam_desc,
                double* W, int64_t ldw, int64_t* k_out, int* status, double* diag8, void* ws, size_t ws_bytes,
                void* stream) {
  HP_REQUIRE(H && lam_desc && W && k_out && status && ws, "hp_syev_tri: null argument");
  HP_REQUIRE(floor_rel >= 0.0 && relgap_min >= 0.0, "hp_syev_tri: negative threshold");
  return syev_tri_run(H, ldh, n, floor_rel, relgap_min, lam_desc, W, ldw, k_out, status, diag8, ws, ws_bytes,
                      (cudaStream_t)stream);
}

int hp_truncate(const double* lam_desc, int64_t n, double eps, double cutoff, int64_t m, double* sigma, double* info4,
                void* stream) {
  HP_REQUIRE(n >= 0 && eps >= 0.0, "hp_truncate: bad arguments");
  return truncate_run(lam_desc, n, eps, cutoff, m, sigma, info4, (cudaStream_t)stream);
}

size_t hp_assemble_workspace_bytes(int64_t d, int64_t m, int64_t N) { return gemm_workspace_bytes(d, N, m, 0, 0); }

int hp_assemble(hp_vecset S, int64_t d, int64_t m, const double* V, int64_t ldv, const double* sigma, int64_t N,
                double* U, int64_t ldu, void* ws, size_t ws_bytes, void* stream) {
  HP_REQUIRE(N >= 0 && N <= m && ldu >= d && ldv >= m, "hp_assemble: bad dimensions");
  VecSet b{V, ldv, nullptr};
  return gemm_run(false, true, d, N, m, vs(S), b, S.aligned16 && (ldv % 2 == 0), 1.0, 0.0, U, ldu, nullptr, nullptr,
                  sigma, 0, 0, ws, ws_bytes, (cudaStream_t)stream);
}

size_t hp_drift_workspace_bytes(int64_t d, int64_t N) { return gemm_workspace_bytes(N, N, d, 1, 0); }

int hp_drift(const double* U, int64_t ldu, int64_t d, int64_t N, double* C, int64_t ldc, double* drift_out, void* ws,
             size_t ws_bytes, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  int rc = gram_sym(U, ldu, d, N, C, ldc, ws, ws_bytes, st);
  if (rc) return rc;
  return drift_run(C, ldc, N, drift_out, st);
}

size_t hp_reortho_workspace_bytes(int64_t d, int64_t N) {
  const int64_t ldx = (d + 1) & ~int64_t(1);
  return reortho_layout(d, N, ldx).total;
}

// U <- Q of the QR factorisation of U: CholQR (one pass when the drift is
// small enough that kappa(U)^2 ~ 1 + 2 drift makes a single pass accurate to
// the rounding level, else CholQR2; shifted CholQR3 when the first Cholesky
// breaks down).  C holds U^T U on entry (from hp_drift) and is destroyed.
// Same span and column order as the MGS sweep of pod.py:227-237.
int hp_reorthonormalize(double* U, int64_t ldu, int64_t d, int64_t N, double* C, int64_t ldc, double drift,
                        int* passes_out, void* ws, size_t ws_bytes, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (passes_out) *passes_out = 0;
  if (N == 0) return HP_OK;
  const int64_t ldx = (d + 1) & ~int64_t(1);
  const ReorthoLayout L = reortho_layout(d, N, ldx);
  HP_REQUIRE(ws_bytes >= L.total, "hp_reorthonormalize: workspace too small");
  char* base = static_cast<char*>(ws);
  double* X = reinterpret_cast<double*>(base + L.off_X);
  double* A = reinterpret_cast<double*>(base + L.off_A);
  const int64_t ldn = (N + 1) & ~int64_t(1);
  void* gws = base + L.off_gemm;
  const size_t gwsb = ws_bytes - L.off_gemm;
  char* pin = pinned_scratch();
  HP_REQUIRE(pin != nullptr, "hp_reorthonormalize: pinned host scratch unavailable");
  int* hinfo = reinterpret_cast<int*>(pin + 64);
  double* htrace = reinterpret_cast<double*>(pin + 80);
  int rc = HP_OK;
  int passes = 0;
  // stream sync + the Cholesky breakdown flag of the pass just queued (flag may be null)
  auto sync_checked = [&](const int* flag, const char* what) -> int {
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
      set_error(std::string("reortho: ") + cudaGetErrorString(e));
      return HP_ECUDA;
    }
    if (flag && *flag != 0) {
      set_error(std::string("reortho: ") + what);
      return HP_ELINALG;
    }
    return HP_OK;
  };
  // keep a copy of C in case the first factorisation fails
  rc = scale_run(C, ldc, N, N, nullptr, nullptr, nullptr, A, ldn, st);
  if (!rc) rc = cholqr_pass(U, ldu, d, N, C, ldc, X, ldx, L, base, ws_bytes, st, &hinfo[0]);
  if (!rc) rc = sync_checked(nullptr, "");
  if (!rc && hinfo[0] != 0) {
    // shifted CholQR (Fukaya et al.): s = 11 (d N + N (N+1)) u ||U||_2^2, ||U||_2^2 <= trace(U^T U)
    trace_kernel<<<1, 256, 0, st>>>(A, ldn, N, C);
    HP_CHECK_LAUNCH("trace_kernel");
    HP_CHECK_CUDA(d2h_small(htrace, C, sizeof(double), st));
    rc = sync_checked(nullptr, "");
    if (rc) return rc;
    const double shift = 11.0 * ((double)d * N + (double)N * (N + 1)) * 1.1102230246251565e-16 * htrace[0];
    add_diag<<<(unsigned)ceil_div(N, 256), 256, 0, st>>>(A, ldn, N, shift);
    HP_CHECK_LAUNCH("add_diag");
    rc = cholqr_pass(U, ldu, d, N, A, ldn, X, ldx, L, base, ws_bytes, st, &hinfo[1]);
    if (!rc) rc = sync_checked(&hinfo[1], "shifted Cholesky broke down (modes numerically rank deficient)");
    // bring the shifted result back into U, then a plain pass (checked here) and the second pass
    if (!rc) rc = scale_run(X, ldx, d, N, nullptr, nullptr, nullptr, U, ldu, st);
    if (!rc) rc = gram_sym(U, ldu, d, N, A, ldn, gws, gwsb, st);
    if (!rc) rc = cholqr_pass(U, ldu, d, N, A, ldn, X, ldx, L, base, ws_bytes, st, &hinfo[0]);
    if (!rc) rc = sync_checked(&hinfo[0], "Cholesky after the shifted pass broke down");
    passes += 1;
    if (rc) {
      if (passes_out) *passes_out = passes;
      return rc;
    }
  }
  passes += 1;
  const bool single = (passes == 1) && (drift >= 0.0) && (drift <= kSinglePassDrift);
  if (single) {
    if (!rc) rc = scale_run(X, ldx, d, N, nullptr, nullptr, nullptr, U, ldu, st);
    if (passes_out) *passes_out = passes;
    if (!rc) {
      cudaError_t e = cudaStreamSynchronize(st);
      if (e != cudaSuccess) {
        set_error(std::string("reortho: ") + cudaGetErrorString(e));
        rc = HP_ECUDA;
      }
    }
    return rc;
  }
  // second pass: X -> U
  if (!rc) rc = gram_sym(X, ldx, d, N, A, ldn, gws, gwsb, st);
  if (!rc) rc = cholqr_pass(X, ldx, d, N, A, ldn, U, ldu, L, base, ws_bytes, st, &hinfo[0]);
  passes += 1;
  if (!rc) {
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
      set_error(std::string("reortho: ") + cudaGetErrorString(e));
      rc = HP_ECUDA;
    } else if (hinfo[0] != 0) {
      set_error("reortho: Cholesky of the re-orthonormalised modes broke down");
      rc = HP_ELINALG;
    }
  }
  if (passes_out) *passes_out = passes;
  return rc;
}

int hp_signs(double* U, int64_t ldu, int64_t d, int64_t N, double* R, int64_t ldr, int64_t mr, double* sign_out,
             void* stream) {
  return signs_run(U, ldu, d, N, R, ldr, mr, sign_out, (cudaStream_t)stream);
}

int hp_transpose_rm_to_cm(const double* src, int64_t rows, int64_t cols, double* dst, int64_t ldd, void* stream) {
  return transpose_run(src, rows, cols, dst, ldd, (cudaStream_t)stream);
}

int hp_scale(const double* src, int64_t lds, int64_t rows, int64_t cols, const double* row_mul, const double* row_div,
             const double* col_mul, double* dst, int64_t ldd, void* stream) {
  return scale_run(src, lds, rows, cols, row_mul, row_div, col_mul, dst, ldd, (cudaStream_t)stream);
}

int hp_finite_check(const double* src, int64_t lds, int64_t rows, int64_t cols, int* bad, void* stream) {
  return finite_check_run(src, lds, rows, cols, bad, (cudaStream_t)stream);
}

int hp_read_small(const void* src, void* pinned_dst, int64_t bytes, void* stream) {
  HP_REQUIRE(bytes >= 0 && bytes % 4 == 0, "hp_read_small: size must be a multiple of 4 bytes");
  HP_CHECK_CUDA(d2h_small(pinned_dst, src, (size_t)bytes, (cudaStream_t)stream));
  count_launches(1);
  return HP_OK;
}

size_t hp_pstrf_workspace_bytes(int64_t m) { return pstrf_workspace_bytes(m); }

int hp_pstrf(const double* G, int64_t ldg, int64_t m, double* L, int64_t ldl, int* piv, double tol_rel,
             double tol_lam, int64_t* rank, void* ws, size_t ws_bytes, void* stream) {
  HP_REQUIRE(m >= 0 && ldg >= m && ldl >= m, "hp_pstrf: bad dimensions");
  return pstrf_run(G, ldg, m, L, ldl, piv, tol_rel, tol_lam, rank, ws, ws_bytes, (cudaStream_t)stream);
}

int hp_add_diag(double* C, int64_t ldc, int64_t n, double s, void* stream) {
  if (n <= 0) return HP_OK;
  add_diag<<<(unsigned)ceil_div(n, 256), 256, 0, (cudaStream_t)stream>>>(C, ldc, n, s);
  HP_CHECK_LAUNCH("add_diag");
  return HP_OK;
}

int hp_gram_drift(const double* C, int64_t ldc, int64_t N, double* drift_out, void* stream) {
  HP_REQUIRE(N >= 0 && ldc >= std::max<int64_t>(N, 1), "hp_gram_drift: bad dimensions");
  return drift_run(C, ldc, N, drift_out, (cudaStream_t)stream);
}

int hp_col_absmax(const double* U, int64_t ldu, int64_t rows, int64_t N, int64_t row_offset, double* vals,
                  int64_t* idx, void* stream) {
  HP_REQUIRE(rows >= 0 && N >= 0 && ldu >= std::max<int64_t>(rows, 1), "hp_col_absmax: bad dimensions");
  return col_absmax_run(U, ldu, rows, N, row_offset, vals, idx, (cudaStream_t)stream);
}

int hp_add(double* dst, const double* src, int64_t n, void* stream) {
  HP_REQUIRE(n >= 0, "hp_add: negative length");
  return add_run(dst, src, n, (cudaStream_t)stream);
}

int hp_col_norms_sq(const double* A, int64_t lda, int64_t rows, int64_t cols, const double* weights, double* out,
                    void* stream) {
  HP_REQUIRE(rows >= 0 && cols >= 0 && lda >= std::max<int64_t>(rows, 1), "hp_col_norms_sq: bad dimensions");
  return col_norms_sq_run(A, lda, rows, cols, weights, out, (cudaStream_t)stream);
}

static size_t tbytes(int64_t N) {
  return (size_t)((std::max<int64_t>(N, 1) + 1) & ~int64_t(1)) * chol_t_cols(N) * 8;
}

size_t hp_chol_inverse_workspace_bytes(int64_t N) {
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  return al(tbytes(N)) + al(16) + al(kSplitKMax) + 256;
}

int hp_chol_inverse(double* C, int64_t ldc, int64_t N, double* Linv, int64_t ldl, int* info_out, void* ws,
                    size_t ws_bytes, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  HP_REQUIRE(N >= 0 && ldc >= N && ldl >= N, "hp_chol_inverse: bad dimensions");
  HP_REQUIRE(ws_bytes >= hp_chol_inverse_workspace_bytes(N), "hp_chol_inverse: workspace too small");
  if (info_out) *info_out = 0;
  if (N == 0) return HP_OK;
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  char* base = static_cast<char*>(ws);
  double* T = reinterpret_cast<double*>(base);
  int* info = reinterpret_cast<int*>(base + al(tbytes(N)));
  char* gws = base + al(tbytes(N)) + al(16);
  const size_t gwsb = ws_bytes - (size_t)(gws - base);
  const bool trace = (debug_flags() & DBG_CHOL_TRACE) != 0;
  cudaEvent_t ev[3];
  if (trace)
    for (auto& e : ev) cudaEventCreate(&e);
  if (trace) cudaEventRecord(ev[0], st);
  int rc = chol_inv_run(C, ldc, N, Linv, ldl, T, info, gws, gwsb, st);
  if (trace) cudaEventRecord(ev[1], st);
  if (trace) {
    cudaEventRecord(ev[2], st);
    cudaEventSynchronize(ev[2]);
    float a = 0.f, b = 0.f;
    cudaEventElapsedTime(&a, ev[0], ev[1]);
    cudaEventElapsedTime(&b, ev[1], ev[2]);
    fprintf(stderr, "[hp_chol_inverse n=%lld] chol_inv %.2f ms (+%.2f)\n", (long long)N, a, b);
    for (auto& e : ev) cudaEventDestroy(e);
  }
  if (rc) return rc;
  int* h = reinterpret_cast<int*>(pinned_scratch() + 160);  // pinned: see pstrf_run
  HP_CHECK_CUDA(d2h_small(h, info, sizeof(int), st));
  HP_CHECK_CUDA(cudaStreamSynchronize(st));
  if (info_out) *info_out = *h;
  return HP_OK;
}

size_t hp_sumsq_workspace_bytes(void) { return 1024 * sizeof(double); }

int hp_sumsq(const double* A, int64_t lda, int64_t rows, int64_t cols, double* out, void* ws, size_t ws_bytes,
             void* stream) {
  HP_REQUIRE(ws_bytes >= 1024 * sizeof(double), "hp_sumsq: workspace too small");
  return sumsq_run(A, lda, rows, cols, out, static_cast<double*>(ws), (cudaStream_t)stream);
}

}  // extern "C"
