/*
 * hapod_b200.h -- C-ABI of libhapod_b200.so, the sm_100a kernels behind the
 * HAPOD hot path (arXiv:1607.05210).
 *
 * The reference package (hapod v0.1.0, pure Python + NumPy/SciPy) has no FFI:
 * its per-node arithmetic is NumPy `@` (BLAS dgemm) and scipy.linalg.eigh
 * (LAPACK dsyevr).  Each entry point below replaces one of those call sites;
 * the Python host package `paper_1607_05210_b200` binds them with ctypes and
 * keeps the reference's Python entry points (pod, block_gramian_pod,
 * run_hapod, run_parallel, IncrementalSession ...).
 *
 * Conventions
 *   - all matrices float64, column-major, leading dimension >= rows;
 *   - all data pointers are DEVICE pointers; `stream` is a cudaStream_t;
 *   - calls are stream-ordered and asynchronous unless stated otherwise;
 *   - every call returns an hp_status; hp_last_error() gives the message
 *     (thread-local).  HP_EINVAL maps to ValueError, HP_ELINALG to
 *     numpy.linalg.LinAlgError (CLI exit 3, cli.py:572-574), HP_ECUDA to
 *     RuntimeError;
 *   - workspaces are caller-allocated; query their size with the matching
 *     *_workspace_bytes function.
 */
#ifndef HAPOD_B200_H
#define HAPOD_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HP_ABI_VERSION 1

enum hp_status { HP_OK = 0, HP_EINVAL = 1, HP_ECUDA = 2, HP_ELINALG = 3, HP_ENOMEM = 4 };

/* A set of contiguous float64 vectors: vector i starts at table[i] when
 * table != NULL (a device array of pointers), else at base + i*ld.  Used to
 * read a node's input as the concatenation of its children's mode blocks
 * without the hstack copy of hierarchy.py:286-290.  aligned16 != 0 promises
 * every vector start is 16-byte aligned (enables 16-byte async copies). */
typedef struct hp_vecset {
  const double* base;
  int64_t ld;
  const double* const* table;
  int aligned16;
} hp_vecset;

int hp_abi_version(void);
/* Number of kernels this library has launched in the process (monotonic). */
long long hp_launch_count(void);
/* Diagnostics (no reference counterpart; never changes a result): bit 0 prints one line per
 * Jacobi sweep, bit 1 adds CUDA-event timing of one mid-sweep round, bit 2 times the CholQR
 * factorisation, bit 3 times the stages of hp_syev_tri, bit 4
 * launches the Jacobi sweeps directly instead of replaying CUDA graphs (for per-kernel profilers).  Returns the previous flags.  The library reads no environment variables. */
int hp_set_debug(int flags);
const char* hp_last_error(void);
int hp_device_sm_count(int device);

/* Generic FP64 DMMA GEMM  C = alpha * op(A) op(B) + beta * C, then
 * C(m,n) *= row_scale[m] * col_scale[n], C(m,n) /= col_div[n] (each nullable).
 *   a_kmajor: A(m,k) = A.vec(m)[k]  else A(m,k) = A.vec(k)[m]
 *   b_kmajor: B(k,n) = B.vec(n)[k]  else B(k,n) = B.vec(k)[n]
 *   sym:      1: M == N, only the upper triangle is computed and mirrored;
 *             2: the same without the mirror (the lower triangle of C is left untouched)
 *   b_upper:  B is upper triangular (B(k,n) = 0 for k > n)
 * Long contractions are split over K with a fixed-order reduction
 * (deterministic; the plan depends only on M, N, K). */
size_t hp_gemm_workspace_bytes(int64_t M, int64_t N, int64_t K, int sym, int b_upper);
int hp_gemm(int a_kmajor, int b_kmajor, int64_t M, int64_t N, int64_t K, hp_vecset A, hp_vecset B, double alpha,
            double beta, double* C, int64_t ldc, const double* row_scale, const double* col_scale,
            const double* col_div, int sym, int b_upper, void* ws, size_t ws_bytes, void* stream);

/* K1 -- Gramian G = D S^T S D, D = diag(colscale) (nullable), exactly
 * symmetric.  Replaces gramian() / InnerProductSpace.gram
 * (pod.py:208-211, 87-91); with colscale = sigma it is the Gramian of
 * ModeSet.scaled() (pod.py:160-162) without the copy. */
size_t hp_gram_workspace_bytes(int64_t d, int64_t m);
int hp_gram(hp_vecset S, int64_t d, int64_t m, const double* colscale, double* G, int64_t ldg, void* ws,
            size_t ws_bytes, void* stream);

/* K1, one child pair at a time (a star's root under run_parallel, parallel.py:77-142 evaluates the
 * parent only after the whole wave; the Gramian of hstack(children) at hierarchy.py:284-291 +
 * pod.py:208-211 can start as soon as two children exist): G (na x nb) = diag(sa) Ua^T Ub diag(sb)
 * with the tile arithmetic of an UNSPLIT hp_gram -- every output entry summed over all d rows by one
 * CTA -- so that the block equals the corresponding block of hp_gram on the concatenation bit for bit
 * whenever hp_gram_single_split(m, d) != 0 for the concatenation's order m.  same != 0: Ua == Ub
 * (diagonal block, exactly symmetric).  hp_gram forms the entries with row <= column and mirrors them
 * (row scale applied before the column scale), so an off-diagonal pair is computed as the UPPER
 * block -- rows = the child that comes first -- and hp_mirror_upper copies the strictly upper
 * triangle of the assembled n x n matrix onto the lower one. */
int hp_gram_single_split(int64_t m, int64_t d);
int hp_gram_pair(hp_vecset Ua, const double* sa, int64_t na, hp_vecset Ub, const double* sb, int64_t nb, int64_t d,
                 int same, double* G, int64_t ldg, void* stream);
int hp_mirror_upper(double* G, int64_t ldg, int64_t n, void* stream);

/* K1b -- block Gramian of [Phi*diag(sigma) | F*diag(fscale)] for the
 * incremental merge (pod.py:376-384): top-left diag(sigma^2) written down,
 * mixed block sigma o (Phi^T F), fresh block F^T F, exactly symmetric.
 * fscale nullable. */
size_t hp_block_gram_workspace_bytes(int64_t d, int64_t n_old, int64_t m);
int hp_block_gram(hp_vecset Phi, const double* sigma, int64_t n_old, hp_vecset F, const double* fscale, int64_t m,
                  int64_t d, double* G, int64_t ldg, void* ws, size_t ws_bytes, void* stream);

/* K2a -- eigensolver preconditioner: pivoted Cholesky G = L L^T + E with
 * complete diagonal pivoting, L (m x r) with rows in the ORIGINAL order, until
 * the largest remaining pivot <= max(tol_rel * max|G_ii|, tol_lam * lam_est), lam_est a
 * power-iteration lower bound of lambda_max (8 GEMVs; skipped when tol_lam = 0).
 * The eigenvalues of G are those of H = L^T L; its eigenvectors
 * V = L W Lambda^{-1/2} (W = eigenvectors of H).  piv (device, m ints)
 * receives the pivot order; rank (host) receives r.  Synchronises once per
 * 128-column panel. */
size_t hp_pstrf_workspace_bytes(int64_t m);
int hp_pstrf(const double* G, int64_t ldg, int64_t m, double* L, int64_t ldl, int* piv, double tol_rel,
             double tol_lam, int64_t* rank, void* ws, size_t ws_bytes, void* stream);

/* K2 -- all eigenpairs of the symmetric n x n G, eigenvalues descending,
 * first nvec eigenvectors in V.  Replaces scipy.linalg.eigh + reversal
 * (pod.py:329-331, 386-388).  Parallel two-sided block Jacobi; synchronises
 * the stream once per sweep.  Returns HP_ELINALG if max_sweeps is reached.
 * A pair (i,j) is rotated iff |g_ij| > tol_abs*max|g_ii|, |g_ij| > tol_rel*sqrt|g_ii g_jj|,
 * |g_ij| > tol_angle*|g_jj - g_ii| (the rotation angle is not negligible) and
 * max(g_ii, g_jj) >= keep_floor (mixing among eigenvalues that are all below the
 * floor never reaches the output).  refine != 0: eigenvalues are Rayleigh quotients
 * v^T G v / v^T v against the input (one extra n^3 GEMM), else the converged diagonal.
 * sweeps / flops (nullable, host) receive the sweep count and the algorithmic flops of
 * its DMMA products. */
size_t hp_syev_workspace_bytes(int64_t n);
int hp_syev(const double* G, int64_t ldg, int64_t n, double* lam_desc, double* V, int64_t ldv, int64_t nvec,
            double tol_rel, double tol_abs, double tol_angle, double keep_floor, int max_sweeps, int refine,
            int* sweeps, double* flops, void* ws, size_t ws_bytes, void* stream);

/* K2, one rank's share of a replicated eigensolve (multi-GPU root): the same
 * iteration as hp_syev without Rayleigh refinement -- identical eigenvalues, sweeps and rotations on
 * every rank -- but the eigenvector accumulation V <- V J (half of a round's DMMA products) is
 * restricted to the rows [vrow0, vrow1) of the padded matrix (whole 64-row slabs of
 * hp_syev_padded_order(n) rows; vrow1 < 0: all rows).  Rows of V outside the range are not
 * meaningful; the ranks all-gather their row ranges.  The reference computes the whole
 * decomposition in one LAPACK call (pod.py:329-331); its wave executor (parallel.py:77-142) has no
 * counterpart for a single node's eigensolve. */
int64_t hp_syev_padded_order(int64_t n);
int hp_syev_rows(const double* G, int64_t ldg, int64_t n, double* lam_desc, double* V, int64_t ldv, int64_t nvec,
                 double tol_rel, double tol_abs, double tol_angle, double keep_floor, int max_sweeps, int* sweeps,
                 double* flops, int64_t vrow0, int64_t vrow1, void* ws, size_t ws_bytes, void* stream);

/* K2t -- the eigenpairs with lambda >= floor_rel * lambda_max of a symmetric positive
 * semidefinite n x n H by Householder tridiagonalisation (one cooperative launch + one DMMA GEMM
 * per 64-column panel), relative-accuracy Sturm multisection and one twisted factorisation per
 * eigenvalue on a single definite representation T - sigma I = L D L^T (no re-orthogonalisation),
 * and a compact-WY back-transformation.  Replaces scipy.linalg.eigh (pod.py:329-331) for the
 * large preconditioned eigenproblems H = L^T L of a node POD: ~4/3 n^3 flops + 8 n^3 / 3 bytes of
 * matrix reads instead of the block Jacobi's ~90 n^3 flops.  lam_desc (n, device): the K
 * eigenvalues descending, the rest zero; W (n x n, ldw even): eigenvectors in the first K columns.
 * status (host): 0 = done; 1 = declined -- the spectrum has a relative gap below relgap_min (the
 * eigenvectors of a cluster would not be orthogonal) or no definite representation exists -- and
 * the caller uses hp_syev instead; outputs are then not meaningful.  diag8 (nullable, host):
 * {smallest relative gap, largest relative residual, sigma, K, tridiagonalisation ms, tridiagonal
 * eigensolve ms (CUDA events on the stream), max Rayleigh-quotient iterations, 0}.
 * 2 <= n <= hp_syev_tri_max_order(). */
int64_t hp_syev_tri_max_order(void);
size_t hp_syev_tri_workspace_bytes(int64_t n);
int hp_syev_tri(const double* H, int64_t ldh, int64_t n, double floor_rel, double relgap_min, double* lam_desc,
                double* W, int64_t ldw, int64_t* k_out, int* status, double* diag8, void* ws, size_t ws_bytes,
                void* stream);

/* K3 -- truncation (pod.py:278-289 with truncation_rank pod.py:190-205):
 * keep = lam >= cutoff*lam_max*m, sigma = sqrt(lam_keep), N = smallest rank
 * whose tail sum_{n>=N} sigma_n^2 <= eps^2, tail = sum lam_keep[N:].
 * info4 (device) = {lam_max, nkeep, N, tail}. */
int hp_truncate(const double* lam_desc, int64_t n, double eps, double cutoff, int64_t m, double* sigma, double* info4,
                void* stream);

/* K4 -- mode reconstruction U = (S V[:, :N]) / sigma[:N]  (pod.py:333-334).
 * For column-scaled inputs pre-scale the rows of V. */
size_t hp_assemble_workspace_bytes(int64_t d, int64_t m, int64_t N);
int hp_assemble(hp_vecset S, int64_t d, int64_t m, const double* V, int64_t ldv, const double* sigma, int64_t N,
                double* U, int64_t ldu, void* ws, size_t ws_bytes, void* stream);

/* K5a -- C = U^T U and drift = max |C - I| (pod.py:245-247), drift_out device scalar. */
size_t hp_drift_workspace_bytes(int64_t d, int64_t N);
int hp_drift(const double* U, int64_t ldu, int64_t d, int64_t N, double* C, int64_t ldc, double* drift_out, void* ws,
             size_t ws_bytes, void* stream);

/* K5b -- U <- Q factor of U (CholQR: one pass when drift <= 1e-1, else
 * CholQR2; shifted CholQR3 on breakdown; pass drift < 0 to force two passes):
 * the same span and Gram-Schmidt column order as the MGS sweep of
 * pod.py:227-237.  C = U^T U on entry (destroyed).  Synchronises the stream. */
size_t hp_reortho_workspace_bytes(int64_t d, int64_t N);
int hp_reorthonormalize(double* U, int64_t ldu, int64_t d, int64_t N, double* C, int64_t ldc, double drift,
                        int* passes_out, void* ws, size_t ws_bytes, void* stream);

/* K6 -- sign convention (pod.py:214-224): per column, the largest-|.| entry
 * (first index on ties) made positive; R (m_r x N, nullable) flipped alike;
 * sign_out (nullable) receives the +-1 applied. */
int hp_signs(double* U, int64_t ldu, int64_t d, int64_t N, double* R, int64_t ldr, int64_t mr, double* sign_out,
             void* stream);

/* Row-sharded root (multi-GPU, one row block of the modes per rank):
 * hp_col_absmax -- per column of the local row block, the largest |u| and the GLOBAL row index
 *   (row_offset + local row, first index on ties) of that entry: the local half of _fix_signs's
 *   argmax (pod.py:214-224); the ranks' candidates are combined by the caller.  vals: N doubles,
 *   idx: N int64 (device).
 * hp_chol_inverse -- Linv = L^{-1} for C = L L^T (N x N, lower part of C used, C destroyed):
 *   the factor of one CholQR pass when C = sum over ranks of U_q^T U_q (replaces MGS,
 *   pod.py:227-237); U_q <- U_q Linv^T is then an hp_gemm with b_upper.  *info_out (host) is
 *   non-zero when the factorisation broke down.  Synchronises the stream. */
/* drift = max |C - I| of a given N x N Gram (the sum over ranks of U_q^T U_q); device scalar. */
int hp_gram_drift(const double* C, int64_t ldc, int64_t N, double* drift_out, void* stream);
int hp_col_absmax(const double* U, int64_t ldu, int64_t rows, int64_t N, int64_t row_offset, double* vals,
                  int64_t* idx, void* stream);
/* hp_add -- dst[i] += src[i], i < n (contiguous, device): the fixed-order binary-tree sum of the
 *   row-distributed root's per-shard Gram partials (replaces the BLAS sum inside the reference's
 *   one-GPU Gram, pod.py:208-211, when the root is split by rows). */
int hp_add(double* dst, const double* src, int64_t n, void* stream);
/* hp_col_norms_sq -- out[j] = sum_i w_i A(i,j)^2 (weights nullable = Euclidean): the reference's
 *   InnerProductSpace.norms_sq (pod.py:93-97).  out: cols doubles (device). */
int hp_col_norms_sq(const double* A, int64_t lda, int64_t rows, int64_t cols, const double* weights, double* out,
                    void* stream);
size_t hp_chol_inverse_workspace_bytes(int64_t N);
int hp_chol_inverse(double* C, int64_t ldc, int64_t N, double* Linv, int64_t ldl, int* info_out, void* ws,
                    size_t ws_bytes, void* stream);

/* Layout helpers: row-major (NumPy C-order) upload -> column-major, row/column
 * scaling (weighted spaces: InnerProductSpace.weigh/unweigh pod.py:76-84),
 * finiteness check (SnapshotBlock, pod.py:115-116; bad = device int). */
int hp_transpose_rm_to_cm(const double* src, int64_t rows, int64_t cols, double* dst, int64_t ldd, void* stream);
int hp_scale(const double* src, int64_t lds, int64_t rows, int64_t cols, const double* row_mul, const double* row_div,
             const double* col_mul, double* dst, int64_t ldd, void* stream);
int hp_finite_check(const double* src, int64_t lds, int64_t rows, int64_t cols, int* bad, void* stream);
/* Stream-ordered read of `bytes` (multiple of 4) device bytes into PINNED host memory by a kernel
   (no copy engine: a D2H memcpy queues behind pending host-to-device uploads).  The host side of
   every small read-back on the node path -- the finiteness flag of SnapshotBlock (pod.py:115-116),
   the truncation counts of _from_spectrum (pod.py:284-289), the drift of _finish_modes
   (pod.py:245-247) and the singular values of the ModeSet (pod.py:142-154). */
int hp_read_small(const void* src, void* pinned_dst, int64_t bytes, void* stream);
/* C(i,i) += s for i < n (Bjorck / Newton-Schulz orthonormalisation of the Ritz basis). */
int hp_add_diag(double* C, int64_t ldc, int64_t n, double s, void* stream);

/* Deterministic sum of squares of a column-major block (residual energy of
 * actual_mean_error, hierarchy.py:237-253); out = device scalar. */
size_t hp_sumsq_workspace_bytes(void);
int hp_sumsq(const double* A, int64_t lda, int64_t rows, int64_t cols, double* out, void* ws, size_t ws_bytes,
             void* stream);

#ifdef __cplusplus
}
#endif

#endif /* HAPOD_B200_H */
