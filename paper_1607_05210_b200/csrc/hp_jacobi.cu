// K2: symmetric eigensolve of the node Gramian by two-sided parallel block
// Jacobi (replaces scipy.linalg.eigh / LAPACK dsyevr, pod.py:329-331,386-388).
//
// The padded n_p x n_p matrix (n_p = nb*32, nb even) is split into nb block
// columns of width 32.  A sweep is nb-1 rounds of a round-robin tournament;
// in each round the nb/2 disjoint block pairs (p,q) are processed at once:
//
//   local solve (first CTAs of jac_round): one CTA per pair loads the 64x64 sub-problem G[I,I],
//               I = block p U block q, into shared memory.  If any off-diagonal
//               entry exceeds tol_abs * max|g_ii| it diagonalises the copy with
//               cyclic parallel-order Jacobi (32 disjoint rotations per step,
//               63 steps per local sweep, relative threshold
//               |a_ij| > tol_rel sqrt|a_ii a_jj|) while accumulating the 64x64
//               rotation W, then re-orthonormalises W with one Bjorck step
//               (W += W (I - W^T W) / 2).  Only W is written.
//   jac_apply : G <- J^T G J and V <- V J for the block-diagonal J built from
//               the W's, as 64x64x64 DMMA products in shared memory: one CTA
//               per upper 64x64 tile pair of G (the pair's own diagonal tile
//               included) and per 64-row slab of V.  Every tile sees the same
//               orthonormal W, so each round is a similarity transform up to
//               GEMM rounding -- the backward error stays at the u*||G|| level
//               instead of growing with the number of rotations.
//
// A sweep in which no pair needed work ends the iteration; a sweep whose
// largest off-diagonal ratio no longer halves while sitting at the rounding
// floor (< 512 u) is accepted as converged as well.  Eigenvalues are then the
// Rayleigh quotients v^T G0 v / v^T v against the ORIGINAL Gramian, sorted
// descending (ties by index), with V's columns permuted to match -- the
// "eigh then reverse" order of pod.py:329-331.
// Padding rows/columns are exactly zero and are never rotated against real
// indices (their off-diagonal entries stay exactly 0), so they are dropped
// by index at the end.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "hp_common.cuh"

namespace hp {
int gemm_run(bool a_kmajor, bool b_kmajor, int64_t M, int64_t N, int64_t K, VecSet A, VecSet B, bool aligned16,
             double alpha, double beta, double* C, int64_t ldc, const double* row_scale, const double* col_scale,
             const double* col_div, int sym, int b_upper, void* ws, size_t ws_bytes, cudaStream_t st);
size_t gemm_workspace_bytes(int64_t M, int64_t N, int64_t K, int sym, int b_upper);
namespace jac {

constexpr int BW = 32;        // block width
constexpr int PS = 2 * BW;    // local problem size
constexpr int LS = PS + 1;    // local smem stride
constexpr int TS = PS + 4;    // apply-kernel smem stride (= 4 mod 16: conflict-free DMMA fragments)
constexpr int AT = 256;       // apply threads
constexpr int64_t GRAPH_MAX_ORDER = 2048;  // padded orders up to this replay their sweeps as CUDA graphs
constexpr int GRAPH_MIN_CONCURRENCY = 3;   // ... when at least this many solves are in flight on host threads

struct Params {
  double* G;          // n_p x n_p, ld = n_p
  double* V;          // n_p x n_p, ld = n_p
  int64_t np;
  int nb;             // number of 32-wide blocks (even)
  int round;
  double* W;          // (nb/2) x 64 x 64, col-major per pair
  int* flags;         // nb/2
  int* counter;       // pairs that needed work in this sweep
  double* maxoff;     // max |g_ij| / max|g_ii| seen in this sweep (atomic max on the bit pattern)
  unsigned long long* mm_count;  // 64x64x64 DMMA products performed by jac_apply (flop accounting)
  unsigned long long* task_counter;  // dynamic task scheduler of the "rest" apply pass
  const double* scal; // scal[0] = max |g_ii| of the input
  double tol_rel, tol_abs;
  double keep_floor;  // pairs whose diagonal entries are both below this never rotate
  double tol_angle;   // pairs whose rotation angle |g_ij| / |g_jj - g_ii| is below this never rotate
  int max_local_sweeps;
  int* tile_mark;     // per G tile: stamp of the round whose "needed" pass already applied it
  int stamp;
  int phase;          // apply: 1 = tiles needed by the next round's local solves, 2 = the rest
  int slab_extra;     // one more slab accumulated besides the range (-1: none): the slab holding the padding rows
  int slab0, nslab;   // V accumulation restricted to the 64-row slabs [slab0, slab0 + nslab) (all of them by default):
                      // a rank of the row-distributed root accumulates only its own rows of V
};

__device__ __forceinline__ void circle_pair(int nplayers, int r, int k, int& a, int& b) {
  // round-robin "circle method": player nplayers-1 fixed, others rotate (0 <= r, k < m)
  const int m = nplayers - 1;
  if (k == 0) {
    a = m;
    b = r;
  } else {
    a = r + k;
    if (a >= m) a -= m;
    b = r - k + m;
    if (b >= m) b -= m;
  }
}

__device__ __forceinline__ void block_pair(const Params& p, int k, int& bp, int& bq) {
  int a, b;
  circle_pair(p.nb, p.round, k, a, b);
  bp = min(a, b);
  bq = max(a, b);
}

// index k of the pair that contains block x in round r (inverse of circle_pair)
__device__ __forceinline__ int pair_of(int nb, int r, int x) {
  const int m = nb - 1;
  if (x == m || x == r) return 0;
  int k = x - r;
  if (k < 0) k += m;
  return k <= (m - 1) / 2 ? k : m - k;
}

__device__ __forceinline__ int64_t local_index(int bp, int bq, int i) {
  return i < BW ? (int64_t)bp * BW + i : (int64_t)bq * BW + (i - BW);
}

__device__ __forceinline__ bool needs_rotation(double aij, double aii, double ajj, double tr, double ta,
                                               double floor_ = 0.0, double tang = 0.0) {
  const double a = fabs(aij);
  return a > ta && a > tr * sqrt(fabs(aii) * fabs(ajj)) && (floor_ <= 0.0 || fmax(aii, ajj) >= floor_) &&
         a > tang * fabs(ajj - aii);
}

// needs_rotation with the relative test squared (a^2 > tr^2 |a_ii a_jj|): no square root on the
// rotation's critical path (entries here are far from the under/overflow range of the square)
__device__ __forceinline__ bool needs_rotation_sq(double aij, double aii, double ajj, double tr, double ta,
                                                  double floor_ = 0.0, double tang = 0.0) {
  const double a = fabs(aij);
  return a > ta && a * a > tr * tr * fabs(aii * ajj) && (floor_ <= 0.0 || fmax(aii, ajj) >= floor_) &&
         a > tang * fabs(ajj - aii);
}

// C(64x64) = op(X) * Y with operands in smem, col-major stride TS.
//  transX = false: X(m,k) at X[k*TS + m];  transX = true: X(m,k) = X[m*TS + k]
// 8 warps: warp w owns rows (w&3)*16..+16 and cols (w>>2)*32..+32.
template <bool TRANSX, int SX = TS, int SY = TS>
__device__ __forceinline__ void mm64(const double* X, const double* Y, double (&acc)[2][4][2]) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int r0 = (warp & 3) * 16, c0 = (warp >> 2) * 32;
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  // per-thread fragment base pointers; the fully unrolled k loop then addresses shared memory
  // with immediate offsets (no per-step index arithmetic between the loads and the DMMAs)
  const double* xa0 = TRANSX ? X + (r0 + g) * SX + t : X + t * SX + r0 + g;
  const double* xa1 = TRANSX ? xa0 + 8 * SX : xa0 + 8;
  const double* yb = Y + (c0 + g) * SY + t;
  constexpr int XK = TRANSX ? 1 : SX;  // stride of k in X
#pragma unroll
  for (int k0 = 0; k0 < PS; k0 += 4) {
    const double a0 = xa0[k0 * XK], a1 = xa1[k0 * XK];
    double b[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) b[j] = yb[j * 8 * SY + k0];
#pragma unroll
    for (int j = 0; j < 4; ++j) dmma_8x8x4(acc[0][j], a0, b[j]);
#pragma unroll
    for (int j = 0; j < 4; ++j) dmma_8x8x4(acc[1][j], a1, b[j]);
  }
}

template <int SC = TS>
__device__ __forceinline__ void store_acc(double* C, const double (&acc)[2][4][2]) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int r0 = (warp & 3) * 16, c0 = (warp >> 2) * 32;
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) C[(c0 + j * 8 + 2 * t + e) * SC + r0 + i * 8 + g] = acc[i][j][e];
}

// Jacobi rotation of the 2x2 problem [[aii, aij], [aij, ajj]] (identity when r == 0):
// t = sgn(theta) / (|theta| + sqrt(1 + theta^2)), theta = (ajj - aii) / (2 aij), written with one
// square root and one division: t = 2 aij sgn(d) / (|d| + sqrt(d^2 + 4 aij^2))
__device__ __forceinline__ void rotation(double aii, double ajj, double aij, int r, double& c, double& s, double& t) {
  const double dd = ajj - aii, a2 = 2.0 * aij;
  const double tt = (dd >= 0.0 ? a2 : -a2) / (fabs(dd) + sqrt(fma(dd, dd, a2 * a2)));
  const double cc = rsqrt(fma(tt, tt, 1.0));
  t = r ? tt : 0.0;
  c = r ? cc : 1.0;
  s = r ? tt * cc : 0.0;
}

// n = R_P^T B R_Q for the 2x2 block B (rows of pair P, columns of pair Q), explicit fma order so
// the owner warps and the look-ahead produce the same bits
__device__ __forceinline__ void two_sided(double b00, double b01, double b10, double b11, double cp, double sp,
                                          double c, double s, double (&n)[4]) {
  const double m00 = fma(cp, b00, -(sp * b10)), m01 = fma(cp, b01, -(sp * b11));
  const double m10 = fma(sp, b00, cp * b10), m11 = fma(sp, b01, cp * b11);
  n[0] = fma(c, m00, -(s * m01));
  n[1] = fma(s, m00, c * m01);
  n[2] = fma(c, m10, -(s * m11));
  n[3] = fma(s, m10, c * m11);
}

// One pair's local solve (block k of round p.round) by a CTA of NT threads (NT/32 warps; warp w
// owns row pairs w, w + NT/32, ... and W rows w, w + NT/32, ...).  `sm` holds 3 PS x LS doubles.
template <int NT>
__device__ __forceinline__ void local_solve(const Params& p, int k, double* sm) {
  constexpr int NW = NT / 32;
  // A is double-buffered (each rotation step reads one copy and writes the other, so one
  // barrier per step suffices); W is column-major (Wl[j*LS + i] = w_ij) and its rows are
  // owned by warps (row % NW == warp), so W needs only __syncwarp between steps.
  double* Acur = sm;
  double* Anx = sm + PS * LS;
  double* Wl = sm + 2 * PS * LS;
  __shared__ int sperm[PS];

  int bp, bq;
  block_pair(p, k, bp, bq);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const double tr = p.tol_rel, ta = p.tol_abs * p.scal[0];
  // local floor: with an absolute trigger, entries below u*max|g_ii| are rounding noise -- do
  // not chase them; with a relative trigger (tol_abs tiny) the local solve follows it
  const double tloc = fmin(2.220446049250313e-16 * p.scal[0], ta);

  for (int e = tid; e < PS * PS; e += NT) {
    const int j = e / PS, i = e % PS;
    Acur[i * LS + j] = p.G[local_index(bp, bq, j) * p.np + local_index(bp, bq, i)];
  }
  __syncthreads();
  // anything to do?  |g_ij| > max(tol_abs * max|g_ii|, tol_rel * sqrt|g_ii g_jj|)
  int mine = 0;
  double moff = 0.0;
  for (int e = tid; e < PS * PS; e += NT) {
    const int i = e / PS, j = e % PS;
    if (i < j) {
      const double aij = Acur[i * LS + j];
      moff = fmax(moff, fabs(aij));
      if (needs_rotation(aij, Acur[i * LS + i], Acur[j * LS + j], tr, ta, p.keep_floor, p.tol_angle)) mine = 1;
    }
  }
  {
    // sweep-level maximum off-diagonal ratio (non-negative doubles order like their bits)
    double r = moff / p.scal[0];
    for (int o = 16; o > 0; o >>= 1) r = fmax(r, __shfl_xor_sync(0xffffffffu, r, o));
    if (lane == 0 && r > 0.0)
      atomicMax(reinterpret_cast<unsigned long long*>(p.maxoff), (unsigned long long)__double_as_longlong(r));
  }
  if (!__syncthreads_or(mine)) {
    if (tid == 0) p.flags[k] = 0;
    return;
  }
  for (int e = tid; e < PS * PS; e += NT) {
    const int j = e / PS, i = e % PS;
    Wl[j * LS + i] = (i == j) ? 1.0 : 0.0;
  }
  __syncthreads();

  // Rotation table, double-buffered by step parity: (c, s, t, r) of the 32 pairs of a step,
  // computed ONCE by warp 0 instead of redundantly by every warp (the FP64 pipe is shared with
  // the DMMA products of the apply CTAs co-resident in the fused round).  Look-ahead: during
  // step s warp 0 already forms the three entries of A_next each pair of step s+1 needs (the
  // same 2x2 transforms the owner warps apply, so the same bits) and that pair's rotation, so
  // a step still needs only its one closing barrier.
  __shared__ double tab_c[2][32], tab_s[2][32], tab_t[2][32];
  __shared__ int tab_r[2][32];
  auto make_rot = [&](double aii, double ajj, double aij, int buf) {
    const int r = needs_rotation_sq(aij, aii, ajj, tr, tloc, p.keep_floor, p.tol_angle);
    double c, s, t;
    rotation(aii, ajj, aij, r, c, s, t);
    tab_c[buf][lane] = c;
    tab_s[buf][lane] = s;
    tab_t[buf][lane] = t;
    tab_r[buf][lane] = r;
  };
  if (warp == 0) {
    int a, b;
    circle_pair(PS, 0, lane, a, b);
    make_rot(Acur[a * LS + a], Acur[b * LS + b], Acur[a * LS + b], 0);
  }
  __syncthreads();
  int cur = 0;
  for (int sweep = 0; sweep < p.max_local_sweeps; ++sweep) {
    int rotated = 0;
    for (int step = 0; step < PS - 1; ++step) {
      // rotation of pair `lane` from the table.  Branch-free: non-rotating pairs carry
      // (c, s, t) = (1, 0, 0), which leaves every entry bit-identical.
      int a, b;
      circle_pair(PS, step, lane, a, b);
      const double c = tab_c[cur][lane], s = tab_s[cur][lane], t = tab_t[cur][lane];
      const int r = tab_r[cur][lane];
      rotated |= r;
      if (warp == 0) {
        // look-ahead: pair `lane` of the next step is (x, y); x sits in pair kx of this step, y in ky
        const int ns = step + 1 < PS - 1 ? step + 1 : 0;
        int x, y, ax, bx, ay, by;
        circle_pair(PS, ns, lane, x, y);
        const int kx = pair_of(PS, step, x), ky = pair_of(PS, step, y);
        circle_pair(PS, step, kx, ax, bx);
        circle_pair(PS, step, ky, ay, by);
        const double txx = tab_t[cur][kx], tyy = tab_t[cur][ky];
        const double xx = x == ax ? fma(-txx, Acur[ax * LS + bx], Acur[ax * LS + ax])
                                  : fma(txx, Acur[ax * LS + bx], Acur[bx * LS + bx]);
        const double yy = y == ay ? fma(-tyy, Acur[ay * LS + by], Acur[ay * LS + ay])
                                  : fma(tyy, Acur[ay * LS + by], Acur[by * LS + by]);
        double n[4];
        two_sided(Acur[ax * LS + ay], Acur[ax * LS + by], Acur[bx * LS + ay], Acur[bx * LS + by], tab_c[cur][kx],
                  tab_s[cur][kx], tab_c[cur][ky], tab_s[cur][ky], n);
        const double xy = x == ax ? (y == ay ? n[0] : n[1]) : (y == ay ? n[2] : n[3]);
        make_rot(xx, yy, xy, cur ^ 1);
      }
      // A_next = R^T A R : this warp owns row pairs P = warp + NW h, column pair Q = lane; all
      // operands are loaded before any store
      {
        constexpr int NH = 32 / NW;
        int i1s[NH], j1s[NH];
        double cps[NH], sps[NH], v[NH][4];
#pragma unroll
        for (int h = 0; h < NH; ++h) {
          const int P = warp + NW * h;
          cps[h] = tab_c[cur][P];
          sps[h] = tab_s[cur][P];
          circle_pair(PS, step, P, i1s[h], j1s[h]);
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
          const double b00 = v[h][0], b01 = v[h][1], b10 = v[h][2], b11 = v[h][3];
          double n[4];
          two_sided(b00, b01, b10, b11, cps[h], sps[h], c, s, n);
          // the pair's own 2x2 block (b00 = a_ii, b01 = b10 = a_ij, b11 = a_jj): exact annihilation
          const double d00 = fma(-t, b01, b00), d11 = fma(t, b01, b11), od = r ? 0.0 : b01;
          const int i1 = i1s[h], j1 = j1s[h];
          Anx[i1 * LS + a] = dg ? d00 : n[0];
          Anx[i1 * LS + b] = dg ? od : n[1];
          Anx[j1 * LS + a] = dg ? od : n[2];
          Anx[j1 * LS + b] = dg ? d11 : n[3];
        }
      }
      // W <- W R on this warp's rows (identity for non-rotating pairs)
      {
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
      __syncwarp();
      double* tmp = Acur;
      Acur = Anx;
      Anx = tmp;
      cur ^= 1;
      __syncthreads();
    }
    if (!__syncthreads_or(rotated)) break;
  }
  // sorted Jacobi: order the local eigenvalues descending so large eigenvalues
  // migrate to the low blocks (the rank-of-diagonal permutation of W's columns)
  if (tid < PS) {
    const double di = Acur[tid * LS + tid];
    int rk = 0;
    for (int j = 0; j < PS; ++j) {
      const double dj = Acur[j * LS + j];
      rk += (dj > di) || (dj == di && j < tid);
    }
    sperm[rk] = tid;
  }
  __syncthreads();
  // one Bjorck step on DMMA (warps 0-7), W column-major in Wl:
  //   E = W^T W - I ;  W_new = W - W E / 2     (E in Anx, W_new staged in Acur)
  double* E = Anx;
  double* Wn = Acur;
  {
    double acc[2][4][2];
    if (warp < 8) mm64<true, LS, LS>(Wl, Wl, acc);   // A(m,k) = Wl[m*LS+k] = W(k,m), B(k,n) = Wl[n*LS+k] = W(k,n)
    __syncthreads();
    if (warp < 8) store_acc<LS>(E, acc);
    __syncthreads();
    for (int e = tid; e < PS; e += NT) E[e * LS + e] -= 1.0;
    __syncthreads();
    if (warp < 8) mm64<false, LS, LS>(Wl, E, acc);  // A(m,k) = Wl[k*LS+m] = W(m,k), B(k,n) = E(k,n)
    __syncthreads();
    if (warp < 8) {
      const int g = lane >> 2, t4 = lane & 3;
      const int r0 = (warp & 3) * 16, c0 = (warp >> 2) * 32;
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
          for (int e2 = 0; e2 < 2; ++e2) {
            const int m = r0 + i * 8 + g, n = c0 + j * 8 + 2 * t4 + e2;
            Wn[n * LS + m] = Wl[n * LS + m] - 0.5 * acc[i][j][e2];
          }
    }
    __syncthreads();
  }
  for (int e = tid; e < PS * PS; e += NT) {
    const int j = e / PS, i = e % PS;
    p.W[(int64_t)k * PS * PS + j * PS + i] = Wn[sperm[j] * LS + i];
  }
  if (tid == 0) {
    p.flags[k] = 1;
    atomicAdd(p.counter, 1);
  }
}

// async 16-byte copies: a 64x64 column-major W (contiguous) into smem stride TS
__device__ __forceinline__ void load_w(double* dst, const double* W) {
  for (int e = threadIdx.x; e < PS * PS / 2; e += AT) {
    const int j = e / (PS / 2), i = (e % (PS / 2)) * 2;
    cp_async_16(dst + j * TS + i, W + j * PS + i, 16);
  }
}

// async gather of the 64x64 tile M[I_rows, I_cols] (column-major, leading dimension ld)
__device__ __forceinline__ void load_tile(double* dst, const double* M, int64_t ld, int rp, int rq, int cp_, int cq) {
  for (int e = threadIdx.x; e < PS * PS / 2; e += AT) {
    const int j = e / (PS / 2), i = (e % (PS / 2)) * 2;
    const int64_t col = local_index(cp_, cq, j), row = local_index(rp, rq, i);
    cp_async_16(dst + j * TS + i, M + col * ld + row, 16);
  }
}

__device__ __forceinline__ void load_slab(double* dst, const double* V, int64_t ld, int64_t row0, int cp_, int cq) {
  for (int e = threadIdx.x; e < PS * PS / 2; e += AT) {
    const int j = e / (PS / 2), i = (e % (PS / 2)) * 2;
    cp_async_16(dst + j * TS + i, V + local_index(cp_, cq, j) * ld + row0 + i, 16);
  }
}

// Result tile (mm64 fragment layout: acc[i][j][e] = C[r0 + 8i + g][c0 + 8j + 2t + e]) straight from
// the accumulators to global memory.  G tile (rows of pair (rp, rq), columns of pair (cp_, cq)):
// the tile and its mirror (the mirror as 16-byte stores of two consecutive rows); a diagonal
// tile writes only its r <= c entries, both ways, so G stays exactly symmetric.
__device__ __forceinline__ void write_acc_g(const Params& p, const double (&acc)[2][4][2], int rp, int rq, int cp_,
                                            int cq, bool diag) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int r0 = (warp & 3) * 16, c0 = (warp >> 2) * 32;
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int r = r0 + i * 8 + g;
    const int64_t ri = local_index(rp, rq, r);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = c0 + j * 8 + 2 * t;
      const int64_t ci = local_index(cp_, cq, c);
      const double v0 = acc[i][j][0], v1 = acc[i][j][1];
      if (!diag) {
        p.G[ci * p.np + ri] = v0;
        p.G[(ci + 1) * p.np + ri] = v1;
        *reinterpret_cast<double2*>(p.G + ri * p.np + ci) = make_double2(v0, v1);
      } else {
        if (r <= c) {
          p.G[ci * p.np + ri] = v0;
          p.G[ri * p.np + ci] = v0;
        }
        if (r <= c + 1) {
          p.G[(ci + 1) * p.np + ri] = v1;
          p.G[ri * p.np + ci + 1] = v1;
        }
      }
    }
  }
}

__device__ __forceinline__ void write_acc_v(const Params& p, const double (&acc)[2][4][2], int cp_, int cq,
                                            int64_t row0) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int r0 = (warp & 3) * 16, c0 = (warp >> 2) * 32;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int c = c0 + j * 8 + 2 * t;
    double* v = p.V + local_index(cp_, cq, c) * p.np + row0 + r0 + g;
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      v[i * 8] = acc[i][j][0];
      v[p.np + i * 8] = acc[i][j][1];
    }
  }
}

// One task of the apply step (a G tile or a V slab); returns after its stores.
__device__ __forceinline__ void apply_task(const Params& p, int64_t b, int64_t ng, int npairs, double* X,
                                           double* WQ, double* WP, int& wq_loaded) {
  double acc[2][4][2];
  if (b < ng) {
    // G tile (P, Q), P <= Q: column-major enumeration of the upper triangle, b = Q(Q+1)/2 + P
    int Q = (int)((sqrt(8.0 * (double)b + 1.0) - 1.0) * 0.5);
    while ((int64_t)(Q + 1) * (Q + 2) / 2 <= b) ++Q;
    while ((int64_t)Q * (Q + 1) / 2 > b) --Q;
    const int P = (int)(b - (int64_t)Q * (Q + 1) / 2);
    if (p.phase == 2 && p.tile_mark[b] == p.stamp) return;  // applied by the "needed" pass
    const int fP = p.flags[P], fQ = p.flags[Q];
    if (!fP && !fQ) return;
    int pp, pq, qp, qq;
    block_pair(p, P, pp, pq);
    block_pair(p, Q, qp, qq);
    load_tile(X, p.G, p.np, pp, pq, qp, qq);
    if (fQ && wq_loaded != Q) load_w(WQ, p.W + (int64_t)Q * PS * PS);
    if (fQ) wq_loaded = Q;
    if (fP) load_w(WP, p.W + (int64_t)P * PS * PS);
    cp_async_commit();
    if (threadIdx.x == 0) atomicAdd(p.mm_count, (unsigned long long)(fP + fQ));
    cp_async_wait<0>();
    __syncthreads();
    if (fQ) {
      mm64<false>(X, WQ, acc);  // X W_Q
      if (!fP) {
        write_acc_g(p, acc, pp, pq, qp, qq, P == Q);
        return;
      }
      __syncthreads();
      store_acc(X, acc);
      __syncthreads();
    }
    mm64<true>(WP, X, acc);     // W_P^T X  (fP set here)
    write_acc_g(p, acc, pp, pq, qp, qq, P == Q);
    return;
  }
  // V slab: rows [rc*64, rc*64+64), columns of pair Q (Q-major, so consecutive tasks share W_Q)
  const int64_t vb = b - ng;
  const int64_t nrc = p.nslab + (p.slab_extra >= 0);
  const int Q = (int)(vb / nrc);
  const int64_t ri = vb % nrc;
  const int64_t rc = ri < p.nslab ? p.slab0 + ri : p.slab_extra;
  if (!p.flags[Q]) return;
  int qp, qq;
  block_pair(p, Q, qp, qq);
  load_slab(X, p.V, p.np, rc * PS, qp, qq);
  if (wq_loaded != Q) load_w(WQ, p.W + (int64_t)Q * PS * PS);
  wq_loaded = Q;
  cp_async_commit();
  if (threadIdx.x == 0) atomicAdd(p.mm_count, 1ull);
  cp_async_wait<0>();
  __syncthreads();
  mm64<false>(X, WQ, acc);
  write_acc_v(p, acc, qp, qq, rc * PS);
}

__device__ __forceinline__ void rest_tasks(const Params& p, double* X, double* WQ, double* WP);


// Persistent apply: a fixed grid (2 CTAs per SM) walks all tasks; tasks of pairs that
// needed no rotation cost two flag loads instead of a CTA launch.
__global__ void __launch_bounds__(AT, 2) jac_apply(Params p) {
  extern __shared__ double sm[];
  double* X = sm;
  double* WQ = X + PS * TS;
  double* WP = WQ + PS * TS;
  const int npairs = p.nb / 2;
  const int64_t ng = (int64_t)npairs * (npairs + 1) / 2;
  if (p.phase == 1) {
    if (blockIdx.x == 0 && threadIdx.x == 0) *p.task_counter = 0ull;  // for the "rest" pass that follows
    // the tiles the next round's local solves read: every pair's diagonal tile and, for each
    // pair (x, y) of round r+1, the tile holding block (x, y); claimed with the round stamp
    __shared__ int go;
    const int rn = (p.round + 1) % (p.nb - 1);
    int wq_loaded = -1;
    for (int t = blockIdx.x; t < 2 * npairs; t += gridDim.x) {
      int P, Q;
      if (t < npairs) {
        P = Q = t;
      } else {
        int x, y;
        circle_pair(p.nb, rn, t - npairs, x, y);
        const int P1 = pair_of(p.nb, p.round, x), P2 = pair_of(p.nb, p.round, y);
        P = min(P1, P2);
        Q = max(P1, P2);
      }
      const int64_t b = (int64_t)Q * (Q + 1) / 2 + P;
      if (threadIdx.x == 0) go = atomicExch(p.tile_mark + b, p.stamp) != p.stamp;
      __syncthreads();
      if (go) apply_task(p, b, ng, npairs, X, WQ, WP, wq_loaded);
      __syncthreads();
    }
    return;
  }
  rest_tasks(p, X, WQ, WP);
}

// The "rest" apply pass of round p.round: every G tile / V slab not already applied by the
// "needed" pass, dynamically scheduled.
__device__ __forceinline__ void rest_tasks(const Params& p, double* X, double* WQ, double* WP) {
  const int npairs = p.nb / 2;
  const int64_t ng = (int64_t)npairs * (npairs + 1) / 2;
  const int64_t ntasks = ng + (int64_t)(p.nslab + (p.slab_extra >= 0)) * npairs;
  // dynamic scheduling in chunks of consecutive tasks (which mostly share the column pair Q, whose
  // rotation then stays in shared memory): the heavy G tiles (two 64^3 products) come first, the
  // V slabs (one product) last, and CTAs sharing an SM with a local solve simply take fewer chunks
  constexpr int CH = 4;
  __shared__ long long s_next;
  int wq_loaded = -1;
  for (;;) {
    if (threadIdx.x == 0) s_next = (long long)atomicAdd(p.task_counter, (unsigned long long)CH);
    __syncthreads();
    const int64_t b0 = s_next;
    __syncthreads();
    if (b0 >= ntasks) break;
    const int64_t b1 = min(ntasks, b0 + CH);
    for (int64_t b = b0; b < b1; ++b) {
      apply_task(p, b, ng, npairs, X, WQ, WP, wq_loaded);
      __syncthreads();  // smem reuse by the next task
    }
  }
}

// One Jacobi round after its "needed" pass: CTAs 0..npairs-1 first solve the local problems of
// round r+1 (they only read tiles the needed pass of round r has finished), then every CTA takes
// chunks of round r's remaining apply tasks.  One launch, one stream: the local solves (the
// round's critical path) start at once and the apply fills the SMs around them.
__global__ void __launch_bounds__(AT, 2) jac_round(Params pa, Params pl, int do_local, int do_rest) {
  extern __shared__ double sm[];
  if (do_local && blockIdx.x < pl.nb / 2) {
    local_solve<AT>(pl, blockIdx.x, sm);
    __syncthreads();
  }
  if (do_rest) rest_tasks(pa, sm, sm + PS * TS, sm + 2 * PS * TS);
}

__global__ void pad_copy(const double* G, int64_t ldg, int64_t n, double* Gp, double* Vp, int64_t np) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= np * np) return;
  const int64_t j = e / np, i = e % np;
  Gp[e] = (i < n && j < n) ? G[j * ldg + i] : 0.0;
  Vp[e] = (i == j) ? 1.0 : 0.0;
}

__global__ void max_abs_diag(const double* Gp, int64_t np, int64_t n, double* out) {
  __shared__ double red[256];
  double m = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) m = fmax(m, fabs(Gp[i * np + i]));
  red[threadIdx.x] = m;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = red[0] > 0.0 ? red[0] : 1.0;
}

// Rayleigh quotients against the ORIGINAL Gramian: rq_i = v_i^T (G0 v_i), one
// warp per column, fixed summation order (deterministic).  Removes the
// eigenvalue drift that the accumulated local rotations leave in diag(G).
// Columns whose real part (rows < n) vanishes are padding eigenvectors (exact
// unit vectors of the zero padding, never mixed with real coordinates): -inf.
// Y == nullptr: no refinement, the value is the converged diagonal entry Y0[col*ldy0 + col].
__global__ void rq_diag(const double* V, int64_t ldv, const double* Y, int64_t ldy, int64_t n, int64_t ncols,
                        double* out, const double* diag_src = nullptr, int64_t ld_diag = 0, int by_padding_rows = 0) {
  const int64_t col = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (col >= ncols) return;
  if (by_padding_rows) {
    // partial V (only some row slabs accumulated): a padding eigenvector is a unit vector of the
    // padding rows [n, ncols) -- rows every partial call accumulates -- a real one vanishes there
    double pp = 0.0;
    for (int64_t k = n + lane; k < ncols; k += 32) {
      const double v = V[col * ldv + k];
      pp += v * v;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) pp += __shfl_xor_sync(0xffffffffu, pp, o);
    if (lane == 0) out[col] = pp > 0.5 ? -INFINITY : diag_src[col * ld_diag + col];
    return;
  }
  double s = 0.0, nn = 0.0;
  for (int64_t k = lane; k < n; k += 32) {
    const double v = V[col * ldv + k];
    if (Y) s += v * Y[col * ldy + k];
    nn += v * v;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s += __shfl_xor_sync(0xffffffffu, s, o);
    nn += __shfl_xor_sync(0xffffffffu, nn, o);
  }
  if (lane == 0) out[col] = nn > 0.5 ? (Y ? s / nn : diag_src[col * ld_diag + col]) : -INFINITY;
}

// rank of each value in descending order, ties broken by index
__global__ void sort_rank(const double* dvals, int64_t n, int64_t keep, double* lam, int* perm) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double di = dvals[i];
  int64_t r = 0;
  for (int64_t j = 0; j < n; ++j) {
    const double dj = dvals[j];
    r += (dj > di) || (dj == di && j < i);
  }
  if (r < keep) {
    lam[r] = di;
    perm[r] = (int)i;
  }
}

__global__ void gather_vectors(const double* Vp, int64_t np, int64_t n, const int* perm, int64_t nvec, double* V,
                               int64_t ldv) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n * nvec) return;
  const int64_t k = e / n, i = e % n;
  V[k * ldv + i] = Vp[(int64_t)perm[k] * np + i];
}

struct Layout {
  int64_t np;
  int nb;
  size_t off_G, off_V, off_W, off_flags, off_marks, off_counter, off_scal, off_perm, off_rq, off_gemm, total;
};

Layout layout(int64_t n) {
  Layout L;
  int nb = (int)ceil_div(std::max<int64_t>(n, 1), BW);
  if (nb < 2) nb = 2;
  if (nb & 1) ++nb;
  L.nb = nb;
  L.np = (int64_t)nb * BW;
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  size_t o = 0;
  L.off_G = o;
  o = al(o + (size_t)L.np * L.np * 8);
  L.off_V = o;
  o = al(o + (size_t)L.np * L.np * 8);
  L.off_W = o;
  o = al(o + 2 * (size_t)(nb / 2) * PS * PS * 8);  // double-buffered by round parity
  L.off_flags = o;
  o = al(o + 2 * (size_t)(nb / 2) * 4);
  L.off_marks = o;
  o = al(o + (size_t)(nb / 2) * (nb / 2 + 1) / 2 * 4);
  L.off_counter = o;
  o = al(o + 64);
  L.off_scal = o;
  o = al(o + 16);
  L.off_perm = o;
  o = al(o + (size_t)L.np * 4);
  L.off_rq = o;
  o = al(o + (size_t)L.np * 8);
  L.off_gemm = o;
  o = al(o + gemm_workspace_bytes(n, L.np, n, 0, 0));
  L.total = o;
  return L;
}

}  // namespace jac

size_t syev_workspace_bytes(int64_t n) { return jac::layout(n).total; }
int64_t syev_padded_order(int64_t n) { return jac::layout(n).np; }

int syev_run(const double* G, int64_t ldg, int64_t n, double* lam_desc, double* V, int64_t ldv, int64_t nvec,
             double tol_rel, double tol_abs, double tol_angle, double keep_floor, int max_sweeps, int refine,
             int* sweeps_out, double* flops_out, void* ws, size_t ws_bytes, cudaStream_t st, int64_t vrow0,
             int64_t vrow1) {
  using namespace jac;
  HP_REQUIRE(n >= 0, "syev: negative order");
  if (sweeps_out) *sweeps_out = 0;
  if (n == 0) return HP_OK;
  HP_REQUIRE(ldg >= n && ldv >= n, "syev: leading dimension too small");
  HP_REQUIRE(nvec >= 0 && nvec <= n, "syev: nvec out of range");
  const Layout L = layout(n);
  HP_REQUIRE(ws_bytes >= L.total, "syev: workspace too small");
  char* base = static_cast<char*>(ws);
  Params p{};
  p.G = reinterpret_cast<double*>(base + L.off_G);
  p.V = reinterpret_cast<double*>(base + L.off_V);
  double* W_base = reinterpret_cast<double*>(base + L.off_W);
  int* flags_base = reinterpret_cast<int*>(base + L.off_flags);
  p.W = W_base;
  p.flags = flags_base;
  p.tile_mark = reinterpret_cast<int*>(base + L.off_marks);
  p.counter = reinterpret_cast<int*>(base + L.off_counter);
  p.maxoff = reinterpret_cast<double*>(base + L.off_counter + 16);
  p.mm_count = reinterpret_cast<unsigned long long*>(base + L.off_counter + 24);
  p.task_counter = reinterpret_cast<unsigned long long*>(base + L.off_counter + 32);
  double* scal = reinterpret_cast<double*>(base + L.off_scal);
  p.scal = scal;
  int* perm = reinterpret_cast<int*>(base + L.off_perm);
  p.np = L.np;
  p.nb = L.nb;
  // rows of V this call accumulates: whole 64-row slabs [vrow0, vrow1) (vrow1 < 0: all rows).  The
  // eigenvalues and every other row of the iteration do not depend on the range.
  if (vrow1 < 0) {
    vrow0 = 0;
    vrow1 = L.np;
  }
  HP_REQUIRE(vrow0 >= 0 && vrow0 <= vrow1 && vrow1 <= L.np && vrow0 % PS == 0 && (vrow1 % PS == 0 || vrow1 == L.np),
             "syev: V row range must be whole 64-row slabs");
  const bool partial = !(vrow0 == 0 && vrow1 == L.np);
  HP_REQUIRE(!partial || !refine, "syev: Rayleigh refinement needs all rows of V");
  p.slab0 = (int)(vrow0 / PS);
  p.nslab = (int)(ceil_div(vrow1, (int64_t)PS) - p.slab0);
  // a partial call also accumulates the last slab: it holds the padding rows (np - n < 64 of them),
  // whose entries tell padding eigenvectors from real ones without the other ranks' rows
  const int last_slab = (int)(L.np / PS) - 1;
  p.slab_extra = (partial && L.np > n && p.slab0 + p.nslab <= last_slab) ? last_slab : -1;
  p.tol_rel = tol_rel;
  p.tol_abs = tol_abs;
  p.keep_floor = keep_floor;
  p.tol_angle = tol_angle;
  // Local cyclic sweeps per pair: a large matrix in its first (full-apply) phase has its local
  // solves hidden under the apply of the fused round, so two local sweeps buy fewer outer sweeps
  // (root H phase 820 -> 778 ms); small problems (leaves, merges) and the nearly diagonal polish
  // (keep_floor > 0, few active pairs) have the local solve on the critical path: one sweep.
  p.max_local_sweeps = (layout(n).nb / 2 >= 32 && keep_floor <= 0.0) ? 2 : 1;

  static std::atomic<unsigned long long> configured{0};
  const int apply_smem = 3 * PS * TS * 8;
  const int rc0 = once_per_device(configured, [&]() -> int {
    HP_CHECK_CUDA(cudaFuncSetAttribute(jac_round, cudaFuncAttributeMaxDynamicSharedMemorySize, apply_smem));
    HP_CHECK_CUDA(cudaFuncSetAttribute(jac_apply, cudaFuncAttributeMaxDynamicSharedMemorySize, apply_smem));
    return (int)HP_OK;
  });
  if (rc0 != HP_OK) return rc0;
  const int64_t npn = L.np * L.np;
  pad_copy<<<(unsigned)ceil_div(npn, 256), 256, 0, st>>>(G, ldg, n, p.G, p.V, L.np);
  HP_CHECK_LAUNCH("pad_copy");
  max_abs_diag<<<1, 256, 0, st>>>(p.G, L.np, n, scal);
  HP_CHECK_LAUNCH("max_abs_diag");

  const int npairs = L.nb / 2;
  const int64_t napply = (int64_t)npairs * (npairs + 1) / 2 + (int64_t)(p.nslab + (p.slab_extra >= 0)) * npairs;
  int nsm = 148, dev = 0;
  HP_CHECK_CUDA(cudaGetDevice(&dev));
  HP_CHECK_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));

  char* host_buf = pinned_scratch();
  HP_REQUIRE(host_buf != nullptr, "syev: pinned host scratch unavailable");
  HP_CHECK_CUDA(zero_async(p.mm_count, 8, st));
  int status = HP_ELINALG;
  int sweep = 0;
  double prev_off = INFINITY;
  unsigned long long mm_total = 0;
  const double floor_ratio = 512.0 * 2.220446049250313e-16;
  const int dbg = debug_flags();
  const int trace = (dbg & DBG_JACOBI_ROUND_TIMING) ? 2 : (dbg & DBG_JACOBI_TRACE) ? 1 : 0;
  cudaEvent_t ev[3];
  if (trace > 1)
    for (auto& e : ev) cudaEventCreate(&e);
  const unsigned needed_grid = (unsigned)std::min<int64_t>(2 * (int64_t)npairs, 2 * (int64_t)nsm);  // one task per CTA (2 per SM)
  // small problems (leaves, merges) get a grid sized to their work -- about four apply tasks per
  // CTA, never fewer CTAs than local solves -- so that concurrent node streams do not flood the
  // SMs with idle apply CTAs; large ones use every SM twice
  const unsigned rest_grid =
      (unsigned)std::min<int64_t>(std::max<int64_t>(npairs, ceil_div(napply, 4)), 2 * (int64_t)nsm);
  // One sweep = 2 R + 4 dependent launches with the same arguments every sweep (round stamps restart at 1;
  // the tile marks are cleared per sweep).  Small problems (leaves, chain merges: kernels of a few
  // microseconds, 16 host threads launching at once in a leaf wave) replay the sweep as a CUDA graph
  // captured on this thread's side stream, so a sweep costs one launch call instead of ~30-130.
  const int R = L.nb - 1;
  auto enqueue_sweep = [&](cudaStream_t ls) -> cudaError_t {
    cudaError_t e = zero_async(p.counter, 24, ls);
    if (e != cudaSuccess) return e;
    e = zero_async(p.tile_mark, (size_t)npairs * (npairs + 1) / 2 * 4, ls);
    if (e != cudaSuccess) return e;
    // Per round r: needed(r), then ONE fused launch in which CTAs 0..npairs-1 solve the local
    // problems of round r+1 before joining the dynamically scheduled rest of round r's apply.
    auto round_params = [&](int r) {
      Params q = p;
      q.round = r;
      q.W = W_base + (size_t)(r & 1) * npairs * PS * PS;
      q.flags = flags_base + (size_t)(r & 1) * npairs;
      q.stamp = r + 1;
      return q;
    };
    jac_round<<<npairs, AT, apply_smem, ls>>>(round_params(0), round_params(0), 1, 0);
    for (int r = 0; r < R; ++r) {
      Params q = round_params(r);
      q.phase = 1;
      jac_apply<<<needed_grid, AT, apply_smem, ls>>>(q);
      if (trace > 1 && r == R / 2) cudaEventRecord(ev[0], ls);
      q.phase = 2;
      jac_round<<<rest_grid, AT, apply_smem, ls>>>(q, round_params(r + 1 < R ? r + 1 : 0), r + 1 < R, 1);
      if (trace > 1 && r == R / 2) {
        cudaEventRecord(ev[1], ls);
        cudaEventRecord(ev[2], ls);
      }
    }
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    return d2h_small(host_buf, p.counter, 32, ls);  // counter, maxoff, mm_count
  };
  struct GraphHolder {
    cudaGraphExec_t exec = nullptr;
    ~GraphHolder() {
      if (exec) cudaGraphExecDestroy(exec);
    }
  } graph;
  // ... when several host threads are in this routine at once (a leaf wave on stream workers): a
  // single stream's launches already run ahead of the GPU, and capturing + instantiating a graph per
  // solve then costs more than it saves (config 2's chain merges: +1.2 ms per merge).
  static std::atomic<int> active_solves{0};
  struct ActiveGuard {
    std::atomic<int>& c;
    int seen;
    explicit ActiveGuard(std::atomic<int>& a) : c(a), seen(a.fetch_add(1, std::memory_order_relaxed) + 1) {}
    ~ActiveGuard() { c.fetch_sub(1, std::memory_order_relaxed); }
  } guard(active_solves);
  bool use_graph = L.np <= GRAPH_MAX_ORDER && trace < 2 && guard.seen >= GRAPH_MIN_CONCURRENCY && !(dbg & DBG_NO_GRAPHS);
  cudaStream_t ls = st;
  if (use_graph) {
    // the side stream starts after everything queued on st; every sweep ends in a host sync of the
    // side stream, so the work queued on st afterwards is ordered behind it
    thread_local cudaStream_t side = nullptr;
    thread_local cudaEvent_t dep = nullptr;
    if (!side) {
      // highest priority: the sweeps are chains of microsecond kernels that would otherwise queue
      // behind the other leaves' full-chip GEMM tiles
      int lo_pri = 0, hi_pri = 0;
      cudaDeviceGetStreamPriorityRange(&lo_pri, &hi_pri);
      if (cudaStreamCreateWithPriority(&side, cudaStreamNonBlocking, hi_pri) != cudaSuccess) side = nullptr;
    }
    if (!dep && cudaEventCreateWithFlags(&dep, cudaEventDisableTiming) != cudaSuccess) dep = nullptr;
    if (side && dep && cudaEventRecord(dep, st) == cudaSuccess && cudaStreamWaitEvent(side, dep, 0) == cudaSuccess)
      ls = side;
    else
      use_graph = false;
    (void)cudaGetLastError();
  }
  for (; sweep < max_sweeps; ++sweep) {
    cudaError_t e = cudaSuccess;
    if (use_graph && !graph.exec) {
      cudaGraph_t g = nullptr;
      e = cudaStreamBeginCapture(ls, cudaStreamCaptureModeThreadLocal);
      if (e == cudaSuccess) {
        const cudaError_t eq = enqueue_sweep(ls);
        e = cudaStreamEndCapture(ls, &g);
        if (e == cudaSuccess) e = eq;
      }
      if (e == cudaSuccess) e = cudaGraphInstantiate(&graph.exec, g, 0);
      if (g) cudaGraphDestroy(g);
      if (e != cudaSuccess) {  // no capture on this stream / driver: launch directly
        (void)cudaGetLastError();
        graph.exec = nullptr;
        use_graph = false;
        e = cudaSuccess;
      }
    }
    if (use_graph)
      e = cudaGraphLaunch(graph.exec, ls);
    else
      e = enqueue_sweep(ls);
    count_launches(2 * R + 4);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ls);
    if (e != cudaSuccess) {
      set_error(std::string("syev sweep: ") + cudaGetErrorString(e));
      return HP_ECUDA;
    }
    const int worked = *reinterpret_cast<int*>(host_buf);
    const double off = *reinterpret_cast<double*>(host_buf + 16);
    mm_total = *reinterpret_cast<unsigned long long*>(host_buf + 24);
    if (trace) {
      float t_local = 0.f, t_apply = 0.f;
      if (trace > 1) {
        cudaEventElapsedTime(&t_local, ev[0], ev[1]);
        cudaEventElapsedTime(&t_apply, ev[1], ev[2]);
      }
      fprintf(stderr, "[hp_syev n=%lld] sweep %d: pairs worked %d / %d, max off/diag %.3e  (mid-round: local %.1f us, apply %.1f us)\n",
              (long long)n, sweep, worked, npairs * (L.nb - 1), off, 1e3f * t_local, 1e3f * t_apply);
    }
    if (worked == 0 || (off < floor_ratio && off > 0.5 * prev_off)) {
      status = HP_OK;
      break;
    }
    prev_off = off;
  }
  if (sweeps_out) *sweeps_out = sweep + (status == HP_OK ? 1 : 0);
  // algorithmic flops of the DMMA rotation products (+ the Rayleigh-quotient GEMM below)
  if (flops_out) *flops_out = (double)mm_total * 2.0 * PS * PS * PS + (refine ? 2.0 * (double)n * n * (double)L.np : 0.0);
  if (status != HP_OK) {
    set_error("syev: Jacobi iteration did not converge");
    return HP_ELINALG;
  }
  // Rayleigh-quotient refinement (refine != 0): Y = G0 V (Y reuses the padded G buffer),
  // rq_i = v_i . y_i / v_i . v_i; otherwise the converged diagonal.  Padding columns -> -inf.
  {
    double* rq = reinterpret_cast<double*>(base + L.off_rq);
    if (refine) {
      VecSet a{G, ldg, nullptr};
      VecSet b{p.V, L.np, nullptr};
      const bool al16 = (ldg % 2 == 0) && ((uintptr_t)G % 16 == 0);
      int rc = gemm_run(false, true, n, L.np, n, a, b, al16, 1.0, 0.0, p.G, L.np, nullptr, nullptr, nullptr, 0, 0,
                        base + L.off_gemm, L.total - L.off_gemm, st);
      if (rc) return rc;
      rq_diag<<<(unsigned)ceil_div(L.np, 8), 256, 0, st>>>(p.V, L.np, p.G, L.np, n, L.np, rq);
    } else {
      rq_diag<<<(unsigned)ceil_div(L.np, 8), 256, 0, st>>>(p.V, L.np, nullptr, 0, n, L.np, rq, p.G, L.np, partial ? 1 : 0);
    }
    HP_CHECK_LAUNCH("rq_diag");
    // rank all n_p columns (padding last), keep the first n
    sort_rank<<<(unsigned)ceil_div(L.np, 256), 256, 0, st>>>(rq, L.np, n, lam_desc, perm);
    HP_CHECK_LAUNCH("sort_rank");
  }
  if (nvec > 0) {
    gather_vectors<<<(unsigned)ceil_div(n * nvec, 256), 256, 0, st>>>(p.V, L.np, n, perm, nvec, V, ldv);
    HP_CHECK_LAUNCH("gather_vectors");
  }
  return HP_OK;
}

}  // namespace hp
