// FP64 DMMA GEMM engine for the HAPOD node contractions (sm_100a).
//
//   K1  Gram SYRK      G = S^T S                 (pod.py:208-211, 87-91)   "TN", sym
//   K1b mixed block    sigma o (Phi^T F)         (pod.py:376-384)          "TN", row scale
//   K4  reconstruction U = (S V[:, :N]) / sigma  (pod.py:333-334)          "NN", column divide
//   K5  drift check    U^T U                     (pod.py:245-247)          "TN", sym
//   CholQR / Cholesky trailing updates                                     "NN" / "NT"
//
// FP64 tensor work on sm_100a is warp-level DMMA (mma.sync m8n8k4 f64 ->
// SASS DMMA.8x8x4); tcgen05 has no f64 kind.  Measured on this pool's B200:
// DMMA peaks at 37.1 TFLOP/s (tools/microbench/fp64_peak.cu).
//
// Tiling: 128x128 CTA tile, 8 warps as 2 (m) x 4 (n), warp tile 64x32 =
// 8x4 DMMA fragments (64 fp64 accumulators / thread), K tile 16, 4-stage
// cp.async (LDGSTS) ring with zero-fill at every edge.  The k index is
// permuted inside a K tile (k = 4t + s when both operands are K-major) so
// each lane fetches its fragments with 128-bit shared loads; row strides are
// padded so those loads are bank-conflict free.
//
// Operands are VecSets (base+ld or a per-vector pointer table), so a node's
// input can be the concatenation of its children's mode blocks without an
// hstack copy.  Split-K over long contractions writes per-split partial tiles
// that a second kernel sums in a FIXED order: results are bit-identical run to
// run and independent of how many GPUs take part (no atomics).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>
#include <vector>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "hp_common.cuh"

namespace hp {
namespace gemm {

constexpr int BM = 128, BN = 128, BK = 16, STAGES = 4, THREADS = 256;
constexpr int LDM = BM + 2;  // [k][m] rows: LD = 2 mod 8 -> conflict-free 128-bit fragment loads

struct Params {
  int64_t M, N, K;
  VecSet A, B;
  double* C;
  int64_t ldc;
  double alpha, beta;
  const double* row_scale;
  const double* col_scale;
  const double* col_div;
  int sym;  // 0 general; 1 symmetric output: tiles bi <= bj computed, entries mirrored; 2 the same, upper part only (no mirror)
  int b_upper;
  int splits;
  int64_t kspan;
  double* partial;
  int tiles_m, tiles_n;
  int64_t ntiles;
  int bn;  // tile width in n: 128, or 96 / 64 for narrow NN / TN outputs on the TMA path (K-major B)
};

template <bool AK, bool BKM>
struct Layout {
  static constexpr bool MODEP = AK && BKM;       // both operands K-major: k = 4t + s
  static constexpr int LDK = MODEP ? 18 : 20;    // [row][k] stride
  static constexpr int A_ELEMS = AK ? BM * LDK : BK * LDM;
  static constexpr int B_ELEMS = BKM ? BN * LDK : BK * LDM;
  static constexpr int STAGE_ELEMS = A_ELEMS + B_ELEMS;
  static constexpr int SMEM_BYTES = STAGES * STAGE_ELEMS * 8;
};

// Tile order (L2 reuse): tiles are rasterised in groups of GN column panels, row-major inside a
// group, so the ~148 tiles of one wave share ~18 row panels and GN column panels instead of
// reading 148 different row panels against one column panel (the plain column-major order read
// the A operand of the config-1 reconstruction 36 times from HBM: 478 GB for 13 GB of input).
// The order only relabels tiles -- every tile is still one CTA over its full K range (or the
// same fixed split-K slices) -- so results are bitwise unchanged.
constexpr int GN = 8;

__device__ __forceinline__ void tile_coords(const Params& p, int64_t t, int& bi, int& bj) {
  if (p.sym) {
    // strictly upper triangle (bi < bj) in super-columns of GN tile columns -- group g holds columns
    // [g GN, g GN + gn): first the full rows bi < g GN (gn tiles each), then the group's own triangle
    // -- and the T diagonal tiles last.  A diagonal tile costs about half a tile on the TMA path
    // (mma_ktile_diag): in the middle of a launch it would take its SM out of step with the wave
    // that shares its operand panels in L2 (ncu: root Gram DRAM reads 115 -> 177 GB); at the end
    // the diagonal tiles fill the last, partial wave.  Also the order make_plan's makespan model
    // and the kernel's longest-first block order of small split-K outputs assume.
    const int T = p.tiles_m;
    const int64_t off = (int64_t)T * (T - 1) / 2;
    if (t >= off) {
      bi = bj = (int)(t - off);
    } else {
      int g = 0;
      while (true) {
        const int64_t c1 = (int64_t)min(T, (g + 1) * GN);
        if (c1 * (c1 - 1) / 2 > t) break;
        ++g;
      }
      const int c0 = g * GN, gn = min(T, c0 + GN) - c0;
      int64_t r = t - (int64_t)c0 * (c0 - 1) / 2;
      if (r < (int64_t)c0 * gn) {
        bi = (int)(r / gn);
        bj = c0 + (int)(r % gn);
      } else {
        r -= (int64_t)c0 * gn;
        int i = 0;
        while (r >= gn - 1 - i) {
          r -= gn - 1 - i;
          ++i;
        }
        bi = c0 + i;
        bj = c0 + i + 1 + (int)r;
      }
    }
  } else {
    const int64_t per_group = (int64_t)p.tiles_m * GN;
    const int g = (int)(t / per_group);
    const int c0 = g * GN, gn = min(p.tiles_n, c0 + GN) - c0;
    const int64_t r = t - (int64_t)g * per_group;
    bi = (int)(r / gn);
    bj = c0 + (int)(r % gn);
    // upper-triangular B: tiles of later columns contract over longer K -- schedule them first
    if (p.b_upper) bj = p.tiles_n - 1 - bj;
  }
}

// Load one operand tile into shared memory.
//  kmajor: `rows` vectors (m or n) of BK contiguous k's      -> s[row][k]  (LDK)
//  else  : BK vectors (k) of `rows` contiguous m's (or n's)  -> s[k][row]  (LDM)
template <bool KMAJOR, bool VEC, int LDK>
__device__ __forceinline__ void load_operand(double* s, const VecSet& op, int64_t r0, int64_t rlim, int64_t k0,
                                             int64_t kend, int tid) {
#pragma unroll
  for (int it = 0; it < 4; ++it) {
    const int c = tid + it * THREADS;
    int srow, scol;  // smem coordinates
    int64_t vec_idx, off;
    int nvalid;
    if (KMAJOR) {
      const int row = c >> 3, kc = (c & 7) * 2;
      const int64_t gr = r0 + row, gk = k0 + kc;
      vec_idx = gr < rlim ? gr : 0;
      off = gk;
      nvalid = gr < rlim ? (int)max((int64_t)0, min((int64_t)2, kend - gk)) : 0;
      srow = row;
      scol = kc;
    } else {
      const int krow = c >> 6, rc = (c & 63) * 2;
      const int64_t gk = k0 + krow, gr = r0 + rc;
      vec_idx = gk < kend ? gk : 0;
      off = gr;
      nvalid = gk < kend ? (int)max((int64_t)0, min((int64_t)2, rlim - gr)) : 0;
      srow = krow;
      scol = rc;
    }
    double* dst = KMAJOR ? s + srow * LDK + scol : s + srow * LDM + scol;
    const double* vp = op.vec(vec_idx);
    if (VEC) {
      const double* src = nvalid ? vp + off : vp;
      cp_async_16(dst, src, nvalid * 8);
    } else {
      cp_async_8(dst, nvalid >= 1 ? vp + off : vp, nvalid >= 1 ? 8 : 0);
      cp_async_8(dst + 1, nvalid >= 2 ? vp + off + 1 : vp, nvalid >= 2 ? 8 : 0);
    }
  }
}

// One BK-deep k tile of the 128x128 CTA tile: this warp's 64x32 sub-tile, DMMA m8n8k4.
template <bool AK, bool BKM>
__device__ __forceinline__ void mma_ktile(const double* as, const double* bs, double (&acc)[8][4][2], int wm, int wn,
                                          int g, int t) {
  using L = Layout<AK, BKM>;
  if (L::MODEP) {
#pragma unroll
    for (int sp = 0; sp < 2; ++sp) {
      double2 af[8], bf[4];
#pragma unroll
      for (int i = 0; i < 8; ++i)
        af[i] = *reinterpret_cast<const double2*>(as + (wm * 64 + i * 8 + g) * L::LDK + 4 * t + 2 * sp);
#pragma unroll
      for (int j = 0; j < 4; ++j)
        bf[j] = *reinterpret_cast<const double2*>(bs + (wn * 32 + j * 8 + g) * L::LDK + 4 * t + 2 * sp);
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          dmma_8x8x4(acc[i][j], af[i].x, bf[j].x);
        }
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          dmma_8x8x4(acc[i][j], af[i].y, bf[j].y);
        }
    }
  } else {
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      double af[8], bf[4];
      const int kk = 4 * s + t;
      if (AK) {
#pragma unroll
        for (int i = 0; i < 8; ++i) af[i] = as[(wm * 64 + i * 8 + g) * L::LDK + kk];
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          double2 v = *reinterpret_cast<const double2*>(as + kk * LDM + wm * 64 + g * 8 + 2 * q);
          af[2 * q] = v.x;
          af[2 * q + 1] = v.y;
        }
      }
      if (BKM) {
#pragma unroll
        for (int j = 0; j < 4; ++j) bf[j] = bs[(wn * 32 + j * 8 + g) * L::LDK + kk];
      } else {
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          double2 v = *reinterpret_cast<const double2*>(bs + kk * LDM + wn * 32 + g * 4 + 2 * q);
          bf[2 * q] = v.x;
          bf[2 * q + 1] = v.y;
        }
      }
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma_8x8x4(acc[i][j], af[i], bf[j]);
    }
  }
}

// Epilogue: split-K partial tile, or alpha/beta/row-col scale/divide + symmetric mirror into C.
template <bool AK, bool BKM, int NJ = 4>
__device__ __forceinline__ void epilogue(const Params& p, const double (&acc)[8][NJ][2], int64_t tile, int z, int64_t m0,
                                         int64_t n0, int wm, int wn, int g, int t) {
  if (p.splits > 1) {
    double* out = p.partial + ((int64_t)z * p.ntiles + tile) * (BM * (8 * NJ * 4));
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < NJ; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int ml = wm * 64 + (AK ? i * 8 + g : g * 8 + i);
          const int nl = wn * (8 * NJ) + (BKM ? j * 8 + 2 * t + e : (2 * t + e) * 4 + j);
          out[nl * BM + ml] = acc[i][j][e];
        }
    return;
  }
  if constexpr (!AK) {
    // M-major A: a thread's 8 row fragments are 8 CONSECUTIVE rows of one output column -- stored as
    // four 16-byte words instead of eight scattered 8-byte ones (same arithmetic, same order)
    // (also the read-modify-write of a symmetric update on a tile strictly above the diagonal, where
    // every entry is wanted; sym == 1 adds the mirrored entries as single words)
    const bool whole = !p.sym || m0 + BM <= n0;
    if (whole && (p.ldc & 1) == 0 && (reinterpret_cast<uintptr_t>(p.C) & 15) == 0) {
      const int64_t mb = m0 + wm * 64 + g * 8;
      if constexpr (!BKM && NJ == 4) {
        // symmetric update with a mirror and an N-major B (the tridiagonalisation's rank-2k updates): a
        // thread's fragments j, j + 1 are CONSECUTIVE columns, so the mirrored entries of one row go
        // out as 16-byte words too
        if (p.sym == 1 && !p.row_scale && !p.col_scale && !p.col_div) {
#pragma unroll
          for (int e = 0; e < 2; ++e)
#pragma unroll
            for (int jp = 0; jp < 4; jp += 2) {
              const int64_t na = n0 + wn * 32 + (2 * t + e) * 4 + jp;
              if (na >= p.N) continue;
              const bool hb = na + 1 < p.N;
              double* da = p.C + na * p.ldc + mb;
              double* db = da + p.ldc;
#pragma unroll
              for (int i = 0; i < 8; i += 2) {
                if (mb + i >= p.M) break;
                const bool h1 = mb + i + 1 < p.M;
                double a0 = p.alpha * acc[i][jp][e], a1 = p.alpha * acc[i + 1][jp][e];
                double b0 = p.alpha * acc[i][jp + 1][e], b1 = p.alpha * acc[i + 1][jp + 1][e];
                if (p.beta != 0.0) {
                  if (h1) {
                    const double2 oa = *reinterpret_cast<const double2*>(da + i);
                    a0 += p.beta * oa.x;
                    a1 += p.beta * oa.y;
                    if (hb) {
                      const double2 ob = *reinterpret_cast<const double2*>(db + i);
                      b0 += p.beta * ob.x;
                      b1 += p.beta * ob.y;
                    }
                  } else {
                    a0 += p.beta * da[i];
                    if (hb) b0 += p.beta * db[i];
                  }
                }
                if (h1) {
                  *reinterpret_cast<double2*>(da + i) = make_double2(a0, a1);
                  if (hb) *reinterpret_cast<double2*>(db + i) = make_double2(b0, b1);
                } else {
                  da[i] = a0;
                  if (hb) db[i] = b0;
                }
                double* r0 = p.C + (mb + i) * p.ldc + na;  // mirrored: row mb + i, columns na, na + 1
                if (hb) {
                  *reinterpret_cast<double2*>(r0) = make_double2(a0, b0);
                  if (h1) *reinterpret_cast<double2*>(r0 + p.ldc) = make_double2(a1, b1);
                } else {
                  r0[0] = a0;
                  if (h1) r0[p.ldc] = a1;
                }
              }
            }
          return;
        }
      }
#pragma unroll
      for (int j = 0; j < NJ; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int64_t n = n0 + wn * (8 * NJ) + (BKM ? j * 8 + 2 * t + e : (2 * t + e) * 4 + j);
          if (n >= p.N) continue;
          const bool cs = p.col_scale != nullptr, cd = p.col_div != nullptr;
          const double csv = cs ? p.col_scale[n] : 1.0, cdv = cd ? p.col_div[n] : 1.0;
          double* dst = p.C + n * p.ldc + mb;
#pragma unroll
          for (int i = 0; i < 8; i += 2) {
            if (mb + i >= p.M) break;
            double v0 = p.alpha * acc[i][j][e], v1 = p.alpha * acc[i + 1][j][e];
            if (p.beta != 0.0) {
              if (mb + i + 1 < p.M) {
                const double2 old = *reinterpret_cast<const double2*>(dst + i);
                v0 += p.beta * old.x;
                v1 += p.beta * old.y;
              } else {
                v0 += p.beta * dst[i];
              }
            }
            if (p.row_scale) {
              v0 *= p.row_scale[mb + i];
              if (mb + i + 1 < p.M) v1 *= p.row_scale[mb + i + 1];
            }
            if (cs) {
              v0 *= csv;
              v1 *= csv;
            }
            if (cd) {
              v0 /= cdv;
              v1 /= cdv;
            }
            if (mb + i + 1 < p.M)
              *reinterpret_cast<double2*>(dst + i) = make_double2(v0, v1);
            else
              dst[i] = v0;
            if (p.sym == 1) {
              p.C[(mb + i) * p.ldc + n] = v0;
              if (mb + i + 1 < p.M) p.C[(mb + i + 1) * p.ldc + n] = v1;
            }
          }
        }
      return;
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < NJ; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int64_t m = m0 + wm * 64 + (AK ? i * 8 + g : g * 8 + i);
        const int64_t n = n0 + wn * (8 * NJ) + (BKM ? j * 8 + 2 * t + e : (2 * t + e) * 4 + j);
        if (m >= p.M || n >= p.N) continue;
        if (p.sym && m > n) continue;
        double v = p.alpha * acc[i][j][e];
        if (p.beta != 0.0) v += p.beta * p.C[n * p.ldc + m];
        if (p.row_scale) v *= p.row_scale[m];
        if (p.col_scale) v *= p.col_scale[n];
        if (p.col_div) v /= p.col_div[n];
        p.C[n * p.ldc + m] = v;
        if (p.sym == 1 && m != n) p.C[m * p.ldc + n] = v;
      }
}

template <bool AK, bool BKM, bool VEC>
__global__ void __launch_bounds__(THREADS, 1) gemm_kernel(Params p) {
  using L = Layout<AK, BKM>;
  extern __shared__ __align__(16) double smem[];
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp & 1, wn = warp >> 1;

  const int64_t tile = blockIdx.x;
  const int z = blockIdx.z;
  int bi, bj;
  tile_coords(p, tile, bi, bj);
  const int64_t m0 = (int64_t)bi * BM, n0 = (int64_t)bj * BN;

  const int64_t kbeg = (int64_t)z * p.kspan;
  int64_t kend = min(p.K, kbeg + p.kspan);
  if (p.b_upper) kend = min(kend, n0 + BN);
  const int nk = kend > kbeg ? (int)((kend - kbeg + BK - 1) / BK) : 0;

  double acc[8][4][2];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  auto stage_a = [&](int s) { return smem + s * L::STAGE_ELEMS; };
  auto stage_b = [&](int s) { return smem + s * L::STAGE_ELEMS + L::A_ELEMS; };
  auto load_stage = [&](int s, int64_t k0) {
    load_operand<AK, VEC, L::LDK>(stage_a(s), p.A, m0, p.M, k0, kend, tid);
    load_operand<BKM, VEC, L::LDK>(stage_b(s), p.B, n0, p.N, k0, kend, tid);
  };

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nk) load_stage(s, kbeg + (int64_t)s * BK);
    cp_async_commit();
  }

  for (int kt = 0; kt < nk; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    const int nxt = kt + STAGES - 1;
    if (nxt < nk) load_stage(nxt % STAGES, kbeg + (int64_t)nxt * BK);
    cp_async_commit();

    mma_ktile<AK, BKM>(stage_a(kt % STAGES), stage_b(kt % STAGES), acc, wm, wn, g, t);
  }
  cp_async_wait<0>();

  epilogue<AK, BKM>(p, acc, tile, z, m0, n0, wm, wn, g, t);
}

// ---------------------------------------------------------------------------------------------
// TMA-staged variant (plain strided operands, 16-byte aligned): warp 8 is the producer and
// moves every operand tile with tensor TMA (cp.async.bulk.tensor.2d, SWIZZLE_128B, hardware
// zero fill outside the matrix); warps 0-7 consume.  Each of the TSTAGES ring slots has a
// "full" mbarrier (producer arrive + transaction bytes) and an "empty" mbarrier (one arrive
// per consumer warp): no CTA-wide barrier and no load instruction in the main loop of the
// consumer warps, and no edge code at all (partial tiles in M, N and K are zero-filled by the
// TMA unit).
//   K-major operand : one box {16 k, 128 vectors}: row r = 128 B, 16-byte chunk c of row r
//                     stored at chunk c ^ (r & 7)
//   M-major operand : 8 boxes {16 m, 16 k}: box b holds m in [16b, 16b+16), k-row kk = 128 B,
//                     chunk c of row kk stored at c ^ (kk & 7)
// With these swizzles the fragment loads of both the 128-bit (both K-major) and the M-major
// paths are bank-conflict free.
constexpr int TSTAGES = 6, TTHREADS = 384;  // 2 consumer warpgroups + 1 producer warpgroup
constexpr int TILE_BYTES = BM * BK * 8;     // 16 KB per operand per stage

struct TmaParams {
  CUtensorMap ta, tb;  // 64-byte aligned (CUtensorMap is declared alignas(64))
  Params p;
};

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::
          "r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

// byte offset of element (row, k) in a K-major tile / (m, k) in an M-major tile
__device__ __forceinline__ int kmaj_off(int row, int k) {
  return row * 128 + ((((k >> 1) ^ row) & 7) << 4) + (k & 1) * 8;
}
__device__ __forceinline__ int mmaj_off(int m, int k) {
  return (m >> 4) * 2048 + k * 128 + (((((m & 15) >> 1) ^ k) & 7) << 4) + (m & 1) * 8;
}

template <bool AK, bool BKM, int NJ>
__device__ __forceinline__ void mma_ktile_sw(const char* as, const char* bs, double (&acc)[8][NJ][2], int wm, int wn,
                                             int g, int t) {
  static_assert(BKM || NJ == 4, "narrow n tiles need a K-major B operand");
  if constexpr (AK && BKM) {
#pragma unroll
    for (int sp = 0; sp < 2; ++sp) {
      double2 af[8], bf[NJ];
      const int kk = 4 * t + 2 * sp;
#pragma unroll
      for (int i = 0; i < 8; ++i) af[i] = *reinterpret_cast<const double2*>(as + kmaj_off(wm * 64 + i * 8 + g, kk));
#pragma unroll
      for (int j = 0; j < NJ; ++j) bf[j] = *reinterpret_cast<const double2*>(bs + kmaj_off(wn * (8 * NJ) + j * 8 + g, kk));
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < NJ; ++j) dmma_8x8x4(acc[i][j], af[i].x, bf[j].x);
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < NJ; ++j) dmma_8x8x4(acc[i][j], af[i].y, bf[j].y);
    }
  } else {
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      double af[8], bf[NJ];
      const int kk = 4 * s + t;
      if constexpr (AK) {
#pragma unroll
        for (int i = 0; i < 8; ++i) af[i] = *reinterpret_cast<const double*>(as + kmaj_off(wm * 64 + i * 8 + g, kk));
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const double2 v = *reinterpret_cast<const double2*>(as + mmaj_off(wm * 64 + g * 8 + 2 * q, kk));
          af[2 * q] = v.x;
          af[2 * q + 1] = v.y;
        }
      }
      if constexpr (BKM) {
#pragma unroll
        for (int j = 0; j < NJ; ++j) bf[j] = *reinterpret_cast<const double*>(bs + kmaj_off(wn * (8 * NJ) + j * 8 + g, kk));
      } else {
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const double2 v = *reinterpret_cast<const double2*>(bs + mmaj_off(wn * 32 + g * 4 + 2 * q, kk));
          bf[2 * q] = v.x;
          bf[2 * q + 1] = v.y;
        }
      }
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < NJ; ++j) dmma_8x8x4(acc[i][j], af[i], bf[j]);
    }
  }
}


// ---------------------------------------------------------------------------------------------
// Diagonal tile of a symmetric product (both operands K-major, 128-wide tile): only the entries
// with row <= column are wanted, i.e. 136 of the tile's 256 8x8 accumulator fragments.  The
// regular 2 x 4 warp grid would leave two warps idle and six at full load, so the fragments are
// re-dealt: the tile is cut into strips of 16 columns; a strip of the full upper-right 64 x 64
// block takes 8 row fragments, strip s of a diagonal 64 x 64 block 2 (s + 1).  Every consumer
// warp gets up to two strips (18 +- 2 fragments of 8 x 16) such that the two warps sharing an
// SM sub-partition (w, w + 4) carry 36 fragments together instead of 64: the tile costs ~56 % of
// a full one.  Each output entry is still one accumulator summed over k in the same order, so
// the result equals the regular path's bit for bit.
struct DiagTask {
  int rb[2], lim[2], cb[2];  // per strip: first row, row fragments (0 = none), first column
};

__device__ __forceinline__ DiagTask diag_task(int warp) {
  DiagTask k;
  k.rb[1] = 0;
  k.lim[1] = 0;
  k.cb[1] = 0;
  switch (warp) {
    case 0: k.rb[0] = 0, k.lim[0] = 8, k.cb[0] = 64, k.rb[1] = 0, k.lim[1] = 2, k.cb[1] = 0; break;
    case 1: k.rb[0] = 0, k.lim[0] = 8, k.cb[0] = 80, k.rb[1] = 64, k.lim[1] = 2, k.cb[1] = 64; break;
    case 2: k.rb[0] = 0, k.lim[0] = 8, k.cb[0] = 96; break;
    case 3: k.rb[0] = 0, k.lim[0] = 8, k.cb[0] = 112; break;
    case 4: k.rb[0] = 0, k.lim[0] = 8, k.cb[0] = 48; break;
    case 5: k.rb[0] = 64, k.lim[0] = 8, k.cb[0] = 112; break;
    case 6: k.rb[0] = 0, k.lim[0] = 4, k.cb[0] = 16, k.rb[1] = 0, k.lim[1] = 6, k.cb[1] = 32; break;
    default: k.rb[0] = 64, k.lim[0] = 4, k.cb[0] = 80, k.rb[1] = 64, k.lim[1] = 6, k.cb[1] = 96; break;
  }
  return k;
}

__device__ __forceinline__ void mma_ktile_diag(const char* as, const char* bs, double (&acc)[8][4][2],
                                               const DiagTask& tk, int g, int t) {
#pragma unroll
  for (int sp = 0; sp < 2; ++sp) {
    const int kk = 4 * t + 2 * sp;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int lim = tk.lim[h];
      if (lim == 0) continue;  // warp-uniform
      double2 af[8], bf[2];
#pragma unroll
      for (int i = 0; i < 8; ++i)
        if (i < lim) af[i] = *reinterpret_cast<const double2*>(as + kmaj_off(tk.rb[h] + i * 8 + g, kk));
#pragma unroll
      for (int j = 0; j < 2; ++j) bf[j] = *reinterpret_cast<const double2*>(bs + kmaj_off(tk.cb[h] + j * 8 + g, kk));
#pragma unroll
      for (int i = 0; i < 8; ++i)
        if (i < lim) {
#pragma unroll
          for (int j = 0; j < 2; ++j) dmma_8x8x4(acc[i][2 * h + j], af[i].x, bf[j].x);
        }
#pragma unroll
      for (int i = 0; i < 8; ++i)
        if (i < lim) {
#pragma unroll
          for (int j = 0; j < 2; ++j) dmma_8x8x4(acc[i][2 * h + j], af[i].y, bf[j].y);
        }
    }
  }
}

// epilogue of a diagonal tile (same arithmetic as `epilogue`, the strip mapping of DiagTask)
__device__ __forceinline__ void epilogue_diag(const Params& p, const double (&acc)[8][4][2], int64_t tile, int z,
                                              int64_t m0, int64_t n0, const DiagTask& tk, int g, int t) {
  double* out = p.splits > 1 ? p.partial + ((int64_t)z * p.ntiles + tile) * (BM * BN) : nullptr;
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int h = j >> 1;
      if (i >= tk.lim[h]) continue;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int ml = tk.rb[h] + i * 8 + g;
        const int nl = tk.cb[h] + (j & 1) * 8 + 2 * t + e;
        if (out) {
          out[nl * BM + ml] = acc[i][j][e];
          continue;
        }
        const int64_t m = m0 + ml, n = n0 + nl;
        if (m >= p.M || n >= p.N || m > n) continue;
        double v = p.alpha * acc[i][j][e];
        if (p.beta != 0.0) v += p.beta * p.C[n * p.ldc + m];
        if (p.row_scale) v *= p.row_scale[m];
        if (p.col_scale) v *= p.col_scale[n];
        if (p.col_div) v /= p.col_div[n];
        p.C[n * p.ldc + m] = v;
        if (p.sym == 1 && m != n) p.C[m * p.ldc + n] = v;
      }
    }
}

template <bool AK, bool BKM, int NJ>
__global__ void __launch_bounds__(TTHREADS, 1) gemm_tma_kernel(const __grid_constant__ TmaParams tp) {
  const Params& p = tp.p;
  extern __shared__ __align__(16) double smem[];
  __shared__ __align__(8) uint64_t full_bar[TSTAGES], empty_bar[TSTAGES];
  // 128B-swizzled TMA destinations must be 1024-byte aligned
  char* sbase = reinterpret_cast<char*>(smem) + ((1024u - (smem_u32(smem) & 1023u)) & 1023u);
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;

  int64_t tile = blockIdx.x;
  int z = blockIdx.z;
  if (p.sym && p.splits > 1) {
    // split symmetric output: block order = all splits of the (full-cost) off-diagonal tiles first,
    // then the diagonal tiles -- longest jobs first, and neighbouring CTAs still share a k range
    const int64_t T = p.tiles_m, n_off = T * (T - 1) / 2;
    const int64_t lin = blockIdx.x + p.ntiles * (int64_t)blockIdx.z, cut = n_off * p.splits;
    if (lin < cut) {
      z = (int)(lin / n_off);
      tile = lin % n_off;
    } else {
      z = (int)((lin - cut) / T);
      tile = n_off + (lin - cut) % T;
    }
  }
  int bi, bj;
  tile_coords(p, tile, bi, bj);
  constexpr int TBN = 32 * NJ;                 // tile width in n (4 n-warps x NJ fragments of 8)
  constexpr int B_BYTES = TBN * BK * 8;
  constexpr int STAGE_BYTES = TILE_BYTES + B_BYTES;
  const int64_t m0 = (int64_t)bi * BM, n0 = (int64_t)bj * TBN;
  const int64_t kbeg = (int64_t)z * p.kspan;
  int64_t kend = min(p.K, kbeg + p.kspan);
  if (p.b_upper) kend = min(kend, n0 + TBN);
  const int nk = kend > kbeg ? (int)((kend - kbeg + BK - 1) / BK) : 0;

  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < TSTAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 8);
    }
    mbar_fence_init();
  }
  __syncthreads();

  if (warp >= 8) {
    // ------------------------------------------------------------------ producer
    // the producer warpgroup hands its registers to the consumers (setmaxnreg: per-SMSP
    // register files hold 2 consumer warps at 224 + 1 producer warp at 56)
    asm volatile("setmaxnreg.dec.sync.aligned.u32 56;\n" ::: "memory");
    if (warp != 8 || lane != 0) return;
    for (int kt = 0; kt < nk; ++kt) {
      const int s = kt % TSTAGES;
      if (kt >= TSTAGES) mbar_wait(&empty_bar[s], ((kt / TSTAGES) - 1) & 1);
      const int k0 = (int)(kbeg + (int64_t)kt * BK);
      char* sa = sbase + s * STAGE_BYTES;
      char* sb = sa + TILE_BYTES;
      mbar_arrive_expect_tx(&full_bar[s], STAGE_BYTES);
      if (AK) {
        tma_load_2d(sa, &tp.ta, k0, (int)m0, &full_bar[s]);
      } else {
#pragma unroll
        for (int b = 0; b < BM / 16; ++b) tma_load_2d(sa + b * 2048, &tp.ta, (int)m0 + 16 * b, k0, &full_bar[s]);
      }
      if (BKM) {
        tma_load_2d(sb, &tp.tb, k0, (int)n0, &full_bar[s]);
      } else {
#pragma unroll
        for (int b = 0; b < TBN / 16; ++b) tma_load_2d(sb + b * 2048, &tp.tb, (int)n0 + 16 * b, k0, &full_bar[s]);
      }
    }
    return;
  }

  // -------------------------------------------------------------------- consumers (warps 0-7)
  asm volatile("setmaxnreg.inc.sync.aligned.u32 224;\n" ::: "memory");
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp & 1, wn = warp >> 1;
  double acc[8][NJ][2];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < NJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  if constexpr (AK && BKM && NJ == 4) {
    if (p.sym && bi == bj) {
      const DiagTask tk = diag_task(warp);
      for (int kt = 0; kt < nk; ++kt) {
        const int s = kt % TSTAGES;
        mbar_wait(&full_bar[s], (kt / TSTAGES) & 1);
        const char* sa = sbase + s * STAGE_BYTES;
        mma_ktile_diag(sa, sa + TILE_BYTES, acc, tk, g, t);
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty_bar[s]);
      }
      epilogue_diag(p, acc, tile, z, m0, n0, tk, g, t);
      return;
    }
  }
  for (int kt = 0; kt < nk; ++kt) {
    const int s = kt % TSTAGES;
    mbar_wait(&full_bar[s], (kt / TSTAGES) & 1);
    const char* sa = sbase + s * STAGE_BYTES;
    mma_ktile_sw<AK, BKM, NJ>(sa, sa + TILE_BYTES, acc, wm, wn, g, t);
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty_bar[s]);
  }
  epilogue<AK, BKM, NJ>(p, acc, tile, z, m0, n0, wm, wn, g, t);
}

// Fixed-order split-K reduction + epilogue.  One thread per tile element.
__global__ void splitk_reduce(Params p) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int bn = p.bn;
  const int64_t tile = idx / (BM * bn);
  if (tile >= p.ntiles) return;
  const int e = (int)(idx % (BM * bn));
  const int nl = e / BM, ml = e % BM;
  int bi, bj;
  tile_coords(p, tile, bi, bj);
  const int64_t m = (int64_t)bi * BM + ml, n = (int64_t)bj * bn + nl;
  if (m >= p.M || n >= p.N) return;
  if (p.sym && m > n) return;
  double s = 0.0;
  for (int z = 0; z < p.splits; ++z) s += p.partial[((int64_t)z * p.ntiles + tile) * (BM * bn) + e];
  double v = p.alpha * s;
  if (p.beta != 0.0) v += p.beta * p.C[n * p.ldc + m];
  if (p.row_scale) v *= p.row_scale[m];
  if (p.col_scale) v *= p.col_scale[n];
  if (p.col_div) v /= p.col_div[n];
  p.C[n * p.ldc + m] = v;
  if (p.sym == 1 && m != n) p.C[m * p.ldc + n] = v;
}

struct Plan {
  int tiles_m, tiles_n;
  int64_t ntiles;
  int splits;
  int64_t kspan;
  size_t ws_bytes;
  int bn;
};

// Tile width in n for an output of N columns: the width of {128, 96, 64} that pads N the least
// (ties go to the wider tile).  A chain merge reconstructs N ~ 78-95 (config 2) or ~ 287
// (config 4) columns: 96-wide tiles are 81-99 % full where 128-wide ones are 61-75 % full; a
// config-3 leaf's 300 modes take five 64-wide tiles (320) instead of three 128-wide ones (384).
// Depends on N only, so the plan -- and with it every bit of the result -- is shape-determined.
int narrow_bn(int64_t N) {
  int best = BN;
  int64_t pad = ceil_div(N, (int64_t)BN) * BN;
  for (int bn : {96, 64}) {
    const int64_t pd = ceil_div(N, (int64_t)bn) * bn;
    if (pd < pad) {
      pad = pd;
      best = bn;
    }
  }
  return best;
}

// Split count of a small symmetric product whose diagonal tiles take the re-dealt path
// (mma_ktile_diag, ~56 % of a full tile): the CTAs of a launch are handed to the SMs in block order
// (all splits of the off-diagonal tiles, then the diagonal ones; one CTA per SM at a time), so the
// launch ends when the slowest SM does.  Among the split counts around the default one, take the
// one with the shortest modelled makespan (cost of a CTA in 16-deep k steps + 2 for its prologue
// and epilogue).  A function of the shape only -- 148 is a constant here, not a device query.
int diag_aware_splits(int T, int64_t K, int64_t base, int64_t min_k) {
  static std::mutex mu;
  static std::map<std::tuple<int, int64_t, int64_t>, int> cache;
  const auto key = std::make_tuple(T, K, base);
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
  }
  const int P = 148;
  const int64_t n_off = (int64_t)T * (T - 1) / 2;
  const int64_t lo = std::max<int64_t>(1, base / 2), hi = std::max<int64_t>(1, std::min<int64_t>(2 * base, K / min_k));
  int best = (int)base;
  double best_span = 0.0;
  std::vector<double> heap;
  for (int64_t s0 = lo; s0 <= hi; ++s0) {
    const int64_t kspan = ceil_div(ceil_div(K, s0), BK) * BK;
    const int64_t sp = std::max<int64_t>(1, ceil_div(K, kspan));
    if (sp != s0) continue;  // not a distinct plan
    const double n = (double)(kspan / BK);
    const double c_full = n + 2.0, c_diag = 0.5625 * n + 2.0;
    heap.assign(P, 0.0);  // min-heap of the SMs' free times
    auto cmp = [](double a, double b) { return a > b; };
    double span = 0.0;
    for (int64_t c = 0; c < (n_off + T) * sp; ++c) {  // launch order: every full tile, then the diagonal ones
      std::pop_heap(heap.begin(), heap.end(), cmp);
      heap.back() += c < n_off * sp ? c_full : c_diag;
      span = std::max(span, heap.back());
      std::push_heap(heap.begin(), heap.end(), cmp);
    }
    if (best_span == 0.0 || span < best_span * (1.0 - 1e-9)) {
      best_span = span;
      best = (int)sp;
    }
  }
  std::lock_guard<std::mutex> lk(mu);
  cache[key] = best;
  return best;
}

// Split count (1..4) of a LARGE symmetric product whose tile count leaves the last wave mostly empty
// (666 tiles on 148 SMs = 4.5 waves cost 5): the same makespan model as diag_aware_splits over the
// kernel's block order (all splits of the off-diagonal tiles, then the diagonal ones), plus the
// second-pass reduction of the partial tiles.  Only used where the caller allows it
// (gemm_set_wavesplit: the orthonormality SYRKs); a split is taken only for a gain above 3 %.
int wave_splits(int T, int64_t K) {
  static std::mutex mu;
  static std::map<std::pair<int, int64_t>, int> cache;
  const auto key = std::make_pair(T, K);
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
  }
  const int P = 148;
  const int64_t n_off = (int64_t)T * (T - 1) / 2;
  int best = 1;
  double best_span = 0.0, span1 = 0.0;
  std::vector<double> heap;
  for (int64_t s0 = 1; s0 <= 4 && K / s0 >= 512; ++s0) {
    const int64_t kspan = ceil_div(ceil_div(K, s0), BK) * BK;
    const int64_t sp = std::max<int64_t>(1, ceil_div(K, kspan));
    if (sp != s0) continue;
    const double n = (double)(kspan / BK);
    const double c_full = n + 2.0, c_diag = 0.5625 * n + 2.0;
    heap.assign(P, 0.0);
    auto cmp = [](double a, double b) { return a > b; };
    double span = 0.0;
    for (int64_t c = 0; c < (n_off + T) * sp; ++c) {
      std::pop_heap(heap.begin(), heap.end(), cmp);
      heap.back() += c < n_off * sp ? c_full : c_diag;
      span = std::max(span, heap.back());
      std::push_heap(heap.begin(), heap.end(), cmp);
    }
    if (sp > 1) span += 0.025 * (double)sp * (double)(n_off + T);  // partial tiles written and re-read
    if (sp == 1) span1 = span;
    if (best_span == 0.0 || span < best_span) {
      best_span = span;
      best = (int)sp;
    }
  }
  if (best > 1 && !(best_span < 0.97 * span1)) best = 1;
  std::lock_guard<std::mutex> lk(mu);
  cache[key] = best;
  return best;
}

Plan make_plan(int64_t M, int64_t N, int64_t K, int sym, int b_upper, int bn = BN, bool diag_aware = false,
               bool wave_split = false) {
  Plan pl;
  pl.bn = bn;
  pl.tiles_m = (int)ceil_div(M, BM);
  pl.tiles_n = (int)ceil_div(N, (int64_t)bn);
  pl.ntiles = sym ? (int64_t)pl.tiles_m * (pl.tiles_m + 1) / 2 : (int64_t)pl.tiles_m * pl.tiles_n;
  // Split-K only when the output alone cannot fill the chip.  Depends on the
  // shape only (never on the device count) so results are reproducible.
  const int64_t target = 2 * 148;
  int64_t splits = 1;
  if (!b_upper && pl.ntiles < target) {
    splits = target / std::max<int64_t>(pl.ntiles, 1);
    // >= 512 k per split; a GEMM of at most 16 output tiles (the deep levels of chol_inv_run, small
    // node products) splits down to 64 k: one 128x128 tile contracts 16 k per ~2 us on its SM, so
    // a single-tile GEMM with K = 256 was ~35 us of one SM's DMMA pipe
    const int64_t min_k = pl.ntiles <= 16 ? 64 : 512;
    splits = std::min<int64_t>(splits, std::max<int64_t>(K / min_k, 1));
    splits = std::min<int64_t>(splits, target);  // a one-tile output over a long K (a chain merge's drift SYRK) spreads over the whole chip
    splits = std::max<int64_t>(splits, 1);
    if (diag_aware && sym && bn == BN && splits > 1 && pl.tiles_m >= 2 && pl.tiles_m <= GN)
      splits = diag_aware_splits(pl.tiles_m, K, splits, min_k);
  } else if (wave_split && diag_aware && sym && !b_upper && bn == BN) {
    splits = wave_splits(pl.tiles_m, K);
  }
  pl.kspan = ceil_div(ceil_div(K, splits), BK) * BK;
  splits = std::max<int64_t>(1, ceil_div(K, std::max<int64_t>(pl.kspan, 1)));
  pl.splits = (int)splits;
  pl.ws_bytes = pl.splits > 1 ? (size_t)pl.splits * pl.ntiles * BM * bn * sizeof(double) : 0;
  return pl;
}

template <bool AK, bool BKM, bool VEC>
int launch_t(const Params& p, cudaStream_t st) {
  using L = Layout<AK, BKM>;
  static std::atomic<unsigned long long> configured{0};
  int rc0 = once_per_device(configured, []() -> int {
    HP_CHECK_CUDA(cudaFuncSetAttribute(gemm_kernel<AK, BKM, VEC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       L::SMEM_BYTES));
    return (int)HP_OK;
  });
  if (rc0 != HP_OK) return rc0;
  dim3 grid((unsigned)p.ntiles, 1, (unsigned)p.splits);
  gemm_kernel<AK, BKM, VEC><<<grid, THREADS, L::SMEM_BYTES, st>>>(p);
  HP_CHECK_LAUNCH("gemm_kernel");
  return HP_OK;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda link)
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }();
  return fn;
}

// 2-d map over `outer` vectors of `inner` contiguous float64 (vector stride ld elements)
bool encode_map(CUtensorMap* map, const double* base, int64_t inner, int64_t outer, int64_t ld, int box_inner,
                int box_outer) {
  auto enc = tensor_map_encoder();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)std::max<int64_t>(inner, 1), (cuuint64_t)std::max<int64_t>(outer, 1)};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 8)};
  cuuint32_t box[2] = {(cuuint32_t)box_inner, (cuuint32_t)box_outer};
  cuuint32_t estr[2] = {1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <bool AK, bool BKM, int NJ = 4>
int launch_tma(const Params& p, cudaStream_t st, bool& done) {
  constexpr int TBN = 32 * NJ;
  constexpr int SMEM = TSTAGES * (TILE_BYTES + TBN * BK * 8) + 1024;
  done = false;
  static std::atomic<unsigned long long> configured{0};
  TmaParams tp;
  tp.p = p;
  // K-major: inner = K (contiguous k of each vector), outer = M / N vectors, box {16, 128}
  // M-major: inner = M / N (contiguous rows of each k-vector), outer = K, box {16, 16}
  const bool ok_a = AK ? encode_map(&tp.ta, p.A.base, p.K, p.M, p.A.ld, BK, BM)
                       : encode_map(&tp.ta, p.A.base, p.M, p.K, p.A.ld, 16, BK);
  const bool ok_b = BKM ? encode_map(&tp.tb, p.B.base, p.K, p.N, p.B.ld, BK, TBN)
                        : encode_map(&tp.tb, p.B.base, p.N, p.K, p.B.ld, 16, BK);
  if (!ok_a || !ok_b) return HP_OK;  // not encodable: caller uses the cp.async kernel
  const int rc0 = once_per_device(configured, []() -> int {
    HP_CHECK_CUDA(cudaFuncSetAttribute(gemm_tma_kernel<AK, BKM, NJ>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       SMEM));
    return (int)HP_OK;
  });
  if (rc0 != HP_OK) return rc0;
  dim3 grid((unsigned)p.ntiles, 1, (unsigned)p.splits);
  gemm_tma_kernel<AK, BKM, NJ><<<grid, TTHREADS, SMEM, st>>>(tp);
  HP_CHECK_LAUNCH("gemm_tma_kernel");
  done = true;
  return HP_OK;
}

}  // namespace gemm

// Calling-thread switch for the next gemm_run calls: never split the contraction and keep the 128-wide
// tiles, whatever the output size -- every output entry is then summed over all K by one CTA in the
// order of a large (unsplit) launch, so a block of a big Gramian computed on its own equals the
// corresponding block of the monolithic launch bit for bit (hp_gram_pair).
static thread_local bool tl_nosplit = false;
void gemm_set_nosplit(bool on) { tl_nosplit = on; }
// Calling-thread switch: the next symmetric gemm_run calls may split a LARGE output's contraction to
// even out the last wave (gemm::wave_splits).  Off for the node Gramians, whose pair blocks must equal
// the monolithic launch bit for bit; on for the orthonormality SYRKs (drift, CholQR).
static thread_local bool tl_wavesplit = false;
void gemm_set_wavesplit(bool on) { tl_wavesplit = on; }
bool gemm_plan_is_single_split(int64_t M, int64_t N, int64_t K, int sym) {
  return gemm::make_plan(M, N, K, sym, 0).splits == 1;
}

// Host entry used by the C-ABI and by the other modules.
int gemm_run(bool a_kmajor, bool b_kmajor, int64_t M, int64_t N, int64_t K, VecSet A, VecSet B, bool aligned16,
             double alpha, double beta, double* C, int64_t ldc, const double* row_scale, const double* col_scale,
             const double* col_div, int sym, int b_upper, void* ws, size_t ws_bytes, cudaStream_t st) {
  using namespace gemm;
  HP_REQUIRE(M >= 0 && N >= 0 && K >= 0, "gemm: negative dimension");
  HP_REQUIRE(!sym || M == N, "gemm: symmetric output needs M == N");
  if (M == 0 || N == 0) return HP_OK;
  Params p{};
  p.M = M;
  p.N = N;
  p.K = K;
  p.A = A;
  p.B = B;
  p.C = C;
  p.ldc = ldc;
  p.alpha = alpha;
  p.beta = beta;
  p.row_scale = row_scale;
  p.col_scale = col_scale;
  p.col_div = col_div;
  p.sym = sym;
  p.b_upper = b_upper;
  auto apply_plan = [&](const Plan& pl) {
    p.bn = pl.bn;
    p.tiles_m = pl.tiles_m;
    p.tiles_n = pl.tiles_n;
    p.ntiles = pl.ntiles;
    p.splits = pl.splits;
    p.kspan = pl.kspan;
    p.partial = nullptr;
    if (pl.splits > 1) {
      if (ws_bytes < pl.ws_bytes) {
        // not enough workspace: fall back to a single split (same arithmetic class, one more wave)
        p.splits = 1;
        p.kspan = ceil_div(std::max<int64_t>(K, 1), BK) * BK;
      } else {
        p.partial = static_cast<double*>(ws);
      }
    }
  };
  const bool tma_ok = aligned16 && !A.table && !B.table && M < (1ll << 31) && N < (1ll << 31) && K < (1ll << 31);
  // narrow n tiles (96 / 64 wide) exist on the TMA path with a K-major B operand only
  const int bn = (tma_ok && b_kmajor && !sym && !b_upper && !tl_nosplit) ? narrow_bn(N) : BN;
  // diagonal tiles of a symmetric K-major x K-major product take the re-dealt path on the TMA kernel
  const bool diag_aware = tma_ok && a_kmajor && b_kmajor && sym && !b_upper && !tl_nosplit;
  apply_plan(make_plan(M, N, K, sym, b_upper, bn, diag_aware, tl_wavesplit));
  if (tl_nosplit) {
    p.splits = 1;
    p.kspan = ceil_div(std::max<int64_t>(K, 1), BK) * BK;
    p.partial = nullptr;
  }
  int rc = HP_OK;
  bool done = false;
  if (tma_ok) {
    if (a_kmajor && b_kmajor)
      rc = bn == 96 ? launch_tma<true, true, 3>(p, st, done)
                    : bn == 64 ? launch_tma<true, true, 2>(p, st, done) : launch_tma<true, true>(p, st, done);
    else if (!a_kmajor && b_kmajor)
      rc = bn == 96 ? launch_tma<false, true, 3>(p, st, done)
                    : bn == 64 ? launch_tma<false, true, 2>(p, st, done) : launch_tma<false, true>(p, st, done);
    else if (!a_kmajor && !b_kmajor)
      rc = launch_tma<false, false>(p, st, done);
    else
      rc = launch_tma<true, false>(p, st, done);
  }
  if (!rc && !done && bn != BN) apply_plan(make_plan(M, N, K, sym, b_upper, BN));  // tensor map not encodable
  if (rc || done) {
  } else if (a_kmajor && b_kmajor)
    rc = aligned16 ? launch_t<true, true, true>(p, st) : launch_t<true, true, false>(p, st);
  else if (!a_kmajor && b_kmajor)
    rc = aligned16 ? launch_t<false, true, true>(p, st) : launch_t<false, true, false>(p, st);
  else if (!a_kmajor && !b_kmajor)
    rc = aligned16 ? launch_t<false, false, true>(p, st) : launch_t<false, false, false>(p, st);
  else
    rc = aligned16 ? launch_t<true, false, true>(p, st) : launch_t<true, false, false>(p, st);
  if (rc) return rc;
  if (p.splits > 1) {
    const int64_t total = p.ntiles * BM * p.bn;
    splitk_reduce<<<(unsigned)ceil_div(total, 256), 256, 0, st>>>(p);
    HP_CHECK_LAUNCH("splitk_reduce");
  }
  return HP_OK;
}

size_t gemm_workspace_bytes(int64_t M, int64_t N, int64_t K, int sym, int b_upper) {
  if (M <= 0 || N <= 0) return 0;
  size_t need = gemm::make_plan(M, N, K, sym, b_upper).ws_bytes;
  if (sym && !b_upper)
    need = std::max({need, gemm::make_plan(M, N, K, sym, b_upper, gemm::BN, true).ws_bytes,
                     gemm::make_plan(M, N, K, sym, b_upper, gemm::BN, true, true).ws_bytes});
  if (!sym && !b_upper)  // the narrow-tile plan of the same shape (gemm_run picks it on the TMA path)
    need = std::max(need, gemm::make_plan(M, N, K, sym, b_upper, gemm::narrow_bn(N)).ws_bytes);
  return need;
}

}  // namespace hp
