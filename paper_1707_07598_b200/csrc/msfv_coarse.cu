// Coarse (Galerkin) system: assembly of A_k = P^T A P from the per-block 8x8
// contributions, banded tiled Cholesky, and the coarse solves.
//
// Reference: forward.py:101-142 forms A_k densely and calls LAPACK dpotrf
// (cho_factor) for k <= 5000, SuperLU above.  A_k couples coarse nodes only
// within a 27-point stencil, so in lexicographic coarse order its half
// bandwidth is pc = (nb1+1)(nb2+1) + (nb1+1) + 1 and Cholesky fill stays
// inside that band: the banded factorization below is the same Cholesky
// factor as the reference's dense one, computed without the zero blocks.
//
// Buffer layout (one allocation of MSFV_INFO_AK_DOUBLES doubles):
//   A     NT*(PT+1) tiles   lower band of A_k; tile column J holds (J+t, J),
//                           t = 0..PT, each TB x TB row-major.  Updated in
//                           place by the factorization (trailing tiles).
//   Dinv  NT tiles          L_JJ^{-1}
//   Lo    NT*(PT+1) tiles   the factor: slot 0 = L_JJ, slot t = L_{J+t,J}
//   LF,LB NT*(PT+1) tiles   solve copies (slot 0 = L_JJ^{-1}) in DMMA fragment
//                           order, forward and transposed (k_coarse_pack)
//   Y     (NT*TB)^2         dense L^{-1} (row-major, lower part), only when
//                           k <= COARSE_INV_MAX: a solve becomes two streaming
//                           products instead of 2*NT dependent tile steps.
// Padding rows (>= kc) are identity.
//
// The factorization is one cooperative launch with one grid barrier per tile
// column: after the barrier every CTA takes trailing-update tasks
// (recomputing the panel products it needs, so the panel TRSM costs no extra
// barrier) and L^{-1} row-panel tasks; CTA 0 first takes the task that
// updates the next diagonal tile and then factors it (one-step lookahead).
#include <cooperative_groups.h>

#include <algorithm>

#include "msfv_common.cuh"
#include "msfv_kernels.h"

namespace cg = cooperative_groups;

namespace msfv {

constexpr int TB = COARSE_TB;
constexpr int TT = TB * TB;

struct CoarseBufs {
  double* A;
  double* Dinv;
  double* Lo;
  double* LF;  // solve copy of (Dinv_J, L_{J+t,J}) in forward fragment order (k_coarse_pack)
  double* LB;  // the same tiles in backward (transposed) fragment order
  double* Y;   // may be null
};

__host__ __device__ __forceinline__ size_t band_tiles(const Geo& g) { return (size_t)g.NT * (g.PT + 1); }
__host__ __device__ __forceinline__ bool coarse_has_inverse(const Geo& g) { return g.coarse_inv != 0; }
__host__ __device__ __forceinline__ size_t y_dim(const Geo& g) { return (size_t)g.NT * TB; }

__host__ __device__ __forceinline__ CoarseBufs coarse_bufs(const Geo& g, double* base) {
  CoarseBufs b;
  b.A = base;
  b.Dinv = b.A + band_tiles(g) * TT;
  b.Lo = b.Dinv + (size_t)g.NT * TT;
  b.LF = b.Lo + band_tiles(g) * TT;
  b.LB = b.LF + band_tiles(g) * TT;
  b.Y = coarse_has_inverse(g) ? b.LB + band_tiles(g) * TT : nullptr;
  return b;
}

size_t coarse_doubles(const Geo& g) {
  size_t n = 4 * band_tiles(g) * TT + (size_t)g.NT * TT;
  if (coarse_has_inverse(g)) n += y_dim(g) * y_dim(g);
  return n;
}
size_t coarse_scratch_doubles(const Geo& g, int nrhs) { return (size_t)g.kc * nrhs; }

__device__ __forceinline__ double* tile(double* A, const Geo& g, int J, int t) {
  return A + ((size_t)J * (g.PT + 1) + t) * TT;
}
__device__ __forceinline__ const double* tile(const double* A, const Geo& g, int J, int t) {
  return A + ((size_t)J * (g.PT + 1) + t) * TT;
}

// Thread per (coarse row c, lower neighbour o): A_k[c][c'] = sum over blocks
// having both as corners (fixed order) of Kloc, + shift on the diagonal.
__global__ void k_coarse_assemble(Geo g, const double* __restrict__ Kloc, double shift, double* __restrict__ Ak) {
  long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  long long tot = (long long)g.NT * TB * 14;
  if (t >= tot) return;
  int o = (int)(t % 14);
  int c = (int)(t / 14);
  if (c >= g.kc) {
    if (o == 0) {
      int J = c / TB, r = c % TB;
      tile(Ak, g, J, 0)[r * TB + r] = 1.0;    // padding rows: identity
    }
    return;
  }
  // enumerate the 14 lexicographically-lower offsets (dz, dy, dx) <= 0
  int dz, dy, dx;
  if (o < 9) { dz = -1; dy = o / 3 - 1; dx = o % 3 - 1; }
  else if (o < 12) { dz = 0; dy = -1; dx = (o - 9) - 1; }
  else { dz = 0; dy = 0; dx = (o - 12) - 1; }
  int ci = c % (g.nb1 + 1), r = c / (g.nb1 + 1), cj = r % (g.nb2 + 1), ck = r / (g.nb2 + 1);
  int di = ci + dx, dj = cj + dy, dk = ck + dz;
  if (di < 0 || dj < 0 || dk < 0 || di > g.nb1 || dj > g.nb2 || dk > g.nb3) return;
  int c2 = coarse_of(g, di, dj, dk);
  double v = 0.0;
  for (int bk = max(ck, dk) - 1; bk <= min(ck, dk); ++bk) {
    if (bk < 0 || bk >= g.nb3) continue;
    for (int bj = max(cj, dj) - 1; bj <= min(cj, dj); ++bj) {
      if (bj < 0 || bj >= g.nb2) continue;
      for (int bi = max(ci, di) - 1; bi <= min(ci, di); ++bi) {
        if (bi < 0 || bi >= g.nb1) continue;
        int l1 = (ci - bi) + 2 * (cj - bj) + 4 * (ck - bk);
        int l2 = (di - bi) + 2 * (dj - bj) + 4 * (dk - bk);
        v += Kloc[(size_t)block_of(g, bi, bj, bk) * 64 + l1 * 8 + l2];
      }
    }
  }
  if (c2 == c) v += shift;
  int I = c / TB, J = c2 / TB;
  tile(Ak, g, J, I - J)[(c % TB) * TB + (c2 % TB)] = v;
}

__global__ void k_coarse_diag(Geo g, const double* __restrict__ Ak, double* __restrict__ diag) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= g.kc) return;
  diag[c] = tile(Ak, g, c / TB, 0)[(c % TB) * TB + (c % TB)];
}

// ------------------------------------------------------------ factorization

struct FactorSmem {
  double P[TB][TB + 1];    // tile operands / POTRF workspace
  double Q[TB][TB + 1];
  double R[TB][TB + 1];
  double D[TB][TB + 1];    // Dinv of the current column
};

__device__ __forceinline__ void load_tile(double (*S)[TB + 1], const double* src) {
  for (int t = threadIdx.x; t < TT; t += blockDim.x) S[t / TB][t % TB] = src[t];
}
__device__ __forceinline__ void store_tile(double* dst, double (*S)[TB + 1]) {
  for (int t = threadIdx.x; t < TT; t += blockDim.x) dst[t] = S[t / TB][t % TB];
}

// 32x32 tile products by 256 threads, each owning a 2x2 output block.
template <bool XT, bool YT>
__device__ __forceinline__ void mm22(double acc[4], double (*X)[TB + 1], double (*Y)[TB + 1], int r0, int c0) {
  acc[0] = acc[1] = acc[2] = acc[3] = 0.0;
#pragma unroll 8
  for (int m = 0; m < TB; ++m) {
    const double x0 = XT ? X[m][r0] : X[r0][m], x1 = XT ? X[m][r0 + 1] : X[r0 + 1][m];
    const double y0 = YT ? Y[c0][m] : Y[m][c0], y1 = YT ? Y[c0 + 1][m] : Y[m][c0 + 1];
    acc[0] += x0 * y0; acc[1] += x0 * y1; acc[2] += x1 * y0; acc[3] += x1 * y1;
  }
}
// O = op(X) op(Y)  (X^T when XT, Y^T when YT)
template <bool XT, bool YT>
__device__ __forceinline__ void mm(double (*O)[TB + 1], double (*X)[TB + 1], double (*Y)[TB + 1]) {
  const int r0 = 2 * (threadIdx.x >> 4), c0 = 2 * (threadIdx.x & 15);
  double a[4];
  mm22<XT, YT>(a, X, Y, r0, c0);
  O[r0][c0] = a[0]; O[r0][c0 + 1] = a[1]; O[r0 + 1][c0] = a[2]; O[r0 + 1][c0 + 1] = a[3];
}
// G (global, leading dimension ld) -= op(X) op(Y)
template <bool XT, bool YT>
__device__ __forceinline__ void gsub(double* G, size_t ld, double (*X)[TB + 1], double (*Y)[TB + 1]) {
  const int r0 = 2 * (threadIdx.x >> 4), c0 = 2 * (threadIdx.x & 15);
  double a[4];
  mm22<XT, YT>(a, X, Y, r0, c0);
  G[r0 * ld + c0] -= a[0]; G[r0 * ld + c0 + 1] -= a[1];
  G[(r0 + 1) * ld + c0] -= a[2]; G[(r0 + 1) * ld + c0 + 1] -= a[3];
}

// Cholesky of diagonal tile J (in A) -> L_JJ (Lo slot 0) and L_JJ^{-1} (Dinv),
// by warp 0 alone: lane r owns row r of L in registers (right-looking with
// shuffles; compile-time unrolled by template recursion so the row stays in
// registers), then lane c owns column c of L^{-1} (forward substitution with
// broadcast shared-memory reads of L).  rsqrt keeps the pivot chain short.
template <int C>
__device__ __forceinline__ void potrf_row_step(double (&x)[TB], double& invd, int r, bool& bad) {
  if constexpr (C < TB) {
    double d = __shfl_sync(0xffffffffu, x[C], C);
    if (!(d > 0.0)) { bad = true; d = 1.0; }
    const double inv = rsqrt(d);
    if (r > C) x[C] *= inv;
    if (r == C) { x[C] = d * inv; invd = inv; }
    const double lrc = x[C];
#pragma unroll
    for (int q = C + 1; q < TB; ++q) {
      const double lqc = __shfl_sync(0xffffffffu, lrc, q);
      if (r >= q) x[q] -= lrc * lqc;
    }
    potrf_row_step<C + 1>(x, invd, r, bad);
  }
}
template <int R>
__device__ __forceinline__ void inv_col_step(double (&d)[TB], int c, const double (*P)[TB + 1], const double* invd) {
  if constexpr (R < TB) {
    double a0 = (R == c) ? 1.0 : 0.0, a1 = 0.0;
#pragma unroll
    for (int m = 0; m + 1 < R; m += 2) {
      a0 -= P[R][m] * d[m];
      a1 -= P[R][m + 1] * d[m + 1];
    }
    if (R & 1) a0 -= P[R][R - 1] * d[R - 1];
    d[R] = (R < c) ? 0.0 : (a0 + a1) * invd[R];
    inv_col_step<R + 1>(d, c, P, invd);
  }
}

__device__ void coarse_potrf(const Geo& g, int J, const CoarseBufs& B, int* flags, FactorSmem& sm) {
  const int tid = threadIdx.x;
  auto& P = sm.P;
  auto& D = sm.D;
  load_tile(P, tile(B.A, g, J, 0));
  __syncthreads();
  if (tid < 32) {
    const int r = tid;
    double x[TB];
#pragma unroll
    for (int q = 0; q < TB; ++q) x[q] = P[r][q];
    double invd = 1.0;
    bool bad = false;
    potrf_row_step<0>(x, invd, r, bad);
    if (bad && r == 0) atomicOr(flags, FLAG_COARSE_NOT_SPD);
#pragma unroll
    for (int q = 0; q < TB; ++q) P[r][q] = q <= r ? x[q] : 0.0;
    sm.Q[0][r] = invd;                // 1 / L[r][r]
    __syncwarp();
    double d[TB];
    inv_col_step<0>(d, r, P, sm.Q[0]);
#pragma unroll
    for (int rr = 0; rr < TB; ++rr) D[rr][r] = d[rr];
  }
  __syncthreads();
  store_tile(B.Dinv + (size_t)J * TT, D);
  store_tile(tile(B.Lo, g, J, 0), P);
  __syncthreads();
}

// Task f of tile column J: f < npairs -> trailing tile (t1, t2); else L^{-1}
// row-panel J restricted to column tile f - npairs.  sm.D holds Dinv_J.
__device__ void coarse_task(const Geo& g, int J, int f, int npairs, const CoarseBufs& B, FactorSmem& sm) {
  auto& X1 = sm.P;
  auto& X2 = sm.Q;
  auto& T = sm.R;
  auto& D = sm.D;
  if (f < npairs) {
    int t1 = (int)((1.0 + sqrt(1.0 + 8.0 * f)) * 0.5);
    while (t1 * (t1 - 1) / 2 > f) --t1;
    while ((t1 + 1) * t1 / 2 <= f) ++t1;
    const int t2 = f - t1 * (t1 - 1) / 2 + 1;
    load_tile(T, tile(B.A, g, J, t1));
    __syncthreads();
    mm<false, true>(X1, T, D);                  // L_{J+t1,J} = A_{J+t1,J} Dinv^T
    __syncthreads();
    if (t2 != t1) {
      load_tile(T, tile(B.A, g, J, t2));
      __syncthreads();
      mm<false, true>(X2, T, D);
      __syncthreads();
      gsub<false, true>(tile(B.A, g, J + t2, t1 - t2), TB, X1, X2);
    } else {
      gsub<false, true>(tile(B.A, g, J + t1, 0), TB, X1, X1);
      store_tile(tile(B.Lo, g, J, t1), X1);
    }
    __syncthreads();
  } else {
    // Yf = Dinv_J Y_J ; W = Dinv_J^T Yf ; Y_{J+t} -= A_{J+t,J} W  (= L_{J+t,J} Yf)
    const int cidx = f - npairs;
    const size_t ld = y_dim(g);
    double* Yj = B.Y + (size_t)J * TB * ld + (size_t)cidx * TB;
    for (int t = threadIdx.x; t < TT; t += blockDim.x) T[t / TB][t % TB] = Yj[(t / TB) * ld + (t % TB)];
    __syncthreads();
    mm<false, false>(X1, D, T);
    __syncthreads();
    for (int t = threadIdx.x; t < TT; t += blockDim.x) Yj[(t / TB) * ld + (t % TB)] = X1[t / TB][t % TB];
    mm<true, false>(X2, D, X1);
    __syncthreads();
    const int pt = min(g.PT, g.NT - 1 - J);
    for (int t = 1; t <= pt; ++t) {
      load_tile(T, tile(B.A, g, J, t));
      __syncthreads();
      gsub<false, false>(B.Y + (size_t)(J + t) * TB * ld + (size_t)cidx * TB, ld, T, X2);
      __syncthreads();
    }
  }
}

__global__ void __launch_bounds__(256) k_coarse_factor(Geo g, double* __restrict__ base, int* __restrict__ flags) {
  __shared__ FactorSmem sm;
  cg::grid_group grid = cg::this_grid();
  const CoarseBufs B = coarse_bufs(g, base);
  const bool withY = B.Y != nullptr;
  if (withY) {
    const size_t ld = y_dim(g);
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < ld; i += (size_t)gridDim.x * blockDim.x)
      B.Y[i * ld + i] = 1.0;
  }
  if (blockIdx.x == 0) coarse_potrf(g, 0, B, flags, sm);
  grid.sync();
  for (int J = 0; J < g.NT; ++J) {
    const int pt = min(g.PT, g.NT - 1 - J);
    const int npairs = pt * (pt + 1) / 2;
    const int ntasks = npairs + (withY ? J + 1 : 0);
    load_tile(sm.D, B.Dinv + (size_t)J * TT);
    __syncthreads();
    if (blockIdx.x == 0 && pt >= 1) {
      coarse_task(g, J, 0, npairs, B, sm);       // pair (1,1): next diagonal tile
      __threadfence_block();
      coarse_potrf(g, J + 1, B, flags, sm);      // lookahead factor of column J+1
    }
    // the other CTAs share everything except the lookahead pair
    const int first = (pt >= 1) ? 1 : 0;
    const int nw = gridDim.x > 1 ? gridDim.x - 1 : 1;
    if (gridDim.x == 1 || blockIdx.x > 0) {
      const int me = gridDim.x > 1 ? blockIdx.x - 1 : 0;
      for (int f = first + me; f < ntasks; f += nw) coarse_task(g, J, f, npairs, B, sm);
    }
    grid.sync();
  }
}

// -------------------------------------------------- solves with L^{-1}

constexpr int SCH = 16;   // sources per pass

// Z[r][s] = sum_{c <= r} Y[r][c] X[c][s]; CTA per row tile, warp w owns rows
// w, w+8, w+16, w+24, lanes run over the 32 columns of each column tile.
__global__ void __launch_bounds__(256) k_coarse_inv_lower(Geo g, const double* __restrict__ Y, const double* __restrict__ X,
                                                          double* __restrict__ Z, int nrhs) {
  __shared__ double Xs[TB][SCH + 1];
  const int I = blockIdx.x;
  const size_t ld = y_dim(g);
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  for (int s0 = 0; s0 < nrhs; s0 += SCH) {
    double acc[4][SCH];
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int s = 0; s < SCH; ++s) acc[q][s] = 0.0;
    for (int C = 0; C <= I; ++C) {
      __syncthreads();
      for (int t = tid; t < TB * SCH; t += blockDim.x) {
        int c = t / SCH, s = t % SCH, row = C * TB + c;
        Xs[c][s] = (row < g.kc && s0 + s < nrhs) ? X[(size_t)row * nrhs + s0 + s] : 0.0;
      }
      __syncthreads();
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const double yv = __ldg(Y + (size_t)(I * TB + w + 8 * q) * ld + (size_t)C * TB + lane);
#pragma unroll
        for (int s = 0; s < SCH; ++s) acc[q][s] += yv * Xs[lane][s];
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
#pragma unroll
      for (int s = 0; s < SCH; ++s) {
        double v = acc[q][s];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
        acc[q][s] = v;
      }
      const int row = I * TB + w + 8 * q;
      if (lane < SCH && row < g.kc && s0 + lane < nrhs) {
        double v = 0.0;
#pragma unroll
        for (int s = 0; s < SCH; ++s) v = (s == lane) ? acc[q][s] : v;
        Z[(size_t)row * nrhs + s0 + lane] = v;
      }
    }
  }
}

// X[c][s] = sum_{r >= c} Y[r][c] Z[r][s]; CTA per column tile, lanes over its
// 32 columns, warps over rows, smem reduction across warps.
__global__ void __launch_bounds__(256) k_coarse_inv_upper(Geo g, const double* __restrict__ Y, const double* __restrict__ Z,
                                                          double* __restrict__ X, int nrhs) {
  __shared__ double Zs[TB][SCH + 1];
  __shared__ double red[8][TB][SCH + 1];
  const int C = blockIdx.x;
  const size_t ld = y_dim(g);
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  for (int s0 = 0; s0 < nrhs; s0 += SCH) {
    double acc[SCH];
#pragma unroll
    for (int s = 0; s < SCH; ++s) acc[s] = 0.0;
    for (int I = C; I < g.NT; ++I) {
      __syncthreads();
      for (int t = tid; t < TB * SCH; t += blockDim.x) {
        int rr = t / SCH, s = t % SCH, row = I * TB + rr;
        Zs[rr][s] = (row < g.kc && s0 + s < nrhs) ? Z[(size_t)row * nrhs + s0 + s] : 0.0;
      }
      __syncthreads();
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int rr = w + 8 * q;
        const double yv = __ldg(Y + (size_t)(I * TB + rr) * ld + (size_t)C * TB + lane);
#pragma unroll
        for (int s = 0; s < SCH; ++s) acc[s] += yv * Zs[rr][s];
      }
    }
#pragma unroll
    for (int s = 0; s < SCH; ++s) red[w][lane][s] = acc[s];
    __syncthreads();
    for (int t = tid; t < TB * SCH; t += blockDim.x) {
      int c = t / SCH, s = t % SCH;
      double v = 0.0;
#pragma unroll
      for (int p = 0; p < 8; ++p) v += red[p][c][s];
      const int row = C * TB + c;
      if (row < g.kc && s0 + s < nrhs) X[(size_t)row * nrhs + s0 + s] = v;
    }
    __syncthreads();
  }
}

// ------------------------------------------------ banded trsv (large k)

// Forward then backward substitution with the banded tiled factor for RC
// right-hand sides per CTA.  X is [kc][nrhs] row-major.  The factor tiles
// stream through a RING-slot cp.async pipeline in shared memory in exactly
// the order they are consumed (forward: Dinv_J, L_{J+1,J}..L_{J+pt,J};
// backward: L_{J+1,J}..L_{J+pt,J}, Dinv_J); the active right-hand-side rows
// (PT+1 tile rows) live in a shared-memory ring, so global X is read and
// written once per sweep.
namespace {
__device__ __forceinline__ void cpa16(void* smem, const void* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cpa_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// tile sequence iterator: forward (dir=+1) or backward (dir=-1)
struct TileSeq {
  int J, t, NT, PT, dir;
  __device__ int pt() const { return min(PT, NT - 1 - J); }
  __device__ bool valid() const { return J >= 0 && J < NT; }
  // forward order: t = 0 (Dinv), 1..pt ; backward order: t = 1..pt, then 0 (Dinv)
  __device__ void next() {
    if (dir > 0) {
      if (t < pt()) ++t; else { ++J; t = 0; }
    } else {
      if (t == 0) { --J; t = (J >= 0 && pt() > 0) ? 1 : 0; }
      else if (t < pt()) ++t;
      else t = 0;
    }
  }
};
}  // namespace

template <int RC>
__global__ void __launch_bounds__(256) k_coarse_trsv(Geo g, const double* __restrict__ Lk, const double* __restrict__ Dinv,
                                                     double* __restrict__ X, int nrhs) {
  constexpr int RING = 4;
  extern __shared__ __align__(16) double tsm[];
  double* ring = tsm;                              // [RING][TB*TB]
  double* Xw = ring + RING * TT;              // [PT+1][TB][RC]
  double* Ys = Xw + (size_t)(g.PT + 1) * TB * RC;  // [TB][RC]
  const int tid = threadIdx.x, nt = blockDim.x;
  const int s0 = blockIdx.x * RC;
  const int ns = min(RC, nrhs - s0);
  const int W = g.PT + 1;
  auto src_of = [&](const TileSeq& q) -> const double* {
    return q.t == 0 ? Dinv + (size_t)q.J * TT : tile(Lk, g, q.J, q.t);
  };
  auto issue = [&](TileSeq& q, int slot) {
    if (q.valid()) {
      const double* src = src_of(q);
      double* dst = ring + slot * TT;
      for (int i = tid; i < TT / 2; i += nt) cpa16(dst + 2 * i, src + 2 * i);
    }
    cpa_commit();
    q.next();
  };
  auto load_rows = [&](int I, double* dst) {
    for (int t = tid; t < TB * RC; t += nt) {
      int r = t / RC, s = t % RC, row = I * TB + r;
      dst[t] = (I < g.NT && s < ns && row < g.kc) ? X[(size_t)row * nrhs + s0 + s] : 0.0;
    }
  };
    {
    TileSeq pf{0, 0, g.NT, g.PT, 1};
    int issued = 0, consumed = 0;
    for (; issued < RING - 1; ++issued) issue(pf, issued % RING);
    for (int I = 0; I <= g.PT; ++I) load_rows(I, Xw + (size_t)(I % W) * TB * RC);
    for (int J = 0; J < g.NT; ++J) {
      const int pt = min(g.PT, g.NT - 1 - J);
      for (int t = 0; t <= pt; ++t) {
        cpa_wait<RING - 2>();
        __syncthreads();
        issue(pf, issued % RING);
        ++issued;
        const double* T = ring + (consumed % RING) * TT;
        ++consumed;
        if (t == 0) {
          const double* xj = Xw + (size_t)(J % W) * TB * RC;
          for (int q = tid; q < TB * RC; q += nt) {
            int r = q / RC, s = q % RC;
            double v = 0.0;
#pragma unroll 8
            for (int c = 0; c < TB; ++c) v += T[r * TB + c] * xj[c * RC + s];
            Ys[q] = v;
            int row = J * TB + r;
            if (s < ns && row < g.kc) X[(size_t)row * nrhs + s0 + s] = v;
          }
        } else {
          double* xt = Xw + (size_t)((J + t) % W) * TB * RC;
          for (int q = tid; q < TB * RC; q += nt) {
            int r = q / RC, s = q % RC;
            double v = 0.0;
#pragma unroll 8
            for (int c = 0; c < TB; ++c) v += T[r * TB + c] * Ys[c * RC + s];
            xt[q] -= v;
          }
        }
      }
      __syncthreads();
      load_rows(J + 1 + g.PT, Xw + (size_t)(J % W) * TB * RC);   // slot of row J is free now
    }
    cpa_wait<0>();
    __syncthreads();
  }
    {
    TileSeq pf{g.NT - 1, 0, g.NT, g.PT, -1};
    pf.t = (pf.pt() > 0) ? 1 : 0;
    int issued = 0, consumed = 0;
    for (; issued < RING - 1; ++issued) issue(pf, issued % RING);
    for (int J = g.NT - 1; J >= 0; --J) {
      const int pt = min(g.PT, g.NT - 1 - J);
      // acc = y_J
      for (int q = tid; q < TB * RC; q += nt) {
        int r = q / RC, s = q % RC, row = J * TB + r;
        Ys[q] = (s < ns && row < g.kc) ? X[(size_t)row * nrhs + s0 + s] : 0.0;
      }
      for (int k = 0; k <= pt; ++k) {
        const int t = (k < pt) ? k + 1 : 0;
        cpa_wait<RING - 2>();
        __syncthreads();
        issue(pf, issued % RING);
        ++issued;
        const double* T = ring + (consumed % RING) * TT;
        ++consumed;
        if (t > 0) {
          const double* xt = Xw + (size_t)((J + t) % W) * TB * RC;
          for (int q = tid; q < TB * RC; q += nt) {
            int c = q / RC, s = q % RC;
            double v = 0.0;
#pragma unroll 8
            for (int r = 0; r < TB; ++r) v += T[r * TB + c] * xt[r * RC + s];
            Ys[q] -= v;
          }
        } else {
          double* xj = Xw + (size_t)(J % W) * TB * RC;
          for (int q = tid; q < TB * RC; q += nt) {
            int r = q / RC, s = q % RC;
            double v = 0.0;
            for (int c = r; c < TB; ++c) v += T[c * TB + r] * Ys[c * RC + s];
            int row = J * TB + r;
            if (row >= g.kc || s >= ns) v = 0.0;
            xj[q] = v;
            if (s < ns && row < g.kc) X[(size_t)row * nrhs + s0 + s] = v;
          }
        }
      }
      __syncthreads();
    }
    cpa_wait<0>();
  }
}

// Step-buffered variant: all PT+1 factor tiles of a column step are staged
// in shared memory at once (double-buffered with cp.async one step ahead; row
// stride TB+2 doubles to avoid bank conflicts), so each step is two
// barrier-separated GEMV phases over all 256 threads.
constexpr int TS = TB + 2;            // padded smem row stride (16-byte granules)
constexpr int TTS = TB * TS;
template <int RC>
__global__ void __launch_bounds__(256) k_coarse_trsv_step(Geo g, const double* __restrict__ Lk,
                                                          const double* __restrict__ Dinv, double* __restrict__ X,
                                                          int nrhs) {
  extern __shared__ __align__(16) double tsm[];
  const int W = g.PT + 1;
  double* buf[2] = {tsm, tsm + (size_t)W * TTS};                // slot 0 = Dinv_J, slot t = L_{J+t,J}
  double* Xw = tsm + (size_t)2 * W * TTS;                         // [PT+1][TB][RC] rhs ring
  double* Ys = Xw + (size_t)W * TB * RC;                          // [TB][RC]
  const int tid = threadIdx.x, nt = blockDim.x;
  const int s0 = blockIdx.x * RC;
  const int ns = min(RC, nrhs - s0);
  auto cp_tile = [&](double* dst, const double* src) {
    for (int i = tid; i < TT / 2; i += nt) {
      const int r = (2 * i) / TB, c = (2 * i) % TB;
      cpa16(dst + r * TS + c, src + 2 * i);
    }
  };
  auto issue = [&](int J, double* dst) {
    if (J >= 0 && J < g.NT) {
      const int pt = min(g.PT, g.NT - 1 - J);
      cp_tile(dst, Dinv + (size_t)J * TT);
      for (int t = 1; t <= pt; ++t) cp_tile(dst + (size_t)t * TTS, tile(Lk, g, J, t));
    }
    cpa_commit();
  };
  auto load_rows = [&](int I, double* dst) {
    for (int t = tid; t < TB * RC; t += nt) {
      int r = t / RC, s = t % RC, row = I * TB + r;
      dst[t] = (I < g.NT && s < ns && row < g.kc) ? X[(size_t)row * nrhs + s0 + s] : 0.0;
    }
  };
  // ---------------- forward: y_J = Dinv_J x_J ; x_{J+t} -= L_{J+t,J} y_J
  issue(0, buf[0]);
  issue(1, buf[1]);
  for (int I = 0; I <= g.PT; ++I) load_rows(I, Xw + (size_t)(I % W) * TB * RC);
  for (int J = 0; J < g.NT; ++J) {
    const int pt = min(g.PT, g.NT - 1 - J);
    double* T = buf[J & 1];
    cpa_wait<1>();
    __syncthreads();
    const double* xj = Xw + (size_t)(J % W) * TB * RC;
    for (int q = tid; q < TB * RC; q += nt) {
      const int r = q / RC, s = q % RC;
      const double* tr = T + r * TS;
      double v0 = 0.0, v1 = 0.0;
#pragma unroll 8
      for (int c = 0; c < TB; c += 2) { v0 += tr[c] * xj[c * RC + s]; v1 += tr[c + 1] * xj[(c + 1) * RC + s]; }
      const double v = v0 + v1;
      Ys[q] = v;
      const int row = J * TB + r;
      if (s < ns && row < g.kc) X[(size_t)row * nrhs + s0 + s] = v;
    }
    __syncthreads();
    for (int q = tid; q < pt * TB * RC; q += nt) {
      const int tt = 1 + q / (TB * RC), rem = q % (TB * RC), r = rem / RC, s = rem % RC;
      const double* L = T + (size_t)tt * TTS + r * TS;
      double v0 = 0.0, v1 = 0.0;
#pragma unroll 8
      for (int c = 0; c < TB; c += 2) { v0 += L[c] * Ys[c * RC + s]; v1 += L[c + 1] * Ys[(c + 1) * RC + s]; }
      Xw[(size_t)((J + tt) % W) * TB * RC + rem] -= v0 + v1;
    }
    __syncthreads();
    load_rows(J + 1 + g.PT, Xw + (size_t)(J % W) * TB * RC);
    issue(J + 2, buf[J & 1]);
  }
  cpa_wait<0>();
  __syncthreads();
  // ---------------- backward: x_J = Dinv_J^T (y_J - sum_t L_{J+t,J}^T x_{J+t})
  issue(g.NT - 1, buf[0]);
  issue(g.NT - 2, buf[1]);
  constexpr int SPLIT = 256 / (TB * RC) > 0 ? 256 / (TB * RC) : 1;   // threads per output
  for (int it = 0; it < g.NT; ++it) {
    const int J = g.NT - 1 - it;
    const int pt = min(g.PT, g.NT - 1 - J);
    double* T = buf[it & 1];
    cpa_wait<1>();
    __syncthreads();
    {
      const int q = tid / SPLIT, part = tid % SPLIT;
      double v0 = 0.0, v1 = 0.0;
      if (q < TB * RC) {
        const int c = q / RC, s = q % RC;
        for (int tt = 1 + part; tt <= pt; tt += SPLIT) {
          const double* L = T + (size_t)tt * TTS + c;
          const double* xt = Xw + (size_t)((J + tt) % W) * TB * RC + s;
#pragma unroll 8
          for (int r = 0; r < TB; r += 2) { v0 += L[r * TS] * xt[r * RC]; v1 += L[(r + 1) * TS] * xt[(r + 1) * RC]; }
        }
      }
      double v = v0 + v1;
#pragma unroll
      for (int off = SPLIT / 2; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off, SPLIT);
      if (q < TB * RC && part == 0) {
        const int c = q / RC, s = q % RC, row = J * TB + c;
        const double y = (s < ns && row < g.kc) ? X[(size_t)row * nrhs + s0 + s] : 0.0;
        Ys[q] = y - v;
      }
    }
    __syncthreads();
    double* xo = Xw + (size_t)(J % W) * TB * RC;
    for (int q = tid; q < TB * RC; q += nt) {
      const int r = q / RC, s = q % RC, row = J * TB + r;
      double v = 0.0;
      for (int c = r; c < TB; ++c) v += T[c * TS + r] * Ys[c * RC + s];
      if (row >= g.kc || s >= ns) v = 0.0;
      xo[q] = v;
      if (s < ns && row < g.kc) X[(size_t)row * nrhs + s0 + s] = v;
    }
    __syncthreads();
    issue(J - 2, buf[it & 1]);
  }
  cpa_wait<0>();
}

namespace {
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}
}  // namespace

// ----------------------------------------------------------- bulk solves
//
// Solve-side copies of the factor.  Both sweeps carry the right-hand sides
// transposed (8 sources x 32 rows per tile row, as four 8x8 accumulator-layout
// pieces), so every product is D += X Y^T of two accumulator-layout 8x8
// pieces (chunk h of k = columns {2k+h}, the layout's slot h).  A 32x32 tile T
// is stored as 16 pieces of 64 doubles at lane*2 (one 512-byte conflict-free
// warp load each):
//   LF piece (mi, kb) = T  block (mi, kb)          (forward:  y^T = r^T Dinv^T, r^T -= y^T L^T)
//   LB piece (nb, kb) = T^T block (nb, kb)         (backward: x^T = (y^T - x^T L) Dinv)
// with slot 0 of tile column J holding Dinv_J.  Tiles below the band end are 0.
__global__ void k_coarse_pack(Geo g, const double* __restrict__ Lo, const double* __restrict__ Dinv,
                              double* __restrict__ LF, double* __restrict__ LB) {
  const int J = blockIdx.x / (g.PT + 1), t = blockIdx.x % (g.PT + 1);
  const bool valid = t == 0 || J + t < g.NT;
  const double* src = t == 0 ? Dinv + (size_t)J * TT : tile(Lo, g, J, t);
  double* f = LF + (size_t)blockIdx.x * TT;
  double* b = LB + (size_t)blockIdx.x * TT;
  for (int e = threadIdx.x; e < TT; e += blockDim.x) {
    const int p = e >> 6, w = e & 63, lane = w >> 1, sl = w & 1, m = lane >> 2, q = lane & 3;
    const int hi = p >> 2, kb = p & 3;
    f[e] = valid ? src[(8 * hi + m) * TB + 8 * kb + 2 * q + sl] : 0.0;
    b[e] = valid ? src[(8 * kb + 2 * q + sl) * TB + 8 * hi + m] : 0.0;
  }
}

namespace {
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(bar)));
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase) {
  unsigned done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
  }
}
// D += X Y^T, X / Y accumulator-layout pieces given as (x0, x1) / (y0, y1)
__device__ __forceinline__ void mma_xyt(double& c0, double& c1, double x0, double x1, double y0, double y1) {
  dmma(c0, c1, x0, y0);
  dmma(c0, c1, x1, y1);
}
}  // namespace

// Forward then backward substitution for 8 right-hand sides per CTA.  The
// factor tiles of a step (tile column J of LF / LB) are cut into nch chunks
// of up to CHT contiguous tiles; the chunk sequence (forward: J ascending,
// chunks in order; backward: J descending, chunks reversed so the Dinv chunk
// comes last) streams through a ring of TRSV_STAGES shared-memory stages, one
// bulk TMA copy per chunk, prefetched TRSV_STAGES-1 chunks ahead.  The active
// right-hand-side rows live in a shared-memory ring of transposed pieces.
constexpr int TRSV_MAX_STAGES = 3;

__global__ void __launch_bounds__(256) k_coarse_trsv_bulk(Geo g, const double* __restrict__ LF,
                                                          const double* __restrict__ LB, double* __restrict__ X,
                                                          int nrhs, int CHT, int NS) {
  extern __shared__ __align__(128) double bsm[];
  __shared__ __align__(8) unsigned long long bar[TRSV_MAX_STAGES];
  const int W = g.PT + 1;
  const int nch = (W + CHT - 1) / CHT;
  const size_t stage_dbl = (size_t)CHT * TT;
  double* Rt = bsm + NS * stage_dbl;   // [W][4][64] rhs ring (transposed pieces)
  double* Ys = Rt + (size_t)W * 256;             // [4][64]
  double* Pt = Ys + 256;                         // [8][64]
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int c = lane >> 2, q = lane & 3;
  const int col = blockIdx.x * 8 + c;
  const bool cok = col < nrhs;
  auto ldx = [&](int R, int pi, double& a, double& b) {
    const int r0 = R * TB + 8 * pi + 2 * q;
    a = (cok && R < g.NT && r0 < g.kc) ? X[(size_t)r0 * nrhs + col] : 0.0;
    b = (cok && R < g.NT && r0 + 1 < g.kc) ? X[(size_t)(r0 + 1) * nrhs + col] : 0.0;
  };
  auto stx = [&](int R, int pi, double a, double b) {
    const int r0 = R * TB + 8 * pi + 2 * q;
    if (cok && r0 < g.kc) X[(size_t)r0 * nrhs + col] = a;
    if (cok && r0 + 1 < g.kc) X[(size_t)(r0 + 1) * nrhs + col] = b;
  };
  auto piece = [&](const double* base, int p) -> const double* { return base + p * 64 + 2 * lane; };
  auto ring = [&](int jm, int t) { const int r = jm + t; return r >= W ? r - W : r; };   // (J + t) % W, jm = J % W
  const int nf = g.NT * nch, total = 2 * nf;
  // chunk sequence iterator (no integer division in the loop)
  struct It {
    int J, ch, jm;
    bool fwd;
  };
  auto advance = [&](It& c) {
    if (c.fwd) {
      if (++c.ch == nch) {
        c.ch = 0;
        ++c.J;
        c.jm = c.jm + 1 == W ? 0 : c.jm + 1;
        if (c.J == g.NT) {
          c.fwd = false;
          c.J = g.NT - 1;
          c.ch = nch - 1;
          c.jm = (g.NT - 1) % W;
        }
      }
    } else if (--c.ch < 0) {
      c.ch = nch - 1;
      --c.J;
      c.jm = c.jm == 0 ? W - 1 : c.jm - 1;
    }
  };
  It ld = {0, 0, 0, true};          // next chunk to load
  int ld_i = 0, ld_st = 0;
  auto issue_next = [&]() {
    if (ld_i >= total) return;
    const int nt = min(CHT, W - ld.ch * CHT);
    const double* src = (ld.fwd ? LF : LB) + ((size_t)ld.J * W + (size_t)ld.ch * CHT) * TT;
    bulk_load(bsm + (size_t)ld_st * stage_dbl, src, (unsigned)(nt * TT * sizeof(double)), &bar[ld_st]);
    advance(ld);
    ++ld_i;
    ld_st = ld_st + 1 == NS ? 0 : ld_st + 1;
  };
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) mbar_init(&bar[s]);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (tid == 0)
    for (int i = 0; i < NS - 1; ++i) issue_next();
  for (int i = tid; i < W * 128; i += blockDim.x) {         // rows 0..PT enter the ring
    const int R = i / 128, pi = (i / 32) & 3;
    if ((i & 31) == lane) {
      double a, b;
      ldx(R, pi, a, b);
      Rt[(R * 4 + pi) * 64 + 2 * lane] = a;
      Rt[(R * 4 + pi) * 64 + 2 * lane + 1] = b;
    }
  }
  __syncthreads();
  double p0 = 0.0, p1 = 0.0;        // backward partial sums of this warp, across the step's chunks
  double ya = 0.0, yb = 0.0;
  It cu = {0, 0, 0, true};
  int st = 0;
  unsigned par = 0u;
  for (int i = 0; i < total; ++i, advance(cu), st = st + 1 == NS ? 0 : st + 1) {
    if (tid == 0) issue_next();
    const int J = cu.J, ch = cu.ch, jm = cu.jm;
    const int pt = min(g.PT, g.NT - 1 - J);
    const int t0 = ch * CHT, t1 = min(W, t0 + CHT) - 1;
    const double* T = bsm + (size_t)st * stage_dbl;           // local tile (t - t0)
    if (i == nf) {                                           // backward: the ring keeps x^T
      for (int k = tid; k < W * 256; k += blockDim.x) Rt[k] = 0.0;
      __syncthreads();
    }
    if (i >= nf && ch == nch - 1) {                         // first chunk of a backward step
      p0 = p1 = 0.0;
      if (wid < 4) ldx(J, wid, ya, yb);
    }
    double ra = 0.0, rb = 0.0;
    if (i < nf && ch == nch - 1 && wid < 4) ldx(J + 1 + g.PT, wid, ra, rb);   // in flight during the step
    mbar_wait(&bar[st], (par >> st) & 1u);
    par ^= 1u << st;
    if (i < nf) {
      // ---------- forward: y_J^T = r_J^T Dinv_J^T ; r_{J+t}^T -= y_J^T L_{J+t,J}^T
      if (ch == 0) {
        if (wid < 4) {
          const int mi = wid;
          const double* RJ = Rt + (size_t)jm * 256;
          double c0 = 0.0, c1 = 0.0, e0 = 0.0, e1 = 0.0;
#pragma unroll
          for (int kb = 0; kb < 4; kb += 2) {
            const double* x = piece(RJ, kb);
            const double* y = piece(T, mi * 4 + kb);
            const double* x2 = piece(RJ, kb + 1);
            const double* y2 = piece(T, mi * 4 + kb + 1);
            mma_xyt(c0, c1, x[0], x[1], y[0], y[1]);
            mma_xyt(e0, e1, x2[0], x2[1], y2[0], y2[1]);
          }
          c0 += e0;
          c1 += e1;
          Ys[mi * 64 + 2 * lane] = c0;
          Ys[mi * 64 + 2 * lane + 1] = c1;
          stx(J, mi, c0, c1);
        }
        __syncthreads();
      }
      const int ta = max(t0, 1), tb = min(t1, pt);
      {
        const int np = (tb - ta + 1) * 4;
        for (int p = wid; p < np; p += 8) {
          const int t = ta + (p >> 2), mi = p & 3;
          double* acc = Rt + (size_t)(ring(jm, t) * 4 + mi) * 64 + 2 * lane;
          double c0 = acc[0], c1 = acc[1];
          const double* Tt = T + (size_t)(t - t0) * TT;
#pragma unroll
          for (int kb = 0; kb < 4; ++kb) {
            const double* x = piece(Ys, kb);
            const double* y = piece(Tt, mi * 4 + kb);
            mma_xyt(c0, c1, -x[0], -x[1], y[0], y[1]);
          }
          acc[0] = c0;
          acc[1] = c1;
        }
      }
      __syncthreads();
      if (ch == nch - 1 && wid < 4) {                        // row J + 1 + PT enters the ring
        const double a = ra, b = rb;
        double* d = Rt + (size_t)(jm * 4 + wid) * 64 + 2 * lane;
        d[0] = a;
        d[1] = b;
      }
    } else {
      // ---------- backward: x_J^T = (y_J^T - sum_t x_{J+t}^T L_{J+t,J}) Dinv_J
      {
        const int nb = wid & 3, half = wid >> 2;
        const int ta = max(t0, 1), tb = min(t1, pt);
        double e0 = 0.0, e1 = 0.0;
        for (int t = ta + ((ta & 1) != half ? 1 : 0); t <= tb; t += 2) {
          const double* xr = Rt + (size_t)ring(jm, t) * 256;
          const double* Tt = T + (size_t)(t - t0) * TT;
#pragma unroll
          for (int kb = 0; kb < 4; kb += 2) {
            const double* x = piece(xr, kb);
            const double* y = piece(Tt, nb * 4 + kb);
            const double* x2 = piece(xr, kb + 1);
            const double* y2 = piece(Tt, nb * 4 + kb + 1);
            mma_xyt(p0, p1, x[0], x[1], y[0], y[1]);
            mma_xyt(e0, e1, x2[0], x2[1], y2[0], y2[1]);
          }
        }
        p0 += e0;
        p1 += e1;
      }
      if (ch == 0) {
        Pt[wid * 64 + 2 * lane] = p0;
        Pt[wid * 64 + 2 * lane + 1] = p1;
        __syncthreads();
        if (wid < 4) {
          const int nb = wid;
          Ys[nb * 64 + 2 * lane] = (ya + Pt[nb * 64 + 2 * lane]) + Pt[(nb + 4) * 64 + 2 * lane];
          Ys[nb * 64 + 2 * lane + 1] = (yb + Pt[nb * 64 + 2 * lane + 1]) + Pt[(nb + 4) * 64 + 2 * lane + 1];
        }
        __syncthreads();
        if (wid < 4) {
          const int nb = wid;
          double c0 = 0.0, c1 = 0.0, e0 = 0.0, e1 = 0.0;
#pragma unroll
          for (int kb = 0; kb < 4; kb += 2) {
            const double* x = piece(Ys, kb);
            const double* y = piece(T, nb * 4 + kb);
            const double* x2 = piece(Ys, kb + 1);
            const double* y2 = piece(T, nb * 4 + kb + 1);
            mma_xyt(c0, c1, x[0], x[1], y[0], y[1]);
            mma_xyt(e0, e1, x2[0], x2[1], y2[0], y2[1]);
          }
          c0 += e0;
          c1 += e1;
          const int r0 = J * TB + 8 * nb + 2 * q;
          if (r0 >= g.kc) c0 = 0.0;
          if (r0 + 1 >= g.kc) c1 = 0.0;
          double* xo = Rt + (size_t)(jm * 4 + nb) * 64 + 2 * lane;   // ring keeps -x^T
          xo[0] = cok ? -c0 : 0.0;
          xo[1] = cok ? -c1 : 0.0;
          stx(J, nb, c0, c1);
        }
      }
      __syncthreads();
    }
  }
}

// One whole tile column per stage (2 stages) when it fits, else chunks
// through 3 stages.
static void trsv_bulk_shape(const Geo& g, int& cht, int& ns, size_t& smem) {
  const int W = g.PT + 1;
  const size_t fixed = ((size_t)W * 256 + 256 + 8 * 64) * sizeof(double);
  const size_t budget = 220 * 1024, tile_b = (size_t)TT * sizeof(double);
  cht = 0;
  ns = 0;
  smem = 0;
  if (fixed + 2 * W * tile_b <= budget) {
    cht = W;
    ns = 2;
  } else {
    if (fixed + (size_t)TRSV_MAX_STAGES * tile_b > budget) return;
    const int maxc = (int)((budget - fixed) / (TRSV_MAX_STAGES * tile_b));
    const int nch = (W + maxc - 1) / maxc;
    cht = (W + nch - 1) / nch;
    ns = TRSV_MAX_STAGES;
  }
  smem = fixed + (size_t)ns * cht * tile_b;
}

// ------------------------------------------------------------- launchers

static inline unsigned nblk(long long n, int t) { return (unsigned)((n + t - 1) / t); }

cudaError_t launch_coarse_assemble(const Geo& g, const double* Kloc, double shift, double* Ak, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(Ak, 0, band_tiles(g) * TT * sizeof(double), st);
  if (e != cudaSuccess) return e;
  long long tot = (long long)g.NT * TB * 14;
  k_coarse_assemble<<<nblk(tot, 256), 256, 0, st>>>(g, Kloc, shift, Ak);
  count_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_coarse_diag(const Geo& g, const double* Ak, double* diag, cudaStream_t st) {
  k_coarse_diag<<<nblk(g.kc, 256), 256, 0, st>>>(g, Ak, diag);
  count_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_coarse_factor(const Geo& g, double* Ak, int* flags, cudaStream_t st) {
  static int coop_grid = -1;
  if (coop_grid < 0) {
    int dev = 0, sms = 0, per_sm = 0, coop = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_coarse_factor, 256, 0);
    coop_grid = (coop && per_sm > 0) ? sms : 0;
  }
  if (coop_grid <= 0) return cudaErrorNotSupported;
  CoarseBufs B = coarse_bufs(g, Ak);
  if (B.Y) {
    cudaError_t e = cudaMemsetAsync(B.Y, 0, y_dim(g) * y_dim(g) * sizeof(double), st);
    if (e != cudaSuccess) return e;
  }
  Geo gg = g;
  void* args[] = {(void*)&gg, (void*)&Ak, (void*)&flags};
  cudaError_t e = cudaLaunchCooperativeKernel((void*)k_coarse_factor, dim3(coop_grid), dim3(256), args, 0, st);
  count_launches(1);
  if (e != cudaSuccess) return e;
  k_coarse_pack<<<(unsigned)band_tiles(g), 256, 0, st>>>(g, B.Lo, B.Dinv, B.LF, B.LB);
  count_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_coarse_solve(const Geo& g, const double* Ak, double* X, double* scratch, int nrhs, cudaStream_t st) {
  if (nrhs == 0) return cudaSuccess;
  CoarseBufs B = coarse_bufs(g, const_cast<double*>(Ak));
  if (B.Y) {
    k_coarse_inv_lower<<<g.NT, 256, 0, st>>>(g, B.Y, X, scratch, nrhs);
    count_launches(1);
    k_coarse_inv_upper<<<g.NT, 256, 0, st>>>(g, B.Y, scratch, X, nrhs);
    count_launches(1);
    return cudaGetLastError();
  }
  constexpr int RC = 4;
  int cht = 0, ns = 0;
  size_t smem_b = 0;
  trsv_bulk_shape(g, cht, ns, smem_b);
  if (cht > 0) {
    cudaError_t e = cudaFuncSetAttribute(k_coarse_trsv_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_b);
    if (e != cudaSuccess) return e;
    k_coarse_trsv_bulk<<<nblk(nrhs, 8), 256, smem_b, st>>>(g, B.LF, B.LB, X, nrhs, cht, ns);
    count_launches(1);
    return cudaGetLastError();
  }
  const size_t smem_s = ((size_t)2 * (g.PT + 1) * TTS + ((size_t)g.PT + 2) * TB * RC) * sizeof(double);
  if (smem_s <= 200 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k_coarse_trsv_step<RC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_s);
    if (e != cudaSuccess) return e;
    k_coarse_trsv_step<RC><<<nblk(nrhs, RC), 256, smem_s, st>>>(g, B.Lo, B.Dinv, X, nrhs);
    count_launches(1);
    return cudaGetLastError();
  }
  size_t smem = ((size_t)4 * TT + ((size_t)g.PT + 2) * TB * RC) * sizeof(double);
  cudaError_t e = cudaFuncSetAttribute(k_coarse_trsv<RC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k_coarse_trsv<RC><<<nblk(nrhs, RC), 256, smem, st>>>(g, B.Lo, B.Dinv, X, nrhs);
  count_launches(1);
  return cudaGetLastError();
}

}  // namespace msfv
