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
//   Lo    NT*(PT+1) tiles   the factor: slot t = L_{J+t,J} (slot 0 unused)
//   LF,LB NT*(PT+1) tiles   solve copies (slot 0 = L_JJ^{-1}) in DMMA fragment
//                           order, forward and transposed (k_coarse_pack)
// Padding rows (>= kc) are identity.
//
// The factorization is one cooperative launch with one grid barrier per tile
// column: after the barrier every CTA takes trailing-update tasks
// (recomputing the panel products it needs, so the panel TRSM costs no extra
// barrier); CTA 0 first takes the task that updates the next diagonal tile
// and then factors it (one-step lookahead).  All tile products are DMMA.
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
};

__host__ __device__ __forceinline__ size_t band_tiles(const Geo& g) { return (size_t)g.NT * (g.PT + 1); }

__host__ __device__ __forceinline__ CoarseBufs coarse_bufs(const Geo& g, double* base) {
  CoarseBufs b;
  b.A = base;
  b.Dinv = b.A + band_tiles(g) * TT;
  b.Lo = b.Dinv + (size_t)g.NT * TT;
  b.LF = b.Lo + band_tiles(g) * TT;
  b.LB = b.LF + band_tiles(g) * TT;
  return b;
}

size_t coarse_doubles(const Geo& g) {
  return 4 * band_tiles(g) * TT + (size_t)g.NT * TT;
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
//
// Tile products run on the FP64 tensor cores (DMMA m8n8k4) in the
// transposed-operand form: with both operands in accumulator (C) layout,
// D += X Y^T (chunk h of k = columns {2k+h}, the layout's slot h), so a 32x32
// tile product O = X Y^T is 16 output 8x8 blocks x 4 k-blocks x 2 DMMAs; warp
// w owns output blocks w and w+8.  Shared tiles use a padded row stride LDT
// (320 bytes) so the 16-byte fragment loads are bank-conflict free.
constexpr int LDT = TB + 8;

struct FactorSmem {
  double T[TB * LDT];      // operand tile (A_{J+t,J}) / diagonal tile under POTRF
  double X1[TB * LDT];     // L_{J+t1,J}
  double X2[TB * LDT];     // L_{J+t2,J}
  double D[TB * LDT];      // Dinv_J
  double Li[4][64];        // POTRF: L_kk^{-1} of the diagonal 8x8 blocks (C layout)
  double Is[64];           // potrf8 output
};

struct F2c {
  double x, y;
};
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}
__device__ __forceinline__ void mxyt(F2c& c, const F2c& x, const F2c& y) {
  dmma(c.x, c.y, x.x, y.x);
  dmma(c.x, c.y, x.y, y.y);
}
// C-layout fragment of 8x8 block (bi, bj) of a tile with row stride ld
__device__ __forceinline__ F2c frag(const double* S, int ld, int bi, int bj, int lane) {
  const double2 v = *reinterpret_cast<const double2*>(S + (8 * bi + (lane >> 2)) * ld + 8 * bj + 2 * (lane & 3));
  return {v.x, v.y};
}
__device__ __forceinline__ void put(double* S, int ld, int bi, int bj, int lane, const F2c& f) {
  *reinterpret_cast<double2*>(S + (8 * bi + (lane >> 2)) * ld + 8 * bj + 2 * (lane & 3)) = make_double2(f.x, f.y);
}
__device__ __forceinline__ void load_tile(double* S, const double* src) {
  for (int t = threadIdx.x; t < TT / 2; t += blockDim.x) {
    const int r = (2 * t) / TB, c = (2 * t) % TB;
    *reinterpret_cast<double2*>(S + r * LDT + c) = *reinterpret_cast<const double2*>(src + 2 * t);
  }
}
__device__ __forceinline__ void store_tile(double* dst, const double* S) {
  for (int t = threadIdx.x; t < TT / 2; t += blockDim.x) {
    const int r = (2 * t) / TB, c = (2 * t) % TB;
    *reinterpret_cast<double2*>(dst + 2 * t) = *reinterpret_cast<const double2*>(S + r * LDT + c);
  }
}
// O = X Y^T (32x32 tiles in shared memory), then op(O block) by the caller
template <class F>
__device__ __forceinline__ void tile_xyt(const double* X, const double* Y, F&& out) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int o = w + 8 * h, bi = o >> 2, bj = o & 3;
    F2c c = {0.0, 0.0}, e = {0.0, 0.0};
#pragma unroll
    for (int kb = 0; kb < 4; kb += 2) {
      mxyt(c, frag(X, LDT, bi, kb, lane), frag(Y, LDT, bj, kb, lane));
      mxyt(e, frag(X, LDT, bi, kb + 1, lane), frag(Y, LDT, bj, kb + 1, lane));
    }
    c.x += e.x;
    c.y += e.y;
    out(bi, bj, c);
  }
}

// Cholesky of one 8x8 SPD block -> L^{-1} (row-major in Is[0..63]).  Every
// lane factors the block redundantly from shared memory (no shuffles on the
// pivot chain: ~2x shorter than a row-per-lane factorization); lanes 0..7
// then form the columns of L^{-1}.
template <int R>
__device__ __forceinline__ void c8_inv(double (&d)[8], int c, const double (&a)[8][8], const double (&inv)[8]) {
  if constexpr (R < 8) {
    double acc = (R == c) ? 1.0 : 0.0;
#pragma unroll
    for (int m = 0; m < R; ++m) acc -= a[R][m] * d[m];
    d[R] = (R < c) ? 0.0 : acc * inv[R];
    c8_inv<R + 1>(d, c, a, inv);
  }
}
__device__ __forceinline__ void potrf_inv8w(const double* S, int ld, double* Is, int lane, int* flags) {
  double a[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j <= i; ++j) a[i][j] = S[i * ld + j];
  double inv[8];
  bool bad = false;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    double d = a[c][c];
    if (!(d > 0.0)) { bad = true; d = 1.0; }
    inv[c] = rsqrt(d);
#pragma unroll
    for (int i = c + 1; i < 8; ++i) a[i][c] *= inv[c];
#pragma unroll
    for (int j = c + 1; j < 8; ++j)
#pragma unroll
      for (int i = j; i < 8; ++i) a[i][j] -= a[i][c] * a[j][c];
  }
  if (bad && lane == 0) atomicOr(flags, FLAG_COARSE_NOT_SPD);
  if (lane < 8) {
    double d[8];
    c8_inv<0>(d, lane, a, inv);
#pragma unroll
    for (int rr = 0; rr < 8; ++rr) Is[rr * 8 + lane] = d[rr];
  }
  __syncwarp();
}

// Blocked Cholesky of the diagonal tile J (in A, full symmetric 32x32) by one
// CTA: four 8x8 diagonal blocks (potrf8 + inverse on warp 0), DMMA panel and
// trailing updates; then Dinv_J = L_JJ^{-1} by block forward substitution in
// transposed form, DT[i][j] = Dinv[i][j]^T = -(sum_k DT[k][j] L[i][k]^T) Li_i^T.
// Writes Dinv_J (row-major) to the factor buffer.
// tile_in_smem: sm.T already holds the (updated) diagonal tile.  Dinv_J is
// also left row-major in sm.D for the caller's next column.
__device__ void coarse_potrf(const Geo& g, int J, const CoarseBufs& B, int* flags, FactorSmem& sm,
                             bool tile_in_smem = false, long long* tprof = nullptr) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  auto stamp = [&](int k) {
    if (tprof && tid == 0) tprof[k] += clock64();
  };
  stamp(0);
  double* P = sm.T;
  if (!tile_in_smem) load_tile(P, tile(B.A, g, J, 0));
  __syncthreads();
  for (int kb = 0; kb < 4; ++kb) {
    if (w == 0) {
      potrf_inv8w(P + 8 * kb * LDT + 8 * kb, LDT, sm.Is, lane, flags);
      const int m = lane >> 2, q = lane & 3;
      sm.Li[kb][2 * lane] = sm.Is[m * 8 + 2 * q];          // L_kk^{-1}, C layout
      sm.Li[kb][2 * lane + 1] = sm.Is[m * 8 + 2 * q + 1];
    }
    __syncthreads();
    stamp(1 + 3 * kb);
    if (w < 3 - kb) {                                      // L[i][kb] = A[i][kb] L_kk^{-T}
      const int i = kb + 1 + w;
      F2c c = {0.0, 0.0};
      const F2c li = {sm.Li[kb][2 * lane], sm.Li[kb][2 * lane + 1]};
      mxyt(c, frag(P, LDT, i, kb, lane), li);
      put(P, LDT, i, kb, lane, c);
    }
    __syncthreads();
    stamp(2 + 3 * kb);
    {                                                      // trailing A[i][j] -= L[i][kb] L[j][kb]^T
      int cnt = 0;
      for (int i = kb + 1; i < 4; ++i)
        for (int j = kb + 1; j <= i; ++j, ++cnt)
          if (cnt == w) {
            F2c c = frag(P, LDT, i, j, lane);
            const F2c a = frag(P, LDT, i, kb, lane), b = frag(P, LDT, j, kb, lane);
            mxyt(c, {-a.x, -a.y}, b);
            put(P, LDT, i, j, lane, c);
          }
    }
    __syncthreads();
    stamp(3 + 3 * kb);
  }
  // Dinv in transposed blocks, held in sm.X2 (block (i,j) C layout of Dinv[i][j]^T)
  double* DT = sm.X2;
  if (w < 4) {                                             // DT[i][i] = Li_i^T
    const int m = lane >> 2, q = lane & 3;
    // C layout of Li^T: lane (m,q) holds Li[2q][m], Li[2q+1][m]; Li row-major is
    // recovered from its C layout: Li[r][c] sits at lane 4r + c/2, slot c%2
    const double* L = sm.Li[w];
    const F2c f = {L[2 * (4 * (2 * q) + m / 2) + (m & 1)], L[2 * (4 * (2 * q + 1) + m / 2) + (m & 1)]};
    put(DT, LDT, w, w, lane, f);
  }
  __syncthreads();
  for (int d = 1; d < 4; ++d) {
    if (w < 4 - d) {
      const int j = w, i = j + d;
      F2c z = {0.0, 0.0};
      for (int k = j; k < i; ++k) mxyt(z, frag(DT, LDT, k, j, lane), frag(P, LDT, i, k, lane));
      F2c o = {0.0, 0.0};
      const F2c li = {sm.Li[i][2 * lane], sm.Li[i][2 * lane + 1]};
      mxyt(o, {-z.x, -z.y}, li);
      put(DT, LDT, i, j, lane, o);
    }
    __syncthreads();
  }
  stamp(13);
  // Dinv row-major: Dinv[8i + 2q (+1)][8j + m] = DT[i][j] slot 0 (1) at lane (m, q)
  double* dst = B.Dinv + (size_t)J * TT;
  for (int o = w; o < 16; o += 8) {
    const int i = o >> 2, j = o & 3, m = lane >> 2, q = lane & 3;
    F2c f = {0.0, 0.0};
    if (j <= i) f = frag(DT, LDT, i, j, lane);
    dst[(8 * i + 2 * q) * TB + 8 * j + m] = f.x;
    dst[(8 * i + 2 * q + 1) * TB + 8 * j + m] = f.y;
    sm.D[(8 * i + 2 * q) * LDT + 8 * j + m] = f.x;
    sm.D[(8 * i + 2 * q + 1) * LDT + 8 * j + m] = f.y;
  }
  __syncthreads();
  stamp(14);
}

// Pair task f of tile column J: trailing tile (t1, t2), t2 <= t1, recomputing
// the panel tiles it needs, L_{J+t,J} = A_{J+t,J} Dinv_J^T (so the panel TRSM
// costs no grid barrier).  sm.D holds Dinv_J.
// diag_to_smem (lookahead pair (1,1)): the updated diagonal tile goes to
// sm.T for the POTRF that follows instead of back to global memory.
__device__ void coarse_task(const Geo& g, int J, int f, const CoarseBufs& B, FactorSmem& sm,
                            bool diag_to_smem = false) {
  const int lane = threadIdx.x & 31;
  int t1 = (int)((1.0 + sqrt(1.0 + 8.0 * f)) * 0.5);
  while (t1 * (t1 - 1) / 2 > f) --t1;
  while ((t1 + 1) * t1 / 2 <= f) ++t1;
  const int t2 = f - t1 * (t1 - 1) / 2 + 1;
  load_tile(sm.T, tile(B.A, g, J, t1));
  __syncthreads();
  tile_xyt(sm.T, sm.D, [&](int bi, int bj, const F2c& c) { put(sm.X1, LDT, bi, bj, lane, c); });
  __syncthreads();
  if (t2 != t1) {
    load_tile(sm.T, tile(B.A, g, J, t2));
    __syncthreads();
    tile_xyt(sm.T, sm.D, [&](int bi, int bj, const F2c& c) { put(sm.X2, LDT, bi, bj, lane, c); });
    __syncthreads();
  } else {
    store_tile(tile(B.Lo, g, J, t1), sm.X1);
  }
  const double* Y = (t2 != t1) ? sm.X2 : sm.X1;
  double* G = tile(B.A, g, J + t2, t1 - t2);
  // G -= X1 Y^T, block by block straight from / to global
  const int wv = threadIdx.x >> 5;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int o = wv + 8 * h, bi = o >> 2, bj = o & 3;
    F2c c = frag(G, TB, bi, bj, lane), e = {0.0, 0.0};
#pragma unroll
    for (int kb = 0; kb < 4; kb += 2) {
      const F2c a = frag(sm.X1, LDT, bi, kb, lane), a2 = frag(sm.X1, LDT, bi, kb + 1, lane);
      mxyt(c, {-a.x, -a.y}, frag(Y, LDT, bj, kb, lane));
      mxyt(e, {-a2.x, -a2.y}, frag(Y, LDT, bj, kb + 1, lane));
    }
    c.x += e.x;
    c.y += e.y;
    if (diag_to_smem)
      put(sm.T, LDT, bi, bj, lane, c);
    else
      put(G, TB, bi, bj, lane, c);
  }
  __syncthreads();
}

__global__ void __launch_bounds__(256, 1) k_coarse_factor(Geo g, double* __restrict__ base, int* __restrict__ flags) {
  __shared__ __align__(16) FactorSmem sm;
  cg::grid_group grid = cg::this_grid();
  const CoarseBufs B = coarse_bufs(g, base);
  if (blockIdx.x == 0) coarse_potrf(g, 0, B, flags, sm);
  grid.sync();
  for (int J = 0; J < g.NT; ++J) {
    const int pt = min(g.PT, g.NT - 1 - J);
    const int npairs = pt * (pt + 1) / 2;
    if (blockIdx.x != 0) load_tile(sm.D, B.Dinv + (size_t)J * TT);   // CTA 0 kept it from its POTRF
    __syncthreads();
    if (blockIdx.x == 0 && pt >= 1) {
      coarse_task(g, J, 0, B, sm, true);         // pair (1,1): next diagonal tile, into sm.T
      coarse_potrf(g, J + 1, B, flags, sm, true);  // lookahead factor of column J+1
    }
    // the other CTAs share everything except the lookahead pair
    const int first = (pt >= 1) ? 1 : 0;
    const int nw = gridDim.x > 1 ? gridDim.x - 1 : 1;
    if (gridDim.x == 1 || blockIdx.x > 0) {
      const int me = gridDim.x > 1 ? blockIdx.x - 1 : 0;
      for (int f = first + me; f < npairs; f += nw) coarse_task(g, J, f, B, sm);
    }
    grid.sync();
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
                                                          int nrhs, int CHT, int NS, long long* tprof = nullptr) {
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
    long long tclk = 0, tw = 0;
    if (tprof && tid == 0) tclk = clock64();
    mbar_wait(&bar[st], (par >> st) & 1u);
    par ^= 1u << st;
    if (tprof && tid == 0) {
      tw = clock64();
      tprof[i < nf ? 0 : 3] += tw - tclk;
    }
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
        if (tprof && tid == 0) tprof[1] += clock64() - tw;
      }
      const int ta = max(t0, 1), tb = min(t1, pt);
      {
        // each warp owns pieces wid, wid+8, ...: up to UP of them run as
        // independent DMMA chains (kb outermost) so the chains overlap
        constexpr int UP = 5;
        double ny[4][2];
#pragma unroll
        for (int kb = 0; kb < 4; ++kb) {
          ny[kb][0] = -Ys[kb * 64 + 2 * lane];
          ny[kb][1] = -Ys[kb * 64 + 2 * lane + 1];
        }
        const int np = (tb - ta + 1) * 4;
        for (int p0 = wid; p0 < np; p0 += 8 * UP) {
          double acc[UP][2];
          double* ap[UP];
          const double* tp[UP];
#pragma unroll
          for (int q = 0; q < UP; ++q) {
            const int p = p0 + 8 * q;
            const bool v = p < np;
            const int t = ta + (v ? (p >> 2) : 0), mi = p & 3;
            ap[q] = Rt + (size_t)(ring(jm, t) * 4 + mi) * 64 + 2 * lane;
            tp[q] = T + (size_t)(t - t0) * TT + mi * 4 * 64 + 2 * lane;
            acc[q][0] = v ? ap[q][0] : 0.0;
            acc[q][1] = v ? ap[q][1] : 0.0;
          }
#pragma unroll
          for (int kb = 0; kb < 4; ++kb)
#pragma unroll
            for (int q = 0; q < UP; ++q)
              if (p0 + 8 * q < np) mma_xyt(acc[q][0], acc[q][1], ny[kb][0], ny[kb][1], tp[q][kb * 64], tp[q][kb * 64 + 1]);
#pragma unroll
          for (int q = 0; q < UP; ++q)
            if (p0 + 8 * q < np) {
              ap[q][0] = acc[q][0];
              ap[q][1] = acc[q][1];
            }
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
        // up to UB tiles of this warp's parity as independent DMMA chains
        constexpr int UB = 3;
        double e0 = 0.0, e1 = 0.0;
        const int tstart = ta + ((ta & 1) != half ? 1 : 0);
        for (int tq = tstart; tq <= tb; tq += 2 * UB) {
          double ac[UB][2];
          const double* xp[UB];
          const double* yp[UB];
#pragma unroll
          for (int q = 0; q < UB; ++q) {
            const int t = min(tq + 2 * q, tb);
            xp[q] = Rt + (size_t)ring(jm, t) * 256 + 2 * lane;
            yp[q] = T + (size_t)(t - t0) * TT + nb * 4 * 64 + 2 * lane;
            ac[q][0] = ac[q][1] = 0.0;
          }
#pragma unroll
          for (int kb = 0; kb < 4; ++kb)
#pragma unroll
            for (int q = 0; q < UB; ++q)
              if (tq + 2 * q <= tb)
                mma_xyt(ac[q][0], ac[q][1], xp[q][kb * 64], xp[q][kb * 64 + 1], yp[q][kb * 64], yp[q][kb * 64 + 1]);
#pragma unroll
          for (int q = 0; q < UB; ++q) {
            e0 += ac[q][0];
            e1 += ac[q][1];
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
    if (tprof && tid == 0) tprof[i < nf ? 2 : 5] += clock64() - tclk;
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
  size_t smem = ((size_t)4 * TT + ((size_t)g.PT + 2) * TB * RC) * sizeof(double);
  cudaError_t e = cudaFuncSetAttribute(k_coarse_trsv<RC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k_coarse_trsv<RC><<<nblk(nrhs, RC), 256, smem, st>>>(g, B.Lo, B.Dinv, X, nrhs);
  count_launches(1);
  return cudaGetLastError();
}

}  // namespace msfv
