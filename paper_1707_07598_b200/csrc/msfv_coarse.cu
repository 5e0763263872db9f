// Coarse (Galerkin) system: assembly of A_k = P^T A P from the per-block 8x8
// contributions, its Cholesky factorization and the coarse solves.
//
// Reference: forward.py:101-142 forms A_k densely and calls LAPACK dpotrf
// (cho_factor) for k <= 5000, SuperLU above.  A_k couples coarse nodes only
// within a 27-point stencil, so in lexicographic coarse order its half
// bandwidth is pc = (nb1+1)(nb2+1) + (nb1+1) + 1 and Cholesky fill stays
// inside that band: the banded factorization below is the Cholesky factor of
// the (permuted) matrix, computed without the zero blocks.
//
// Nested dissection by coarse z-planes (coarse_nd): the middle plane zs is a
// separator C; the planes below (part 0, natural order) and above (part 1,
// planes in reverse order so the plane next to C comes last) are independent
// banded systems factored concurrently, half the sequential depth of the
// single band.  With L_q the part factors, the coupling blocks are
// Z_q = L_q^{-1} A_{q,C} (non-zero only from the part's last plane on, since
// A_{q,C} couples C to that plane), the separator Schur complement is
// S = A_CC - Z_0^T Z_0 - Z_1^T Z_1 (dense P x P, P = plane size), factored as a
// dense band.  Solves: forward sweeps on both parts, x_C -= Z^T y, full
// separator solve, y -= Z x_C, backward sweeps.  Without coarse_nd the whole
// system is one band (b[0]).
//
// Per band (one allocation, see coarse_layout):
//   A     NT*(PT+1) tiles   lower band; tile column J holds (J+t, J), t = 0..PT,
//                           each TB x TB row-major.  Updated in place.
//   Dinv  NT tiles          L_JJ^{-1}
//   Lo    NT*(PT+1) tiles   the factor: slot t = L_{J+t,J} (slot 0 unused)
//   LF,LB NT*(PT+1) tiles   solve copies (slot 0 = L_JJ^{-1}) in DMMA fragment
//                           order, forward and transposed (k_coarse_pack)
//   SF,SB NT*(PT+1) tiles   block-row-scaled solve copies for the cluster
//                           sweeps (k_coarse_pack_scaled): SF[J][t] =
//                           Dinv_{J+t} L_{J+t,J}, SB[J][t] = Dinv_{J-t}^T
//                           L_{J,J-t}^T, slot 0 = Dinv_J / Dinv_J^T
// Padding rows (>= n) are identity.
//
// The band factorization is one cooperative launch with one grid barrier per
// tile column (both parts advance together): every CTA takes trailing-update
// tasks (recomputing the panel products it needs, so the panel TRSM costs no
// extra barrier); CTA b first takes the task that updates band b's next
// diagonal tile and then factors it (one-step lookahead).  All tile products
// are DMMA.
#include <cooperative_groups.h>

#include <algorithm>
#include <array>
#include <vector>
#include <cstdio>
#include <cstdlib>
#include <climits>

#include "msfv_common.cuh"
#include "msfv_kernels.h"

namespace cg = cooperative_groups;

namespace msfv {

constexpr int TB = COARSE_TB;
constexpr int TT = TB * TB;

struct Band {
  double* A;
  double* Dinv;
  double* Lo;
  double* LF;
  double* LB;
  double* SF;   // scaled solve copies for the cluster sweeps (k_coarse_pack_scaled)
  double* SB;
  int n;        // valid rows
  int NT, PT;   // tile rows, band tiles
};

struct Coarse {
  int nd;               // 1: z-plane nested dissection, 0: one band
  int P, zs, planes;    // coarse plane size, separator plane, planes
  int nb;               // bands in use (1 or 3)
  Band b[3];            // part 0, part 1, separator (b[0] = whole system when !nd)
  int J0[2];            // first tile row of each part's last plane
  double* Z[2];         // rows [J0*TB, NT*TB) of Z_q, row-major, P columns
  size_t total;         // doubles
};

__host__ __device__ __forceinline__ Band make_band(double* base, size_t& off, int n, int ptcap) {
  Band B;
  B.n = n;
  B.NT = (n + TB - 1) / TB;
  B.PT = ptcap < B.NT - 1 ? ptcap : B.NT - 1;
  const size_t bt = (size_t)B.NT * (B.PT + 1) * TT;
  B.A = base ? base + off : nullptr;        off += bt;
  B.Dinv = base ? base + off : nullptr;     off += (size_t)B.NT * TT;
  B.Lo = base ? base + off : nullptr;       off += bt;
  B.LF = base ? base + off : nullptr;       off += bt;
  B.LB = base ? base + off : nullptr;       off += bt;
  B.SF = base ? base + off : nullptr;       off += bt;
  B.SB = base ? base + off : nullptr;       off += bt;
  return B;
}

__host__ __device__ __forceinline__ Coarse coarse_layout(const Geo& g, double* base) {
  Coarse L{};
  L.P = (g.nb1 + 1) * (g.nb2 + 1);
  L.planes = g.nb3 + 1;
  L.nd = g.coarse_nd != 0 && L.planes >= 3;
  const int ptcap = (g.pc + TB - 1) / TB;
  size_t off = 0;
  if (!L.nd) {
    L.nb = 1;
    L.b[0] = make_band(base, off, g.kc, ptcap);
    L.total = off;
    return L;
  }
  L.nb = 3;
  L.zs = (L.planes - 1) / 2;
  const int n0 = L.zs * L.P, n1 = (L.planes - 1 - L.zs) * L.P;
  L.b[0] = make_band(base, off, n0, ptcap);
  L.b[1] = make_band(base, off, n1, ptcap);
  L.b[2] = make_band(base, off, L.P, INT_MAX);
  for (int q = 0; q < 2; ++q) {
    L.J0[q] = (L.b[q].n - L.P) / TB;
    L.Z[q] = base ? base + off : nullptr;
    off += (size_t)(L.b[q].NT - L.J0[q]) * TB * L.P;
  }
  L.total = off;
  return L;
}

__device__ __forceinline__ double* btile(double* A, const Band& B, int J, int t) {
  return A + ((size_t)J * (B.PT + 1) + t) * TT;
}
__device__ __forceinline__ const double* btile(const double* A, const Band& B, int J, int t) {
  return A + ((size_t)J * (B.PT + 1) + t) * TT;
}

// natural coarse index -> (band, local row)
__device__ __forceinline__ void coarse_map(const Coarse& L, int c, int& part, int& local) {
  if (!L.nd) {
    part = 0;
    local = c;
    return;
  }
  const int ck = c / L.P, w = c - ck * L.P;
  if (ck < L.zs) { part = 0; local = c; }
  else if (ck > L.zs) { part = 1; local = (L.planes - 1 - ck) * L.P + w; }
  else { part = 2; local = w; }
}

size_t mf_doubles(const Geo& g);
int mf_tile_rows(const Geo& g);
size_t coarse_doubles(const Geo& g) { return g.coarse_nd == 2 ? mf_doubles(g) : coarse_layout(g, nullptr).total; }
size_t coarse_scratch_doubles(const Geo& g, int nrhs) {
  if (g.coarse_nd == 2) return (size_t)mf_tile_rows(g) * TB * nrhs;   // mf_tile_rows already counts Vin + Vout
  const Coarse L = coarse_layout(g, nullptr);
  size_t rows = 0;
  for (int b = 0; b < L.nb; ++b) rows += (size_t)L.b[b].NT * TB;
  return rows * nrhs;
}
int coarse_tile_rows(const Geo& g) {
  if (g.coarse_nd == 2) return mf_tile_rows(g);
  const Coarse L = coarse_layout(g, nullptr);
  int r = 0;
  for (int b = 0; b < L.nb; ++b) r += L.b[b].NT;
  return r;
}

// A_k[c][c2] for the o-th lexicographically lower stencil neighbour c2 of c:
// sum over blocks having both as corners (fixed order) of Kloc, + shift on the
// diagonal.  Returns false when the neighbour is outside the grid.
__device__ __forceinline__ bool coarse_entry(const Geo& g, const double* __restrict__ Kloc, double shift, int c, int o,
                                             int& c2, double& v) {
  int dz, dy, dx;
  if (o < 9) { dz = -1; dy = o / 3 - 1; dx = o % 3 - 1; }
  else if (o < 12) { dz = 0; dy = -1; dx = (o - 9) - 1; }
  else { dz = 0; dy = 0; dx = (o - 12) - 1; }
  const int ci = c % (g.nb1 + 1), r = c / (g.nb1 + 1), cj = r % (g.nb2 + 1), ck = r / (g.nb2 + 1);
  const int di = ci + dx, dj = cj + dy, dk = ck + dz;
  if (di < 0 || dj < 0 || dk < 0 || di > g.nb1 || dj > g.nb2 || dk > g.nb3) return false;
  c2 = coarse_of(g, di, dj, dk);
  v = 0.0;
  for (int bk = max(ck, dk) - 1; bk <= min(ck, dk); ++bk) {
    if (bk < 0 || bk >= g.nb3) continue;
    for (int bj = max(cj, dj) - 1; bj <= min(cj, dj); ++bj) {
      if (bj < 0 || bj >= g.nb2) continue;
      for (int bi = max(ci, di) - 1; bi <= min(ci, di); ++bi) {
        if (bi < 0 || bi >= g.nb1) continue;
        const int l1 = (ci - bi) + 2 * (cj - bj) + 4 * (ck - bk);
        const int l2 = (di - bi) + 2 * (dj - bj) + 4 * (dk - bk);
        v += Kloc[(size_t)block_of(g, bi, bj, bk) * 64 + l1 * 8 + l2];
      }
    }
  }
  if (c2 == c) v += shift;
  return true;
}

// Thread per (coarse row c, lower neighbour o); scatters into the permuted bands
// and coupling blocks.  Then padding rows of every band get identity.
__global__ void k_coarse_assemble(Geo g, Coarse L, const double* __restrict__ Kloc, double shift) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long main = (long long)g.kc * 14;
  if (t >= main) {
    const long long u = t - main;              // padding: band u / TB, row n + u % TB
    const int b = (int)(u / TB), r = (int)(u % TB);
    if (b < L.nb) {
      const Band& B = L.b[b];
      const int row = B.n + r;
      if (row < B.NT * TB) btile(B.A, B, row / TB, 0)[(row % TB) * (TB + 1)] = 1.0;
    }
    return;
  }
  const int o = (int)(t % 14), c = (int)(t / 14);
  int c2;
  double v;
  if (!coarse_entry(g, Kloc, shift, c, o, c2, v)) return;
  int p1, l1, p2, l2;
  coarse_map(L, c, p1, l1);
  coarse_map(L, c2, p2, l2);
  if (p1 == p2) {
    const Band& B = L.b[p1];
    const int r = max(l1, l2), s = min(l1, l2);
    btile(B.A, B, s / TB, r / TB - s / TB)[(r % TB) * TB + (s % TB)] = v;
  } else {
    // part q node lr (in its last plane) couples to separator node ls
    const int q = p1 == 2 ? p2 : p1, lr = p1 == 2 ? l2 : l1, ls = p1 == 2 ? l1 : l2;
    L.Z[q][(size_t)(lr - L.J0[q] * TB) * L.P + ls] = v;
  }
}

__global__ void k_coarse_diag(Geo g, Coarse L, double* __restrict__ diag) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= g.kc) return;
  int p, l;
  coarse_map(L, c, p, l);
  const Band& B = L.b[p];
  diag[c] = btile(B.A, B, l / TB, 0)[(l % TB) * (TB + 1)];
}

// Dense natural-order A_k (both triangles), for the host-side `A_k` attribute.
__global__ void k_coarse_dense(Geo g, const double* __restrict__ Kloc, double shift, double* __restrict__ out) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= (long long)g.kc * 14) return;
  const int o = (int)(t % 14), c = (int)(t / 14);
  int c2;
  double v;
  if (!coarse_entry(g, Kloc, shift, c, o, c2, v)) return;
  out[(size_t)c * g.kc + c2] = v;
  out[(size_t)c2 * g.kc + c] = v;
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
// 1/sqrt(d) for a positive normal d: MUFU seed and one cubic Newton-type
// step (relative error ~2^-60 before rounding), no special-case branches --
// the pivot chain of the 32x32 POTRF is the critical path of every tile column
__device__ __forceinline__ double rsq_seeded(double d) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
  const double e = fma(-d * y, y, 1.0);
  const double t = fma(0.375, e, 0.5);
  return fma(y * e, t, y);
}
__device__ __forceinline__ void potrf_inv8w(const double* S, int ld, double* Is, int lane, int* flags) {
  double a[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j <= i; ++j) a[i][j] = S[i * ld + j];
  // column ci of L^{-1} rides along the pivots (right-looking forward
  // substitution of e_ci: independent of the trailing update, so it adds no
  // latency to the pivot chain)
  const int ci = lane & 7;
  double acc[8], dc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = i == ci ? 1.0 : 0.0;
  bool bad = false;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    double d = a[c][c];
    if (!(d > 0.0)) { bad = true; d = 1.0; }
    const double inv = rsq_seeded(d);
#pragma unroll
    for (int i = c + 1; i < 8; ++i) a[i][c] *= inv;
#pragma unroll
    for (int j = c + 1; j < 8; ++j)
#pragma unroll
      for (int i = j; i < 8; ++i) a[i][j] -= a[i][c] * a[j][c];
    dc[c] = acc[c] * inv;
#pragma unroll
    for (int i = c + 1; i < 8; ++i) acc[i] = fma(-a[i][c], dc[c], acc[i]);
  }
  if (bad && lane == 0) atomicOr(flags, FLAG_COARSE_NOT_SPD);
  if (lane < 8) {
#pragma unroll
    for (int rr = 0; rr < 8; ++rr) Is[rr * 8 + lane] = dc[rr];
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
__device__ void coarse_potrf(const Band& B, int J, int* flags, FactorSmem& sm,
                             bool tile_in_smem = false, long long* tprof = nullptr) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  auto stamp = [&](int k) {
    if (tprof && tid == 0) tprof[k] += clock64();
  };
  stamp(0);
  double* P = sm.T;
  if (!tile_in_smem) load_tile(P, btile(B.A, B, J, 0));
  __syncthreads();
  // The whole chain runs on warp 0 (warp barriers only): four 8x8 POTRF +
  // inverse steps, each followed by its panel and trailing DMMA updates, then
  // Dinv in transposed blocks (sm.X2, block (i,j) = C layout of Dinv[i][j]^T):
  // DT[i][j] = -(sum_k DT[k][j] L[i][k]^T) Li_i^T.
  double* DT = sm.X2;
  if (w == 0) {
    const int m = lane >> 2, q = lane & 3;
#pragma unroll
    for (int kb = 0; kb < 4; ++kb) {
      potrf_inv8w(P + 8 * kb * LDT + 8 * kb, LDT, sm.Is, lane, flags);
      const F2c li = {sm.Is[m * 8 + 2 * q], sm.Is[m * 8 + 2 * q + 1]};     // L_kk^{-1}, C layout
      sm.Li[kb][2 * lane] = li.x;
      sm.Li[kb][2 * lane + 1] = li.y;
      stamp(1 + 3 * kb);
      // panel L[i][kb] = A[i][kb] L_kk^{-T} and trailing A[i][j] -= L[i][kb] L[j][kb]^T,
      // all operands loaded before any store (independent DMMA chains)
      F2c pl[4], tr[4][4];
#pragma unroll
      for (int i = kb + 1; i < 4; ++i) {
        pl[i] = frag(P, LDT, i, kb, lane);
#pragma unroll
        for (int j = kb + 1; j <= i; ++j) tr[i][j] = frag(P, LDT, i, j, lane);
      }
#pragma unroll
      for (int i = kb + 1; i < 4; ++i) {
        F2c c = {0.0, 0.0};
        mxyt(c, pl[i], li);
        pl[i] = c;
      }
#pragma unroll
      for (int i = kb + 1; i < 4; ++i)
#pragma unroll
        for (int j = kb + 1; j <= i; ++j) mxyt(tr[i][j], {-pl[i].x, -pl[i].y}, pl[j]);
#pragma unroll
      for (int i = kb + 1; i < 4; ++i) {
        put(P, LDT, i, kb, lane, pl[i]);
#pragma unroll
        for (int j = kb + 1; j <= i; ++j) put(P, LDT, i, j, lane, tr[i][j]);
      }
      __syncwarp();
      stamp(3 + 3 * kb);
    }
    for (int i = 0; i < 4; ++i) {                          // DT[i][i] = Li_i^T
      // C layout of Li^T: lane (m,q) holds Li[2q][m], Li[2q+1][m]; Li[r][c] sits
      // at lane 4r + c/2, slot c%2 of its C layout
      const double* L = sm.Li[i];
      const F2c f = {L[2 * (4 * (2 * q) + m / 2) + (m & 1)], L[2 * (4 * (2 * q + 1) + m / 2) + (m & 1)]};
      put(DT, LDT, i, i, lane, f);
    }
    __syncwarp();
    // block forward substitution by diagonals; Li and L blocks in registers
    F2c lb[4][4], dt[4][4], lid[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      lid[i] = {sm.Li[i][2 * lane], sm.Li[i][2 * lane + 1]};
#pragma unroll
      for (int k = 0; k < i; ++k) lb[i][k] = frag(P, LDT, i, k, lane);
      dt[i][i] = frag(DT, LDT, i, i, lane);
    }
#pragma unroll
    for (int d = 1; d < 4; ++d)
#pragma unroll
      for (int j = 0; j + d < 4; ++j) {
        const int i = j + d;
        F2c z = {0.0, 0.0};
#pragma unroll
        for (int k = j; k < i; ++k) mxyt(z, dt[k][j], lb[i][k]);
        F2c o = {0.0, 0.0};
        mxyt(o, {-z.x, -z.y}, lid[i]);
        dt[i][j] = o;
      }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < i; ++j) put(DT, LDT, i, j, lane, dt[i][j]);
  }
  __syncthreads();
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

// Pair task of tile column J: trailing tile (t1, t2), t2 <= t1, recomputing
// the panel tiles it needs, L_{J+t,J} = A_{J+t,J} Dinv_J^T (so the panel TRSM
// costs no grid barrier).  sm.D holds Dinv_J.  The two panel tiles and the
// target tile's fragments are read together (one L2 round trip per task).
// (The lookahead pair (1,1) is coarse_chain_task.)
__device__ void coarse_pair(const Band& B, int J, int t1, int t2, FactorSmem& sm) {
  const int lane = threadIdx.x & 31, wv = threadIdx.x >> 5;
  double* G = btile(B.A, B, J + t2, t1 - t2);
  F2c c[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int o = wv + 8 * h;
    c[h] = frag(G, TB, o >> 2, o & 3, lane);
  }
  load_tile(sm.T, btile(B.A, B, J, t1));
  if (t2 != t1) load_tile(sm.X2, btile(B.A, B, J, t2));
  __syncthreads();
  tile_xyt(sm.T, sm.D, [&](int bi, int bj, const F2c& v) { put(sm.X1, LDT, bi, bj, lane, v); });
  __syncthreads();
  if (t2 != t1) {
    tile_xyt(sm.X2, sm.D, [&](int bi, int bj, const F2c& v) { put(sm.T, LDT, bi, bj, lane, v); });
    __syncthreads();
  } else {
    store_tile(btile(B.Lo, B, J, t1), sm.X1);
  }
  const double* Y = (t2 != t1) ? sm.T : sm.X1;
  // G -= X1 Y^T, block by block
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int o = wv + 8 * h, bi = o >> 2, bj = o & 3;
    F2c e = {0.0, 0.0};
#pragma unroll
    for (int kb = 0; kb < 4; kb += 2) {
      const F2c a = frag(sm.X1, LDT, bi, kb, lane), a2 = frag(sm.X1, LDT, bi, kb + 1, lane);
      mxyt(c[h], {-a.x, -a.y}, frag(Y, LDT, bj, kb, lane));
      mxyt(e, {-a2.x, -a2.y}, frag(Y, LDT, bj, kb + 1, lane));
    }
    c[h].x += e.x;
    c[h].y += e.y;
    put(G, TB, bi, bj, lane, c[h]);
  }
  __syncthreads();
}
// pair f of the band enumeration: f = t1 (t1 - 1) / 2 + t2 - 1
__device__ void coarse_task(const Band& B, int J, int f, FactorSmem& sm) {
  int t1 = (int)((1.0 + sqrt(1.0 + 8.0 * f)) * 0.5);
  while (t1 * (t1 - 1) / 2 > f) --t1;
  while ((t1 + 1) * t1 / 2 <= f) ++t1;
  coarse_pair(B, J, t1, f - t1 * (t1 - 1) / 2 + 1, sm);
}
// Panel tile only: L_{J+t1,J} = A_{J+t1,J} Dinv_J^T to Lo (rows whose trailing
// updates are deferred, see k_mf_factor).
__device__ void coarse_panel_only(const Band& B, int J, int t1, FactorSmem& sm) {
  const int lane = threadIdx.x & 31;
  load_tile(sm.T, btile(B.A, B, J, t1));
  __syncthreads();
  tile_xyt(sm.T, sm.D, [&](int bi, int bj, const F2c& v) { put(sm.X1, LDT, bi, bj, lane, v); });
  __syncthreads();
  store_tile(btile(B.Lo, B, J, t1), sm.X1);
  __syncthreads();
}
// Deferred update of tile (R, C), both beyond the NE eliminated tile columns:
// A_{R,C} -= sum_{J < NE} L_{R,J} L_{C,J}^T from the stored factor tiles.
__device__ void coarse_deferred(const Band& B, int NE, int R, int C, FactorSmem& sm) {
  const int lane = threadIdx.x & 31, wv = threadIdx.x >> 5;
  double* G = btile(B.A, B, C, R - C);
  F2c c[2], e[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int o = wv + 8 * h;
    c[h] = frag(G, TB, o >> 2, o & 3, lane);
    e[h] = {0.0, 0.0};
  }
  for (int J = 0; J < NE; ++J) {
    double* X = (J & 1) ? sm.T : sm.X1;       // two (X, Y) buffer pairs: the next loads overlap this product
    double* Y = (J & 1) ? sm.D : sm.X2;
    load_tile(X, btile(B.Lo, B, J, R - J));
    if (R != C) load_tile(Y, btile(B.Lo, B, J, C - J));
    __syncthreads();
    const double* Yr = R != C ? Y : X;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int o = wv + 8 * h, bi = o >> 2, bj = o & 3;
#pragma unroll
      for (int kb = 0; kb < 4; kb += 2) {
        const F2c a = frag(X, LDT, bi, kb, lane), a2 = frag(X, LDT, bi, kb + 1, lane);
        mxyt(c[h], {-a.x, -a.y}, frag(Yr, LDT, bj, kb, lane));
        mxyt(e[h], {-a2.x, -a2.y}, frag(Yr, LDT, bj, kb + 1, lane));
      }
    }
  }
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int o = wv + 8 * h;
    c[h].x += e[h].x;
    c[h].y += e[h].y;
    put(G, TB, o >> 2, o & 3, lane, c[h]);
  }
  __syncthreads();
}

// Lookahead pair (1,1) of tile column J on the chain CTA (sm.D holds Dinv_J):
// L_{J+1,J} = A_{J+1,J} Dinv_J^T goes to Lo, the updated next diagonal tile to
// sm.T for the POTRF that follows.  Both global reads (the panel tile and the
// diagonal tile's fragments) are in flight together: one L2 round trip on
// the critical path of the tile column instead of two.
__device__ void coarse_chain_task(const Band& B, int J, FactorSmem& sm) {
  const int lane = threadIdx.x & 31, wv = threadIdx.x >> 5;
  const double* G = btile(B.A, B, J + 1, 0);
  F2c c[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int o = wv + 8 * h;
    c[h] = frag(G, TB, o >> 2, o & 3, lane);
  }
  load_tile(sm.T, btile(B.A, B, J, 1));
  __syncthreads();
  tile_xyt(sm.T, sm.D, [&](int bi, int bj, const F2c& v) { put(sm.X1, LDT, bi, bj, lane, v); });
  __syncthreads();
  store_tile(btile(B.Lo, B, J, 1), sm.X1);
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int o = wv + 8 * h, bi = o >> 2, bj = o & 3;
    F2c e = {0.0, 0.0};
#pragma unroll
    for (int kb = 0; kb < 4; kb += 2) {
      const F2c a = frag(sm.X1, LDT, bi, kb, lane), a2 = frag(sm.X1, LDT, bi, kb + 1, lane);
      mxyt(c[h], {-a.x, -a.y}, frag(sm.X1, LDT, bj, kb, lane));
      mxyt(e, {-a2.x, -a2.y}, frag(sm.X1, LDT, bj, kb + 1, lane));
    }
    c[h].x += e.x;
    c[h].y += e.y;
    put(sm.T, LDT, bi, bj, lane, c[h]);
  }
  __syncthreads();
}

// One cooperative launch factors up to two independent bands in lockstep
// (one grid barrier per tile column).
struct FactorJob {
  Band b[2];
  int nb;
};

__global__ void __launch_bounds__(256, 1) k_coarse_factor(FactorJob job, int* __restrict__ flags) {
  __shared__ __align__(16) FactorSmem sm;
  cg::grid_group grid = cg::this_grid();
  const int nb = job.nb;
  const int mine = blockIdx.x < nb ? (int)blockIdx.x : -1;        // lookahead band of this CTA
  if (mine >= 0) coarse_potrf(mine ? job.b[1] : job.b[0], 0, flags, sm);
  grid.sync();
  int ntmax = 0;
  for (int b = 0; b < nb; ++b) ntmax = max(ntmax, job.b[b].NT);
  const int nw = (int)gridDim.x - nb > 0 ? (int)gridDim.x - nb : (int)gridDim.x;
  const int me = (int)gridDim.x - nb > 0 ? (int)blockIdx.x - nb : (int)blockIdx.x;
  for (int J = 0; J < ntmax; ++J) {
    if (mine >= 0) {
      const Band B = mine ? job.b[1] : job.b[0];
      if (J < B.NT - 1) {
        coarse_chain_task(B, J, sm);              // pair (1,1): next diagonal tile, into sm.T
        coarse_potrf(B, J + 1, flags, sm, true);  // lookahead factor of column J+1 (keeps Dinv in sm.D)
      }
    }
    if (me >= 0) {
      // trailing tasks of all bands (minus each band's lookahead pair) in one index space
      int first[2] = {0, 0}, ntask[2] = {0, 0};
      for (int b = 0; b < nb; ++b) {
        const Band& B = job.b[b];
        const int pt = J < B.NT ? min(B.PT, B.NT - 1 - J) : 0;
        first[b] = pt >= 1 ? 1 : 0;
        ntask[b] = pt * (pt + 1) / 2 - first[b];
      }
      int loaded = -1;
      for (int gi = me; gi < ntask[0] + ntask[1]; gi += nw) {
        const int b = gi < ntask[0] ? 0 : 1;
        const int f = gi - (b ? ntask[0] : 0);
        const Band B = b ? job.b[1] : job.b[0];
        if (loaded != b) {
          load_tile(sm.D, B.Dinv + (size_t)J * TT);
          __syncthreads();
          loaded = b;
        }
        coarse_task(B, J, first[b] + f, sm);
      }
    }
    grid.sync();
  }
}

// S_CC -= sum_q Z_q^T Z_q on the separator band (dense), CTA per lower 32x32
// tile.  DMMA in the transposed-operand form, D[i][j] += sum_r Z[r][i] Z[r][j]:
// warp w takes the 8-row chunks w, w+8, ... of both parts for all 16 output
// blocks of the tile (4 X and 4 Y fragments per chunk feed 16 MMA pairs);
// the 8 warp partials are summed in a fixed order through shared memory.
__global__ void __launch_bounds__(256) k_schur_update(Coarse L) {
  extern __shared__ __align__(16) double red[];   // [8 warps][16 blocks][64]
  const Band& C = L.b[2];
  int I = 0, K = blockIdx.x;                      // blockIdx -> lower tile (I, K), I >= K
  while (K > I) { K -= I + 1; ++I; }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, m = lane >> 2, q = lane & 3;
  double acc[16][2];
#pragma unroll
  for (int o = 0; o < 16; ++o) acc[o][0] = acc[o][1] = 0.0;
  const int nc0 = (L.b[0].NT - L.J0[0]) * TB / 8, nc1 = (L.b[1].NT - L.J0[1]) * TB / 8;
  for (int ch = w; ch < nc0 + nc1; ch += 8) {
    const int p = ch < nc0 ? 0 : 1;
    const double* Z = L.Z[p] + (size_t)(8 * (ch - (p ? nc0 : 0)) + 2 * q) * L.P;
    double x[4][2], y[4][2];
#pragma unroll
    for (int bb = 0; bb < 4; ++bb) {
      const int i = I * TB + 8 * bb + m, j = K * TB + 8 * bb + m;
      x[bb][0] = i < L.P ? Z[i] : 0.0;
      x[bb][1] = i < L.P ? Z[L.P + i] : 0.0;
      y[bb][0] = j < L.P ? Z[j] : 0.0;
      y[bb][1] = j < L.P ? Z[L.P + j] : 0.0;
    }
#pragma unroll
    for (int o = 0; o < 16; ++o) {
      dmma(acc[o][0], acc[o][1], x[o >> 2][0], y[o & 3][0]);
      dmma(acc[o][0], acc[o][1], x[o >> 2][1], y[o & 3][1]);
    }
  }
#pragma unroll
  for (int o = 0; o < 16; ++o) {
    red[(w * 16 + o) * 64 + 2 * lane] = acc[o][0];
    red[(w * 16 + o) * 64 + 2 * lane + 1] = acc[o][1];
  }
  __syncthreads();
  double* G = btile(C.A, C, K, I - K);
  for (int e = threadIdx.x; e < 16 * 64; e += blockDim.x) {
    const int o = e >> 6, idx = e & 63, ln = idx >> 1, sl = idx & 1;
    double v = 0.0;
#pragma unroll
    for (int ww = 0; ww < 8; ++ww) v += red[(ww * 16 + o) * 64 + idx];
    const int bi = o >> 2, bj = o & 3, mm = ln >> 2, qq = ln & 3;
    G[(8 * bi + mm) * TB + 8 * bj + 2 * qq + sl] -= v;
  }
}

// x_C[ls][s] -= sum_q sum_r Z_q[r][ls] y_q[J0_q*TB + r][s]: CTA per 8 separator
// rows x 8 sources, 8 warps over the 8-row chunks of both parts (DMMA,
// D[ls][s] += sum_r Z[r][ls] y[r][s]), fixed-order warp reduction.
__global__ void __launch_bounds__(256) k_schur_rhs(Coarse L, const double* __restrict__ y0,
                                                   const double* __restrict__ y1, double* __restrict__ xc, int nrhs) {
  __shared__ double red[8][64];
  const int ls0 = blockIdx.x * 8, s0 = blockIdx.y * 8;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, m = lane >> 2, q = lane & 3;
  const int nc0 = (L.b[0].NT - L.J0[0]) * TB / 8, nc1 = (L.b[1].NT - L.J0[1]) * TB / 8;
  const int ls = ls0 + m, s = s0 + m;
  double c[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
  int u = 0;
  for (int ch = w; ch < nc0 + nc1; ch += 8, u ^= 1) {
    const int p = ch < nc0 ? 0 : 1;
    const int r = 8 * (ch - (p ? nc0 : 0)) + 2 * q;
    const double* Z = L.Z[p] + (size_t)r * L.P;
    const double* y = (p == 0 ? y0 : y1) + ((size_t)L.J0[p] * TB + r) * nrhs;
    const double x0 = ls < L.P ? Z[ls] : 0.0, x1 = ls < L.P ? Z[L.P + ls] : 0.0;
    const double v0 = s < nrhs ? y[s] : 0.0, v1 = s < nrhs ? y[nrhs + s] : 0.0;
    dmma(c[u][0], c[u][1], x0, v0);
    dmma(c[u][0], c[u][1], x1, v1);
  }
  red[w][2 * lane] = c[0][0] + c[1][0];
  red[w][2 * lane + 1] = c[0][1] + c[1][1];
  __syncthreads();
  if (threadIdx.x < 64) {
    const int idx = threadIdx.x, ln = idx >> 1, sl = idx & 1;
    double v = 0.0;
#pragma unroll
    for (int ww = 0; ww < 8; ++ww) v += red[ww][idx];
    const int r = ls0 + (ln >> 2), cidx = s0 + 2 * (ln & 3) + sl;
    if (r < L.P && cidx < nrhs) xc[(size_t)r * nrhs + cidx] -= v;
  }
}

// y_q[J0_q*TB + r][s] -= sum_ls Z_q[r][ls] x_C[ls][s]: CTA per 8 part rows x
// 8 sources, 8 warps over the 8-column chunks of Z (DMMA,
// D[r][s] += sum_ls Z[r][ls] x_C[ls][s]), fixed-order warp reduction.
__global__ void __launch_bounds__(256) k_schur_back(Coarse L, double* __restrict__ y0, double* __restrict__ y1,
                                                    const double* __restrict__ xc, int nrhs) {
  __shared__ double red[8][64];
  const int rb = blockIdx.x * 8, s0 = blockIdx.y * 8;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, m = lane >> 2, q = lane & 3;
  const int r0 = (L.b[0].NT - L.J0[0]) * TB;
  const int p = rb < r0 ? 0 : 1;
  const int rloc = (p == 0 ? rb : rb - r0) + m;                // Z row of this lane
  const double* Z = L.Z[p] + (size_t)rloc * L.P;
  const int s = s0 + m;
  double c[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
  int u = 0;
  for (int ls = 8 * w + 2 * q; ls < L.P + 6; ls += 64, u ^= 1) {
    const double x0 = ls < L.P ? Z[ls] : 0.0, x1 = ls + 1 < L.P ? Z[ls + 1] : 0.0;
    const double v0 = (ls < L.P && s < nrhs) ? xc[(size_t)ls * nrhs + s] : 0.0;
    const double v1 = (ls + 1 < L.P && s < nrhs) ? xc[(size_t)(ls + 1) * nrhs + s] : 0.0;
    dmma(c[u][0], c[u][1], x0, v0);
    dmma(c[u][0], c[u][1], x1, v1);
  }
  red[w][2 * lane] = c[0][0] + c[1][0];
  red[w][2 * lane + 1] = c[0][1] + c[1][1];
  __syncthreads();
  if (threadIdx.x < 64) {
    const int idx = threadIdx.x, ln = idx >> 1, sl = idx & 1;
    double v = 0.0;
#pragma unroll
    for (int ww = 0; ww < 8; ++ww) v += red[ww][idx];
    const int r = (p == 0 ? rb : rb - r0) + (ln >> 2), cidx = s0 + 2 * (ln & 3) + sl;
    if (L.J0[p] * TB + r < L.b[p].n && cidx < nrhs)
      ((p == 0 ? y0 : y1) + ((size_t)L.J0[p] * TB + r) * nrhs)[cidx] -= v;
  }
}

// natural X <-> part-local vectors (dir 0: gather, 1: scatter)
__global__ void k_coarse_permute(Geo g, Coarse L, double* __restrict__ X, double* __restrict__ x0,
                                 double* __restrict__ x1, double* __restrict__ xc, int nrhs, int dir) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= (long long)g.kc * nrhs) return;
  const int c = (int)(t / nrhs), s = (int)(t % nrhs);
  int p, l;
  coarse_map(L, c, p, l);
  double* d = (p == 0 ? x0 : (p == 1 ? x1 : xc)) + (size_t)l * nrhs + s;
  if (dir == 0) *d = X[t];
  else X[t] = *d;
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
__global__ void k_coarse_pack(Band B) {
  const int J = blockIdx.x / (B.PT + 1), t = blockIdx.x % (B.PT + 1);
  const bool valid = t == 0 || J + t < B.NT;
  const double* src = t == 0 ? B.Dinv + (size_t)J * TT : btile(B.Lo, B, J, t);
  double* f = B.LF + (size_t)blockIdx.x * TT;
  double* b = B.LB + (size_t)blockIdx.x * TT;
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


// One sweep job: a band's solve copies, its right-hand sides (row r of the
// band at X[r*nrhs]), first tile row J0 and mode (1 forward, 2 backward).
struct SweepJob {
  const double* LF;
  const double* LB;
  double* X;
  int NT, PT, n, nrhs, J0, mode;
};
struct SweepJobs {
  SweepJob j[2];
  int groups;   // CTAs (8 right-hand sides each) per job
};

// Banded substitution sweeps for 8 right-hand sides per CTA, one launch
// serving up to two independent jobs (e.g. the two nested-dissection parts);
// each job sweeps forward from tile row J0 (mode bit 1) and/or backward down
// to J0 (mode bit 2).  The factor tiles of a step (tile column J of LF / LB) are cut into nch chunks
// of up to CHT contiguous tiles; the chunk sequence (forward: J ascending,
// chunks in order; backward: J descending, chunks reversed so the Dinv chunk
// comes last) streams through a ring of TRSV_STAGES shared-memory stages, one
// bulk TMA copy per chunk, prefetched TRSV_STAGES-1 chunks ahead.  The active
// right-hand-side rows live in a shared-memory ring of transposed pieces.
constexpr int TRSV_MAX_STAGES = 3;

__global__ void __launch_bounds__(256) k_coarse_trsv_bulk(SweepJobs jobs, int CHT, int NS,
                                                          long long* tprof = nullptr) {
  extern __shared__ __align__(128) double bsm[];
  __shared__ __align__(8) unsigned long long bar[TRSV_MAX_STAGES];
  const SweepJob& job = jobs.j[blockIdx.x / jobs.groups];
  const int group = blockIdx.x % jobs.groups;
  const double* __restrict__ LF = job.LF;
  const double* __restrict__ LB = job.LB;
  double* __restrict__ X = job.X;
  const int NTj = job.NT, nrow = job.n, nrhs = job.nrhs, J0 = job.J0, mode = job.mode, PTj = job.PT;
  const int W = PTj + 1;
  const int nch = (W + CHT - 1) / CHT;
  const size_t stage_dbl = (size_t)CHT * TT;
  double* Rt = bsm + NS * stage_dbl;   // [W][4][64] rhs ring (transposed pieces)
  double* Ys = Rt + (size_t)W * 256;             // [4][64]
  double* Pt = Ys + 256;                         // [8][64]
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int c = lane >> 2, q = lane & 3;
  const int col = group * 8 + c;
  const bool cok = col < nrhs;
  auto ldx = [&](int R, int pi, double& a, double& b) {
    const int r0 = R * TB + 8 * pi + 2 * q;
    a = (cok && R < NTj && r0 < nrow) ? X[(size_t)r0 * nrhs + col] : 0.0;
    b = (cok && R < NTj && r0 + 1 < nrow) ? X[(size_t)(r0 + 1) * nrhs + col] : 0.0;
  };
  auto stx = [&](int R, int pi, double a, double b) {
    const int r0 = R * TB + 8 * pi + 2 * q;
    if (cok && r0 < nrow) X[(size_t)r0 * nrhs + col] = a;
    if (cok && r0 + 1 < nrow) X[(size_t)(r0 + 1) * nrhs + col] = b;
  };
  auto piece = [&](const double* base, int p) -> const double* { return base + p * 64 + 2 * lane; };
  auto ring = [&](int jm, int t) { const int r = jm + t; return r >= W ? r - W : r; };   // (J + t) % W, jm = J % W
  const int nsteps = (NTj - J0) * nch;
  const int nf = (mode & 1) ? nsteps : 0, total = nf + ((mode & 2) ? nsteps : 0);
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
        if (c.J == NTj) {
          c.fwd = false;
          c.J = NTj - 1;
          c.ch = nch - 1;
          c.jm = (NTj - 1) % W;
        }
      }
    } else if (--c.ch < 0) {
      c.ch = nch - 1;
      --c.J;
      c.jm = c.jm == 0 ? W - 1 : c.jm - 1;
    }
  };
  const It start = (mode & 1) ? It{J0, 0, J0 % W, true} : It{NTj - 1, nch - 1, (NTj - 1) % W, false};
  It ld = start;                    // next chunk to load
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
  if (mode & 1)
    for (int i = tid; i < W * 128; i += blockDim.x) {       // rows J0..J0+PT enter the ring
      const int R = J0 + i / 128, pi = (i / 32) & 3;
      if ((i & 31) == lane) {
        double a, b;
        ldx(R, pi, a, b);
        Rt[((R % W) * 4 + pi) * 64 + 2 * lane] = a;
        Rt[((R % W) * 4 + pi) * 64 + 2 * lane + 1] = b;
      }
    }
  __syncthreads();
  double p0 = 0.0, p1 = 0.0;        // backward partial sums of this warp, across the step's chunks
  double ya = 0.0, yb = 0.0;
  It cu = start;
  int st = 0;
  unsigned par = 0u;
  for (int i = 0; i < total; ++i, advance(cu), st = st + 1 == NS ? 0 : st + 1) {
    if (tid == 0) issue_next();
    const int J = cu.J, ch = cu.ch, jm = cu.jm;
    const int pt = min(PTj, NTj - 1 - J);
    const int t0 = ch * CHT, t1 = min(W, t0 + CHT) - 1;
    const double* T = bsm + (size_t)st * stage_dbl;           // local tile (t - t0)
    if (i == nf) {                                           // backward: the ring keeps x^T
      for (int k = tid; k < W * 256; k += blockDim.x) Rt[k] = 0.0;
      __syncthreads();
    }
    if (i >= nf && ch == nch - 1) {                         // first chunk of a backward step
      p0 = p1 = 0.0;
#ifndef TRSV_SKIP_LDX
      if (wid < 4) ldx(J, wid, ya, yb);
#endif
    }
    double ra = 0.0, rb = 0.0;
#ifndef TRSV_SKIP_LDX
    if (i < nf && ch == nch - 1 && wid < 4) ldx(J + 1 + PTj, wid, ra, rb);   // in flight during the step
#endif
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
          if (r0 >= nrow) c0 = 0.0;
          if (r0 + 1 >= nrow) c1 = 0.0;
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
static void trsv_bulk_shape(int PT, int& cht, int& ns, size_t& smem) {
  const int W = PT + 1;
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

// ------------------------------------------------ cluster-parallel sweeps
//
// Block-row-scaled forms of the two triangular systems:
//   forward   (Dinv L) y = Dinv b,        tiles SF[J][t] = Dinv_{J+t} L_{J+t,J}
//   backward  (Dinv^T L^T) x = Dinv^T y,  tiles SB[J][t] = Dinv_{J-t}^T L_{J,J-t}^T
// have identity diagonal blocks, so a right-looking sweep needs no diagonal
// solve: once row J is final, every row J+t (J-t) subtracts M_t * row_J, and
// the next row is final after ONE tile product.  Rows are spread over the C
// CTAs of a thread-block cluster (row R owned by CTA R mod C, each CTA holding
// its rows' accumulators in a shared-memory ring and streaming only its own
// tiles), so a step costs one tile product plus one DSMEM broadcast of the
// final row instead of a whole tile column on one SM.
//
// Broadcast protocol (all in shared memory, no grid barrier): the owner of
// the row final at global step u writes its 8x32 transposed value with
// st.async into slot u % CS_NB of every CTA's Ybuf, completing 2 KB of
// transaction bytes on that CTA's full[slot] barrier (armed by the receiver
// one use ahead).  A receiver releases a slot (remote arrive on empty[slot] of
// the CTA that will write its next use) as soon as the row is in registers.
// Warp w always owns 8-row piece w of every row, so the ring needs no
// CTA-wide synchronisation; one __syncthreads per step guards tile-stage reuse.
__global__ void __launch_bounds__(256) k_coarse_pack_scaled(Band B) {
  constexpr int LD = TB + 1;                             // padded rows: conflict-free columns
  __shared__ double Ms[TB * LD], Ds[TB * LD];
  const int J = blockIdx.x / (B.PT + 1), t = blockIdx.x % (B.PT + 1);
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // output (r = ty + 8i, col = tx)
  for (int dir = 0; dir < 2; ++dir) {
    const int R = dir == 0 ? J + t : J - t;              // row block whose Dinv scales
    const bool valid = R >= 0 && R < B.NT;
    double* out = (dir == 0 ? B.SF : B.SB) + (size_t)blockIdx.x * TT;
    __syncthreads();
    if (valid) {
      const double* L = t == 0 ? nullptr : btile(B.Lo, B, dir == 0 ? J : R, t);
      for (int e = threadIdx.x; e < TT; e += blockDim.x) {
        const int r = e / TB, cc = e % TB;
        Ds[r * LD + cc] = B.Dinv[(size_t)R * TT + e];
        Ms[r * LD + cc] = L ? L[e] : (r == cc ? 1.0 : 0.0);
      }
    }
    __syncthreads();
    // forward: (Dinv M)[r][col]; backward: (M Dinv)^T[r][col] = sum_k M[col][k] Dinv[k][r]
    double v[4] = {0.0, 0.0, 0.0, 0.0};
    if (valid) {
#pragma unroll 8
      for (int kk = 0; kk < TB; ++kk) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int r = ty + 8 * i;
          v[i] = dir == 0 ? fma(Ds[r * LD + kk], Ms[kk * LD + tx], v[i]) : fma(Ms[tx * LD + kk], Ds[kk * LD + r], v[i]);
        }
      }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {                        // element (r, tx) -> piece layout
      const int r = ty + 8 * i, p = (r >> 3) * 4 + (tx >> 3), lane = (r & 7) * 4 + ((tx & 7) >> 1);
      out[p * 64 + lane * 2 + (tx & 1)] = v[i];
    }
  }
}

constexpr int CS_CWARPS = 4;                      // compute warps
constexpr int CS_THREADS = (CS_CWARPS + 1) * 32;  // + one producer warp
constexpr int CS_NB = 4;      // broadcast slots
constexpr int CS_MAXNS = 3;   // tile stages (2 when 3 do not fit)
constexpr int CS_MAXC = 8;

struct CsJob {
  const double* SF;
  const double* SB;
  double* X;
  int NT, PT, n, nrhs, J0, mode;   // mode bit 1 forward (rows J0..NT-1), bit 2 backward (NT-1..J0)
};
struct CsJobs {
  CsJob j[2];
  int groups;   // clusters (8 right-hand sides each) per job
  int C;        // CTAs per cluster
  int SLT;      // tiles per stage
  int NS;       // tile stages
};

namespace {
__device__ __forceinline__ unsigned cs_mapa(unsigned a, int rank) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
// CTA-scope acquire: the st.async / bulk-copy data completes through the
// barrier's transaction count (async proxy); a cluster-scope acquire would
// also invalidate L1 (CCTL.IVALL) on every wait.
__device__ __forceinline__ void cs_wait(unsigned bar, unsigned parity) {
  unsigned done = 0;
  while (!done)
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
}
__device__ __forceinline__ void cs_arm(unsigned bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
// Relaxed remote arrive: a release at cluster scope compiles to a GPU-wide
// MEMBAR that waits for the thread's outstanding global stores.  The only
// accesses it must order are the shared-memory reads of the slot, which the
// caller makes complete first through a register dependency (dep == 0).
__device__ __forceinline__ void cs_remote_arrive(unsigned rbar, unsigned dep) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(rbar + dep) : "memory");
}
// 0, computed from v so that it cannot issue before v's loads complete
__device__ __forceinline__ unsigned cs_dep(double v) {
  unsigned z;
  asm volatile("{\n .reg .b32 lo, hi;\n mov.b64 {lo, hi}, %1;\n and.b32 %0, lo, 0;\n}\n" : "=r"(z) : "d"(v));
  return z;
}
__device__ __forceinline__ void cs_st_async(unsigned raddr, double a, double b, unsigned rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];\n" ::"r"(raddr),
               "d"(a), "d"(b), "r"(rbar)
               : "memory");
}
__device__ __forceinline__ void cs_bulk(double* dst, const double* src, unsigned bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"((unsigned)(TT * sizeof(double))), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void cs_cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ int cs_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return (int)r;
}
}  // namespace

__global__ void __launch_bounds__(CS_THREADS) k_coarse_sweep_cluster(CsJobs jobs) {
  extern __shared__ __align__(128) double csm[];
  __shared__ __align__(8) unsigned long long full[CS_NB], empty[CS_NB], tbar[CS_MAXNS], tfree[CS_MAXNS];
  const int C = jobs.C, cm = C - 1, SLT = jobs.SLT, NS = jobs.NS;
  const int cl = blockIdx.x / C, k = cs_rank();
  const bool j1 = cl >= jobs.groups;                          // (no dynamic param indexing)
  CsJob job;
#define CS_SEL(f) job.f = j1 ? jobs.j[1].f : jobs.j[0].f
  CS_SEL(SF); CS_SEL(SB); CS_SEL(X); CS_SEL(NT); CS_SEL(PT); CS_SEL(n); CS_SEL(nrhs); CS_SEL(J0); CS_SEL(mode);
#undef CS_SEL
  const int group = j1 ? cl - jobs.groups : cl;
  const int NT = job.NT, PT = job.PT, W = PT + 1, J0 = job.J0, nrow = job.n, nrhs = job.nrhs;
  const int nV = NT - J0;
  const int nph = ((job.mode & 1) ? 1 : 0) + ((job.mode & 2) ? 1 : 0);
  const int total = nph * nV;
  const bool fwd0 = (job.mode & 1) != 0;
  double* __restrict__ X = job.X;
  double* stage = csm;                                          // [NS][SLT][TT]
  double* ring = stage + (size_t)NS * SLT * TT;                 // [W][4][64]
  double* ybuf = ring + (size_t)W * 256;                        // [CS_NB][4][64]
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int q = lane & 3, col = group * 8 + (lane >> 2);
  const bool cok = col < nrhs;
  const unsigned full0 = smem_u32(&full[0]), empty0 = smem_u32(&empty[0]);
  const unsigned tbar0 = smem_u32(&tbar[0]), tfree0 = smem_u32(&tfree[0]);
  const unsigned ybuf0 = smem_u32(ybuf);

  // step u: direction, local index v, band row R; this CTA's rows updated at
  // step u are R +- t for t = t1, t1 + C, ... <= tmax; `entry`: the row of
  // local step v + PT + 1 (band row Re) enters this CTA's ring at step u
  struct Step {
    bool fwd, entry;
    int v, R, t1, tmax, Re;
  };
  auto geom = [&](int u) {
    Step s;
    s.fwd = fwd0 && u < nV;
    s.v = u < nV ? u : u - nV;
    s.R = s.fwd ? J0 + s.v : NT - 1 - s.v;
    s.t1 = (s.fwd ? k - s.R : s.R - k) & cm;
    if (s.t1 == 0) s.t1 = C;
    s.tmax = min(PT, nV - 1 - s.v);
    s.Re = s.fwd ? s.R + W : s.R - W;
    s.entry = s.v + W < nV && (s.Re & cm) == k;
    return s;
  };
  auto row_of = [&](int u) {
    const int v = u < nV ? u : u - nV;
    return (fwd0 && u < nV) ? J0 + v : NT - 1 - v;
  };
  auto ldx = [&](int R, int pi, double& a, double& b) {
    const int r0 = R * TB + 8 * pi + 2 * q;
    a = (cok && r0 < nrow) ? X[(size_t)r0 * nrhs + col] : 0.0;
    b = (cok && r0 + 1 < nrow) ? X[(size_t)(r0 + 1) * nrhs + col] : 0.0;
  };
  auto stx = [&](int R, int pi, double a, double b) {
    const int r0 = R * TB + 8 * pi + 2 * q;
    if (cok && r0 < nrow) X[(size_t)r0 * nrhs + col] = a;
    if (cok && r0 + 1 < nrow) X[(size_t)(r0 + 1) * nrhs + col] = b;
  };

  if (tid == 0) {
    for (int s = 0; s < CS_NB; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(full0 + 8u * s));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(empty0 + 8u * s), "r"(CS_CWARPS * C));
    }
    for (int s = 0; s < NS; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(tbar0 + 8u * s));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(tfree0 + 8u * s), "r"(CS_CWARPS));
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    for (int s = 0; s < CS_NB && s < total; ++s) cs_arm(full0 + 8u * s, 256u * sizeof(double));
  }
  cs_cluster_sync();

  if (w == CS_CWARPS) {
    // ---------------- producer warp: this CTA's tiles of every step, NS ahead
    if (lane == 0) {
      int st = 0;
      unsigned it = 0;
      for (int u = 0; u < total; ++u) {
        if (it > 0) cs_wait(tfree0 + 8u * st, (it - 1) & 1u);
        const Step s = geom(u);
        const int nt = (s.t1 <= s.tmax ? (s.tmax - s.t1) / C + 1 : 0) + (s.entry ? 1 : 0);
        const unsigned bar = tbar0 + 8u * st;
        cs_arm(bar, (unsigned)(nt * TT * sizeof(double)));
        const double* T = s.fwd ? job.SF : job.SB;
        double* dst = stage + (size_t)st * SLT * TT;
        int i = 0;
        for (int t = s.t1; t <= s.tmax; t += C, ++i)
          cs_bulk(dst + (size_t)i * TT, T + ((size_t)s.R * W + t) * TT, bar);
        if (s.entry) cs_bulk(dst + (size_t)i * TT, T + (size_t)s.Re * W * TT, bar);
        if (++st == NS) {
          st = 0;
          ++it;
        }
      }
    }
  } else {
    // ---------------- compute warps: warp w owns piece w of every row
    unsigned eph = 0u;               // empty-barrier parity per slot
    auto publish = [&](int u, double a, double b) {      // row of step u is final
      stx(row_of(u), w, a, b);
      const int s = u & (CS_NB - 1);
      if (u >= CS_NB) {
        cs_wait(empty0 + 8u * s, (eph >> s) & 1u);
        eph ^= 1u << s;
      }
      const unsigned la = ybuf0 + (unsigned)((s * 256 + w * 64 + 2 * lane) * sizeof(double));
      const unsigned lb = full0 + 8u * s;
      for (int c = 0; c < C; ++c) cs_st_async(cs_mapa(la, c), a, b, cs_mapa(lb, c));
    };
    auto prod = [&](const double* tp, const double (&x)[4][2], double& c0, double& c1) {
      double e0 = 0.0, e1 = 0.0;
#pragma unroll
      for (int kb = 0; kb < 4; kb += 2) {
        mma_xyt(c0, c1, x[kb][0], x[kb][1], tp[kb * 64], tp[kb * 64 + 1]);
        mma_xyt(e0, e1, x[kb + 1][0], x[kb + 1][1], tp[(kb + 1) * 64], tp[(kb + 1) * 64 + 1]);
      }
      c0 += e0;
      c1 += e1;
    };
    int st = 0;
    unsigned it = 0;
    int vs = 0;                      // v % W
    for (int u = 0; u < total; ++u) {
      const Step s = geom(u);
      if (s.v == 0) {
        // phase prologue: rows of local steps 0..PT enter (Dinv from global);
        // the first one is final at once
        vs = 0;
        asm volatile("bar.sync 1, %0;\n" ::"r"(CS_CWARPS * 32) : "memory");   // phase-1 results visible
        const double* T = s.fwd ? job.SF : job.SB;
        for (int vv = 0; vv < W && vv < nV; ++vv) {
          const int R = s.fwd ? s.R + vv : s.R - vv;
          if ((R & cm) != k) continue;
          double bv[4][2], m[4][2];
#pragma unroll
          for (int kb = 0; kb < 4; ++kb) {
            ldx(R, kb, bv[kb][0], bv[kb][1]);
            m[kb][0] = T[(size_t)R * W * TT + (w * 4 + kb) * 64 + 2 * lane];
            m[kb][1] = T[(size_t)R * W * TT + (w * 4 + kb) * 64 + 2 * lane + 1];
          }
          double c0 = 0.0, c1 = 0.0;
          double mm[4][2];
#pragma unroll
          for (int kb = 0; kb < 4; ++kb) {
            mm[kb][0] = m[kb][0];
            mm[kb][1] = m[kb][1];
          }
          // acc = M0 b: operands (b^T, M0 pieces)
          {
            double e0 = 0.0, e1 = 0.0;
#pragma unroll
            for (int kb = 0; kb < 4; kb += 2) {
              mma_xyt(c0, c1, bv[kb][0], bv[kb][1], mm[kb][0], mm[kb][1]);
              mma_xyt(e0, e1, bv[kb + 1][0], bv[kb + 1][1], mm[kb + 1][0], mm[kb + 1][1]);
            }
            c0 += e0;
            c1 += e1;
          }
          if (vv == 0) publish(u, c0, c1);
          else {
            ring[(vv * 4 + w) * 64 + 2 * lane] = c0;
            ring[(vv * 4 + w) * 64 + 2 * lane + 1] = c1;
          }
        }
      }
      double bv[4][2];
      if (s.entry) {                                       // in flight during the step
#pragma unroll
        for (int kb = 0; kb < 4; ++kb) ldx(s.Re, kb, bv[kb][0], bv[kb][1]);
      }
      cs_wait(tbar0 + 8u * st, it & 1u);
      const int ys = u & (CS_NB - 1);
      cs_wait(full0 + 8u * ys, (unsigned)((u >> 2) & 1));
      double ny[4][2];
#pragma unroll
      for (int kb = 0; kb < 4; ++kb) {
        ny[kb][0] = -ybuf[ys * 256 + kb * 64 + 2 * lane];
        ny[kb][1] = -ybuf[ys * 256 + kb * 64 + 2 * lane + 1];
      }
      if (tid == 0 && u + CS_NB < total) cs_arm(full0 + 8u * ys, 256u * sizeof(double));
      if (lane == 0 && u + CS_NB < total) {
        double d = 0.0;
#pragma unroll
        for (int kb = 0; kb < 4; ++kb) d += ny[kb][0] + ny[kb][1];
        cs_remote_arrive(cs_mapa(empty0 + 8u * ys, row_of(u + CS_NB) & cm), cs_dep(d));
      }
      const double* Tst = stage + (size_t)st * SLT * TT + w * 4 * 64 + 2 * lane;
      int t = s.t1, i = 0;
      if (t == 1 && t <= s.tmax) {                         // critical: row of step u+1 becomes final
        const int rs = vs + 1 == W ? 0 : vs + 1;
        const double* ap = ring + (rs * 4 + w) * 64 + 2 * lane;
        double c0 = ap[0], c1 = ap[1];
        prod(Tst, ny, c0, c1);
        publish(u + 1, c0, c1);
        t += C;
        ++i;
      }
      for (; t + C <= s.tmax; t += 2 * C, i += 2) {        // two independent tile products
        int ra = vs + t, rb = vs + t + C;
        ra -= ra >= W ? W : 0;
        rb -= rb >= W ? W : 0;
        double* apa = ring + (ra * 4 + w) * 64 + 2 * lane;
        double* apb = ring + (rb * 4 + w) * 64 + 2 * lane;
        double a0 = apa[0], a1 = apa[1], b0 = apb[0], b1 = apb[1];
        prod(Tst + (size_t)i * TT, ny, a0, a1);
        prod(Tst + (size_t)(i + 1) * TT, ny, b0, b1);
        apa[0] = a0;
        apa[1] = a1;
        apb[0] = b0;
        apb[1] = b1;
      }
      if (t <= s.tmax) {
        int ra = vs + t;
        ra -= ra >= W ? W : 0;
        double* apa = ring + (ra * 4 + w) * 64 + 2 * lane;
        double a0 = apa[0], a1 = apa[1];
        prod(Tst + (size_t)i * TT, ny, a0, a1);
        apa[0] = a0;
        apa[1] = a1;
        ++i;
      }
      if (s.entry) {                                       // ring slot of the finished row v
        double c0 = 0.0, c1 = 0.0;
        const double* tp = Tst + (size_t)i * TT;
        double e0 = 0.0, e1 = 0.0;
#pragma unroll
        for (int kb = 0; kb < 4; kb += 2) {
          mma_xyt(c0, c1, bv[kb][0], bv[kb][1], tp[kb * 64], tp[kb * 64 + 1]);
          mma_xyt(e0, e1, bv[kb + 1][0], bv[kb + 1][1], tp[(kb + 1) * 64], tp[(kb + 1) * 64 + 1]);
        }
        double* ap = ring + (vs * 4 + w) * 64 + 2 * lane;
        ap[0] = c0 + e0;
        ap[1] = c1 + e1;
      }
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(tfree0 + 8u * st) : "memory");
      if (++st == NS) {
        st = 0;
        ++it;
      }
      vs = vs + 1 == W ? 0 : vs + 1;
    }
  }
  cs_cluster_sync();
}

static cudaError_t launch_cluster_sweeps(const CsJobs& jobs, int njobs, int nrhs, cudaStream_t st) {
  if (nrhs == 0) return cudaSuccess;
  CsJobs J = jobs;
  int ptmax = 0;
  for (int k = 0; k < njobs; ++k) ptmax = std::max(ptmax, J.j[k].PT);
  J.groups = (nrhs + 7) / 8;
  J.C = 1;
  while (J.C * 2 <= std::min(CS_MAXC, ptmax)) J.C *= 2;      // power of two
  J.SLT = (ptmax + J.C - 1) / J.C + 1;
  const size_t fixed = ((size_t)(ptmax + 1) * 256 + CS_NB * 256) * sizeof(double);
  const size_t stage_b = (size_t)J.SLT * TT * sizeof(double);
  const size_t budget = 225 * 1024;
  J.NS = fixed + CS_MAXNS * stage_b <= budget ? CS_MAXNS : 2;
  const size_t smem = fixed + J.NS * stage_b;
  if (smem > budget) return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(k_coarse_sweep_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(njobs * J.groups * J.C));
  cfg.blockDim = dim3(CS_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)J.C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, k_coarse_sweep_cluster, J);
  count_launches(1);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

static CsJob cs_job(const Band& B, double* X, int nrhs, int J0, int mode) {
  CsJob s;
  s.SF = B.SF;
  s.SB = B.SB;
  s.X = X;
  s.NT = B.NT;
  s.PT = B.PT;
  s.n = B.n;
  s.nrhs = nrhs;
  s.J0 = J0;
  s.mode = mode;
  return s;
}

// ------------------------------------------------------------- launchers

static inline unsigned nblk(long long n, int t) { return (unsigned)((n + t - 1) / t); }

cudaError_t launch_mf_assemble(const Geo& g, const double* Kloc, double shift, double* Ak, cudaStream_t st);
cudaError_t launch_mf_diag(const Geo& g, const double* Ak, double* diag, cudaStream_t st);
cudaError_t launch_mf_factor(const Geo& g, double* Ak, int* flags, cudaStream_t st);
cudaError_t launch_mf_solve(const Geo& g, const double* Ak, double* X, double* scratch, int nrhs, cudaStream_t st);
size_t mf_doubles(const Geo& g);
int mf_tile_rows(const Geo& g);

cudaError_t launch_coarse_assemble(const Geo& g, const double* Kloc, double shift, double* Ak, cudaStream_t st) {
  if (g.coarse_nd == 2) return launch_mf_assemble(g, Kloc, shift, Ak, st);
  const Coarse L = coarse_layout(g, Ak);
  for (int b = 0; b < L.nb; ++b) {
    cudaError_t e = cudaMemsetAsync(L.b[b].A, 0, (size_t)L.b[b].NT * (L.b[b].PT + 1) * TT * sizeof(double), st);
    if (e != cudaSuccess) return e;
  }
  if (L.nd)
    for (int q = 0; q < 2; ++q) {
      cudaError_t e = cudaMemsetAsync(L.Z[q], 0, (size_t)(L.b[q].NT - L.J0[q]) * TB * L.P * sizeof(double), st);
      if (e != cudaSuccess) return e;
    }
  const long long tot = (long long)g.kc * 14 + (long long)L.nb * TB;
  k_coarse_assemble<<<nblk(tot, 256), 256, 0, st>>>(g, L, Kloc, shift);
  count_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_coarse_diag(const Geo& g, const double* Ak, double* diag, cudaStream_t st) {
  if (g.coarse_nd == 2) return launch_mf_diag(g, Ak, diag, st);
  k_coarse_diag<<<nblk(g.kc, 256), 256, 0, st>>>(g, coarse_layout(g, const_cast<double*>(Ak)), diag);
  count_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_coarse_dense(const Geo& g, const double* Kloc, double shift, double* out, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(out, 0, (size_t)g.kc * g.kc * sizeof(double), st);
  if (e != cudaSuccess) return e;
  k_coarse_dense<<<nblk((long long)g.kc * 14, 256), 256, 0, st>>>(g, Kloc, shift, out);
  count_launches(1);
  return cudaGetLastError();
}

static cudaError_t launch_factor_job(const FactorJob& job, int* flags, cudaStream_t st) {
  static PerDevice<int> grid_cache;
  const int coop_grid = grid_cache.get([] {
    int dev = 0, sms = 0, per_sm = 0, coop = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_coarse_factor, 256, 0);
    return (coop && per_sm > 0) ? sms : 0;
  });
  if (coop_grid <= 0) return cudaErrorNotSupported;
  FactorJob j = job;
  void* args[] = {(void*)&j, (void*)&flags};
  cudaError_t e = cudaLaunchCooperativeKernel((void*)k_coarse_factor, dim3(coop_grid), dim3(256), args, 0, st);
  count_launches(1);
  if (e != cudaSuccess) return e;
  for (int b = 0; b < job.nb; ++b) {
    k_coarse_pack<<<(unsigned)(job.b[b].NT * (job.b[b].PT + 1)), 256, 0, st>>>(job.b[b]);
    k_coarse_pack_scaled<<<(unsigned)(job.b[b].NT * (job.b[b].PT + 1)), 256, 0, st>>>(job.b[b]);
    count_launches(2);
  }
  return cudaGetLastError();
}

static cudaError_t launch_sweeps(const SweepJobs& jobs, int njobs, int nrhs, cudaStream_t st) {
  if (nrhs == 0) return cudaSuccess;
  int ptmax = 0;
  for (int k = 0; k < njobs; ++k) ptmax = std::max(ptmax, jobs.j[k].PT);
  int cht = 0, ns = 0;
  size_t smem = 0;
  trsv_bulk_shape(ptmax, cht, ns, smem);
  if (cht <= 0) return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(k_coarse_trsv_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  SweepJobs J = jobs;
  J.groups = (nrhs + 7) / 8;
  k_coarse_trsv_bulk<<<(unsigned)(njobs * J.groups), 256, smem, st>>>(J, cht, ns, nullptr);
  count_launches(1);
  return cudaGetLastError();
}

static SweepJob sweep_job(const Band& B, double* X, int nrhs, int J0, int mode) {
  SweepJob s;
  s.LF = B.LF;
  s.LB = B.LB;
  s.X = X;
  s.NT = B.NT;
  s.PT = B.PT;
  s.n = B.n;
  s.nrhs = nrhs;
  s.J0 = J0;
  s.mode = mode;
  return s;
}

static bool cluster_sweeps_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("MSFV_CLUSTER_SWEEP");
    on = e ? atoi(e) != 0 : 1;
  }
  return on != 0;
}

cudaError_t launch_coarse_factor(const Geo& g, double* Ak, int* flags, cudaStream_t st) {
  if (g.coarse_nd == 2) return launch_mf_factor(g, Ak, flags, st);
  const Coarse L = coarse_layout(g, Ak);
  FactorJob job{};
  job.b[0] = L.b[0];
  if (!L.nd) {
    job.nb = 1;
    return launch_factor_job(job, flags, st);
  }
  job.b[1] = L.b[1];
  job.nb = 2;
  cudaError_t e = launch_factor_job(job, flags, st);                // both parts
  if (e != cudaSuccess) return e;
  if (cluster_sweeps_enabled()) {                                   // Z_q = L_q^{-1} A_{q,C}
    CsJobs zj{};
    for (int q = 0; q < 2; ++q) zj.j[q] = cs_job(L.b[q], L.Z[q] - (size_t)L.J0[q] * TB * L.P, L.P, L.J0[q], 1);
    e = launch_cluster_sweeps(zj, 2, L.P, st);
  } else {
    SweepJobs zj{};
    for (int q = 0; q < 2; ++q) zj.j[q] = sweep_job(L.b[q], L.Z[q] - (size_t)L.J0[q] * TB * L.P, L.P, L.J0[q], 1);
    e = launch_sweeps(zj, 2, L.P, st);
  }
  if (e != cudaSuccess) return e;
  const int ntc = L.b[2].NT;
  const int red_bytes = 8 * 16 * 64 * (int)sizeof(double);
  e = cudaFuncSetAttribute(k_schur_update, cudaFuncAttributeMaxDynamicSharedMemorySize, red_bytes);
  if (e != cudaSuccess) return e;
  k_schur_update<<<(unsigned)(ntc * (ntc + 1) / 2), 256, red_bytes, st>>>(L);  // S = A_CC - sum Z^T Z
  count_launches(1);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  FactorJob jc{};
  jc.b[0] = L.b[2];
  jc.nb = 1;
  return launch_factor_job(jc, flags, st);
}


// Solve sweeps of one or two bands: cluster-parallel (scaled copies) by
// default, the one-CTA-per-8-rhs kernel when MSFV_CLUSTER_SWEEP=0.
static cudaError_t solve_sweeps(const Band* B, double* const* X, int nj, int nrhs, int mode, cudaStream_t st) {
  if (cluster_sweeps_enabled()) {
    CsJobs cj{};
    for (int k = 0; k < nj; ++k) cj.j[k] = cs_job(B[k], X[k], nrhs, 0, mode);
    return launch_cluster_sweeps(cj, nj, nrhs, st);
  }
  SweepJobs sj{};
  for (int k = 0; k < nj; ++k) sj.j[k] = sweep_job(B[k], X[k], nrhs, 0, mode);
  return launch_sweeps(sj, nj, nrhs, st);
}

cudaError_t launch_coarse_solve(const Geo& g, const double* Ak, double* X, double* scratch, int nrhs, cudaStream_t st) {
  if (nrhs == 0) return cudaSuccess;
  if (g.coarse_nd == 2) return launch_mf_solve(g, Ak, X, scratch, nrhs, st);
  const Coarse L = coarse_layout(g, const_cast<double*>(Ak));
  if (!L.nd) return solve_sweeps(&L.b[0], &X, 1, nrhs, 3, st);
  double* x0 = scratch;
  double* x1 = x0 + (size_t)L.b[0].NT * TB * nrhs;
  double* xc = x1 + (size_t)L.b[1].NT * TB * nrhs;
  double* xp[2] = {x0, x1};
  const long long tot = (long long)g.kc * nrhs;
  k_coarse_permute<<<nblk(tot, 256), 256, 0, st>>>(g, L, X, x0, x1, xc, nrhs, 0);
  count_launches(1);
  cudaError_t e = solve_sweeps(L.b, xp, 2, nrhs, 1, st);             // y_q = L_q^{-1} b_q
  if (e != cudaSuccess) return e;
  k_schur_rhs<<<dim3(nblk(L.P, 8), nblk(nrhs, 8)), 256, 0, st>>>(L, x0, x1, xc, nrhs);
  count_launches(1);
  e = solve_sweeps(&L.b[2], &xc, 1, nrhs, 3, st);                    // x_C = S^{-1}(b_C - sum Z^T y)
  if (e != cudaSuccess) return e;
  const long long rz = (long long)((L.b[0].NT - L.J0[0]) + (L.b[1].NT - L.J0[1])) * TB;
  k_schur_back<<<dim3(nblk(rz, 8), nblk(nrhs, 8)), 256, 0, st>>>(L, x0, x1, xc, nrhs);  // y_q -= Z_q x_C
  count_launches(1);
  e = solve_sweeps(L.b, xp, 2, nrhs, 2, st);                         // x_q = L_q^{-T} y_q
  if (e != cudaSuccess) return e;
  k_coarse_permute<<<nblk(tot, 256), 256, 0, st>>>(g, L, X, x0, x1, xc, nrhs, 1);
  count_launches(1);
  return cudaGetLastError();
}


// ============================================================================
// Multifrontal nested dissection of the coarse system (coarse_nd == 2).
//
// The coarse grid (kx x ky x kz nodes, 27-point stencil) is dissected
// recursively: a box is split by the coordinate plane through the middle of
// its longest extent; boxes of <= MF_LEAF (128) nodes are leaves.  A tree node
// eliminates E (its separator plane, or the whole leaf box); its front is
// [E | B], B = the nodes of ancestor separators adjacent to its box, each part
// padded to whole 32-row tiles (E padding = identity, B padding = 0).  Fronts
// are dense bands of full width (PT = NT - 1), so the tile-task Cholesky of
// the banded path factors them unchanged: the first NE tile columns are
// eliminated, the trailing tiles are left holding the update matrix
// U = F_BB - L_BE L_BE^T, which the parent extend-adds.  All fronts of one
// tree level are factored in one cooperative launch (grid barrier per tile
// column), the sequential depth is the sum over levels of NE instead of the
// band's NT (config 4: 26 tile columns instead of 73 + 10).  On levels with
// more B x B tiles than CTAs the B x B updates are deferred to one K-loop
// task per tile after the last column (coarse_deferred).  Solves walk the
// levels up (y_E = L_EE^-1 v_E, v_B -= L_BE y_E) and down
// (x_E = L_EE^-T (y_E - L_BE^T x_B)); contributions move between fronts by
// gathers through host-built index maps, so every sum has a fixed order.
// ============================================================================

constexpr int MF_LEAF = 128;   // leaf boxes of <= 128 coarse nodes (tuned on config 4: 64 -> 128 saves 0.07 ms per step)
constexpr int MF_MAXF = 1024;   // fronts per level handled by the cooperative kernels
constexpr int MF_GR = 16;       // rows per item of the G products
constexpr int MF_FACTOR_FCACHE = 256;  // front descriptors of a level cached by the factor kernel (dynamic shared memory)
constexpr int MF_KC = 256;      // input rows per chunk of the K-chunked G products (fronts beyond one shared-memory load)
constexpr int MF_INV_W = 8;     // identity columns per item of k_mf_inv_all
constexpr int MF_INV_NS = 6;    // its tile ring stages
constexpr int MF_INV_LD = COARSE_TB + 4;   // padded tile row stride (288 B: conflict-free fragment loads)
constexpr int MF_INV_SMALL = 12;   // fronts of <= 12 E tile columns share the small-footprint launch
constexpr int MF_SMEM_MAX = 226 * 1024;   // dynamic shared memory of the staged solve kernels
// explicit front inverse blocks (G) give one-product-per-front solves where
// the fronts fit the inverse-block budget (MfPlan::use_g); else staged sweeps
// SMs left to the backward basis sweeps (k_basis_bwd, side stream) while the
// multifrontal kernels run: the latency-bound coarse work keeps the rest
int mf_reserved_sms() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("MSFV_BWD_SMS");
    v = e ? std::max(0, atoi(e)) : 32;
  }
  return v;
}

struct MfFront {
  int nE, nB, NE, NT;     // real E / B sizes, tile counts (NT = NE + ceil(nB/TB))
  long long aoff;         // band storage offset (A, Dinv, Lo)
  long long voff;         // solve workspace row offset
  int c[2];               // children (-1: none)
  int goff;               // gid table offset (NT*TB entries, -1 = padding)
  int moff[2];            // child maps (NT*TB entries: child-local row or -1)
  int parent, pslot;      // parent front (-1: root) and which of its children this is
  int upoff;              // up map (NT*TB entries: parent-local row of this front's B rows, else -1)
  long long goff2;        // G = [L_EE^-1 ; -L_BE L_EE^-1] (NT*TB x NE*TB) then G^T, row-major
};

struct MfPlan {
  std::vector<MfFront> fr;
  std::vector<int> lvl, lvl_off;     // fronts per level (leaves first), CSR offsets
  std::vector<int> gid, maps;
  size_t a27 = 0, total = 0, vrows = 0;
  int maxNT = 0;
  // device copies (uploaded on first use)
  MfFront* d_fr = nullptr;
  int* d_lvl = nullptr;
  int* d_gid = nullptr;
  int* d_maps = nullptr;
  int* d_lvloff = nullptr;
  int* d_pre = nullptr;   // per-level prefix sums (solve): rows | forward items | backward items, npre each
  int npre = 0;
  MfFront* d_frl = nullptr;  // front descriptors in level order (one load instead of d_fr[d_lvl[.]])
  int4* d_gtab = nullptr;    // gather tables of the one-launch solve: forward rows then backward rows, level order
  int* d_rowbase = nullptr;  // first table row of every level (nl + 1 entries)
  int4* d_items = nullptr;   // k_mf_inv_all items (front, tile column, slice), longest chain first;
  int nitems[2] = {0, 0};    // group 0: fronts with NE > MF_INV_SMALL, group 1: the rest (own launch, own footprint)
  int inv_nemax[2] = {0, 0};
  bool use_g = true;      // explicit inverse blocks fit the kernels' shared memory (else staged sweeps)
};

__host__ __device__ __forceinline__ Band mf_band(double* base, const MfFront& f) {
  Band B{};
  B.n = f.NT * TB;
  B.NT = f.NT;
  B.PT = f.NT - 1;
  const size_t bt = (size_t)f.NT * f.NT * TT;
  B.A = base + f.aoff;
  B.Dinv = B.A + bt;
  B.Lo = B.Dinv + (size_t)f.NT * TT;
  B.LF = B.LB = B.SF = B.SB = nullptr;
  return B;
}

static void mf_dissect(MfPlan& P, int kx, int ky, int kz, int lo[3], int hi[3], std::vector<int>& anc_seps,
                       std::vector<std::vector<int>>& Elist, std::vector<std::vector<int>>& Blist,
                       std::vector<int>& height, std::vector<std::array<int, 2>>& kids, int& out_id) {
  auto id = [&](int x, int y, int z) { return x + kx * (y + ky * z); };
  const int ext[3] = {hi[0] - lo[0] + 1, hi[1] - lo[1] + 1, hi[2] - lo[2] + 1};
  const long long vol = (long long)ext[0] * ext[1] * ext[2];
  std::vector<int> E;
  std::array<int, 2> ch = {-1, -1};
  int h = 0;
  static int leaf = -1;
  if (leaf < 0) {
    const char* e = getenv("MSFV_MF_LEAF");
    leaf = e ? std::max(8, atoi(e)) : MF_LEAF;
  }
  if (vol <= leaf || (ext[0] < 3 && ext[1] < 3 && ext[2] < 3)) {
    for (int z = lo[2]; z <= hi[2]; ++z)
      for (int y = lo[1]; y <= hi[1]; ++y)
        for (int x = lo[0]; x <= hi[0]; ++x) E.push_back(id(x, y, z));
  } else {
    int ax = 2;
    if (ext[1] > ext[ax]) ax = 1;
    if (ext[0] > ext[ax]) ax = 0;
    const int mid = (lo[ax] + hi[ax]) / 2;
    int slo[3] = {lo[0], lo[1], lo[2]}, shi[3] = {hi[0], hi[1], hi[2]};
    slo[ax] = shi[ax] = mid;
    for (int z = slo[2]; z <= shi[2]; ++z)
      for (int y = slo[1]; y <= shi[1]; ++y)
        for (int x = slo[0]; x <= shi[0]; ++x) E.push_back(id(x, y, z));
    // the separator's own nodes are ancestors of both halves
    const size_t mark = anc_seps.size();
    anc_seps.insert(anc_seps.end(), E.begin(), E.end());
    for (int side = 0; side < 2; ++side) {
      int clo[3] = {lo[0], lo[1], lo[2]}, chi[3] = {hi[0], hi[1], hi[2]};
      if (side == 0) chi[ax] = mid - 1; else clo[ax] = mid + 1;
      if (clo[ax] > chi[ax]) continue;
      int cid;
      mf_dissect(P, kx, ky, kz, clo, chi, anc_seps, Elist, Blist, height, kids, cid);
      ch[side] = cid;
      h = std::max(h, height[cid] + 1);
    }
    anc_seps.resize(mark);
  }
  // B: ancestor separator nodes adjacent (27-point) to the box
  std::vector<int> B;
  for (int u : anc_seps) {
    const int x = u % kx, y = (u / kx) % ky, z = u / (kx * ky);
    if (x >= lo[0] - 1 && x <= hi[0] + 1 && y >= lo[1] - 1 && y <= hi[1] + 1 && z >= lo[2] - 1 && z <= hi[2] + 1)
      B.push_back(u);
  }
  out_id = (int)Elist.size();
  Elist.push_back(E);
  Blist.push_back(B);
  height.push_back(h);
  kids.push_back(ch);
}

static MfPlan* mf_build(const Geo& g) {
  auto* P = new MfPlan;
  const int kx = g.nb1 + 1, ky = g.nb2 + 1, kz = g.nb3 + 1;
  std::vector<std::vector<int>> Elist, Blist;
  std::vector<int> height, anc;
  std::vector<std::array<int, 2>> kids;
  int lo[3] = {0, 0, 0}, hi[3] = {kx - 1, ky - 1, kz - 1}, root;
  mf_dissect(*P, kx, ky, kz, lo, hi, anc, Elist, Blist, height, kids, root);
  const int nf = (int)Elist.size();     // postorder: children before parents
  // B in elimination order (ancestor fronts come later in postorder; within a
  // front E is lexicographic)
  std::vector<int> pos(g.kc, -1);
  {
    int p = 0;
    for (int f = 0; f < nf; ++f)
      for (int u : Elist[f]) pos[u] = p++;
  }
  for (auto& B : Blist) std::sort(B.begin(), B.end(), [&](int a, int b) { return pos[a] < pos[b]; });
  P->fr.resize(nf);
  size_t aoff = 0, voff = 0;
  for (int f = 0; f < nf; ++f) {
    MfFront& F = P->fr[f];
    F.nE = (int)Elist[f].size();
    F.nB = (int)Blist[f].size();
    F.NE = (F.nE + TB - 1) / TB;
    F.NT = F.NE + (F.nB + TB - 1) / TB;
    F.aoff = (long long)aoff;
    aoff += (size_t)F.NT * F.NT * TT * 2 + (size_t)F.NT * TT;
    F.voff = (long long)voff;
    voff += (size_t)F.NT * TB;
    F.c[0] = kids[f][0];
    F.c[1] = kids[f][1];
    P->maxNT = std::max(P->maxNT, F.NT);
    F.goff = (int)P->gid.size();
    for (int r = 0; r < F.NT * TB; ++r) {
      int v = -1;
      if (r < F.NE * TB) { if (r < F.nE) v = Elist[f][r]; }
      else if (r - F.NE * TB < F.nB) v = Blist[f][r - F.NE * TB];
      P->gid.push_back(v);
    }
  }
  for (int f = 0; f < nf; ++f) {
    MfFront& F = P->fr[f];
    for (int s = 0; s < 2; ++s) {
      F.moff[s] = -1;
      const int c = F.c[s];
      if (c < 0) continue;
      const MfFront& C = P->fr[c];
      std::vector<int> where(g.kc, -1);       // node -> child-local row of the child's B part
      for (int i = 0; i < C.nB; ++i) where[Blist[c][i]] = C.NE * TB + i;
      F.moff[s] = (int)P->maps.size();
      for (int r = 0; r < F.NT * TB; ++r) {
        const int u = P->gid[F.goff + r];
        P->maps.push_back(u >= 0 ? where[u] : -1);
      }
    }
  }
  // parents and up maps (child B row -> parent-local row)
  for (int f = 0; f < nf; ++f) {
    P->fr[f].parent = -1;
    P->fr[f].pslot = 0;
  }
  for (int f = 0; f < nf; ++f)
    for (int sl = 0; sl < 2; ++sl)
      if (P->fr[f].c[sl] >= 0) {
        P->fr[P->fr[f].c[sl]].parent = f;
        P->fr[P->fr[f].c[sl]].pslot = sl;
      }
  for (int f = 0; f < nf; ++f) {
    MfFront& F = P->fr[f];
    F.upoff = (int)P->maps.size();
    std::vector<int> prow;
    if (F.parent >= 0) {
      const MfFront& Pa = P->fr[F.parent];
      prow.assign(g.kc, -1);
      for (int r = 0; r < Pa.NT * TB; ++r) {
        const int u = P->gid[Pa.goff + r];
        if (u >= 0) prow[u] = r;
      }
    }
    for (int r = 0; r < F.NT * TB; ++r) {
      const int u = P->gid[F.goff + r];
      P->maps.push_back(F.parent >= 0 && r >= F.NE * TB && u >= 0 ? prow[u] : -1);
    }
  }
  // levels by height (leaves = 0)
  int hmax = 0;
  for (int f = 0; f < nf; ++f) hmax = std::max(hmax, height[f]);
  P->lvl_off.push_back(0);
  for (int h = 0; h <= hmax; ++h) {
    for (int f = 0; f < nf; ++f)
      if (height[f] == h) P->lvl.push_back(f);
    P->lvl_off.push_back((int)P->lvl.size());
  }
  for (int f = 0; f < nf; ++f) {
    MfFront& F = P->fr[f];
    F.goff2 = (long long)aoff;
    aoff += (size_t)2 * F.NT * F.NE * TT;
  }
  P->a27 = aoff;
  P->total = aoff + (size_t)g.kc * 14;
  P->vrows = voff;
  if (getenv("MSFV_MF_DEBUG")) {
    for (size_t l = 0; l + 1 < P->lvl_off.size(); ++l) {
      int ne = 0, nt = 0, nemax = 0;
      for (int i = P->lvl_off[l]; i < P->lvl_off[l + 1]; ++i) {
        ne += P->fr[P->lvl[i]].nE;
        nt = std::max(nt, P->fr[P->lvl[i]].NT);
        nemax = std::max(nemax, P->fr[P->lvl[i]].NE);
      }
      fprintf(stderr, "mf level %zu: %d fronts, sum nE %d, max NE %d tiles, max NT %d tiles\n", l,
              P->lvl_off[l + 1] - P->lvl_off[l], ne, nemax, nt);
    }
  }
  return P;
}

static const MfPlan* mf_plan(const Geo& g) { return static_cast<const MfPlan*>(g.mf); }

static cudaError_t mf_upload(const Geo& g) {
  MfPlan* P = const_cast<MfPlan*>(mf_plan(g));
  if (P->d_fr) return cudaSuccess;
  cudaError_t e = cudaMalloc(&P->d_fr, P->fr.size() * sizeof(MfFront));
  if (e == cudaSuccess) e = cudaMalloc(&P->d_lvl, P->lvl.size() * sizeof(int));
  if (e == cudaSuccess) e = cudaMalloc(&P->d_gid, P->gid.size() * sizeof(int));
  if (e == cudaSuccess) e = cudaMalloc(&P->d_maps, std::max<size_t>(P->maps.size(), 1) * sizeof(int));
  if (e == cudaSuccess) e = cudaMemcpy(P->d_fr, P->fr.data(), P->fr.size() * sizeof(MfFront), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(P->d_lvl, P->lvl.data(), P->lvl.size() * sizeof(int), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(P->d_gid, P->gid.data(), P->gid.size() * sizeof(int), cudaMemcpyHostToDevice);
  if (e == cudaSuccess && !P->maps.empty())
    e = cudaMemcpy(P->d_maps, P->maps.data(), P->maps.size() * sizeof(int), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMalloc(&P->d_lvloff, P->lvl_off.size() * sizeof(int));
  if (e == cudaSuccess)
    e = cudaMemcpy(P->d_lvloff, P->lvl_off.data(), P->lvl_off.size() * sizeof(int), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) {
    // level l's prefixes start at lvl_off[l] + l (nf + 1 entries each)
    const int nl = (int)P->lvl_off.size() - 1;
    P->npre = P->lvl_off[nl] + nl;
    std::vector<int> pre(3 * (size_t)P->npre, 0);
    for (int l = 0; l < nl; ++l) {
      const int l0 = P->lvl_off[l], nf = P->lvl_off[l + 1] - l0, pb = l0 + l;
      for (int i = 0; i < nf; ++i) {
        const MfFront& F = P->fr[P->lvl[l0 + i]];
        pre[pb + i + 1] = pre[pb + i] + F.NT * TB;
        pre[P->npre + pb + i + 1] = pre[P->npre + pb + i] + (F.NT * TB + MF_GR - 1) / MF_GR;
        pre[2 * P->npre + pb + i + 1] = pre[2 * P->npre + pb + i] + (F.nE + MF_GR - 1) / MF_GR;
      }
    }
    e = cudaMalloc(&P->d_pre, pre.size() * sizeof(int));
    if (e == cudaSuccess) e = cudaMemcpy(P->d_pre, pre.data(), pre.size() * sizeof(int), cudaMemcpyHostToDevice);
  }
  if (e == cudaSuccess) {
    // Gather tables of the solve's phase (A), one int4 per front row in level order: forward
    // (V row, X row of an E node or -1, child 0 V row or -1, child 1 V row or -1), backward
    // (V row, own V row for the E tile rows or -1, X row of a B node or -1, 0): a thread needs one table
    // load and then its value loads, instead of descriptor, node id, map and child offset loads in turn.
    const int nl = (int)P->lvl_off.size() - 1;
    std::vector<int> rowbase(nl + 1, 0);
    std::vector<int4> tab(2 * P->vrows);
    int pos = 0;
    for (int l = 0; l < nl; ++l) {
      rowbase[l] = pos;
      for (int i = P->lvl_off[l]; i < P->lvl_off[l + 1]; ++i) {
        const MfFront& F = P->fr[P->lvl[i]];
        for (int r = 0; r < F.NT * TB; ++r, ++pos) {
          const int gidr = P->gid[F.goff + r];
          int4 f = make_int4((int)F.voff + r, (r < F.nE) ? gidr : -1, -1, -1);
          for (int c = 0; c < 2; ++c) {
            if (F.c[c] < 0) continue;
            const int q = P->maps[F.moff[c] + r];
            if (q >= 0) (c == 0 ? f.z : f.w) = (int)P->fr[F.c[c]].voff + q;
          }
          tab[pos] = f;
          tab[P->vrows + pos] = make_int4((int)F.voff + r, r < F.NE * TB ? (int)F.voff + r : -1,
                                          (r >= F.NE * TB && gidr >= 0) ? gidr : -1, 0);
        }
      }
    }
    rowbase[nl] = pos;
    std::vector<MfFront> frl(P->lvl.size());
    for (size_t i = 0; i < P->lvl.size(); ++i) frl[i] = P->fr[P->lvl[i]];
    e = cudaMalloc(&P->d_frl, frl.size() * sizeof(MfFront));
    if (e == cudaSuccess) e = cudaMemcpy(P->d_frl, frl.data(), frl.size() * sizeof(MfFront), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMalloc(&P->d_gtab, tab.size() * sizeof(int4));
    if (e == cudaSuccess) e = cudaMemcpy(P->d_gtab, tab.data(), tab.size() * sizeof(int4), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMalloc(&P->d_rowbase, rowbase.size() * sizeof(int));
    if (e == cudaSuccess)
      e = cudaMemcpy(P->d_rowbase, rowbase.data(), rowbase.size() * sizeof(int), cudaMemcpyHostToDevice);
  }
  if (e == cudaSuccess && P->use_g) {
    std::vector<int4> items[2];
    for (int f = 0; f < (int)P->fr.size(); ++f) {
      const MfFront& F = P->fr[f];
      const int grp = F.NE > MF_INV_SMALL ? 0 : 1;
      P->inv_nemax[grp] = std::max(P->inv_nemax[grp], F.NE);
      for (int c = 0; c < F.NE; ++c) {
        const int cost = (F.NE - c) * (F.NE - c + 1) / 2 + (F.NT - F.NE) * (F.NE - c);
        for (int sl = 0; sl < TB / MF_INV_W; ++sl) items[grp].push_back(make_int4(f, c, sl, cost));
      }
    }
    for (auto& v : items) std::stable_sort(v.begin(), v.end(), [](const int4& a, const int4& b) { return a.w > b.w; });
    P->nitems[0] = (int)items[0].size();
    P->nitems[1] = (int)items[1].size();
    items[0].insert(items[0].end(), items[1].begin(), items[1].end());
    e = cudaMalloc(&P->d_items, std::max<size_t>(items[0].size(), 1) * sizeof(int4));
    if (e == cudaSuccess && !items[0].empty())
      e = cudaMemcpy(P->d_items, items[0].data(), items[0].size() * sizeof(int4), cudaMemcpyHostToDevice);
  }
  return e;
}

void mf_release(Geo& g) {
  auto* P = const_cast<MfPlan*>(mf_plan(g));
  if (!P) return;
  if (P->d_fr) cudaFree(P->d_fr);
  if (P->d_lvl) cudaFree(P->d_lvl);
  if (P->d_gid) cudaFree(P->d_gid);
  if (P->d_maps) cudaFree(P->d_maps);
  if (P->d_lvloff) cudaFree(P->d_lvloff);
  if (P->d_pre) cudaFree(P->d_pre);
  if (P->d_items) cudaFree(P->d_items);
  if (P->d_gtab) cudaFree(P->d_gtab);
  if (P->d_frl) cudaFree(P->d_frl);
  if (P->d_rowbase) cudaFree(P->d_rowbase);
  delete P;
  g.mf = nullptr;
}
// Multifrontal plan when its kernels fit (the explicit-inverse chain keeps a
// front's E rows in shared memory; the one-launch solve keeps the largest
// front's G chunk and vector there, sized for <= 32 right-hand sides).
bool mf_attach(Geo& g) {
  MfPlan* P = mf_build(g);
  int nemax = 0, ntmax = 0;
  for (const MfFront& F : P->fr) {
    nemax = std::max(nemax, F.NE);
    ntmax = std::max(ntmax, F.NT);
  }
  const size_t inv_b = ((size_t)nemax * TB * MF_INV_W + (size_t)MF_INV_NS * TB * MF_INV_LD) * sizeof(double);
  const int nl = (int)P->lvl_off.size() - 1;
  int maxf = 0;
  for (int l = 0; l < nl; ++l) maxf = std::max(maxf, P->lvl_off[l + 1] - P->lvl_off[l]);
  if (maxf > MF_MAXF) {
    delete P;
    g.mf = nullptr;
    return false;
  }
  // explicit inverse blocks whenever a front's 8 inverse columns fit shared
  // memory (k_mf_inv_all); fronts whose G chunk and input vector exceed one
  // shared-memory load take the K-chunked products of the one-launch solve
  // (config 5's top levels).  Otherwise the blocked sweeps.
  (void)ntmax;
  P->use_g = inv_b <= (size_t)MF_SMEM_MAX;
  g.mf = P;
  return true;
}

struct MfDev {
  const MfFront* fr;
  const int* lvl;
  const int* gid;
  const int* maps;
  double* base;
};

// A27[c][o]: the 14 lexicographically lower stencil entries of row c
__global__ void k_mf_a27(Geo g, const double* __restrict__ Kloc, double shift, double* __restrict__ A27) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= (long long)g.kc * 14) return;
  const int o = (int)(t % 14), c = (int)(t / 14);
  int c2;
  double v;
  A27[t] = coarse_entry(g, Kloc, shift, c, o, c2, v) ? v : 0.0;
}
__device__ __forceinline__ double mf_a(const Geo& g, const double* __restrict__ A27, int a, int b) {
  const int c = max(a, b), c2 = min(a, b);
  const int kx = g.nb1 + 1, ky = g.nb2 + 1;
  const int dx = c2 % kx - c % kx, dy = (c2 / kx) % ky - (c / kx) % ky, dz = c2 / (kx * ky) - c / (kx * ky);
  if (dx < -1 || dx > 1 || dy < -1 || dy > 1 || dz < -1 || dz > 1) return 0.0;
  int o;
  if (dz == -1) o = (dy + 1) * 3 + (dx + 1);
  else if (dz == 0 && dy == -1) o = 9 + dx + 1;
  else o = 12 + dx + 1;
  return A27[(size_t)c * 14 + o];
}
// U element (r, c) (child-local, both in the child's B part) of a factored child
__device__ __forceinline__ double mf_u(const Band& C, int r, int c) {
  const int a = max(r, c), b = min(r, c);
  return btile(C.A, C, b / TB, a / TB - b / TB)[(a % TB) * TB + (b % TB)];
}
// Tile-staged assembly: CTA (lower tile, front); the tile's 32 row and 32
// column node ids, their coarse coordinates and child-map entries are staged
// in shared memory once, each thread then assembles 4 elements.
__global__ void __launch_bounds__(256) k_mf_assemble_t(Geo g, MfDev d, int l0, const double* __restrict__ A27) {
  __shared__ int rid[2][TB], rco[2][TB], rm0[2][TB], rm1[2][TB];   // [0] rows, [1] columns
  const MfFront F = d.fr[d.lvl[l0 + blockIdx.y]];
  const int nlow = F.NT * (F.NT + 1) / 2;
  if ((int)blockIdx.x >= nlow) return;
  int J = 0, rem = blockIdx.x;
  while (rem >= F.NT - J) {
    rem -= F.NT - J;
    ++J;
  }
  const int tt = rem;
  const Band B = mf_band(d.base, F);
  const int* gid = d.gid + F.goff;
  const int* m0 = F.c[0] >= 0 ? d.maps + F.moff[0] : nullptr;
  const int* m1 = F.c[1] >= 0 ? d.maps + F.moff[1] : nullptr;
  const int kx = g.nb1 + 1, ky = g.nb2 + 1;
  if (threadIdx.x < 2 * TB) {
    const int w = threadIdx.x / TB, i = threadIdx.x % TB;
    const int r = (w == 0 ? (J + tt) : J) * TB + i;
    const int u = gid[r];
    rid[w][i] = u;
    rco[w][i] = u >= 0 ? (u % kx) | (((u / kx) % ky) << 10) | ((u / (kx * ky)) << 20) : 0;
    rm0[w][i] = m0 ? m0[r] : -1;
    rm1[w][i] = m1 ? m1[r] : -1;
  }
  Band C0{}, C1{};
  if (F.c[0] >= 0) C0 = mf_band(d.base, d.fr[F.c[0]]);
  if (F.c[1] >= 0) C1 = mf_band(d.base, d.fr[F.c[1]]);
  __syncthreads();
  double* T = btile(B.A, B, J, tt);
  for (int e = threadIdx.x; e < TT; e += blockDim.x) {
    const int i = e / TB, j = e % TB;
    const int r = (J + tt) * TB + i, c = J * TB + j;
    const int gr = rid[0][i], gc = rid[1][j];
    double v = 0.0;
    if (gr < 0 || gc < 0) {
      v = (r == c && r < F.NE * TB) ? 1.0 : 0.0;
    } else {
      if (r < F.nE || c < F.nE) {
        // A_k(gr, gc) from the 14 lower stencil entries of max(gr, gc)
        const bool sw = gr < gc;
        const int hi = sw ? gc : gr, pc = sw ? rco[0][i] : rco[1][j], hc = sw ? rco[1][j] : rco[0][i];
        const int dx = (pc & 1023) - (hc & 1023), dy = ((pc >> 10) & 1023) - ((hc >> 10) & 1023),
                  dz = (pc >> 20) - (hc >> 20);
        if (dx >= -1 && dx <= 1 && dy >= -1 && dy <= 1 && dz >= -1 && dz <= 1) {
          const int o = dz == -1 ? (dy + 1) * 3 + (dx + 1) : (dy == -1 ? 9 + dx + 1 : 12 + dx + 1);
          v = A27[(size_t)hi * 14 + o];
        }
      }
      if (rm0[0][i] >= 0 && rm0[1][j] >= 0) v += mf_u(C0, rm0[0][i], rm0[1][j]);
      if (rm1[0][i] >= 0 && rm1[1][j] >= 0) v += mf_u(C1, rm1[0][i], rm1[1][j]);
    }
    T[e] = v;
  }
}
// Partial Cholesky (first NE tile columns) of all fronts of one level, one
// grid barrier per tile column: CTA f (< nf) factors front f's diagonal tiles
// (one-column lookahead), the other CTAs take the trailing tile tasks of all
// fronts in one index space.
struct MfJob {
  MfDev d;
  int l0, nf, jmax;
  int defer;   // 1: B x B trailing updates deferred to one K-loop task per tile (levels with more B x B tiles than CTAs)
  Geo g;
};
__global__ void __launch_bounds__(256, 2) k_mf_factor(MfJob job, int* __restrict__ flags) {
  __shared__ __align__(16) FactorSmem sm;
  __shared__ int pre[MF_MAXF + 1];
  cg::grid_group grid = cg::this_grid();
  const int nf = job.nf, G = (int)gridDim.x;
  const bool split = nf < G;
  // the level's front descriptors are fetched once (dynamic shared memory, the first MF_FACTOR_FCACHE
  // fronts): d.fr[d.lvl[.]] is two dependent global loads, asked for by every task and every tile column
  extern __shared__ __align__(16) unsigned char fcache_raw[];
  MfFront* fcache = reinterpret_cast<MfFront*>(fcache_raw);
  const int ncache = min(nf, MF_FACTOR_FCACHE);
  for (int i = threadIdx.x; i < ncache; i += blockDim.x) fcache[i] = job.d.fr[job.d.lvl[job.l0 + i]];
  __syncthreads();
  auto front = [&](int i) { return i < ncache ? fcache[i] : job.d.fr[job.d.lvl[job.l0 + i]]; };
  // a chain CTA with one front keeps its descriptor in registers (critical path of every tile column)
  MfFront myF{};
  if (split && (int)blockIdx.x < nf) myF = front(blockIdx.x);
  for (int i = blockIdx.x; i < nf; i += G) coarse_potrf(mf_band(job.d.base, split ? myF : front(i)), 0, flags, sm);
  grid.sync();
  const int nw = split ? G - nf : G, me = split ? (int)blockIdx.x - nf : (int)blockIdx.x;
  for (int J = 0; J < job.jmax; ++J) {
    for (int i = blockIdx.x; i < nf && (split ? blockIdx.x < nf : true); i += G) {
      const MfFront F = split ? myF : front(i);
      if (J + 1 < F.NE) {
        const Band B = mf_band(job.d.base, F);
        if (!split) {                              // a chain CTA with one front still holds Dinv_J from its POTRF
          load_tile(sm.D, B.Dinv + (size_t)J * TT);
          __syncthreads();
        }
        coarse_chain_task(B, J, sm);
        coarse_potrf(B, J + 1, flags, sm, true);
      }
    }
    if (me >= 0) {
      // prefix of the task counts (each CTA builds the same table).  Per
      // front: the pairs (t1, t2) whose column J + t2 is still an E column
      // (those tiles feed the next panels), then one panel-only task per B
      // row; the B x B tiles wait for the deferred phase below.
      for (int i = threadIdx.x; i < nf; i += blockDim.x) {
        const MfFront F = front(i);
        int n = 0;
        if (J < F.NE) {
          const int pt = F.NT - 1 - J, ne = F.NE - 1 - J, nep = job.defer ? ne : pt;
          n = nep * pt - nep * (nep - 1) / 2 - (ne >= 1 ? 1 : 0) + (pt - nep);
        }
        pre[i + 1] = n;
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        pre[0] = 0;
        for (int i = 0; i < nf; ++i) pre[i + 1] += pre[i];
      }
      __syncthreads();
      const int total = pre[nf];
      int loaded = -1, fi = 0;
      for (int gi = me; gi < total; gi += nw) {
        while (pre[fi + 1] <= gi) ++fi;
        const MfFront F = front(fi);
        const Band B = mf_band(job.d.base, F);
        const int pt = F.NT - 1 - J, ne = F.NE - 1 - J, nep = job.defer ? ne : pt;
        const int npair = nep * pt - nep * (nep - 1) / 2;
        if (loaded != fi) {
          load_tile(sm.D, B.Dinv + (size_t)J * TT);
          __syncthreads();
          loaded = fi;
        }
        int p = (gi - pre[fi]) + (ne >= 1 ? 1 : 0);    // pair (1,1) belongs to the chain CTA
        if (p < npair) {
          int t2 = 1;
          while (p >= pt - t2 + 1) {
            p -= pt - t2 + 1;
            ++t2;
          }
          coarse_pair(B, J, t2 + p, t2, sm);
        } else {
          coarse_panel_only(B, J, nep + 1 + (p - npair), sm);
        }
      }
    }
    grid.sync();
  }
  // ---- deferred phase: the update matrices U = F_BB - L_BE L_BE^T, one task per lower B x B tile
  if (job.defer) {
    for (int i = threadIdx.x; i < nf; i += blockDim.x) {
      const MfFront F = front(i);
      const int nb = F.NT - F.NE;
      pre[i + 1] = nb * (nb + 1) / 2;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      pre[0] = 0;
      for (int i = 0; i < nf; ++i) pre[i + 1] += pre[i];
    }
    __syncthreads();
    const int total = pre[nf];
    int fi = 0;
    for (int gi = blockIdx.x; gi < total; gi += G) {
      while (pre[fi + 1] <= gi) ++fi;
      const MfFront F = front(fi);
      const Band B = mf_band(job.d.base, F);
      int p = gi - pre[fi], r = 0;                     // p = r (r + 1) / 2 + c, c <= r
      while ((r + 1) * (r + 2) / 2 <= p) ++r;
      coarse_deferred(B, F.NE, F.NE + r, F.NE + p - r * (r + 1) / 2, sm);
    }
  }
}

// Forward solve of the fronts of one level, CTA per front:
// v = [X(E) ; 0] + children's v_B (gathers), y_J = Dinv_J v_J,
// v_I -= L_{I,J} y_J; V keeps y_E and the update v_B for the parent.
__global__ void __launch_bounds__(256) k_mf_fwd(MfDev d, int l0, const double* __restrict__ X, double* __restrict__ V,
                                                int nrhs) {
  extern __shared__ __align__(16) double ys[];     // TB x nrhs
  const MfFront F = d.fr[d.lvl[l0 + blockIdx.x]];
  const Band B = mf_band(d.base, F);
  const int* gid = d.gid + F.goff;
  double* v = V + (size_t)F.voff * nrhs;
  const int rows = F.NT * TB;
  const double* v0 = F.c[0] >= 0 ? V + (size_t)d.fr[F.c[0]].voff * nrhs : nullptr;
  const double* v1 = F.c[1] >= 0 ? V + (size_t)d.fr[F.c[1]].voff * nrhs : nullptr;
  const int* m0 = v0 ? d.maps + F.moff[0] : nullptr;
  const int* m1 = v1 ? d.maps + F.moff[1] : nullptr;
  for (int t = threadIdx.x; t < rows * nrhs; t += blockDim.x) {
    const int r = t / nrhs, s = t % nrhs;
    double a = (r < F.nE) ? X[(size_t)gid[r] * nrhs + s] : 0.0;
    if (m0 && m0[r] >= 0) a += v0[(size_t)m0[r] * nrhs + s];
    if (m1 && m1[r] >= 0) a += v1[(size_t)m1[r] * nrhs + s];
    v[t] = a;
  }
  __syncthreads();
  for (int J = 0; J < F.NE; ++J) {
    const double* Di = B.Dinv + (size_t)J * TT;
    for (int t = threadIdx.x; t < TB * nrhs; t += blockDim.x) {
      const int i = t / nrhs, s = t % nrhs;
      double a = 0.0;
#pragma unroll 8
      for (int k = 0; k < TB; ++k) a += Di[i * TB + k] * v[(size_t)(J * TB + k) * nrhs + s];
      ys[t] = a;
    }
    __syncthreads();
    for (int t = threadIdx.x; t < TB * nrhs; t += blockDim.x) v[(size_t)J * TB * nrhs + t] = ys[t];
    for (int t = threadIdx.x; t < (F.NT - 1 - J) * TB * nrhs; t += blockDim.x) {
      const int rr = t / nrhs, s = t % nrhs, I = J + 1 + rr / TB, i = rr % TB;
      const double* Lt = btile(B.Lo, B, J, I - J) + i * TB;
      double a = 0.0;
#pragma unroll 8
      for (int k = 0; k < TB; ++k) a += Lt[k] * ys[k * nrhs + s];
      v[(size_t)(I * TB + i) * nrhs + s] -= a;
    }
    __syncthreads();
  }
}
// Backward solve, CTA per front (levels root first): x_B from X (solved
// ancestors), x_J = Dinv_J^T (y_J - sum_{I>J} L_{I,J}^T x_I), x_E -> X.
__global__ void __launch_bounds__(256) k_mf_bwd(MfDev d, int l0, double* __restrict__ X, double* __restrict__ V,
                                                int nrhs) {
  extern __shared__ __align__(16) double ys[];     // TB x nrhs
  const MfFront F = d.fr[d.lvl[l0 + blockIdx.x]];
  const Band B = mf_band(d.base, F);
  const int* gid = d.gid + F.goff;
  double* v = V + (size_t)F.voff * nrhs;
  for (int t = threadIdx.x; t < (F.NT - F.NE) * TB * nrhs; t += blockDim.x) {
    const int r = F.NE * TB + t / nrhs, s = t % nrhs;
    v[(size_t)r * nrhs + s] = gid[r] >= 0 ? X[(size_t)gid[r] * nrhs + s] : 0.0;
  }
  __syncthreads();
  for (int J = F.NE - 1; J >= 0; --J) {
    for (int t = threadIdx.x; t < TB * nrhs; t += blockDim.x) {
      const int j = t / nrhs, s = t % nrhs;
      double a = v[(size_t)(J * TB + j) * nrhs + s];
      for (int I = J + 1; I < F.NT; ++I) {
        const double* Lt = btile(B.Lo, B, J, I - J);
#pragma unroll 8
        for (int i = 0; i < TB; ++i) a -= Lt[i * TB + j] * v[(size_t)(I * TB + i) * nrhs + s];
      }
      ys[t] = a;
    }
    __syncthreads();
    const double* Di = B.Dinv + (size_t)J * TT;
    for (int t = threadIdx.x; t < TB * nrhs; t += blockDim.x) {
      const int j = t / nrhs, s = t % nrhs;
      double a = 0.0;
#pragma unroll 8
      for (int k = 0; k < TB; ++k) a += Di[k * TB + j] * ys[k * nrhs + s];
      v[(size_t)(J * TB + j) * nrhs + s] = a;
    }
    __syncthreads();
  }
  for (int t = threadIdx.x; t < F.nE * nrhs; t += blockDim.x) {
    const int r = t / nrhs, s = t % nrhs;
    X[(size_t)gid[r] * nrhs + s] = v[t];
  }
}

// Shared-memory versions (the front vector, Dinv_J and L's tile column J
// staged per step; coalesced tile loads, no global round trips in the dot
// products).  smem: V rows*nrhs + (NT-1) tiles + 1 tile + TB*nrhs.
// Dinv_J and L's tile column J (contiguous) arrive by two bulk copies on one
// mbarrier (issued by thread 0; the caller waits on the returned phase).
__device__ __forceinline__ void mf_stage_tma(double* Dj, double* Ls, const Band& B, int J, int nb,
                                             unsigned long long* bar) {
  if (threadIdx.x == 0) {
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    const unsigned bd = TT * sizeof(double), bl = (unsigned)nb * TT * sizeof(double);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bd + bl)
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     smem_u32(Dj)),
                 "l"(B.Dinv + (size_t)J * TT), "r"(bd), "r"(smem_u32(bar))
                 : "memory");
    if (nb > 0)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                       smem_u32(Ls)),
                   "l"(btile(B.Lo, B, J, 1)), "r"(bl), "r"(smem_u32(bar))
                   : "memory");
  }
}
__global__ void __launch_bounds__(256) k_mf_fwd_s(MfDev d, int l0, const double* __restrict__ X,
                                                  double* __restrict__ Vg, int nrhs, int ntmax) {
  extern __shared__ __align__(16) double sh[];
  const MfFront F = d.fr[d.lvl[l0 + blockIdx.x]];
  const Band B = mf_band(d.base, F);
  const int* gid = d.gid + F.goff;
  const int rows = F.NT * TB;
  double* V = sh;                                   // rows x nrhs
  double* Ls = V + (size_t)ntmax * TB * nrhs;       // (NT-1) tiles
  double* Dj = Ls + (size_t)(ntmax - 1) * TT;       // 1 tile
  double* ys = Dj + TT;                             // TB x nrhs
  const bool pairs = !(nrhs & 1) && nrhs <= 64 && (int)blockDim.x % (nrhs >> 1) == 0;
  __shared__ __align__(8) unsigned long long bar;
  if (threadIdx.x == 0) mbar_init(&bar);
  unsigned phase = 0;
  const double* v0 = F.c[0] >= 0 ? Vg + (size_t)d.fr[F.c[0]].voff * nrhs : nullptr;
  const double* v1 = F.c[1] >= 0 ? Vg + (size_t)d.fr[F.c[1]].voff * nrhs : nullptr;
  const int* m0 = v0 ? d.maps + F.moff[0] : nullptr;
  const int* m1 = v1 ? d.maps + F.moff[1] : nullptr;
  // gather indices first (coalesced), then the values with several loads in
  // flight per thread
  int* ix = reinterpret_cast<int*>(ys + TB * nrhs);   // 3 x rows
  for (int r = threadIdx.x; r < rows; r += blockDim.x) {
    ix[r] = r < F.nE ? gid[r] : -1;
    ix[rows + r] = m0 ? m0[r] : -1;
    ix[2 * rows + r] = m1 ? m1[r] : -1;
  }
  __syncthreads();
#pragma unroll 4
  for (int t = threadIdx.x; t < rows * nrhs; t += blockDim.x) {
    const int r = t / nrhs, s = t % nrhs;
    const int a0 = ix[r], a1 = ix[rows + r], a2 = ix[2 * rows + r];
    double a = a0 >= 0 ? __ldcg(X + (size_t)a0 * nrhs + s) : 0.0;
    if (a1 >= 0) a += __ldcg(v0 + (size_t)a1 * nrhs + s);
    if (a2 >= 0) a += __ldcg(v1 + (size_t)a2 * nrhs + s);
    V[t] = a;
  }
  __syncthreads();
  for (int J = 0; J < F.NE; ++J) {
    const int nb = F.NT - 1 - J;
    mf_stage_tma(Dj, Ls, B, J, nb, &bar);
    mbar_wait(&bar, phase);
    phase ^= 1;
    if (pairs) {
      // 2 rows x 2 right-hand sides per thread, double2 shared loads
      const int ncp = nrhs >> 1, cp = threadIdx.x % ncp, rp = threadIdx.x / ncp, rstep = 2 * (blockDim.x / ncp);
      const double* vJ = V + (size_t)J * TB * nrhs;
      for (int r0 = 2 * rp; r0 < TB; r0 += rstep) {
        double a00 = 0, a01 = 0, a10 = 0, a11 = 0;
#pragma unroll
        for (int k = 0; k < TB; k += 2) {
          const double2 l0 = *reinterpret_cast<const double2*>(Dj + r0 * TB + k);
          const double2 l1 = *reinterpret_cast<const double2*>(Dj + (r0 + 1) * TB + k);
          const double2 y0 = *reinterpret_cast<const double2*>(vJ + k * nrhs + 2 * cp);
          const double2 y1 = *reinterpret_cast<const double2*>(vJ + (k + 1) * nrhs + 2 * cp);
          a00 = fma(l0.x, y0.x, fma(l0.y, y1.x, a00));
          a01 = fma(l0.x, y0.y, fma(l0.y, y1.y, a01));
          a10 = fma(l1.x, y0.x, fma(l1.y, y1.x, a10));
          a11 = fma(l1.x, y0.y, fma(l1.y, y1.y, a11));
        }
        *reinterpret_cast<double2*>(ys + r0 * nrhs + 2 * cp) = make_double2(a00, a01);
        *reinterpret_cast<double2*>(ys + (r0 + 1) * nrhs + 2 * cp) = make_double2(a10, a11);
      }
      __syncthreads();
      for (int t = threadIdx.x; t < TB * nrhs; t += blockDim.x) V[(size_t)J * TB * nrhs + t] = ys[t];
      double* vN = V + (size_t)(J + 1) * TB * nrhs;
      for (int r0 = 2 * rp; r0 < nb * TB; r0 += rstep) {
        double a00 = 0, a01 = 0, a10 = 0, a11 = 0;
#pragma unroll
        for (int k = 0; k < TB; k += 2) {
          const double2 l0 = *reinterpret_cast<const double2*>(Ls + (size_t)r0 * TB + k);
          const double2 l1 = *reinterpret_cast<const double2*>(Ls + (size_t)(r0 + 1) * TB + k);
          const double2 y0 = *reinterpret_cast<const double2*>(ys + k * nrhs + 2 * cp);
          const double2 y1 = *reinterpret_cast<const double2*>(ys + (k + 1) * nrhs + 2 * cp);
          a00 = fma(l0.x, y0.x, fma(l0.y, y1.x, a00));
          a01 = fma(l0.x, y0.y, fma(l0.y, y1.y, a01));
          a10 = fma(l1.x, y0.x, fma(l1.y, y1.x, a10));
          a11 = fma(l1.x, y0.y, fma(l1.y, y1.y, a11));
        }
        double2* o0 = reinterpret_cast<double2*>(vN + (size_t)r0 * nrhs + 2 * cp);
        double2* o1 = reinterpret_cast<double2*>(vN + (size_t)(r0 + 1) * nrhs + 2 * cp);
        const double2 p0 = *o0, p1 = *o1;
        *o0 = make_double2(p0.x - a00, p0.y - a01);
        *o1 = make_double2(p1.x - a10, p1.y - a11);
      }
      __syncthreads();
      continue;
    }
    for (int t = threadIdx.x; t < TB * nrhs; t += blockDim.x) {
      const int i = t / nrhs, s = t % nrhs;
      const double* vj = V + (size_t)J * TB * nrhs + s;
      double a = 0.0, b = 0.0;
#pragma unroll
      for (int k = 0; k < TB; k += 2) {
        a = fma(Dj[i * TB + k], vj[k * nrhs], a);
        b = fma(Dj[i * TB + k + 1], vj[(k + 1) * nrhs], b);
      }
      ys[t] = a + b;
    }
    __syncthreads();
    for (int t = threadIdx.x; t < TB * nrhs; t += blockDim.x) V[(size_t)J * TB * nrhs + t] = ys[t];
    for (int t = threadIdx.x; t < nb * TB * nrhs; t += blockDim.x) {
      const int rr = t / nrhs, s = t % nrhs;
      const double* Lr = Ls + (size_t)rr * TB;
      double a = 0.0, b = 0.0;
#pragma unroll
      for (int k = 0; k < TB; k += 2) {
        a = fma(Lr[k], ys[k * nrhs + s], a);
        b = fma(Lr[k + 1], ys[(k + 1) * nrhs + s], b);
      }
      V[(size_t)((J + 1) * TB + rr) * nrhs + s] -= a + b;
    }
    __syncthreads();
  }
  double* v = Vg + (size_t)F.voff * nrhs;
  for (int t = threadIdx.x; t < rows * nrhs; t += blockDim.x) v[t] = V[t];
}
__global__ void __launch_bounds__(256) k_mf_bwd_s(MfDev d, int l0, double* __restrict__ X, const double* __restrict__ Vg,
                                                  int nrhs, int ntmax) {
  extern __shared__ __align__(16) double sh[];
  const MfFront F = d.fr[d.lvl[l0 + blockIdx.x]];
  const Band B = mf_band(d.base, F);
  const int* gid = d.gid + F.goff;
  const int rows = F.NT * TB;
  double* V = sh;
  double* Ls = V + (size_t)ntmax * TB * nrhs;
  double* Dj = Ls + (size_t)(ntmax - 1) * TT;
  double* ys = Dj + TT;
  const bool pairs = !(nrhs & 1) && nrhs <= 64 && ((int)blockDim.x / 2) % (nrhs >> 1) == 0;
  double* ps = ys + TB * nrhs + (3 * ntmax * TB + 1) / 2;   // 2 x TB x nrhs partial sums (after ix)
  __shared__ __align__(8) unsigned long long bar;
  if (threadIdx.x == 0) mbar_init(&bar);
  unsigned phase = 0;
  const double* v = Vg + (size_t)F.voff * nrhs;
  int* ix = reinterpret_cast<int*>(ys + TB * nrhs);
  for (int r = threadIdx.x; r < rows; r += blockDim.x) ix[r] = gid[r];
  __syncthreads();
#pragma unroll 4
  for (int t = threadIdx.x; t < rows * nrhs; t += blockDim.x) {
    const int r = t / nrhs, s = t % nrhs;
    const int a0 = ix[r];
    V[t] = r < F.NE * TB ? __ldcg(v + t) : (a0 >= 0 ? __ldcg(X + (size_t)a0 * nrhs + s) : 0.0);
  }
  __syncthreads();
  for (int J = F.NE - 1; J >= 0; --J) {
    const int nb = F.NT - 1 - J;
    mf_stage_tma(Dj, Ls, B, J, nb, &bar);
    mbar_wait(&bar, phase);
    phase ^= 1;
    if (pairs) {
      // r = y_J - L^T x: 2 columns x 2 right-hand sides per thread, the
      // row sum split over the two thread halves (partials through Dj's
      // neighbour buffer ps), then x_J = Dinv_J^T r
      const int ncp = nrhs >> 1, half = blockDim.x / 2, th = threadIdx.x % half, hs = threadIdx.x / half;
      const int cp = th % ncp, jp = th / ncp, jstep = 2 * (half / ncp);
      const double* vb = V + (size_t)(J + 1) * TB * nrhs;
      const int R = nb * TB, r0 = hs ? R / 2 : 0, r1 = hs ? R : R / 2;
      for (int j0 = 2 * jp; j0 < TB; j0 += jstep) {
        double a00 = 0, a01 = 0, a10 = 0, a11 = 0;
        for (int rr = r0; rr < r1; ++rr) {
          const double2 l = *reinterpret_cast<const double2*>(Ls + (size_t)rr * TB + j0);
          const double2 x = *reinterpret_cast<const double2*>(vb + (size_t)rr * nrhs + 2 * cp);
          a00 = fma(l.x, x.x, a00);
          a01 = fma(l.x, x.y, a01);
          a10 = fma(l.y, x.x, a10);
          a11 = fma(l.y, x.y, a11);
        }
        double* pp = ps + (size_t)hs * TB * nrhs;
        *reinterpret_cast<double2*>(pp + j0 * nrhs + 2 * cp) = make_double2(a00, a01);
        *reinterpret_cast<double2*>(pp + (j0 + 1) * nrhs + 2 * cp) = make_double2(a10, a11);
      }
      __syncthreads();
      for (int t = threadIdx.x; t < TB * nrhs; t += blockDim.x)
        ys[t] = V[(size_t)J * TB * nrhs + t] - (ps[t] + ps[TB * nrhs + t]);
      __syncthreads();
      {
        const int cq = threadIdx.x % ncp, jq = threadIdx.x / ncp, js = 2 * ((int)blockDim.x / ncp);
        for (int j0 = 2 * jq; j0 < TB; j0 += js) {
          double a00 = 0, a01 = 0, a10 = 0, a11 = 0;
#pragma unroll
          for (int k = 0; k < TB; ++k) {
            const double2 dd = *reinterpret_cast<const double2*>(Dj + k * TB + j0);
            const double2 rr = *reinterpret_cast<const double2*>(ys + k * nrhs + 2 * cq);
            a00 = fma(dd.x, rr.x, a00);
            a01 = fma(dd.x, rr.y, a01);
            a10 = fma(dd.y, rr.x, a10);
            a11 = fma(dd.y, rr.y, a11);
          }
          *reinterpret_cast<double2*>(V + (size_t)(J * TB + j0) * nrhs + 2 * cq) = make_double2(a00, a01);
          *reinterpret_cast<double2*>(V + (size_t)(J * TB + j0 + 1) * nrhs + 2 * cq) = make_double2(a10, a11);
        }
      }
      __syncthreads();
      continue;
    }
    for (int t = threadIdx.x; t < TB * nrhs; t += blockDim.x) {
      const int j = t / nrhs, s = t % nrhs;
      const double* vb = V + (size_t)(J + 1) * TB * nrhs + s;
      double a = V[(size_t)(J * TB + j) * nrhs + s], b = 0.0;
      for (int rr = 0; rr < nb * TB; rr += 2) {
        a = fma(-Ls[(size_t)rr * TB + j], vb[(size_t)rr * nrhs], a);
        b = fma(-Ls[(size_t)(rr + 1) * TB + j], vb[(size_t)(rr + 1) * nrhs], b);
      }
      ys[t] = a + b;
    }
    __syncthreads();
    for (int t = threadIdx.x; t < TB * nrhs; t += blockDim.x) {
      const int j = t / nrhs, s = t % nrhs;
      double a = 0.0, b = 0.0;
#pragma unroll
      for (int k = 0; k < TB; k += 2) {
        a = fma(Dj[k * TB + j], ys[k * nrhs + s], a);
        b = fma(Dj[(k + 1) * TB + j], ys[(k + 1) * nrhs + s], b);
      }
      V[(size_t)(J * TB + j) * nrhs + s] = a + b;
    }
    __syncthreads();
  }
  for (int t = threadIdx.x; t < F.nE * nrhs; t += blockDim.x) {
    const int r = t / nrhs, s = t % nrhs;
    X[(size_t)gid[r] * nrhs + s] = V[t];
  }
}

// Explicit front inverse blocks G = [L_EE^-1; -L_BE L_EE^-1] and G^T
// (k_mf_inv_all below).  With them a front's forward solve is
// [y_E; c_B] = G v_E + [0; v_B] and its backward solve x_E = G^T [y_E; x_B]:
// one matrix product per front, so a coarse solve has the depth of the tree
// (6 levels at config 4) instead of 26 tile steps.
// one bulk copy global -> shared on an mbarrier (thread 0 issues; all wait)
__device__ __forceinline__ void mf_tma1(double* dst, const double* src, unsigned bytes, unsigned long long* bar) {
  if (threadIdx.x == 0) {
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
  }
}
// All explicit inverse blocks of the factorization in ONE launch (replaces the
// per-level k_mf_inv / k_mf_invB pairs, which ran between the levels'
// factor launches although only the solves read G): item = (front, tile
// column c, 8-column slice s).  The CTA (4 warps) runs the forward
// substitution L_EE Y = I(:, 8 columns) with Y (rows x 8) in shared memory,
// then G_B = -L_BE Y.  The tile sequence (Dinv_J, L_{J+1,J} .. L_{NE-1,J} per
// step J, then the B rows) is known in advance, so the 32x32 tiles stream
// through a ring of MF_INV_NS padded shared-memory stages filled by cp.async
// (MF_INV_NS - 1 tiles in flight: the chain is not bound by L2 latency);
// each tile product (32x32 by 32x8) is 8 DMMAs per warp.  Items are sorted by
// chain length (host, mf_upload), longest first.
constexpr int MF_INV2_THREADS = 128;
__device__ __forceinline__ void cp_async16(double* dst, const double* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }
struct MfInvCur {
  int ph, J, I;
};
__global__ void __launch_bounds__(MF_INV2_THREADS) k_mf_inv_all(MfDev d, const int4* __restrict__ items) {
  extern __shared__ __align__(16) double sh[];
  const int4 it = items[blockIdx.x];
  const MfFront F = d.fr[it.x];
  const int c = it.y, s = it.z;
  const Band B = mf_band(d.base, F);
  const int NE = F.NE, NT = F.NT;
  double* V = sh;                                   // NE*TB x 8
  double* ring = V + (size_t)NE * TB * MF_INV_W;    // MF_INV_NS x TB x MF_INV_LD
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, m = lane >> 2, q = lane & 3;
  const int col0 = c * TB + s * MF_INV_W;
  for (int t = tid; t < NE * TB * MF_INV_W; t += MF_INV2_THREADS)
    V[t] = (t / MF_INV_W == col0 + t % MF_INV_W) ? 1.0 : 0.0;
  const int n1 = (NE - c) * (NE - c + 1) / 2, ntot = n1 + (NT - NE) * (NE - c);
  auto next = [&](MfInvCur& u) {
    if (u.ph == 1) {
      if (++u.I >= NE) {
        ++u.J;
        u.I = u.J;
        if (u.J >= NE) u = {2, c, NE};
      }
    } else if (++u.J >= NE) {
      u.J = c;
      ++u.I;
    }
  };
  auto issue = [&](int n, const MfInvCur& u) {
    if (n < ntot) {
      const double* src = u.I == u.J ? B.Dinv + (size_t)u.J * TT : btile(B.Lo, B, u.J, u.I - u.J);
      double* dst = ring + (size_t)(n % MF_INV_NS) * TB * MF_INV_LD;
#pragma unroll
      for (int k = 0; k < TT / 2 / MF_INV2_THREADS; ++k) {
        const int ch = tid + MF_INV2_THREADS * k, r = ch / (TB / 2), c2 = ch % (TB / 2);
        cp_async16(dst + r * MF_INV_LD + 2 * c2, src + r * TB + 2 * c2);
      }
    }
    cp_async_commit();
  };
  MfInvCur ui{1, c, c}, uc{1, c, c};
  for (int n = 0; n < MF_INV_NS - 1; ++n) {
    issue(n, ui);
    next(ui);
  }
  // O (8 rows 8w.., 8 columns) = tile rows 8w.. times Y (32 x 8, stride 8)
  auto prod = [&](const double* T, const double* Y) -> F2c {
    F2c a = {0.0, 0.0}, b = {0.0, 0.0};
    const double* Tr = T + (8 * w + m) * MF_INV_LD + q;
    const double* Yr = Y + q * MF_INV_W + m;
#pragma unroll
    for (int kk = 0; kk < 8; kk += 2) {
      dmma(a.x, a.y, Tr[4 * kk], Yr[4 * kk * MF_INV_W]);
      dmma(b.x, b.y, Tr[4 * kk + 4], Yr[(4 * kk + 4) * MF_INV_W]);
    }
    return {a.x + b.x, a.y + b.y};
  };
  double* G = d.base + F.goff2;
  const int frows = NT * TB, ncol = NE * TB;
  double* GT = G + (size_t)NT * NE * TT;
  F2c acc = {0.0, 0.0};
  for (int n = 0; n < ntot; ++n) {
    cp_async_wait<MF_INV_NS - 2>();
    __syncthreads();                       // tile n landed for every thread; stage (n-1) % NS is free
    issue(n + MF_INV_NS - 1, ui);
    next(ui);
    const double* T = ring + (size_t)(n % MF_INV_NS) * TB * MF_INV_LD;
    double* VJ = V + (size_t)uc.J * TB * MF_INV_W;
    const F2c o = prod(T, VJ);
    if (uc.ph == 1) {
      if (uc.I == uc.J) {                  // Y_J = Dinv_J v_J (every warp has read v_J before any row changes)
        __syncthreads();
        *reinterpret_cast<double2*>(VJ + (8 * w + m) * MF_INV_W + 2 * q) = make_double2(o.x, o.y);
      } else {                             // v_I -= L_{I,J} Y_J (own rows)
        double2* p = reinterpret_cast<double2*>(V + ((size_t)uc.I * TB + 8 * w + m) * MF_INV_W + 2 * q);
        const double2 v = *p;
        *p = make_double2(v.x - o.x, v.y - o.y);
      }
    } else {                               // G_B[I] = -sum_J L_{I,J} Y_J
      acc.x += o.x;
      acc.y += o.y;
      if (uc.J == NE - 1) {
        const int r = uc.I * TB + 8 * w + m, cq = col0 + 2 * q;
        *reinterpret_cast<double2*>(G + (size_t)r * ncol + cq) = make_double2(-acc.x, -acc.y);
        GT[(size_t)cq * frows + r] = -acc.x;
        GT[(size_t)(cq + 1) * frows + r] = -acc.y;
        acc = {0.0, 0.0};
      }
    }
    next(uc);
  }
  __syncthreads();
  const int rows = NE * TB;
  for (int t = tid; t < rows * MF_INV_W; t += MF_INV2_THREADS) {
    const int r = t / MF_INV_W, qq = t % MF_INV_W;
    G[(size_t)r * ncol + col0 + qq] = V[t];
  }
  for (int t = tid; t < rows * MF_INV_W; t += MF_INV2_THREADS) {
    const int qq = t / rows, r = t % rows;
    GT[(size_t)(col0 + qq) * frows + r] = V[(size_t)r * MF_INV_W + qq];
  }
}

// Forward solve of one level with G: CTA (front, 16-row chunk): the chunk of
// G arrives by one bulk copy while v_E is gathered (X on E + the children's
// c_B); out = G v_E (+ the children's c_B on B rows).
__global__ void __launch_bounds__(256) k_mf_gfwd(MfDev d, int l0, const double* __restrict__ X,
                                                 double* __restrict__ Vg, int nrhs) {
  extern __shared__ __align__(16) double sh[];
  __shared__ __align__(8) unsigned long long bar;
  const MfFront F = d.fr[d.lvl[l0 + blockIdx.x]];
  const int rows = F.NT * TB, ncol = F.NE * TB, r0c = blockIdx.y * MF_GR;
  if (r0c >= rows) return;
  const int nr = min(MF_GR, rows - r0c);
  const int* gid = d.gid + F.goff;
  const double* v0 = F.c[0] >= 0 ? Vg + (size_t)d.fr[F.c[0]].voff * nrhs : nullptr;
  const double* v1 = F.c[1] >= 0 ? Vg + (size_t)d.fr[F.c[1]].voff * nrhs : nullptr;
  const int* m0 = v0 ? d.maps + F.moff[0] : nullptr;
  const int* m1 = v1 ? d.maps + F.moff[1] : nullptr;
  double* Gs = sh;                                    // MF_GR x ncol
  double* vE = Gs + (size_t)MF_GR * ncol;             // ncol x nrhs
  if (threadIdx.x == 0) mbar_init(&bar);
  __syncthreads();
  mf_tma1(Gs, d.base + F.goff2 + (size_t)r0c * ncol, (unsigned)(nr * ncol * sizeof(double)), &bar);
  auto gat = [&](int r, int s) {
    double a = (r < F.nE) ? __ldcg(X + (size_t)gid[r] * nrhs + s) : 0.0;
    if (m0) { const int q = m0[r]; if (q >= 0) a += __ldcg(v0 + (size_t)q * nrhs + s); }
    if (m1) { const int q = m1[r]; if (q >= 0) a += __ldcg(v1 + (size_t)q * nrhs + s); }
    return a;
  };
#pragma unroll 4
  for (int t = threadIdx.x; t < ncol * nrhs; t += blockDim.x) vE[t] = gat(t / nrhs, t % nrhs);
  __syncthreads();
  mbar_wait(&bar, 0);
  double* v = Vg + (size_t)F.voff * nrhs;
  for (int t = threadIdx.x; t < nr * nrhs; t += blockDim.x) {
    const int i = t / nrhs, s = t % nrhs, r = r0c + i;
    const double* Gr = Gs + (size_t)i * ncol;
    const int kend = r < ncol ? min(ncol, (r / TB + 1) * TB) : ncol;   // L_EE^-1 is block lower triangular
    double a = 0.0, b = 0.0;
    for (int k = 0; k < kend; k += 2) {
      a = fma(Gr[k], vE[k * nrhs + s], a);
      b = fma(Gr[k + 1], vE[(k + 1) * nrhs + s], b);
    }
    a += b;
    if (r >= ncol) a += gat(r, s);
    v[(size_t)r * nrhs + s] = a;
  }
}
// Backward solve of one level with G^T: CTA (front, 16-row chunk of x_E):
// z = [y_E ; x_B] gathered, x_E = G^T z -> X.
__global__ void __launch_bounds__(256) k_mf_gbwd(MfDev d, int l0, double* __restrict__ X,
                                                 const double* __restrict__ Vg, int nrhs) {
  extern __shared__ __align__(16) double sh[];
  __shared__ __align__(8) unsigned long long bar;
  const MfFront F = d.fr[d.lvl[l0 + blockIdx.x]];
  const int j0 = blockIdx.y * MF_GR;
  if (j0 >= F.nE) return;
  const int nj = min(MF_GR, F.nE - j0);
  const int rows = F.NT * TB, ncol = F.NE * TB;
  const int rz0 = (j0 / TB) * TB;                    // G^T rows of this chunk vanish before their block
  const int* gid = d.gid + F.goff;
  const double* v = Vg + (size_t)F.voff * nrhs;
  double* Gs = sh;                                   // MF_GR x rows (columns rz0.. used)
  double* z = Gs + (size_t)MF_GR * rows;             // rows x nrhs
  if (threadIdx.x == 0) mbar_init(&bar);
  __syncthreads();
  mf_tma1(Gs, d.base + F.goff2 + (size_t)F.NT * F.NE * TT + (size_t)j0 * rows,
          (unsigned)(nj * rows * sizeof(double)), &bar);
#pragma unroll 4
  for (int t = threadIdx.x; t < (rows - rz0) * nrhs; t += blockDim.x) {
    const int r = rz0 + t / nrhs, s = t % nrhs;
    z[(size_t)r * nrhs + s] = r < ncol ? __ldcg(v + (size_t)r * nrhs + s)
                                       : (gid[r] >= 0 ? __ldcg(X + (size_t)gid[r] * nrhs + s) : 0.0);
  }
  __syncthreads();
  mbar_wait(&bar, 0);
  for (int t = threadIdx.x; t < nj * nrhs; t += blockDim.x) {
    const int i = t / nrhs, s = t % nrhs, j = j0 + i;
    const double* Gr = Gs + (size_t)i * rows;
    double a = 0.0, b = 0.0;
    for (int r = rz0; r < rows; r += 2) {
      a = fma(Gr[r], z[(size_t)r * nrhs + s], a);
      b = fma(Gr[r + 1], z[(size_t)(r + 1) * nrhs + s], b);
    }
    X[(size_t)gid[j] * nrhs + s] = a + b;
  }
}

// Both sweeps of a coarse solve in one cooperative launch.  Per level:
// (A) grid-wide gather of every front's input vector into Vin (independent
// loads on all SMs), grid barrier; (B) (front, 16-row chunk) items: the chunk
// of G (forward) or G^T (backward) and the input rows it needs arrive by bulk
// copies, one product, result to Vout (forward) or X (backward); grid barrier.
struct MfSolveJob {
  MfDev d;
  const int* lvl_off;   // device copy of the level offsets
  int nl;
  double* X;            // right-hand sides in, solution out (k x nrhs, natural order)
  double* Vout;         // per-front outputs (y_E | c_B), Σ rows x nrhs
  double* Vin;          // per-front gathered inputs, Σ rows x nrhs
  int nrhs;
  unsigned long long* tstamp;   // debug (MSFV_MF_TIMING): globaltimer after every grid barrier
  const int* pre;       // MfPlan::d_pre
  int npre;
  int kchunk;           // > 0: pipelined K-chunked products with this many input rows per chunk
  const MfFront* frl;   // MfPlan::d_frl
  int lvl_off_total;    // number of fronts
  const int4* gtab;     // MfPlan::d_gtab
  const int* rowbase;   // MfPlan::d_rowbase
  int vrows;
};
__device__ __forceinline__ void mf_bulk_raw(double* dst, const double* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// Work unit of the pipelined products: one (front, MF_GR-row chunk) item of a
// level's phase (B).  Rows of G (forward) or G^T (backward) start at G0 with
// stride gstride; the product runs over input rows [kbeg, kmax) of vin.
struct MfItem {
  const double* G0;
  const double* vin;
  size_t gstride;
  int nr, kbeg, kmax;
  int r0;        // first output row (forward: front row r0c, backward: E row j0)
  int fi;        // front (level-local)
};
__device__ __forceinline__ void mf_stamp(unsigned long long* ts, int i) {
  if (ts && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    ts[i] = t;
  }
}
constexpr int MF_FCACHE = 128;   // front descriptors cached per level in the coop solve
constexpr int MF_PRE_CAP = 640;  // prefix entries (fronts + levels) of a tree cached whole by the coop solve
constexpr int MF_COOP_STATIC = 36864;   // static shared memory of k_mf_solve_coop, rounded up
__global__ void __launch_bounds__(256, 1) k_mf_solve_coop(MfSolveJob job) {
  extern __shared__ __align__(16) double sh[];
  __shared__ __align__(8) unsigned long long bar;
  __shared__ __align__(8) unsigned long long bars2[2];   // the two buffers of the pipelined products
  __shared__ int pre_s[MF_MAXF + 1], preB_s[MF_MAXF + 1];
  __shared__ MfFront fc_s[MF_FCACHE];
  // Small trees (config 4: 63 fronts): the prefix sums of every (pass, level) and all front descriptors
  // are fetched once at kernel start, so a level phase starts without a global round trip and a barrier.
  __shared__ int preAll[3 * MF_PRE_CAP];
  const bool all_cached = job.npre <= MF_PRE_CAP && job.lvl_off_total <= MF_FCACHE;
  if (all_cached) {
    for (int i = threadIdx.x; i < 3 * job.npre; i += blockDim.x)
      preAll[(i / job.npre) * MF_PRE_CAP + i % job.npre] = job.pre[i] * (i < job.npre ? job.nrhs : 1);
    for (int i = threadIdx.x; i < job.lvl_off_total; i += blockDim.x) fc_s[i] = job.frl[i];
  }
  const int* pre = pre_s;
  const int* preB = preB_s;
  const MfFront* fc = fc_s;
  int fcn = 0;                       // descriptors available through fc[]
  int4 t4n[4];                       // prefetched gather-table entries of the next level phase
  bool have_next = false;
  cg::grid_group grid = cg::this_grid();
  if (threadIdx.x == 0) {
    mbar_init(&bar);
    mbar_init(&bars2[0]);
    mbar_init(&bars2[1]);
  }
  __syncthreads();
  unsigned ph = 0, phs2 = 0u;   // phs2: parity bits of bars2
  int nst = 0;
  mf_stamp(job.tstamp, nst++);
  const MfDev& d = job.d;
  const int nrhs = job.nrhs;
  const long long gtid = blockIdx.x * (long long)blockDim.x + threadIdx.x, gstride = (long long)gridDim.x * blockDim.x;
  for (int pass = 0; pass < 2; ++pass) {
    for (int li = 0; li < job.nl; ++li) {
      const int l = pass == 0 ? li : job.nl - 1 - li;
      const int l0 = job.lvl_off[l], nf = job.lvl_off[l + 1] - l0;
      // ---- (A) gather: flat index over the level's fronts (rows x nrhs
      // each); the level's front descriptors are cached in shared memory and
      // each thread keeps four elements' loads in flight
      // (descriptors and both phases' prefix sums in one round of loads)
      if (all_cached) {
        pre = preAll + l0 + l;
        preB = preAll + (pass == 0 ? 1 : 2) * MF_PRE_CAP + l0 + l;
        fc = fc_s + l0;
        fcn = nf;
      } else {
        for (int i = threadIdx.x; i < nf && i < MF_FCACHE; i += blockDim.x) fc_s[i] = job.frl[l0 + i];
        for (int i = threadIdx.x; i <= nf; i += blockDim.x) {
          pre_s[i] = job.pre[l0 + l + i] * nrhs;
          preB_s[i] = job.pre[(pass == 0 ? 1 : 2) * job.npre + l0 + l + i];
        }
        fcn = min(nf, MF_FCACHE);
        __syncthreads();
      }
      {
        // flat index over (front row of the level, right-hand side); four elements' loads in flight per thread
        const long long total = pre[nf];
        const int4* tab = job.gtab + (pass ? job.vrows : 0) + job.rowbase[l];
        for (long long base = gtid; base < total; base += 4 * gstride) {
          double a[4];
          long long dst[4];
          int4 t4[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const long long gi = base + u * gstride;
            if (have_next && base == gtid) t4[u] = t4n[u];     // fetched during the previous level's products
            else t4[u] = gi < total ? __ldg(tab + gi / nrhs) : make_int4(-1, -1, -1, -1);
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const long long gi = base + u * gstride;
            a[u] = 0.0;
            dst[u] = -1;
            if (gi >= total) continue;
            const int s2 = (int)(gi % nrhs);
            const int4 t = t4[u];
            double v = 0.0;
            if (pass == 0) {
              if (t.y >= 0) v = __ldcg(job.X + (size_t)t.y * nrhs + s2);
              if (t.z >= 0) v += __ldcg(job.Vout + (size_t)t.z * nrhs + s2);
              if (t.w >= 0) v += __ldcg(job.Vout + (size_t)t.w * nrhs + s2);
            } else {
              if (t.y >= 0) v = __ldcg(job.Vout + (size_t)t.y * nrhs + s2);
              else if (t.z >= 0) v = __ldcg(job.X + (size_t)t.z * nrhs + s2);
            }
            a[u] = v;
            dst[u] = (long long)t.x * nrhs + s2;
          }
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (dst[u] >= 0) job.Vin[dst[u]] = a[u];
        }
      }
      // the next level phase's table entries (static data) travel while this level's products run
      have_next = false;
      if (all_cached) {
        const int li2 = li + 1 < job.nl ? li + 1 : 0, pass2 = li + 1 < job.nl ? pass : pass + 1;
        if (pass2 < 2) {
          const int l2 = pass2 == 0 ? li2 : job.nl - 1 - li2;
          const int l02 = job.lvl_off[l2], nf2 = job.lvl_off[l2 + 1] - l02;
          const long long total2 = preAll[l02 + l2 + nf2];
          const int4* tab2 = job.gtab + (pass2 ? job.vrows : 0) + job.rowbase[l2];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const long long gi = gtid + u * gstride;
            t4n[u] = gi < total2 ? __ldg(tab2 + gi / nrhs) : make_int4(-1, -1, -1, -1);
          }
          have_next = true;
        }
      }
      grid.sync();
      mf_stamp(job.tstamp, nst++);
      // ---- (B) products
      if (job.kchunk) {
        // Pipelined K-chunked products: the CTA's units (item, chunk of KC
        // input rows) stream through two shared-memory buffers; the copies of
        // the unit after next are issued as soon as a buffer is consumed, so
        // a CTA with many items (config 5: 124 leaf items per CTA) is bound by
        // the copy / FMA time, not by one L2 round trip per item.
        const int KC = job.kchunk, GLD = KC + 4;   // padded G row stride: conflict-free fragment loads
        const size_t bufd = (size_t)MF_GR * GLD + (size_t)KC * nrhs + 8;
        double* red = sh + 2 * bufd;                // k-part partial sums of an item
        // warp (tj, part): 8 right-hand sides tj, k-part `part` of every chunk, both 8-row halves
        const int ntj = (nrhs + 7) >> 3, nparts = max(1, 8 / ntj), RLD = 8 * ntj + 2;
        const int wv = threadIdx.x >> 5, lane = threadIdx.x & 31, mm = lane >> 2, qq = lane & 3;
        const bool wact = wv < ntj * nparts;
        const int tj = wv % ntj, part = wv / ntj;
        const int total = preB[nf];
        auto front = [&](int fi2) { return fi2 < fcn ? fc[fi2] : d.fr[d.lvl[l0 + fi2]]; };
        auto item_of = [&](int gi, int& fi2) {
          while (preB[fi2 + 1] <= gi) ++fi2;
          const MfFront F = front(fi2);
          const int rows = F.NT * TB, ncol = F.NE * TB;
          MfItem it;
          it.vin = job.Vin + (size_t)F.voff * nrhs;
          it.fi = fi2;
          if (pass == 0) {                 // [y_E; c_B] rows r0c.. = G v_E (+ the children's c_B on B rows)
            const int r0c = (gi - preB[fi2]) * MF_GR;
            it.nr = min(MF_GR, rows - r0c);
            it.r0 = r0c;
            it.kbeg = 0;
            it.kmax = r0c < ncol ? min(ncol, ((r0c + it.nr - 1) / TB + 1) * TB) : ncol;
            it.G0 = d.base + F.goff2 + (size_t)r0c * ncol;
            it.gstride = (size_t)ncol;
          } else {                         // x_E rows j0.. = G^T [y_E; x_B]
            const int j0 = (gi - preB[fi2]) * MF_GR;
            it.nr = min(MF_GR, F.nE - j0);
            it.r0 = j0;
            it.kbeg = (j0 / TB) * TB;
            it.kmax = rows;
            it.G0 = d.base + F.goff2 + (size_t)F.NT * F.NE * TT + (size_t)j0 * rows;
            it.gstride = (size_t)rows;
          }
          return it;
        };
        // issue cursor (thread 0 copies; every thread tracks it: cheap and branch-uniform)
        int gi_i = blockIdx.x, fi_i = 0, k_i = 0;
        bool have_i = gi_i < total;
        MfItem it_i{};
        if (have_i) {
          it_i = item_of(gi_i, fi_i);
          k_i = it_i.kbeg;
        }
        auto issue_next = [&](int b) {
          if (!have_i) return;
          const int kc = min(KC, it_i.kmax - k_i);
          if (threadIdx.x < 32) {                  // warp 0: lane 0 arms the barrier, lanes 0..nr-1 copy a row of G each, lane 31 the input rows
            double* Gs = sh + (size_t)b * bufd;
            double* vs = Gs + (size_t)MF_GR * GLD;
            const unsigned bg = (unsigned)(kc * sizeof(double)), bv = (unsigned)(kc * nrhs * sizeof(double));
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            if (threadIdx.x == 0) {
              asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(&bars2[b])),
                           "r"(it_i.nr * bg + bv)
                           : "memory");
            }
            __syncwarp();
            const int ii = threadIdx.x;
            if (ii < it_i.nr)
              mf_bulk_raw(Gs + (size_t)ii * GLD, it_i.G0 + (size_t)ii * it_i.gstride + k_i, bg, &bars2[b]);
            if (ii == 31) mf_bulk_raw(vs, it_i.vin + (size_t)k_i * nrhs, bv, &bars2[b]);
          }
          k_i += KC;
          if (k_i >= it_i.kmax) {
            gi_i += gridDim.x;
            have_i = gi_i < total;
            if (have_i) {
              it_i = item_of(gi_i, fi_i);
              k_i = it_i.kbeg;
            }
          }
        };
        issue_next(0);
        issue_next(1);
        int b = 0, fi_c = 0;
        for (int gi = blockIdx.x; gi < total; gi += gridDim.x) {
          const MfItem it = item_of(gi, fi_c);
          const MfFront F = front(it.fi);
          const int ncol = F.NE * TB;
          double addv[4] = {0.0, 0.0, 0.0, 0.0};
          if (pass == 0 && it.r0 >= ncol) {       // B rows: the children's c_B, fetched while the chunks arrive
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int t = threadIdx.x + 256 * u;
              if (t < it.nr * nrhs) addv[u] = __ldcg(it.vin + (size_t)it.r0 * nrhs + t);
            }
          }
          // (every row of an item has the same k range: an item's 16 rows lie in one 32-row tile)
          F2c c0 = {0.0, 0.0}, c1 = {0.0, 0.0};
          for (int k0 = it.kbeg; k0 < it.kmax; k0 += KC) {
            const int kc = min(KC, it.kmax - k0);
            const double* Gs = sh + (size_t)b * bufd;
            const double* vs = Gs + (size_t)MF_GR * GLD;
            mbar_wait(&bars2[b], (phs2 >> b) & 1u);
            phs2 ^= 1u << b;
            if (wact) {
              const int kp = kc / nparts, kb = part * kp;             // kc is a multiple of 32, nparts of 8
              const double* Ga = Gs + (size_t)mm * GLD + kb + qq;
              const double* Gb = Ga + (size_t)8 * GLD;
              const double* Vb = vs + (size_t)(kb + qq) * nrhs + 8 * tj + mm;
              F2c e0 = {0.0, 0.0}, e1 = {0.0, 0.0};
#pragma unroll 4
              for (int k = 0; k < kp; k += 8) {
                const double b0 = Vb[(size_t)k * nrhs], b1 = Vb[(size_t)(k + 4) * nrhs];
                dmma(c0.x, c0.y, Ga[k], b0);
                dmma(c1.x, c1.y, Gb[k], b0);
                if (k + 4 < kp) {
                  dmma(e0.x, e0.y, Ga[k + 4], b1);
                  dmma(e1.x, e1.y, Gb[k + 4], b1);
                }
              }
              c0.x += e0.x; c0.y += e0.y;
              c1.x += e1.x; c1.y += e1.y;
            }
            __syncthreads();                     // buffer b consumed by every thread
            issue_next(b);
            b ^= 1;
          }
          if (wact) {
            double* rp = red + (size_t)part * 16 * RLD + 8 * tj + 2 * qq;
            rp[(size_t)mm * RLD] = c0.x;
            rp[(size_t)mm * RLD + 1] = c0.y;
            rp[(size_t)(mm + 8) * RLD] = c1.x;
            rp[(size_t)(mm + 8) * RLD + 1] = c1.y;
          }
          __syncthreads();
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int t = threadIdx.x + 256 * u;
            if (t < it.nr * nrhs) {
              const int ii = t / nrhs, s2 = t % nrhs;
              double a = 0.0;
              for (int pp = 0; pp < nparts; ++pp) a += red[((size_t)pp * 16 + ii) * RLD + s2];
              if (pass == 0)
                job.Vout[((size_t)F.voff + it.r0 + ii) * nrhs + s2] = a + addv[u];
              else
                job.X[(size_t)d.gid[F.goff + it.r0 + ii] * nrhs + s2] = a;
            }
          }
        }
      }
      int fi = 0;
      for (int gi = blockIdx.x; gi < preB[nf] && !job.kchunk; gi += gridDim.x) {
        while (preB[fi + 1] <= gi) ++fi;
        const MfFront F = fi < fcn ? fc[fi] : d.fr[d.lvl[l0 + fi]];
        const int rows = F.NT * TB, ncol = F.NE * TB;
        const double* vin = job.Vin + (size_t)F.voff * nrhs;
        if (pass == 0) {
          const int r0c = (gi - preB[fi]) * MF_GR, nr = min(MF_GR, rows - r0c);
          const int kmax = r0c < ncol ? min(ncol, ((r0c + nr - 1) / TB + 1) * TB) : ncol;
          double* Gs = sh;
          double* vs = Gs + (size_t)MF_GR * ncol;
          double* addv = vs + (size_t)ncol * nrhs;
          if (threadIdx.x == 0) {
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            const unsigned bg = (unsigned)(nr * ncol * sizeof(double)), bv = (unsigned)(kmax * nrhs * sizeof(double));
            const unsigned ba = r0c >= ncol ? (unsigned)(nr * nrhs * sizeof(double)) : 0u;
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(&bar)), "r"(bg + bv + ba)
                         : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                             smem_u32(Gs)), "l"(d.base + F.goff2 + (size_t)r0c * ncol), "r"(bg), "r"(smem_u32(&bar))
                         : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                             smem_u32(vs)), "l"(vin), "r"(bv), "r"(smem_u32(&bar))
                         : "memory");
            if (ba)
              asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                               smem_u32(addv)), "l"(vin + (size_t)r0c * nrhs), "r"(ba), "r"(smem_u32(&bar))
                           : "memory");
          }
          mbar_wait(&bar, ph);
          ph ^= 1;
          // rows of the chunk may end at different diagonal blocks: use each row's own bound
          for (int t = threadIdx.x; t < nr * nrhs; t += blockDim.x) {
            const int ii = t / nrhs, s = t % nrhs, r = r0c + ii;
            const double* Gr = Gs + (size_t)ii * ncol;
            const int kend = r < ncol ? min(ncol, (r / TB + 1) * TB) : ncol;
            double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
            int k = 0;
            for (; k + 3 < kend; k += 4) {
              a0 = fma(Gr[k], vs[(size_t)k * nrhs + s], a0);
              a1 = fma(Gr[k + 1], vs[(size_t)(k + 1) * nrhs + s], a1);
              a2 = fma(Gr[k + 2], vs[(size_t)(k + 2) * nrhs + s], a2);
              a3 = fma(Gr[k + 3], vs[(size_t)(k + 3) * nrhs + s], a3);
            }
            for (; k < kend; ++k) a0 = fma(Gr[k], vs[(size_t)k * nrhs + s], a0);
            double a = (a0 + a1) + (a2 + a3);
            if (r >= ncol) a += addv[(size_t)ii * nrhs + s];
            job.Vout[((size_t)F.voff + r) * nrhs + s] = a;
          }
        } else {
          const int j0 = (gi - preB[fi]) * MF_GR, nj = min(MF_GR, F.nE - j0);
          const int rz0 = (j0 / TB) * TB;
          double* Gs = sh;                                 // nj x rows
          double* zs = Gs + (size_t)MF_GR * rows;          // rows x nrhs (from rz0)
          if (threadIdx.x == 0) {
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            const unsigned bg = (unsigned)(nj * rows * sizeof(double)),
                           bz = (unsigned)((rows - rz0) * nrhs * sizeof(double));
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(&bar)), "r"(bg + bz)
                         : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                             smem_u32(Gs)),
                         "l"(d.base + F.goff2 + (size_t)F.NT * F.NE * TT + (size_t)j0 * rows), "r"(bg),
                         "r"(smem_u32(&bar))
                         : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                             smem_u32(zs + (size_t)rz0 * nrhs)), "l"(vin + (size_t)rz0 * nrhs), "r"(bz), "r"(smem_u32(&bar))
                         : "memory");
          }
          mbar_wait(&bar, ph);
          ph ^= 1;
          for (int t = threadIdx.x; t < nj * nrhs; t += blockDim.x) {
            const int ii = t / nrhs, s = t % nrhs, j = j0 + ii;
            const double* Gr = Gs + (size_t)ii * rows;
            double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
            int r = rz0;
            for (; r + 3 < rows; r += 4) {
              a0 = fma(Gr[r], zs[(size_t)r * nrhs + s], a0);
              a1 = fma(Gr[r + 1], zs[(size_t)(r + 1) * nrhs + s], a1);
              a2 = fma(Gr[r + 2], zs[(size_t)(r + 2) * nrhs + s], a2);
              a3 = fma(Gr[r + 3], zs[(size_t)(r + 3) * nrhs + s], a3);
            }
            for (; r < rows; ++r) a0 = fma(Gr[r], zs[(size_t)r * nrhs + s], a0);
            job.X[(size_t)d.gid[F.goff + j] * nrhs + s] = (a0 + a1) + (a2 + a3);
          }
        }
        __syncthreads();
      }
      grid.sync();
      mf_stamp(job.tstamp, nst++);
    }
  }
}

// Solve with scatters instead of gather phases (15 grid barriers instead of
// 29): phase 0 gathers X onto every front's E rows (XE) and zeroes the child
// slots S0/S1; a forward item sums XE + S0 + S1 for its input rows and
// writes y_E (Vout) and its c_B rows straight into its parent's slot
// S_{pslot} at fixed rows (no atomics: each slot row has one writer); a
// backward item reads [y_E; x_B] (x_B in Zb, written by the parent), writes
// x_E to X and to its children's Zb rows.  Zb reuses the XE workspace.
constexpr int MF_CC = 4;     // right-hand sides per CTA of the blocked sweeps (4: more CTAs on the few top fronts)
constexpr int MF_LCH = 8;    // L tiles per streamed chunk (8: half the chunk barriers of 4; config 5 solve 5.8 -> 4.2 ms)
__device__ __forceinline__ void mf_tma_tiles(double* dst, const double* src, int ntile, unsigned long long* bar) {
  if (threadIdx.x == 0) {
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    const unsigned bytes = (unsigned)ntile * TT * sizeof(double);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
  }
}
__global__ void __launch_bounds__(256) k_mf_fwd_c(MfDev d, int l0, const double* __restrict__ X,
                                                  double* __restrict__ Vg, int ld, int ntmax) {
  extern __shared__ __align__(16) double sh[];
  __shared__ __align__(8) unsigned long long bar[3];     // 0, 1: L chunk buffers, 2: Dinv
  const MfFront F = d.fr[d.lvl[l0 + blockIdx.x]];
  const int c0 = blockIdx.y * MF_CC, nc = min(MF_CC, ld - c0);
  if (nc <= 0) return;
  const Band B = mf_band(d.base, F);
  const int rows = F.NT * TB;
  double* V = sh;                                   // rows x MF_CC
  double* Ls = V + (size_t)ntmax * TB * MF_CC;      // 2 x MF_LCH tiles
  double* Dj = Ls + (size_t)2 * MF_LCH * TT;
  double* ys = Dj + TT;                             // TB x MF_CC
  const int* gid = d.gid + F.goff;
  const double* v0 = F.c[0] >= 0 ? Vg + (size_t)d.fr[F.c[0]].voff * ld : nullptr;
  const double* v1 = F.c[1] >= 0 ? Vg + (size_t)d.fr[F.c[1]].voff * ld : nullptr;
  const int* m0 = v0 ? d.maps + F.moff[0] : nullptr;
  const int* m1 = v1 ? d.maps + F.moff[1] : nullptr;
  if (threadIdx.x == 0) {
    mbar_init(&bar[0]);
    mbar_init(&bar[1]);
    mbar_init(&bar[2]);
  }
#pragma unroll 4
  for (int t = threadIdx.x; t < rows * MF_CC; t += blockDim.x) {
    const int r = t / MF_CC, s = t % MF_CC;
    double a = 0.0;
    if (s < nc) {
      if (r < F.nE) a = __ldcg(X + (size_t)gid[r] * ld + c0 + s);
      if (m0) { const int q = m0[r]; if (q >= 0) a += __ldcg(v0 + (size_t)q * ld + c0 + s); }
      if (m1) { const int q = m1[r]; if (q >= 0) a += __ldcg(v1 + (size_t)q * ld + c0 + s); }
    }
    V[t] = a;
  }
  __syncthreads();
  unsigned ph[3] = {0, 0, 0};
  int buf = 0;
  const int cp = threadIdx.x % (MF_CC / 2), rp = threadIdx.x / (MF_CC / 2);   // 2 rows x 2 rhs per thread
  const int rstep = 2 * (blockDim.x / (MF_CC / 2));
  // prologue: Dinv_0 and the first L chunk of column 0
  mf_tma_tiles(Dj, B.Dinv, 1, &bar[2]);
  if (F.NT > 1) mf_tma_tiles(Ls, btile(B.Lo, B, 0, 1), min(MF_LCH, F.NT - 1), &bar[0]);
  bool first_issued = true;                         // the prologue issued column 0's first chunk (if any)
  for (int J = 0; J < F.NE; ++J) {
    const int nb = F.NT - 1 - J;
    if (nb > 0 && !first_issued) mf_tma_tiles(Ls + (size_t)buf * MF_LCH * TT, btile(B.Lo, B, J, 1), min(MF_LCH, nb),
                                              &bar[buf]);
    first_issued = false;
    mbar_wait(&bar[2], ph[2]);
    ph[2] ^= 1;
    for (int r0 = 2 * rp; r0 < TB; r0 += rstep) {
      double a00 = 0, a01 = 0, a10 = 0, a11 = 0;
      const double* vJ = V + (size_t)J * TB * MF_CC;
#pragma unroll 8
      for (int k = 0; k < TB; ++k) {
        const double l0v = Dj[r0 * TB + k], l1v = Dj[(r0 + 1) * TB + k];
        const double2 y = *reinterpret_cast<const double2*>(vJ + k * MF_CC + 2 * cp);
        a00 = fma(l0v, y.x, a00);
        a01 = fma(l0v, y.y, a01);
        a10 = fma(l1v, y.x, a10);
        a11 = fma(l1v, y.y, a11);
      }
      *reinterpret_cast<double2*>(ys + r0 * MF_CC + 2 * cp) = make_double2(a00, a01);
      *reinterpret_cast<double2*>(ys + (r0 + 1) * MF_CC + 2 * cp) = make_double2(a10, a11);
    }
    __syncthreads();                                  // ys complete, Dj consumed
    if (J + 1 < F.NE) mf_tma_tiles(Dj, B.Dinv + (size_t)(J + 1) * TT, 1, &bar[2]);
    for (int t = threadIdx.x; t < TB * MF_CC; t += blockDim.x) V[(size_t)J * TB * MF_CC + t] = ys[t];
    for (int tc = 0; tc < nb; tc += MF_LCH) {
      const int nt = min(MF_LCH, nb - tc);
      // prefetch the next chunk (this column's next, or the next column's first)
      {
        int nJ = J, ntc = tc + MF_LCH;
        if (ntc >= nb) { nJ = J + 1; ntc = 0; }
        const int nnb = F.NT - 1 - nJ;
        if (nJ < F.NE && ntc < nnb) {
          mf_tma_tiles(Ls + (size_t)(buf ^ 1) * MF_LCH * TT, btile(B.Lo, B, nJ, 1 + ntc), min(MF_LCH, nnb - ntc),
                       &bar[buf ^ 1]);
          if (nJ != J) first_issued = true;
        }
      }
      mbar_wait(&bar[buf], ph[buf]);
      ph[buf] ^= 1;
      const double* Lc = Ls + (size_t)buf * MF_LCH * TT;
      double* vN = V + (size_t)(J + 1 + tc) * TB * MF_CC;
      for (int r0 = 2 * rp; r0 < nt * TB; r0 += rstep) {
        double a00 = 0, a01 = 0, a10 = 0, a11 = 0;
#pragma unroll 8
        for (int k = 0; k < TB; ++k) {
          const double l0v = Lc[(size_t)r0 * TB + k], l1v = Lc[(size_t)(r0 + 1) * TB + k];
          const double2 y = *reinterpret_cast<const double2*>(ys + k * MF_CC + 2 * cp);
          a00 = fma(l0v, y.x, a00);
          a01 = fma(l0v, y.y, a01);
          a10 = fma(l1v, y.x, a10);
          a11 = fma(l1v, y.y, a11);
        }
        double2* o0 = reinterpret_cast<double2*>(vN + (size_t)r0 * MF_CC + 2 * cp);
        double2* o1 = reinterpret_cast<double2*>(vN + (size_t)(r0 + 1) * MF_CC + 2 * cp);
        const double2 p0 = *o0, p1 = *o1;
        *o0 = make_double2(p0.x - a00, p0.y - a01);
        *o1 = make_double2(p1.x - a10, p1.y - a11);
      }
      __syncthreads();                                // chunk consumed before its buffer is refilled
      buf ^= 1;
    }
  }
  double* v = Vg + (size_t)F.voff * ld;
  for (int t = threadIdx.x; t < rows * MF_CC; t += blockDim.x) {
    const int r = t / MF_CC, s = t % MF_CC;
    if (s < nc) v[(size_t)r * ld + c0 + s] = V[t];
  }
}
__global__ void __launch_bounds__(256) k_mf_bwd_c(MfDev d, int l0, double* __restrict__ X,
                                                  const double* __restrict__ Vg, int ld, int ntmax) {
  extern __shared__ __align__(16) double sh[];
  __shared__ __align__(8) unsigned long long bar[3];
  const MfFront F = d.fr[d.lvl[l0 + blockIdx.x]];
  const int c0 = blockIdx.y * MF_CC, nc = min(MF_CC, ld - c0);
  if (nc <= 0) return;
  const Band B = mf_band(d.base, F);
  const int rows = F.NT * TB;
  double* V = sh;
  double* Ls = V + (size_t)ntmax * TB * MF_CC;      // 2 x MF_LCH tiles
  double* Dj = Ls + (size_t)2 * MF_LCH * TT;
  double* ys = Dj + TT;                             // TB x MF_CC
  const int* gid = d.gid + F.goff;
  const double* v = Vg + (size_t)F.voff * ld;
  if (threadIdx.x == 0) {
    mbar_init(&bar[0]);
    mbar_init(&bar[1]);
    mbar_init(&bar[2]);
  }
#pragma unroll 4
  for (int t = threadIdx.x; t < rows * MF_CC; t += blockDim.x) {
    const int r = t / MF_CC, s = t % MF_CC;
    double a = 0.0;
    if (s < nc) {
      if (r < F.NE * TB) a = __ldcg(v + (size_t)r * ld + c0 + s);
      else if (gid[r] >= 0) a = __ldcg(X + (size_t)gid[r] * ld + c0 + s);
    }
    V[t] = a;
  }
  __syncthreads();
  unsigned ph[3] = {0, 0, 0};
  int buf = 0;
  const int j = threadIdx.x / MF_CC, s = threadIdx.x % MF_CC;   // one output per thread (32 x 8)
  {
    const int J = F.NE - 1, nb = F.NT - 1 - J;
    mf_tma_tiles(Dj, B.Dinv + (size_t)J * TT, 1, &bar[2]);
    if (nb > 0) mf_tma_tiles(Ls, btile(B.Lo, B, J, 1), min(MF_LCH, nb), &bar[0]);
  }
  bool first_issued = true;                         // the prologue issued step NE-1's first chunk (if any)
  for (int J = F.NE - 1; J >= 0; --J) {
    const int nb = F.NT - 1 - J;
    double acc0 = 0.0, acc1 = 0.0;
    if (nb > 0 && !first_issued) mf_tma_tiles(Ls + (size_t)buf * MF_LCH * TT, btile(B.Lo, B, J, 1), min(MF_LCH, nb),
                                              &bar[buf]);
    first_issued = false;
    for (int tc = 0; tc < nb; tc += MF_LCH) {
      const int nt = min(MF_LCH, nb - tc);
      {
        int nJ = J, ntc = tc + MF_LCH;
        if (ntc >= nb) { nJ = J - 1; ntc = 0; }
        const int nnb = F.NT - 1 - nJ;
        if (nJ >= 0 && ntc < nnb) {
          mf_tma_tiles(Ls + (size_t)(buf ^ 1) * MF_LCH * TT, btile(B.Lo, B, nJ, 1 + ntc), min(MF_LCH, nnb - ntc),
                       &bar[buf ^ 1]);
          if (nJ != J) first_issued = true;
        }
      }
      mbar_wait(&bar[buf], ph[buf]);
      ph[buf] ^= 1;
      const double* Lc = Ls + (size_t)buf * MF_LCH * TT;
      if (j < TB) {
        const double* vb = V + (size_t)(J + 1 + tc) * TB * MF_CC + s;
        for (int rr = 0; rr < nt * TB; rr += 2) {
          acc0 = fma(Lc[(size_t)rr * TB + j], vb[(size_t)rr * MF_CC], acc0);
          acc1 = fma(Lc[(size_t)(rr + 1) * TB + j], vb[(size_t)(rr + 1) * MF_CC], acc1);
        }
      }
      __syncthreads();
      buf ^= 1;
    }
    if (j < TB) ys[j * MF_CC + s] = V[(size_t)(J * TB + j) * MF_CC + s] - (acc0 + acc1);
    mbar_wait(&bar[2], ph[2]);
    ph[2] ^= 1;
    __syncthreads();
    if (j < TB) {
      double a = 0.0, b = 0.0;
#pragma unroll 8
      for (int k = 0; k < TB; k += 2) {
        a = fma(Dj[k * TB + j], ys[k * MF_CC + s], a);
        b = fma(Dj[(k + 1) * TB + j], ys[(k + 1) * MF_CC + s], b);
      }
      V[(size_t)(J * TB + j) * MF_CC + s] = a + b;
    }
    __syncthreads();                                  // Dj consumed, x_J in V
    if (J >= 1) mf_tma_tiles(Dj, B.Dinv + (size_t)(J - 1) * TT, 1, &bar[2]);
  }
  for (int t = threadIdx.x; t < F.nE * MF_CC; t += blockDim.x) {
    const int r = t / MF_CC, s2 = t % MF_CC;
    if (s2 < nc) X[(size_t)gid[r] * ld + c0 + s2] = V[t];
  }
}

static MfDev mf_dev(const Geo& g, double* base) {
  const MfPlan* P = mf_plan(g);
  return MfDev{P->d_fr, P->d_lvl, P->d_gid, P->d_maps, base};
}

cudaError_t launch_mf_assemble(const Geo& g, const double* Kloc, double shift, double* Ak, cudaStream_t st) {
  cudaError_t e = mf_upload(g);
  if (e != cudaSuccess) return e;
  k_mf_a27<<<nblk((long long)g.kc * 14, 256), 256, 0, st>>>(g, Kloc, shift, Ak + mf_plan(g)->a27);
  count_launches(1);
  return cudaGetLastError();
}
cudaError_t launch_mf_diag(const Geo& g, const double* Ak, double* diag, cudaStream_t st) {
  // diagonal entries are A27[c][13]
  cudaError_t e = cudaMemcpy2DAsync(diag, sizeof(double), Ak + mf_plan(g)->a27 + 13, 14 * sizeof(double),
                                    sizeof(double), g.kc, cudaMemcpyDeviceToDevice, st);
  return e;
}
cudaError_t launch_mf_factor(const Geo& g, double* Ak, int* flags, cudaStream_t st) {
  cudaError_t e = mf_upload(g);
  if (e != cudaSuccess) return e;
  const MfPlan* P = mf_plan(g);
  static PerDevice<int> grid_cache;
  const int coop_grid = grid_cache.get([] {
    int dev = 0, sms = 0, per_sm = 0, coop = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
    if (cudaFuncSetAttribute(k_mf_factor, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)(MF_FACTOR_FCACHE * sizeof(MfFront))) != cudaSuccess)
      return 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_mf_factor, 256, MF_FACTOR_FCACHE * sizeof(MfFront));
    return (coop && per_sm > 0) ? std::max(1, sms - mf_reserved_sms()) * std::min(per_sm, 2) : 0;
  });
  if (coop_grid <= 0) return cudaErrorNotSupported;
  const MfDev d = mf_dev(g, Ak);
  for (size_t l = 0; l + 1 < P->lvl_off.size(); ++l) {
    const int l0 = P->lvl_off[l], nf = P->lvl_off[l + 1] - l0;
    if (nf <= 0) continue;
    if (nf > MF_MAXF) return cudaErrorInvalidValue;
    int jmax = 0, ntmax = 0;
    for (int i = 0; i < nf; ++i) {
      jmax = std::max(jmax, P->fr[P->lvl[l0 + i]].NE);
      ntmax = std::max(ntmax, P->fr[P->lvl[l0 + i]].NT);
    }
    k_mf_assemble_t<<<dim3(ntmax * (ntmax + 1) / 2, nf), 256, 0, st>>>(g, d, l0, Ak + P->a27);
    count_launches(1);
    // defer the B x B updates where a tile column has more of them than CTAs (throughput-bound levels:
    // fewer, cheaper tasks); latency-bound levels keep the per-column updates (no extra phase at the end)
    long long nbb = 0;
    for (int i = 0; i < nf; ++i) {
      const long long nb = P->fr[P->lvl[l0 + i]].NT - P->fr[P->lvl[l0 + i]].NE;
      nbb += nb * (nb + 1) / 2;
    }
    MfJob job{d, l0, nf, jmax, nbb > coop_grid ? 1 : 0, g};
    void* args[] = {(void*)&job, (void*)&flags};
    e = cudaLaunchCooperativeKernel((void*)k_mf_factor, dim3(coop_grid), dim3(256), args,
                                    (size_t)std::min(nf, MF_FACTOR_FCACHE) * sizeof(MfFront), st);
    count_launches(1);
    if (e != cudaSuccess) return e;
  }
  if (P->use_g) {
    // every explicit inverse block after the last level (only the solves read G):
    // one launch per footprint group
    static PerDevice<cudaError_t> attr;
    e = attr.get([] { return cudaFuncSetAttribute(k_mf_inv_all, cudaFuncAttributeMaxDynamicSharedMemorySize, MF_SMEM_MAX); });
    if (e != cudaSuccess) return e;
    int off = 0;
    for (int grp = 0; grp < 2; ++grp) {
      if (P->nitems[grp] > 0) {
        const size_t smi =
            ((size_t)P->inv_nemax[grp] * TB * MF_INV_W + (size_t)MF_INV_NS * TB * MF_INV_LD) * sizeof(double);
        if (smi > (size_t)MF_SMEM_MAX) return cudaErrorInvalidValue;
        k_mf_inv_all<<<P->nitems[grp], MF_INV2_THREADS, smi, st>>>(d, P->d_items + off);
        count_launches(1);
      }
      off += P->nitems[grp];
    }
  }
  return cudaGetLastError();
}
cudaError_t launch_mf_solve(const Geo& g, const double* Ak, double* X, double* scratch, int nrhs, cudaStream_t st) {
  if (nrhs == 0) return cudaSuccess;
  const bool force_c = getenv("MSFV_MF_FORCE_CHUNKED") != nullptr;   // test hook: the blocked sweeps at any size
  cudaError_t e = mf_upload(g);
  if (e != cudaSuccess) return e;
  const MfPlan* P = mf_plan(g);
  const MfDev d = mf_dev(g, const_cast<double*>(Ak));
  const size_t sm = (size_t)TB * nrhs * sizeof(double);
  if (sm > 48 * 1024) {
    e = cudaFuncSetAttribute(k_mf_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_mf_bwd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
  }
  const int nl = (int)P->lvl_off.size() - 1;
  auto level_nt = [&](int l) {
    int nt = 1;
    for (int i = P->lvl_off[l]; i < P->lvl_off[l + 1]; ++i) nt = std::max(nt, P->fr[P->lvl[i]].NT);
    return nt;
  };
  auto smem_s = [&](int nt) {
    return ((size_t)nt * TB * nrhs + (size_t)nt * TT + (size_t)3 * TB * nrhs) * sizeof(double) +
           (size_t)3 * nt * TB * sizeof(int) + 16;
  };
  auto smem_c = [&](int nt) {
    return ((size_t)nt * TB * MF_CC + (size_t)2 * MF_LCH * TT + TT + (size_t)TB * MF_CC) * sizeof(double);
  };
  static PerDevice<cudaError_t> attr;
  e = attr.get([] {
    cudaError_t r = cudaFuncSetAttribute(k_mf_fwd_s, cudaFuncAttributeMaxDynamicSharedMemorySize, MF_SMEM_MAX);
    if (r == cudaSuccess) r = cudaFuncSetAttribute(k_mf_bwd_s, cudaFuncAttributeMaxDynamicSharedMemorySize, MF_SMEM_MAX);
    if (r == cudaSuccess) r = cudaFuncSetAttribute(k_mf_fwd_c, cudaFuncAttributeMaxDynamicSharedMemorySize, MF_SMEM_MAX - 8192);
    if (r == cudaSuccess) r = cudaFuncSetAttribute(k_mf_bwd_c, cudaFuncAttributeMaxDynamicSharedMemorySize, MF_SMEM_MAX - 8192);
    return r;
  });
  if (e != cudaSuccess) return e;
  if (P->use_g && nrhs <= 64 && !force_c) {
    // one cooperative launch for both sweeps
    size_t smc = 0;
    for (int l = 0; l < nl; ++l) {
      const int nt = level_nt(l);
      smc = std::max(smc, ((size_t)MF_GR * nt * TB + (size_t)nt * TB * nrhs + (size_t)MF_GR * nrhs) * sizeof(double));
    }
    static PerDevice<int> grid_cache;
    const int coop_grid = grid_cache.get([] {
      int dev = 0, sms = 0, coop = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
      if (cudaFuncSetAttribute(k_mf_solve_coop, cudaFuncAttributeMaxDynamicSharedMemorySize, MF_SMEM_MAX - MF_COOP_STATIC) !=
          cudaSuccess)
        return 0;
      return coop ? std::max(1, sms - mf_reserved_sms()) : 0;
    });
    // fronts whose G chunk + input vector exceed one shared-memory load: K-chunked products
    // (MSFV_MF_FORCE_KCHUNK: test hook, the chunked products at any size)
    const bool kchunk = smc > (size_t)MF_SMEM_MAX - MF_COOP_STATIC || getenv("MSFV_MF_FORCE_KCHUNK") != nullptr;
    int KC = MF_KC;                                   // largest chunk whose two buffers fit
    auto smem_k = [&](int kc) { return (2 * ((size_t)MF_GR * (kc + 4) + (size_t)kc * nrhs + 8) + 1280) * sizeof(double); };
    while (KC > 32 && smem_k(KC) > (size_t)MF_SMEM_MAX - MF_COOP_STATIC) KC /= 2;
    if (kchunk) smc = smem_k(KC);
    if (coop_grid > 0 && smc <= (size_t)MF_SMEM_MAX - MF_COOP_STATIC && !getenv("MSFV_MF_NOCOOP")) {
      const bool timing = getenv("MSFV_MF_TIMING") != nullptr;
      static PerDevice<unsigned long long*> tst_cache;
      unsigned long long* tst = timing ? tst_cache.get([] {
        unsigned long long* p = nullptr;
        cudaMalloc(&p, 256 * sizeof(unsigned long long));
        return p;
      }) : nullptr;
      MfSolveJob job{d, P->d_lvloff, nl, X, scratch, scratch + P->vrows * nrhs, nrhs, timing ? tst : nullptr, P->d_pre,
                     P->npre, kchunk ? KC : 0, P->d_frl, (int)P->lvl.size(), P->d_gtab, P->d_rowbase, (int)P->vrows};
      void* args[] = {(void*)&job};
      e = cudaLaunchCooperativeKernel((void*)k_mf_solve_coop, dim3(coop_grid), dim3(256), args, smc, st);
      count_launches(1);
      if (e != cudaSuccess) return e;
      if (timing) {   // debug: per-phase durations (us) of this solve, stderr
        unsigned long long h[256];
        const int n = 1 + 4 * nl;
        cudaStreamSynchronize(st);
        cudaMemcpy(h, tst, n * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
        fprintf(stderr, "[mf solve nrhs=%d] total %.1f us:", nrhs, (h[n - 1] - h[0]) * 1e-3);
        for (int i = 1; i < n; ++i) fprintf(stderr, " %s%.1f", (i % 2) ? "A" : "B", (h[i] - h[i - 1]) * 1e-3);
        fprintf(stderr, "\n");
      }
      return cudaGetLastError();
    }
  }
  bool g_fits = !force_c;
  for (int l = 0; l < nl; ++l) {
    const int nt = level_nt(l);
    if (((size_t)MF_GR * nt * TB + (size_t)nt * TB * nrhs) * sizeof(double) > (size_t)MF_SMEM_MAX) g_fits = false;
  }
  if (P->use_g && g_fits) {
    static PerDevice<cudaError_t> gattr;
    e = gattr.get([] {
      cudaError_t r = cudaFuncSetAttribute(k_mf_gfwd, cudaFuncAttributeMaxDynamicSharedMemorySize, MF_SMEM_MAX);
      if (r == cudaSuccess) r = cudaFuncSetAttribute(k_mf_gbwd, cudaFuncAttributeMaxDynamicSharedMemorySize, MF_SMEM_MAX);
      return r;
    });
    if (e != cudaSuccess) return e;
    for (int l = 0; l < nl; ++l) {
      const int l0 = P->lvl_off[l], nf = P->lvl_off[l + 1] - l0, nt = level_nt(l);
      int ne = 1;
      for (int i = l0; i < l0 + nf; ++i) ne = std::max(ne, P->fr[P->lvl[i]].NE);
      const size_t smf = ((size_t)MF_GR * ne * TB + (size_t)ne * TB * nrhs) * sizeof(double);
      if (smf > (size_t)MF_SMEM_MAX) return cudaErrorInvalidValue;   // unreachable: checked below
      k_mf_gfwd<<<dim3(nf, (nt * TB + MF_GR - 1) / MF_GR), 256, smf, st>>>(d, l0, X, scratch, nrhs);
    }
    for (int l = nl - 1; l >= 0; --l) {
      const int l0 = P->lvl_off[l], nf = P->lvl_off[l + 1] - l0, nt = level_nt(l);
      int ne = 1;
      for (int i = l0; i < l0 + nf; ++i) ne = std::max(ne, P->fr[P->lvl[i]].NE);
      const size_t smb = ((size_t)MF_GR * nt * TB + (size_t)nt * TB * nrhs) * sizeof(double);
      if (smb > (size_t)MF_SMEM_MAX) return cudaErrorInvalidValue;
      k_mf_gbwd<<<dim3(nf, (ne * TB + MF_GR - 1) / MF_GR), 256, smb, st>>>(d, l0, X, scratch, nrhs);
    }
    count_launches(2 * nl);
    return cudaGetLastError();
  }
  for (int l = 0; l < nl; ++l) {
    const int l0 = P->lvl_off[l], nf = P->lvl_off[l + 1] - l0, nt = level_nt(l);
    if (smem_s(nt) <= MF_SMEM_MAX && !force_c)
      k_mf_fwd_s<<<nf, 256, smem_s(nt), st>>>(d, l0, X, scratch, nrhs, nt);
    else if (smem_c(nt) <= MF_SMEM_MAX - 8192)
      k_mf_fwd_c<<<dim3(nf, (nrhs + MF_CC - 1) / MF_CC), 256, smem_c(nt), st>>>(d, l0, X, scratch, nrhs, nt);
    else
      k_mf_fwd<<<nf, 256, sm, st>>>(d, l0, X, scratch, nrhs);
  }
  for (int l = nl - 1; l >= 0; --l) {
    const int l0 = P->lvl_off[l], nf = P->lvl_off[l + 1] - l0, nt = level_nt(l);
    if (smem_s(nt) <= MF_SMEM_MAX && !force_c)
      k_mf_bwd_s<<<nf, 256, smem_s(nt), st>>>(d, l0, X, scratch, nrhs, nt);
    else if (smem_c(nt) <= MF_SMEM_MAX - 8192)
      k_mf_bwd_c<<<dim3(nf, (nrhs + MF_CC - 1) / MF_CC), 256, smem_c(nt), st>>>(d, l0, X, scratch, nrhs, nt);
    else
      k_mf_bwd<<<nf, 256, sm, st>>>(d, l0, X, scratch, nrhs);
  }
  count_launches(2 * nl);
  return cudaGetLastError();
}
size_t mf_doubles(const Geo& g) { return mf_plan(g)->total; }
int mf_tile_rows(const Geo& g) { return (int)(4 * mf_plan(g)->vrows / TB); }   // Vout, XE/Zb, S0, S1 workspaces

}  // namespace msfv
