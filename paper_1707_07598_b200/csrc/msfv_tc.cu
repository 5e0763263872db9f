// FP64 tensor-core (DMMA, mma.sync m8n8k4 f64) tile-band kernels for the
// per-block interior problems -- the hot path of the basis build
// (basis.py:511-563) and of every blockdiag(A_II^-1) application
// (MultiscaleBasis.interior_solve, basis.py:339-353).
//
// One warp owns one coarse block.  A_II (nI x nI, half bandwidth p, interior
// nodes in lexicographic order) is processed in 8x8 tiles: tile column J has
// the diagonal tile and PT = ceil(p/8) sub-diagonal tiles.  The right-looking
// blocked Cholesky keeps its whole active window -- the (PT+1)(PT+2)/2 tiles
// that still receive updates -- in registers (DMMA accumulator layout), so the
// trailing update is 2 DMMAs per tile with no shared-memory traffic.  The 8
// Lagrange right-hand sides ride along as one extra tile column (fused
// forward substitution); the backward substitution re-reads the factor tiles
// from L2/HBM.  The per-block 8x8 Galerkin block is a DMMA reduction over the
// block's owned edges.
//
// Factor storage ("LT"), per block, per tile column J, PT+1 tiles of 64
// doubles stored in A-fragment lane order:  slot 0 = L_JJ^{-1},
// slot t = L_{J+t,J}.   Fragment layouts (m8n8k4 f64):
//   A[m][k] at lane 4m+k ; B[k][n] at lane 4n+k ; C[m][n] at lane 4m+n/2, slot n%2
// An 8x8 tile in "A-frag" form is two A fragments (k = 0..3 and 4..7).
#include <mutex>
#include <cstdlib>
#include "msfv_common.cuh"
#include "msfv_kernels.h"
#include "msfv_dmma.cuh"

namespace msfv {
namespace {

constexpr unsigned FULL = 0xffffffffu;

using namespace dmma;

// Interior coordinates, packed x | y << 10 | z << 20 (one table per CTA).
__device__ __forceinline__ void fill_coords(const Geo& g, int* crd) {
  for (int a = threadIdx.x; a < g.nI; a += blockDim.x) {
    const int x = 1 + a % g.ni1, y = 1 + (a / g.ni1) % g.ni2, z = 1 + a / (g.ni1 * g.ni2);
    crd[a] = x | (y << 10) | (z << 20);
  }
}

// Transposed-operand DMMA form.  With BOTH operands in accumulator (C) layout,
// mma(D, X, Y) computes D += X Y^T: chunk h of the k dimension is the column
// set {2k + h}, i.e. slot h of the C layout, for X and Y alike.  Every product
// the Cholesky and the substitutions need (X_t = A_t L^-T, A -= X_a X_b^T,
// y^T = r^T L^-T, r^T -= y^T X^T, x^T = (.) L^-1) is of that form once the
// right-hand sides are carried transposed, so no register shuffles are needed.
// Tiles are stored row-major (the C layout at lane*2); ld_t loads the C layout
// of a stored tile's transpose.

// Per-block stencil table in shared memory: one row of AROW doubles per
// interior node, padding rows (up to 8*NTI) are identity:
//   [A_ii, A_{i,i-1}, A_{i,i-ni1}, A_{i,i-p}, 0]
// Coinciding offsets (ni1 == 1 or ni2 == 1) are merged into the first slot
// that the selector (sel_code) tests.  The Lagrange right-hand sides -A_IB x_B
// (basis.py:548) of the 8 corners are written to the block's Sint rows, which
// then park the forward-substitution result y and finally hold S_I.  The
// conductances of the boundary-interior edges go to Fk (face-major, (u, v)
// in-face order) for the local Galerkin block.
constexpr int AROW = 5;

__device__ __forceinline__ int face_off(const Geo& g, int face) {
  const int ax = face >> 1;
  const int a0 = 0, a1 = 2 * g.ni2 * g.ni3, a2 = a1 + 2 * g.ni1 * g.ni3;
  const int sz = ax == 0 ? g.ni2 * g.ni3 : (ax == 1 ? g.ni1 * g.ni3 : g.ni1 * g.ni2);
  return (ax == 0 ? a0 : (ax == 1 ? a1 : a2)) + (face & 1) * sz;
}

__device__ __forceinline__ void stencil_table(const Geo& g, const double* __restrict__ w, int X0, int Y0, int Z0,
                                              int NR, double* As, double* Fk, double* Sb, int lane, int jb) {
  const double s1 = g.ih1 * g.ih1, s2 = g.ih2 * g.ih2, s3 = g.ih3 * g.ih3;
  for (int i = lane; i < NR; i += 32) {
    double* row = As + i * AROW;
    if (i >= g.nI) {
      row[0] = 1.0;
      row[1] = row[2] = row[3] = row[4] = 0.0;
      continue;
    }
    int x, y, z;
    decode3f(i, g.ni1, g.r_ni1, g.ni2, g.r_ni2, x, y, z);
    ++x; ++y; ++z;
    const long long I = X0 + x, J = Y0 + y, K = Z0 + z;
    const double kxm = __ldg(w + ex_id(g, I - 1, J, K)) * s1;
    const double kxp = __ldg(w + ex_id(g, I, J, K)) * s1;
    const double kym = __ldg(w + ey_id(g, I, J - 1, K)) * s2;
    const double kyp = __ldg(w + ey_id(g, I, J, K)) * s2;
    const double kzm = __ldg(w + ez_id(g, I, J, K - 1)) * s3;
    const double kzp = __ldg(w + ez_id(g, I, J, K)) * s3;
    const double v1 = x > 1 ? -kxm : 0.0, v2 = y > 1 ? -kym : 0.0, v3 = z > 1 ? -kzm : 0.0;
    const int D2 = g.ni1, D3 = g.p;
    row[0] = ((((kxm + kxp) + kym) + kyp) + kzm) + kzp;
    row[1] = v1 + (D2 == 1 ? v2 : 0.0) + (D3 == 1 ? v3 : 0.0);
    row[2] = v2 + (D3 == D2 ? v3 : 0.0);
    row[3] = v3;
    row[4] = 0.0;
    // boundary-face conductances (x == 1 and x == ni1 may both hold)
    if (x == 1) Fk[face_off(g, 0) + (z - 1) * g.ni2 + (y - 1)] = kxm;
    if (x == g.ni1) Fk[face_off(g, 1) + (z - 1) * g.ni2 + (y - 1)] = kxp;
    if (y == 1) Fk[face_off(g, 2) + (z - 1) * g.ni1 + (x - 1)] = kym;
    if (y == g.ni2) Fk[face_off(g, 3) + (z - 1) * g.ni1 + (x - 1)] = kyp;
    if (z == 1) Fk[face_off(g, 4) + (y - 1) * g.ni1 + (x - 1)] = kzm;
    if (z == g.ni3) Fk[face_off(g, 5) + (y - 1) * g.ni1 + (x - 1)] = kzp;
    // Lagrange rhs of corner cc: sum over boundary faces of k_f * hat_cc(face
    // point); the face-normal hat factor is exactly 1 or 0
    const double fx0 = x == 1 ? kxm : 0.0, fx1 = x == g.ni1 ? kxp : 0.0;
    const double fy0 = y == 1 ? kym : 0.0, fy1 = y == g.ni2 ? kyp : 0.0;
    const double fz0 = z == 1 ? kzm : 0.0, fz1 = z == g.ni3 ? kzp : 0.0;
    if (g.bx) {
      // reduced boundary conditions: the skeleton values of the bound box table
      // instead of the hats (same sum over the boundary faces)
      for (int cc = 0; cc < 8; ++cc) {
        double v = 0.0;
        if (x == 1) v += fx0 * skel_value(g, jb, cc, 0, y, z);
        if (x == g.ni1) v += fx1 * skel_value(g, jb, cc, g.b1, y, z);
        if (y == 1) v += fy0 * skel_value(g, jb, cc, x, 0, z);
        if (y == g.ni2) v += fy1 * skel_value(g, jb, cc, x, g.b2, z);
        if (z == 1) v += fz0 * skel_value(g, jb, cc, x, y, 0);
        if (z == g.ni3) v += fz1 * skel_value(g, jb, cc, x, y, g.b3);
        Sb[(size_t)cc * g.nI + i] = v;
      }
      continue;
    }
    const double hx0 = hatf1(x, g.ib1), hx1 = hatf1(x - g.b1, g.ib1);
    const double hy0 = hatf1(y, g.ib2), hy1 = hatf1(y - g.b2, g.ib2);
    const double hz0 = hatf1(z, g.ib3), hz1 = hatf1(z - g.b3, g.ib3);
#pragma unroll
    for (int cc = 0; cc < 8; ++cc) {
      const bool cx = cc & 1, cy = cc & 2, cz = cc & 4;
      const double hx = cx ? hx1 : hx0, hy = cy ? hy1 : hy0, hz = cz ? hz1 : hz0;
      double v = 0.0;
      v += (cx ? 0.0 : fx0) * (hy * hz);
      v += (cx ? fx1 : 0.0) * (hy * hz);
      v += (cy ? 0.0 : fy0) * (hx * hz);
      v += (cy ? fy1 : 0.0) * (hx * hz);
      v += (cz ? 0.0 : fz0) * (hx * hy);
      v += (cz ? fz1 : 0.0) * (hx * hy);
      Sb[(size_t)cc * g.nI + i] = v;
    }
  }
}

// Stencil-table slot of A(i, i - d) (4 = structural zero).
__device__ __forceinline__ unsigned sel_code(const Geo& g, int d) {
  return d == 0 ? 0u : d == 1 ? 1u : d == g.ni1 ? 2u : d == g.p ? 3u : 4u;
}

// Transposed right-hand-side tile I of corner column c = lane/4 (rows 8I+2q, +1).
__device__ __forceinline__ F2 ld_rt(const Geo& g, const double* Sb, int I, int lane) {
  const int c = lane >> 2, r0 = 8 * I + 2 * (lane & 3);
  const double* p = Sb + (size_t)c * g.nI + r0;
  return {r0 < g.nI ? __ldcg(p) : 0.0, r0 + 1 < g.nI ? __ldcg(p + 1) : 0.0};
}
__device__ __forceinline__ void st_rt(const Geo& g, double* Sb, int I, int lane, const F2& v) {
  const int c = lane >> 2, r0 = 8 * I + 2 * (lane & 3);
  double* p = Sb + (size_t)c * g.nI + r0;
  if (r0 < g.nI) p[0] = v.x;
  if (r0 + 1 < g.nI) p[1] = v.y;
}

// Cholesky of one 8x8 SPD tile (C layout); returns L^{-1} in C layout.  Lanes
// 0..7 own rows of L in registers (shuffle right-looking factorization, rsqrt
// pivots), then columns of L^{-1}; shared memory re-lays the tile.
template <int C>
__device__ __forceinline__ void p8_step(double (&x)[8], double& invd, int r, bool& bad) {
  if constexpr (C < 8) {
    double d = __shfl_sync(FULL, x[C], C);
    if (!(d > 0.0)) { bad = true; d = 1.0; }
    const double inv = rsqrt(d);
    if (r > C) x[C] *= inv;
    if (r == C) { x[C] = d * inv; invd = inv; }
    const double lrc = x[C];
#pragma unroll
    for (int q = C + 1; q < 8; ++q) {
      const double lqc = __shfl_sync(FULL, lrc, q);
      if (r >= q) x[q] -= lrc * lqc;
    }
    p8_step<C + 1>(x, invd, r, bad);
  }
}
template <int R>
__device__ __forceinline__ void i8_step(double (&d)[8], int c, const double* Ds, const double* invd) {
  if constexpr (R < 8) {
    double acc = (R == c) ? 1.0 : 0.0;
#pragma unroll
    for (int m = 0; m < R; ++m) acc -= Ds[R * 8 + m] * d[m];
    d[R] = (R < c) ? 0.0 : acc * invd[R];
    i8_step<R + 1>(d, c, Ds, invd);
  }
}

__device__ __forceinline__ F2 potrf_inv8(const F2& t, double* Ds, double* Is, int lane, int* flags) {
  st2(Ds + lane * 2, t);
  __syncwarp();
  const int r = lane & 7;
  double x[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) x[q] = Ds[r * 8 + q];
  bool bad = false;
  double invd = 1.0;
  p8_step<0>(x, invd, r, bad);
  if (bad && lane == 0) atomicOr(flags, FLAG_LOCAL_NOT_SPD);
  __syncwarp();
  if (lane < 8) {
#pragma unroll
    for (int q = 0; q < 8; ++q) Ds[r * 8 + q] = x[q];
    Is[64 + r] = invd;
  }
  __syncwarp();
  if (lane < 8) {
    double d[8];
    i8_step<0>(d, lane, Ds, Is + 64);
#pragma unroll
    for (int rr = 0; rr < 8; ++rr) Is[rr * 8 + lane] = d[rr];
  }
  __syncwarp();
  const F2 li = ld2(Is + lane * 2);
  __syncwarp();
  return li;
}

// ---- software-pipelined POTRF: the factorization of the next diagonal tile
// runs with the current step's other trailing DMMAs interleaved between its
// pivots (one warp's in-order stream then overlaps the pivot chain latency
// with tensor-core work).  Trailing pairs (a, b), 2 <= a <= PT, 1 <= b <= a,
// in descending rows so X tiles die early.
__host__ __device__ constexpr int tr_a(int PT, int k) {
  for (int a = PT; a >= 2; --a) {
    if (k < a) return a;
    k -= a;
  }
  return 1;
}
__host__ __device__ constexpr int tr_b(int PT, int k) {
  for (int a = PT; a >= 2; --a) {
    if (k < a) return k + 1;
    k -= a;
  }
  return 1;
}
template <int PT, int LO, int HI>
__device__ __forceinline__ void trail(F2 (&W)[PT + 1][PT + 1], const F2 (&X)[PT + 1]) {
  if constexpr (LO < HI) {
    constexpr int a = tr_a(PT, LO), b = tr_b(PT, LO);
    mma(W[a][b], neg(X[a]), X[b]);
    trail<PT, LO + 1, HI>(W, X);
  }
}
constexpr int PIPE_STAGES = 17;   // after load, after each of 8 pivots, after each of 8 inverse rows
template <int PT>
struct TrailPipe {
  F2 (&W)[PT + 1][PT + 1];
  const F2 (&X)[PT + 1];
  template <int K>
  __device__ __forceinline__ void at() {
    constexpr int NP = PT * (PT + 1) / 2 - 1;
    trail<PT, (K * NP) / PIPE_STAGES, ((K + 1) * NP) / PIPE_STAGES>(W, X);
  }
};
template <int C, class P>
__device__ __forceinline__ void p8_pipe(double (&x)[8], double& invd, int r, bool& bad, P& pipe) {
  if constexpr (C < 8) {
    double d = __shfl_sync(FULL, x[C], C);
    if (!(d > 0.0)) { bad = true; d = 1.0; }
    const double inv = rsqrt(d);
    if (r > C) x[C] *= inv;
    if (r == C) { x[C] = d * inv; invd = inv; }
    const double lrc = x[C];
#pragma unroll
    for (int q = C + 1; q < 8; ++q) {
      const double lqc = __shfl_sync(FULL, lrc, q);
      if (r >= q) x[q] -= lrc * lqc;
    }
    pipe.template at<C + 1>();
    p8_pipe<C + 1>(x, invd, r, bad, pipe);
  }
}
template <int R, class P>
__device__ __forceinline__ void i8_pipe(double (&d)[8], int c, const double* Ds, const double* invd, P& pipe) {
  if constexpr (R < 8) {
    double acc = (R == c) ? 1.0 : 0.0;
#pragma unroll
    for (int m = 0; m < R; ++m) acc -= Ds[R * 8 + m] * d[m];
    d[R] = (R < c) ? 0.0 : acc * invd[R];
    pipe.template at<9 + R>();
    i8_pipe<R + 1>(d, c, Ds, invd, pipe);
  }
}
// potrf_inv8 with the pipe's DMMA groups interleaved (all lanes convergent)
template <class P>
__device__ __forceinline__ F2 potrf_inv8_pipe(const F2& t, double* Ds, double* Is, int lane, int* flags, P& pipe) {
  st2(Ds + lane * 2, t);
  __syncwarp();
  const int r = lane & 7;
  double x[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) x[q] = Ds[r * 8 + q];
  pipe.template at<0>();
  bool bad = false;
  double invd = 1.0;
  p8_pipe<0>(x, invd, r, bad, pipe);
  if (bad && lane == 0) atomicOr(flags, FLAG_LOCAL_NOT_SPD);
  __syncwarp();
  if (lane < 8) {
#pragma unroll
    for (int q = 0; q < 8; ++q) Ds[r * 8 + q] = x[q];
    Is[64 + r] = invd;
  }
  __syncwarp();
  double d[8];
  i8_pipe<0>(d, r, Ds, Is + 64, pipe);
  if (lane < 8) {
#pragma unroll
    for (int rr = 0; rr < 8; ++rr) Is[rr * 8 + lane] = d[rr];
  }
  __syncwarp();
  const F2 li = ld2(Is + lane * 2);
  __syncwarp();
  return li;
}

}  // namespace

// ----------------------------------------------------------------- basis

// Backward substitution of block jb: Sb holds y = L^{-1} R (parked by the
// forward sweep) and receives S_I = L^{-T} y:
//   x_J^T = (y_J^T - sum_t x_{J+t}^T X_t) L_JJ^{-1};
// the window keeps -x^T of the last PT tiles; the next steps' transposed
// factor tiles and y are prefetched into registers.
// SPX (p = 8 PT - 7): the transposed offset-PT tile has its one entry in
// column 0, so its product needs only the chunk-0 DMMA.
template <int PT, bool SPX = false>
__device__ __forceinline__ void backward_sweep(const Geo& g, const double* __restrict__ LT, double* Sb, int jb,
                                               int lane) {
  const int NTI = (g.nI + 7) >> 3;
  if (NTI == 0) return;
    F2 Xw[PT > 0 ? PT : 1];
#pragma unroll
    for (int t = 0; t < (PT > 0 ? PT : 1); ++t) Xw[t] = {0.0, 0.0};
    F2 nLt[2][PT + 1], nY[2];
    auto load_bwd = [&](int J, F2 (&Lt)[PT + 1], F2& Y) {
      const double* p = LT + ((size_t)jb * NTI + J) * (PT + 1) * 64;
#pragma unroll
      for (int t = 0; t <= PT; ++t) Lt[t] = (t == 0 || J + t < NTI) ? ld_t(p + t * 64, lane) : F2{0.0, 0.0};
      Y = ld_rt(g, Sb, J, lane);
    };
    load_bwd(NTI - 1, nLt[0], nY[0]);
    if (NTI > 1) load_bwd(NTI - 2, nLt[1], nY[1]);
    for (int J = NTI - 1; J >= 0; --J) {
      F2 cLt[PT + 1];
#pragma unroll
      for (int t = 0; t <= PT; ++t) {
        cLt[t] = nLt[0][t];
        nLt[0][t] = nLt[1][t];
      }
      F2 acc = nY[0];
      nY[0] = nY[1];
      if (J > 1) load_bwd(J - 2, nLt[1], nY[1]);
#pragma unroll
      for (int t = 1; t <= PT; ++t)
        if (J + t < NTI) {
          if (SPX && t == PT)
            mma884(acc.x, acc.y, Xw[t - 1].x, cLt[t].x);
          else
            mma(acc, Xw[t - 1], cLt[t]);
        }
      F2 xj = {0.0, 0.0};
      mma(xj, acc, cLt[0]);
      st_rt(g, Sb, J, lane, xj);
#pragma unroll
      for (int t = PT - 1; t >= 1; --t) Xw[t] = Xw[t - 1];
      if (PT > 0) Xw[0] = neg(xj);
    }
  __syncwarp();
}


// ---- lean main loop (compile-time stencil tile mask OM: bit o set when tile
// offset o below the diagonal can hold stencil entries; 0xC3 = {0,1,6,7} for
// 7x7x7 interiors).  Differences from the generic loop:
//  * the window slide costs no register moves: every trailing update writes
//    its result straight into the shifted slot (D != C form of the DMMA);
//  * the diagonal 8x8 POTRF is predicate-free (rows above the pivot carry
//    junk in their upper part, never read) with a MUFU-seeded rsqrt and one
//    cubic correction instead of the library's special-case branches;
//  * L_JJ^{-1} is a right-looking column solve (chain of 8 FMA+MUL pairs)
//    over a column-major copy of L in shared memory;
//  * only the tile offsets in OM are fetched from the stencil table.
__device__ __forceinline__ void mma_to(F2& d, const F2& c, const F2& a, const F2& b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};\n"
      : "=d"(d.x), "=d"(d.y)
      : "d"(a.x), "d"(b.x), "d"(c.x), "d"(c.y));
  mma884(d.x, d.y, a.y, b.y);
}
// d = c + X Y^T when one operand's even columns (chunk 0) are exactly zero:
// one DMMA instead of two
__device__ __forceinline__ void mma_to_h1(F2& d, const F2& c, const F2& a, const F2& b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};\n"
      : "=d"(d.x), "=d"(d.y)
      : "d"(a.y), "d"(b.y), "d"(c.x), "d"(c.y));
}
// 1/sqrt(d) for a positive normal d: MUFU seed (>= 2^-22) and one cubic
// Newton-type step y (1 + e/2 + 3e^2/8), e = 1 - d y^2 (relative error ~2^-60
// before rounding).
__device__ __forceinline__ double rsq(double d) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
  const double e = fma(-d * y, y, 1.0);
  const double t = fma(0.375, e, 0.5);
  return fma(y * e, t, y);
}
// SPX: the band is p = 8 PT - 7 (7x7x7 interiors: p = 49, PT = 7), so the
// offset-PT factor tile L_{J+PT,J} holds one entry, (0, 7): its chunk 0 (even
// columns) is exactly zero and every product with it needs one DMMA.
template <int PT, bool SPX = false>
struct TrailPipe2 {
  F2 (&Wn)[PT + 1][PT + 1];
  const F2 (&W)[PT + 1][PT + 1];
  const F2 (&X)[PT + 1];
  template <int K>
  __device__ __forceinline__ void at() {
    constexpr int NP = PT * (PT + 1) / 2 - 1;
    run<(K * NP) / PIPE_STAGES, ((K + 1) * NP) / PIPE_STAGES>();
  }
  template <int LO, int HI>
  __device__ __forceinline__ void run() {
    if constexpr (LO < HI) {
      constexpr int a = tr_a(PT, LO), b = tr_b(PT, LO);
      if constexpr (SPX && a == PT)
        mma_to_h1(Wn[a - 1][b - 1], W[a][b], neg(X[a]), X[b]);
      else
        mma_to(Wn[a - 1][b - 1], W[a][b], neg(X[a]), X[b]);
      run<LO + 1, HI>();
    }
  }
};
template <int C, class P>
__device__ __forceinline__ void p8_lean(double (&x)[8], bool& bad, double* Is, int lane, P& pipe) {
  if constexpr (C < 8) {
    double d = __shfl_sync(FULL, x[C], C);
    if (!(d > 0.0)) { bad = true; d = 1.0; }
    const double inv = rsq(d);
    x[C] *= inv;                      // L(r, C) on rows r >= C (sqrt(d) on r == C)
    if (lane == 0) Is[C] = inv;
#pragma unroll
    for (int q = C + 1; q < 8; ++q) x[q] = fma(-x[C], __shfl_sync(FULL, x[C], q), x[q]);
    pipe.template at<C + 1>();
    p8_lean<C + 1>(x, bad, Is, lane, pipe);
  }
}
template <int K, class P>
__device__ __forceinline__ void inv_lean(double (&acc)[8], const double* Ds, const double* Is, P& pipe) {
  if constexpr (K < 8) {
    acc[K] *= Is[K];
#pragma unroll
    for (int R = K + 1; R < 8; ++R) acc[R] = fma(-Ds[K * 8 + R], acc[K], acc[R]);
    pipe.template at<9 + K>();
    inv_lean<K + 1>(acc, Ds, Is, pipe);
  }
}
// returns L^{-1} (C layout) of the SPD 8x8 tile t (C layout); Ds: 64 doubles,
// Is: 72 doubles of warp-private shared memory
template <class P>
__device__ __forceinline__ F2 potrf_inv8_lean(const F2& t, double* Ds, double* Is, int lane, int* flags, P& pipe) {
  st2(Ds + lane * 2, t);
  __syncwarp();
  const int r = lane & 7;
  double x[8];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const double2 v = reinterpret_cast<const double2*>(Ds + r * 8)[k];
    x[2 * k] = v.x;
    x[2 * k + 1] = v.y;
  }
  pipe.template at<0>();
  bool bad = false;
  p8_lean<0>(x, bad, Is, lane, pipe);
  if (bad && lane == 0) atomicOr(flags, FLAG_LOCAL_NOT_SPD);
  __syncwarp();
  if (lane < 8) {                     // column-major copy of L: Ds[q * 8 + r] = L(r, q)
#pragma unroll
    for (int q = 0; q < 8; ++q) Ds[q * 8 + r] = x[q];
  }
  __syncwarp();
  // column c = r of L^{-1}, right-looking: z_k = acc_k / L(k,k); acc_R -= L(R,k) z_k
  double acc[8];
#pragma unroll
  for (int R = 0; R < 8; ++R) acc[R] = R == r ? 1.0 : 0.0;
  inv_lean<0>(acc, Ds, Is, pipe);
  if (lane < 8) {
#pragma unroll
    for (int R = 0; R < 8; ++R) Is[8 + R * 8 + r] = acc[R];
  }
  __syncwarp();
  const F2 li = ld2(Is + 8 + lane * 2);
  __syncwarp();
  return li;
}

// 1D bulk copy shared -> global (async proxy) for the factor tiles: the
// registers are free once the tiles are in shared memory (a plain STG keeps
// its source registers locked until the LSU drains them, which stalled the
// next step's DMMAs writing the same registers).
__device__ __forceinline__ void bulk_s2g(double* gdst, const double* ssrc, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(gdst),
               "r"((unsigned)__cvta_generic_to_shared(ssrc)), "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;\n" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

// Transposed Lagrange right-hand-side tile I (corner lane/4, rows 8I+2q, +1)
// evaluated from the face conductances in shared memory, in the summation
// order of stencil_table (bit-identical to the parked copy in Sint): the
// first window of the factorization does not wait on a global round trip of
// the values stencil_table has just stored.
__device__ __forceinline__ double rhs_value(const Geo& g, const double* Fk, int i, int cc) {
  if (i >= g.nI) return 0.0;
  int x, y, z;
  decode3f(i, g.ni1, g.r_ni1, g.ni2, g.r_ni2, x, y, z);
  ++x; ++y; ++z;
  const bool cx = cc & 1, cy = cc & 2, cz = cc & 4;
  const double hx = cx ? hatf1(x - g.b1, g.ib1) : hatf1(x, g.ib1);
  const double hy = cy ? hatf1(y - g.b2, g.ib2) : hatf1(y, g.ib2);
  const double hz = cz ? hatf1(z - g.b3, g.ib3) : hatf1(z, g.ib3);
  const double fx0 = x == 1 ? Fk[face_off(g, 0) + (z - 1) * g.ni2 + (y - 1)] : 0.0;
  const double fx1 = x == g.ni1 ? Fk[face_off(g, 1) + (z - 1) * g.ni2 + (y - 1)] : 0.0;
  const double fy0 = y == 1 ? Fk[face_off(g, 2) + (z - 1) * g.ni1 + (x - 1)] : 0.0;
  const double fy1 = y == g.ni2 ? Fk[face_off(g, 3) + (z - 1) * g.ni1 + (x - 1)] : 0.0;
  const double fz0 = z == 1 ? Fk[face_off(g, 4) + (y - 1) * g.ni1 + (x - 1)] : 0.0;
  const double fz1 = z == g.ni3 ? Fk[face_off(g, 5) + (y - 1) * g.ni1 + (x - 1)] : 0.0;
  double v = 0.0;
  v += (cx ? 0.0 : fx0) * (hy * hz);
  v += (cx ? fx1 : 0.0) * (hy * hz);
  v += (cy ? 0.0 : fy0) * (hx * hz);
  v += (cy ? fy1 : 0.0) * (hx * hz);
  v += (cz ? 0.0 : fz0) * (hx * hy);
  v += (cz ? fz1 : 0.0) * (hx * hy);
  return v;
}
__device__ __forceinline__ F2 rhs_rt(const Geo& g, const double* Fk, int I, int lane) {
  const int c = lane >> 2, r0 = 8 * I + 2 * (lane & 3);
  return {rhs_value(g, Fk, r0, c), rhs_value(g, Fk, r0 + 1, c)};
}

// B = sum over the six boundary faces of k_f h h^T for 7x7 faces: per face
// row v two DMMAs (u = 1..4 | 5..7, lane slot = u offset), the hats separable
// (same products as the generic loop, summed in row order).
__device__ __forceinline__ void galerkin_faces7(const Geo& g, const double* Fk, int lane, F2& K) {
  const int cc = lane >> 2, slot = lane & 3;
  const int cx = cc & 1, cy = (cc >> 1) & 1, cz = (cc >> 2) & 1;
#pragma unroll
  for (int face = 0; face < 6; ++face) {
    const int ax = face >> 1, hi = face & 1;
    const bool on = (ax == 0 ? cx : (ax == 1 ? cy : cz)) == hi;
    const int cu = ax == 0 ? cy * g.b2 : cx * g.b1, cv = ax == 2 ? cy * g.b2 : cz * g.b3;
    const double ibu = ax == 0 ? g.ib2 : g.ib1, ibv = ax == 2 ? g.ib2 : g.ib3;
    const double* F = Fk + 49 * face;
    const double hu0 = on ? hatf1(1 + slot - cu, ibu) : 0.0;
    const double hu1 = (on && slot < 3) ? hatf1(5 + slot - cu, ibu) : 0.0;
#pragma unroll
    for (int v = 1; v <= 7; ++v) {
      const double hv = hatf1(v - cv, ibv);
      const double b0 = hu0 * hv, b1 = hu1 * hv;
      const double a0 = F[(v - 1) * 7 + slot] * b0;
      const double a1 = slot < 3 ? F[(v - 1) * 7 + 4 + slot] * b1 : 0.0;
      mma884(K.x, K.y, a0, b0);
      mma884(K.x, K.y, a1, b1);
    }
  }
}

struct NoPipe {
  template <int K>
  __device__ __forceinline__ void at() {}
};
template <int PT, unsigned OM, int RF>
__device__ __forceinline__ void factor_forward_lean(const Geo& g, const double* As, const double* Fk, double* Sb,
                                                    double* LT, int jb,
                                                    int lane, double* Ds, double* Is, double* Lst, int* flags,
                                                    F2& G) {
  const int NTI = (g.nI + 7) >> 3;
  const int m = lane >> 2, q = lane & 3;
  // 7x7x7 interiors (OM = {0,1,6,7}): p = 49 = 8 PT - 7, see TrailPipe2
  constexpr bool SPX = PT == 7 && OM == 0xC3u;
  // per-lane stencil slots (3 bits each) of element (b, s) of W[PT][b]:
  // A(i, i - d), d = 8 (PT - b) + m - 2q - s
  unsigned long long sel = 0;
#pragma unroll
  for (int b = 0; b <= PT; ++b)
#pragma unroll
    for (int s = 0; s < 2; ++s)
      sel |= (unsigned long long)sel_code(g, 8 * (PT - b) + m - 2 * q - s) << (6 * b + 3 * s);
  auto fetch = [&](int I, int b) -> F2 {
    const double* row = As + (8 * I + m) * AROW;
    return {row[(sel >> (6 * b)) & 7u], row[(sel >> (6 * b + 3)) & 7u]};
  };
  F2 W[PT + 1][PT + 1];
  F2 Rt[PT + 1];
#pragma unroll
  for (int a = 0; a <= PT; ++a) {
#pragma unroll
    for (int b = 0; b <= PT; ++b) {
      W[a][b] = {0.0, 0.0};
      if (b <= a && ((OM >> (a - b)) & 1u) && a < NTI) W[a][b] = fetch(a, PT - a + b);
    }
    Rt[a] = RF ? rhs_rt(g, Fk, a, lane) : ld_rt(g, Sb, a, lane);
  }
  NoPipe nop;
  F2 Li = potrf_inv8_lean(W[0][0], Ds, Is, lane, flags, nop);
#pragma unroll 1
  for (int J = 0; J < NTI; ++J) {
    const int In = J + 1 + PT;       // tile row entering the window after this step
    const F2 nR = In < NTI ? (RF == 2 ? rhs_rt(g, Fk, In, lane) : ld_rt(g, Sb, In, lane)) : F2{0.0, 0.0};
    F2 X[PT + 1];
    // factor tiles of this step: staged in shared memory (double buffer),
    // one bulk copy to LT
    double* Ls = Lst + (J & 1) * (PT + 1) * 64;
    if (lane == 0) bulk_wait_read<1>();          // the copy that last read this buffer is done
    __syncwarp();
    st2(Ls + lane * 2, Li);
#pragma unroll
    for (int t = 1; t <= PT; ++t) {
      X[t] = {0.0, 0.0};
      if (SPX && t == PT)
        mma884(X[t].x, X[t].y, W[t][0].y, Li.y);   // A_{J+PT,J} = its (0, 7) entry (never updated)
      else
        mma(X[t], W[t][0], Li);      // X_t = A_t L^{-T}
      st2(Ls + t * 64 + lane * 2, X[t]);
    }
    fence_async_smem();
    __syncwarp();
    if (lane == 0) bulk_s2g(LT + ((size_t)jb * NTI + J) * (PT + 1) * 64, Ls, (PT + 1) * 64 * sizeof(double));
    F2 Wn[PT + 1][PT + 1];
    F2 Rn[PT + 1];
    // fused forward substitution of the 8 Lagrange columns (transposed)
    F2 Yt = {0.0, 0.0};
    mma(Yt, Rt[0], Li);              // y^T = r^T L^{-T}
    mma(G, Yt, Yt);
    {
      const F2 nY = neg(Yt);
#pragma unroll
      for (int t = 1; t <= PT; ++t) {
        if (SPX && t == PT)
          mma_to_h1(Rn[t - 1], Rt[t], nY, X[t]);
        else
          mma_to(Rn[t - 1], Rt[t], nY, X[t]);
      }
    }
    st_rt(g, Sb, J, lane, Yt);       // y parks in the consumed rhs rows
    Rn[PT] = nR;
    if constexpr (PT >= 1) {
      mma_to(Wn[0][0], W[1][1], neg(X[1]), X[1]);
      TrailPipe2<PT, SPX> pipe{Wn, W, X};
      if (J + 1 < NTI) {
        Li = potrf_inv8_lean(Wn[0][0], Ds, Is, lane, flags, pipe);
      } else {
        pipe.template run<0, PT * (PT + 1) / 2 - 1>();
      }
    }
#pragma unroll
    for (int b = 0; b <= PT; ++b)
      Wn[PT][b] = (In < NTI && ((OM >> (PT - b)) & 1u)) ? fetch(In, b) : F2{0.0, 0.0};
#pragma unroll
    for (int a = 0; a <= PT; ++a) {
#pragma unroll
      for (int b = 0; b <= a; ++b) W[a][b] = Wn[a][b];
      Rt[a] = Rn[a];
    }
  }
  if (lane == 0) bulk_wait_all();
  __syncwarp();
}

template <int PT, bool BWD, unsigned OM, int RF>
__global__ void __launch_bounds__(TC_WARPS * 32)
k_basis_tc(Geo g, const double* __restrict__ w, double* __restrict__ LT, double* __restrict__ Sint,
           double* __restrict__ Kloc, int* __restrict__ flags, int jb0, int jb1) {
  __shared__ __align__(16) double Dsh[TC_WARPS][64];
  __shared__ __align__(16) double Ish[TC_WARPS][72];
  extern __shared__ __align__(16) double tcsm[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int jb = jb0 + blockIdx.x * TC_WARPS + wid;
  if (jb >= jb1) return;
  const int NTI = (g.nI + 7) >> 3, NR = 8 * NTI;
  const int NF = face_off(g, 5) + g.ni1 * g.ni2;
  const int AFE = (NR * AROW + NF + 1) & ~1;   // stencil table + face conductances, even
  double* As = tcsm + (size_t)wid * (AFE + (OM ? 2 * (PT + 1) * 64 : 0));
  double* Fk = As + NR * AROW;
  double* Sb = Sint + (size_t)jb * 8 * g.nI;
  const int bi = jb % g.nb1, bj = (jb / g.nb1) % g.nb2, bk = jb / (g.nb1 * g.nb2);
  const int X0 = bi * g.b1, Y0 = bj * g.b2, Z0 = bk * g.b3;
  const int m = lane >> 2, q = lane & 3;
  double* Ds = Dsh[wid];
  double* Is = Ish[wid];
  stencil_table(g, w, X0, Y0, Z0, NR, As, Fk, Sb, lane, jb);
  __syncwarp();
  // tile offsets (I - K) that can hold stencil entries: d in {0, 1, ni1, p}
  unsigned omask = 1u;
  {
    const int ds[3] = {g.ni1 >= 2 ? 1 : 0, g.ni2 >= 2 ? g.ni1 : 0, g.ni3 >= 2 ? g.p : 0};
#pragma unroll
    for (int s = 0; s < 3; ++s) {
      const int d = ds[s];
      if (d <= 0) continue;
      for (int o = d / 8; o <= (d + 7) / 8; ++o) omask |= 1u << o;
    }
  }
  // per-lane table slots of the entering row: element (b, s) of W[PT][b]
  // is A(i, i - d) with d = 8 (PT - b) + m - 2q - s
  unsigned long long sel = 0;
#pragma unroll
  for (int b = 0; b <= PT; ++b)
#pragma unroll
    for (int s = 0; s < 2; ++s)
      sel |= (unsigned long long)sel_code(g, 8 * (PT - b) + m - 2 * q - s) << (6 * b + 3 * s);
  // tile (I, I - (PT - b)) of A, C layout, from the stencil table
  auto fetch = [&](int I, int b) -> F2 {
    const double* row = As + (8 * I + m) * AROW;
    return {row[(sel >> (6 * b)) & 7u], row[(sel >> (6 * b + 3)) & 7u]};
  };
  F2 G = {0.0, 0.0};                   // sum_J y_J^T y_J  (= R^T S_I, see the Galerkin block)
  if constexpr (OM != 0) {
    if (NTI > 0) {
      double* Lst = As + AFE;                    // 2 x (PT + 1) tiles, 16-byte aligned
      factor_forward_lean<PT, OM, RF>(g, As, Fk, Sb, LT, jb, lane, Ds, Is, Lst, flags, G);
      __syncwarp();
      if constexpr (BWD) backward_sweep<PT, PT == 7 && OM == 0xC3u>(g, LT, Sb, jb, lane);
      __syncwarp();
    }
  } else if (NTI > 0) {
    F2 W[PT + 1][PT + 1];
    F2 Rt[PT + 1];
#pragma unroll
    for (int a = 0; a <= PT; ++a) {
#pragma unroll
      for (int b = 0; b <= PT; ++b) {
        W[a][b] = {0.0, 0.0};
        if (b <= a && ((omask >> (a - b)) & 1u)) W[a][b] = fetch(a, PT - a + b);
      }
      Rt[a] = ld_rt(g, Sb, a, lane);
    }
    F2 Li = potrf_inv8(W[0][0], Ds, Is, lane, flags);
    for (int J = 0; J < NTI; ++J) {
      const int In = J + 1 + PT;       // tile row entering the window after this step
      const F2 nR = In < NTI ? ld_rt(g, Sb, In, lane) : F2{0.0, 0.0};
      F2 X[PT + 1];
      double* Lt = LT + ((size_t)jb * NTI + J) * (PT + 1) * 64 + lane * 2;
      st2(Lt, Li);
#pragma unroll
      for (int t = 1; t <= PT; ++t) {
        X[t] = {0.0, 0.0};
        mma(X[t], W[t][0], Li);                // X_t = A_t L^{-T}
        st2(Lt + t * 64, X[t]);
      }
      // fused forward substitution of the 8 Lagrange columns (transposed)
      F2 Yt = {0.0, 0.0};
      mma(Yt, Rt[0], Li);                      // y^T = r^T L^{-T}
      mma(G, Yt, Yt);
      {
        const F2 nY = neg(Yt);
#pragma unroll
        for (int t = 1; t <= PT; ++t) mma(Rt[t], nY, X[t]);   // r_t^T -= y^T X_t^T
      }
      st_rt(g, Sb, J, lane, Yt);               // y parks in the consumed rhs rows
      // trailing update: the next diagonal tile first, then its POTRF with
      // the remaining tile updates interleaved between the pivots
      if constexpr (PT >= 1) {
        mma(W[1][1], neg(X[1]), X[1]);
        TrailPipe<PT> pipe{W, X};
        if (J + 1 < NTI) {
          Li = potrf_inv8_pipe(W[1][1], Ds, Is, lane, flags, pipe);
        } else {
          trail<PT, 0, PT * (PT + 1) / 2 - 1>(W, X);
        }
      }
      // slide the window by one tile
#pragma unroll
      for (int a = 1; a <= PT; ++a) {
#pragma unroll
        for (int b = 1; b <= a; ++b) W[a - 1][b - 1] = W[a][b];
        Rt[a - 1] = Rt[a];
      }
#pragma unroll
      for (int b = 0; b <= PT; ++b)
        W[PT][b] = (In < NTI && ((omask >> (PT - b)) & 1u)) ? fetch(In, b) : F2{0.0, 0.0};
      Rt[PT] = nR;
    }
    __syncwarp();
    if constexpr (BWD) backward_sweep<PT>(g, LT, Sb, jb, lane);
    __syncwarp();
  }

  // ---- local Galerkin block K_j = sum_{owned e} (w_e/h^2) dS_e dS_e^T (interior part).
  // Edges touching the interior contribute S_I^T(A S)_I + S_B^T(A^I S)_B and
  // (A S)_I = 0 is the local problem just solved, so only the boundary-interior
  // edges remain: sum_e k_e h(x_e) (h(x_e) - S_I(i_e))^T = B - R^T S_I with
  // B = sum_e k_e h h^T and R the Lagrange rhs; R^T S_I = R^T A_II^-1 R = Y^T Y
  // with Y = L^-1 R, accumulated during the forward sweep (G).  Skeleton-only
  // owned edges (model-independent hats) are added by k_skel_galerkin.
  // B is a DMMA reduction, 4 edges (k) x 8 corners per instruction: lane
  // (corner cc = lane/4, edge slot lane%4).
  const int cc = lane >> 2, slot = lane & 3;
  const int cx = cc & 1, cy = (cc >> 1) & 1, cz = (cc >> 2) & 1;
  F2 K = {0.0, 0.0};
  if constexpr (OM != 0) {
    galerkin_faces7(g, Fk, lane, K);
  } else if (NTI > 0) {   // blocks one cell thick along an axis have no interior: no boundary-interior edges
#pragma unroll 1
  for (int face = 0; face < 6; ++face) {
    const int ax = face >> 1, hi = face & 1;
    const int nu = ax == 0 ? g.ni2 : g.ni1, nv = ax == 2 ? g.ni2 : g.ni3;
    const int tot = nu * nv;
    // hat factors: face normal exactly 0/1, in-face axes u, v
    const bool on = (ax == 0 ? cx : (ax == 1 ? cy : cz)) == hi;
    const int cu = ax == 0 ? cy * g.b2 : cx * g.b1, cv = ax == 2 ? cy * g.b2 : cz * g.b3;
    const double ibu = ax == 0 ? g.ib2 : g.ib1, ibv = ax == 2 ? g.ib2 : g.ib3;
    const double* F = Fk + face_off(g, face);
    int u = 1 + slot, v = 1;
    while (u > nu) { u -= nu; ++v; }
    for (int base = 0; base < tot; base += 4) {
      const int f = base + slot;
      double a = 0.0, b = 0.0;
      if (f < tot && on) {
        b = hatf1(u - cu, ibu) * hatf1(v - cv, ibv);
        a = F[f] * b;
      }
      mma884(K.x, K.y, a, b);
      u += 4;
      while (u > nu) { u -= nu; ++v; }
    }
  }
  }
  K.x -= G.x;
  K.y -= G.y;
  st2(Kloc + (size_t)jb * 64 + lane * 2, K);
}

// Backward sweeps only (S_I from the parked y): a small persistent grid (one
// 2-warp CTA per two SMs) so it can run beside the cooperative coarse
// factorization, which needs a CTA slot on every SM.
constexpr int BWD_WARPS = 8;   // one 256-thread CTA per SM (register-limited)
template <int PT, bool SPX>
__global__ void __launch_bounds__(BWD_WARPS * 32) k_basis_bwd(Geo g, const double* __restrict__ LT,
                                                              double* __restrict__ Sint) {
  const int lane = threadIdx.x & 31;
  for (int jb = blockIdx.x * BWD_WARPS + (threadIdx.x >> 5); jb < g.nbl; jb += gridDim.x * BWD_WARPS)
    backward_sweep<PT, SPX>(g, LT, Sint + (size_t)jb * 8 * g.nI, jb, lane);
}

// ------------------------------------------------------- skeleton Galerkin

// Kloc[j] += sum over the skeleton-only edges owned by block j of
// (w_e/h^2) dH_e dH_e^T, where dH_e are the (model-independent) hat
// differences across the edge.  Runs after k_basis_tc (fixed summation order).
// One warp per block, DMMA reduction (lane = corner cc x edge slot) over the
// host-built edge table g.skel (entries needing a "last block" flag the block
// lacks are skipped; the pinned node has no row of S).
constexpr int SKEL_WARPS = 4;
__global__ void __launch_bounds__(SKEL_WARPS * 32) k_skel_galerkin(Geo g, const double* __restrict__ w,
                                                                  double* __restrict__ Kloc, int jb0, int jb1) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int jb = jb0 + blockIdx.x * SKEL_WARPS + wid;
  if (jb >= jb1) return;
  const int bi = jb % g.nb1, bj = (jb / g.nb1) % g.nb2, bk = jb / (g.nb1 * g.nb2);
  const int X0 = bi * g.b1, Y0 = bj * g.b2, Z0 = bk * g.b3;
  const int lx = bi == g.nb1 - 1, ly = bj == g.nb2 - 1, lz = bk == g.nb3 - 1;
  const int cc = lane >> 2, slot = lane & 3;
  const int cb[3] = {(cc & 1) ? g.b1 : 0, (cc & 2) ? g.b2 : 0, (cc & 4) ? g.b3 : 0};
  F2 K = {0.0, 0.0};
#pragma unroll
  for (int ax = 0; ax < 3; ++ax) {
    // transverse axes p (u) and q (v), their block sizes / "last" flags / hat data
    const int pa = ax == 0 ? 1 : 0, qa = ax == 2 ? 1 : 2;
    const int bax = ax == 0 ? g.b1 : (ax == 1 ? g.b2 : g.b3);
    const int bp = pa == 0 ? g.b1 : g.b2, bq = qa == 1 ? g.b2 : g.b3;
    const int lp = pa == 0 ? lx : ly, lq = qa == 1 ? ly : lz;
    const double ibax = ax == 0 ? g.ib1 : (ax == 1 ? g.ib2 : g.ib3);
    const double ibp = pa == 0 ? g.ib1 : g.ib2, ibq = qa == 1 ? g.ib2 : g.ib3;
    const double ihs = ax == 0 ? g.ih1 * g.ih1 : (ax == 1 ? g.ih2 * g.ih2 : g.ih3 * g.ih3);
    const int np_ = bp + lp, nq = bq + lq;
    const long long sx = ax == 0 ? 1 : (ax == 1 ? (long long)(g.n1 + 1) : (long long)(g.n1 + 1) * (g.n2 + 1));
    for (int v = 0; v < nq; ++v) {
      const bool vedge = v == 0 || v == bq;
      for (int u = 0; u < np_; ++u) {
        if (!(vedge || u == 0 || u == bp || bax == 1)) {
          u = bp - 1;            // skip the inner part of the row (u in (0, bp))
          continue;
        }
        const double ht = hatf1(u - cb[pa], ibp) * hatf1(v - cb[qa], ibq);
        int x = 0, y = 0, z = 0;
        if (ax == 0) { y = u; z = v; } else if (ax == 1) { x = u; z = v; } else { x = u; y = v; }
        const long long e0 = ax == 0 ? ex_id(g, X0 + x, Y0 + y, Z0 + z)
                                     : (ax == 1 ? ey_id(g, X0 + x, Y0 + y, Z0 + z) : ez_id(g, X0 + x, Y0 + y, Z0 + z));
        for (int xa0 = 0; xa0 < bax; xa0 += 4) {
          const int xa = xa0 + slot;
          double a = 0.0, b = 0.0;
          if (xa < bax) {
            const bool n0 = jb == 0 && xa == 0 && u == 0 && v == 0;   // pinned node: no row of S
            const double h1 = hatf1(xa + 1 - cb[ax], ibax) * ht;
            const double h0 = n0 ? 0.0 : hatf1(xa - cb[ax], ibax) * ht;
            b = h1 - h0;
            a = (__ldg(w + e0 + xa * sx) * ihs) * b;
          }
          mma884(K.x, K.y, a, b);
        }
      }
    }
  }
  double* kl = Kloc + (size_t)jb * 64 + lane * 2;
  kl[0] += K.x;
  kl[1] += K.y;
}

// Skeleton Galerkin by lines: along an owned skeleton line (axis ax,
// transverse position (u, v)) every hat difference is the same,
// dH_c = s_c ht_c / b_ax with s_c = +-1 (the hats are linear along the
// line) and ht_c the transverse hat product, so the line contributes
// (sum_e w_e / h^2) dH dH^T: the edge weights of a line are summed first and
// the 8x8 block is a DMMA reduction over lines.  Lines are enumerated as in
// the edge loop above (v = 0 all u; 0 < v < bq: u in {0, bp (last block)};
// v = bq (last block) all u).  The pinned node (block 0, first edge of each
// axis' (0,0) line) has no row of S: that edge is its own record with
// dH = H(node 1).  Lanes own lines; records go through shared memory.
// Requires every block extent >= 2 (the edge loop handles extent 1).
constexpr int SKL_WARPS = 4;
__host__ __device__ inline int skel_lines_axis(int bp, int bq, int lp, int lq) {
  return (bp + lp) + (bq - 1) * (1 + lp) + lq * (bp + lp);
}
__global__ void __launch_bounds__(SKL_WARPS * 32) k_skel_lines(Geo g, const double* __restrict__ w,
                                                              double* __restrict__ Kloc, int rec_max, int jb0,
                                                              int jb1, int overwrite) {
  extern __shared__ __align__(16) double skl[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int jb = jb0 + blockIdx.x * SKL_WARPS + wid;
  if (jb >= jb1) return;
  double* ra = skl + (size_t)wid * rec_max * 16;   // record r: a[8] at 16r, b[8] at 16r + 8
  const int bi = jb % g.nb1, bj = (jb / g.nb1) % g.nb2, bk = jb / (g.nb1 * g.nb2);
  const int X0 = bi * g.b1, Y0 = bj * g.b2, Z0 = bk * g.b3;
  const int lx = bi == g.nb1 - 1, ly = bj == g.nb2 - 1, lz = bk == g.nb3 - 1;
  const int nl0 = skel_lines_axis(g.b2, g.b3, ly, lz);
  const int nl1 = skel_lines_axis(g.b1, g.b3, lx, lz);
  const int nl2 = skel_lines_axis(g.b1, g.b2, lx, ly);
  const int NL = nl0 + nl1 + nl2, NR = NL + (jb == 0 ? 3 : 0);
  for (int r = lane; r < NR; r += 32) {
    int ax, L;
    if (r < NL) {
      ax = r < nl0 ? 0 : (r < nl0 + nl1 ? 1 : 2);
      L = r - (ax == 0 ? 0 : (ax == 1 ? nl0 : nl0 + nl1));
    } else {
      ax = r - NL;                                  // pinned-node records
      L = 0;
    }
    const int pa = ax == 0 ? 1 : 0, qa = ax == 2 ? 1 : 2;
    const int bax = ax == 0 ? g.b1 : (ax == 1 ? g.b2 : g.b3);
    const int bp = pa == 0 ? g.b1 : g.b2, bq = qa == 1 ? g.b2 : g.b3;
    const int lp = pa == 0 ? lx : ly;
    const double ibax = ax == 0 ? g.ib1 : (ax == 1 ? g.ib2 : g.ib3);
    const double ibp = pa == 0 ? g.ib1 : g.ib2, ibq = qa == 1 ? g.ib2 : g.ib3;
    const double ihs = ax == 0 ? g.ih1 * g.ih1 : (ax == 1 ? g.ih2 * g.ih2 : g.ih3 * g.ih3);
    const long long sx = ax == 0 ? 1 : (ax == 1 ? (long long)(g.n1 + 1) : (long long)(g.n1 + 1) * (g.n2 + 1));
    const int np_ = bp + lp, nU = 1 + lp;
    int u, v;
    if (L < np_) {
      v = 0;
      u = L;
    } else if (L < np_ + (bq - 1) * nU) {
      const int L2 = L - np_;
      v = 1 + L2 / nU;
      u = (L2 % nU) ? bp : 0;
    } else {
      v = bq;
      u = L - np_ - (bq - 1) * nU;
    }
    int x = 0, y = 0, z = 0;
    if (ax == 0) { y = u; z = v; } else if (ax == 1) { x = u; z = v; } else { x = u; y = v; }
    const long long e0 = ax == 0 ? ex_id(g, X0 + x, Y0 + y, Z0 + z)
                                 : (ax == 1 ? ey_id(g, X0 + x, Y0 + y, Z0 + z) : ez_id(g, X0 + x, Y0 + y, Z0 + z));
    const bool pin_line = jb == 0 && u == 0 && v == 0;
    double wsum, scale;
    if (r < NL) {
      wsum = 0.0;
#pragma unroll 8
      for (int xa = pin_line ? 1 : 0; xa < bax; ++xa) wsum += __ldg(w + e0 + xa * sx);
      scale = ibax;                                 // |dH| along the line, times s_c below
    } else {
      wsum = __ldg(w + e0);
      scale = 0.0;                                  // pinned edge: H(node 1) (set per corner)
    }
    const double wl = wsum * ihs;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int cbp = ((pa == 0 ? c & 1 : (c >> 1) & 1)) ? bp : 0;
      const int cbq = ((qa == 1 ? (c >> 1) & 1 : (c >> 2) & 1)) ? bq : 0;
      const int cba = (ax == 0 ? c & 1 : (ax == 1 ? (c >> 1) & 1 : (c >> 2) & 1));
      const double ht = hatf1(u - cbp, ibp) * hatf1(v - cbq, ibq);
      double d;
      if (r < NL) d = (cba ? scale : -scale) * ht;
      else d = hatf1(1 - (cba ? bax : 0), ibax) * ht;
      ra[16 * r + c] = wl * d;
      ra[16 * r + 8 + c] = d;
    }
  }
  __syncwarp();
  const int cc = lane >> 2, slot = lane & 3;
  F2 K = {0.0, 0.0};
  for (int r0 = 0; r0 < NR; r0 += 4) {
    const int r = r0 + slot;
    const double a = r < NR ? ra[16 * r + cc] : 0.0;
    const double b = r < NR ? ra[16 * r + 8 + cc] : 0.0;
    mma884(K.x, K.y, a, b);
  }
  double* kl = Kloc + (size_t)jb * 64 + lane * 2;
  if (overwrite) {
    kl[0] = K.x;
    kl[1] = K.y;
  } else {
    kl[0] += K.x;
    kl[1] += K.y;
  }
}

__global__ void k_kloc_add(double* __restrict__ Kloc, const double* __restrict__ Ks, long long i0, long long i1) {
  const long long i = i0 + blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < i1) Kloc[i] += Ks[i];
}

// The skeleton line sums depend only on the edge weights: they run on a side
// stream beside the basis kernel (into a scratch copy, added to Kloc once
// both are done).  Per device: stream, two events, scratch.
namespace {
struct SkelSide {
  cudaStream_t st = nullptr;
  cudaEvent_t ew = nullptr, ed = nullptr, ek = nullptr;   // w ready | sums done | scratch consumed
  bool ek_live = false;
  double* buf = nullptr;
  size_t cap = 0;
  std::mutex mu;                                           // host-side sequence (one build at a time per device)
};
SkelSide g_skel_side[64];
}

// ------------------------------------------------------------ block solve

// out = blockdiag(A_II^{-1}) rhs on block interiors (full node fields); out
// may alias rhs.  NCH chunks of 8 right-hand sides ride through one sweep so
// each factor tile is read once per NCH*8 sources; the next step's tiles are
// prefetched into registers.  Right-hand sides are carried transposed (lane
// 4c+q: rows 8I+2q, 8I+2q+1 of column c) so every product is X Y^T of two
// C-layout tiles (see ld_t).  y is parked in out between the sweeps.
// With compact != 0 the warps run over nlist blocks (blist[slot], or slot
// itself when blist is null) and rhs/out are compact per-block interior
// fields (row slot*nI + a).
template <int PT, int NCH>
__global__ void __launch_bounds__(TC_WARPS * 32)
k_block_solve_tc(Geo g, const double* __restrict__ LT, const double* rhs, double* out, int nrhs,
                 const int* __restrict__ blist, int nlist, int compact) {
  extern __shared__ int crd[];
  fill_coords(g, crd);
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int widx = blockIdx.x * TC_WARPS + wid;
  if (widx >= (compact ? nlist : g.nbl)) return;
  const int jb = blist ? blist[widx] : widx;
  const int NTI = (g.nI + 7) >> 3;
  if (NTI == 0) return;
  const int bi = jb % g.nb1, bj = (jb / g.nb1) % g.nb2, bk = jb / (g.nb1 * g.nb2);
  const int X0 = bi * g.b1, Y0 = bj * g.b2, Z0 = bk * g.b3;
  const int c = lane >> 2, q = lane & 3;
  auto node_of = [&](int a) -> long long {
    if (a >= g.nI) return -1;
    if (compact) return (long long)widx * g.nI + a;
    const int v = crd[a];
    return node_id(g, X0 + (v & 1023), Y0 + ((v >> 10) & 1023), Z0 + (v >> 20));
  };
  const double* LTb = LT + (size_t)jb * NTI * (PT + 1) * 64;
  auto load_fwd = [&](int J, F2* Lt) {
    const double* p = LTb + (size_t)J * (PT + 1) * 64 + lane * 2;
#pragma unroll
    for (int t = 0; t <= PT; ++t) Lt[t] = (t == 0 || J + t < NTI) ? ld2(p + t * 64) : F2{0.0, 0.0};
  };
  auto load_bwd = [&](int J, F2* Lt) {
    const double* p = LTb + (size_t)J * (PT + 1) * 64;
#pragma unroll
    for (int t = 0; t <= PT; ++t) Lt[t] = (t == 0 || J + t < NTI) ? ld_t(p + t * 64, lane) : F2{0.0, 0.0};
  };
  for (int s0 = 0; s0 < nrhs; s0 += 8 * NCH) {
    auto load_tile = [&](const double* src, int I, F2* v) {
      const long long n0 = node_of(8 * I + 2 * q), n1 = node_of(8 * I + 2 * q + 1);
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch) {
        const int col = s0 + 8 * ch + c;
        v[ch] = {0.0, 0.0};
        if (col < nrhs) {
          if (n0 >= 0) v[ch].x = src[n0 * nrhs + col];
          if (n1 >= 0) v[ch].y = src[n1 * nrhs + col];
        }
      }
    };
    auto store_tile = [&](int I, const F2* v) {
      const long long n0 = node_of(8 * I + 2 * q), n1 = node_of(8 * I + 2 * q + 1);
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch) {
        const int col = s0 + 8 * ch + c;
        if (col < nrhs) {
          if (n0 >= 0) out[n0 * nrhs + col] = v[ch].x;
          if (n1 >= 0) out[n1 * nrhs + col] = v[ch].y;
        }
      }
    };
    F2 R[PT + 1][NCH];
#pragma unroll
    for (int a = 0; a <= PT; ++a) load_tile(rhs, a, R[a]);
    F2 nL[PT + 1];
    load_fwd(0, nL);
    // forward: y_J^T = r_J^T L_JJ^{-T} ; r_{J+t}^T -= y_J^T L_{J+t,J}^T
    for (int J = 0; J < NTI; ++J) {
      F2 cL[PT + 1];
#pragma unroll
      for (int t = 0; t <= PT; ++t) cL[t] = nL[t];
      if (J + 1 < NTI) load_fwd(J + 1, nL);
      F2 nxt[NCH];
      load_tile(rhs, J + 1 + PT, nxt);            // read ahead before y_J lands (out may alias rhs)
      F2 Yc[NCH];
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch) {
        Yc[ch] = {0.0, 0.0};
        mma(Yc[ch], R[0][ch], cL[0]);
        const F2 nY = neg(Yc[ch]);
#pragma unroll
        for (int t = 1; t <= PT; ++t)
          if (J + t < NTI) mma(R[t][ch], nY, cL[t]);
      }
      __syncwarp();
      store_tile(J, Yc);
#pragma unroll
      for (int a = 1; a <= PT; ++a)
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) R[a - 1][ch] = R[a][ch];
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch) R[PT][ch] = nxt[ch];
    }
    __syncwarp();
    // backward: x_J^T = (y_J^T - sum_t x_{J+t}^T L_{J+t,J}) L_JJ^{-1}; the
    // window keeps -x^T
    F2 Xw[PT > 0 ? PT : 1][NCH];
#pragma unroll
    for (int t = 0; t < (PT > 0 ? PT : 1); ++t)
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch) Xw[t][ch] = {0.0, 0.0};
    load_bwd(NTI - 1, nL);
    for (int J = NTI - 1; J >= 0; --J) {
      F2 cT[PT + 1];
#pragma unroll
      for (int t = 0; t <= PT; ++t) cT[t] = nL[t];
      if (J > 0) load_bwd(J - 1, nL);
      F2 acc[NCH];
      load_tile(out, J, acc);
      F2 xj[NCH];
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch) {
#pragma unroll
        for (int t = 1; t <= PT; ++t)
          if (J + t < NTI) mma(acc[ch], Xw[t - 1][ch], cT[t]);
        xj[ch] = {0.0, 0.0};
        mma(xj[ch], acc[ch], cT[0]);
      }
      __syncwarp();
      store_tile(J, xj);
#pragma unroll
      for (int t = PT - 1; t >= 1; --t)
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) Xw[t][ch] = Xw[t - 1][ch];
      if (PT > 0)
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) Xw[0][ch] = neg(xj[ch]);
    }
    __syncwarp();
  }
}

// ------------------------------------------------------------- launchers

int tc_band(const Geo& g) {
  const int nti = (g.nI + 7) / 8;
  if (nti == 0) return 0;
  int pt = (g.p + 7) / 8;
  if (pt > nti - 1) pt = nti - 1;
  return pt;
}

bool tc_supported(const Geo& g) { return tc_band(g) <= TC_MAX_PT; }

size_t tc_factor_doubles(const Geo& g) {
  const size_t nti = (g.nI + 7) / 8;
  return (size_t)g.nbl * nti * (tc_band(g) + 1) * 64;
}
size_t tc_scratch_doubles(const Geo&) { return 0; }

template <int PT, unsigned OM, int RF = 0>
static cudaError_t launch_basis_tc_k(const Geo& g, const double* w, double* LT, double* Sint, double* Kloc,
                                     int* flags, bool bwd, cudaStream_t st, int jb0, int jb1) {
  const unsigned grid = (unsigned)((jb1 - jb0 + TC_WARPS - 1) / TC_WARPS);
  if (grid == 0) return cudaSuccess;
  const size_t nf = 2 * ((size_t)g.ni2 * g.ni3 + (size_t)g.ni1 * g.ni3 + (size_t)g.ni1 * g.ni2);
  const size_t smem =
      (size_t)TC_WARPS * (((((g.nI + 7) / 8) * 8 * AROW + nf + 1) & ~(size_t)1) + (OM ? 2 * (PT + 1) * 64 : 0)) *
      sizeof(double);
  cudaError_t e =
      cudaFuncSetAttribute(k_basis_tc<PT, true, OM, RF>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_basis_tc<PT, false, OM, RF>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (bwd)
    k_basis_tc<PT, true, OM, RF><<<grid, TC_WARPS * 32, smem, st>>>(g, w, LT, Sint, Kloc, flags, jb0, jb1);
  else
    k_basis_tc<PT, false, OM, RF><<<grid, TC_WARPS * 32, smem, st>>>(g, w, LT, Sint, Kloc, flags, jb0, jb1);
  return cudaSuccess;
}
// lean main loop for 7x7x7 interiors (every 3D BASELINE config: 8^3-cell
// blocks); MSFV_BASIS_VARIANT=0 forces the generic loop (1..3: rhs tiles from
// Sint / first window evaluated in place / all evaluated in place)
static int basis_variant(const Geo& g) {
  const char* e = getenv("MSFV_BASIS_VARIANT");
  const int v = e ? atoi(e) : 1;
  return g.ni1 == 7 && g.ni2 == 7 && g.ni3 == 7 ? v : 0;
}
template <int PT>
static cudaError_t launch_basis_tc_t(const Geo& g, const double* w, double* LT, double* Sint,
                                     double* Kloc, int* flags, bool bwd, cudaStream_t st, int jb0, int jb1) {
  cudaError_t e;
  // reduced boundary conditions (g.bx): the kernel factors, solves and parks its (hat-based) Galerkin block;
  // the caller recomputes Kloc from the actual skeleton values (launch_lg_galerkin) -- no hat skeleton sums here
  const bool reduced = g.bx != nullptr;
  const bool lines = !reduced && g.b1 >= 2 && g.b2 >= 2 && g.b3 >= 2;   // k_skel_galerkin: blocks one cell thick
  const int rec_max = skel_lines_axis(g.b2, g.b3, 1, 1) + skel_lines_axis(g.b1, g.b3, 1, 1) +
                      skel_lines_axis(g.b1, g.b2, 1, 1) + 3;
  const size_t skl_sm = (size_t)SKL_WARPS * rec_max * 16 * sizeof(double);
  if (lines && skl_sm > 48 * 1024) {
    e = cudaFuncSetAttribute(k_skel_lines, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)skl_sm);
    if (e != cudaSuccess) return e;
  }
  SkelSide* side = nullptr;
  std::unique_lock<std::mutex> side_lock;
  if (lines && !getenv("MSFV_SKEL_SERIAL")) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev >= 0 && dev < 64) {
      side = &g_skel_side[dev];
      side_lock = std::unique_lock<std::mutex>(side->mu);
      if (!side->st) {
        e = cudaStreamCreateWithFlags(&side->st, cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&side->ew, cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&side->ed, cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&side->ek, cudaEventDisableTiming);
        if (e != cudaSuccess) return e;
      }
      const size_t need = (size_t)g.nbl * 64;
      if (side->cap < need) {
        if (side->buf) {
          cudaDeviceSynchronize();
          cudaFree(side->buf);
        }
        side->buf = nullptr;
        side->cap = 0;
        e = cudaMalloc(&side->buf, need * sizeof(double));
        if (e != cudaSuccess) return e;
        side->cap = need;
      }
      // skeleton sums first (their CTAs take SMs before the long basis kernel fills them)
      e = cudaEventRecord(side->ew, st);
      if (e == cudaSuccess) e = cudaStreamWaitEvent(side->st, side->ew, 0);
      // the scratch is reused: the previous build's add (possibly on another stream) must have read it
      if (e == cudaSuccess && side->ek_live) e = cudaStreamWaitEvent(side->st, side->ek, 0);
      if (e != cudaSuccess) return e;
      k_skel_lines<<<(unsigned)((jb1 - jb0 + SKL_WARPS - 1) / SKL_WARPS), SKL_WARPS * 32, skl_sm, side->st>>>(
          g, w, side->buf, rec_max, jb0, jb1, 1);
      count_launches(1);
      e = cudaGetLastError();
      if (e == cudaSuccess) e = cudaEventRecord(side->ed, side->st);
      if (e != cudaSuccess) return e;
    }
  }
  if constexpr (PT == 7) {
    const int v = reduced ? (basis_variant(g) ? 1 : 0) : basis_variant(g);   // reduced: right-hand sides from Sint only
    if (v == 1)
      e = launch_basis_tc_k<7, 0xC3u, 0>(g, w, LT, Sint, Kloc, flags, bwd, st, jb0, jb1);
    else if (v == 2)
      e = launch_basis_tc_k<7, 0xC3u, 1>(g, w, LT, Sint, Kloc, flags, bwd, st, jb0, jb1);
    else if (v == 3)
      e = launch_basis_tc_k<7, 0xC3u, 2>(g, w, LT, Sint, Kloc, flags, bwd, st, jb0, jb1);
    else
      e = launch_basis_tc_k<PT, 0u>(g, w, LT, Sint, Kloc, flags, bwd, st, jb0, jb1);
  } else {
    e = launch_basis_tc_k<PT, 0u>(g, w, LT, Sint, Kloc, flags, bwd, st, jb0, jb1);
  }
  if (e != cudaSuccess) return e;
  count_launches(1);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (side) {
    e = cudaStreamWaitEvent(st, side->ed, 0);
    if (e != cudaSuccess) return e;
    const long long i0 = (long long)jb0 * 64, i1 = (long long)jb1 * 64;
    k_kloc_add<<<(unsigned)((i1 - i0 + 255) / 256), 256, 0, st>>>(Kloc, side->buf, i0, i1);
    e = cudaEventRecord(side->ek, st);
    if (e != cudaSuccess) return e;
    side->ek_live = true;
  } else if (lines) {
    k_skel_lines<<<(unsigned)((jb1 - jb0 + SKL_WARPS - 1) / SKL_WARPS), SKL_WARPS * 32, skl_sm, st>>>(
        g, w, Kloc, rec_max, jb0, jb1, 0);
  } else if (reduced) {
    return cudaSuccess;
  } else
    k_skel_galerkin<<<(unsigned)((jb1 - jb0 + SKEL_WARPS - 1) / SKEL_WARPS), SKEL_WARPS * 32, 0, st>>>(g, w, Kloc,
                                                                                                     jb0, jb1);
  count_launches(1);
  return cudaGetLastError();
}
template <int PT>
static cudaError_t launch_solve_tc_t(const Geo& g, const double* LT, const double* rhs, double* out, int nrhs,
                                     const int* blist, int nlist, int compact, cudaStream_t st) {
  const int nw = compact ? nlist : g.nbl;
  const unsigned grid = (unsigned)((nw + TC_WARPS - 1) / TC_WARPS);
  const size_t smem = (size_t)g.nI * sizeof(int);
  if (nrhs > 8)
    k_block_solve_tc<PT, 2><<<grid, TC_WARPS * 32, smem, st>>>(g, LT, rhs, out, nrhs, blist, nlist, compact);
  else
    k_block_solve_tc<PT, 1><<<grid, TC_WARPS * 32, smem, st>>>(g, LT, rhs, out, nrhs, blist, nlist, compact);
  count_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_basis_tc(const Geo& g, const double* w, double* LT, double* Sint, double* Kloc,
                            int* flags, cudaStream_t st, bool bwd, int jb0, int jb1) {
  if (jb1 < 0) jb1 = g.nbl;
  if (jb1 <= jb0) return cudaSuccess;
  switch (tc_band(g)) {
    case 0: return launch_basis_tc_t<0>(g, w, LT, Sint, Kloc, flags, bwd, st, jb0, jb1);
    case 1: return launch_basis_tc_t<1>(g, w, LT, Sint, Kloc, flags, bwd, st, jb0, jb1);
    case 2: return launch_basis_tc_t<2>(g, w, LT, Sint, Kloc, flags, bwd, st, jb0, jb1);
    case 3: return launch_basis_tc_t<3>(g, w, LT, Sint, Kloc, flags, bwd, st, jb0, jb1);
    case 4: return launch_basis_tc_t<4>(g, w, LT, Sint, Kloc, flags, bwd, st, jb0, jb1);
    case 5: return launch_basis_tc_t<5>(g, w, LT, Sint, Kloc, flags, bwd, st, jb0, jb1);
    case 6: return launch_basis_tc_t<6>(g, w, LT, Sint, Kloc, flags, bwd, st, jb0, jb1);
    case 7: return launch_basis_tc_t<7>(g, w, LT, Sint, Kloc, flags, bwd, st, jb0, jb1);
    default: return cudaErrorInvalidValue;
  }
}

template <int PT>
static cudaError_t launch_basis_bwd_t(const Geo& g, const double* LT, double* Sint, cudaStream_t st) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // persistent, one 8-warp CTA on all but a few SMs: the register file of a
  // busy SM is then full, so the latency-bound coarse sweeps this kernel runs
  // beside land on the SMs left free
  static int free_sms = -1;
  if (free_sms < 0) {
    const char* e = getenv("MSFV_BWD_FREE_SMS");
    free_sms = e ? std::max(0, atoi(e)) : 12;
  }
  // multifrontal coarse path: the sweeps start right after the forward part
  // and run on the SMs the coarse kernels leave free (mf_reserved_sms)
  const int want = g.coarse_nd == 2 ? std::max(1, mf_reserved_sms()) : sms - free_sms;
  const int grid = std::max(1, std::min((g.nbl + BWD_WARPS - 1) / BWD_WARPS, want));
  if (PT == 7 && g.p == 8 * PT - 7 && g.ni1 == 7 && g.ni2 == 7)
    k_basis_bwd<PT, true><<<grid, BWD_WARPS * 32, 0, st>>>(g, LT, Sint);
  else
    k_basis_bwd<PT, false><<<grid, BWD_WARPS * 32, 0, st>>>(g, LT, Sint);
  count_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_basis_bwd(const Geo& g, const double* LT, double* Sint, cudaStream_t st) {
  switch (tc_band(g)) {
    case 0: return launch_basis_bwd_t<0>(g, LT, Sint, st);
    case 1: return launch_basis_bwd_t<1>(g, LT, Sint, st);
    case 2: return launch_basis_bwd_t<2>(g, LT, Sint, st);
    case 3: return launch_basis_bwd_t<3>(g, LT, Sint, st);
    case 4: return launch_basis_bwd_t<4>(g, LT, Sint, st);
    case 5: return launch_basis_bwd_t<5>(g, LT, Sint, st);
    case 6: return launch_basis_bwd_t<6>(g, LT, Sint, st);
    case 7: return launch_basis_bwd_t<7>(g, LT, Sint, st);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_block_solve_tc(const Geo& g, const double* LT, const double* rhs, double* out, int nrhs,
                                  cudaStream_t st, const int* blist, int nlist, int compact) {
  if (g.nI == 0 || nrhs == 0 || (compact && nlist == 0)) return cudaSuccess;
  switch (tc_band(g)) {
    case 0: return launch_solve_tc_t<0>(g, LT, rhs, out, nrhs, blist, nlist, compact, st);
    case 1: return launch_solve_tc_t<1>(g, LT, rhs, out, nrhs, blist, nlist, compact, st);
    case 2: return launch_solve_tc_t<2>(g, LT, rhs, out, nrhs, blist, nlist, compact, st);
    case 3: return launch_solve_tc_t<3>(g, LT, rhs, out, nrhs, blist, nlist, compact, st);
    case 4: return launch_solve_tc_t<4>(g, LT, rhs, out, nrhs, blist, nlist, compact, st);
    case 5: return launch_solve_tc_t<5>(g, LT, rhs, out, nrhs, blist, nlist, compact, st);
    case 6: return launch_solve_tc_t<6>(g, LT, rhs, out, nrhs, blist, nlist, compact, st);
    case 7: return launch_solve_tc_t<7>(g, LT, rhs, out, nrhs, blist, nlist, compact, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace msfv
