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
#include "msfv_common.cuh"
#include "msfv_kernels.h"

namespace msfv {
namespace {

constexpr unsigned FULL = 0xffffffffu;

struct F2 {
  double x, y;
};

__device__ __forceinline__ void mma884(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}
// C (accumulator layout) += A (A-frag) * B (B-frag), k = 8
__device__ __forceinline__ void mma(F2& c, const F2& a, const F2& b) {
  mma884(c.x, c.y, a.x, b.x);
  mma884(c.x, c.y, a.y, b.y);
}
__device__ __forceinline__ F2 neg(const F2& f) { return {-f.x, -f.y}; }

// accumulator tile T -> A-frag of T
__device__ __forceinline__ F2 c_to_a(const F2& c, int lane) {
  const int m = lane >> 2, k = lane & 3;
  const int s0 = (m << 2) | (k >> 1), s1 = (m << 2) | (2 + (k >> 1));
  double x0 = __shfl_sync(FULL, c.x, s0), y0 = __shfl_sync(FULL, c.y, s0);
  double x1 = __shfl_sync(FULL, c.x, s1), y1 = __shfl_sync(FULL, c.y, s1);
  const bool odd = k & 1;
  return {odd ? y0 : x0, odd ? y1 : x1};
}
// accumulator tile T -> B-frag of T (B[k][n] = T[k][n])
__device__ __forceinline__ F2 c_to_b(const F2& c, int lane) {
  const int k = lane & 3, n = lane >> 2;
  const int s0 = (k << 2) | (n >> 1), s1 = ((k + 4) << 2) | (n >> 1);
  double x0 = __shfl_sync(FULL, c.x, s0), y0 = __shfl_sync(FULL, c.y, s0);
  double x1 = __shfl_sync(FULL, c.x, s1), y1 = __shfl_sync(FULL, c.y, s1);
  const bool odd = n & 1;
  return {odd ? y0 : x0, odd ? y1 : x1};
}
// A-frag of T -> A-frag of T^T (equivalently the B-frag of T)
__device__ __forceinline__ F2 a_to_t(const F2& f, int lane) {
  const int k = lane & 3, n = lane >> 2;
  const int s0 = (k << 2) | (n & 3), s1 = ((k + 4) << 2) | (n & 3);
  double p0 = __shfl_sync(FULL, f.x, s0), q0 = __shfl_sync(FULL, f.y, s0);
  double p1 = __shfl_sync(FULL, f.x, s1), q1 = __shfl_sync(FULL, f.y, s1);
  const bool hi = n >= 4;
  return {hi ? q0 : p0, hi ? q1 : p1};
}

__device__ __forceinline__ F2 ld2(const double* p) {
  double2 v = *reinterpret_cast<const double2*>(p);
  return {v.x, v.y};
}
__device__ __forceinline__ F2 ld2cg(const double* p) {
  double2 v = __ldcg(reinterpret_cast<const double2*>(p));
  return {v.x, v.y};
}
__device__ __forceinline__ void st2(double* p, const F2& f) {
  *reinterpret_cast<double2*>(p) = make_double2(f.x, f.y);
}

// Stencil row of interior node i of a block: the six edge conductances / h^2.
struct Row {
  bool valid;
  int x, y, z;
  double kxm, kxp, kym, kyp, kzm, kzp;
};

// Interior coordinates, packed x | y << 10 | z << 20 (one table per CTA).
__device__ __forceinline__ void fill_coords(const Geo& g, int* crd) {
  for (int a = threadIdx.x; a < g.nI; a += blockDim.x) {
    const int x = 1 + a % g.ni1, y = 1 + (a / g.ni1) % g.ni2, z = 1 + a / (g.ni1 * g.ni2);
    crd[a] = x | (y << 10) | (z << 20);
  }
}

__device__ __forceinline__ Row load_row(const Geo& g, const double* __restrict__ w, const int* crd, int X0, int Y0,
                                        int Z0, int i) {
  Row r;
  r.valid = i < g.nI;
  if (!r.valid) {
    r.x = r.y = r.z = 0;
    r.kxm = r.kxp = r.kym = r.kyp = r.kzm = r.kzp = 0.0;
    return r;
  }
  const int c = crd[i];
  r.x = c & 1023;
  r.y = (c >> 10) & 1023;
  r.z = c >> 20;
  const long long I = X0 + r.x, J = Y0 + r.y, K = Z0 + r.z;
  r.kxm = __ldg(w + ex_id(g, I - 1, J, K)) * g.ih1 * g.ih1;
  r.kxp = __ldg(w + ex_id(g, I, J, K)) * g.ih1 * g.ih1;
  r.kym = __ldg(w + ey_id(g, I, J - 1, K)) * g.ih2 * g.ih2;
  r.kyp = __ldg(w + ey_id(g, I, J, K)) * g.ih2 * g.ih2;
  r.kzm = __ldg(w + ez_id(g, I, J, K - 1)) * g.ih3 * g.ih3;
  r.kzp = __ldg(w + ez_id(g, I, J, K)) * g.ih3 * g.ih3;
  return r;
}

// A_II[i][l] for l <= i (padding rows are identity).
__device__ __forceinline__ double a_entry(const Geo& g, const Row& r, int i, int l) {
  if (!r.valid) return i == l ? 1.0 : 0.0;
  if (l > i) return 0.0;
  const int d = i - l;
  if (d == 0) return ((((r.kxm + r.kxp) + r.kym) + r.kyp) + r.kzm) + r.kzp;
  double v = 0.0;
  if (d == 1 && r.x > 1) v -= r.kxm;
  if (d == g.ni1 && r.y > 1) v -= r.kym;
  if (d == g.p && r.z > 1) v -= r.kzm;
  return v;
}

// Lagrange right-hand side -A_IB x_B (basis.py:548) of node row r, corner cc.
__device__ __forceinline__ double rhs_entry(const Geo& g, const Row& r, int cc) {
  if (!r.valid) return 0.0;
  double v = 0.0;
  if (r.x == 1) v += r.kxm * hatf(g, cc, 0, r.y, r.z);
  if (r.x == g.ni1) v += r.kxp * hatf(g, cc, g.b1, r.y, r.z);
  if (r.y == 1) v += r.kym * hatf(g, cc, r.x, 0, r.z);
  if (r.y == g.ni2) v += r.kyp * hatf(g, cc, r.x, g.b2, r.z);
  if (r.z == 1) v += r.kzm * hatf(g, cc, r.x, r.y, 0);
  if (r.z == g.ni3) v += r.kzp * hatf(g, cc, r.x, r.y, g.b3);
  return v;
}

// Cholesky of one 8x8 SPD tile (accumulator layout); returns L^{-1} as an
// A-frag.  Lanes 0..7 own rows of L in registers (shuffle right-looking
// factorization, rsqrt pivots), then columns of L^{-1}; shared memory is used
// only to re-layout the tile.
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
  const int m = lane >> 2, n0 = 2 * (lane & 3);
  Ds[m * 8 + n0] = t.x;
  Ds[m * 8 + n0 + 1] = t.y;
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
  const int k = lane & 3;
  F2 li = {Is[m * 8 + k], Is[m * 8 + 4 + k]};
  __syncwarp();
  return li;
}

}  // namespace

// ----------------------------------------------------------------- basis

template <int PT>
__global__ void __launch_bounds__(TC_WARPS * 32)
k_basis_tc(Geo g, const double* __restrict__ w, double* __restrict__ LT, double* __restrict__ Sint,
           double* __restrict__ Ysc, double* __restrict__ Kloc, int* __restrict__ flags) {
  __shared__ double Dsh[TC_WARPS][64];
  __shared__ double Ish[TC_WARPS][72];
  extern __shared__ __align__(16) double tcsm[];
  int* crd = reinterpret_cast<int*>(tcsm + (size_t)TC_WARPS * g.nI * 8);
  fill_coords(g, crd);
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double* Sx = tcsm + (size_t)wid * g.nI * 8;     // this block's interior basis values [a][corner]
  const int jb = blockIdx.x * TC_WARPS + wid;
  if (jb >= g.nbl) return;
  const int bi = jb % g.nb1, bj = (jb / g.nb1) % g.nb2, bk = jb / (g.nb1 * g.nb2);
  const int X0 = bi * g.b1, Y0 = bj * g.b2, Z0 = bk * g.b3;
  const int NTI = (g.nI + 7) >> 3;
  const int m = lane >> 2, n0 = 2 * (lane & 3);
  double* Ds = Dsh[wid];
  double* Is = Ish[wid];
  // tile offsets (I - K) that can hold stencil entries: d in {0, 1, ni1, p}
  unsigned omask = 1u;
  {
    const int ds[3] = {g.ni1 >= 2 ? 1 : 0, g.ni2 >= 2 ? g.ni1 : 0, g.ni3 >= 2 ? g.p : 0};
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      const int d = ds[q];
      if (d <= 0) continue;
      for (int o = (d - 7 + 7) / 8; o <= (d + 7) / 8; ++o) omask |= 1u << o;
    }
  }
  if (NTI > 0) {
    F2 W[PT + 1][PT + 1];
    F2 R[PT + 1];
    // ---- initial window: tile rows 0..PT
#pragma unroll
    for (int a = 0; a <= PT; ++a) {
      const int i = 8 * a + m;
      Row rw = load_row(g, w, crd, X0, Y0, Z0, i);
#pragma unroll
      for (int b = 0; b <= PT; ++b) {
        if (b <= a && ((omask >> (a - b)) & 1u)) {
          const int l = 8 * b + n0;
          W[a][b] = {a_entry(g, rw, i, l), a_entry(g, rw, i, l + 1)};
        } else {
          W[a][b] = {0.0, 0.0};
        }
      }
      R[a] = {rhs_entry(g, rw, n0), rhs_entry(g, rw, n0 + 1)};
    }
    for (int J = 0; J < NTI; ++J) {
      // prefetch the stencil row entering the window at the end of this step
      const int inext = 8 * (J + 1 + PT) + m;
      Row rn = load_row(g, w, crd, X0, Y0, Z0, inext);

      const F2 Li = potrf_inv8(W[0][0], Ds, Is, lane, flags);
      F2 X[PT + 1];
#pragma unroll
      for (int t = 1; t <= PT; ++t) {
        F2 c = {0.0, 0.0};
        mma(c, c_to_a(W[t][0], lane), Li);     // X_t = A_t L^{-T}
        X[t] = c_to_a(c, lane);
      }
      // fused forward substitution for the 8 Lagrange columns
      F2 Yc = {0.0, 0.0};
      mma(Yc, Li, c_to_b(R[0], lane));         // y_J = L_JJ^{-1} r_J
      {
        const F2 Yb = c_to_b(Yc, lane);
#pragma unroll
        for (int t = 1; t <= PT; ++t) mma(R[t], neg(X[t]), Yb);
      }
      // trailing update of the register window
#pragma unroll
      for (int a = 1; a <= PT; ++a) {
        const F2 nXa = neg(X[a]);
#pragma unroll
        for (int b = 1; b <= a; ++b) mma(W[a][b], nXa, X[b]);
      }
      // factor tiles and y to global memory
      {
        double* Lt = LT + ((size_t)jb * NTI + J) * (PT + 1) * 64;
        st2(Lt + lane * 2, Li);
#pragma unroll
        for (int t = 1; t <= PT; ++t) st2(Lt + t * 64 + lane * 2, X[t]);
        st2(Ysc + ((size_t)jb * NTI + J) * 64 + lane * 2, Yc);
      }
      // slide the window by one tile
#pragma unroll
      for (int a = 1; a <= PT; ++a) {
#pragma unroll
        for (int b = 1; b <= a; ++b) W[a - 1][b - 1] = W[a][b];
        R[a - 1] = R[a];
      }
      {
        const int In = J + 1 + PT;
#pragma unroll
        for (int b = 0; b <= PT; ++b) {
          if ((omask >> (PT - b)) & 1u) {
            const int l = 8 * (In - PT + b) + n0;
            W[PT][b] = {a_entry(g, rn, inext, l), a_entry(g, rn, inext, l + 1)};
          } else {
            W[PT][b] = {0.0, 0.0};
          }
        }
        R[PT] = {rhs_entry(g, rn, n0), rhs_entry(g, rn, n0 + 1)};
      }
    }
    __syncwarp();
    // ---- backward substitution L^T x = y, window of solved tiles as B-frags;
    // the next step's factor tiles are prefetched into registers.
    F2 Xw[PT > 0 ? PT : 1];
#pragma unroll
    for (int t = 0; t < (PT > 0 ? PT : 1); ++t) Xw[t] = {0.0, 0.0};
    F2 nLt[PT + 1], nY;
    {
      const int J = NTI - 1;
      const double* Lt = LT + ((size_t)jb * NTI + J) * (PT + 1) * 64;
#pragma unroll
      for (int t = 0; t <= PT; ++t) nLt[t] = (t == 0 || J + t < NTI) ? ld2cg(Lt + t * 64 + lane * 2) : F2{0.0, 0.0};
      nY = ld2cg(Ysc + ((size_t)jb * NTI + J) * 64 + lane * 2);
    }
    for (int J = NTI - 1; J >= 0; --J) {
      F2 cLt[PT + 1];
#pragma unroll
      for (int t = 0; t <= PT; ++t) cLt[t] = nLt[t];
      F2 acc = nY;
      if (J > 0) {
        const double* Lt = LT + ((size_t)jb * NTI + J - 1) * (PT + 1) * 64;
#pragma unroll
        for (int t = 0; t <= PT; ++t) nLt[t] = (t == 0 || J - 1 + t < NTI) ? ld2cg(Lt + t * 64 + lane * 2) : F2{0.0, 0.0};
        nY = ld2cg(Ysc + ((size_t)jb * NTI + J - 1) * 64 + lane * 2);
      }
#pragma unroll
      for (int t = 1; t <= PT; ++t) {
        if (J + t < NTI) mma(acc, neg(a_to_t(cLt[t], lane)), Xw[t - 1]);
      }
      F2 xj = {0.0, 0.0};
      mma(xj, a_to_t(cLt[0], lane), c_to_b(acc, lane));
      const int a0 = 8 * J + m;
      if (a0 < g.nI) {
        Sint[((size_t)jb * 8 + n0) * g.nI + a0] = xj.x;
        Sint[((size_t)jb * 8 + n0 + 1) * g.nI + a0] = xj.y;
        st2(Sx + a0 * 8 + n0, xj);
      }
#pragma unroll
      for (int t = PT - 1; t >= 1; --t) Xw[t] = Xw[t - 1];
      if (PT > 0) Xw[0] = c_to_b(xj, lane);
    }
    __syncwarp();
  }

  // ---- local Galerkin block K_j = sum_{owned e} (w_e/h^2) dS_e dS_e^T (interior part).
  // Edges touching the interior contribute S_I^T(A S)_I + S_B^T(A^I S)_B and
  // (A S)_I = 0 is the local problem just solved, so only the boundary-interior
  // edges remain: k_e S(x_e) (S(x_e) - S(i_e))^T.  Skeleton-only owned edges
  // contribute k_e dH dH^T with the model-independent hats.  DMMA reduction,
  // 4 edges (k) x 8 corners per instruction: lane (corner cc = lane/4, edge
  // slot lane%4).
  const int cc = lane >> 2, slot = lane & 3;
  F2 K = {0.0, 0.0};
  // (1) boundary-interior edges, face by face
#pragma unroll 1
  for (int face = 0; face < 6; ++face) {
    const int ax = face >> 1, hi = face & 1;
    const int nu = ax == 0 ? g.ni2 : g.ni1, nv = ax == 2 ? g.ni2 : g.ni3;
    const int tot = nu * nv;
    const double ihs = ax == 0 ? g.ih1 * g.ih1 : (ax == 1 ? g.ih2 * g.ih2 : g.ih3 * g.ih3);
    for (int base = 0; base < tot; base += 4) {
      const int f = base + slot;
      double a = 0.0, b = 0.0;
      if (f < tot) {
        const int u = 1 + f % nu, v = 1 + f / nu;
        int xb, yb, zb, xi, yi, zi, xe, ye, ze;
        if (ax == 0) {
          xb = hi ? g.b1 : 0; yb = u; zb = v; xi = hi ? g.b1 - 1 : 1; yi = u; zi = v;
        } else if (ax == 1) {
          xb = u; yb = hi ? g.b2 : 0; zb = v; xi = u; yi = hi ? g.b2 - 1 : 1; zi = v;
        } else {
          xb = u; yb = v; zb = hi ? g.b3 : 0; xi = u; yi = v; zi = hi ? g.b3 - 1 : 1;
        }
        xe = min(xb, xi); ye = min(yb, yi); ze = min(zb, zi);
        const long long e = ax == 0 ? ex_id(g, X0 + xe, Y0 + ye, Z0 + ze)
                                    : (ax == 1 ? ey_id(g, X0 + xe, Y0 + ye, Z0 + ze) : ez_id(g, X0 + xe, Y0 + ye, Z0 + ze));
        const double sb = hatf(g, cc, xb, yb, zb);
        const double si = Sx[interior_index(g, xi, yi, zi) * 8 + cc];
        b = sb - si;
        a = (__ldg(w + e) * ihs) * sb;
      }
      mma884(K.x, K.y, a, b);
    }
  }
  // (2) skeleton-only owned edges: added by k_skel_galerkin (model-independent hats)
  Kloc[(size_t)jb * 64 + m * 8 + n0] = K.x;
  Kloc[(size_t)jb * 64 + m * 8 + n0 + 1] = K.y;
}

// ------------------------------------------------------- skeleton Galerkin

// Kloc[j] += sum over the skeleton-only edges owned by block j of
// (w_e/h^2) dH_e dH_e^T, where dH_e are the (model-independent) hat
// differences across the edge.  Runs after k_basis_tc (fixed summation order).
__global__ void __launch_bounds__(64) k_skel_galerkin(Geo g, const double* __restrict__ w, double* __restrict__ Kloc) {
  __shared__ double red[36][65];
  const int jb = blockIdx.x;
  const int tid = threadIdx.x;
  const int bi = jb % g.nb1, bj = (jb / g.nb1) % g.nb2, bk = jb / (g.nb1 * g.nb2);
  const int X0 = bi * g.b1, Y0 = bj * g.b2, Z0 = bk * g.b3;
  const int lx = (bi == g.nb1 - 1), ly = (bj == g.nb2 - 1), lz = (bk == g.nb3 - 1);
  const bool has0 = (jb == 0);
  double acc[36];
#pragma unroll
  for (int q = 0; q < 36; ++q) acc[q] = 0.0;
  for (int ax = 0; ax < 3; ++ax) {
    const int xm = g.b1 + (ax == 0 ? 0 : lx), ym = g.b2 + (ax == 1 ? 0 : ly), zm = g.b3 + (ax == 2 ? 0 : lz);
    const int bax = ax == 0 ? g.b1 : (ax == 1 ? g.b2 : g.b3);
    const double ihs = ax == 0 ? g.ih1 * g.ih1 : (ax == 1 ? g.ih2 * g.ih2 : g.ih3 * g.ih3);
    const int tot = xm * ym * zm;
    for (int f = tid; f < tot; f += blockDim.x) {
      const int x = f % xm, q = f / xm, y = q % ym, z = q / ym;
      bool skel;
      if (ax == 0) skel = (y == 0 || y == g.b2 || z == 0 || z == g.b3);
      else if (ax == 1) skel = (x == 0 || x == g.b1 || z == 0 || z == g.b3);
      else skel = (x == 0 || x == g.b1 || y == 0 || y == g.b2);
      if (!(skel || bax == 1)) continue;
      const int x1 = x + (ax == 0), y1 = y + (ax == 1), z1 = z + (ax == 2);
      const long long e = ax == 0 ? ex_id(g, X0 + x, Y0 + y, Z0 + z)
                                  : (ax == 1 ? ey_id(g, X0 + x, Y0 + y, Z0 + z) : ez_id(g, X0 + x, Y0 + y, Z0 + z));
      const double kc = __ldg(w + e) * ihs;
      const bool n0 = has0 && x == 0 && y == 0 && z == 0;
      double dh[8];
#pragma unroll
      for (int cc = 0; cc < 8; ++cc) dh[cc] = hatf(g, cc, x1, y1, z1) - (n0 ? 0.0 : hatf(g, cc, x, y, z));
#pragma unroll
      for (int c1 = 0; c1 < 8; ++c1) {
        const double kd = kc * dh[c1];
#pragma unroll
        for (int c2 = 0; c2 <= c1; ++c2) acc[c1 * (c1 + 1) / 2 + c2] += kd * dh[c2];
      }
    }
  }
#pragma unroll
  for (int q = 0; q < 36; ++q) red[q][tid] = acc[q];
  __syncthreads();
  if (tid < 36) {
    double v = 0.0;
    for (int t = 0; t < blockDim.x; ++t) v += red[tid][t];
    int c1 = 0;
    while ((c1 + 1) * (c1 + 2) / 2 <= tid) ++c1;
    const int c2 = tid - c1 * (c1 + 1) / 2;
    Kloc[(size_t)jb * 64 + c1 * 8 + c2] += v;
    if (c1 != c2) Kloc[(size_t)jb * 64 + c2 * 8 + c1] += v;
  }
}

// ------------------------------------------------------------ block solve

// out = blockdiag(A_II^{-1}) rhs on block interiors (full node fields); out
// may alias rhs.  NCH chunks of 8 right-hand sides ride through one sweep so
// each factor tile is read once per NCH*8 sources; the next step's tiles are
// prefetched into registers.  y is parked in out between the sweeps.
template <int PT, int NCH>
__global__ void __launch_bounds__(TC_WARPS * 32)
k_block_solve_tc(Geo g, const double* __restrict__ LT, const double* rhs, double* out, int nrhs) {
  extern __shared__ int crd[];
  fill_coords(g, crd);
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int jb = blockIdx.x * TC_WARPS + wid;
  if (jb >= g.nbl) return;
  const int NTI = (g.nI + 7) >> 3;
  if (NTI == 0) return;
  const int bi = jb % g.nb1, bj = (jb / g.nb1) % g.nb2, bk = jb / (g.nb1 * g.nb2);
  const int X0 = bi * g.b1, Y0 = bj * g.b2, Z0 = bk * g.b3;
  const int m = lane >> 2, n0 = 2 * (lane & 3);
  auto node_of = [&](int a) -> long long {
    const int c = crd[a];
    return node_id(g, X0 + (c & 1023), Y0 + ((c >> 10) & 1023), Z0 + (c >> 20));
  };
  const double* LTb = LT + (size_t)jb * NTI * (PT + 1) * 64;
  auto load_step = [&](int J, F2* Lt) {
    const double* p = LTb + (size_t)J * (PT + 1) * 64 + lane * 2;
#pragma unroll
    for (int t = 0; t <= PT; ++t) Lt[t] = (t == 0 || J + t < NTI) ? ld2(p + t * 64) : F2{0.0, 0.0};
  };
  for (int s0 = 0; s0 < nrhs; s0 += 8 * NCH) {
    auto load_tile = [&](const double* src, int I, F2* v) {
      const int a = 8 * I + m;
      long long nd = (a < g.nI) ? node_of(a) : -1;
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch) {
        const int sA = s0 + 8 * ch + n0;
        v[ch] = {0.0, 0.0};
        if (nd >= 0) {
          if (sA < nrhs) v[ch].x = src[nd * nrhs + sA];
          if (sA + 1 < nrhs) v[ch].y = src[nd * nrhs + sA + 1];
        }
      }
    };
    auto store_tile = [&](int I, const F2* v) {
      const int a = 8 * I + m;
      if (a >= g.nI) return;
      const long long nd = node_of(a);
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch) {
        const int sA = s0 + 8 * ch + n0;
        if (sA < nrhs) out[nd * nrhs + sA] = v[ch].x;
        if (sA + 1 < nrhs) out[nd * nrhs + sA + 1] = v[ch].y;
      }
    };
    F2 R[PT + 1][NCH];
#pragma unroll
    for (int a = 0; a <= PT; ++a) load_tile(rhs, a, R[a]);
    F2 nL[PT + 1];
    load_step(0, nL);
    // forward: y_J = L_JJ^{-1} r_J ; r_{J+t} -= L_{J+t,J} y_J
    for (int J = 0; J < NTI; ++J) {
      F2 cL[PT + 1];
#pragma unroll
      for (int t = 0; t <= PT; ++t) cL[t] = nL[t];
      if (J + 1 < NTI) load_step(J + 1, nL);
      F2 nxt[NCH];
      load_tile(rhs, J + 1 + PT, nxt);            // read ahead before y_J lands (out may alias rhs)
      F2 Yc[NCH];
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch) {
        Yc[ch] = {0.0, 0.0};
        mma(Yc[ch], cL[0], c_to_b(R[0][ch], lane));
        const F2 Yb = c_to_b(Yc[ch], lane);
#pragma unroll
        for (int t = 1; t <= PT; ++t)
          if (J + t < NTI) mma(R[t][ch], neg(cL[t]), Yb);
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
    // backward: x_J = L_JJ^{-T} (y_J - sum_t L_{J+t,J}^T x_{J+t})
    F2 Xw[PT > 0 ? PT : 1][NCH];
#pragma unroll
    for (int t = 0; t < (PT > 0 ? PT : 1); ++t)
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch) Xw[t][ch] = {0.0, 0.0};
    load_step(NTI - 1, nL);
    for (int J = NTI - 1; J >= 0; --J) {
      F2 cT[PT + 1];
#pragma unroll
      for (int t = 0; t <= PT; ++t) cT[t] = a_to_t(nL[t], lane);   // transposed tiles
      if (J > 0) load_step(J - 1, nL);
      F2 acc[NCH];
      load_tile(out, J, acc);
      F2 xj[NCH];
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch) {
#pragma unroll
        for (int t = 1; t <= PT; ++t)
          if (J + t < NTI) mma(acc[ch], neg(cT[t]), Xw[t - 1][ch]);
        xj[ch] = {0.0, 0.0};
        mma(xj[ch], cT[0], c_to_b(acc[ch], lane));
      }
      __syncwarp();
      store_tile(J, xj);
#pragma unroll
      for (int t = PT - 1; t >= 1; --t)
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) Xw[t][ch] = Xw[t - 1][ch];
      if (PT > 0)
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) Xw[0][ch] = c_to_b(xj[ch], lane);
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
size_t tc_scratch_doubles(const Geo& g) { return (size_t)g.nbl * ((g.nI + 7) / 8) * 64; }

template <int PT>
static cudaError_t launch_basis_tc_t(const Geo& g, const double* w, double* LT, double* Sint, double* Ysc,
                                     double* Kloc, int* flags, cudaStream_t st) {
  const unsigned grid = (unsigned)((g.nbl + TC_WARPS - 1) / TC_WARPS);
  const size_t smem = (size_t)TC_WARPS * g.nI * 8 * sizeof(double) + (size_t)g.nI * sizeof(int);
  cudaError_t e = cudaFuncSetAttribute(k_basis_tc<PT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k_basis_tc<PT><<<grid, TC_WARPS * 32, smem, st>>>(g, w, LT, Sint, Ysc, Kloc, flags);
  count_launches(1);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  k_skel_galerkin<<<g.nbl, 64, 0, st>>>(g, w, Kloc);
  count_launches(1);
  return cudaGetLastError();
}
template <int PT>
static cudaError_t launch_solve_tc_t(const Geo& g, const double* LT, const double* rhs, double* out, int nrhs,
                                     cudaStream_t st) {
  const unsigned grid = (unsigned)((g.nbl + TC_WARPS - 1) / TC_WARPS);
  const size_t smem = (size_t)g.nI * sizeof(int);
  if (nrhs > 8)
    k_block_solve_tc<PT, 2><<<grid, TC_WARPS * 32, smem, st>>>(g, LT, rhs, out, nrhs);
  else
    k_block_solve_tc<PT, 1><<<grid, TC_WARPS * 32, smem, st>>>(g, LT, rhs, out, nrhs);
  count_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_basis_tc(const Geo& g, const double* w, double* LT, double* Sint, double* Ysc, double* Kloc,
                            int* flags, cudaStream_t st) {
  switch (tc_band(g)) {
    case 0: return launch_basis_tc_t<0>(g, w, LT, Sint, Ysc, Kloc, flags, st);
    case 1: return launch_basis_tc_t<1>(g, w, LT, Sint, Ysc, Kloc, flags, st);
    case 2: return launch_basis_tc_t<2>(g, w, LT, Sint, Ysc, Kloc, flags, st);
    case 3: return launch_basis_tc_t<3>(g, w, LT, Sint, Ysc, Kloc, flags, st);
    case 4: return launch_basis_tc_t<4>(g, w, LT, Sint, Ysc, Kloc, flags, st);
    case 5: return launch_basis_tc_t<5>(g, w, LT, Sint, Ysc, Kloc, flags, st);
    case 6: return launch_basis_tc_t<6>(g, w, LT, Sint, Ysc, Kloc, flags, st);
    case 7: return launch_basis_tc_t<7>(g, w, LT, Sint, Ysc, Kloc, flags, st);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_block_solve_tc(const Geo& g, const double* LT, const double* rhs, double* out, int nrhs,
                                  cudaStream_t st) {
  if (g.nI == 0 || nrhs == 0) return cudaSuccess;
  switch (tc_band(g)) {
    case 0: return launch_solve_tc_t<0>(g, LT, rhs, out, nrhs, st);
    case 1: return launch_solve_tc_t<1>(g, LT, rhs, out, nrhs, st);
    case 2: return launch_solve_tc_t<2>(g, LT, rhs, out, nrhs, st);
    case 3: return launch_solve_tc_t<3>(g, LT, rhs, out, nrhs, st);
    case 4: return launch_solve_tc_t<4>(g, LT, rhs, out, nrhs, st);
    case 5: return launch_solve_tc_t<5>(g, LT, rhs, out, nrhs, st);
    case 6: return launch_solve_tc_t<6>(g, LT, rhs, out, nrhs, st);
    case 7: return launch_solve_tc_t<7>(g, LT, rhs, out, nrhs, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace msfv
