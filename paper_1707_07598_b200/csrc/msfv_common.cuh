// Shared geometry and index helpers for the MSFV B200 kernels.
//
// Index conventions follow the reference exactly (bit-exact patterns):
//   nodes  x-fastest, (n1+1)(n2+1)(n3+1)           mesh.py:51-54
//   cells  x-fastest, n1 n2 n3                      mesh.py:62-64
//   edges  x-edges, then y-edges, then z-edges; i fastest inside each axis
//                                                   operators.py:36-50
//   pinned space drops global node 0                operators.py:20,140
//   coarse columns = coarse nodes in global order   basis.py:95-116
//   block j = bi + nb1 (bj + nb2 bk)                mesh.py:112-118
// Device layouts (all float64, owned by the caller):
//   "full node fields"  F[node][s], node over ALL Nn nodes, F[0][*] == 0
//   interior basis      Sint[block][corner][a], a = lexicographic interior index
//   local factor        Lc[block][col][r] = L[col+r][col] (r=0: 1/L[col][col])
//                       Lr[block][row][d] = L[row][row-d] (d=0: 1/L[row][row])
//   coarse operator     tiled lower band, see coarse kernels
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace msfv {

// One skeleton-only edge of a block's owned set (model-independent, built on
// the host): local lower node, axis, which "last block along x/y/z" flags it
// needs (bits 1/2/4), whether its lower node is the block origin (the pinned
// node for block 0), and the 8 corner hats at its two nodes.
struct SkelEdge {
  int ax, x, y, z, req, origin, pad0, pad1;
  double h1[8], h0[8];
};

struct Geo {
  int n1, n2, n3;          // cells per axis
  int b1, b2, b3;          // cells per block per axis
  int nb1, nb2, nb3;       // blocks per axis
  int ni1, ni2, ni3;       // interior nodes per block per axis (b - 1)
  int nI;                  // interior nodes per block
  int p;                   // half bandwidth of A_II (ni1 * ni2)
  int P1;                  // p + 1
  int P1s;                 // P1 rounded up to even (row stride of Lc/Lr)
  int nbl;                 // number of blocks
  int kc;                  // number of coarse nodes (columns of S)
  int pc;                  // half bandwidth of A_k in coarse lexicographic order
  int TB, NT, PT;          // coarse tile size, tile rows, tile band
  int nwx, nwy, nwz;       // closed-box edge counts per block
  long long Nn, Nm, Ex, Ey, Ez, E;
  double h1, h2, h3;
  double ih1, ih2, ih3;    // 1/h per axis (as the reference's 1.0/h)
  double qv;               // 0.25 * cell volume (operators.py:83)
  double ib1, ib2, ib3;    // 1/b per axis (device-side hats)
  int coarse_nd;           // 1: z-plane nested dissection, 2: multifrontal nested dissection (msfv_coarse.cu)
  const void* mf;          // host-side multifrontal plan (coarse_nd == 2), owned by the msfv_plan
  const SkelEdge* skel;    // device table of the skeleton-only owned edges (msfv_basis_build)
  int nskel;
  int gtab8;               // 1: the 8^3 closure template (hats + edge table) is on the device (grad_template_init)
  // reduced-dimension boundary conditions (msfv_reduced.cu): per-block closed-box
  // skeleton values bx[block][corner][nbox] bound by msfv_plan_bind_boundary;
  // nullptr: the trilinear hats (basis.py:84-116)
  const double* bx;
  int nbox;                // (b1+1)(b2+1)(b3+1)
  int reduced;             // plan built for reduced boundary conditions
  // float reciprocals for division-free index decoding (see fdiv)
  float r_n1, r_n2, r_n1p, r_n2p, r_b1, r_b2, r_b3, r_ni1, r_ni2, r_nI, r_nb1, r_nb2;
};

// floor(x / d) for 0 <= x < 2^31 from a float reciprocal, corrected to exact.
__host__ __device__ __forceinline__ int fdiv(long long x, int d, float rd) {
  long long q = (long long)((float)x * rd);
  long long r = x - q * d;
  while (r < 0) { --q; r += d; }
  while (r >= d) { ++q; r -= d; }
  return (int)q;
}
// idx -> (i, j, k) for an (d1, d2, *) box, x fastest
__host__ __device__ __forceinline__ void decode3f(long long idx, int d1, float r1, int d2, float r2, int& i, int& j,
                                                  int& k) {
  const int q = fdiv(idx, d1, r1);
  i = (int)(idx - (long long)q * d1);
  k = fdiv(q, d2, r2);
  j = q - k * d2;
}

__host__ __device__ __forceinline__ long long node_id(const Geo& g, long long i, long long j, long long k) {
  return i + (long long)(g.n1 + 1) * (j + (long long)(g.n2 + 1) * k);
}
__host__ __device__ __forceinline__ long long cell_id(const Geo& g, long long i, long long j, long long k) {
  return i + (long long)g.n1 * (j + (long long)g.n2 * k);
}
__host__ __device__ __forceinline__ long long ex_id(const Geo& g, long long i, long long j, long long k) {
  return i + (long long)g.n1 * (j + (long long)(g.n2 + 1) * k);
}
__host__ __device__ __forceinline__ long long ey_id(const Geo& g, long long i, long long j, long long k) {
  return g.Ex + i + (long long)(g.n1 + 1) * (j + (long long)g.n2 * k);
}
__host__ __device__ __forceinline__ long long ez_id(const Geo& g, long long i, long long j, long long k) {
  return g.Ex + g.Ey + i + (long long)(g.n1 + 1) * (j + (long long)(g.n2 + 1) * k);
}

// Trilinear hat factor along one axis, evaluated exactly like basis.py:91:
//   max(0, 1 - |x - c| / b)   (IEEE division, no contraction).
__host__ __device__ __forceinline__ double hat1(int d, int b) {
  double a = fabs((double)d) / (double)b;
  double v = 1.0 - a;
  return v > 0.0 ? v : 0.0;
}
// Hat of local corner cc = cx + 2 cy + 4 cz at local node (x, y, z) of a block.
// Product order ((1*fx)*fy)*fz as in basis.py:89-91.
__host__ __device__ __forceinline__ double hat_corner(int cc, int x, int y, int z, int b1, int b2, int b3) {
  const int cx = (cc & 1) ? b1 : 0, cy = (cc & 2) ? b2 : 0, cz = (cc & 4) ? b3 : 0;
  double w = hat1(x - cx, b1);
  w = w * hat1(y - cy, b2);
  w = w * hat1(z - cz, b3);
  return w;
}
// Division-free device hat (1 - |d| * (1/b)); equal to hat1 whenever 1/b is
// exact (b a power of two, e.g. the 8-cell blocks of the configs) and within
// one ulp otherwise.  Used only inside device arithmetic; the skeleton values
// of the returned CSC S come from the host (bit-exact with the reference).
__device__ __forceinline__ double hatf1(int d, double ib) {
  double v = 1.0 - fabs((double)d) * ib;
  return v > 0.0 ? v : 0.0;
}
__device__ __forceinline__ double hatf(const Geo& g, int cc, int x, int y, int z) {
  const int cx = (cc & 1) ? g.b1 : 0, cy = (cc & 2) ? g.b2 : 0, cz = (cc & 4) ? g.b3 : 0;
  double w = hatf1(x - cx, g.ib1);
  w = w * hatf1(y - cy, g.ib2);
  w = w * hatf1(z - cz, g.ib3);
  return w;
}

// Owner block of a node / edge for sums that must count each item once:
// coordinate X belongs to block min(X / b, nb - 1) along each axis.
__host__ __device__ __forceinline__ int own1(long long X, int b, int nb) {
  long long q = X / b;
  return (int)(q < nb - 1 ? q : nb - 1);
}

// 32-bit decode of a linear index (all index spaces here are < 2^31; 64-bit
// division is a long instruction sequence on the GPU).
__host__ __device__ __forceinline__ void decode3(long long idx, int d1, int d2, int& i, int& j, int& k) {
  const unsigned u = (unsigned)idx;
  const unsigned q = u / (unsigned)d1;
  i = (int)(u - q * (unsigned)d1);
  const unsigned q2 = q / (unsigned)d2;
  j = (int)(q - q2 * (unsigned)d2);
  k = (int)q2;
}
__host__ __device__ __forceinline__ int own1i(int X, int b, int nb) {
  const int q = (int)((unsigned)X / (unsigned)b);
  return q < nb - 1 ? q : nb - 1;
}

__host__ __device__ __forceinline__ int block_of(const Geo& g, int bi, int bj, int bk) {
  return bi + g.nb1 * (bj + g.nb2 * bk);
}
__host__ __device__ __forceinline__ int coarse_of(const Geo& g, int ci, int cj, int ck) {
  return ci + (g.nb1 + 1) * (cj + (g.nb2 + 1) * ck);
}
// Coarse column of local corner cc of block (bi,bj,bk).
__host__ __device__ __forceinline__ int corner_col(const Geo& g, int bi, int bj, int bk, int cc) {
  return coarse_of(g, bi + (cc & 1), bj + ((cc >> 1) & 1), bk + ((cc >> 2) & 1));
}

// Local interior index of local node (x, y, z) or -1 when on the block boundary.
__host__ __device__ __forceinline__ int interior_index(const Geo& g, int x, int y, int z) {
  if (x <= 0 || x >= g.b1 || y <= 0 || y >= g.b2 || z <= 0 || z >= g.b3) return -1;
  return (x - 1) + g.ni1 * ((y - 1) + g.ni2 * (z - 1));
}

// Skeleton value of corner cc at local node (x, y, z) of block jb: the bound
// reduced-boundary table, or the model-independent hat.
__device__ __forceinline__ double skel_value(const Geo& g, int jb, int cc, int x, int y, int z) {
  if (g.bx) return g.bx[((size_t)jb * 8 + cc) * g.nbox + x + (g.b1 + 1) * (y + (g.b2 + 1) * z)];
  return hatf(g, cc, x, y, z);
}
// Basis value S(node, corner cc) of a node given in local coordinates of block
// jb.  Interior values come from the per-block solve, skeleton values are the
// hats (or the bound reduced-boundary values), and the pinned global node 0
// has no row (value 0).
__device__ __forceinline__ double s_value(const Geo& g, const double* __restrict__ Sint_b, int jb,
                                          int cc, int x, int y, int z, bool is_node0) {
  int a = interior_index(g, x, y, z);
  if (a >= 0) return Sint_b[(size_t)cc * g.nI + a];
  if (is_node0) return 0.0;
  return skel_value(g, jb, cc, x, y, z);
}

}  // namespace msfv
