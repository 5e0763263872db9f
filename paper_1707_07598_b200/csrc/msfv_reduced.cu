// Reduced-dimension boundary conditions for the multiscale basis (SURVEY 8(f)
// N4; BASELINE.json north_star: "reduced 1D tangential-flux boundary problems
// on dual-block edges and faces").  The reference evaluates trilinear hats on
// the skeleton instead (generate_bc_lagrange, basis.py:84-116; SPEC.md:328
// "no reduced-dimension edge problems"), so this is a flagged extension with
// its own CPU oracle (oracle/msfv_reduced.py):
//   lines  (1D): u = normalized cumulative resistance sum(1/w_e) along each
//          segment between adjacent coarse nodes;
//   faces  (2D): the 5-point problem of each face patch's in-plane edges
//          (w_e / h_e^2) with the line values as Dirichlet data, 4 corners;
//   boxes      : every block's closed-box skeleton values of its 8 corners,
//          bx[block][corner][(b1+1)(b2+1)(b3+1)] (interior entries 0), which
//          the basis kernels read instead of the hats (Geo::bx).
// One warp per face patch: lines in lanes 0..3, the banded Cholesky of the
// patch (half bandwidth bu - 1) with lane-parallel column updates in shared
// memory, 4 right-hand sides.  Latency-bound (13 056 patches at config 4).
#include <algorithm>
#include "msfv_common.cuh"
#include "msfv_kernels.h"

namespace msfv {
namespace {

constexpr int RF_WARPS = 4;

__host__ __device__ inline int face_count(const Geo& g, int ax) {
  return ax == 0 ? (g.nb1 + 1) * g.nb2 * g.nb3 : (ax == 1 ? g.nb1 * (g.nb2 + 1) * g.nb3 : g.nb1 * g.nb2 * (g.nb3 + 1));
}
__host__ __device__ inline int bsize(const Geo& g, int a) { return a == 0 ? g.b1 : (a == 1 ? g.b2 : g.b3); }
__device__ inline double hsq_inv(const Geo& g, int a) {
  return a == 0 ? g.ih1 * g.ih1 : (a == 1 ? g.ih2 * g.ih2 : g.ih3 * g.ih3);
}
__device__ inline long long edge_id(const Geo& g, int ax, long long i, long long j, long long k) {
  return ax == 0 ? ex_id(g, i, j, k) : (ax == 1 ? ey_id(g, i, j, k) : ez_id(g, i, j, k));
}
// face f of orientation ax -> patch coordinates (position along ax, block
// indices along ua, va) and its base node
__device__ inline void face_decode(const Geo& g, int ax, int f, int p[3]) {
  const int n0 = ax == 0 ? g.nb1 + 1 : g.nb1, n1 = ax == 1 ? g.nb2 + 1 : g.nb2;
  p[0] = f % n0;
  p[1] = (f / n0) % n1;
  p[2] = f / (n0 * n1);
}
__host__ __device__ inline size_t face_stride(const Geo& g) {
  const int m = std::max(g.b1, std::max(g.b2, g.b3)) + 1;
  return (size_t)4 * m * m;
}

// Face values: fv[face][c4][(bu+1)(bv+1)], c4 = du + 2 dv (corner offsets along ua, va).
__global__ void __launch_bounds__(RF_WARPS * 32)
k_red_faces(Geo g, const double* __restrict__ w, double* __restrict__ fv, int* __restrict__ flags, int smem_w) {
  extern __shared__ double rsm[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  long long gf = (long long)blockIdx.x * RF_WARPS + wid;
  int ax = 0;
  while (ax < 3 && gf >= face_count(g, ax)) gf -= face_count(g, ax++);
  if (ax >= 3) return;
  const int f = (int)gf;
  const int ua = ax == 0 ? 1 : 0, va = ax == 2 ? 1 : 2;
  const int bu = bsize(g, ua), bv = bsize(g, va);
  const int NU = bu + 1, NG = (bu + 1) * (bv + 1);
  int pc[3];
  face_decode(g, ax, f, pc);
  int base[3];
  for (int a = 0; a < 3; ++a) base[a] = pc[a] * bsize(g, a);
  double* grid = rsm + (size_t)wid * smem_w;      // [4][NG]
  const int nu = bu - 1, nv = bv - 1, n2 = nu * nv, P = nu;   // interior unknowns, half bandwidth
  double* Cb = grid + 4 * NG;                      // [n2][P + 1] column band
  double* X = Cb + (size_t)n2 * (P + 1);           // [n2][4]
  double* invd = X + (size_t)n2 * 4;               // [n2]
  for (int i = lane; i < 4 * NG; i += 32) grid[i] = 0.0;
  __syncwarp();
  // corners and the four perimeter lines (lane l: line l)
  if (lane < 4) grid[lane * NG + (lane & 1) * bu + NU * ((lane >> 1) * bv)] = 1.0;
  if (lane < 4) {
    const bool along_u = lane < 2;                 // lines along ua at v = 0 (lane 0) / v = bv (lane 1)
    const int side = lane & 1;
    const int L = along_u ? bu : bv, lax = along_u ? ua : va;
    double R = 0.0;
    for (int s = 0; s < L; ++s) {
      int q[3] = {base[0], base[1], base[2]};
      if (along_u) { q[ua] += s; q[va] += side * bv; }
      else { q[va] += s; q[ua] += side * bu; }
      R += 1.0 / w[edge_id(g, lax, q[0], q[1], q[2])];
    }
    double acc = 0.0;                              // sum of r_s for s < t
    for (int t = 1; t < L; ++t) {
      int q[3] = {base[0], base[1], base[2]};
      if (along_u) { q[ua] += t - 1; q[va] += side * bv; }
      else { q[va] += t - 1; q[ua] += side * bu; }
      acc += 1.0 / w[edge_id(g, lax, q[0], q[1], q[2])];
      const double hi = acc / R;                   // upper end's value
      double suf = 0.0;                            // sum of r_s for s >= t (lower end), same order as the oracle
      for (int s = t; s < L; ++s) {
        int r3[3] = {base[0], base[1], base[2]};
        if (along_u) { r3[ua] += s; r3[va] += side * bv; }
        else { r3[va] += s; r3[ua] += side * bu; }
        suf += 1.0 / w[edge_id(g, lax, r3[0], r3[1], r3[2])];
      }
      const double lo = suf / R;
      int u, v, clo, chi;
      if (along_u) { u = t; v = side * bv; clo = 2 * side; chi = 2 * side + 1; }
      else { u = side * bu; v = t; clo = side; chi = side + 2; }
      grid[clo * NG + u + NU * v] = lo;
      grid[chi * NG + u + NU * v] = hi;
    }
  }
  __syncwarp();
  if (n2 > 0) {
    // band + right-hand sides of the patch problem
    const double cu = hsq_inv(g, ua), cv = hsq_inv(g, va);
    for (int a = lane; a < n2; a += 32) {
      const int u = 1 + a % nu, v = 1 + a / nu;
      int q[3] = {base[0], base[1], base[2]};
      q[ua] += u; q[va] += v;
      int qm[3] = {q[0], q[1], q[2]}, qn[3] = {q[0], q[1], q[2]};
      qm[ua] -= 1; qn[va] -= 1;
      const double kum = w[edge_id(g, ua, qm[0], qm[1], qm[2])] * cu, kup = w[edge_id(g, ua, q[0], q[1], q[2])] * cu;
      const double kvm = w[edge_id(g, va, qn[0], qn[1], qn[2])] * cv, kvp = w[edge_id(g, va, q[0], q[1], q[2])] * cv;
      double* col = Cb + (size_t)a * (P + 1);
      for (int r = 0; r <= P; ++r) col[r] = 0.0;
      col[0] = ((kum + kup) + kvm) + kvp;
      if (u < nu) col[1] = -kup;
      if (v < nv) col[P] = -kvp;
      for (int c = 0; c < 4; ++c) {
        double r = 0.0;
        if (u == 1) r += kum * grid[c * NG + 0 + NU * v];
        if (u == nu) r += kup * grid[c * NG + bu + NU * v];
        if (v == 1) r += kvm * grid[c * NG + u + 0];
        if (v == nv) r += kvp * grid[c * NG + u + NU * bv];
        X[a * 4 + c] = r;
      }
    }
    __syncwarp();
    for (int j = 0; j < n2; ++j) {
      double* col = Cb + (size_t)j * (P + 1);
      const int rmax = min(P, n2 - 1 - j);
      if (lane == 0) {
        double d = col[0];
        if (!(d > 0.0)) {
          atomicOr(flags, FLAG_LOCAL_NOT_SPD);
          d = 1.0;
        }
        col[0] = sqrt(d);
        invd[j] = 1.0 / col[0];
      }
      __syncwarp();
      for (int r = 1 + lane; r <= rmax; r += 32) col[r] *= invd[j];
      __syncwarp();
      const int nup = rmax * (rmax + 1) / 2;
      for (int t = lane; t < nup; t += 32) {
        int r = (int)((1.0 + sqrt(1.0 + 8.0 * t)) * 0.5);
        while (r * (r - 1) / 2 > t) --r;
        while ((r + 1) * r / 2 <= t) ++r;
        const int qd = t - r * (r - 1) / 2 + 1;
        Cb[(size_t)(j + qd) * (P + 1) + (r - qd)] -= col[r] * col[qd];
      }
      __syncwarp();
    }
    // L y = rhs, then L^T x = y (4 right-hand sides)
    for (int i = 0; i < n2; ++i) {
      const int rmax = min(P, n2 - 1 - i);
      const double* col = Cb + (size_t)i * (P + 1);
      if (lane < 4) X[i * 4 + lane] *= invd[i];
      __syncwarp();
      for (int t = lane; t < rmax * 4; t += 32) {
        const int r = 1 + t / 4, c = t & 3;
        X[(i + r) * 4 + c] -= col[r] * X[i * 4 + c];
      }
      __syncwarp();
    }
    for (int i = n2 - 1; i >= 0; --i) {
      if (lane < 4) X[i * 4 + lane] *= invd[i];
      __syncwarp();
      const int dmax = min(P, i);
      for (int t = lane; t < dmax * 4; t += 32) {
        const int d = 1 + t / 4, c = t & 3;
        X[(i - d) * 4 + c] -= Cb[(size_t)(i - d) * (P + 1) + d] * X[i * 4 + c];
      }
      __syncwarp();
    }
    for (int t = lane; t < n2 * 4; t += 32) {
      const int a = t >> 2, c = t & 3;
      grid[c * NG + (1 + a % nu) + NU * (1 + a / nu)] = X[t];
    }
    __syncwarp();
  }
  double* out = fv + ((size_t)f + (ax > 0 ? face_count(g, 0) : 0) + (ax > 1 ? face_count(g, 1) : 0)) * face_stride(g);
  for (int i = lane; i < 4 * NG; i += 32) out[i] = grid[i];
}

// bx[block][cc][box node]: skeleton values of the block's 8 corners on its
// closed box from the face patches (interior entries 0; the pinned node 0).
__global__ void k_red_box(Geo g, const double* __restrict__ fv, double* __restrict__ bx) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= (long long)g.nbl * 8 * g.nbox) return;
  const int n = (int)(t % g.nbox);
  const int cc = (int)((t / g.nbox) & 7);
  const int jb = (int)(t / (8LL * g.nbox));
  const int B1 = g.b1 + 1, B2 = g.b2 + 1;
  const int l[3] = {n % B1, (n / B1) % B2, n / (B1 * B2)};
  const int bi = jb % g.nb1, bj = (jb / g.nb1) % g.nb2, bk = jb / (g.nb1 * g.nb2);
  const int blk[3] = {bi, bj, bk};
  double v = 0.0;
  int ax = -1;
  for (int a = 0; a < 3 && ax < 0; ++a)
    if (l[a] == 0 || l[a] == bsize(g, a)) ax = a;
  if (ax >= 0 && !(jb == 0 && n == 0)) {
    const int side = l[ax] == 0 ? 0 : 1;
    const int cbit[3] = {cc & 1, (cc >> 1) & 1, (cc >> 2) & 1};
    if (cbit[ax] == side) {
      const int ua = ax == 0 ? 1 : 0, va = ax == 2 ? 1 : 2;
      int pc[3] = {blk[0], blk[1], blk[2]};
      pc[ax] += side;
      const int n0 = ax == 0 ? g.nb1 + 1 : g.nb1, n1 = ax == 1 ? g.nb2 + 1 : g.nb2;
      const long long f = pc[0] + (long long)n0 * (pc[1] + (long long)n1 * pc[2]) +
                          (ax > 0 ? face_count(g, 0) : 0) + (ax > 1 ? face_count(g, 1) : 0);
      const int NU = bsize(g, ua) + 1, NG = NU * (bsize(g, va) + 1);
      const int c4 = cbit[ua] + 2 * cbit[va];
      v = fv[f * face_stride(g) + (size_t)c4 * NG + l[ua] + NU * l[va]];
    }
  }
  bx[t] = v;
}

__global__ void k_basis_csc_box(long long nnz, const double* __restrict__ Sint, const long long* __restrict__ src,
                                const long long* __restrict__ bsrc, const double* __restrict__ bx,
                                double* __restrict__ vals) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= nnz) return;
  vals[t] = src[t] >= 0 ? Sint[src[t]] : bx[bsrc[t]];
}

}  // namespace

size_t red_face_doubles(const Geo& g) {
  return (size_t)(face_count(g, 0) + face_count(g, 1) + face_count(g, 2)) * face_stride(g);
}
size_t red_box_doubles(const Geo& g) { return (size_t)g.nbl * 8 * g.nbox; }

cudaError_t launch_reduced_boundary(const Geo& g, const double* w, double* fv, double* bx, int* flags,
                                    cudaStream_t st) {
  const int bmax = std::max(g.b1, std::max(g.b2, g.b3));
  const int n2max = (bmax - 1) * (bmax - 1), Pmax = bmax - 1;
  const int smem_w = 4 * (bmax + 1) * (bmax + 1) + n2max * (Pmax + 1) + n2max * 4 + n2max + 2;
  const size_t smem = (size_t)RF_WARPS * smem_w * sizeof(double);
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(k_red_faces, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const long long nf = (long long)face_count(g, 0) + face_count(g, 1) + face_count(g, 2);
  k_red_faces<<<(unsigned)((nf + RF_WARPS - 1) / RF_WARPS), RF_WARPS * 32, smem, st>>>(g, w, fv, flags, smem_w);
  count_launches(1);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  const long long nb = (long long)g.nbl * 8 * g.nbox;
  k_red_box<<<(unsigned)((nb + 255) / 256), 256, 0, st>>>(g, fv, bx);
  count_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_basis_csc_box(long long nnz, const double* Sint, const long long* src, const long long* bsrc,
                                 const double* bx, double* vals, cudaStream_t st) {
  if (nnz == 0) return cudaSuccess;
  k_basis_csc_box<<<(unsigned)((nnz + 255) / 256), 256, 0, st>>>(nnz, Sint, src, bsrc, bx, vals);
  count_launches(1);
  return cudaGetLastError();
}

}  // namespace msfv
