// Fine-mesh kernels (SURVEY 8(f) N1 and the Gauss-Newton objective, N3):
//  * A(w) X over every pinned node for the full forward solve and block CG
//    (forward_full / block_cg, forward.py:78-98, solvers.py:57-136), node
//    fields [node][nrhs] with the pinned node 0 kept at zero;
//  * xi_e = sum_s dU_e dV_e / h_e^2 for the full-mesh sensitivity
//    (FullSensitivity.rapply, forward.py:170-175: sum_j G_j^T v_j with
//    G_j = d(A u_j)/dm = G^T diag(G u_j) C diag(sigma), operators.py:168-194),
//    gathered onto the cells by k_cell_gather (msfv_block.cu);
//  * the Tikhonov term alpha/2 ||L (m - m_ref)||^2 with L the cell-centre
//    difference operator (inversion.py:32-88): alpha L^T L v and the squared
//    face differences.
// All are HBM-bound stencil sweeps: one thread per (node or cell, lane group
// of right-hand sides), coalesced along the x-fastest index.
#include "msfv_common.cuh"
#include "msfv_kernels.h"

namespace msfv {
namespace {

inline unsigned nblk(long long n, int t) { return (unsigned)((n + t - 1) / t); }

// out(node, s) = sum over the node's edges of (w_e / h^2) (X(node) - X(nb)),
// the pinned operator row (operators.py:138-141); out(0, *) = 0.  One thread
// per (node, s): x-consecutive nodes are consecutive threads for nrhs == 1,
// and a node's nrhs values are consecutive otherwise.
__global__ void k_apply_full(Geo g, const double* __restrict__ w, const double* __restrict__ X, int nrhs,
                             double* __restrict__ out) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= g.Nn * nrhs) return;
  const long long nd = t / nrhs;
  if (nd == 0) {
    out[t] = 0.0;
    return;
  }
  int i, j, k;
  decode3f(nd, g.n1 + 1, g.r_n1p, g.n2 + 1, g.r_n2p, i, j, k);
  const double xc = X[t];
  const double c1 = g.ih1 * g.ih1, c2 = g.ih2 * g.ih2, c3 = g.ih3 * g.ih3;
  const long long sy = (long long)(g.n1 + 1) * nrhs, sz = (long long)(g.n1 + 1) * (g.n2 + 1) * nrhs;
  double v = 0.0;
  if (i > 0) v += w[ex_id(g, i - 1, j, k)] * c1 * (xc - X[t - nrhs]);
  if (i < g.n1) v += w[ex_id(g, i, j, k)] * c1 * (xc - X[t + nrhs]);
  if (j > 0) v += w[ey_id(g, i, j - 1, k)] * c2 * (xc - X[t - sy]);
  if (j < g.n2) v += w[ey_id(g, i, j, k)] * c2 * (xc - X[t + sy]);
  if (k > 0) v += w[ez_id(g, i, j, k - 1)] * c3 * (xc - X[t - sz]);
  if (k < g.n3) v += w[ez_id(g, i, j, k)] * c3 * (xc - X[t + sz]);
  out[t] = v;
}

// Edge e of the reference's edge order (x-, y-, z-edges, i fastest;
// operators.py:36-74): end nodes a < b and 1/h_e.
__device__ __forceinline__ void edge_ends(const Geo& g, long long e, long long& a, long long& b, double& ih) {
  int i, j, k;
  if (e < g.Ex) {
    decode3f(e, g.n1, g.r_n1, g.n2 + 1, g.r_n2p, i, j, k);
    a = node_id(g, i, j, k);
    b = a + 1;
    ih = g.ih1;
  } else if (e < g.Ex + g.Ey) {
    decode3f(e - g.Ex, g.n1 + 1, g.r_n1p, g.n2, g.r_n2, i, j, k);
    a = node_id(g, i, j, k);
    b = a + (g.n1 + 1);
    ih = g.ih2;
  } else {
    decode3f(e - g.Ex - g.Ey, g.n1 + 1, g.r_n1p, g.n2 + 1, g.r_n2p, i, j, k);
    a = node_id(g, i, j, k);
    b = a + (long long)(g.n1 + 1) * (g.n2 + 1);
    ih = g.ih3;
  }
}

// out(e, c) = (X(b, c) - X(a, c)) / h_e: the pinned nodal gradient G_p X of
// ncol node fields (row 0 of X is the pinned node, kept at zero).
__global__ void k_edge_grad(Geo g, const double* __restrict__ X, int ncol, double* __restrict__ out) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= g.E * ncol) return;
  const long long e = t / ncol;
  const int c = (int)(t - e * ncol);
  long long a, b;
  double ih;
  edge_ends(g, e, a, b, ih);
  out[t] = (X[b * ncol + c] - X[a * ncol + c]) * ih;
}

// out(node, c) = (G_p^T F)(node, c): +F/h for the edges ending at the node,
// -F/h for the edges starting there, axes x, y, z in order; out(0, *) = 0.
__global__ void k_edge_div(Geo g, const double* __restrict__ F, int ncol, double* __restrict__ out) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= g.Nn * ncol) return;
  const long long nd = t / ncol;
  const int c = (int)(t - nd * ncol);
  if (nd == 0) {
    out[t] = 0.0;
    return;
  }
  int i, j, k;
  decode3f(nd, g.n1 + 1, g.r_n1p, g.n2 + 1, g.r_n2p, i, j, k);
  double v = 0.0;
  if (i > 0) v += F[ex_id(g, i - 1, j, k) * ncol + c] * g.ih1;
  if (i < g.n1) v -= F[ex_id(g, i, j, k) * ncol + c] * g.ih1;
  if (j > 0) v += F[ey_id(g, i, j - 1, k) * ncol + c] * g.ih2;
  if (j < g.n2) v -= F[ey_id(g, i, j, k) * ncol + c] * g.ih2;
  if (k > 0) v += F[ez_id(g, i, j, k - 1) * ncol + c] * g.ih3;
  if (k < g.n3) v -= F[ez_id(g, i, j, k) * ncol + c] * g.ih3;
  out[t] = v;
}

// xi_e = sum_s (U_b - U_a)(V_b - V_a) / h_e^2, sources summed in order.
__global__ void k_full_xi(Geo g, const double* __restrict__ U, const double* __restrict__ V, int nrhs,
                          double* __restrict__ xi) {
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= g.E) return;
  long long a, b;
  double ih;
  int i, j, k;
  if (e < g.Ex) {
    decode3f(e, g.n1, g.r_n1, g.n2 + 1, g.r_n2p, i, j, k);
    a = node_id(g, i, j, k);
    b = a + 1;
    ih = g.ih1;
  } else if (e < g.Ex + g.Ey) {
    decode3f(e - g.Ex, g.n1 + 1, g.r_n1p, g.n2, g.r_n2, i, j, k);
    a = node_id(g, i, j, k);
    b = a + (g.n1 + 1);
    ih = g.ih2;
  } else {
    decode3f(e - g.Ex - g.Ey, g.n1 + 1, g.r_n1p, g.n2 + 1, g.r_n2p, i, j, k);
    a = node_id(g, i, j, k);
    b = a + (long long)(g.n1 + 1) * (g.n2 + 1);
    ih = g.ih3;
  }
  double acc = 0.0;
  for (int s = 0; s < nrhs; ++s)
    acc += (U[b * nrhs + s] - U[a * nrhs + s]) * (V[b * nrhs + s] - V[a * nrhs + s]);
  xi[e] = acc * (ih * ih);
}

// out_c = alpha * (L^T L v)_c in the reference's CSR order (inversion.py:84-88):
// row c of L^T L holds the z-, y-, x- neighbours, the diagonal (sum of
// (1/h)^2 over the cell's faces, x faces then y then z), then x+, y+, z+.
__global__ void k_reg_apply(Geo g, double alpha, const double* __restrict__ v, double* __restrict__ out) {
  const long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (c >= g.Nm) return;
  int i, j, k;
  decode3f(c, g.n1, g.r_n1, g.n2, g.r_n2, i, j, k);
  const double q1 = g.ih1 * g.ih1, q2 = g.ih2 * g.ih2, q3 = g.ih3 * g.ih3;
  const long long sy = g.n1, sz = (long long)g.n1 * g.n2;
  double diag = 0.0;
  if (i > 0) diag += q1;
  if (i < g.n1 - 1) diag += q1;
  if (j > 0) diag += q2;
  if (j < g.n2 - 1) diag += q2;
  if (k > 0) diag += q3;
  if (k < g.n3 - 1) diag += q3;
  double s = 0.0;
  if (k > 0) s += -q3 * v[c - sz];
  if (j > 0) s += -q2 * v[c - sy];
  if (i > 0) s += -q1 * v[c - 1];
  s += diag * v[c];
  if (i < g.n1 - 1) s += -q1 * v[c + 1];
  if (j < g.n2 - 1) s += -q2 * v[c + sy];
  if (k < g.n3 - 1) s += -q3 * v[c + sz];
  out[c] = alpha * s;
}

// out_c = sum over the faces (c, c + e_axis) of ((d_{c+e} - d_c) / h)^2, i.e.
// the rows of L d owned by cell c, squared (||L d||^2 = sum_c out_c).
__global__ void k_reg_faces(Geo g, const double* __restrict__ d, double* __restrict__ out) {
  const long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (c >= g.Nm) return;
  int i, j, k;
  decode3f(c, g.n1, g.r_n1, g.n2, g.r_n2, i, j, k);
  double s = 0.0;
  if (i < g.n1 - 1) { const double t = -g.ih1 * d[c] + g.ih1 * d[c + 1]; s += t * t; }
  if (j < g.n2 - 1) { const double t = -g.ih2 * d[c] + g.ih2 * d[c + g.n1]; s += t * t; }
  if (k < g.n3 - 1) { const double t = -g.ih3 * d[c] + g.ih3 * d[c + (long long)g.n1 * g.n2]; s += t * t; }
  out[c] = s;
}

}  // namespace

cudaError_t launch_apply_full(const Geo& g, const double* w, const double* X, int nrhs, double* out,
                              cudaStream_t st) {
  if (nrhs <= 0) return cudaSuccess;
  k_apply_full<<<nblk(g.Nn * nrhs, 256), 256, 0, st>>>(g, w, X, nrhs, out);
  count_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_full_gradient(const Geo& g, const double* sigma, const double* U, const double* V, int nrhs,
                                 double* xi, double* gout, cudaStream_t st) {
  k_full_xi<<<nblk(g.E, 256), 256, 0, st>>>(g, U, V, nrhs, xi);
  count_launches(1);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return launch_cell_gather(g, sigma, xi, gout, st);
}

cudaError_t launch_edge_grad(const Geo& g, const double* X, int ncol, double* out, cudaStream_t st) {
  if (ncol <= 0) return cudaSuccess;
  k_edge_grad<<<nblk(g.E * ncol, 256), 256, 0, st>>>(g, X, ncol, out);
  count_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_edge_div(const Geo& g, const double* F, int ncol, double* out, cudaStream_t st) {
  if (ncol <= 0) return cudaSuccess;
  k_edge_div<<<nblk(g.Nn * ncol, 256), 256, 0, st>>>(g, F, ncol, out);
  count_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_reg_apply(const Geo& g, double alpha, const double* v, double* out, cudaStream_t st) {
  k_reg_apply<<<nblk(g.Nm, 256), 256, 0, st>>>(g, alpha, v, out);
  count_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_reg_faces(const Geo& g, const double* d, double* out, cudaStream_t st) {
  k_reg_faces<<<nblk(g.Nm, 256), 256, 0, st>>>(g, d, out);
  count_launches(1);
  return cudaGetLastError();
}

}  // namespace msfv
