// FP64 tensor-core (DMMA, mma.sync.m8n8k4.f64) tile helpers shared by the
// per-block local solvers (msfv_tc.cu: register-window band for half
// bandwidths <= 56; msfv_large.cu: L2-resident band for larger blocks).
//
// Tiles are 8x8 row-major (64 doubles).  The accumulator (C) layout of a
// stored tile is the pair at lane*2 (element (m, n) at lane 4m + n/2, slot n%2).
// With BOTH operands in C layout, mma(D, X, Y) computes D += X Y^T (chunk h of
// the k dimension is the column set {2k + h}, slot h of the layout), so the
// Cholesky panel/trailing products and the transposed substitutions need no
// register shuffles; ld_t gives the C layout of a stored tile's transpose.
#pragma once

namespace msfv {
namespace dmma {

struct F2 {
  double x, y;
};

__device__ __forceinline__ void mma884(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}
// D += X Y^T for C-layout tiles X, Y (k = 8)
__device__ __forceinline__ void mma(F2& c, const F2& a, const F2& b) {
  mma884(c.x, c.y, a.x, b.x);
  mma884(c.x, c.y, a.y, b.y);
}
__device__ __forceinline__ F2 neg(const F2& f) { return {-f.x, -f.y}; }

__device__ __forceinline__ F2 ld2(const double* p) {
  double2 v = *reinterpret_cast<const double2*>(p);
  return {v.x, v.y};
}
__device__ __forceinline__ void st2(double* p, const F2& f) {
  *reinterpret_cast<double2*>(p) = make_double2(f.x, f.y);
}
// L2-coherent forms (data written earlier by other warps of the same kernel)
__device__ __forceinline__ F2 ld2cg(const double* p) {
  double2 v = __ldcg(reinterpret_cast<const double2*>(p));
  return {v.x, v.y};
}
__device__ __forceinline__ void st2cg(double* p, const F2& f) {
  __stcg(reinterpret_cast<double2*>(p), make_double2(f.x, f.y));
}
// C layout of the transpose of the row-major tile at p
__device__ __forceinline__ F2 ld_t(const double* p, int lane) {
  const int m = lane >> 2, q = lane & 3;
  return {__ldcg(p + 16 * q + m), __ldcg(p + 16 * q + 8 + m)};
}

}  // namespace dmma
}  // namespace msfv
