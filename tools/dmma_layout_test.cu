// Verifies the m8n8k4 f64 fragment layouts assumed by msfv_tc.cu:
//  A[m][k] at lane 4m+k ; B[k][n] at lane 4n+k ; C[m][n] at lane 4m+n/2, slot n%2
#include <cstdio>
__global__ void k(double* out) {
  int L = threadIdx.x;
  double a = 0, b = 0, c0 = 0, c1 = 0;
  // A = ones at (m,k): A[m][k] = m*10+k ; B[k][n] = (k==n%4) ? 1 : 0 ... use general values
  int m = L >> 2, kk = L & 3;
  a = m * 10.0 + kk;          // A[m][k]
  int n = L >> 2, kb = L & 3;
  b = (kb == (n & 3)) ? (n >= 4 ? 2.0 : 1.0) : 0.0;   // B[k][n]
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n" : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
  out[L * 2] = c0; out[L * 2 + 1] = c1;
}
int main() {
  double* d; cudaMalloc(&d, 64 * 8); k<<<1, 32>>>(d); double h[64]; cudaMemcpy(h, d, 512, cudaMemcpyDeviceToHost);
  // expected C[m][n] = sum_k A[m][k] B[k][n] = A[m][n%4] * (n>=4?2:1)
  int bad = 0;
  for (int L = 0; L < 32; ++L) for (int v = 0; v < 2; ++v) {
    int m = L >> 2, n = 2 * (L & 3) + v;
    double e = (m * 10.0 + (n & 3)) * (n >= 4 ? 2.0 : 1.0);
    if (h[L * 2 + v] != e) { bad++; printf("L%d v%d got %g exp %g\n", L, v, h[L*2+v], e); }
  }
  printf("dmma layout %s\n", bad ? "MISMATCH" : "OK");
  return 0;
}
