// Checks the m8n8k4 f64 fragment layout assumed by the DMMA trilinear kernel:
//   A: a = A[lane >> 2][lane & 3]; B: b = B[lane & 3][lane >> 2];
//   C/D: d[h] = C[lane >> 2][2 (lane & 3) + h]
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(const double* A, const double* B, double* D) {
  const int l = threadIdx.x;
  double a = A[(l >> 2) * 4 + (l & 3)];
  double b = B[(l & 3) * 8 + (l >> 2)];
  double d0 = 0.0, d1 = 0.0;
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
  D[(l >> 2) * 8 + 2 * (l & 3)] = d0;
  D[(l >> 2) * 8 + 2 * (l & 3) + 1] = d1;
}
int main() {
  double hA[32], hB[32], hD[64], ref[64];
  for (int i = 0; i < 32; ++i) { hA[i] = 1.0 + i * 0.37; hB[i] = 2.0 - i * 0.11; }
  for (int r = 0; r < 8; ++r)
    for (int c = 0; c < 8; ++c) {
      double s = 0;
      for (int kk = 0; kk < 4; ++kk) s += hA[r * 4 + kk] * hB[kk * 8 + c];
      ref[r * 8 + c] = s;
    }
  double *A, *B, *D;
  cudaMalloc(&A, 256); cudaMalloc(&B, 256); cudaMalloc(&D, 512);
  cudaMemcpy(A, hA, 256, cudaMemcpyHostToDevice);
  cudaMemcpy(B, hB, 256, cudaMemcpyHostToDevice);
  k<<<1, 32>>>(A, B, D);
  cudaMemcpy(hD, D, 512, cudaMemcpyDeviceToHost);
  double err = 0;
  for (int i = 0; i < 64; ++i) err = fmax(err, fabs(hD[i] - ref[i]));
  printf("{\"dmma_layout_max_err\": %.3e, \"ok\": %s, \"err\": \"%s\"}\n", err, err < 1e-12 ? "true" : "false",
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
