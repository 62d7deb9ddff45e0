// FP64 FMA throughput microbenchmark (development aid; the roofline denominator for the
// FP64-ALU-bound trilinear kernel): every thread runs 8 independent DFMA chains.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x[8];
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-9 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
  }
  double s = 0;
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 1234.5) out[threadIdx.x] = s;   // keep the chains alive
}
int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 1024 * sizeof(double));
  const int iters = 1 << 16, threads = 512, blocks = sms * 4;
  dfma_kernel<<<blocks, threads>>>(out, 1024, 0.999999, 1e-7);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  double best = 0;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    dfma_kernel<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double tf = 2.0 * 8 * iters * (double)threads * blocks / (ms * 1e-3) / 1e12;
    if (tf > best) best = tf;
  }
  printf("{\"fp64_fma_tflops\": %.3f, \"sms\": %d}\n", best, sms);
  return 0;
}
