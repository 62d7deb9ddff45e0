// FP64 tensor-core (DMMA, mma.sync m8n8k4 f64) throughput microbenchmark on sm_100a
// (development aid: decides whether the trilinear / high-p contractions go to DMMA).
// Every warp runs 8 independent accumulator chains of m8n8k4 (256 FMA each).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
__global__ void dmma_kernel(double* out, int iters, double a, double b) {
  double c[8][2];
  for (int k = 0; k < 8; ++k) c[k][0] = c[k][1] = threadIdx.x * 1e-9 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) dmma(c[k][0], c[k][1], a, b);
  }
  double s = 0;
  for (int k = 0; k < 8; ++k) s += c[k][0] + c[k][1];
  if (s == 1234.5) out[threadIdx.x] = s;
}
int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 1024 * sizeof(double));
  const int iters = 1 << 14;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int threads : {128, 256, 512}) {
    const int blocks = sms * (1024 / threads);
    dmma_kernel<<<blocks, threads>>>(out, 64, 1e-6, 1e-7);
    double best = 0;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0);
      dmma_kernel<<<blocks, threads>>>(out, iters, 1e-6, 1e-7);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      const double flops = 2.0 * 256 * 8 * (double)iters * (threads / 32) * blocks;
      const double tf = flops / (ms * 1e-3) / 1e12;
      if (tf > best) best = tf;
    }
    printf("{\"dmma_f64_tflops\": %.3f, \"threads\": %d, \"sms\": %d, \"err\": \"%s\"}\n", best, threads,
           sms, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
