// DMMA (mma.sync.m8n8k4.f64) throughput vs warps per SM and independent
// accumulator chains per warp (development probe).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
template <int C>
__global__ void k(double* out, int iters) {
  const int lane = threadIdx.x & 31;
  const double a = 1.0 + lane * 1e-9, b = 1e-9;
  double d[C][2];
#pragma unroll
  for (int q = 0; q < C; ++q) d[q][0] = d[q][1] = q;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int q = 0; q < C; ++q) dmma(d[q][0], d[q][1], a, b);
  }
  double s = 0;
#pragma unroll
  for (int q = 0; q < C; ++q) s += d[q][0] + d[q][1];
  if (s == 1234.5) out[0] = s;
}
template <int C>
void run(int wps, int sms) {
  double* o; cudaMalloc(&o, 8);
  const int iters = 4096;
  // one CTA per SM with wps warps
  k<C><<<sms, 32 * wps>>>(o, 64);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<C><<<sms, 32 * wps>>>(o, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double flops = 2.0 * 256 * C * (double)iters * wps * sms;
  printf("warps/SM %2d chains %d : %7.2f TF/s\n", wps, C, flops / ms / 1e9);
  cudaFree(o);
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int w : {4, 8, 12, 16, 24, 32}) { run<1>(w, sms); run<2>(w, sms); run<4>(w, sms); run<8>(w, sms); }
  return 0;
}
