// Do DMMA (mma.sync.m8n8k4.f64) and DFMA share one pipe on sm_100a?
// Warps of a CTA run either DMMA chains or DFMA chains; the aggregate rate
// of a mixed CTA against the pure ones answers it (development probe).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
// warps [0, wm) run DMMA, warps [wm, wm + wf) run DFMA
__global__ void k(double* out, int iters, int wm) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const double a = 1.0 + lane * 1e-9, b = 1e-9;
  double d[8][2];
#pragma unroll
  for (int q = 0; q < 8; ++q) d[q][0] = d[q][1] = q;
  if (w < wm) {
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int q = 0; q < 8; ++q) dmma(d[q][0], d[q][1], a, b);
    }
  } else {
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        d[q][0] = fma(d[q][0], a, b);
        d[q][1] = fma(d[q][1], a, b);
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) s += d[q][0] + d[q][1];
  if (s == 1234.5) out[0] = s;
}
void run(int wm, int wf, int sms) {
  double* o; cudaMalloc(&o, 8);
  const int iters = 8192;
  k<<<sms, 32 * (wm + wf)>>>(o, 64, wm);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<<<sms, 32 * (wm + wf)>>>(o, iters, wm);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  // per warp per iteration: DMMA 8 x 512 flops, DFMA 16 x 64 flops
  const double fm = 8.0 * 512 * iters * wm * sms, ff = 16.0 * 64 * iters * wf * sms;
  printf("dmma warps %2d dfma warps %2d : %8.3f ms  dmma %6.2f TF/s  dfma %6.2f TF/s  sum %6.2f\n",
         wm, wf, ms, fm / ms / 1e9, ff / ms / 1e9, (fm + ff) / ms / 1e9);
  cudaFree(o);
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run(16, 0, sms); run(0, 16, sms); run(0, 32, sms);
  // the DFMA warps do 1/4 of the flops per iteration: in a shared pipe the
  // mixed time is the sum of the parts, in separate pipes the max
  run(16, 16, sms); run(8, 32, sms); run(4, 16, sms); run(8, 8, sms); run(16, 32, sms);
  return 0;
}
