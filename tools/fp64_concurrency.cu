// Do DMMA (FP64 tensor) and DFMA (FP64 vector) share throughput?  Half the warps of every CTA run
// back-to-back DMMAs, the other half back-to-back DFMAs; compare against each alone.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n" : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
__global__ void mixed(double* out, int iters, int mode) {   // mode 0: dmma only, 1: dfma only, 2: half/half
  const int warp = threadIdx.x >> 5;
  const bool do_mma = mode == 0 || (mode == 2 && (warp & 1) == 0);
  double s = 0;
  if (do_mma) {
    double c[8][2];
    for (int q = 0; q < 8; ++q) { c[q][0] = q; c[q][1] = threadIdx.x; }
    double a = threadIdx.x * 1e-3, b = 1.0;
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int q = 0; q < 8; ++q) dmma(c[q][0], c[q][1], a, b);
    for (int q = 0; q < 8; ++q) s += c[q][0] + c[q][1];
  } else {
    double acc[16];
    for (int q = 0; q < 16; ++q) acc[q] = q + threadIdx.x;
    for (int it = 0; it < iters * 4; ++it)
#pragma unroll
      for (int q = 0; q < 16; ++q) acc[q] = fma(acc[q], 1.0000001, 1e-7);
    for (int q = 0; q < 16; ++q) s += acc[q];
  }
  if (s == 1.2345) out[0] = s;
}
int main() {
  double* d; cudaMalloc(&d, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 2000, threads = 512, grid = sms * 2;
  for (int mode = 0; mode < 3; ++mode) {
    mixed<<<grid, threads>>>(d, 10, mode); cudaDeviceSynchronize();
    cudaEventRecord(e0); mixed<<<grid, threads>>>(d, iters, mode); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    // flops: dmma warp: 8*iters MMAs * 512 flop; dfma warp: 16*4*iters * 2 flop * 32 lanes
    const double wp = (double)grid * threads / 32;
    const double fm = 8.0 * iters * 512, ff = 16.0 * 4 * iters * 2 * 32;
    double flops = mode == 0 ? wp * fm : mode == 1 ? wp * ff : wp / 2 * (fm + ff);
    printf("mode %d (%s): %.3f ms  %.2f TFLOP/s\n", mode, mode == 0 ? "dmma" : mode == 1 ? "dfma" : "half/half", ms, flops / ms / 1e9);
  }
  return 0;
}
