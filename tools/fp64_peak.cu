// Microbenchmark: sustained FP64 DFMA and DMMA (mma.sync m8n8k4 f64) throughput on sm_100a,
// plus random-index LDS.128 throughput on a p-entry complex128 table in shared memory
// (the twiddle-table access pattern of the exp-sum kernel). Used to fix the FP64 roofline
// denominator that MEASURED_PEAKS.json does not provide.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)

template<int CH>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double acc[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) acc[c] = threadIdx.x * 1e-9 + c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += acc[c];
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[8][2];
#pragma unroll
  for (int q = 0; q < 8; ++q) { c[q][0] = q; c[q][1] = -q; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[q][0]), "+d"(c[q][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) s += c[q][0] + c[q][1];
  if (s == 12345.678) out[0] = s;
}

// random-index 16B smem gathers: idx_{t+1} = (idx_t + u) mod p, lanes start at (lane*u) mod p
__global__ void lds_kernel(double* out, int iters, int p, int u) {
  extern __shared__ double2 tab[];
  for (int i = threadIdx.x; i < p; i += blockDim.x) tab[i] = make_double2(i, -i);
  __syncthreads();
  int idx = (int)(((long long)(threadIdx.x + blockIdx.x) * u) % p);
  double sx = 0, sy = 0;
  for (int it = 0; it < iters; ++it) {
    double2 v = tab[idx];
    sx += v.x; sy += v.y;
    idx += u; if (idx >= p) idx -= p;
  }
  if (sx + sy == 12345.678) out[0] = sx;
}

int main() {
  double* d; CK(cudaMalloc(&d, 8));
  cudaDeviceProp pr; CK(cudaGetDeviceProperties(&pr, 0));
  int sms = pr.multiProcessorCount;
  printf("device %s sms %d clock(kHz) %d\n", pr.name, sms, pr.clockRate);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int blocksPerSm : {2, 4, 8}) {
    int threads = 256, iters = 20000, grid = sms * blocksPerSm;
    dfma_kernel<16><<<grid, threads>>>(d, 100, 1.0000001, 1e-7);
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0); dfma_kernel<16><<<grid, threads>>>(d, iters, 1.0000001, 1e-7); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    double flops = 2.0 * 16 * (double)iters * threads * grid;
    printf("DFMA blocks/SM %d: %.3f ms  %.2f TFLOP/s\n", blocksPerSm, best, flops / best / 1e9);
  }
  // sustained: 3 s loop
  {
    int threads = 256, iters = 20000, grid = sms * 4;
    cudaEventRecord(e0); int n = 0;
    for (; n < 60; ++n) dfma_kernel<16><<<grid, threads>>>(d, iters, 1.0000001, 1e-7);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 16 * (double)iters * threads * grid * n;
    printf("DFMA sustained (%d launches, %.1f ms): %.2f TFLOP/s\n", n, ms, flops / ms / 1e9);
  }
  for (int blocksPerSm : {2, 4, 8}) {
    int threads = 256, iters = 4000, grid = sms * blocksPerSm;
    dmma_kernel<<<grid, threads>>>(d, 10); CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0); dmma_kernel<<<grid, threads>>>(d, iters); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    double flops = 2.0 * 8 * 8 * 4 * 8 * (double)iters * (threads / 32) * grid;
    printf("DMMA m8n8k4 blocks/SM %d: %.3f ms  %.2f TFLOP/s\n", blocksPerSm, best, flops / best / 1e9);
  }
  for (int u : {1, 7, 1234, 2501, 3777}) {
    int p = 5003, threads = 512, iters = 20000, grid = sms * 2;
    size_t sm = (size_t)p * 16;
    CK(cudaFuncSetAttribute(lds_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    lds_kernel<<<grid, threads, sm>>>(d, 10, p, u); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); lds_kernel<<<grid, threads, sm>>>(d, iters, p, u); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1);
    double warpLds = (double)iters * (threads / 32) * grid;
    double clk = pr.clockRate * 1e3;  // nominal
    printf("LDS.128 random p=%d u=%d: %.3f ms, %.2f warp-LDS/us/SM, ~%.2f cyc/warp-LDS at %.0f MHz\n", p, u, ms,
           warpLds / sms / (ms * 1e3), (ms * 1e-3 * clk) / (warpLds / sms), clk / 1e6);
  }
  return 0;
}
