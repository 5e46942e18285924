// Microbenchmark: DMMA (mma.sync m8n8k4 f64) throughput for the exp-sum's complex MMA pattern:
// per k-step MB x NB complex blocks, 4 real MMAs each (Ar Br, Ar Bi, Ai (-Bi), Ai Br), operands
// changing every step.  Compares against back-to-back MMAs on fixed operands.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n" : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
__device__ __forceinline__ double dneg(double x) { return __longlong_as_double(__double_as_longlong(x) ^ (long long)0x8000000000000000ULL); }

template <int MB, int NB, int NEG, int ORDER>
__global__ void pattern(double* out, int iters) {
  double ar[MB][NB][2], ai[MB][NB][2];
#pragma unroll
  for (int a = 0; a < MB; ++a)
#pragma unroll
    for (int b = 0; b < NB; ++b) { ar[a][b][0] = ar[a][b][1] = ai[a][b][0] = ai[a][b][1] = threadIdx.x; }
  double2 tw[MB], cv[NB];
#pragma unroll
  for (int a = 0; a < MB; ++a) tw[a] = make_double2(1e-3 * a + threadIdx.x * 1e-6, 2e-3);
#pragma unroll
  for (int b = 0; b < NB; ++b) cv[b] = make_double2(1e-3 * b, 1.0 + 1e-6 * threadIdx.x);
  for (int it = 0; it < iters; ++it) {
    if (ORDER == 0) {
#pragma unroll
      for (int b = 0; b < NB; ++b)
#pragma unroll
        for (int a = 0; a < MB; ++a) {
          dmma(ar[a][b][0], ar[a][b][1], tw[a].x, cv[b].x);
          dmma(ai[a][b][0], ai[a][b][1], tw[a].x, cv[b].y);
        }
#pragma unroll
      for (int b = 0; b < NB; ++b)
#pragma unroll
        for (int a = 0; a < MB; ++a) {
          dmma(ar[a][b][0], ar[a][b][1], tw[a].y, NEG ? dneg(cv[b].y) : cv[b].y);
          dmma(ai[a][b][0], ai[a][b][1], tw[a].y, cv[b].x);
        }
    } else {
#pragma unroll
      for (int b = 0; b < NB; ++b)
#pragma unroll
        for (int a = 0; a < MB; ++a) {
          dmma(ar[a][b][0], ar[a][b][1], tw[a].x, cv[b].x);
          dmma(ar[a][b][0], ar[a][b][1], tw[a].y, NEG ? dneg(cv[b].y) : cv[b].y);
          dmma(ai[a][b][0], ai[a][b][1], tw[a].x, cv[b].y);
          dmma(ai[a][b][0], ai[a][b][1], tw[a].y, cv[b].x);
        }
    }
    // perturb operands so the compiler cannot hoist
#pragma unroll
    for (int a = 0; a < MB; ++a) tw[a].x = __longlong_as_double(__double_as_longlong(tw[a].x) ^ (it & 1));
  }
  double s = 0;
#pragma unroll
  for (int a = 0; a < MB; ++a)
#pragma unroll
    for (int b = 0; b < NB; ++b) s += ar[a][b][0] + ar[a][b][1] + ai[a][b][0] + ai[a][b][1];
  if (s == 1.2345) out[0] = s;
}

template <int MB, int NB, int NEG, int ORDER>
void run(const char* name, int warps, int blocksPerSm, double* d, int sms) {
  int iters = 2000;
  int grid = sms * blocksPerSm, threads = warps * 32;
  pattern<MB, NB, NEG, ORDER><<<grid, threads>>>(d, 10);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(e0); pattern<MB, NB, NEG, ORDER><<<grid, threads>>>(d, iters); cudaEventRecord(e1);
    cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  double flops = 512.0 * 4 * MB * NB * (double)iters * warps * grid;
  cudaError_t err = cudaGetLastError();
  printf("%-28s warps/blk %2d blk/SM %d : %6.2f TFLOP/s %s\n", name, warps, blocksPerSm, flops / best / 1e9,
         err == cudaSuccess ? "" : cudaGetErrorString(err));
}

int main() {
  double* d; cudaMalloc(&d, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<2, 7, 1, 0>("MB2 NB7 neg sweep", 8, 1, d, sms);
  run<2, 7, 0, 0>("MB2 NB7 noneg sweep", 8, 1, d, sms);
  run<2, 7, 1, 1>("MB2 NB7 neg pairs", 8, 1, d, sms);
  run<2, 7, 1, 0>("MB2 NB7 neg sweep", 16, 1, d, sms);
  run<2, 4, 1, 0>("MB2 NB4 neg sweep", 16, 1, d, sms);
  run<1, 7, 1, 0>("MB1 NB7 neg sweep", 16, 1, d, sms);
  run<2, 2, 1, 0>("MB2 NB2 neg sweep", 8, 2, d, sms);
  run<1, 1, 1, 0>("MB1 NB1 neg sweep", 8, 2, d, sms);
  run<4, 4, 1, 0>("MB4 NB4 neg sweep", 8, 1, d, sms);
  return 0;
}
