// tc_i8_rate.cu -- issue-rate microbenchmark of tcgen05.mma.kind::i8 (M = 128) on B200: one CTA per SM,
// one elected lane issues R MMAs back to back (A from TMEM, B from shared memory), committed once;
// reports cycles per MMA and the fraction of the int8 peak (8192 MAC/clk/SM).  Variants: N, number
// of distinct accumulators cycled through, MMAs per accumulator run.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 tools/tc_i8_rate.cu -o tools/tc_i8_rate
#include <cstdio>
#include <cstdlib>

#include "../paper_1606_07407_b200/csrc/tc_i8.cuh"

using namespace sfft;

__global__ void __launch_bounds__(128, 1) rate(int N, int R, int nacc, int run, long long* cyc) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tb;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 256 * 32 * 4 / 4; i += 128) reinterpret_cast<int*>(smem)[i] = i * 2654435761u;
  if (threadIdx.x == 0) {
    tc::mbar_init(&bar, 1);
    tc::fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc<512>(&tb);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t base = tb;
  const uint32_t idesc = tc::idesc_i8(128, N);
  const int a_col = 512 - 64;
  if (warp == 1) {
    long long t0 = clock64();
    for (int i = 0; i < R; ++i) {
      const int acc = (i / run) % nacc;
      const uint32_t d = base + acc * N;
      const uint64_t bd = tc::sdesc_kmajor(tc::smem_u32(smem + (i & 3) * N * 32), 128, 256);
      tc::mma_i8_ts_elect(d, base + a_col + (i & 7) * 8, bd, idesc, i >= nacc * run ? 1u : 0u);
    }
    tc::mma_commit_elect(&bar);
    tc::mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (threadIdx.x == 32 && blockIdx.x == 0) *cyc = t1 - t0;
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<512>(base);
}

// tight variant: descriptors precomputed, 8 MMAs unrolled per iteration with constant offsets
template <int N, bool SS>
__global__ void __launch_bounds__(128, 1) rate2(int R, long long* cyc) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tb;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 256 * 32 * 4 / 4; i += 128) reinterpret_cast<int*>(smem)[i] = i * 2654435761u;
  if (threadIdx.x == 0) {
    tc::mbar_init(&bar, 1);
    tc::fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc<512>(&tb);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t base = tb;
  constexpr uint32_t idesc = tc::idesc_i8(128, N);
  if (warp == 1) {
    const uint64_t bd0 = tc::sdesc_kmajor(tc::smem_u32(smem), 128, 256);
    const uint64_t ad0 = tc::sdesc_kmajor(tc::smem_u32(smem + 65536), 128, 256);
    long long t0 = clock64();
    for (int i = 0; i < R; i += 8) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const uint64_t bd = bd0 + (uint64_t)((u & 3) * N * 32 / 16);
        if constexpr (SS) {
          const uint64_t ad = ad0 + (uint64_t)((u & 3) * 128 * 32 / 16);
          asm volatile("{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(base), "l"(ad), "l"(bd),
                       "r"(idesc), "r"(1) : "memory");
        } else {
          tc::mma_i8_ts_elect(base, base + 448 + u * 8, bd, idesc, 1u);
        }
      }
    }
    tc::mma_commit_elect(&bar);
    tc::mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (threadIdx.x == 32 && blockIdx.x == 0) *cyc = t1 - t0;
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<512>(base);
}

template <int N, bool SS>
void run2(long long* d) {
  cudaFuncSetAttribute(rate2<N, SS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  const int R = 4000;
  rate2<N, SS><<<148, 128, 160 * 1024>>>(R, d);
  cudaDeviceSynchronize();
  long long c;
  cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  const double per = (double)c / R, ideal = 128.0 * N * 32 / 8192.0;
  printf("tight %s N=%3d: %.1f cycles/MMA (ideal %.1f) -> %.0f%% of int8 peak\n", SS ? "SS" : "TS", N, per, ideal,
         100.0 * ideal / per);
}

int main() {
  long long* d;
  cudaMalloc(&d, 8);
  cudaFuncSetAttribute(rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  struct V { int N, nacc, run; } vs[] = {{112, 1, 1}, {112, 3, 1}, {112, 3, 5}, {112, 2, 8}, {128, 1, 1}, {128, 3, 4},
                                         {256, 1, 1}, {64, 1, 1}, {64, 6, 1}, {16, 1, 1}, {48, 5, 3}};
  for (auto v : vs) {
    if (v.nacc * v.N > 448) continue;
    const int R = 4000;
    rate<<<148, 128, 160 * 1024>>>(v.N, R, v.nacc, v.run, d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    long long c;
    cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    const double per = (double)c / R, ideal = 128.0 * v.N * 32 / 8192.0;
    printf("N=%3d nacc=%d run=%d: %.1f cycles/MMA (ideal %.1f) -> %.0f%% of int8 peak\n", v.N, v.nacc, v.run, per, ideal,
           100.0 * ideal / per);
  }
  run2<64, false>(d); run2<112, false>(d); run2<128, false>(d); run2<256, false>(d);
  run2<64, true>(d); run2<112, true>(d); run2<128, true>(d); run2<256, true>(d);
  return 0;
}
