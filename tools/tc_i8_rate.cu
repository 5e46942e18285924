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

// the exp-sum pass pattern: per stage, all products (s, t) with s + t in [3, 5] (15 MMAs) into 3
// accumulators at columns acc_stride * (w - 3), A slots at a_base + sa * 48 + 8 s, then commits
template <int WL, int WH>
__device__ __forceinline__ void stage_mmas(uint32_t base, uint32_t a0, uint64_t bd0, uint32_t acc_stride, uint32_t ntd,
                                           uint32_t idesc) {
#pragma unroll
  for (int w = WL; w <= WH; ++w)
#pragma unroll
    for (int sl = 0; sl <= w; ++sl)
      tc::mma_i8_ts(base + (w - WL) * acc_stride, a0 + 8 * sl, bd0 + (uint64_t)((w - sl) * ntd), idesc, 1u);
}
__global__ void __launch_bounds__(128, 1) pattern(int stages, int acc_stride, int a_base, int commits, long long* cyc) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar[8];
  __shared__ uint32_t tb;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 8; ++i) tc::mbar_init(bar + i, 1);
    tc::fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc<512>(&tb);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t base = tb;
  const uint32_t idesc = tc::idesc_i8(128, 112);
  if (warp == 1) {
    long long t0 = clock64();
    for (int st = 0; st < stages; ++st) {
      const int sb = st & 3, sa = st % 3;
      const uint64_t bd0 = tc::sdesc_kmajor(tc::smem_u32(smem + sb * 6 * 112 * 32), 128, 256);
      const uint32_t a0 = base + a_base + sa * 48;
      if (tc::elect_one()) {
        stage_mmas<3, 5>(base, a0, bd0, acc_stride, 112 * 2, idesc);
        if (commits) {
          tc::mma_commit(bar + sb);
          tc::mma_commit(bar + 4 + sa);
        }
      }
      __syncwarp();
    }
    if (tc::elect_one()) tc::mma_commit(bar + 7);
    __syncwarp();
    while (!tc::mbar_try_wait(bar + 7, 0)) {}
    long long t1 = clock64();
    if (threadIdx.x == 32 && blockIdx.x == 0) *cyc = t1 - t0;
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<512>(base);
}

// pattern + a per-stage wait on an mbarrier that completed long ago (phase 0 done, waiting parity 0)
__device__ __forceinline__ bool test_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
               "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(tc::smem_u32(bar)), "r"(parity) : "memory");
  return ok != 0;
}
__global__ void __launch_bounds__(128, 1) pattern_wait(int stages, int mode, long long* cyc) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar[9];
  __shared__ uint32_t tb;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 9; ++i) tc::mbar_init(bar + i, 1);
    tc::fence_mbar_init();
    tc::mbar_arrive(bar + 8);            // phase 0 of bar[8] completes now
  }
  if (warp == 0) tc::tmem_alloc<512>(&tb);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t base = tb;
  const uint32_t idesc = tc::idesc_i8(128, 64);
  if (warp == 1) {
    long long t0 = clock64();
    for (int st = 0; st < stages; ++st) {
      const int sb = st & 3, sa = st & 1;
      if (mode == 1) tc::mbar_wait(bar + 8, 0);
      if (mode == 2) while (!test_wait(bar + 8, 0)) {}
      tc::fence_after_sync();
      const uint64_t bd0 = tc::sdesc_kmajor(tc::smem_u32(smem + sb * 6 * 64 * 32), 128, 256);
      const uint32_t a0 = base + 384 + sa * 48;
      if (tc::elect_one()) {
        stage_mmas<0, 5>(base, a0, bd0, 64, 64 * 2, idesc);
        tc::mma_commit(bar + sb);
      }
      __syncwarp();
    }
    if (tc::elect_one()) tc::mma_commit(bar + 7);
    __syncwarp();
    while (!tc::mbar_try_wait(bar + 7, 0)) {}
    long long t1 = clock64();
    if (threadIdx.x == 32 && blockIdx.x == 0) *cyc = t1 - t0;
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<512>(base);
}
void run_pattern_wait(long long* d, int mode) {
  cudaFuncSetAttribute(pattern_wait, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  const int stages = 400;
  pattern_wait<<<148, 128, 160 * 1024>>>(stages, mode, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long c = 0;
  cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  printf("pattern_wait N=64 S=6 mode=%d (0 none, 1 try_wait, 2 test_wait spin): %.1f cycles/stage (ideal %.1f) %s\n", mode,
         (double)c / stages, 21 * 32.0, cudaGetErrorString(e));
}

// sweep: weights [WL, WH], width N, accumulators at w * N, A slots after them
template <int WL, int WH>
__global__ void __launch_bounds__(128, 1) pattern_sweep(int stages, int N, long long* cyc) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar[8];
  __shared__ uint32_t tb;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 8; ++i) tc::mbar_init(bar + i, 1);
    tc::fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc<512>(&tb);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t base = tb;
  const uint32_t idesc = tc::idesc_i8(128, N);
  constexpr int nl = WH + 1;
  if (warp == 1) {
    long long t0 = clock64();
    for (int st = 0; st < stages; ++st) {
      const int sb = st & 3, sa = st & 1;
      const uint64_t bd0 = tc::sdesc_kmajor(tc::smem_u32(smem + sb * 6 * 64 * 32), 128, 256);
      const uint32_t a0 = base + (WH - WL + 1) * N + sa * nl * 8;
      if (tc::elect_one()) {
        stage_mmas<WL, WH>(base, a0, bd0, N, N * 2, idesc);
        tc::mma_commit(bar + sb);
      }
      __syncwarp();
    }
    if (tc::elect_one()) tc::mma_commit(bar + 7);
    __syncwarp();
    while (!tc::mbar_try_wait(bar + 7, 0)) {}
    long long t1 = clock64();
    if (threadIdx.x == 32 && blockIdx.x == 0) *cyc = t1 - t0;
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<512>(base);
}
template <int WL, int WH>
void run_sweep(long long* d, int N) {
  if ((WH - WL + 1) * N + 2 * (WH + 1) * 8 > 512) return;
  cudaFuncSetAttribute(pattern_sweep<WL, WH>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  const int stages = 400;
  pattern_sweep<WL, WH><<<148, 128, 160 * 1024>>>(stages, N, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long c = 0;
  cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  int prods = 0;
  for (int w = WL; w <= WH; ++w) prods += w + 1;
  const double ideal = prods * N / 2.0;
  printf("sweep w[%d,%d] N=%3d: %.1f cycles/stage, ideal %.1f -> %.0f%% %s\n", WL, WH, N, (double)c / stages, ideal,
         100.0 * ideal * stages / c, cudaGetErrorString(e));
}

// pattern S=6 N=64 fed by a real producer: bulk copies of 12 KB stages from global (L2-resident) into an
// 8-slot ring, MMA warp waits bfull per stage (mode 0) or not at all (mode 1, copies still running)
__global__ void __launch_bounds__(96, 1) pattern_copy(int stages, int mode, const int8_t* gB, long long* cyc) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ __align__(8) uint64_t bfull[8], bempty[8], fin;
  __shared__ uint32_t tb;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 8; ++i) { tc::mbar_init(bfull + i, 1); tc::mbar_init(bempty + i, 1); }
    tc::mbar_init(&fin, 1);
    tc::fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc<512>(&tb);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t base = tb;
  const uint32_t idesc = tc::idesc_i8(128, 64);
  const uint32_t bytes = 6 * 64 * 32;
  if (warp == 2 && lane == 0) {
    for (int st = 0; st < stages; ++st) {
      const int sb = st & 7;
      const uint32_t par = ((st >> 3) & 1) ^ 1;
      while (!tc::mbar_try_wait(bempty + sb, par)) __nanosleep(100);
      tc::mbar_expect_tx(bfull + sb, bytes);
      tc::bulk_g2s(smem + sb * bytes, gB + ((size_t)(blockIdx.x * 7 + st) % 160) * bytes, bytes, bfull + sb);
    }
  }
  if (warp == 1) {
    long long t0 = clock64();
    for (int st = 0; st < stages; ++st) {
      const int sb = st & 7, sa = st & 1;
      if (mode == 0) tc::mbar_wait(bfull + sb, (st >> 3) & 1);
      tc::fence_after_sync();
      const uint64_t bd0 = tc::sdesc_kmajor(tc::smem_u32(smem + sb * bytes), 128, 256);
      const uint32_t a0 = base + 384 + sa * 48;
      if (tc::elect_one()) {
        stage_mmas<0, 5>(base, a0, bd0, 64, 64 * 2, idesc);
        tc::mma_commit(bempty + sb);
      }
      __syncwarp();
    }
    if (tc::elect_one()) tc::mma_commit(&fin);
    __syncwarp();
    while (!tc::mbar_try_wait(&fin, 0)) {}
    long long t1 = clock64();
    if (threadIdx.x == 32 && blockIdx.x == 0) *cyc = t1 - t0;
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<512>(base);
}
void run_pattern_copy(long long* d, int mode) {
  static int8_t* gB = nullptr;
  if (!gB) { cudaMalloc(&gB, 160 * 6 * 64 * 32); cudaMemset(gB, 1, 160 * 6 * 64 * 32); }
  cudaFuncSetAttribute(pattern_copy, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  const int stages = 800;
  pattern_copy<<<148, 96, 160 * 1024>>>(stages, mode, gB, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long c = 0;
  cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  printf("pattern_copy mode=%d: %.1f cycles/stage (ideal 672) %s\n", mode, (double)c / stages, cudaGetErrorString(e));
}

void run_pattern(long long* d, int acc_stride, int a_base, int commits) {
  cudaFuncSetAttribute(pattern, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  const int stages = 400;
  pattern<<<148, 128, 160 * 1024>>>(stages, acc_stride, a_base, commits, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long c = 0;
  cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  printf("pattern acc_stride=%d a_base=%d commits=%d: %.1f cycles/stage (ideal %.1f) %s\n", acc_stride, a_base, commits,
         (double)c / stages, 15 * 56.0, cudaGetErrorString(e));
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
  run_pattern_copy(d, 0);
  run_pattern_copy(d, 1);
  run_sweep<0, 5>(d, 64);
  run_pattern_wait(d, 0);
  run_pattern_wait(d, 1);
  run_pattern_wait(d, 2);
  run_pattern(d, 112, 336, 1);
  run2<64, false>(d); run2<112, false>(d); run2<128, false>(d); run2<256, false>(d);
  run2<64, true>(d); run2<112, true>(d); run2<128, true>(d); run2<256, true>(d);
  return 0;
}
