// tc_i8_probe2.cu -- hardware check of the CTA-pair (cta_group::2) kind::i8 MMA: a cluster of 2 CTAs,
// A rows 0-127 in CTA 0's TMEM and 128-255 in CTA 1's (same TMEM address), B columns [0, N/2) in CTA 0's
// shared memory and [N/2, N) in CTA 1's (same offset), D rows of each CTA in its own TMEM; the leader CTA
// issues, the commit is multicast to both CTAs' mbarriers.  Checks D = A B^T exactly for several N.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 tools/tc_i8_probe2.cu -o tools/tc_i8_probe2
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_1606_07407_b200/csrc/tc_i8.cuh"

using namespace sfft;

constexpr int KS = 2;

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128) probe2(const int8_t* A, const int8_t* Bt, int32_t* D, int N) {
  __shared__ __align__(128) int8_t sB[KS * 128 * 32];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  const uint32_t rank = cluster_rank();
  const int Nh = N / 2;
  // this CTA's half of B: columns [rank * N/2, (rank + 1) * N/2), per K step a (N/2) x 32 K-major tile
  for (int i = tid; i < KS * Nh * 32 / 4; i += 128)
    reinterpret_cast<int32_t*>(sB)[i] = reinterpret_cast<const int32_t*>(Bt + (size_t)rank * KS * Nh * 32)[i];
  if (tid == 0) {
    tc::mbar_init(&bar, 1);
    tc::fence_mbar_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(tc::smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc::fence_before_sync();
  __syncthreads();
  cluster_sync();
  tc::fence_after_sync();
  const uint32_t base = tbase;
  const uint32_t lane_addr = base + ((uint32_t)(warp * 32) << 16);
  const int a_col = 256;
  for (int ks = 0; ks < KS; ++ks) {
    uint32_t w[8];
    for (int c = 0; c < 8; ++c) {
      const int8_t* a = A + ((size_t)rank * 128 + tid) * (KS * 32) + ks * 32 + 4 * c;
      w[c] = (uint32_t)(uint8_t)a[0] | ((uint32_t)(uint8_t)a[1] << 8) | ((uint32_t)(uint8_t)a[2] << 16) |
             ((uint32_t)(uint8_t)a[3] << 24);
    }
    tc::tmem_st8(lane_addr + a_col + ks * 8, w);
  }
  tc::tmem_wait_st();
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc::fence_before_sync();
  __syncthreads();
  cluster_sync();
  tc::fence_after_sync();
  if (rank == 0 && tid == 0) {
    const uint32_t idesc = tc::idesc_i8(256, N);
    for (int ks = 0; ks < KS; ++ks) {
      const uint64_t bd = tc::sdesc_kmajor(tc::smem_u32(sB + ks * Nh * 32), 128, 256);
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::2.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(base),
          "r"(base + a_col + ks * 8), "l"(bd), "r"(idesc), "r"(ks > 0 ? 1u : 0u)
          : "memory");
    }
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            tc::smem_u32(&bar)),
        "h"((uint16_t)3)
        : "memory");
  }
  __syncwarp();
  tc::mbar_wait(&bar, 0);
  tc::fence_after_sync();
  for (int c0 = 0; c0 < N; c0 += 16) {
    int32_t v[16];
    tc::tmem_ld16(lane_addr + c0, v);
    tc::tmem_wait_ld();
    for (int i = 0; i < 16; ++i)
      if (c0 + i < N) D[((size_t)rank * 128 + tid) * N + c0 + i] = v[i];
  }
  tc::fence_before_sync();
  __syncthreads();
  cluster_sync();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(base));
}

int main() {
  int bad_total = 0;
  for (int N : {32, 48, 64, 96, 112, 128}) {
    const int Nh = N / 2;
    std::vector<int8_t> A(256 * KS * 32), B((size_t)N * KS * 32), Bt((size_t)2 * KS * Nh * 32);
    srand(99 + N);
    for (auto& x : A) x = (int8_t)(rand() % 256 - 128);
    for (auto& x : B) x = (int8_t)(rand() % 256 - 128);
    for (int h = 0; h < 2; ++h)
      for (int ks = 0; ks < KS; ++ks)
        for (int n = 0; n < Nh; ++n)
          for (int k = 0; k < 32; ++k)
            Bt[(size_t)h * KS * Nh * 32 + (size_t)ks * Nh * 32 + (n / 8) * 256 + (k / 16) * 128 + (n % 8) * 16 + k % 16] =
                B[(size_t)(h * Nh + n) * KS * 32 + ks * 32 + k];
    int8_t *dA, *dB;
    int32_t* dD;
    cudaMalloc(&dA, A.size());
    cudaMalloc(&dB, Bt.size());
    cudaMalloc(&dD, 4 * 256 * N);
    cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dB, Bt.data(), Bt.size(), cudaMemcpyHostToDevice);
    cudaMemset(dD, 0, 4 * 256 * N);
    probe2<<<2, 128>>>(dA, dB, dD, N);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("N=%d CUDA error %s\n", N, cudaGetErrorString(e));
      return 2;
    }
    std::vector<int32_t> D(256 * N);
    cudaMemcpy(D.data(), dD, 4 * D.size(), cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int m = 0; m < 256; ++m)
      for (int n = 0; n < N; ++n) {
        int32_t ref = 0;
        for (int k = 0; k < KS * 32; ++k) ref += (int32_t)A[m * KS * 32 + k] * (int32_t)B[(size_t)n * KS * 32 + k];
        if (ref != D[m * N + n]) {
          if (bad < 4) printf("N=%d mismatch m=%d n=%d got %d want %d\n", N, m, n, D[m * N + n], ref);
          ++bad;
        }
      }
    printf("cta_group::2 N=%d: %d / %d mismatches\n", N, bad, 256 * N);
    bad_total += bad;
    cudaFree(dA);
    cudaFree(dB);
    cudaFree(dD);
  }
  printf(bad_total ? "PROBE2 FAIL\n" : "PROBE2 OK\n");
  return bad_total ? 1 : 0;
}
