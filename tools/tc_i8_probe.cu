// tc_i8_probe.cu -- hardware check of the tcgen05 building blocks used by k_expsum_i8.cu:
// kind::i8 MMA with A in TMEM (tcgen05.st, 4 K-bytes per 32-bit column) and B in shared memory
// (K-major, no swizzle, core matrices 8 rows x 16 B, LBO 128 B, SBO 256 B), s32 accumulator read
// back with tcgen05.ld 32x32b.  One CTA, M = 128, several K steps accumulated, N in {16, 112, 256}.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 tools/tc_i8_probe.cu -o tools/tc_i8_probe
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../paper_1606_07407_b200/csrc/tc_i8.cuh"

using namespace sfft;

constexpr int KS = 3;   // K steps of 32

__global__ void __launch_bounds__(128) probe(const int8_t* A, const int8_t* Bt, int32_t* D, int N) {
  __shared__ __align__(128) int8_t sB[KS * 256 * 32];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  // B tiles already in the UMMA layout in global memory: plain copy
  for (int i = tid; i < KS * N * 32 / 4; i += 128) reinterpret_cast<int32_t*>(sB)[i] = reinterpret_cast<const int32_t*>(Bt)[i];
  if (tid == 0) {
    tc::mbar_init(&bar, 1);
    tc::fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc<512>(&tbase);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t base = tbase;
  const uint32_t lane_addr = base + ((uint32_t)(warp * 32) << 16);
  const int a_col = 256;
  // A rows -> TMEM: row m = tid, K bytes packed 4 per column (byte 0 = lowest K)
  for (int ks = 0; ks < KS; ++ks) {
    uint32_t w[8];
    for (int c = 0; c < 8; ++c) {
      const int8_t* a = A + (size_t)tid * (KS * 32) + ks * 32 + 4 * c;
      w[c] = (uint32_t)(uint8_t)a[0] | ((uint32_t)(uint8_t)a[1] << 8) | ((uint32_t)(uint8_t)a[2] << 16) |
             ((uint32_t)(uint8_t)a[3] << 24);
    }
    tc::tmem_st8(lane_addr + a_col + ks * 8, w);
  }
  tc::tmem_wait_st();
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic smem writes -> async proxy
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  if (tid == 0) {
    const uint32_t idesc = tc::idesc_i8(128, N);
    for (int ks = 0; ks < KS; ++ks) {
      const uint64_t bd = tc::sdesc_kmajor(tc::smem_u32(sB + ks * N * 32), 128, 256);
      tc::mma_i8_ts(base, base + a_col + ks * 8, bd, idesc, ks > 0);
    }
    tc::mma_commit(&bar);
  }
  __syncwarp();
  tc::mbar_wait(&bar, 0);
  tc::fence_after_sync();
  for (int c0 = 0; c0 < N; c0 += 16) {
    int32_t v[16];
    tc::tmem_ld16(lane_addr + c0, v);
    tc::tmem_wait_ld();
    for (int i = 0; i < 16; ++i) D[(size_t)tid * N + c0 + i] = v[i];
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<512>(base);
}

int main() {
  int bad_total = 0;
  for (int N : {16, 112, 256}) {
    std::vector<int8_t> A(128 * KS * 32), B((size_t)N * KS * 32), Bt((size_t)KS * N * 32);
    srand(1234 + N);
    for (auto& x : A) x = (int8_t)(rand() % 256 - 128);
    for (auto& x : B) x = (int8_t)(rand() % 256 - 128);
    // B[n][k] (k over KS*32) -> per K step tile: off(n,k) = (n/8)*256 + (k/16)*128 + (n%8)*16 + k%16
    for (int ks = 0; ks < KS; ++ks)
      for (int n = 0; n < N; ++n)
        for (int k = 0; k < 32; ++k)
          Bt[(size_t)ks * N * 32 + (n / 8) * 256 + (k / 16) * 128 + (n % 8) * 16 + k % 16] = B[(size_t)n * KS * 32 + ks * 32 + k];
    int8_t *dA, *dB;
    int32_t* dD;
    cudaMalloc(&dA, A.size());
    cudaMalloc(&dB, Bt.size());
    cudaMalloc(&dD, 4 * 128 * N);
    cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dB, Bt.data(), Bt.size(), cudaMemcpyHostToDevice);
    cudaMemset(dD, 0, 4 * 128 * N);
    probe<<<1, 128>>>(dA, dB, dD, N);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("N=%d CUDA error %s\n", N, cudaGetErrorString(e));
      return 2;
    }
    std::vector<int32_t> D(128 * N);
    cudaMemcpy(D.data(), dD, 4 * D.size(), cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int m = 0; m < 128; ++m)
      for (int n = 0; n < N; ++n) {
        int32_t ref = 0;
        for (int k = 0; k < KS * 32; ++k) ref += (int32_t)A[m * KS * 32 + k] * (int32_t)B[(size_t)n * KS * 32 + k];
        if (ref != D[m * N + n]) {
          if (bad < 8) printf("N=%d mismatch m=%d n=%d got %d want %d\n", N, m, n, D[m * N + n], ref);
          ++bad;
        }
      }
    printf("N=%d: %d / %d mismatches\n", N, bad, 128 * N);
    bad_total += bad;
    cudaFree(dA);
    cudaFree(dB);
    cudaFree(dD);
  }
  printf(bad_total ? "PROBE FAIL\n" : "PROBE OK\n");
  return bad_total ? 1 : 0;
}
