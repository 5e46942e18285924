// k_expsum.cu -- SURVEY 8(a) row a3 (the hot kernel): the residual exponential sum f - g on
// every line of one iteration (Algorithm 2 l.13-14; Eq. (41)):
//
//   s_n[h] = sum_{j < K} C[j][n] * W_p[(h * u_j) mod p],   h in [0, p), n in [0, L)
//
// with u_j = v_{j,m} mod p, W_p[q] = e^{+2 pi i q / p} and C[j][n] the line coefficient of term j
// (a_j or -a_e times e^{2 pi i (v_{j,n-1} mod E)/E}).  Mathematically s_n[h] = f(x) - g(x) at the
// sample point x = unwrap_time((h/p) e_m + (1/E) e_{n-1}); the phase index is an exact integer.
//
// B200 mapping: a (p x K) . (K x L) complex contraction on the FP64 pipe whose left operand is
// generated on the fly from a p-entry root table held in shared memory.  Lanes run along h
// (TH samples per thread, 32 apart), warps split the block tile into WH x WN warp tiles of
// (32*TH) x TN, terms are staged through shared memory in chunks of BK with cp.async double
// buffering.  One complex MAC = 4 DFMA; C values are warp-broadcast LDS.128, roots are
// random-index LDS.128.
#include "sfft_internal.cuh"

namespace sfft {

constexpr int kBK = 16;   // terms per staged chunk

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  const int sz = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

template <int TN, int TH, int WARPS>
__global__ void __launch_bounds__(WARPS * 32)
expsum_kernel(DevParams P, int32_t wn_count, int32_t n_htiles, int32_t n_ntiles) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int BN = TN * wn_count;
  const int WH = WARPS / wn_count;
  const int BM = 32 * TH * WH;

  int bid = blockIdx.x;
  const int nt = bid % n_ntiles;
  bid /= n_ntiles;
  const int ht = bid % n_htiles;
  const int s = bid / n_htiles;
  if (s >= P.batch || P.st_status[s] != ST_RUN) return;
  const int p = P.st_p[s];
  if (ht * BM >= p) return;
  const int m = P.st_m[s];
  const int K = P.k + P.st_nR[s];

  double2* sW = reinterpret_cast<double2*>(smem_raw);
  const int p_pad = (p + 1) & ~1;
  double2* sC = sW + p_pad;                                    // [2][kBK][BN]
  int* sU = reinterpret_cast<int*>(sC + 2 * kBK * BN);          // [2][kBK]
  int* sDU = sU + 2 * kBK;                                     // [2][kBK]

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wn = warp % wn_count, wh = warp / wn_count;

  // root table of this signal's prime (computed by the prep kernel)
  const double2* Wg = P.W_tab + (int64_t)s * P.p_stride;
  for (int q = tid; q < p; q += WARPS * 32) sW[q] = Wg[q];

  const int64_t* vm = P.v_all + ((int64_t)s * P.r + m) * P.kk;     // column m of the term keys
  const double2* Cg = P.C_all + (int64_t)s * P.kk * P.Lp + (int64_t)nt * BN;
  const int n_chunks = (K + kBK - 1) / kBK;

  auto stage = [&](int buf, int chunk) {
    const int j0 = chunk * kBK;
    double2* dst = sC + buf * kBK * BN;
    for (int e = tid; e < kBK * BN; e += WARPS * 32) {
      const int jj = e / BN, n = e - jj * BN;
      const int j = j0 + jj;
      const bool ok = j < K;
      cp_async16(dst + e, ok ? (const void*)(Cg + (int64_t)j * P.Lp + n) : (const void*)Cg, ok);
    }
    if (tid < kBK) {
      const int j = j0 + tid;
      int u = 0;
      if (j < K) u = (int)mod_pos64(vm[j], p);
      sU[buf * kBK + tid] = u;
      sDU[buf * kBK + tid] = (int)(((int64_t)u * 32) % p);
    }
  };

  double2 acc[TH][TN];
#pragma unroll
  for (int t = 0; t < TH; ++t)
#pragma unroll
    for (int n = 0; n < TN; ++n) acc[t][n] = make_double2(0.0, 0.0);

  const unsigned h0 = (unsigned)(ht * BM + wh * 32 * TH + lane);
  const unsigned magic = 0xFFFFFFFFu / (unsigned)p + 1u;      // ceil(2^32 / p): x mod p for x < 2^32 / 64
  const int pp = p;

  stage(0, 0);
  cp_async_commit();
  for (int ch = 0; ch < n_chunks; ++ch) {
    const int buf = ch & 1;
    if (ch + 1 < n_chunks) {
      stage(buf ^ 1, ch + 1);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const double2* cb = sC + buf * kBK * BN + wn * TN;
    const int* ub = sU + buf * kBK;
    const int* dub = sDU + buf * kBK;
#pragma unroll 2
    for (int jj = 0; jj < kBK; ++jj) {
      const unsigned u = (unsigned)ub[jj];
      const int du = dub[jj];
      const unsigned x = h0 * u;
      int r = (int)(x - __umulhi(x, magic) * (unsigned)pp);
      r += (r >> 31) & pp;
      double2 tw[TH];
#pragma unroll
      for (int t = 0; t < TH; ++t) {
        tw[t] = sW[r];
        r += du;
        r -= (r >= pp) ? pp : 0;
      }
      const double2* crow = cb + jj * BN;
#pragma unroll
      for (int n = 0; n < TN; ++n) {
        const double2 c = crow[n];
#pragma unroll
        for (int t = 0; t < TH; ++t) {
          acc[t][n].x = fma(tw[t].x, c.x, acc[t][n].x);
          acc[t][n].x = fma(-tw[t].y, c.y, acc[t][n].x);
          acc[t][n].y = fma(tw[t].x, c.y, acc[t][n].y);
          acc[t][n].y = fma(tw[t].y, c.x, acc[t][n].y);
        }
      }
    }
    __syncthreads();
  }

  double2* out = P.lines + (int64_t)s * P.L * P.p_stride;
  const int n_base = nt * BN + wn * TN;
#pragma unroll
  for (int n = 0; n < TN; ++n) {
    const int nn = n_base + n;
    if (nn >= P.L) break;
#pragma unroll
    for (int t = 0; t < TH; ++t) {
      const unsigned h = h0 + 32u * t;
      if (h < (unsigned)p) out[(int64_t)nn * P.p_stride + h] = acc[t][n];
    }
  }
}

// ---------------------------------------------------------------- host side
static const int kTNs[] = {1, 2, 3, 4, 5, 6, 7, 8, 11, 13, 16};
constexpr int kWarps = 8;
constexpr int kTH = 2;

ExpsumShape choose_expsum_shape(int L) {
  ExpsumShape best{};
  long best_pad = -1;
  for (int tn : kTNs)
    for (int wn : {1, 2, 4, 8}) {
      const int bn = tn * wn;
      const int nt = (L + bn - 1) / bn;
      const long pad = (long)nt * bn;
      bool better = best_pad < 0 || pad < best_pad || (pad == best_pad && tn > best.tn) ||
                    (pad == best_pad && tn == best.tn && wn < best.wn);
      if (better) {
        best_pad = pad;
        best.tn = tn; best.wn = wn; best.th = kTH; best.warps = kWarps;
        best.bm = 32 * kTH * (kWarps / wn); best.bn = bn; best.nt = nt;
      }
    }
  return best;
}

template <int TN>
static cudaError_t launch_tn(const DevParams& P, const ExpsumShape& S, int32_t max_p, int32_t n_signals,
                             cudaStream_t st) {
  const int n_htiles = (max_p + S.bm - 1) / S.bm;
  const size_t smem = sizeof(double2) * (size_t)(((max_p + 1) & ~1) + 2 * kBK * S.bn) + sizeof(int) * 4 * kBK;
  auto kern = expsum_kernel<TN, kTH, kWarps>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const long grid = (long)n_signals * n_htiles * S.nt;
  if (grid <= 0) return cudaSuccess;
  kern<<<(unsigned)grid, kWarps * 32, smem, st>>>(P, S.wn, n_htiles, S.nt);
  return cudaGetLastError();
}

cudaError_t launch_expsum(const DevParams& P, const ExpsumShape& S, int32_t max_p, int32_t n_signals,
                          cudaStream_t st) {
  switch (S.tn) {
    case 1: return launch_tn<1>(P, S, max_p, n_signals, st);
    case 2: return launch_tn<2>(P, S, max_p, n_signals, st);
    case 3: return launch_tn<3>(P, S, max_p, n_signals, st);
    case 4: return launch_tn<4>(P, S, max_p, n_signals, st);
    case 5: return launch_tn<5>(P, S, max_p, n_signals, st);
    case 6: return launch_tn<6>(P, S, max_p, n_signals, st);
    case 7: return launch_tn<7>(P, S, max_p, n_signals, st);
    case 8: return launch_tn<8>(P, S, max_p, n_signals, st);
    case 11: return launch_tn<11>(P, S, max_p, n_signals, st);
    case 13: return launch_tn<13>(P, S, max_p, n_signals, st);
    case 16: return launch_tn<16>(P, S, max_p, n_signals, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace sfft
