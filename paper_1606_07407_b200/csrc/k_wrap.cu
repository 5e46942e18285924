// k_wrap.cu -- SURVEY 8(a) row a8: back to d dimensions (Algorithm 2 l.36).
//   untilt every tilted pair: u = T^T v / hypo^2, rejecting non-integers (Alg. 3 l.38-39, reading R17)
//   wrap every block by balanced digits: digit = ((u + N/2) mod N) - N/2, u <- (u - digit)/N
//   canonical order: lexicographic by frequency vector (rank sort, keys of the first two
//   coordinates in shared memory, full compare only on ties)
#include "sfft_internal.cuh"

namespace sfft {

__global__ void wrap_kernel(DevParams P, int32_t* __restrict__ out_freqs, double2* __restrict__ out_coeffs,
                            int32_t* __restrict__ out_count, int32_t* __restrict__ out_status) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  unsigned long long* key = reinterpret_cast<unsigned long long*>(smem_raw);    // [k]
  __shared__ int bad;
  const int s = blockIdx.x, tid = threadIdx.x;
  const int nR = P.st_nR[s];
  int status = P.st_status[s];
  if (status == ST_RUN) status = SFFT_PARTIAL;
  if (tid == 0) bad = 0;
  __syncthreads();
  const int64_t* vreg = P.v_all + (int64_t)s * P.r * P.kk + P.k;
  int32_t* wt = P.wtmp + (int64_t)s * P.k * P.d;
  const int64_t N = P.N, h2 = N / 2;
  for (int e = tid; e < nR; e += blockDim.x) {
    int32_t* row = wt + (int64_t)e * P.d;
    for (int q = 0; q < P.r; ++q) {
      int64_t u = vreg[(int64_t)q * P.kk + e];
      const int at = P.axis_tilt[q];
      if (at >= 0) {
        const int64_t* T = P.tilts + 5 * (at >> 1);
        const int64_t v0 = vreg[T[0] * P.kk + e], v1 = vreg[T[1] * P.kk + e];
        const int64_t b = T[2], h = T[3], c2 = T[4] * T[4];
        const int64_t num = (at & 1) ? (-h * v0 + b * v1) : (b * v0 + h * v1);
        if (num % c2 != 0) { bad = 1; u = 0; }
        else u = num / c2;
      }
      const int dq = P.block_dims[q], off = P.block_off[q];
      int64_t geo = 0, pw = 1;
      for (int t = 0; t < dq; ++t) { geo += pw; pw *= N; }
      if (u < -h2 * geo || u > (h2 - 1) * geo) { bad = 1; u = 0; }
      for (int t = 0; t < dq; ++t) {
        const int64_t digit = mod_pos64(u + h2, N) - h2;
        row[off + t] = (int32_t)digit;
        u = (u - digit) / N;
      }
    }
    const unsigned long long k0 = (unsigned long long)(row[0] + h2);
    const unsigned long long k1 = P.d > 1 ? (unsigned long long)(row[1] + h2) : 0ull;
    key[e] = (k0 << 32) | k1;
  }
  __syncthreads();
  int32_t* of = out_freqs + (int64_t)s * P.k * P.d;
  double2* oc = out_coeffs + (int64_t)s * P.k;
  const double2* areg = P.a_reg + (int64_t)s * P.k;
  for (int e = tid; e < nR; e += blockDim.x) {
    const unsigned long long ke = key[e];
    const int32_t* re = wt + (int64_t)e * P.d;
    int rank = 0;
    for (int f = 0; f < nR; ++f) {
      const unsigned long long kf = key[f];
      if (kf < ke) ++rank;
      else if (kf == ke && f != e) {
        const int32_t* rf = wt + (int64_t)f * P.d;
        for (int l = 2; l < P.d; ++l) {
          if (rf[l] != re[l]) { rank += rf[l] < re[l]; break; }
        }
      }
    }
    for (int l = 0; l < P.d; ++l) of[(int64_t)rank * P.d + l] = re[l];
    oc[rank] = areg[e];
  }
  for (int64_t i = (int64_t)nR * P.d + tid; i < (int64_t)P.k * P.d; i += blockDim.x) of[i] = 0;
  for (int i = nR + tid; i < P.k; i += blockDim.x) oc[i] = make_double2(0.0, 0.0);
  __syncthreads();
  if (tid == 0) {
    if (bad) status = SFFT_ECORRUPT;
    out_count[s] = nR;
    if (out_status) out_status[s] = status;
    P.st_status[s] = status;
  }
}

cudaError_t launch_wrap(const DevParams& P, int32_t n_signals, int32_t* out_freqs, double* out_coeffs,
                        int32_t* out_count, int32_t* out_status, cudaStream_t st) {
  const size_t smem = sizeof(unsigned long long) * (size_t)P.k;
  cudaError_t e = cudaFuncSetAttribute(wrap_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (n_signals > 0)
    wrap_kernel<<<n_signals, 256, smem, st>>>(P, out_freqs, reinterpret_cast<double2*>(out_coeffs), out_count,
                                              out_status);
  return cudaGetLastError();
}

}  // namespace sfft
