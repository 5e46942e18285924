// k_project.cu -- SURVEY 8(a) row a1: reduced (tilted) frequencies and line coefficients.
//
//   v_{j,q} = sum_{t < d_q} omega_{j, off_q + t} N^t          (Eq. (35); powers 0..d_q-1)
//   (v_{j,a0}, v_{j,a1}) <- (b v0 - h v1, h v0 + b v1)          (Eq. (27)) per tilt
//   C[j][0]   = a_j                                            (unshifted line)
//   C[j][1+n] = a_j e^{2 pi i (v_{j,n} mod E)/E}                (line shifted by eps = 1/E along axis n)
//
// These are the only d-long dot products of the method; they run once per solve.  The exact
// integer reduction (v mod E) keeps the phase exact (reading R1).
#include "sfft_internal.cuh"

namespace sfft {

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// one warp per (signal, term); the term's r reduced coordinates stay in shared memory (tilts, line factors)
// and are written to v_all once.  Dynamic smem: 8 r bytes per warp (SMEM = false for very long keys: v_all
// itself, stride kk).
template <bool SMEM>
__global__ void __launch_bounds__(256) project_kernel(DevParams P, int32_t batch, const int32_t* __restrict__ freqs,
                                                      const double2* __restrict__ coeffs) {
  extern __shared__ int64_t vsm_all[];
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (gw >= (int64_t)batch * P.k) return;
  const int s = (int)(gw / P.k), j = (int)(gw % P.k);
  int64_t* vs = P.v_all + (int64_t)s * P.r * P.kk;
  const int64_t vstr = SMEM ? 1 : P.kk;
  int64_t* vsm = SMEM ? vsm_all + (int64_t)(threadIdx.x >> 5) * P.r : vs + j;
  const int si = P.spec_slots > 1 ? s / P.spec_slots : s;      // the input signal of slot s (R26)
  const int32_t* w = freqs + ((int64_t)si * P.k + j) * P.d;
  for (int q = lane; q < P.r; q += 32) {
    const int off = P.block_off[q], dq = P.block_dims[q];
    int64_t acc = 0, pw = 1;
    int t = 0;
    for (; t + 2 <= dq; t += 2) {                       // two independent loads in flight
      const int64_t w0 = __ldg(w + off + t), w1 = __ldg(w + off + t + 1);
      acc += w0 * pw + w1 * (pw * P.N);
      pw *= P.N * P.N;
    }
    if (t < dq) acc += (int64_t)__ldg(w + off + t) * pw;
    vsm[q * vstr] = acc;
  }
  __syncwarp();
  for (int t = lane; t < P.n_tilts; t += 32) {
    const int64_t* T = P.tilts + 5 * t;
    const int64_t a0 = T[0], a1 = T[1], b = T[2], h = T[3];
    const int64_t u0 = vsm[a0 * vstr], u1 = vsm[a1 * vstr];
    vsm[a0 * vstr] = b * u0 - h * u1;
    vsm[a1 * vstr] = h * u0 + b * u1;
  }
  __syncwarp();
  if (SMEM)
    for (int q = lane; q < P.r; q += 32) vs[(int64_t)q * P.kk + j] = vsm[q];
  const double2 a = coeffs[(int64_t)si * P.k + j];
  double2* Crow = P.C_all + ((int64_t)s * P.kk + j) * P.Lp;
  for (int n = lane; n < P.Lp; n += 32) {
    double2 c;
    if (n == 0) c = a;
    else if (n < P.L) c = cmul(a, line_factor_exact(vsm[(int64_t)(P.line_lo + n - 1) * vstr], P.E));
    else c = make_double2(0.0, 0.0);
    Crow[n] = c;
  }
}

__global__ void init_state_kernel(DevParams P, int32_t batch) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= batch) return;
  P.st_status[s] = ST_RUN;
  P.st_nR[s] = 0;
  P.st_p[s] = 0;
  P.st_m[s] = 0;
  P.st_M[s] = 0;
  P.st_stall[s] = 0;
  P.st_iters[s] = 0;
  P.st_samples[s] = 0;
  P.st_cmacs[s] = 0;
  P.st_cmacs_i8[s] = 0;
  P.st_fftw[2 * s] = 0.0;
  P.st_fftw[2 * s + 1] = 0.0;
  P.st_lvl[s] = 0;
  P.st_il[s] = 0;
  P.st_retilt[s] = 0;
}

cudaError_t launch_project(const DevParams& P, int32_t batch, const int32_t* freqs, const double* coeffs,
                           cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(P.htab, 0, sizeof(int32_t) * (size_t)batch * P.H, st);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(P.st_log, 0, sizeof(int32_t) * 2 * kLogIters, st);
  if (e != cudaSuccess) return e;
  init_state_kernel<<<(batch + 255) / 256, 256, 0, st>>>(P, batch);
  const int64_t warps = (int64_t)batch * P.k;
  const int threads = 256;
  const int64_t blocks = (warps * 32 + threads - 1) / threads;
  const size_t smem = sizeof(int64_t) * (size_t)(threads / 32) * P.r;
  if (smem <= 160 * 1024) {
    e = ensure_smem(project_kernel<true>, smem);
    if (e != cudaSuccess) return e;
    project_kernel<true><<<(unsigned)blocks, threads, smem, st>>>(P, batch, freqs,
                                                                  reinterpret_cast<const double2*>(coeffs));
  } else {
    project_kernel<false><<<(unsigned)blocks, threads, 0, st>>>(P, batch, freqs,
                                                                reinterpret_cast<const double2*>(coeffs));
  }
  return cudaGetLastError();
}

// C rows of signal 0 for K arbitrary terms whose v already sits in v_all[0] (stage entry point).
__global__ void line_coeffs_kernel(DevParams P, int32_t K, const double2* __restrict__ c) {
  const int lane = threadIdx.x & 31;
  const int64_t j = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (j >= K) return;
  const double2 a = c[j];
  double2* Crow = P.C_all + j * P.Lp;
  for (int n = lane; n < P.Lp; n += 32) {
    double2 v;
    if (n == 0) v = a;
    else if (n < P.L) v = cmul(a, line_factor_exact(P.v_all[(int64_t)(P.line_lo + n - 1) * P.kk + j], P.E));
    else v = make_double2(0.0, 0.0);
    Crow[n] = v;
  }
}

cudaError_t launch_line_coeffs(const DevParams& P, int32_t K, const double* c, cudaStream_t st) {
  const int threads = 256;
  const int64_t blocks = ((int64_t)K * 32 + threads - 1) / threads;
  if (blocks > 0)
    line_coeffs_kernel<<<(unsigned)blocks, threads, 0, st>>>(P, K, reinterpret_cast<const double2*>(c));
  return cudaGetLastError();
}

}  // namespace sfft
