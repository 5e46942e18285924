// decode_common.cuh -- device building blocks of SURVEY 8(a) rows a5 (select) and a6 (collision test +
// decode), shared by the fused FFT epilogue (k_fft.cu: line-0 CTAs select, line-n CTAs test their line)
// and the teacher-forced stage entry point (k_decode.cu).  Algorithm 2 l.18-29.
#pragma once
#include "sfft_internal.cuh"

namespace sfft {

// exclusive prefix sum over the block (blockDim a multiple of 32, <= 1024); *total gets the sum.
// scratch: >= 32 ints of shared memory.
__device__ __forceinline__ int block_excl_scan(int v, int* scratch, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) scratch[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int t = lane < nw ? scratch[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    if (lane < nw) scratch[lane] = t;       // inclusive warp-prefix
  }
  __syncthreads();
  const int before = warp > 0 ? scratch[warp - 1] : 0;
  *total = scratch[nw - 1];
  __syncthreads();
  return before + x - v;
}

// a5 select (Alg. 2 l.18, readings R5/R6): bins b < p with |F_0[b]| >= floor_abs in ascending b; if more than
// kstar qualify, the kstar largest |F_0| (ties -> smaller b), still ascending.  f0(b) returns F_0[b].
// Shared memory: cand[p], mag[p], flag[p], scratch[>= 32].  Returns the candidate count (all threads).
// Needs ceil(nc / blockDim) <= 32 (p <= 32 blockDim).
template <class F0>
__device__ int select_candidates(F0 f0, int p, int kstar, double floor_abs, int* cand, double* mag, int* flag,
                                 int* scratch) {
  const int tid = threadIdx.x;
  int total = 0;
  // thread t owns the contiguous bins [t per, (t + 1) per): flags in a register mask, one block scan
  const int per = (p + blockDim.x - 1) / blockDim.x;     // <= 32
  const int b0 = tid * per, b1 = min(p, b0 + per);
  unsigned mask = 0u;
  for (int b = b0; b < b1; ++b) {
    const double2 f = f0(b);
    if (hypot(f.x, f.y) >= floor_abs) mask |= 1u << (b - b0);
  }
  int pos = block_excl_scan(__popc(mask), scratch, &total);
  for (int b = b0; b < b1; ++b)
    if (mask >> (b - b0) & 1u) {
      const double2 f = f0(b);
      cand[pos] = b;
      mag[pos] = hypot(f.x, f.y);
      ++pos;
    }
  __syncthreads();
  int nc = total;
  if (nc > kstar) {
    for (int i = tid; i < nc; i += blockDim.x) {
      const double mi = mag[i];
      const int bi = cand[i];
      int rank = 0;
      for (int j = 0; j < nc; ++j) rank += (mag[j] > mi) || (mag[j] == mi && cand[j] < bi);
      flag[i] = rank < kstar;
    }
    __syncthreads();
    const int per2 = (nc + blockDim.x - 1) / blockDim.x;
    const int i0 = tid * per2, i1 = min(nc, i0 + per2);
    int c2 = 0, keep_b[32], nk = 0;
    for (int i = i0; i < i1; ++i) c2 += flag[i];
    const int pos2 = block_excl_scan(c2, scratch, &total);
    for (int i = i0; i < i1 && nk < 32; ++i)
      if (flag[i]) keep_b[nk++] = cand[i];
    __syncthreads();
    for (int t = 0; t < nk; ++t) cand[pos2 + t] = keep_b[t];
    __syncthreads();
    nc = total;
  }
  return nc;
}

// a6 for one (candidate, shifted line): Eq. (42) |F_n| / |F_0| within tol of 1, then Eq. (41)
// v = round(Arg(F_n conj F_0) E / 2 pi) with |x - v| <= round_tol and (range) lo <= v <= hi.
__device__ __forceinline__ bool test_decode(double2 f0, double2 fv, double tol, int64_t E, double round_tol,
                                            bool range, int64_t lo, int64_t hi, int64_t* v_out) {
  const double mag0 = hypot(f0.x, f0.y);
  const double rho = hypot(fv.x, fv.y) / mag0;
  if (!(fabs(rho - 1.0) < tol)) return false;
  // q = F_n conj(F_0), written without contraction to mirror the plain formula
  const double qr = __dadd_rn(__dmul_rn(fv.x, f0.x), __dmul_rn(fv.y, f0.y));
  const double qi = __dsub_rn(__dmul_rn(fv.y, f0.x), __dmul_rn(fv.x, f0.y));
  const double twopi = 6.283185307179586476925286766559;
  const double x = __ddiv_rn(__dmul_rn(atan2(qi, qr), (double)E), twopi);
  const double xr = rint(x);
  bool good = fabs(x - xr) <= round_tol;
  const int64_t v = (int64_t)xr;
  if (range) good = good && v >= lo && v <= hi;
  *v_out = v;
  return good;
}

// bin-domain residual (reading R21): F_n[b] + p sum_{e in bin b} C_reg[e][n], entries in ascending e
// (the per-bin order of terms_kernel), rounded as written (no contraction)
__device__ __forceinline__ double2 add_bin_residual(double2 f, const int32_t* bstart, const int32_t* border,
                                                    const double2* Creg, int Lp, int n, int b, double pd) {
  const int q0 = bstart[b], q1 = bstart[b + 1];
  if (q0 == q1) return f;
  double2 acc = make_double2(0.0, 0.0);
  for (int q = q0; q < q1; ++q) {
    const double2 c = Creg[(int64_t)border[q] * Lp + n];
    acc.x = __dadd_rn(acc.x, c.x);
    acc.y = __dadd_rn(acc.y, c.y);
  }
  return make_double2(__dadd_rn(f.x, __dmul_rn(pd, acc.x)), __dadd_rn(f.y, __dmul_rn(pd, acc.y)));
}

}  // namespace sfft
