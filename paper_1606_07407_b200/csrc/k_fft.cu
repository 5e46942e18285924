// k_fft.cu -- SURVEY 8(a) row a4: batched prime-length DFTs (Algorithm 2 l.16-17)
//
//   F_n[b] = sum_{h < p} s_n[h] e^{-2 pi i h b / p}     (unnormalised, so Eq. (3)'s factor p appears)
//
// p is prime (no Cooley-Tukey split), so each line is transformed with Bluestein's identity
// hb = (h^2 + b^2 - (b-h)^2)/2:
//   F[b] = w[b] * sum_h (s[h] w[h]) conj(w[b-h]),  w[n] = e^{-pi i (n^2 mod 2p)/p}  (exact index)
// i.e. a cyclic convolution of length M >= 2p-1 done as DIF-FFT -> pointwise product with the
// precomputed kernel spectrum -> DIT-inverse FFT.  M is 7-smooth (radices 2,3,4,5,7,8) and the
// whole length-M work array lives in shared memory (M <= 14112 -> 221 KB).  The forward FFT is
// in-place decimation in frequency (natural order in, digit-reversed out); the kernel spectrum
// is produced by the same routine, so the pointwise product happens in digit-reversed order and
// the in-place decimation-in-time inverse returns natural order: no permutation pass.
// Twiddles e^{-2 pi i q/M} = T_hi[q >> 7] * T_lo[q & 127], two small tables in shared memory.
#include "fft_consts.cuh"
#include <algorithm>
#include <cstdlib>

#include "decode_common.cuh"
#include "sfft_internal.cuh"

namespace sfft {

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmulx(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cmulconj(double2 a, double2 b) {   // a * conj(b)
  return make_double2(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}
__device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
// multiply by -i (forward) or +i (inverse)
template <bool INV>
__device__ __forceinline__ double2 mul_mi(double2 a) {
  return INV ? make_double2(-a.y, a.x) : make_double2(a.y, -a.x);
}

// cos / sin of 2 pi k / R for the odd radices
__device__ __constant__ double kCos3[3] = {1.0, -0.5, -0.5};
__device__ __constant__ double kSin3[3] = {0.0, 0.86602540378443864676, -0.86602540378443864676};
__device__ __constant__ double kCos5[5] = {1.0, 0.30901699437494742410, -0.80901699437494742410,
                                           -0.80901699437494742410, 0.30901699437494742410};
__device__ __constant__ double kSin5[5] = {0.0, 0.95105651629515357212, 0.58778525229247312917,
                                           -0.58778525229247312917, -0.95105651629515357212};
__device__ __constant__ double kCos7[7] = {1.0, 0.62348980185873353053, -0.22252093395631440429,
                                           -0.90096886790241912624, -0.90096886790241912624,
                                           -0.22252093395631440429, 0.62348980185873353053};
__device__ __constant__ double kSin7[7] = {0.0, 0.78183148246802980871, 0.97492791218182360702,
                                           0.43388373911755812048, -0.43388373911755812048,
                                           -0.97492791218182360702, -0.78183148246802980871};

// in-register DFT of size R; forward uses e^{-2 pi i nk/R}, inverse e^{+2 pi i nk/R}
template <int R, bool INV>
__device__ __forceinline__ void dft_small(double2 (&x)[R]) {
  if constexpr (R == 2) {
    const double2 a = x[0], b = x[1];
    x[0] = cadd(a, b);
    x[1] = csub(a, b);
  } else if constexpr (R == 4) {
    const double2 a0 = cadd(x[0], x[2]), a1 = csub(x[0], x[2]);
    const double2 b0 = cadd(x[1], x[3]), b1 = mul_mi<INV>(csub(x[1], x[3]));
    x[0] = cadd(a0, b0);
    x[2] = csub(a0, b0);
    x[1] = cadd(a1, b1);
    x[3] = csub(a1, b1);
  } else if constexpr (R == 8) {
    const double h = 0.70710678118654752440;
    double2 a[4], b[4];
#pragma unroll
    for (int n = 0; n < 4; ++n) {
      a[n] = cadd(x[n], x[n + 4]);
      b[n] = csub(x[n], x[n + 4]);
    }
    // b[n] *= w8^n, w8 = e^{-+ 2 pi i / 8}
    b[1] = INV ? make_double2(h * (b[1].x - b[1].y), h * (b[1].x + b[1].y))
               : make_double2(h * (b[1].x + b[1].y), h * (b[1].y - b[1].x));
    b[2] = mul_mi<INV>(b[2]);
    b[3] = INV ? make_double2(-h * (b[3].x + b[3].y), h * (b[3].x - b[3].y))
               : make_double2(h * (b[3].y - b[3].x), -h * (b[3].x + b[3].y));
    dft_small<4, INV>(a);
    dft_small<4, INV>(b);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      x[2 * k] = a[k];
      x[2 * k + 1] = b[k];
    }
  } else if constexpr (R == 3 || R == 5 || R == 7) {
    // odd prime R: pair n with R-n
    const double* C = (R == 3) ? kCos3 : (R == 5) ? kCos5 : kCos7;
    const double* S = (R == 3) ? kSin3 : (R == 5) ? kSin5 : kSin7;
    constexpr int H = (R - 1) / 2;
    double2 sp[H], sm[H];
    double2 y0 = x[0];
#pragma unroll
    for (int n = 1; n <= H; ++n) {
      sp[n - 1] = cadd(x[n], x[R - n]);
      sm[n - 1] = csub(x[n], x[R - n]);
      y0 = cadd(y0, sp[n - 1]);
    }
    double2 out[R];
    out[0] = y0;
#pragma unroll
    for (int k = 1; k <= H; ++k) {
      double2 re = x[0], im = make_double2(0.0, 0.0);
#pragma unroll
      for (int n = 1; n <= H; ++n) {
        const int q = (n * k) % R;
        re = make_double2(re.x + C[q] * sp[n - 1].x, re.y + C[q] * sp[n - 1].y);
        im = make_double2(im.x + S[q] * sm[n - 1].x, im.y + S[q] * sm[n - 1].y);
      }
      // forward: y[k] = re - i im, y[R-k] = re + i im
      const double2 mi = make_double2(im.y, -im.x);   // -i * im
      out[k] = INV ? csub(re, mi) : cadd(re, mi);
      out[R - k] = INV ? cadd(re, mi) : csub(re, mi);
    }
#pragma unroll
    for (int k = 0; k < R; ++k) x[k] = out[k];
  } else {
    // composite R = A B (in registers): n = B n1 + n2, k = k1 + A k2
    //   t[n2][k1] = DFT_A over n1 of x[B n1 + n2], times w_R^(n2 k1); y[k1 + A k2] = DFT_B over n2
    constexpr int A = (R == 16) ? 4 : (R == 12) ? 4 : (R == 9) ? 3 : (R == 15) ? 3 : (R == 6) ? 3 : (R == 10) ? 5 : 7;
    constexpr int B = R / A;
    const double* C = (R == 6) ? kCos6 : (R == 9) ? kCos9 : (R == 10) ? kCos10 : (R == 12) ? kCos12
                    : (R == 14) ? kCos14 : (R == 15) ? kCos15 : kCos16;
    const double* S = (R == 6) ? kSin6 : (R == 9) ? kSin9 : (R == 10) ? kSin10 : (R == 12) ? kSin12
                    : (R == 14) ? kSin14 : (R == 15) ? kSin15 : kSin16;
#pragma unroll
    for (int n2 = 0; n2 < B; ++n2) {
      double2 u[A];
#pragma unroll
      for (int n1 = 0; n1 < A; ++n1) u[n1] = x[B * n1 + n2];
      dft_small<A, INV>(u);
#pragma unroll
      for (int k1 = 0; k1 < A; ++k1) {
        const int q = (n2 * k1) % R;
        double2 t = u[k1];
        // e^{-+ 2 pi i q / R}; quarter and half turns and odd eighths are done without full products
        if (q == 0) {
        } else if (2 * q == R) {
          t = make_double2(-t.x, -t.y);
        } else if (4 * q == R) {
          t = mul_mi<INV>(t);
        } else if (4 * q == 3 * R) {
          t = mul_mi<!INV>(t);
        } else if (8 * q == R || 8 * q == 3 * R || 8 * q == 5 * R || 8 * q == 7 * R) {
          const double h = 0.70710678118654752440;                // (c, s) = (+-h, +-h)
          const double c = (8 * q == R || 8 * q == 7 * R) ? h : -h;
          const double sn = (8 * q < 4 * R) ? -h : h;             // forward sine sign: -sin(2 pi q / R)
          const double s = INV ? -sn : sn;
          t = c == s ? make_double2(c * (t.x - t.y), c * (t.x + t.y)) : make_double2(c * (t.x + t.y), c * (t.y - t.x));
        } else {
          const double c = C[q], s = INV ? S[q] : -S[q];
          t = make_double2(t.x * c - t.y * s, t.x * s + t.y * c);
        }
        x[B * k1 + n2] = t;
      }
    }
    double2 y[R];
#pragma unroll
    for (int k1 = 0; k1 < A; ++k1) {
      double2 w[B];
#pragma unroll
      for (int n2 = 0; n2 < B; ++n2) w[n2] = x[B * k1 + n2];
      dft_small<B, INV>(w);
#pragma unroll
      for (int k2 = 0; k2 < B; ++k2) y[k1 + A * k2] = w[k2];
    }
#pragma unroll
    for (int k = 0; k < R; ++k) x[k] = y[k];
  }
}

// Per-pass base twiddles (precomputed once per plan for every FFT size, exact index) are copied
// into shared memory next to the data: base[n1] = e^{-2 pi i n1 / S} for n1 < Q = S/R; the
// butterfly forms e^{-2 pi i n1 k / S} = base^k by repeated products (error ~k ulp, k < 8).
// Two butterflies per loop trip with all loads issued before any store (ILP across the
// shared-memory latency).
template <int R, bool INV>
__device__ __forceinline__ void bfly_load(const double2* x, int base, int Q, double2 (&v)[R]) {
#pragma unroll
  for (int n = 0; n < R; ++n) v[n] = x[base + Q * n];
}

// w[k] = b^k for 1 <= k < R by a product tree: w[2^j] = w[2^(j-1)]^2, w[2^j + i] = w[2^j] w[i] -- the same
// R - 2 products as a running power, dependency depth ceil(log2 R) instead of R - 2 (and error ~log2 k ulp)
template <int R>
__device__ __forceinline__ void twiddle_powers(double2 b, double2 (&w)[R]) {
  w[0] = make_double2(1.0, 0.0);
  if constexpr (R > 1) w[1] = b;
#pragma unroll
  for (int k = 2; k < R; ++k) {
    int hi = 1;
    while (2 * hi <= k) hi *= 2;
    w[k] = hi == k ? cmulx(w[k / 2], w[k / 2]) : cmulx(w[hi], w[k - hi]);
  }
}

template <int R, bool INV, bool ZT = false>
__device__ __forceinline__ void bfly_finish(double2* x, int base, int Q, double2 b, double2 (&v)[R], int nz = 0) {
  double2 w[R];
  twiddle_powers<R>(b, w);
  if (!INV) {
    dft_small<R, false>(v);
    x[base] = v[0];
#pragma unroll
    for (int k = 1; k < R; ++k) x[base + Q * k] = cmulx(v[k], w[k]);
  } else {
#pragma unroll
    for (int k = 1; k < R; ++k) v[k] = cmulconj(v[k], w[k]);
    dft_small<R, true>(v);
#pragma unroll
    for (int n = 0; n < R; ++n)
      if (!ZT || base + Q * n < nz) x[base + Q * n] = v[n];   // ZT (last DIT pass): outputs >= nz are not needed
  }
}

// ZT, forward: the first DIF pass of a zero-padded input -- points at index >= nz are zero and are neither stored
// by the load phase nor read here (the pass writes every point, so the buffer needs no zero fill).
// ZT, inverse: the last DIT pass stores only the outputs below nz (the Bluestein result needs b < p)
template <int R, bool INV, bool ZT = false>
__device__ __forceinline__ void pass_loop(double2* x, int M, int S, const double2* __restrict__ tb, int nz = 0) {
  const int Q = S / R;
  const int nb = M / R;
  for (int bi = threadIdx.x; bi < nb; bi += blockDim.x) {
    const int blk = bi / Q, n1 = bi - blk * Q;
    const int base = blk * S + n1;
    double2 v[R];
    if (ZT && !INV) {
#pragma unroll
      for (int n = 0; n < R; ++n) v[n] = base + Q * n < nz ? x[base + Q * n] : make_double2(0.0, 0.0);
    } else {
      bfly_load<R, INV>(x, base, Q, v);
    }
    bfly_finish<R, INV, ZT && INV>(x, base, Q, tb[n1], v, nz);
  }
}

// First DIF pass fused with the load of a discrete-log line (int8 exp-sum iterations, ksplit = 1): the butterfly
// of base n1 gathers its inputs h = n1 + Q n < p straight from the line (position f = log_g h, the h = 0 row at
// f = p - 1) times the chirp -- the products of the load phase's x[h] = line[f] chirp[h] (chirp[h] = chl[f]: one
// chirp_value) followed by the ZT first pass, up to the FMA contraction of the product into the butterfly, without
// the scattered shared-memory sweep and its barrier.
template <int R>
__device__ __forceinline__ void pass_loop_gather(double2* x, int M, int p, const double2* __restrict__ tb,
                                                 const double2* __restrict__ line, const double2* __restrict__ ch,
                                                 const int32_t* __restrict__ dlog) {
  const int Q = M / R;
  for (int n1 = threadIdx.x; n1 < Q; n1 += blockDim.x) {
    int f[R];
#pragma unroll
    for (int n = 0; n < R; ++n) {
      const int h = n1 + Q * n;
      f[n] = h < p ? (h ? __ldg(dlog + h) : p - 1) : -1;
    }
    double2 v[R];
#pragma unroll
    for (int n = 0; n < R; ++n)
      v[n] = f[n] >= 0 ? cmulx(line[f[n]], __ldg(ch + n1 + Q * n)) : make_double2(0.0, 0.0);
    bfly_finish<R, false>(x, n1, Q, tb[n1], v);
  }
}

// Warp-local pass: after the first passes of a DIF FFT the array splits into independent blocks (the butterflies
// of a pass with span S only touch one aligned block of S points).  Once the leading radices' product is a multiple
// of the warp count W, warp w owns the contiguous region [w Mw, (w + 1) Mw), Mw = M / W, and runs the remaining
// passes on it with __syncwarp only: the same butterflies with the same twiddles as pass_loop (bitwise identical
// results), no block barrier, and warps drift out of phase so that one warp's shared-memory loads / stores overlap
// another's FP64 butterflies.
template <int R, bool INV>
__device__ __forceinline__ void pass_loop_w(double2* xw, int Mw, int S, const double2* __restrict__ tb) {
  const int Q = S / R;
  const int nb = Mw / R;
  for (int bi = threadIdx.x & 31; bi < nb; bi += 32) {
    const int blk = bi / Q, n1 = bi - blk * Q;
    const int base = blk * S + n1;
    double2 v[R];
    bfly_load<R, INV>(xw, base, Q, v);
    bfly_finish<R, INV>(xw, base, Q, tb[n1], v);
  }
  __syncwarp();
}

template <bool INV, bool BIG>
__device__ void fft_pass_w(double2* xw, int Mw, int S, int R, const double2* tb) {
  if constexpr (BIG) {
    switch (R) {
      case 9: pass_loop_w<9, INV>(xw, Mw, S, tb); return;
      case 10: pass_loop_w<10, INV>(xw, Mw, S, tb); return;
      case 12: pass_loop_w<12, INV>(xw, Mw, S, tb); return;
      case 14: pass_loop_w<14, INV>(xw, Mw, S, tb); return;
      case 15: pass_loop_w<15, INV>(xw, Mw, S, tb); return;
      case 16: pass_loop_w<16, INV>(xw, Mw, S, tb); return;
    }
  }
  switch (R) {
    case 2: pass_loop_w<2, INV>(xw, Mw, S, tb); break;
    case 3: pass_loop_w<3, INV>(xw, Mw, S, tb); break;
    case 4: pass_loop_w<4, INV>(xw, Mw, S, tb); break;
    case 5: pass_loop_w<5, INV>(xw, Mw, S, tb); break;
    case 6: pass_loop_w<6, INV>(xw, Mw, S, tb); break;
    case 7: pass_loop_w<7, INV>(xw, Mw, S, tb); break;
    case 8: pass_loop_w<8, INV>(xw, Mw, S, tb); break;
  }
}

// first pass index from which every pass is warp-local: the smallest ps >= 1 whose leading radix product
// R_0 ... R_{ps-1} is a multiple of the warp count (npass: none)
__device__ __forceinline__ int warp_local_from(const DevParams& P, int fi) {
  if (blockDim.x & 31) return kMaxFftPasses;
  const int W = blockDim.x >> 5;
  const int8_t* radix = P.fft_radix + fi * kMaxFftPasses;
  const int npass = P.fft_npass[fi];
  int prod = radix[0];
  for (int ps = 1; ps < npass; ++ps) {
    if (prod % W == 0) return ps;
    prod *= radix[ps];
  }
  return kMaxFftPasses;
}

template <bool INV, bool BIG, bool ZT = false>
__device__ void fft_pass(double2* x, int M, int S, int R, const double2* tb, int nz = 0) {
  if constexpr (BIG) {
    switch (R) {
      case 6: pass_loop<6, INV, ZT>(x, M, S, tb, nz); __syncthreads(); return;
      case 9: pass_loop<9, INV, ZT>(x, M, S, tb, nz); __syncthreads(); return;
      case 10: pass_loop<10, INV, ZT>(x, M, S, tb, nz); __syncthreads(); return;
      case 12: pass_loop<12, INV, ZT>(x, M, S, tb, nz); __syncthreads(); return;
      case 14: pass_loop<14, INV, ZT>(x, M, S, tb, nz); __syncthreads(); return;
      case 15: pass_loop<15, INV, ZT>(x, M, S, tb, nz); __syncthreads(); return;
      case 16: pass_loop<16, INV, ZT>(x, M, S, tb, nz); __syncthreads(); return;
    }
  }
  switch (R) {
    case 2: pass_loop<2, INV, ZT>(x, M, S, tb, nz); break;
    case 3: pass_loop<3, INV, ZT>(x, M, S, tb, nz); break;
    case 4: pass_loop<4, INV, ZT>(x, M, S, tb, nz); break;
    case 5: pass_loop<5, INV, ZT>(x, M, S, tb, nz); break;
    case 6: pass_loop<6, INV, ZT>(x, M, S, tb, nz); break;
    case 7: pass_loop<7, INV, ZT>(x, M, S, tb, nz); break;
    case 8: pass_loop<8, INV, ZT>(x, M, S, tb, nz); break;
  }
  __syncthreads();
}

template <bool BIG>
__device__ void fft_first_gather(const DevParams& P, double2* x, int fi, const double2* tb, int p,
                                 const double2* __restrict__ line, const double2* __restrict__ ch,
                                 const int32_t* __restrict__ dlog) {
  const int M = P.fft_M[fi];
  const int R = P.fft_radix[fi * kMaxFftPasses];
  if constexpr (BIG) {
    switch (R) {
      case 6: pass_loop_gather<6>(x, M, p, tb, line, ch, dlog); __syncthreads(); return;
      case 9: pass_loop_gather<9>(x, M, p, tb, line, ch, dlog); __syncthreads(); return;
      case 10: pass_loop_gather<10>(x, M, p, tb, line, ch, dlog); __syncthreads(); return;
      case 12: pass_loop_gather<12>(x, M, p, tb, line, ch, dlog); __syncthreads(); return;
      case 14: pass_loop_gather<14>(x, M, p, tb, line, ch, dlog); __syncthreads(); return;
      case 15: pass_loop_gather<15>(x, M, p, tb, line, ch, dlog); __syncthreads(); return;
      case 16: pass_loop_gather<16>(x, M, p, tb, line, ch, dlog); __syncthreads(); return;
    }
  }
  switch (R) {
    case 2: pass_loop_gather<2>(x, M, p, tb, line, ch, dlog); break;
    case 3: pass_loop_gather<3>(x, M, p, tb, line, ch, dlog); break;
    case 4: pass_loop_gather<4>(x, M, p, tb, line, ch, dlog); break;
    case 5: pass_loop_gather<5>(x, M, p, tb, line, ch, dlog); break;
    case 6: pass_loop_gather<6>(x, M, p, tb, line, ch, dlog); break;
    case 7: pass_loop_gather<7>(x, M, p, tb, line, ch, dlog); break;
    case 8: pass_loop_gather<8>(x, M, p, tb, line, ch, dlog); break;
  }
  __syncthreads();
}

// copy the base-twiddle tables of FFT size fi into shared memory (after the data array)
__device__ void load_twiddles(const DevParams& P, int fi, double2* tb) {
  const int32_t* off = P.fft_tw_off + fi * kMaxFftPasses;
  const int npass = P.fft_npass[fi];
  const int n = off[npass] - off[0];
  const double2* src = P.fft_tw + off[0];
  for (int q = threadIdx.x; q < n; q += blockDim.x) tb[q] = src[q];
}

// Fused middle of the Bluestein convolution: the last DIF pass (S = R, Q = 1: contiguous groups of
// R, unit twiddles), the pointwise product with the kernel spectrum V and the first DIT pass (the
// same groups) in registers -- three shared-memory sweeps replaced by one.
template <int R, bool BIG>
__device__ __forceinline__ void mid_loop(double2* x, int M, const double2* __restrict__ V, const bool wl,
                                         const double2* __restrict__ VB = nullptr) {
  // U groups per trip with all their loads (shared x, global V -- L2-resident) issued first: the V loads are
  // latency-bound.  wl: warp w runs the groups of its region [w M/W, (w + 1) M/W) (warp-local passes); VB: the
  // spectrum blocked for this warp count, so that the lanes' loads of element k are consecutive (coalesced)
  constexpr int U = 1;
  if (VB) {
    const int Mw = M / (int)(blockDim.x >> 5), w = threadIdx.x >> 5, Gw = Mw / R;
    x += w * Mw;
    VB += w * Mw;
    for (int g = threadIdx.x & 31; g < Gw; g += 32) {
      double2 v[R], wv[R];
#pragma unroll
      for (int k = 0; k < R; ++k) {
        v[k] = x[g * R + k];
        wv[k] = __ldg(VB + k * Gw + g);
      }
      dft_small<R, false>(v);
#pragma unroll
      for (int k = 0; k < R; ++k) v[k] = cmulx(v[k], wv[k]);
      dft_small<R, true>(v);
#pragma unroll
      for (int k = 0; k < R; ++k) x[g * R + k] = v[k];
    }
    return;
  }
  int G = M / R, t0 = threadIdx.x, step = blockDim.x;
  if (wl) {
    const int Mw = M / (int)(blockDim.x >> 5), w = threadIdx.x >> 5;
    x += w * Mw;
    V += w * Mw;
    G = Mw / R;
    t0 = threadIdx.x & 31;
    step = 32;
  }
  for (int g0 = t0; g0 < G; g0 += U * step) {
    double2 v[U][R], w[U][R];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int g = g0 + u * step;
#pragma unroll
      for (int k = 0; k < R; ++k) {
        v[u][k] = g < G ? x[g * R + k] : make_double2(0.0, 0.0);
        w[u][k] = g < G ? __ldg(V + g * R + k) : make_double2(0.0, 0.0);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int g = g0 + u * step;
      dft_small<R, false>(v[u]);
#pragma unroll
      for (int k = 0; k < R; ++k) v[u][k] = cmulx(v[u][k], w[u][k]);
      dft_small<R, true>(v[u]);
      if (g < G) {
#pragma unroll
        for (int k = 0; k < R; ++k) x[g * R + k] = v[u][k];
      }
    }
  }
}

template <bool BIG, bool WL = false>
__device__ void fft_mid(const DevParams& P, double2* x, int fi, const double2* __restrict__ V, bool wl = false,
                        const double2* __restrict__ VB = nullptr) {
  if constexpr (!WL) wl = false;
  const int M = P.fft_M[fi];
  const int R = P.fft_radix[fi * kMaxFftPasses + P.fft_npass[fi] - 1];
  // the blocked copy only when this launch's warp count is the plan's (the fill blocked it for that count)
  if (!WL || !wl || P.fft_radix[fi * kMaxFftPasses + kFftVwSlot] != (int)(blockDim.x >> 5)) VB = nullptr;
  switch (R) {
    case 2: mid_loop<2, BIG>(x, M, V, wl, VB); break;
    case 3: mid_loop<3, BIG>(x, M, V, wl, VB); break;
    case 4: mid_loop<4, BIG>(x, M, V, wl, VB); break;
    case 5: mid_loop<5, BIG>(x, M, V, wl, VB); break;
    case 6: mid_loop<6, BIG>(x, M, V, wl, VB); break;
    case 7: mid_loop<7, BIG>(x, M, V, wl, VB); break;
    case 8: mid_loop<8, BIG>(x, M, V, wl, VB); break;
  }
  if constexpr (BIG) {
    switch (R) {
      case 9: mid_loop<9, BIG>(x, M, V, wl, VB); break;
      case 10: mid_loop<10, BIG>(x, M, V, wl, VB); break;
      case 12: mid_loop<12, BIG>(x, M, V, wl, VB); break;
      case 14: mid_loop<14, BIG>(x, M, V, wl, VB); break;
      case 15: mid_loop<15, BIG>(x, M, V, wl, VB); break;
      case 16: mid_loop<16, BIG>(x, M, V, wl, VB); break;
    }
  }
  if (wl) __syncwarp();
  else __syncthreads();
}

// forward DIF FFT, natural -> digit-reversed; tb = shared copy of this size's tables
template <bool BIG, bool WL = false>
// nz < M: only x[0, nz) holds data, the rest is implicit zero padding (never stored, see pass_loop ZT)
// WL: passes >= wl are warp-local (pass_loop_w); a warp-local last pass ends with a block barrier unless the
// caller continues on the warp's own region (skip_last: the fused middle)
// ps0 = 1: the first pass already ran (fft_first_gather)
__device__ void fft_dif(const DevParams& P, double2* x, int fi, const double2* tb, int skip_last = 0, int nz = -1,
                        int wl = kMaxFftPasses, int ps0 = 0) {
  if constexpr (!WL) wl = kMaxFftPasses;
  const int M = P.fft_M[fi];
  const int8_t* radix = P.fft_radix + fi * kMaxFftPasses;
  const int32_t* off = P.fft_tw_off + fi * kMaxFftPasses;
  const int npass = P.fft_npass[fi];
  int S = M;
  for (int ps = 0; ps < ps0; ++ps) S /= radix[ps];
  for (int ps = ps0; ps < npass - skip_last; ++ps) {
    const int R = radix[ps];
    if (ps == 0 && nz >= 0 && nz < M) fft_pass<false, BIG, true>(x, M, S, R, tb + (off[ps] - off[0]), nz);
    else if (WL && ps >= wl) {
      const int Mw = M / (int)(blockDim.x >> 5);
      fft_pass_w<false, BIG>(x + (threadIdx.x >> 5) * Mw, Mw, S, R, tb + (off[ps] - off[0]));
    } else fft_pass<false, BIG>(x, M, S, R, tb + (off[ps] - off[0]));
    S /= R;
  }
  if (WL && !skip_last && npass - 1 >= wl) __syncthreads();
}
// inverse (unnormalised, x M) DIT FFT, digit-reversed -> natural
template <bool BIG, bool WL = false>
// WL: passes >= wl are warp-local (they come first in DIT order); a block barrier follows the last of them
__device__ void fft_dit(const DevParams& P, double2* x, int fi, const double2* tb, int skip_first = 0, int nz = -1,
                        int wl = kMaxFftPasses) {
  if constexpr (!WL) wl = kMaxFftPasses;
  const int M = P.fft_M[fi];
  const int8_t* radix = P.fft_radix + fi * kMaxFftPasses;
  const int32_t* off = P.fft_tw_off + fi * kMaxFftPasses;
  const int npass = P.fft_npass[fi];
  int S = 1;
  for (int ps = npass - 1; ps >= 0; --ps) {
    const int R = radix[ps];
    S *= R;
    if (ps == npass - 1 && skip_first) continue;
    if (WL && ps == wl - 1) __syncthreads();         // the first block-wide pass after the warp-local ones
    if (ps == 0 && nz >= 0 && nz < M) fft_pass<true, BIG, true>(x, M, S, R, tb + (off[ps] - off[0]), nz);
    else if (WL && ps >= wl) {
      const int Mw = M / (int)(blockDim.x >> 5);
      fft_pass_w<true, BIG>(x + (threadIdx.x >> 5) * Mw, Mw, S, R, tb + (off[ps] - off[0]));
    } else fft_pass<true, BIG>(x, M, S, R, tb + (off[ps] - off[0]));
  }
}

__device__ int find_fft_index(const DevParams& P, int p) {
  const int need = 2 * p - 1;
  int lo = 0, hi = P.n_fft - 1;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (P.fft_M[mid] >= need) hi = mid; else lo = mid + 1;
  }
  return lo;
}

// one segment of the base-twiddle tables: e^{-2 pi i n1 / S} for n1 < S/R
__global__ void fft_twiddle_kernel(double2* __restrict__ tw, const int4* __restrict__ seg) {
  const int4 g = seg[blockIdx.x];            // (offset, S, R, unused)
  const int S = g.y, R = g.z, Q = S / R;
  for (int n1 = threadIdx.x; n1 < Q; n1 += blockDim.x) {
    double s, c;
    sincospi(-2.0 * (double)n1 / (double)S, &s, &c);
    tw[g.x + n1] = make_double2(c, s);
  }
}

cudaError_t launch_fft_twiddles(double2* tw, const int4* seg, int n_seg, cudaStream_t st) {
  if (n_seg > 0) fft_twiddle_kernel<<<n_seg, 256, 0, st>>>(tw, seg);
  return cudaGetLastError();
}

__device__ __forceinline__ double2 chirp_value(int64_t q, int64_t p) {
  // e^{-pi i (q^2 mod 2p) / p}
  const int64_t e = (q * q) % (2 * p);
  double s, c;
  sincospi((double)e / (double)p, &s, &c);
  return make_double2(c, -s);
}

// ---- discrete-log row order of the int8-limb exp-sum (reading R22) ----
__device__ __forceinline__ uint32_t mulmod32(uint32_t a, uint32_t b, uint32_t p) { return (uint32_t)(((uint64_t)a * b) % p); }
__device__ uint32_t powmod32(uint32_t g, uint32_t e, uint32_t p) {
  uint32_t r = 1 % p;
  while (e) {
    if (e & 1) r = mulmod32(r, g, p);
    g = mulmod32(g, g, p);
    e >>= 1;
  }
  return r;
}
// smallest primitive root of the prime p: g^((p-1)/q) != 1 for every prime factor q of p - 1
__device__ uint32_t primitive_root(uint32_t p) {
  if (p == 2) return 1;
  uint32_t f[16];
  int nf = 0;
  uint32_t n = p - 1;
  for (uint32_t q = 2; q * q <= n; ++q)
    if (n % q == 0) {
      f[nf++] = q;
      while (n % q == 0) n /= q;
    }
  if (n > 1) f[nf++] = n;
  for (uint32_t g = 2; g < p; ++g) {
    bool ok = true;
    for (int i = 0; i < nf && ok; ++i) ok = powmod32(g, (p - 1) / f[i], p) != 1;
    if (ok) return g;
  }
  return 1;
}
// Tables of the discrete-log row order (reading R22): T[f] = T[f + p - 1] = limbs of W_p[g^f] (f < p-1, stored
// twice so row f + e_j needs no wrap), T[2(p-1)] = limbs of W_p[0] = 1; pw[f] = g^f (pw[p-1] = 0: the h = 0
// row); e_j = log_g u_j of the iteration's terms, -1 for u_j = 0 and for the padding up to a multiple of 16.
__device__ void i8_log_tables(const DevParams& P, int slot, int p) {
  __shared__ uint32_t s_g;
  if (threadIdx.x == 0) s_g = primitive_root((uint32_t)p);
  __syncthreads();
  const uint32_t g = s_g, n1 = (uint32_t)p - 1;
  const int64_t base = (int64_t)slot * P.i8_tstride;
  const uint32_t per = (n1 + blockDim.x - 1) / blockDim.x;
  const uint32_t f0 = threadIdx.x * per;
  uint32_t x = f0 < n1 ? powmod32(g, f0, (uint32_t)p) : 0;
  for (uint32_t f = f0; f < n1 && f < f0 + per; ++f) {
    P.i8_pw[base + f] = (int32_t)x;
    P.i8_dlog[base + x] = (int32_t)f;
    P.i8_chl[base + f] = chirp_value(x, p);
    double sn, cs;
    sincospi(2.0 * (double)x / (double)p, &sn, &cs);   // W_p[x] = e^{+2 pi i x / p}, exact rational argument
    if (P.i8_S > 0) {
      uint2 lo;
      uint32_t hi;
      i8_root_entry(cs, sn, P.i8_S, lo, hi);
      P.i8_tlo[base + f] = lo;
      P.i8_thi[base + f] = hi;
      P.i8_tlo[base + n1 + f] = lo;
      P.i8_thi[base + n1 + f] = hi;
    }
    if (P.dl_root) {
      P.dl_root[base + f] = make_double2(cs, sn);
      P.dl_root[base + n1 + f] = make_double2(cs, sn);
    }
    x = mulmod32(x, g, (uint32_t)p);
  }
  if (threadIdx.x == 0) {
    if (P.i8_S > 0) {
      uint2 lo;
      uint32_t hi;
      i8_root_entry(1.0, 0.0, P.i8_S, lo, hi);
      P.i8_tlo[base + 2 * n1] = lo;
      P.i8_thi[base + 2 * n1] = hi;
    }
    if (P.dl_root) P.dl_root[base + 2 * n1] = make_double2(1.0, 0.0);
    P.i8_pw[base + n1] = 0;
    P.i8_chl[base + n1] = chirp_value(0, p);
  }
}

__device__ __forceinline__ long long global_ns() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// spin until *flag == v; after 2 s (the scheduling assumption failed) flag the plan's error word and go on
// instead of hanging the GPU -- the execute then fails with SFFT_ECUDA
__device__ __forceinline__ void wait_stamp(const int32_t* flag, int32_t v, int32_t* err, int ns = 64) {
  int got;
  long long t0 = 0;
  for (int it = 0;; ++it) {
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(got) : "l"(flag) : "memory");
    if (got == v) return;
    if ((it & 255) == 0) {
      const long long t = global_ns();
      if (it == 0) t0 = t;
      else if (t - t0 > 2000000000ll) { atomicExch(err, 1); return; }
    }
    __nanosleep(ns);
  }
}


// ---- table cache: slot assignment (one CTA) ----
// Hits reuse their slot; the distinct missing primes get slots not used in this epoch (at most n_active slots
// are in use, the cache has n_active + 16 or more), which are queued in fill[] for tables_fill.  The primes of
// the slots are looked up through a shared-memory hash map (prime -> slot) built at entry, O(1) per signal.
__device__ __forceinline__ int tab_hash(int p, int mask) { return (int)(((uint32_t)p * 2654435761u) >> 7) & mask; }

// sm: 2 HS + 2 * 2048 + C ints (HS = power of two >= max(2048, 2C)).  fillers: also record, for every slot
// refilled in this epoch, the lowest active index whose signal uses the prime (the CTA that fills it in
// prep_iter_kernel: every other user has a higher block index)
__device__ void assign_slots(const DevParams& P, int32_t epoch, int* sm, bool fillers) {
  const int C = P.n_tslots;
  int HS = 2048;
  while (HS < 2 * C) HS <<= 1;
  const int hm = HS - 1;
  int* mk = sm;                                      // [HS] map keys: prime of a slot (0 = empty)
  int* mv = mk + HS;                                 // [HS] map values: slot
  int* hkey = mv + HS;                               // [2048] hash of missing primes
  int* hidx = hkey + 2048;                           // [2048] their rank
  int* ep = hidx + 2048;                             // [C] slot epochs (victim choice)
  int* hfill = ep + C;                               // [2048] lowest active index using the missing prime
  __shared__ int n_miss, n_free;
  const int n_active = P.ctrl[0];
  if (P.ctrl_next && threadIdx.x < 8) P.ctrl_next[threadIdx.x] = 0;   // the next iteration's control block
  for (int i = threadIdx.x; i < HS; i += blockDim.x) mk[i] = 0;
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) { hkey[i] = 0; hfill[i] = 0x7fffffff; }
  if (threadIdx.x == 0) { n_miss = 0; n_free = 0; }
  __syncthreads();
  for (int i = threadIdx.x; i < C; i += blockDim.x) {
    const int p = P.slot_p[i];
    if (p == 0) continue;
    int h = tab_hash(p, hm);
    while (atomicCAS(&mk[h], 0, p) != 0) h = (h + 1) & hm;        // each prime occupies at most one slot
    mv[h] = i;
  }
  __syncthreads();
  auto lookup = [&](int p) -> int {
    for (int h = tab_hash(p, hm);; h = (h + 1) & hm) {
      const int k = mk[h];
      if (k == p) return mv[h];
      if (k == 0) return -1;
    }
  };
  for (int a = threadIdx.x; a < n_active; a += blockDim.x) {
    const int s = P.active[a];
    const int p = P.st_p[s];
    const int hit = lookup(p);
    if (hit >= 0) {
      P.st_slot[s] = hit;
      P.slot_epoch[hit] = epoch;
    } else {
      int h = (p * 40503) & 2047;
      for (;;) {
        const int old = atomicCAS(&hkey[h], 0, p);
        if (old == 0) { hidx[h] = atomicAdd(&n_miss, 1); break; }
        if (old == p) break;
        h = (h + 1) & 2047;
      }
      atomicMin(&hfill[h], a);
    }
  }
  __syncthreads();
  // victims for the missing primes: least recently used first (empty slots have epoch -1), ties -> lower index;
  // warp 0 picks them one by one (deterministic; n_miss is 0 in the steady state)
  if (threadIdx.x < 32 && n_miss > 0) {
    for (int i = threadIdx.x; i < C; i += 32) ep[i] = P.slot_epoch[i];
    __syncwarp();
    int got = 0;
    for (; got < n_miss; ++got) {
      int best = 0x7fffffff, bi = -1;
      for (int i = threadIdx.x; i < C; i += 32)
        if (ep[i] != epoch && ep[i] < best) { best = ep[i]; bi = i; }
      for (int o = 16; o; o >>= 1) {
        const int ob = __shfl_xor_sync(0xffffffffu, best, o), oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ob < best || (ob == best && oi >= 0 && (bi < 0 || oi < bi))) { best = ob; bi = oi; }
      }
      if (bi < 0) break;
      if (threadIdx.x == 0) { P.fill[got] = bi; ep[bi] = epoch; }
      __syncwarp();
    }
    if (threadIdx.x == 0) n_free = got;
  }
  __syncthreads();
  if (n_miss == 0) {
    if (threadIdx.x == 0) P.ctrl[3] = 0;
    return;
  }
  // the filled slots: new primes into the map (the victims' old primes are not looked up in this epoch)
  for (int h = threadIdx.x; h < 2048; h += blockDim.x) {
    const int p = hkey[h];
    if (p == 0 || hidx[h] >= n_free) continue;
    const int slot = P.fill[hidx[h]];
    P.slot_p[slot] = p;
    P.slot_epoch[slot] = epoch;
    if (fillers) { P.fill_by[slot] = hfill[h]; P.fill_ep[slot] = epoch; }
    int g = tab_hash(p, hm);
    while (atomicCAS(&mk[g], 0, p) != 0) g = (g + 1) & hm;
    mv[g] = slot;
  }
  __syncthreads();
  for (int a = threadIdx.x; a < n_active; a += blockDim.x) {
    const int s = P.active[a];
    const int slot = lookup(P.st_p[s]);
    if (slot >= 0) P.st_slot[s] = slot;
  }
  if (threadIdx.x == 0) P.ctrl[3] = min(n_miss, n_free);
}

__global__ void __launch_bounds__(1024) tables_assign_kernel(DevParams P, int32_t epoch) {
  pdl_wait();
  extern __shared__ int sm[];
  assign_slots(P, epoch, sm, false);
}


// ---- per-signal term phases of the iteration: u_j = v_{j,m} mod p, 8 u_j mod p, e_j = log_g u_j ----
// cnt: >= p + 3k ints of shared memory; scratch: >= 32 ints.  phases: kTermsU (u_j and the bin sort; needs no
// table slot; u_j also kept in cnt[p + k ..)) | kTermsE (e_j, from the slot's discrete-log table; alone, it
// reads u_j from shared memory, or back from u_all when `u_smem` is false -- the table fill reused the smem)
constexpr int kTermsU = 1, kTermsE = 2;
__device__ void terms_body(const DevParams& P, int s, int* cnt, int* scratch, int phases = kTermsU | kTermsE,
                           bool u_smem = false) {
  const int p = P.st_p[s];
  if (!(phases & kTermsU)) {
    if (!P.log_tables) return;
    const int K = P.k + P.st_nR[s];
    const int Kp = (K + 15) & ~15;
    const int2* ug = P.u_all + (int64_t)s * P.kk;
    const int* us = cnt + p + P.k;
    const int64_t base = (int64_t)P.st_slot[s] * P.i8_tstride;
    int32_t* eg = P.i8_elog + (int64_t)s * P.i8_estride;
    for (int j = threadIdx.x; j < Kp; j += blockDim.x) {
      const int u = j < K ? (u_smem ? us[j] : ug[j].x) : 0;
      eg[j] = u ? P.i8_dlog[base + u] : -1;
    }
    return;
  }
  if (threadIdx.x == 0) P.st_M[s] = find_fft_index(P, p);
  const int m = P.st_m[s];
  const int K = P.k + P.st_nR[s];
  const int64_t* vm = P.v_all + ((int64_t)s * P.r + m) * P.kk;
  int2* ug = P.u_all + (int64_t)s * P.kk;
  const int Kp = (K + 15) & ~15;
  const int64_t base = (int64_t)P.st_slot[s] * P.i8_tstride;
  int32_t* eg = P.log_tables && (phases & kTermsE) ? P.i8_elog + (int64_t)s * P.i8_estride : nullptr;
  int* ub = cnt + p;                                 // [nR] bins of the registry entries (smem copy)
  int* us = cnt + p + P.k;                           // [K] u_j (smem copy for a later kTermsE pass)
  for (int j = threadIdx.x; j < (eg ? Kp : K); j += blockDim.x) {
    const int u = j < K ? (int)mod_pos64(vm[j], p) : 0;
    if (j < K) { ug[j] = make_int2(u, (8 * u) % p); us[j] = u; }
    if (j >= P.k && j < K) ub[j - P.k] = u;
    // e_j: -1 for u_j = 0 and for the padding up to a multiple of 16 (reading R22)
    if (eg) eg[j] = u ? P.i8_dlog[base + u] : -1;
  }
  // the FP64 exp-sum stages the phases in 16-byte pairs: the partner of the last term must be a valid index
  if (threadIdx.x == 0 && (K & 1)) ug[K] = make_int2(0, 0);
  // registry entries grouped by their bin u_e (bin-domain residual, reading R21): counting sort, stable in e
  const int nR = P.st_nR[s];
  if (P.literal || nR == 0) return;
  int32_t* bstart = P.bin_start + (int64_t)s * (P.p_stride + 1);
  int32_t* border = P.bin_order + (int64_t)s * P.k;
  for (int b = threadIdx.x; b < p; b += blockDim.x) cnt[b] = 0;
  __syncthreads();
  for (int e = threadIdx.x; e < nR; e += blockDim.x) atomicAdd(&cnt[ub[e]], 1);
  __syncthreads();
  {
    const int per = (p + blockDim.x - 1) / blockDim.x;
    const int b0 = threadIdx.x * per, b1 = min(p, b0 + per);
    int c0 = 0;
    for (int b = b0; b < b1; ++b) c0 += cnt[b];
    int tot;
    int run = block_excl_scan(c0, scratch, &tot);
    for (int b = b0; b < b1; ++b) { const int c = cnt[b]; bstart[b] = run; cnt[b] = run; run += c; }
    if (threadIdx.x == 0) bstart[p] = nR;
    __syncthreads();
  }
  if (threadIdx.x < 32) {                            // stable placement, 32 entries at a time
    const int lane = threadIdx.x;
    for (int e0 = 0; e0 < nR; e0 += 32) {
      const int e = e0 + lane;
      const int b = e < nR ? ub[e] : -1 - lane;
      const unsigned peers = __match_any_sync(0xffffffffu, b);
      const int rank = __popc(peers & ((1u << lane) - 1u));
      int base = 0;
      if (e < nR) base = cnt[b];
      __syncwarp();
      if (e < nR) {
        border[base + rank] = e;
        if (rank == __popc(peers) - 1) cnt[b] = base + rank + 1;
      }
      __syncwarp();
    }
  }
}

__global__ void terms_kernel(DevParams P, int32_t direct) {
  pdl_wait();
  if (!direct && (int)blockIdx.x >= P.ctrl[0]) return;   // grid sized before the host read n_active
  extern __shared__ int cnt[];                       // [p]: entries per bin, then the running end; [nR] bins; [K] u
  __shared__ int scratch[32];
  terms_body(P, P.active[blockIdx.x], cnt, scratch);
}

// per active signal: expsum root table, Bluestein chirp and the kernel spectrum for its prime
// BIG: sizes >= 4096 whose plans use in-register radices up to 16 (512 threads, 128 registers);
// small sizes use radices <= 8 with 64 registers so that several CTAs share an SM.
// tables of prime p into cache slot `slot`: W_p roots, Bluestein chirp, kernel spectrum V = DIF(conj chirp)/M,
// int8 root tables in discrete-log order; smem: the FFT buffer of size M and its twiddles
template <bool BIG>
__device__ void fill_tables(const DevParams& P, int slot, int p, unsigned char* smem_raw) {
  const int fi = find_fft_index(P, p);
  const int M = P.fft_M[fi];
  double2* x = reinterpret_cast<double2*>(smem_raw);
  double2* tb = x + M;
  load_twiddles(P, fi, tb);
  double2* W = P.W_tab + (int64_t)slot * P.p_stride;
  double2* ch = P.chirp + (int64_t)slot * P.p_stride;
  for (int q = threadIdx.x; q < M; q += blockDim.x) x[q] = make_double2(0.0, 0.0);
  __syncthreads();
  for (int q = threadIdx.x; q < p; q += blockDim.x) {
    double sn, cs;
    sincospi(2.0 * (double)q / (double)p, &sn, &cs);   // e^{+2 pi i q/p}
    W[q] = make_double2(cs, sn);
    const double2 w = chirp_value(q, p);
    ch[q] = w;
    const double2 vq = make_double2(w.x, -w.y);        // conj(w[q]) = kernel value at +-q
    x[q] = vq;
    if (q > 0) x[M - q] = vq;
  }
  if (P.log_tables) i8_log_tables(P, slot, p);
  __syncthreads();
  fft_dif<BIG>(P, x, fi, tb);
  const double inv = 1.0 / (double)M;
  double2* V = P.V + (int64_t)slot * P.M_stride;
  for (int q = threadIdx.x; q < M; q += blockDim.x) V[q] = cscale(x[q], inv);
  const int vw = P.fft_radix[fi * kMaxFftPasses + kFftVwSlot];
  if (vw && P.VB) {
    // warp-blocked copy for the warp-local middle (kFftVwSlot): element k of group g of warp region w
    const int R = P.fft_radix[fi * kMaxFftPasses + P.fft_npass[fi] - 1], Mt = M / vw, Gt = Mt / R;
    double2* VB = P.VB + (int64_t)slot * P.M_stride;
    for (int q = threadIdx.x; q < M; q += blockDim.x) {
      const int w = q / Mt, rr = q - w * Mt, g = rr / R, k = rr - g * R;
      VB[w * Mt + k * Gt + g] = cscale(x[q], inv);
    }
  }
}

// stage entry points (direct): the tables of every listed signal's prime; else the queued fills of the iteration
template <bool BIG>
__global__ void __launch_bounds__(BIG ? 512 : 1024, 1) fft_prep_kernel(DevParams P, int32_t direct) {
  pdl_wait();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  if (direct) {
    const int s = P.active[blockIdx.x];
    fill_tables<BIG>(P, P.st_slot[s], P.st_p[s], smem_raw);
    return;
  }
  // the queued fills of this iteration (a device-side count, usually 0 once the cache is warm): a grid of at most
  // one wave of these large-smem CTAs loops over them -- a grid of one CTA per active signal would spend several
  // waves of empty CTAs (C2, 1024 signals: ~20 us per iteration)
  const int n_fill = P.ctrl[3];
  for (int f = blockIdx.x; f < n_fill; f += gridDim.x) {
    const int slot = P.fill[f];
    fill_tables<BIG>(P, slot, P.slot_p[slot], smem_raw);
    __syncthreads();
  }
}

// One kernel per iteration for the table prep (CTA per active-signal slot of the previous count): CTA 0 maps
// the primes to cache slots and releases a stamp; every CTA then fills its prime's slot if it is the filler
// (lowest active index using the prime) and releases the slot's stamp, or waits for that stamp (the filler
// has a lower block index: resident or finished -- the decoupled look-back progress argument); then the
// signal's terms.  Replaces tables_assign + fft_prep + terms launches.
__device__ __forceinline__ void release_stamp(int32_t* flag, int32_t v) {
  __threadfence();
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(flag), "r"(v) : "memory");
}

template <bool BIG>
__global__ void __launch_bounds__(BIG ? 512 : 1024, 1) prep_iter_kernel(DevParams P, int32_t epoch) {
  pdl_wait();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int scratch[32];
  // CTA 0 assigns the slots; meanwhile the others do the slot-independent half of their terms
  const int a = blockIdx.x;
  if (a == 0) {
    assign_slots(P, epoch, reinterpret_cast<int*>(smem_raw), true);
    __syncthreads();
    if (threadIdx.x == 0) release_stamp(P.assign_ready, epoch);
    __syncthreads();
  }
  if (a >= P.ctrl[0]) return;
  const int s = P.active[a];
  terms_body(P, s, reinterpret_cast<int*>(smem_raw), scratch, kTermsU);
  if (a > 0 && threadIdx.x == 0) wait_stamp(P.assign_ready, epoch, P.spin_err);
  __syncthreads();
  const int slot = P.st_slot[s];
  bool filled = false;
  if (P.fill_ep[slot] == epoch) {
    if (P.fill_by[slot] == a) {
      filled = true;                                 // the FFT buffer overwrites the smem copy of u_j
      fill_tables<BIG>(P, slot, P.st_p[s], smem_raw);
      __syncthreads();
      if (threadIdx.x == 0) release_stamp(P.slot_ready + slot, epoch);
    } else if (threadIdx.x == 0) {
      wait_stamp(P.slot_ready + slot, epoch, P.spin_err);
    }
    __syncthreads();
  }
  terms_body(P, s, reinterpret_cast<int*>(smem_raw), scratch, kTermsE, !filled);
}


// ---- fused decode epilogue: no HBM round trip of the lines n >= 1 ----
// line-0 CTA: F_0[b] = chirp[b] conv[b] + registry bins (reading R21), kept in shared memory; select (a5) the
// candidates, publish them with F_0 at the candidates (the commit's a = F_0[b] / p) and pass flags = 1, then
// release sel_ready[s] = it_epoch
__device__ void fused_select(const DevParams& P, int s, int p, double2* x, const double2* __restrict__ ch,
                             double2* line) {
  const int tid = threadIdx.x;
  const int nR = P.st_nR[s];
  const bool resid = !P.literal && nR > 0;
  const double pd = (double)p;
  const int32_t* bstart = P.bin_start + (int64_t)s * (P.p_stride + 1);
  const int32_t* border = P.bin_order + (int64_t)s * P.k;
  const double2* Creg = P.C_all + ((int64_t)s * P.kk + P.k) * P.Lp;
  for (int b0 = tid; b0 < p; b0 += 4 * blockDim.x) {
    double2 c[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int b = b0 + u * blockDim.x;
      c[u] = b < p ? __ldg(ch + b) : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int b = b0 + u * blockDim.x;
      if (b < p) {
        double2 f = cmulx(x[b], c[u]);
        if (resid) f = add_bin_residual(f, bstart, border, Creg, P.Lp, 0, b, pd);
        x[b] = f;
      }
    }
  }
  __syncthreads();
  // x[p ..) is free after the transform: mag[p] double, cand[p], flag[p], scratch[32] (smem budget: radix_plan)
  double* mag = reinterpret_cast<double*>(x + p);
  int* cand = reinterpret_cast<int*>(mag + p);
  int* flag = cand + p;
  int* scratch = flag + p;
  const int nc = select_candidates([&](int b) { return x[b]; }, p, P.k - nR, P.floor_rel * pd, cand, mag, flag,
                                   scratch);
  int32_t* sendf = reinterpret_cast<int32_t*>(P.rec_send + (int64_t)s * P.rec_words);
  // distributed speculation (R26): the record's tail carries (nc, p, m), the bins and F_0 at them for the ranks
  int64_t* tail = P.spec_dist ? P.rec_send + (int64_t)s * P.rec_words + P.spec_tail : nullptr;
  for (int ci = tid; ci < nc; ci += blockDim.x) {
    const int b = cand[ci];
    P.rec_cand[(int64_t)s * P.k + ci] = b;
    P.rec_f0[(int64_t)s * P.k + ci] = x[b];
    if (P.peer_mode) peer_put_flag(P, s, ci, 1);
    else sendf[ci] = 1;
    if (tail) {
      reinterpret_cast<int32_t*>(tail + 2)[ci] = b;
      double* f0t = reinterpret_cast<double*>(tail + 2 + (P.k + 1) / 2);
      f0t[2 * ci] = x[b].x;
      f0t[2 * ci + 1] = x[b].y;
    }
  }
  if (tid == 0) {
    P.rec_nc[s] = nc;
    if (tail) {
      int32_t* h = reinterpret_cast<int32_t*>(tail);
      h[0] = nc;
      h[1] = p;
      h[2] = P.st_m[s];
    }
  }
  // fused exchange: the flags just stored in the peers' memory must land before the line-n CTAs' clears, which
  // follow their acquire of sel_ready -- every thread fences at system scope, the release is system scope
  if (P.peer_mode) __threadfence_system();
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    if (P.peer_mode)
      asm volatile("st.release.sys.global.b32 [%0], %1;" ::"l"(P.sel_ready + s), "r"(P.it_epoch) : "memory");
    else
      asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(P.sel_ready + s), "r"(P.it_epoch) : "memory");
  }
}

// line-n CTA (n >= 1 local line): after the line-0 CTA of the signal published, test + decode (a6) every
// candidate on this line: F_n[b] = chirp[b] conv[b] + registry bins, Eq. (42) ratio and Eq. (41) decode;
// a pass writes v into the record, a failure clears the candidate's flag (benign race: all writers store 0)
__device__ __forceinline__ void fused_test_wait(const DevParams& P, int s) {
  if (threadIdx.x == 0) wait_stamp(P.sel_ready + s, P.it_epoch, P.spin_err, 256);
  __syncthreads();
}
__device__ void fused_test(const DevParams& P, int s, int p, int n, const double2* x, const double2* __restrict__ ch) {
  const int tid = threadIdx.x;
  const int nR = P.st_nR[s];
  const bool resid = !P.literal && nR > 0;
  const double pd = (double)p;
  const int32_t* bstart = P.bin_start + (int64_t)s * (P.p_stride + 1);
  const int32_t* border = P.bin_order + (int64_t)s * P.k;
  const double2* Creg = P.C_all + ((int64_t)s * P.kk + P.k) * P.Lp;
  const int lvl = P.st_lvl[s];
  const int64_t Ev = P.lvl_E[lvl];
  const int ng = P.line_lo + n - 1;                       // reduced axis of the line
  const int64_t lo = P.lvl_lo[(int64_t)lvl * P.r + ng], hi = P.lvl_hi[(int64_t)lvl * P.r + ng];
  const int nc = *(volatile const int32_t*)(P.rec_nc + s);
  const int32_t* cand = P.rec_cand + (int64_t)s * P.k;
  const double2* f0s = P.rec_f0 + (int64_t)s * P.k;
  int32_t* sendf = reinterpret_cast<int32_t*>(P.rec_send + (int64_t)s * P.rec_words);
  int64_t* sendv = P.rec_send + (int64_t)s * P.rec_words + P.rec_fw + (int64_t)(n - 1) * P.k;
  for (int ci = tid; ci < nc; ci += blockDim.x) {
    const int b = cand[ci];
    double2 f = cmulx(x[b], __ldg(ch + b));
    if (resid) f = add_bin_residual(f, bstart, border, Creg, P.Lp, n, b, pd);
    int64_t v = 0;
    const bool pass = test_decode(f0s[ci], f, P.tol, Ev, P.round_tol, P.extra & 1, lo, hi, &v);
    if (P.peer_mode) {
      if (pass) peer_put_coord(P, s, n, ci, v);
      else peer_put_flag(P, s, ci, 0);
    } else {
      if (pass) sendv[ci] = v;
      else sendf[ci] = 0;
    }
  }
}

#ifdef SFFT_FFT_PROF
// tuning builds only: cycles per phase summed over the CTAs of pfft_kernel (thread 0's clock)
__device__ unsigned long long g_fft_prof[8];
#define FFT_PROF_MARK(i)                                                     \
  do {                                                                       \
    __syncthreads();                                                         \
    if (threadIdx.x == 0) {                                                  \
      const long long t_ = clock64();                                        \
      atomicAdd(&g_fft_prof[i], (unsigned long long)(t_ - prof_t0));         \
      prof_t0 = t_;                                                          \
    }                                                                        \
  } while (0)
#else
#define FFT_PROF_MARK(i) do {} while (0)
#endif

// one block per (signal, line): F = Bluestein DFT_p(s), in place in `lines`
// WL small sizes (M < fft_big_m) launch with at most 256 threads (two CTAs per SM, 128 registers)
template <bool BIG, bool WL>
__global__ void __launch_bounds__(BIG ? 512 : (WL ? 256 : 1024), BIG ? 1 : (WL ? 2 : 1))
pfft_kernel(DevParams P, int32_t n_lines, int32_t ksplit, const double2* __restrict__ part, int32_t p_part) {
  pdl_wait();
  extern __shared__ __align__(16) unsigned char smem_raw[];
#ifdef SFFT_FFT_PROF
  long long prof_t0 = clock64();
#endif
  // fused decode: CTAs [0, n_signals) are the line-0 CTAs (they select and publish the candidates), the
  // rest line n >= 1 of each signal; they wait for their signal's line-0 CTA, which has a lower block index
  // (already resident or finished when a later block starts: the forward-progress argument of decoupled
  // look-back scans)
  int slot, n;
  if (P.fuse_decode) {
    const int na = (int)gridDim.x / n_lines;
    if ((int)blockIdx.x < na) { slot = blockIdx.x; n = 0; }
    else { const int t = blockIdx.x - na; slot = t / (n_lines - 1); n = 1 + t % (n_lines - 1); }
  } else {
    slot = blockIdx.x / n_lines;
    n = blockIdx.x % n_lines;
  }
  const int s = P.active[slot];
  const int p = P.st_p[s];
  const int fi = P.st_M[s];
  const int M = P.fft_M[fi];
  double2* x = reinterpret_cast<double2*>(smem_raw);
  double2* tb = x + M;
  load_twiddles(P, fi, tb);
  const int tslot = P.st_slot[s];                     // table slot of the signal's prime
  const double2* ch = P.chirp + (int64_t)tslot * P.p_stride;
  double2* line = P.lines + ((int64_t)s * n_lines + n) * P.p_stride;
  const bool gather_first = M <= P.fused_load && P.lines_log && !P.fused_sample && ksplit == 1 && P.fft_npass[fi] >= 2;
  if (P.fused_sample) {
    // NEXT #3 fusion: this CTA samples its own line (Alg. 2 l.13-14; Eq. (41)) -- s_n[h] = sum_j C[j][n] W_p^{h u_j}
    // with rows f in discrete-log order (h = g^f, root of (f, j) = dl_root[f + e_j], W_p[0] = 1 for e_j < 0 and
    // for the h = 0 row) -- and multiplies by the chirp into the FFT buffer; the samples never leave shared memory.
    // shared memory after the FFT buffer and its twiddles: roots [2(p - 1) + 1], C column [K], e_j [K]
    const int K = P.k;
    const int ntw = P.fft_tw_off[fi * kMaxFftPasses + P.fft_npass[fi]] - P.fft_tw_off[fi * kMaxFftPasses];
    double2* sroot = tb + ((ntw + 1) & ~1);
    const int nroot = 2 * (p - 1) + 1;
    double2* scol = sroot + ((nroot + 1) & ~1);
    int* se = reinterpret_cast<int*>(scol + K);
    const double2* rsrc = P.dl_root + (int64_t)tslot * P.i8_tstride;
    for (int q = threadIdx.x; q < nroot; q += blockDim.x) sroot[q] = rsrc[q];
    const double2* Cs = P.C_all + (int64_t)s * P.kk * P.Lp + n;
    const int32_t* eg = P.i8_elog + (int64_t)s * P.i8_estride;
    for (int j = threadIdx.x; j < K; j += blockDim.x) {
      scol[j] = Cs[(int64_t)j * P.Lp];
      se[j] = eg[j];
    }
    __syncthreads();
    const int32_t* pw = P.i8_pw + (int64_t)tslot * P.i8_tstride;
    const double2* chl = P.i8_chl + (int64_t)tslot * P.i8_tstride;
    const int one = 2 * (p - 1);
    // two rows per thread and trip share the broadcast loads of e_j and C[j][n]; the h = 0 row (f = p - 1, every
    // root 1) takes the table's W_p[0] entry through e = -1 semantics: its index is forced to `one`
    for (int f0 = threadIdx.x; f0 < p; f0 += 2 * blockDim.x) {
      const int f1 = f0 + blockDim.x;
      const bool z0 = f0 == p - 1, z1 = f1 == p - 1, v1 = f1 < p;
      double ar0 = 0.0, ai0 = 0.0, ar1 = 0.0, ai1 = 0.0;
#pragma unroll 4
      for (int j = 0; j < K; ++j) {
        const int e = se[j];
        const double2 c = scol[j];
        const double2 w0 = sroot[(e < 0 || z0) ? one : f0 + e];
        const double2 w1 = sroot[(e < 0 || z1 || !v1) ? one : f1 + e];
        ar0 = fma(c.x, w0.x, fma(-c.y, w0.y, ar0));
        ai0 = fma(c.x, w0.y, fma(c.y, w0.x, ai0));
        ar1 = fma(c.x, w1.x, fma(-c.y, w1.y, ar1));
        ai1 = fma(c.x, w1.y, fma(c.y, w1.x, ai1));
      }
      x[__ldg(pw + f0)] = cmulx(make_double2(ar0, ai0), __ldg(chl + f0));
      if (v1) x[__ldg(pw + f1)] = cmulx(make_double2(ar1, ai1), __ldg(chl + f1));
    }
  } else if (gather_first) {
    // the first DIF pass gathers the line itself (below)
  } else if (P.lines_log) {
    // the int8 exp-sum wrote the samples in discrete-log order: position f holds h = pw[f]; all of a
    // thread's loads in flight (latency-bound phase), then the chirp products scattered
    const int32_t* pw = P.i8_pw + (int64_t)tslot * P.i8_tstride;
    const double2* chl = P.i8_chl + (int64_t)tslot * P.i8_tstride;
    const int n_slots = gridDim.x / n_lines;
    constexpr int U = BIG ? 8 : 4;
    for (int f0 = threadIdx.x; f0 < p; f0 += U * blockDim.x) {
      double2 v[U], c[U];
      int h[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int f = f0 + u * blockDim.x;
        h[u] = f < p ? __ldg(pw + f) : -1;
        c[u] = f < p ? __ldg(chl + f) : make_double2(0.0, 0.0);
        if (ksplit == 1) {
          v[u] = f < p ? line[f] : make_double2(0.0, 0.0);
        } else {
          v[u] = make_double2(0.0, 0.0);
          for (int ks = 0; ks < ksplit && f < p; ++ks) {
            const double2 t = part[(((int64_t)ks * n_slots + slot) * n_lines + n) * p_part + f];
            v[u].x += t.x;
            v[u].y += t.y;
          }
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (h[u] >= 0) x[h[u]] = cmulx(v[u], c[u]);
    }
  } else if (ksplit == 1) {
    // 4 independent loads in flight per thread (latency-bound phase)
    for (int q0 = threadIdx.x; q0 < p; q0 += 4 * blockDim.x) {
      double2 a[4], c[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int q = q0 + u * blockDim.x;
        a[u] = q < p ? line[q] : make_double2(0.0, 0.0);
        c[u] = q < p ? ch[q] : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int q = q0 + u * blockDim.x;
        if (q < p) x[q] = cmulx(a[u], c[u]);
      }
    }
  } else {
    // sum the exp-sum partials over the term splits in fixed order (deterministic)
    const int n_slots = gridDim.x / n_lines;
    for (int q = threadIdx.x; q < p; q += blockDim.x) {
      double2 v = make_double2(0.0, 0.0);
      for (int ks = 0; ks < ksplit; ++ks) {
        const double2 t = part[(((int64_t)ks * n_slots + slot) * n_lines + n) * p_part + q];
        v.x += t.x;
        v.y += t.y;
      }
      x[q] = cmulx(v, ch[q]);
    }
  }
  if (P.fft_npass[fi] <= 1)                           // a single-pass size has no DIF pass to treat the padding
    for (int q = p + threadIdx.x; q < M; q += blockDim.x) x[q] = make_double2(0.0, 0.0);
  __syncthreads();
  FFT_PROF_MARK(0);
  // warp-local from pass wl on (the middle included), unless disabled or the middle would not be warp-local
  // (WL instantiation: launched when the iteration's largest size qualifies; smaller sizes of the same launch fall
  // back to block-wide passes)
  int wl = kMaxFftPasses;
  if constexpr (WL) {
    wl = warp_local_from(P, fi);
    if (wl > P.fft_npass[fi] - 1) wl = kMaxFftPasses;
  }
  if (gather_first) fft_first_gather<BIG>(P, x, fi, tb, p, line, ch, P.i8_dlog + (int64_t)tslot * P.i8_tstride);
  fft_dif<BIG, WL>(P, x, fi, tb, 1, p, wl, gather_first ? 1 : 0);   // x[p, M) is implicit zero padding
  FFT_PROF_MARK(1);
  fft_mid<BIG, WL>(P, x, fi, P.V + (int64_t)tslot * P.M_stride, wl < kMaxFftPasses,
                   P.VB ? P.VB + (int64_t)tslot * P.M_stride : nullptr);
  FFT_PROF_MARK(2);
  fft_dit<BIG, WL>(P, x, fi, tb, 1, p, wl);           // only F[b], b < p, is used
  FFT_PROF_MARK(3);
  if (P.fuse_decode) {
    if (n == 0) {
      fused_select(P, s, p, x, ch, line);
      FFT_PROF_MARK(4);
    } else {
      fused_test_wait(P, s);
      FFT_PROF_MARK(5);
      fused_test(P, s, p, n, x, ch);
      FFT_PROF_MARK(6);
    }
    if (P.peer_mode) peer_release_line(P, s, n);
    if (P.fuse_commit) {
      // the last of the signal's n_lines CTAs to arrive commits it (a7): every thread fences its record
      // writes, thread 0 counts the arrival; the last one resets the counter for the next iteration
      __shared__ int last;
      __threadfence();
      __syncthreads();
      if (threadIdx.x == 0) {
        last = atomicAdd(P.commit_cnt + s, 1) == n_lines - 1;
        if (last) {
          P.commit_cnt[s] = 0;
          __threadfence();
        }
      }
      __syncthreads();
      if (last) commit_signal<false>(P, P.cur_iter, s, smem_raw);   // not with R26 (api.cu)
    }
    return;
  }
  // F[b] = w[b] * (conv)[b]: 4 chirp loads in flight per thread (the chirp is L2-resident, latency-bound)
  for (int b0 = threadIdx.x; b0 < p; b0 += 4 * blockDim.x) {
    double2 c[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int b = b0 + u * blockDim.x;
      c[u] = b < p ? __ldg(ch + b) : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int b = b0 + u * blockDim.x;
      if (b < p) line[b] = cmulx(x[b], c[u]);
    }
  }
  FFT_PROF_MARK(4);
}

#ifdef SFFT_FFT_PROF
cudaError_t fft_prof_read(unsigned long long* out, bool reset) {
  cudaError_t e = cudaMemcpyFromSymbol(out, g_fft_prof, sizeof(unsigned long long) * 8);
  if (e == cudaSuccess && reset) {
    unsigned long long z[8] = {0};
    e = cudaMemcpyToSymbol(g_fft_prof, z, sizeof z);
  }
  return e;
}
#endif

cudaError_t launch_prep_iter(const DevParams& P, int32_t n_bound, int32_t smem_bytes, cudaStream_t st, int32_t epoch) {
  if (n_bound <= 0) return cudaSuccess;
  size_t hs = 2048;
  while (hs < 2 * (size_t)P.n_tslots) hs <<= 1;
  const size_t smem = std::max<size_t>((size_t)smem_bytes,
                                       std::max(sizeof(int) * (2 * hs + 2 * 4096 + (size_t)P.n_tslots),
                                                sizeof(int) * ((size_t)P.p_stride + 3 * (size_t)P.k)));
  cudaError_t e = ensure_smem(prep_iter_kernel<true>, smem);
  if (e != cudaSuccess) return e;
  return launch_pdl(prep_iter_kernel<true>, dim3(n_bound), dim3(512), smem, st, P, epoch);
}

cudaError_t launch_fft_prep(const DevParams& P, int32_t n_signals, int32_t smem_bytes, int32_t threads, int32_t big,
                            cudaStream_t st, int32_t epoch, bool direct) {
  if (n_signals <= 0) return cudaSuccess;
  if (!direct) {
    size_t hs = 2048;
    while (hs < 2 * (size_t)P.n_tslots) hs <<= 1;
    const size_t sm = sizeof(int) * (2 * hs + 2 * 4096 + (size_t)P.n_tslots);
    cudaError_t e = ensure_smem(tables_assign_kernel, sm);
    if (e != cudaSuccess) return e;
    e = launch_pdl(tables_assign_kernel, dim3(1), dim3(1024), sm, st, P, epoch);
    if (e != cudaSuccess) return e;
  }
  const size_t smem = (size_t)smem_bytes;
  auto kern = big ? fft_prep_kernel<true> : fft_prep_kernel<false>;
  cudaError_t e = ensure_smem(kern, smem);
  if (e != cudaSuccess) return e;
  int n_sm = 148;
  {
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
  }
  const int fill_grid = direct ? n_signals : std::min(n_signals, n_sm);   // queued fills: one wave, looping
  e = launch_pdl(kern, dim3(fill_grid), dim3(threads), smem, st, P, direct ? 1 : 0);
  if (e != cudaSuccess) return e;
  e = ensure_smem(terms_kernel, sizeof(int) * ((size_t)P.p_stride + 3 * (size_t)P.k));
  if (e != cudaSuccess) return e;
  e = launch_pdl(terms_kernel, dim3(n_signals), dim3(256), sizeof(int) * ((size_t)P.p_stride + 3 * (size_t)P.k), st, P,
                 direct ? 1 : 0);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

cudaError_t launch_pfft(const DevParams& P, int32_t n_signals, int32_t n_lines, int32_t smem_bytes, int32_t threads,
                        int32_t big, int32_t ksplit, const double2* part, int32_t p_part, cudaStream_t st, bool wl) {
  const size_t smem = (size_t)smem_bytes;
  wl = wl && (big || threads <= 256);
  auto kern = big ? (wl ? pfft_kernel<true, true> : pfft_kernel<true, false>)
                  : (wl ? pfft_kernel<false, true> : pfft_kernel<false, false>);
  cudaError_t e = ensure_smem(kern, smem);
  if (e != cudaSuccess) return e;
  const long grid = (long)n_signals * n_lines;
  if (grid > 0) return launch_pdl(kern, dim3((unsigned)grid), dim3(threads), smem, st, P, n_lines, ksplit, part, p_part);
  return cudaGetLastError();
}

}  // namespace sfft
