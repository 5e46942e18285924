// k_expsum_i8.cu -- SURVEY 8(a) row a3 on the 5th-generation tensor cores: the exponential sum of
// one iteration (Algorithm 2 l.13-14; Eq. (41))
//
//   s_n[h] = sum_{j < K} C[j][n] * W_p[(h * u_j) mod p],   h in [0, p), n in [0, L)
//
// computed EXACTLY in integer arithmetic on fixed-point limbs, then combined in FP64.
//
// Fixed point.  A root component x in [-1, 1] is X = rint(x * 127 * 256^(S-1)) split into S balanced
// base-256 digits x_0 .. x_{S-1} (x_0 most significant, every digit in [-128, 127], |x_0| <= 127),
// so x = sum_s x_s 256^-s / 127 up to the rounding of X.  A line coefficient component y (of a
// signal whose largest coefficient component is sigma) is Y = rint(y / sigma * 127 * 256^(S-1)) split
// the same way.  Every limb product x_s y_t is an exact int8 x int8 -> int32 product and the int32
// sums over 2K operands (|sum| <= 2K * 127 * 128 < 2^31 for K < 65000) are exact, so
//
//   s = sigma / 127^2 * sum_{w < S} 256^-w * Acc_w,   Acc_w = sum_{s + t = w} sum_j x_s(h, j) y_t(j, n)
//
// with the products of weight w >= S dropped: the result differs from the exact sum of the
// FP64-rounded roots and coefficients by ~2 * 256^-S relative per product (S = 6: 7e-15), which the
// plan turns into a decode bound.  Complex arithmetic is a real GEMM over
// 2K x 2L: A'[h][2j] = Re W, A'[h][2j+1] = Im W; B'[2j][2n] = Re C, B'[2j+1][2n] = -Im C,
// B'[2j][2n+1] = Im C, B'[2j+1][2n+1] = Re C, so column 2n is Re s_n and column 2n+1 is Im s_n.
//
// B200 mapping (one CTA per 128 samples h x NT output columns x a range of 16-term K steps):
//   * A limbs (the roots, gathered per (h, j) from a p-entry limb table in shared memory) are
//     written by 4 generator warps straight into TMEM (tcgen05.st; TMEM lane = sample row), two
//     stages;
//   * B limbs (line coefficients, precomputed once per solve in the UMMA K-major layout) stream
//     through shared memory by 1-D bulk copies (TMA engine) on an mbarrier ring;
//   * one thread issues tcgen05.mma.kind::i8 (A from TMEM, B from smem, s32 accumulators in TMEM),
//     one accumulator per limb weight; weights that do not fit TMEM at once run in separate passes
//     (highest weights first) whose FP64 partials are added in the epilogue;
//   * the epilogue (same 4 warps) reads the accumulators with tcgen05.ld and writes complex128 lines.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "sfft_internal.cuh"
#include "tc_i8.cuh"

namespace sfft {

constexpr int kI8Rows = 128;          // MMA M
constexpr int kI8StepTerms = 16;      // terms per K step (32 int8 K elements: re and im)

// ------------------------------------------------------------------ B limbs (once per solve)
// sigma[s] = max over terms j < K and lines n < L of max(|Re C|, |Im C|)
__global__ void i8_sigma_kernel(DevParams P, int32_t K) {
  const int s = blockIdx.x;
  const double2* Cs = P.C_all + (int64_t)s * P.kk * P.Lp;
  double m = 0.0;
  for (int64_t e = threadIdx.x; e < (int64_t)K * P.L; e += blockDim.x) {
    const int j = (int)(e / P.L), n = (int)(e % P.L);
    const double2 c = Cs[(int64_t)j * P.Lp + n];
    m = fmax(m, fmax(fabs(c.x), fabs(c.y)));
  }
  for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  __shared__ double red[32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = fmax(m, red[w]);
    P.i8_sigma[s] = m > 0.0 ? m : 1.0;
  }
}

// balanced base-256 digits of X (|X| <= 127 * 256^(S-1)), most significant first
__device__ __forceinline__ void digits(int64_t X, int S, int (&d)[8]) {
  for (int t = S - 1; t >= 0; --t) {
    const int64_t r = ((X + 128) & 255) - 128;
    d[t] = (int)r;
    X = (X - r) >> 8;
  }
}

// One thread per (signal, n-tile, K step, output column, 4-byte K word): S words, one per limb.
__global__ void i8_limbs_kernel(DevParams P, int32_t K) {
  const int NT = P.i8_NT, S = P.i8_S;
  const int64_t per_step = (int64_t)NT * 8;                       // (column, K word) pairs
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t steps_all = (int64_t)P.i8_ntiles * P.i8_nks;
  const int64_t total = (int64_t)P.batch * steps_all * per_step;
  if (g >= total) return;
  const int e = (int)(g % per_step);
  const int64_t st = g / per_step;                               // (signal, ntile, kstep)
  const int ks = (int)(st % P.i8_nks);
  const int nt = (int)((st / P.i8_nks) % P.i8_ntiles);
  const int s = (int)(st / steps_all);
  const int col = e >> 3, kw = e & 7;                            // output column, K word (4 K elements)
  const int gc = nt * NT + col;
  const int n = gc >> 1, im_out = gc & 1;
  const double q = 127.0 * ldexp(1.0, 8 * (S - 1)) / P.i8_sigma[s];
  int dg[4][8];
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    const int kp = 4 * kw + b;                                   // K element in the step
    const int j = ks * kI8StepTerms + (kp >> 1);
    double v = 0.0;
    if (j < K && n < P.L) {
      const double2 c = P.C_all[((int64_t)s * P.kk + j) * P.Lp + n];
      const bool a_im = kp & 1;                                   // row 2j+1 multiplies Im W
      v = im_out ? (a_im ? c.x : c.y) : (a_im ? -c.y : c.x);
    }
    digits(llrint(v * q), S, dg[b]);
  }
  int8_t* base = P.i8_B + ((((int64_t)s * P.i8_ntiles + nt) * P.i8_nks + ks) * S) * (int64_t)NT * 32;
  const int off = (col >> 3) * 256 + (kw >> 2) * 128 + (col & 7) * 16 + (kw & 3) * 4;
  for (int t = 0; t < S; ++t) {
    const uint32_t w = (uint32_t)(uint8_t)dg[0][t] | ((uint32_t)(uint8_t)dg[1][t] << 8) |
                       ((uint32_t)(uint8_t)dg[2][t] << 16) | ((uint32_t)(uint8_t)dg[3][t] << 24);
    *reinterpret_cast<uint32_t*>(base + (int64_t)t * NT * 32 + off) = w;
  }
}

// ------------------------------------------------------------------ the exp-sum kernel
constexpr int kI8GenWarps = 8;        // 2 per TMEM lane quarter: warp g covers rows 32 (g % 4) .., terms 8 (g / 4) ..
constexpr int kI8MaxAStages = 8;
constexpr int kI8Threads = 32 * (kI8GenWarps + 2);   // + B producer warp + MMA warp
constexpr int kI8ProdWarp = kI8GenWarps, kI8MmaWarp = kI8GenWarps + 1;

struct I8Args {
  int32_t n_htiles, ksplit, p_part, nsb, npass;
  int32_t pass[4];            // wl | wh << 4 | nsa << 8 | a_base << 16 (TMEM column of A slot 0)
  uint32_t b_stage_bytes;     // S * NT * 32
  uint32_t tab_off, u_off;    // smem offsets of the limb tables and the u list
  int32_t dbg;                // tuning only (SFFT_I8_DBG): 1 conflict-free gathers, 2 no MMAs, 3 no A generation,
                              // 4 MMAs only (no copies, no generation)
};
__device__ __forceinline__ int pass_wl(int v) { return v & 15; }
__device__ __forceinline__ int pass_wh(int v) { return (v >> 4) & 15; }
__device__ __forceinline__ int pass_nsa(int v) { return (v >> 8) & 255; }
__device__ __forceinline__ int pass_abase(int v) { return v >> 16; }

// 8 terms (4 TMEM columns per limb) of one K step for this thread's row h
template <int NL>
__device__ __forceinline__ void gen_stage(uint32_t taddr, const int* __restrict__ sU, const uint2* __restrict__ sTlo,
                                          const uint32_t* __restrict__ sThi, unsigned h, unsigned magic, int p,
                                          int dbg) {
  uint32_t w[NL][4];
  unsigned q[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const unsigned x = h * (unsigned)sU[e];
    int r = (int)(x - __umulhi(x, magic) * (unsigned)p);
    r += (r >> 31) & p;
    q[e] = dbg == 1 ? (h + e) : (unsigned)r;
  }
  uint2 lo[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) lo[e] = sTlo[q[e]];
  uint32_t hi[8];
  if constexpr (NL > 4) {
#pragma unroll
    for (int e = 0; e < 8; ++e) hi[e] = sThi[q[e]];
  }
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const uint2 l0 = lo[2 * c], l1 = lo[2 * c + 1];
    w[0][c] = __byte_perm(l0.x, l1.x, 0x5410);
    if constexpr (NL > 1) w[1][c] = __byte_perm(l0.x, l1.x, 0x7632);
    if constexpr (NL > 2) w[2][c] = __byte_perm(l0.y, l1.y, 0x5410);
    if constexpr (NL > 3) w[3][c] = __byte_perm(l0.y, l1.y, 0x7632);
    if constexpr (NL > 4) {
      w[4][c] = __byte_perm(hi[2 * c], hi[2 * c + 1], 0x5410);
      if constexpr (NL > 5) w[5][c] = __byte_perm(hi[2 * c], hi[2 * c + 1], 0x7632);
    }
  }
#pragma unroll
  for (int t = 0; t < NL; ++t) tc::tmem_st4(taddr + 8 * t, w[t]);
}

// All limb products of one K step for the weights [WL, WH] of a pass, fully unrolled: accumulator of
// weight w at column (w - WL) NT, A limb s at a0 + 8 s, B limb t at descriptor bd0 + t * (NT * 32 / 16).
template <int WL, int WH>
__device__ __forceinline__ void issue_stage(uint32_t tbase, uint32_t a0, uint64_t bd0, uint32_t nt_cols, uint32_t nt_desc,
                                            uint32_t idesc, bool first_k) {
#pragma unroll
  for (int w = WL; w <= WH; ++w)
#pragma unroll
    for (int sl = 0; sl <= w; ++sl)
      tc::mma_i8_ts(tbase + (uint32_t)(w - WL) * nt_cols, a0 + 8 * sl, bd0 + (uint64_t)((w - sl) * nt_desc), idesc,
                    (!first_k || sl > 0) ? 1u : 0u);
}

__device__ __forceinline__ void issue_stage_rt(int wl, int wh, uint32_t tbase, uint32_t a0, uint64_t bd0,
                                               uint32_t nt_cols, uint32_t nt_desc, uint32_t idesc, bool first_k) {
#define SFFT_I8_CASE(a, b) \
  case a * 8 + b: issue_stage<a, b>(tbase, a0, bd0, nt_cols, nt_desc, idesc, first_k); break;
  switch (wl * 8 + wh) {
    SFFT_I8_CASE(0, 0) SFFT_I8_CASE(0, 1) SFFT_I8_CASE(0, 2) SFFT_I8_CASE(0, 3) SFFT_I8_CASE(0, 4) SFFT_I8_CASE(0, 5)
    SFFT_I8_CASE(1, 1) SFFT_I8_CASE(1, 2) SFFT_I8_CASE(1, 3) SFFT_I8_CASE(1, 4) SFFT_I8_CASE(1, 5)
    SFFT_I8_CASE(2, 2) SFFT_I8_CASE(2, 3) SFFT_I8_CASE(2, 4) SFFT_I8_CASE(2, 5)
    SFFT_I8_CASE(3, 3) SFFT_I8_CASE(3, 4) SFFT_I8_CASE(3, 5)
    SFFT_I8_CASE(4, 4) SFFT_I8_CASE(4, 5)
    SFFT_I8_CASE(5, 5)
    default: break;
  }
#undef SFFT_I8_CASE
}

__global__ void __launch_bounds__(kI8Threads, 1) expsum_i8_kernel(DevParams P, I8Args A, double2* part) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  uint64_t* bfull = reinterpret_cast<uint64_t*>(smem_raw);        // [4]
  uint64_t* bempty = bfull + 4;                                      // [4]
  uint64_t* afull = bfull + 8;                                       // [kI8MaxAStages]
  uint64_t* aempty = afull + kI8MaxAStages;                          // [kI8MaxAStages]
  uint64_t* accfull = aempty + kI8MaxAStages;
  uint64_t* accempty = accfull + 1;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(accempty + 1);
  int* spass = reinterpret_cast<int*>(tslot + 1);                   // [4]
  unsigned char* sB = smem_raw + 512;
  uint2* sTlo = reinterpret_cast<uint2*>(smem_raw + A.tab_off);
  const int NT = P.i8_NT, S = P.i8_S;

  int bid = blockIdx.x;
  const int ks_i = bid % A.ksplit;
  bid /= A.ksplit;
  const int nt = bid % P.i8_ntiles;
  bid /= P.i8_ntiles;
  const int ht = bid % A.n_htiles;
  const int slot = bid / A.n_htiles;
  const int s = P.active[slot];
  const int p = P.st_p[s];
  if (ht * kI8Rows >= p) return;
  const int K = P.i8_K;                                             // terms in the B limbs (bin-domain: k)
  const int nks = (K + kI8StepTerms - 1) / kI8StepTerms;
  const int per = (nks + A.ksplit - 1) / A.ksplit;
  const int ks_lo = ks_i * per, ks_hi = min(nks, ks_lo + per);
  const int nk = max(0, ks_hi - ks_lo);
  uint32_t* sThi = reinterpret_cast<uint32_t*>(sTlo + p);
  int* sU = reinterpret_cast<int*>(smem_raw + A.u_off);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == kI8MmaWarp) tc::tmem_alloc<512>(tslot);
  if (tid == 0) {
    for (int i = 0; i < 4; ++i) { tc::mbar_init(bfull + i, 1); tc::mbar_init(bempty + i, 1); }
    for (int i = 0; i < kI8MaxAStages; ++i) { tc::mbar_init(afull + i, kI8GenWarps); tc::mbar_init(aempty + i, 1); }
    tc::mbar_init(accfull, 1);
    tc::mbar_init(accempty, kI8GenWarps);
    tc::fence_mbar_init();
  }
  if (tid < 4) spass[tid] = A.pass[tid];
  // root limb tables of this signal's prime (W_tab from the prep kernel) and the phase indices u_j
  {
    const double2* Wg = P.W_tab + (int64_t)s * P.p_stride;
    const double qa = 127.0 * ldexp(1.0, 8 * (S - 1));
    for (int q = tid; q < p; q += kI8Threads) {
      const double2 w = Wg[q];
      int dr[8], di[8];
      digits(llrint(w.x * qa), S, dr);
      digits(llrint(w.y * qa), S, di);
      uint32_t e[6];
#pragma unroll
      for (int t = 0; t < 6; ++t) e[t] = t < S ? ((uint32_t)(uint8_t)dr[t] | ((uint32_t)(uint8_t)di[t] << 8)) : 0u;
      sTlo[q] = make_uint2(e[0] | (e[1] << 16), e[2] | (e[3] << 16));
      if (S > 4) sThi[q] = e[4] | (e[5] << 16);
    }
    const int2* ug = P.u_all + (int64_t)s * P.kk;
    for (int i = tid; i < nk * kI8StepTerms; i += kI8Threads) {
      const int j = ks_lo * kI8StepTerms + i;
      sU[i] = j < K ? ug[j].x : 0;
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tbase = *tslot;

  if (warp < kI8GenWarps) {
    // ---------------- A generators + epilogue: warp g owns TMEM lanes / rows 32 (g % 4) .., terms 8 (g / 4) ..
    const int quarter = warp & 3, half = warp >> 2;
    const int row = 32 * quarter + lane;
    const unsigned h = (unsigned)(ht * kI8Rows + row);
    const unsigned magic = 0xFFFFFFFFu / (unsigned)p + 1u;
    const uint32_t lane_addr = tbase + ((uint32_t)(32 * quarter) << 16);
    double2* out;
    int64_t pstr;
    if (A.ksplit == 1) {
      out = P.lines + (int64_t)s * P.L * P.p_stride;
      pstr = P.p_stride;
    } else {
      const int n_slots = gridDim.x / (A.ksplit * A.n_htiles * P.i8_ntiles);
      out = part + ((int64_t)ks_i * n_slots + slot) * P.L * (int64_t)A.p_part;
      pstr = A.p_part;
    }
    const double scale = P.i8_sigma[s] / (127.0 * 127.0);
    uint32_t aphase = 0;                                           // parity bit per A slot
    for (int ps = 0; ps < A.npass; ++ps) {
      const int pv = spass[ps];
      const int wl = pass_wl(pv), wh = pass_wh(pv), nsa = pass_nsa(pv), nl = wh + 1;
      const uint32_t ta0 = lane_addr + pass_abase(pv) + 4 * half;
      for (int kq = 0; kq < nk; ++kq) {
        const int sa = kq % nsa;
        tc::mbar_wait(aempty + sa, ((aphase >> sa) & 1) ^ 1);
        aphase ^= 1u << sa;
        const uint32_t ta = ta0 + sa * nl * 8;
        const int* u8 = sU + kq * kI8StepTerms + 8 * half;
        if (A.dbg != 3 && A.dbg != 4) switch (nl) {
          case 1: gen_stage<1>(ta, u8, sTlo, sThi, h, magic, p, A.dbg); break;
          case 2: gen_stage<2>(ta, u8, sTlo, sThi, h, magic, p, A.dbg); break;
          case 3: gen_stage<3>(ta, u8, sTlo, sThi, h, magic, p, A.dbg); break;
          case 4: gen_stage<4>(ta, u8, sTlo, sThi, h, magic, p, A.dbg); break;
          case 5: gen_stage<5>(ta, u8, sTlo, sThi, h, magic, p, A.dbg); break;
          default: gen_stage<6>(ta, u8, sTlo, sThi, h, magic, p, A.dbg); break;
        }
        tc::tmem_wait_st();
        tc::fence_before_sync();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(afull + sa);
      }
      // epilogue of this pass: sum the weights in FP64 (lowest weight first) and add to the lines;
      // the two warps of a lane quarter take alternate 16-column chunks
      tc::mbar_wait(accfull, ps & 1);
      tc::fence_after_sync();
      const bool first = ps == 0;
      for (int c0 = 16 * half; c0 < NT; c0 += 32) {
        double acc[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[i] = 0.0;
        for (int w = wh; w >= wl; --w) {
          int32_t v[16];
          tc::tmem_ld16(lane_addr + (w - wl) * NT + c0, v);
          tc::tmem_wait_ld();
          const double f = ldexp(1.0, -8 * w);
#pragma unroll
          for (int i = 0; i < 16; ++i) acc[i] = fma((double)v[i], f, acc[i]);
        }
        if (h < (unsigned)p) {
          const int n0 = (nt * NT + c0) >> 1;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int nn = n0 + i;
            if (nn < P.L) {
              double2* o = out + (int64_t)nn * pstr + h;
              double2 val = make_double2(acc[2 * i] * scale, acc[2 * i + 1] * scale);
              if (!first) {
                const double2 prev = *o;
                val.x += prev.x;
                val.y += prev.y;
              }
              *o = val;
            }
          }
        }
      }
      tc::fence_before_sync();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(accempty);
    }
  } else if (warp == kI8ProdWarp) {
    // ---------------- B producer: one elected lane streams the B limb tiles (backs off while the ring is full)
    if (lane == 0 && nk > 0) {
      const int8_t* Bg = P.i8_B + (((int64_t)s * P.i8_ntiles + nt) * P.i8_nks) * S * (int64_t)NT * 32;
      int ib = 0;
      for (int ps = 0; ps < A.npass; ++ps) {
        const uint32_t bytes = (uint32_t)(pass_wh(spass[ps]) + 1) * NT * 32;
        for (int kq = 0; kq < nk; ++kq, ++ib) {
          const int sb = ib % A.nsb;
          const uint32_t par = ((ib / A.nsb) & 1) ^ 1;
          while (!tc::mbar_try_wait(bempty + sb, par)) __nanosleep(64);
          if (A.dbg == 4) {
            tc::mbar_arrive(bfull + sb);
          } else {
            tc::mbar_expect_tx(bfull + sb, bytes);
            tc::bulk_g2s(sB + (size_t)sb * A.b_stage_bytes, Bg + (int64_t)(ks_lo + kq) * S * NT * 32, bytes, bfull + sb);
          }
        }
      }
    }
  } else {
    // ---------------- MMA issuer: the whole warp runs the loop (uniform descriptors), one elected lane issues
    {
      const uint32_t idesc = tc::idesc_i8(kI8Rows, NT);
      int ib = 0;
      uint32_t aphase = 0;
      for (int ps = 0; ps < A.npass; ++ps) {
        const int pv = spass[ps];
        const int wl = pass_wl(pv), wh = pass_wh(pv), nsa = pass_nsa(pv), nl = wh + 1;
        if (ps > 0) {
          tc::mbar_wait(accempty, (ps - 1) & 1);
          tc::fence_after_sync();
        }
        for (int kq = 0; kq < nk; ++kq, ++ib) {
          const int sb = ib % A.nsb, sa = kq % nsa;
          tc::mbar_wait(bfull + sb, (ib / A.nsb) & 1);
          tc::mbar_wait(afull + sa, (aphase >> sa) & 1);
          aphase ^= 1u << sa;
          tc::fence_after_sync();
          const uint64_t bd0 = tc::sdesc_kmajor(tc::smem_u32(sB + (size_t)sb * A.b_stage_bytes), 128, 256);
          const uint32_t a0 = tbase + pass_abase(pv) + sa * nl * 8;
          if (tc::elect_one()) {
            if (A.dbg != 2) issue_stage_rt(wl, wh, tbase, a0, bd0, (uint32_t)NT, (uint32_t)NT * 2, idesc, kq == 0);
            tc::mma_commit(bempty + sb);
            tc::mma_commit(aempty + sa);
          }
          __syncwarp();
        }
        if (tc::elect_one()) tc::mma_commit(accfull);
        __syncwarp();
      }
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == kI8MmaWarp) {
    tc::fence_after_sync();
    tc::tmem_dealloc<512>(tbase);
  }
}

// ------------------------------------------------------------------ host side
// Limb count from the decode budget: the int8 path keeps |x - round(x)| of the
// Eq. (41) decode below ~1e-3 and coefficient errors below ~1e-11 relative.
int i8_limbs_for(int64_t E) {
  if (E <= ((int64_t)1 << 28)) return 5;
  if (E <= ((int64_t)1 << 36)) return 6;
  return 0;   // beyond what FP64 roots can feed: use the FP64 tensor (DMMA) path
}

// Passes over the limb weights: a pass [wl, wh] holds (wh - wl + 1) NT s32 accumulator columns and
// nsa A slots of 8 (wh + 1) columns within the 512 TMEM columns; at least 3 A slots per pass so the
// generators run ahead of the tensor core (the MMA completion -> slot free -> regenerate round trip).
static bool i8_passes(int S, int NT, int min_slots, I8Config& c) {
  c.npass = 0;
  int wh = S - 1;
  while (wh >= 0) {
    int wl = wh;
    auto fits = [&](int lo) { return (wh - lo + 1) * NT + min_slots * 8 * (wh + 1) <= 512; };
    if (!fits(wl)) return false;
    while (wl - 1 >= 0 && fits(wl - 1)) --wl;
    if (c.npass == 4) return false;
    const int acc = (wh - wl + 1) * NT;
    c.wl[c.npass] = wl;
    c.wh[c.npass] = wh;
    c.a_base[c.npass] = acc;
    c.nsa[c.npass] = std::min(8, (512 - acc) / (8 * (wh + 1)));
    ++c.npass;
    wh = wl - 1;
  }
  return true;
}

bool i8_configure(int L, int64_t E, int k, I8Config* out) {
  I8Config c{};
  c.S = i8_limbs_for(E);
  if (c.S == 0 || getenv("SFFT_NO_I8")) return false;
  const int N2 = 2 * L;
  double best = 1e30;
  for (int nt = (N2 + 255) / 256; nt <= (N2 + 15) / 16; ++nt) {
    const int NT = ((N2 + nt - 1) / nt + 15) / 16 * 16;
    if (NT > 256) continue;
    I8Config t = c;
    t.NT = NT;
    t.ntiles = nt;
    if (!i8_passes(c.S, NT, 3, t) && !i8_passes(c.S, NT, 2, t)) continue;
    // cycles per (128 rows, 16 terms): MMA (products * NT / 2) vs A generation (~150 per pass) + epilogue
    const int prods = c.S * (c.S + 1) / 2;
    const double cost = nt * (std::max(prods * NT / 2.0, 150.0 * t.npass) + 40.0 * t.npass);
    if (cost < best - 1e-9) { best = cost; c.NT = NT; c.ntiles = nt; c.npass = t.npass;
      for (int i = 0; i < 4; ++i) { c.wl[i] = t.wl[i]; c.wh[i] = t.wh[i]; c.a_base[i] = t.a_base[i]; c.nsa[i] = t.nsa[i]; } }
  }
  if (c.NT == 0) return false;
  c.nks = (2 * k + kI8StepTerms - 1) / kI8StepTerms;
  *out = c;
  return true;
}

size_t i8_limb_bytes(const I8Config& c, int batch) {
  return (size_t)batch * c.ntiles * c.nks * c.S * (size_t)c.NT * 32;
}

static size_t i8_smem(const I8Config& c, int p, int nk_cta, int nsb, uint32_t* tab_off, uint32_t* u_off) {
  size_t o = 512 + (size_t)nsb * c.S * c.NT * 32;
  o = (o + 15) & ~(size_t)15;
  *tab_off = (uint32_t)o;
  o += (size_t)p * 8 + (c.S > 4 ? (size_t)p * 4 : 0);
  o = (o + 15) & ~(size_t)15;
  *u_off = (uint32_t)o;
  o += (size_t)nk_cta * kI8StepTerms * 4;
  return o;
}

bool i8_fits(const I8Config& c, int p, int k, int smem_optin) {
  uint32_t a, b;
  const int nks = (k + kI8StepTerms - 1) / kI8StepTerms;
  return i8_smem(c, p, nks, 2, &a, &b) <= (size_t)smem_optin;
}

int i8_blocks(const I8Config& c, int32_t max_p, int32_t n_signals) {
  return n_signals * ((max_p + kI8Rows - 1) / kI8Rows) * c.ntiles;
}

cudaError_t launch_i8_prepare(const DevParams& P, int32_t n_signals, int32_t K, cudaStream_t st) {
  i8_sigma_kernel<<<n_signals, 256, 0, st>>>(P, K);
  const int64_t total = (int64_t)n_signals * P.i8_ntiles * P.i8_nks * P.i8_NT * 8;
  DevParams Q = P;
  Q.batch = n_signals;
  if (total > 0) i8_limbs_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(Q, K);
  return cudaGetLastError();
}

cudaError_t launch_expsum_i8(const DevParams& P, const I8Config& c, int32_t max_p, int32_t n_signals, int32_t ksplit,
                             double2* part, int32_t p_part, int smem_optin, cudaStream_t st) {
  I8Args A{};
  A.n_htiles = (max_p + kI8Rows - 1) / kI8Rows;
  A.ksplit = ksplit;
  A.p_part = p_part;
  A.npass = c.npass;
  A.dbg = getenv("SFFT_I8_DBG") ? atoi(getenv("SFFT_I8_DBG")) : 0;
  for (int i = 0; i < c.npass; ++i) A.pass[i] = c.wl[i] | (c.wh[i] << 4) | (c.nsa[i] << 8) | (c.a_base[i] << 16);
  A.b_stage_bytes = (uint32_t)c.S * c.NT * 32;
  const int nks = (P.i8_K + kI8StepTerms - 1) / kI8StepTerms;
  const int nk_cta = (nks + ksplit - 1) / ksplit;
  int nsb = 4;
  size_t smem = 0;
  for (; nsb >= 2; --nsb) {
    smem = i8_smem(c, max_p, nk_cta, nsb, &A.tab_off, &A.u_off);
    if (smem <= (size_t)smem_optin) break;
  }
  if (nsb < 2) return cudaErrorInvalidValue;
  A.nsb = nsb;
  // one CTA per SM: the kernel allocates all 512 TMEM columns
  smem = std::max(smem, (size_t)120 * 1024);
  cudaError_t e = cudaFuncSetAttribute(expsum_i8_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const long grid = (long)n_signals * A.n_htiles * c.ntiles * ksplit;
  if (grid > 0) expsum_i8_kernel<<<(unsigned)grid, kI8Threads, smem, st>>>(P, A, part);
  return cudaGetLastError();
}

}  // namespace sfft
