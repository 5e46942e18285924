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
#include <algorithm>
#include <cassert>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "sfft_internal.cuh"

namespace sfft {

#ifndef SFFT_BK
#define SFFT_BK 64
#endif
constexpr int kBK = SFFT_BK;   // terms per staged chunk

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
expsum_kernel(DevParams P, int32_t wn_count, int32_t n_htiles, int32_t n_ntiles, int32_t ksplit, double2* part,
              int32_t p_part) {
  pdl_wait();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int BN = TN * wn_count;
  const int WH = WARPS / wn_count;
  const int BM = 32 * TH * WH;

  int bid = blockIdx.x;
  const int ks = bid % ksplit;
  bid /= ksplit;
  const int nt = bid % n_ntiles;
  bid /= n_ntiles;
  const int ht = bid % n_htiles;
  const int slot = bid / n_htiles;
  const int s = P.active[slot];
  const int p = P.st_p[s];
  if (ht * BM >= p) return;
  const int K = P.k + (P.literal ? P.st_nR[s] : 0);      // bin-domain g: signal terms only

  double2* sW = reinterpret_cast<double2*>(smem_raw);
  const int p_pad = (p + 1) & ~1;
  double2* sC = sW + p_pad;                                    // [2][kBK][BN]
  int* sU = reinterpret_cast<int*>(sC + 2 * kBK * BN);          // [2][kBK]
  int* sDU = sU + 2 * kBK;                                     // [2][kBK]

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wn = warp % wn_count, wh = warp / wn_count;

  // root table of this signal's prime (computed by the prep kernel)
  const double2* Wg = P.W_tab + (int64_t)P.st_slot[s] * P.p_stride;
  for (int q = tid; q < p; q += WARPS * 32) sW[q] = Wg[q];

  const double2* Cg = P.C_all + (int64_t)s * P.kk * P.Lp + (int64_t)nt * BN;
  const int n_chunks_all = (K + kBK - 1) / kBK;
  const int per = (n_chunks_all + ksplit - 1) / ksplit;
  const int c_lo = ks * per, c_hi = min(n_chunks_all, c_lo + per);

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
      const int u = j < K ? P.u_all[(int64_t)s * P.kk + j].x : 0;
      sU[buf * kBK + tid] = u;
      sDU[buf * kBK + tid] = (u * 32) % p;
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

  if (c_lo < c_hi) {
    stage(0, c_lo);
    cp_async_commit();
  }
  for (int ch = c_lo; ch < c_hi; ++ch) {
    const int buf = (ch - c_lo) & 1;
    if (ch + 1 < c_hi) {
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

  double2* out;
  int64_t pstr;
  if (ksplit == 1) {
    out = P.lines + (int64_t)s * P.L * P.p_stride;
    pstr = P.p_stride;
  } else {
    const int n_slots = gridDim.x / (ksplit * n_htiles * n_ntiles);
    out = part + ((int64_t)ks * n_slots + slot) * P.L * (int64_t)p_part;
    pstr = p_part;
  }
  const int n_base = nt * BN + wn * TN;
#pragma unroll
  for (int n = 0; n < TN; ++n) {
    const int nn = n_base + n;
    if (nn >= P.L) break;
#pragma unroll
    for (int t = 0; t < TH; ++t) {
      const unsigned h = h0 + 32u * t;
      if (h < (unsigned)p) out[(int64_t)nn * pstr + h] = acc[t][n];
    }
  }
}

// ---------------------------------------------------------------- FP64 tensor-core variant
// Same contraction on the FP64 tensor pipe: mma.sync.m8n8k4 f64 (SASS DMMA), 4 real MMAs per
// complex 8x8x4 block (Dr += Ar Br + Ai (-Bi), Di += Ar Bi + Ai Br).  Fragments (PTX ISA m8n8k4
// .f64): A[m][k] m = lane>>2, k = lane&3; B[k][n] k = lane&3, n = lane>>2; D[m][n] m = lane>>2,
// n = 2(lane&3)+{0,1}.  Rows m are samples h, columns n are lines, k are terms j: every lane
// fetches ONE root W_p[(h u_j) mod p] per 8x4 A block and ONE line coefficient per 4x8 B block.
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}
__device__ __forceinline__ double dneg(double x) {
  return __longlong_as_double(__double_as_longlong(x) ^ (long long)0x8000000000000000ULL);
}

// Warp roles: the WARPS warps form WG = (NB1 ? 2 : 1) column groups.  Group 0 owns columns
// [0, 8 NB0), group 1 owns [8 NB0, 8 (NB0 + NB1)); inside a group every warp owns 8 MB rows, so a
// block tile is BM = 8 MB WARPS / WG rows x BN = 8 (NB0 + NB1) lines.  Two column groups double
// the resident warps per SM at the same accumulator footprint per warp.
template <int MB, int NB>
struct DmmaAcc {
  double r[MB][NB][2], i[MB][NB][2];
};

template <int MB, int NB, int BN>
__device__ __forceinline__ void dmma_chunk(DmmaAcc<MB, NB>& acc, const double2* __restrict__ sW,
                                           const double2* __restrict__ cb, const int2* __restrict__ ub,
                                           unsigned hrow, int col0, int kl, int nl, unsigned magic, int pp) {
  constexpr int KS = kBK / 4;
  struct Frag { double2 tw[MB]; double2 cv[NB]; };
  auto load_frag = [&](Frag& f, int kk) {
    const int j = kk * 4 + kl;
    const int2 ud = ub[j];
    const unsigned x = hrow * (unsigned)ud.x;
    int r = (int)(x - __umulhi(x, magic) * (unsigned)pp);
    r += (r >> 31) & pp;
#pragma unroll
    for (int a = 0; a < MB; ++a) {
#ifdef SFFT_BOUNDS
      assert(r >= 0 && r < pp && ud.x >= 0 && ud.x < pp && ud.y >= 0 && ud.y < pp);
#endif
      f.tw[a] = sW[r];
      r += ud.y;
      r -= (r >= pp) ? pp : 0;
    }
    const double2* crow = cb + j * BN + col0 + nl;
#pragma unroll
    for (int b = 0; b < NB; ++b) f.cv[b] = crow[8 * b];
  };
  auto mma_frag = [&](const Frag& f) {
#pragma unroll
    for (int b = 0; b < NB; ++b)
#pragma unroll
      for (int a = 0; a < MB; ++a) {
        dmma(acc.r[a][b][0], acc.r[a][b][1], f.tw[a].x, f.cv[b].x);
        dmma(acc.i[a][b][0], acc.i[a][b][1], f.tw[a].x, f.cv[b].y);
      }
#pragma unroll
    for (int b = 0; b < NB; ++b)
#pragma unroll
      for (int a = 0; a < MB; ++a) {
        dmma(acc.r[a][b][0], acc.r[a][b][1], f.tw[a].y, dneg(f.cv[b].y));
        dmma(acc.i[a][b][0], acc.i[a][b][1], f.tw[a].y, f.cv[b].x);
      }
  };
  Frag f0, f1;
  load_frag(f0, 0);
#pragma unroll
  for (int kk = 0; kk < KS; kk += 2) {
    load_frag(f1, kk + 1);
    mma_frag(f0);
    if (kk + 2 < KS) load_frag(f0, kk + 2);
    mma_frag(f1);
  }
}

template <int MB, int NB>
__device__ __forceinline__ void dmma_store(const DmmaAcc<MB, NB>& acc, double2* out, int64_t pstr, int L, int p,
                                           unsigned hrow0, int col0, int kl, int nl) {
#pragma unroll
  for (int a = 0; a < MB; ++a) {
    const unsigned h = hrow0 + a * 8 + nl;
    if (h >= (unsigned)p) continue;
#pragma unroll
    for (int b = 0; b < NB; ++b)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int nn = col0 + b * 8 + 2 * kl + e;
        if (nn < L) out[(int64_t)nn * pstr + h] = make_double2(acc.r[a][b][e], acc.i[a][b][e]);
      }
  }
}

// The whole term loop of one column group (staging is shared by all warps of the block; every
// warp of both groups reaches the same sequence of block barriers).
template <int MB, int NB, int BN, int WARPS, typename StageF>
__device__ __forceinline__ void dmma_group(StageF&& stage, const double2* sW, const double2* sC, const int2* sU,
                                           int c_lo, int c_hi, unsigned hrow0, int col0, int lane, unsigned magic,
                                           int p, double2* out, int64_t pstr, int L, int col_base) {
  DmmaAcc<MB, NB> acc;
#pragma unroll
  for (int a = 0; a < MB; ++a)
#pragma unroll
    for (int b = 0; b < NB; ++b) acc.r[a][b][0] = acc.r[a][b][1] = acc.i[a][b][0] = acc.i[a][b][1] = 0.0;
  const int kl = lane & 3, nl = lane >> 2;
  const unsigned hrow = hrow0 + nl;
  if (c_lo < c_hi) {
    stage(0, c_lo);
    cp_async_commit();
  }
  for (int ch = c_lo; ch < c_hi; ++ch) {
    const int buf = (ch - c_lo) & 1;
    if (ch + 1 < c_hi) {
      stage(buf ^ 1, ch + 1);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    dmma_chunk<MB, NB, BN>(acc, sW, sC + buf * kBK * BN, sU + buf * kBK, hrow, col0, kl, nl, magic, p);
    __syncthreads();
  }
  cp_async_wait<0>();
  dmma_store<MB, NB>(acc, out, pstr, L, p, hrow0, col_base + col0, kl, nl);
}

template <int MB, int NB0, int NB1, int WARPS>
__global__ void __launch_bounds__(WARPS * 32)
expsum_dmma_kernel(DevParams P, int32_t n_htiles, int32_t n_ntiles, int32_t ksplit, double2* part, int32_t p_part) {
  pdl_wait();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int WG = NB1 ? 2 : 1;
  constexpr int WPG = WARPS / WG;                               // warps per column group
  constexpr int BN = 8 * (NB0 + NB1);
  constexpr int BM = 8 * MB * WPG;

  int bid = blockIdx.x;
  const int ks = bid % ksplit;
  bid /= ksplit;
  const int nt = bid % n_ntiles;
  bid /= n_ntiles;
  const int ht = bid % n_htiles;
  const int slot = bid / n_htiles;                              // index into the active-signal list
  const int s = P.active[slot];
#ifdef SFFT_BOUNDS
  assert(s >= 0 && s < P.batch);
#endif
  const int p = P.st_p[s];
  if (ht * BM >= p) return;
  const int K = P.k + (P.literal ? P.st_nR[s] : 0);      // bin-domain g: signal terms only
#ifdef SFFT_BOUNDS
  assert(p >= 2 && p <= P.p_cap && K >= 0 && K <= P.kk);
#endif

  double2* sW = reinterpret_cast<double2*>(smem_raw);
  const int p_pad = (p + 1) & ~1;
  double2* sC = sW + p_pad;                                    // [2][kBK][BN]
  int2* sU = reinterpret_cast<int2*>(sC + 2 * kBK * BN);        // [2][kBK]  (u, (8u) mod p)

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wg = warp / WPG, wr = warp % WPG;
  const double2* Wg = P.W_tab + (int64_t)P.st_slot[s] * P.p_stride;
  for (int q = tid; q < p; q += WARPS * 32) cp_async16(sW + q, Wg + q, true);   // joins the first stage group

  const int2* ug = P.u_all + (int64_t)s * P.kk;
  const double2* Cg = P.C_all + (int64_t)s * P.kk * P.Lp + (int64_t)nt * BN;
  const int n_chunks_all = (K + kBK - 1) / kBK;
  const int per = (n_chunks_all + ksplit - 1) / ksplit;
  const int c_lo = ks * per, c_hi = min(n_chunks_all, c_lo + per);

  auto stage = [&](int buf, int chunk) {
    const int j0 = chunk * kBK;
    double2* dst = sC + buf * kBK * BN;
    for (int e = tid; e < kBK * BN; e += WARPS * 32) {
      const int jj = e / BN, n = e - jj * BN;
      const int j = j0 + jj;
      const bool ok = j < K;
      cp_async16(dst + e, ok ? (const void*)(Cg + (int64_t)j * P.Lp + n) : (const void*)Cg, ok);
    }
    if (tid < kBK / 2) {                                        // 16-byte copies of two (u, 8u mod p) pairs
      const int j = j0 + 2 * tid;
      const bool ok = j < K;                                     // invalid: zero-fill from a safe address
      cp_async16(sU + buf * kBK + 2 * tid, ok ? (const void*)(ug + j) : (const void*)ug, ok);
    }
  };

  double2* out;
  int64_t pstr;
  if (ksplit == 1) {
    out = P.lines + (int64_t)s * P.L * P.p_stride;
    pstr = P.p_stride;
  } else {
    const int n_slots = gridDim.x / (ksplit * n_htiles * n_ntiles);
    out = part + ((int64_t)ks * n_slots + slot) * P.L * (int64_t)p_part;
    pstr = p_part;
  }
  const unsigned hrow0 = (unsigned)(ht * BM + wr * 8 * MB);
  const unsigned magic = 0xFFFFFFFFu / (unsigned)p + 1u;
  if (NB1 == 0 || wg == 0)
    dmma_group<MB, NB0, BN, WARPS>(stage, sW, sC, sU, c_lo, c_hi, hrow0, 0, lane, magic, p, out, pstr, P.L, nt * BN);
  else
    dmma_group<MB, (NB1 ? NB1 : 1), BN, WARPS>(stage, sW, sC, sU, c_lo, c_hi, hrow0, 8 * NB0, lane, magic, p, out,
                                               pstr, P.L, nt * BN);
}

// ---------------------------------------------------------------- host side
static const int kTNs[] = {1, 2, 3, 4, 5, 6, 7, 8, 11, 13, 16};
constexpr int kWarps = 8;
constexpr int kTH = 2;
constexpr int kDmmaMB = 2;

// Throughput model: per (warp, term) the DFMA kernel spends 2 TH TN SM-cycles on the
// FP64 pipe and ~8 TH + TN shared-memory wavefronts (random-index root loads, broadcast C loads);
// the DMMA kernel is FP64-tensor bound (measured 37.1 vs 33.6 TFLOP/s) with padding to 8 lines.
ExpsumShape choose_expsum_shape(int L) {
  ExpsumShape best{};
  best.est = -1.0;
  for (int tn : kTNs)
    for (int wn : {1, 2, 4, 8}) {
      const int bn = tn * wn;
      const int nt = (L + bn - 1) / bn;
      const double util = (double)L / ((double)nt * bn);
      const double fp = 2.0 * kTH * tn, sm = 8.0 * kTH + tn;
      const double est = 0.45 * 33.6 * util * fp / std::max(fp, sm);     // 0.45: measured DFMA efficiency
      if (est > best.est + 1e-9) {
        best = ExpsumShape{0, tn, wn, kTH, kWarps, 32 * kTH * (kWarps / wn), bn, nt, 0, 0, est};
      }
    }
  for (int nb = 1; nb <= 8; ++nb) {
    const int bn = 8 * nb;
    const int nt = (L + bn - 1) / bn;
    const double util = (double)L / ((double)nt * bn);
    const double est = 0.8 * 37.1 * util * (nb >= 2 ? 1.0 : 0.9);      // 0.8: measured DMMA efficiency
    if (est > best.est + 1e-9) best = ExpsumShape{1, 0, 0, 0, kWarps, 8 * kDmmaMB * kWarps, bn, nt, kDmmaMB, nb, est};
  }
  // tuning override: SFFT_EXPSUM=dfma:<tn>:<wn> | dmma:<nb> | dmma:<nb>:<mb>
  if (const char* e = getenv("SFFT_EXPSUM")) {
    int a = 0, b = 0;
    if (sscanf(e, "dmma:%d:%d", &a, &b) == 2) {
      const int bn = 8 * a, nt = (L + bn - 1) / bn;
      const int warps = b == 2 ? 8 : 16;
      const int bm = b == 1 ? 128 : 128;
      best = ExpsumShape{1, 0, 0, 0, warps, bm, bn, nt, b, a, 0.0};
    } else if (sscanf(e, "dfma:%d:%d", &a, &b) == 2) {
      const int bn = a * b, nt = (L + bn - 1) / bn;
      best = ExpsumShape{0, a, b, kTH, kWarps, 32 * kTH * (kWarps / b), bn, nt, 0, 0, 0.0};
    } else if (sscanf(e, "dmma:%d", &a) == 1) {
      const int bn = 8 * a, nt = (L + bn - 1) / bn;
      best = ExpsumShape{1, 0, 0, 0, kWarps, 8 * kDmmaMB * kWarps, bn, nt, kDmmaMB, a, 0.0};
    }
  }
  return best;
}

static size_t expsum_smem(int max_p, int bn) {
  return sizeof(double2) * (size_t)(((max_p + 1) & ~1) + 2 * kBK * bn) + sizeof(int) * 4 * kBK;
}

struct Split { int ksplit; double2* part; int p_part; int* occ_out; };   // occ_out: query only, no launch

template <typename KernT, typename... Args>
static cudaError_t launch_grid(KernT kern, const ExpsumShape& S, int32_t max_p, int32_t n_signals, const Split& sp,
                               cudaStream_t st, Args... args) {
  const size_t smem = expsum_smem(max_p, S.bn);
  cudaError_t e = ensure_smem(kern, smem);
  if (e != cudaSuccess) return e;
  if (sp.occ_out) return cudaOccupancyMaxActiveBlocksPerMultiprocessor(sp.occ_out, kern, S.warps * 32, smem);
  const int n_htiles = (max_p + S.bm - 1) / S.bm;
  const long grid = (long)n_signals * n_htiles * S.nt * sp.ksplit;
  if (grid <= 0) return cudaSuccess;
  return launch_pdl(kern, dim3((unsigned)grid), dim3(S.warps * 32), smem, st, args..., n_htiles, S.nt, sp.ksplit,
                    sp.part, sp.p_part);
}

template <int TN>
static cudaError_t launch_tn(const DevParams& P, const ExpsumShape& S, int32_t max_p, int32_t n_signals,
                             const Split& sp, cudaStream_t st) {
  return launch_grid(expsum_kernel<TN, kTH, kWarps>, S, max_p, n_signals, sp, st, P, (int32_t)S.wn);
}

template <int NB>
static cudaError_t launch_nb(const DevParams& P, const ExpsumShape& S, int32_t max_p, int32_t n_signals,
                             const Split& sp, cudaStream_t st) {
  // mb 1: 16 warps x (8 rows); mb 2: 8 warps x (16 rows); mb 3: 16 warps in two column groups x (16 rows)
  if (S.mb == 1) return launch_grid(expsum_dmma_kernel<1, NB, 0, 16>, S, max_p, n_signals, sp, st, P);
  if (S.mb == 4) return launch_grid(expsum_dmma_kernel<1, NB, 0, 4>, S, max_p, n_signals, sp, st, P);   // 32 rows
  if (S.mb == 5) return launch_grid(expsum_dmma_kernel<2, NB, 0, 4>, S, max_p, n_signals, sp, st, P);   // 64 rows
  if (S.mb == 3 && NB >= 2)
    return launch_grid(expsum_dmma_kernel<2, (NB + 1) / 2, NB / 2, 16>, S, max_p, n_signals, sp, st, P);
  return launch_grid(expsum_dmma_kernel<2, NB, 0, 8>, S, max_p, n_signals, sp, st, P);
}

int expsum_bk() { return kBK; }

// Row tile for the iteration's largest prime: late iterations have p of a few tens to a few hundred,
// where 128-row CTAs would leave most rows idle.
ExpsumShape expsum_for_p(const ExpsumShape& S, int32_t max_p) {
  const char* ov = getenv("SFFT_EXPSUM");
  if (S.kind != 1 || S.mb != 2 || (ov && (!strncmp(ov, "dmma", 4) || !strncmp(ov, "dfma", 4)))) return S;
  ExpsumShape r = S;
  if (max_p <= 48) { r.mb = 4; r.warps = 4; r.bm = 32; }
  else if (max_p <= 320) { r.mb = 5; r.warps = 4; r.bm = 64; }
  return r;
}

int expsum_blocks(const ExpsumShape& S, int32_t max_p, int32_t n_signals) {
  return n_signals * ((max_p + S.bm - 1) / S.bm) * S.nt;
}

int expsum_occupancy(const ExpsumShape& S, int32_t max_p) {
  int occ = 1;
  DevParams P;
  memset(&P, 0, sizeof P);
  if (launch_expsum(P, S, max_p, 1, 1, nullptr, 0, nullptr, &occ) != cudaSuccess) return 1;
  return occ > 0 ? occ : 1;
}

cudaError_t launch_expsum(const DevParams& P, const ExpsumShape& S, int32_t max_p, int32_t n_signals,
                          int32_t ksplit, double2* part, int32_t p_part, cudaStream_t st, int* occ_out) {
  const Split sp{ksplit, part, p_part, occ_out};
  if (S.kind == 1) {
    switch (S.nb) {
      case 1: return launch_nb<1>(P, S, max_p, n_signals, sp, st);
      case 2: return launch_nb<2>(P, S, max_p, n_signals, sp, st);
      case 3: return launch_nb<3>(P, S, max_p, n_signals, sp, st);
      case 4: return launch_nb<4>(P, S, max_p, n_signals, sp, st);
      case 5: return launch_nb<5>(P, S, max_p, n_signals, sp, st);
      case 6: return launch_nb<6>(P, S, max_p, n_signals, sp, st);
      case 7: return launch_nb<7>(P, S, max_p, n_signals, sp, st);
      case 8: return launch_nb<8>(P, S, max_p, n_signals, sp, st);
    }
    return cudaErrorInvalidValue;
  }
  switch (S.tn) {
    case 1: return launch_tn<1>(P, S, max_p, n_signals, sp, st);
    case 2: return launch_tn<2>(P, S, max_p, n_signals, sp, st);
    case 3: return launch_tn<3>(P, S, max_p, n_signals, sp, st);
    case 4: return launch_tn<4>(P, S, max_p, n_signals, sp, st);
    case 5: return launch_tn<5>(P, S, max_p, n_signals, sp, st);
    case 6: return launch_tn<6>(P, S, max_p, n_signals, sp, st);
    case 7: return launch_tn<7>(P, S, max_p, n_signals, sp, st);
    case 8: return launch_tn<8>(P, S, max_p, n_signals, sp, st);
    case 11: return launch_tn<11>(P, S, max_p, n_signals, sp, st);
    case 13: return launch_tn<13>(P, S, max_p, n_signals, sp, st);
    case 16: return launch_tn<16>(P, S, max_p, n_signals, sp, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace sfft
