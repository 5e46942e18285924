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
// the same way.  Every limb product x_s y_t is an exact int8 x int8 -> int32 product.  Accumulator w
// sums the w + 1 <= S limb pairs (s, w - s) over the 2K real operands, |Acc_w| <= S * 2K * 128 * 128,
// so the int32 sums are exact while S * 2K * 2^14 < 2^31, i.e. K < 10922 terms at S = 6 (13107 at
// S = 5); i8_configure refuses larger k (the FP64 path runs, or expsum_path = 2 gets ENOTSUP).  Then
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
//   * one elected lane issues tcgen05.mma.kind::i8 (A from TMEM, B from smem, s32 accumulators in TMEM),
//     one accumulator per limb weight: all S weights of an output tile live in TMEM at once, so the
//     output columns are split into n-tiles of at most NT columns (S NT + slots <= 512 TMEM columns);
//   * the epilogue (the generator warps) reads the accumulators with tcgen05.ld, sums the weights in FP64
//     and writes complex128 lines;
//   * the kernel is persistent (one CTA per SM walks a contiguous range of tiles, so the root table of a
//     signal is built once per CTA) and a ring of full / empty mbarriers couples generators, the B
//     producer and the MMA issuer.
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
// sigma[s] >= every |Re C[j][n]|, |Im C[j][n]|: the line factors have unit modulus, so |C[j][n]| = |C[j][0]|
// up to a few ulp; sigma = (1 + 1e-12) max_j |C[j][0]| (column 0 is the unshifted line, C[j][0] = a_j)
__global__ void i8_sigma_kernel(DevParams P, int32_t K) {
  pdl_wait();
  const int s = blockIdx.x;
  const double2* Cs = P.C_all + (int64_t)s * P.kk * P.Lp;
  double m = 0.0;
  for (int j = threadIdx.x; j < K; j += blockDim.x) {
    const double2 c = Cs[(int64_t)j * P.Lp];
    m = fmax(m, hypot(c.x, c.y));
  }
  for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  __shared__ double red[32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = fmax(m, red[w]);
    P.i8_sigma[s] = m > 0.0 ? m * (1.0 + 1e-12) : 1.0;
  }
}

__host__ __device__ __forceinline__ int i8_tile_width(int nt, int ntiles, int NT, int NT_last) {
  return nt == ntiles - 1 ? NT_last : NT;
}

// B limbs of signal s, n-tile nt (width W), K step ks, limb t: 32 W bytes at
//   i8_B + s * per_signal + nt * nks * S * NT * 32 + (ks * S + t) * W * 32,  per_signal = nks * S * 32 * cols
// in the UMMA K-major layout: (column, K byte) -> (col / 8) 256 + (k / 16) 128 + (col % 8) 16 + k % 16.
// One CTA per (signal, n-tile, K step): the 16 terms x W/2 lines of C are read coalesced into shared
// memory, every (column, K byte) value is split into its S digits in shared memory, and the S limb tiles
// (contiguous in global memory) are written with 16-byte stores.
template <int S>
__global__ void __launch_bounds__(256) i8_limbs_kernel(DevParams P, int32_t K, int32_t only_retilted) {
  pdl_wait();
  // [term][line of the tile] (W <= 96); row stride 49 x 16 B: the terms a warp reads share banks only 2-way
  __shared__ double2 cv[kI8StepTerms][49];
  __shared__ __align__(16) uint8_t tiles[6 * 96 * 32];           // [limb][W * 32]
  const int NT = P.i8_NT, ntiles = P.i8_ntiles, nks = P.i8_nks;
  const int nkt = (K + kI8StepTerms - 1) / kI8StepTerms;        // steps in use (layout stride stays nks)
  const int cols = (ntiles - 1) * NT + P.i8_NT_last;
  int b = blockIdx.x;
  const int ks = b % nkt;
  b /= nkt;
  const int nt = b % ntiles;
  const int s = b / ntiles;
  if (only_retilted && !P.st_retilt[s]) return;
  const int W = i8_tile_width(nt, ntiles, NT, P.i8_NT_last);
  const int n0 = (nt * NT) >> 1, nl = W >> 1;                     // lines of the tile
  const double2* Cs = P.C_all + (int64_t)s * P.kk * P.Lp;
  for (int i = threadIdx.x; i < kI8StepTerms * nl; i += blockDim.x) {
    const int jj = i / nl, l = i - jj * nl;
    const int j = ks * kI8StepTerms + jj, n = n0 + l;
    cv[jj][l] = (j < K && n < P.L) ? Cs[(int64_t)j * P.Lp + n] : make_double2(0.0, 0.0);
  }
  __syncthreads();
  const double q = 127.0 * ldexp(1.0, 8 * (S - 1)) / P.i8_sigma[s];
  // CTA pairs: column halves [0, W/2) and [W/2, W) are separate K-major tiles (one per CTA of the pair)
  const int hw = P.i8_pair ? W / 2 : W;
  uint32_t* tw = reinterpret_cast<uint32_t*>(tiles);
  // thread item: output column col, K bytes 4 k4 .. 4 k4 + 3 (terms 2 k4, 2 k4 + 1; re / im rows) -> one
  // 32-bit word per limb
  for (int i = threadIdx.x; i < W * 8; i += blockDim.x) {
    const int col = i >> 3, k4 = i & 7;
    const bool im_out = col & 1;                                  // column 2n+1 is Im s_n
    uint32_t word[S];
#pragma unroll
    for (int t = 0; t < S; ++t) word[t] = 0u;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int kp = 4 * k4 + u;
      const double2 c = cv[kp >> 1][col >> 1];
      const bool a_im = kp & 1;                                   // row 2j+1 multiplies Im W
      const double v = im_out ? (a_im ? c.x : c.y) : (a_im ? -c.y : c.x);
      // balanced base-256 digits of X (i8_digits, most significant first): X + sum_t 128 * 256^t has the plain
      // base-256 digits r_t + 128 (|X| <= 127 * 256^(S-1)), so limb t is byte S-1-t of it with the top bit
      // flipped -- the same bytes as the digit loop, without its 64-bit arithmetic per digit
      const uint64_t Y = (uint64_t)llrint(v * q) + 0x8080808080808080ull;
#pragma unroll
      for (int t = 0; t < S; ++t)
        word[t] |= (((uint32_t)(Y >> (8 * (S - 1 - t))) & 255u) ^ 128u) << (8 * u);
    }
    const int half = col / hw, cc = col - half * hw, kp0 = 4 * k4;
    const int off = half * S * hw * 32 + (cc >> 3) * 256 + (kp0 >> 4) * 128 + (cc & 7) * 16 + (kp0 & 15);
#pragma unroll
    for (int t = 0; t < S; ++t) tw[(t * hw * 32 + off) >> 2] = word[t];
  }
  __syncthreads();
  int8_t* base = P.i8_B + (int64_t)s * nks * S * 32 * cols + (int64_t)nt * nks * S * NT * 32 + (int64_t)ks * S * W * 32;
  const int4* src = reinterpret_cast<const int4*>(tiles);
  int4* dst = reinterpret_cast<int4*>(base);
  for (int i = threadIdx.x; i < S * W * 2; i += blockDim.x) dst[i] = src[i];
}

// ------------------------------------------------------------------ the exp-sum kernel
constexpr int kI8GenWarps = 8;        // 2 per TMEM lane quarter: warp g covers rows 32 (g % 4) .., terms 8 (g / 4) ..
constexpr int kI8MaxSlots = 8;
constexpr int kI8Threads = 32 * (kI8GenWarps + 3);   // + B producer warp + MMA warp + B forwarder warp
constexpr int kI8ProdWarp = kI8GenWarps, kI8MmaWarp = kI8GenWarps + 1, kI8FwdWarp = kI8GenWarps + 2;

struct I8Args {
  int32_t n_htiles, ksplit, p_part, n_slots;
  int32_t nb;                 // B ring slots (shared memory)
  int32_t nap;                // producer back-off (ns) while the B ring is full
  int32_t gnap;               // generator back-off (ns) while waiting for a free A slot (0: spin)
  int32_t relaxed;            // tuning only (SFFT_I8_RELAXED=-1): release semantics for every cross-CTA arrival
  uint32_t b_stage_bytes;     // S * NT * 32
  uint32_t tab_off, thi_off, u_off;   // smem offsets of the limb tables and the phase list
  int32_t chunk;              // consecutive tiles per CTA visit
  long long* prof;            // tuning only (SFFT_I8_PROF): per-CTA cycle counters
  int32_t dbg;                // tuning only (SFFT_I8_DBG): 1 conflict-free gathers, 2 no MMAs, 3 no A generation
};

// 8 terms (4 TMEM columns per limb) of one K step for this thread's row h: gather the root limbs and pack
// them into the TMEM word layout (4 K bytes per 32-bit column: re_j, im_j, re_j+1, im_j+1)
// 8 terms (4 TMEM columns per limb) of one K step for this thread's row f (discrete-log order, reading R22):
// the root of (f, j) is table entry f + e_j (the table holds T twice, so no wrap), or entry 2(p-1) = W_p[0]
// when e_j < 0 (u_j = 0, padding) or the row is h = 0 / padding (special).  The 32 lanes of a warp (consecutive
// f) read consecutive entries -- conflict-free shared-memory gathers.
template <int NL>
__device__ __forceinline__ void gen_limbs(uint32_t (&w)[NL][4], const int* __restrict__ sE,
                                          const uint2* __restrict__ sTlo, const uint32_t* __restrict__ sThi, int f,
                                          bool special, int one, int dbg) {
  const int4 ea = *reinterpret_cast<const int4*>(sE), eb = *reinterpret_cast<const int4*>(sE + 4);
  const int ev[8] = {ea.x, ea.y, ea.z, ea.w, eb.x, eb.y, eb.z, eb.w};
  int q[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) q[e] = (special || ev[e] < 0) ? one : f + ev[e];
  if (dbg == 1) {
#pragma unroll
    for (int e = 0; e < 8; ++e) q[e] = special ? one : f;
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
}

// All S (S + 1) / 2 limb products of one K step, fully unrolled: accumulator of weight w at column w NT,
// A limb s at a0 + 8 s, B limb t at descriptor bd0 + t * (NT * 32 / 16).
template <int S, bool PAIR>
__device__ __forceinline__ void issue_stage(uint32_t tbase, uint32_t a0, uint64_t bd0, uint32_t nt_cols, uint32_t nt_desc,
                                            uint32_t idesc, bool first_k) {
#pragma unroll
  for (int w = 0; w < S; ++w)
#pragma unroll
    for (int sl = 0; sl <= w; ++sl) {
      if constexpr (PAIR)
        tc::mma_i8_ts2(tbase + (uint32_t)w * nt_cols, a0 + 8 * sl, bd0 + (uint64_t)((w - sl) * nt_desc), idesc,
                       (!first_k || sl > 0) ? 1u : 0u);
      else
        tc::mma_i8_ts(tbase + (uint32_t)w * nt_cols, a0 + 8 * sl, bd0 + (uint64_t)((w - sl) * nt_desc), idesc,
                      (!first_k || sl > 0) ? 1u : 0u);
    }
}

// Tile t of the launch: (slot, h-tile, n-tile, term split) with the split index fastest.
struct I8Tile { int slot, ht, nt, ks; };
__device__ __forceinline__ I8Tile tile_of(int t, const I8Args& A, int ntiles) {
  I8Tile r;
  r.ks = t % A.ksplit;
  t /= A.ksplit;
  r.nt = t % ntiles;
  t /= ntiles;
  r.ht = t % A.n_htiles;
  r.slot = t / A.n_htiles;
  return r;
}

// ring slots of a tile of width W: the S accumulators take S W columns, each slot S * 8 columns
__device__ __forceinline__ int ring_slots(int W, int S) { return min(kI8MaxSlots, (512 - S * W) / (8 * S)); }

// Persistent: CTA c owns the contiguous tile range [c T / G, (c + 1) T / G), so consecutive tiles share a
// signal and the root limb table / phase list is rebuilt only when the signal changes.  Every role walks
// the same tile sequence; the ring parities carry over from tile to tile (one bit per slot).  Two rings:
//   A (TMEM, ring_slots(W, S) slots): afull[i] = 8 generator-warp arrivals, aempty[i] = one tcgen05.commit
//   B (shared memory, A.nb slots, deep enough to cover the L2 latency of the bulk copies):
//     bfull[i] = the producer's arrive.expect_tx + the bytes, bempty[i] = one tcgen05.commit
// A forwarder warp waits for bfull of the step and arrives on afull as its 9th arrival, so the MMA issuer
// waits on one barrier per step (every try_wait costs ~90 cycles even when the phase is complete, and the
// tensor core's instruction queue is too shallow to hide two of them).
// PAIR: clusters of 2 CTAs on one TPC run tcgen05.mma.cta_group::2 over M = 256 rows (128 per CTA): each CTA
// generates its own rows' A limbs in its own TMEM and streams half of the B columns (W/2 per tile) into its own
// shared memory, so the tensor cores' shared-memory B reads and the B copies per SM halve.  The leader CTA
// (rank 0) issues; the peer's generator / forwarder / epilogue warps arrive on the leader's afull / accempty
// barriers through the cluster window; the commits are multicast to both CTAs.
template <int S, bool PROF, bool PAIR>
__global__ void __launch_bounds__(kI8Threads, 1) expsum_i8_kernel(DevParams P, I8Args A, double2* part, int32_t n_tiles) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  uint64_t* afull = reinterpret_cast<uint64_t*>(smem_raw);         // [kI8MaxSlots]
  uint64_t* aempty = afull + kI8MaxSlots;
  uint64_t* bfull = aempty + kI8MaxSlots;
  uint64_t* bempty = bfull + kI8MaxSlots;
  uint64_t* accfull = bempty + kI8MaxSlots;
  uint64_t* accempty = accfull + 1;
  uint64_t* tabbar = accempty + 1;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tabbar + 1);
  unsigned char* sB = smem_raw + 512;
  uint2* sTlo = reinterpret_cast<uint2*>(smem_raw + A.tab_off);
  const uint32_t* sThi = reinterpret_cast<const uint32_t*>(smem_raw + A.thi_off);
  int* sU = reinterpret_cast<int*>(smem_raw + A.u_off);         // e_j of the signal's terms
  const int NT = P.i8_NT, ntiles = P.i8_ntiles, nks = P.i8_nks;
  const int cols = (ntiles - 1) * NT + P.i8_NT_last;
  const int K = P.i8_K;                                             // terms in the B limbs (bin-domain: k)
  const int nkt = (K + kI8StepTerms - 1) / kI8StepTerms;             // K steps in use
  const int per = (nkt + A.ksplit - 1) / A.ksplit;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = PAIR ? tc::cluster_rank() : 0u;
  const int cid = PAIR ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;       // pair (cluster) index
  const int ncl = PAIR ? (int)(gridDim.x >> 1) : (int)gridDim.x;
  constexpr int kRowsTile = PAIR ? 2 * kI8Rows : kI8Rows;
  if (warp == kI8MmaWarp) {
    if (PAIR) tc::tmem_alloc2<512>(tslot);
    else tc::tmem_alloc<512>(tslot);
  }
  if (tid == 0) {
    for (int i = 0; i < kI8MaxSlots; ++i) {
      tc::mbar_init(afull + i, (PAIR ? 2 : 1) * (kI8GenWarps + 1));   // generators + the B forwarder (of both CTAs)
      tc::mbar_init(aempty + i, 1);
      tc::mbar_init(bfull + i, 1);
      tc::mbar_init(bempty + i, 1);
    }
    tc::mbar_init(accfull, 1);
    tc::mbar_init(accempty, (PAIR ? 2 : 1) * kI8GenWarps);
    tc::mbar_init(tabbar, 1);
    tc::fence_mbar_init();
  }
  tc::fence_before_sync();
  __syncthreads();
  if (PAIR) tc::cluster_sync();                                        // barriers of both CTAs initialised
  tc::fence_after_sync();
  const uint32_t tbase = *tslot;
  pdl_wait();       // the prologue above (TMEM, barriers) overlaps the predecessor's tail; its data only from here
  // the leader's afull / accempty as seen from this CTA (cluster window), for the peer's arrivals
  const uint32_t afull_l = PAIR ? tc::mapa(afull, 0) : 0u, accempty_l = PAIR ? tc::mapa(accempty, 0) : 0u;
  // Peer arrivals of the generators / epilogue only signal completed TMEM stores / loads (tcgen05.wait::st /
  // ::ld, then tcgen05.fence::before_thread_sync), so they are relaxed (a release at cluster scope costs
  // ~500 cycles per arrival); the forwarder's arrival publishes the peer's B half (TMA-written shared
  // memory) and keeps release semantics.
  auto arrive_afull = [&](int sl, bool publishes_smem) {
    if (PAIR && rank != 0) {
      if (publishes_smem || A.relaxed < 0) tc::mbar_arrive_cluster(afull_l + 8u * (uint32_t)sl);
      else tc::mbar_arrive_cluster_relaxed(afull_l + 8u * (uint32_t)sl);
    } else {
      tc::mbar_arrive(afull + sl);
    }
  };
  auto arrive_accempty = [&]() {
    if (PAIR && rank != 0) {
      if (A.relaxed < 0) tc::mbar_arrive_cluster(accempty_l);
      else tc::mbar_arrive_cluster_relaxed(accempty_l);
    } else {
      tc::mbar_arrive(accempty);
    }
  };

  uint32_t aring = 0, bring = 0;        // parity bit per ring slot (each role keeps its own copies)
  int bpos = 0;                         // B ring position (producer / MMA)
  int ntile_done = 0;                   // accfull / accempty parity
  int cur_s = -1;
  uint32_t tabphase = 0;
  long long pr_a = 0, pr_b = 0, pr_e = 0, pr_t = 0, pr_g = 0;
  const long long pr_start = clock64();
  // chunks of A.chunk consecutive tiles (same signal, mostly) dealt round robin: the CTAs sweep the signals
  // together, so the B limbs of the few signals in flight stay in L2 while each CTA reuses its table
  const int n_chunks = (n_tiles + A.chunk - 1) / A.chunk;
  for (int t = 0, q = cid, tq = 0; q < n_chunks; ) {
    t = q * A.chunk + tq;
    if (++tq == A.chunk || t + 1 >= n_tiles) { tq = 0; q += ncl; }
    if (t >= n_tiles) continue;
    const I8Tile tl = tile_of(t, A, ntiles);
    const int s = P.active[tl.slot];
    const int p = P.st_p[s];
    if (tl.ht * kRowsTile >= p) continue;                          // uniform across the CTA (pair)
    const int ks_lo = tl.ks * per, ks_hi = min(nkt, ks_lo + per);
    const int nk = max(0, ks_hi - ks_lo);
    if (nk == 0) continue;
    const int W = i8_tile_width(tl.nt, ntiles, NT, P.i8_NT_last);
    const int nsl = ring_slots(W, S);
    if (s != cur_s) {
      const long long ct0 = PROF ? clock64() : 0;
      // root limb table of this signal's prime (written by the prep kernel) and its phase indices u_j: three
      // bulk copies once every warp is done with the previous signal's table
      __syncthreads();
      if (tid == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        const uint32_t nt = 2 * (uint32_t)p - 1;                       // T twice + the W_p[0] entry
        const uint32_t blo = (nt * 8 + 15) & ~15u, bhi = S > 4 ? ((nt * 4 + 15) & ~15u) : 0u;
        const uint32_t bu = ((uint32_t)nkt * kI8StepTerms * 4 + 15) & ~15u;     // i8_elog rows hold kk + 16
        tc::mbar_expect_tx(tabbar, blo + bhi + bu);
        const int64_t tab0 = (int64_t)P.st_slot[s] * P.i8_tstride;     // the signal's table slot
        tc::bulk_g2s(sTlo, P.i8_tlo + tab0, blo, tabbar);
        if (bhi) tc::bulk_g2s(smem_raw + A.thi_off, P.i8_thi + tab0, bhi, tabbar);
        tc::bulk_g2s(sU, P.i8_elog + (int64_t)s * P.i8_estride, bu, tabbar);
      }
      tc::mbar_wait(tabbar, tabphase);
      tabphase ^= 1;
      cur_s = s;
      (void)ct0;
    }

    if (warp < kI8GenWarps) {
      // ---------------- A generators + epilogue: warp g owns TMEM lanes / rows 32 (g % 4) .., terms 8 (g / 4) ..
      const int quarter = warp & 3, half = warp >> 2;
      const int row = 32 * quarter + lane;
      const unsigned h = (unsigned)(tl.ht * kRowsTile + (int)rank * kI8Rows + row);   // row f (discrete-log order)
      const uint32_t lane_addr = tbase + ((uint32_t)(32 * quarter) << 16);
      const uint32_t ta0 = lane_addr + (uint32_t)(S * W) + 4 * half;
      // software pipeline: the limbs of step kq + 1 are gathered while the tensor core works on step kq and
      // before the slot they go to is free; only the TMEM store + arrive sit on the critical path
      uint32_t w[S][4];
      const int* ub = sU + ks_lo * kI8StepTerms + 8 * half;
      const bool special = (int)h >= p - 1;                         // h = 0 row or padding: all roots 1
      if (A.dbg != 3) gen_limbs<S>(w, ub, sTlo, sThi, (int)h, special, 2 * (p - 1), A.dbg);
      int sl = 0;
      for (int kq = 0; kq < nk; ++kq, sl = (sl + 1 == nsl ? 0 : sl + 1)) {
        const long long c0 = PROF ? clock64() : 0;
        if (A.gnap) {
          while (!tc::mbar_try_wait(aempty + sl, ((aring >> sl) & 1) ^ 1)) __nanosleep(A.gnap);
        } else {
          tc::mbar_wait(aempty + sl, ((aring >> sl) & 1) ^ 1);
        }
        aring ^= 1u << sl;
        if (PROF) pr_a += clock64() - c0;
        const uint32_t ta = ta0 + sl * S * 8;
#pragma unroll
        for (int t = 0; t < S; ++t) tc::tmem_st4(ta + 8 * t, w[t]);
        tc::tmem_wait_st();
        tc::fence_before_sync();
        __syncwarp();
        if (lane == 0) arrive_afull(sl, false);
        const long long cg = PROF ? clock64() : 0;
        if (PROF) pr_t += cg - c0 - (pr_a - pr_a);                   // store + arrive (incl. the slot wait, see pr_a)
        if (kq + 1 < nk && A.dbg != 3)
          gen_limbs<S>(w, ub + (kq + 1) * kI8StepTerms, sTlo, sThi, (int)h, special, 2 * (p - 1), A.dbg);
        if (PROF) pr_g += clock64() - cg;
      }
      // epilogue: sum the S weights in FP64 (lowest first); the two warps of a lane quarter take alternate
      // 16-column chunks
      double2* out;
      int64_t pstr;
      if (A.ksplit == 1) {
        out = P.lines + (int64_t)s * P.L * P.p_stride;
        pstr = P.p_stride;
      } else {
        out = part + ((int64_t)tl.ks * A.n_slots + tl.slot) * P.L * (int64_t)A.p_part;
        pstr = A.p_part;
      }
      const double scale = P.i8_sigma[s] / (127.0 * 127.0);
      const long long ce0 = PROF ? clock64() : 0;
      tc::mbar_wait(accfull, ntile_done & 1);
      tc::fence_after_sync();
      const bool live = h < (unsigned)p;
      for (int c0 = 16 * half; c0 < W; c0 += 32) {
        int32_t v[16];
        double acc[16];
        tc::tmem_ld16(lane_addr + (uint32_t)((S - 1) * W + c0), v);
        tc::tmem_wait_ld();
        const double f0 = ldexp(1.0, -8 * (S - 1));
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[i] = (double)v[i] * f0;
        for (int w = S - 2; w >= 0; --w) {
          tc::tmem_ld16(lane_addr + (uint32_t)(w * W + c0), v);
          tc::tmem_wait_ld();
          const double f = ldexp(1.0, -8 * w);
#pragma unroll
          for (int i = 0; i < 16; ++i) acc[i] = fma((double)v[i], f, acc[i]);
        }
        const int n0 = (tl.nt * NT + c0) >> 1;
        if (live) {
#pragma unroll
          for (int i = 0; i < 8; ++i)
            if (n0 + i < P.L) out[(int64_t)(n0 + i) * pstr + h] = make_double2(acc[2 * i] * scale, acc[2 * i + 1] * scale);
        }
      }
      if (PROF) pr_e += clock64() - ce0;
      tc::fence_before_sync();
      __syncwarp();
      if (lane == 0) arrive_accempty();
    } else if (warp == kI8ProdWarp) {
      // ---------------- B producer: one lane streams the B limb tiles (backs off while the ring is full)
      // PAIR: this CTA's half of the columns, [rank W/2, (rank + 1) W/2), stored after the other half
      const uint32_t bytes = (uint32_t)S * (PAIR ? W / 2 : W) * 32;
      const int8_t* Bg = P.i8_B + (int64_t)s * nks * S * 32 * cols + (int64_t)tl.nt * nks * S * NT * 32 + rank * bytes;
      for (int kq = 0; kq < nk; ++kq) {
        const int sb = bpos;
        bpos = bpos + 1 == A.nb ? 0 : bpos + 1;
        const uint32_t par = ((bring >> sb) & 1) ^ 1;
        bring ^= 1u << sb;
        if (lane == 0) {
          while (!tc::mbar_try_wait(bempty + sb, par)) __nanosleep(A.nap);
          tc::mbar_expect_tx(bfull + sb, bytes);
          tc::bulk_g2s(sB + (size_t)sb * A.b_stage_bytes, Bg + (int64_t)(ks_lo + kq) * S * W * 32, bytes,
                       bfull + sb);
        }
      }
    } else if (warp == kI8FwdWarp) {
      // ---------------- B forwarder: the 9th arrival on afull, once the step's B limbs have landed, so the MMA
      // issuer waits on one barrier per step without putting a second wait on a generator's critical path
      int sl = 0;
      for (int kq = 0; kq < nk; ++kq, sl = (sl + 1 == nsl ? 0 : sl + 1)) {
        const int sb = bpos;
        bpos = bpos + 1 == A.nb ? 0 : bpos + 1;
        const long long cb = PROF ? clock64() : 0;
        tc::mbar_wait(aempty + sl, ((aring >> sl) & 1) ^ 1);   // the slot's previous phase is over
        aring ^= 1u << sl;
        tc::mbar_wait(bfull + sb, (bring >> sb) & 1);
        bring ^= 1u << sb;
        if (PROF) pr_b += clock64() - cb;
        if (lane == 0) arrive_afull(sl, true);
      }
    } else if (!PAIR || rank == 0) {
      // ---------------- MMA issuer: the whole warp walks the ring, one elected lane issues
      const uint32_t idesc = tc::idesc_i8(kRowsTile, W);
      if (ntile_done > 0) {
        const long long c0 = PROF ? clock64() : 0;
        tc::mbar_wait(accempty, (ntile_done - 1) & 1);
        if (PROF) pr_e += clock64() - c0;
        tc::fence_after_sync();
      }
      const uint64_t bdesc0 = tc::sdesc_kmajor(tc::smem_u32(sB), 128, 256);
      const uint32_t stage_desc = A.b_stage_bytes >> 4, a_slot0 = tbase + (uint32_t)(S * W);
      int sl = 0;
      for (int kq = 0; kq < nk; ++kq) {
        const int sb = bpos;
        bpos = bpos + 1 == A.nb ? 0 : bpos + 1;
        const long long c1 = PROF ? clock64() : 0;
        tc::mbar_wait(afull + sl, (aring >> sl) & 1);      // implies bfull (the forwarder waited for it)
        aring ^= 1u << sl;
        if (PROF) pr_a += clock64() - c1;
        tc::fence_after_sync();
        if (tc::elect_one()) {
          if (A.dbg != 2)
            issue_stage<S, PAIR>(tbase, a_slot0 + sl * S * 8, bdesc0 + (uint64_t)(sb * stage_desc), (uint32_t)W,
                                 (uint32_t)(PAIR ? W : W * 2), idesc, kq == 0);
          if (PAIR) {
            tc::mma_commit2(bempty + sb);
            tc::mma_commit2(aempty + sl);
          } else {
            tc::mma_commit(bempty + sb);
            tc::mma_commit(aempty + sl);
          }
        }
        __syncwarp();
        sl = sl + 1 == nsl ? 0 : sl + 1;
      }
      if (tc::elect_one()) {
        if (PAIR) tc::mma_commit2(accfull);
        else tc::mma_commit(accfull);
      }
      __syncwarp();
    }
    ++ntile_done;
  }
  if (PROF && lane == 0 && (warp == 0 || warp == kI8MmaWarp)) {
    long long* o = A.prof + (blockIdx.x * 2 + (warp == 0 ? 0 : 1)) * 6;
    o[0] = clock64() - pr_start; o[1] = pr_a; o[2] = pr_b; o[3] = pr_e; o[4] = pr_t; o[5] = pr_g;
  }
  tc::fence_before_sync();
  __syncthreads();
  if (PAIR) tc::cluster_sync();                                        // the peer's MMAs read this CTA's TMEM
  if (warp == kI8MmaWarp) {
    tc::fence_after_sync();
    if (PAIR) tc::tmem_dealloc2<512>(tbase);
    else tc::tmem_dealloc<512>(tbase);
  }
}

// ------------------------------------------------------------------ host side
// Limb count (reading R22): S = 6 keeps every sample within the stage-parity bar 1e-12 sum |c| of
// SURVEY 4 layer 5 (measured; S = 5 missed it for short lines, K = 6: 8e-12 vs 6e-12) and coefficient errors
// ~1e-14 relative; FP64 roots cannot feed more than E = 2^36 (the Eq. (41) decode then needs the FP64 path).
int i8_limbs_for(int64_t E) {
  if (E <= ((int64_t)1 << 36)) return 6;
  return 0;   // beyond what FP64 roots can feed: use the FP64 tensor (DMMA) path
}

// n-tiles: widths NT (multiple of 16) except a narrower last one; every tile keeps its S accumulators plus
// at least 2 ring slots (S * 8 columns each) in the 512 TMEM columns.  Cost model per (128 rows, 16 terms):
// MMA cycles S (S + 1) / 2 * W / 2 per tile, A generation ~250 cycles per tile (overlapped) and a fixed
// ~120 cycles of ring overhead per stage.
bool i8_configure(int L, int64_t E, int k, I8Config* out) {
  I8Config c{};
  c.S = i8_limbs_for(E);
  if (c.S == 0 || getenv("SFFT_NO_I8")) return false;
  // exact int32 accumulation (header): S * 2K * 2^14 < 2^31 for the K = k signal terms of a line
  if ((int64_t)c.S * 2 * k * 16384 >= ((int64_t)1 << 31)) return false;
  const int N2 = 2 * L;
  // very few lines (2L <= 16): one N = 16 MMA per limb product is mostly padding and the A generation
  // dominates; the FP64 kernels are faster there (measured on C2, L = 3) unless forced (expsum_path = 2)
  if (N2 <= 16 && !getenv("SFFT_I8_SMALL_L")) c.small_l = 1;
  const int prods = c.S * (c.S + 1) / 2;
  const int nt_cap = std::min(96, ((512 - 2 * 8 * c.S) / c.S) / 16 * 16);   // 96: limbs kernel staging
  int force = getenv("SFFT_I8_NT") ? atoi(getenv("SFFT_I8_NT")) : 0;
  double best = 1e30;
  for (int NT = 16; NT <= nt_cap; NT += 16) {
    if (force && NT != force) continue;
    const int nt = (N2 + NT - 1) / NT;
    const int last = ((N2 - (nt - 1) * NT) + 15) / 16 * 16;
    double cost = 0;
    for (int i = 0; i < nt; ++i) {
      const int W = i == nt - 1 ? last : NT;
      cost += std::max(prods * W / 2.0, 250.0) + 120.0;
    }
    if (cost < best - 1e-9) { best = cost; c.NT = NT; c.ntiles = nt; c.NT_last = last; }
  }
  if (c.NT == 0) return false;
  c.nks = (2 * k + kI8StepTerms - 1) / kI8StepTerms;
  // CTA pairs (cta_group::2) are exact (parity-tested) but not the default: the peer CTA's arrivals on the
  // leader's barriers cost ~500 cycles each with release semantics, which the two A slots of a 64-column tile
  // cannot hide (measured: 2.38 ms vs 1.93 ms for the C3 iteration-1 exp-sum); SFFT_I8_PAIR=1 enables them.
  c.pair = (c.NT_last >= 32 && c.NT >= 32 && getenv("SFFT_I8_PAIR") && atoi(getenv("SFFT_I8_PAIR")) == 1) ? 1 : 0;
  *out = c;
  return true;
}

size_t i8_limb_bytes(const I8Config& c, int batch) {
  const int cols = (c.ntiles - 1) * c.NT + c.NT_last;
  return (size_t)batch * c.nks * c.S * 32 * (size_t)cols;
}

static size_t i8_smem(const I8Config& c, int p, int nkt, int nb, uint32_t* tab_off, uint32_t* thi_off,
                      uint32_t* u_off) {
  size_t o = 512 + (size_t)nb * c.S * c.NT * 32;
  o = (o + 15) & ~(size_t)15;
  *tab_off = (uint32_t)o;
  const size_t nt = 2 * (size_t)p - 1;                                  // T twice + the W_p[0] entry
  o += (nt * 8 + 15) & ~(size_t)15;
  *thi_off = (uint32_t)o;
  o += c.S > 4 ? ((nt * 4 + 15) & ~(size_t)15) : 0;
  *u_off = (uint32_t)o;
  o += (size_t)nkt * kI8StepTerms * 4 + 16;
  return o;
}

bool i8_fits(const I8Config& c, int p, int k, int smem_optin) {
  uint32_t a, b, d;
  const int nkt = (k + kI8StepTerms - 1) / kI8StepTerms;
  return i8_smem(c, p, nkt, 2, &a, &b, &d) <= (size_t)smem_optin;
}

int i8_blocks(const I8Config& c, int32_t max_p, int32_t n_signals) {
  const int rows = c.pair ? 2 * kI8Rows : kI8Rows;                      // tiles of one persistent unit (CTA or pair)
  return n_signals * ((max_p + rows - 1) / rows) * c.ntiles;
}

cudaError_t launch_i8_prepare(const DevParams& P, int32_t n_signals, int32_t K, cudaStream_t st, bool only_retilted) {
  if (!only_retilted) i8_sigma_kernel<<<n_signals, 256, 0, st>>>(P, K);   // |a_j| do not change on a retilt
  const int64_t ctas = (int64_t)n_signals * P.i8_ntiles * ((K + kI8StepTerms - 1) / kI8StepTerms);
  if (ctas > 0) {
    auto kern = P.i8_S == 6 ? i8_limbs_kernel<6> : i8_limbs_kernel<5>;      // i8_limbs_for: S is 5 or 6
    return launch_pdl(kern, dim3((unsigned)ctas), dim3(256), 0, st, P, K, only_retilted ? 1 : 0);
  }
  return cudaGetLastError();
}

// stage entry point: lines of signal 0 from discrete-log order back to natural order, out [L][p]
__global__ void i8_unpermute_kernel(DevParams P, int32_t p, double2* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)P.L * p) return;
  const int n = (int)(i / p), f = (int)(i % p);
  out[(int64_t)n * p + P.i8_pw[(int64_t)P.st_slot[0] * P.i8_tstride + f]] = P.lines[(int64_t)n * P.p_stride + f];
}

cudaError_t launch_i8_unpermute(const DevParams& P, int32_t p, double* out, cudaStream_t st) {
  const int64_t tot = (int64_t)P.L * p;
  if (tot > 0) i8_unpermute_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(P, p, reinterpret_cast<double2*>(out));
  return cudaGetLastError();
}

cudaError_t launch_expsum_i8(const DevParams& P, const I8Config& c, int32_t max_p, int32_t n_signals, int32_t ksplit,
                             double2* part, int32_t p_part, int smem_optin, cudaStream_t st) {
  I8Args A{};
  A.n_htiles = (max_p + kI8Rows - 1) / kI8Rows;
  A.ksplit = ksplit;
  A.p_part = p_part;
  A.n_slots = n_signals;
  A.dbg = getenv("SFFT_I8_DBG") ? atoi(getenv("SFFT_I8_DBG")) : 0;
  A.nap = getenv("SFFT_I8_NAP") ? atoi(getenv("SFFT_I8_NAP")) : 256;
  // generators sleep 64 ns between polls of a full A ring instead of spinning (their polls compete with the
  // gathers of the generators that do have a slot; C3 / C5 exp-sum -0.5 % / -0.6 %, profiles/r02_experiments.md)
  A.gnap = getenv("SFFT_I8_GNAP") ? atoi(getenv("SFFT_I8_GNAP")) : 64;
  A.relaxed = getenv("SFFT_I8_RELAXED") ? atoi(getenv("SFFT_I8_RELAXED")) : 0;
  static long long* prof_buf = nullptr;
  if (getenv("SFFT_I8_PROF")) {
    if (!prof_buf) cudaMalloc(&prof_buf, sizeof(long long) * 148 * 2 * 6);
    cudaMemsetAsync(prof_buf, 0, sizeof(long long) * 148 * 2 * 6, st);
    A.prof = prof_buf;
  }
  A.b_stage_bytes = (uint32_t)c.S * c.NT * 32;
  const int nkt = (P.i8_K + kI8StepTerms - 1) / kI8StepTerms;
  size_t smem = 0;
  for (A.nb = kI8MaxSlots; A.nb >= 2; --A.nb) {
    smem = i8_smem(c, max_p, nkt, A.nb, &A.tab_off, &A.thi_off, &A.u_off);
    if (smem <= (size_t)smem_optin) break;
  }
  if (A.nb < 2) return cudaErrorInvalidValue;
  // one CTA per SM: the kernel allocates all 512 TMEM columns
  smem = std::max(smem, (size_t)120 * 1024);
  const bool pair = P.i8_pair != 0;
  void (*kern)(DevParams, I8Args, double2*, int32_t);
  if (pair) kern = c.S == 5 ? (A.prof ? expsum_i8_kernel<5, true, true> : expsum_i8_kernel<5, false, true>)
                            : (A.prof ? expsum_i8_kernel<6, true, true> : expsum_i8_kernel<6, false, true>);
  else kern = c.S == 5 ? (A.prof ? expsum_i8_kernel<5, true, false> : expsum_i8_kernel<5, false, false>)
                       : (A.prof ? expsum_i8_kernel<6, true, false> : expsum_i8_kernel<6, false, false>);
  cudaError_t e = ensure_smem(kern, smem);
  if (e != cudaSuccess) return e;
  if (pair) {
    A.n_htiles = (max_p + 2 * kI8Rows - 1) / (2 * kI8Rows);            // 256-row tiles of the pair
  }
  const long tiles = (long)n_signals * A.n_htiles * c.ntiles * ksplit;
  int n_sm = 148;
  cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, 0);
  const long units = pair ? n_sm / 2 : n_sm;                            // persistent CTAs (pairs)
  // chunks of consecutive tiles per CTA visit keep a signal's root table in the CTA (measured, C3 / C4 / C5:
  // 2 tiles when the columns span several n-tiles, one tile otherwise; 4 and more lengthen the tail)
  A.chunk = getenv("SFFT_I8_CHUNK") ? std::max(1, atoi(getenv("SFFT_I8_CHUNK"))) : (c.ntiles >= 2 ? 2 : 1);
  const long grid = std::min<long>((tiles + A.chunk - 1) / A.chunk, units) * (pair ? 2 : 1);
  if (grid > 0) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(kI8Threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = pair ? 2 : 1;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    e = cudaLaunchKernelEx(&cfg, kern, P, A, part, (int32_t)tiles);
    if (e != cudaSuccess) return e;
  }
  if (A.prof && grid > 0) {
    long long h[148 * 2 * 6];
    cudaMemcpyAsync(h, A.prof, sizeof h, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    double g[6] = {0}, m[6] = {0};
    for (int b = 0; b < grid; ++b)
      for (int i = 0; i < 6; ++i) { g[i] += h[b * 12 + i]; m[i] += h[b * 12 + 6 + i]; }
    fprintf(stderr, "[i8prof] p=%d NT=%d/%d x%d | gen(warp 0): total %.0f slot-wait %.0f bfull-wait %.0f "
            "store+arrive %.0f gather %.0f epilogue %.0f | mma: total %.0f afull-wait %.0f accempty %.0f (cycles per CTA)\n",
            max_p, c.NT, c.NT_last, c.ntiles, g[0] / grid, g[1] / grid, g[2] / grid, (g[4] - g[1]) / grid, g[5] / grid,
            g[3] / grid, m[0] / grid, m[1] / grid, m[3] / grid);
  }
  return cudaGetLastError();
}

}  // namespace sfft
