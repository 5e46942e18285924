// sfft_internal.cuh -- shared declarations of the sm_100a implementation of the
// multidimensional phase-shift sparse FFT (arXiv 1606.07407, Algorithm 2).
// Nothing here is shared with oracle/ (test infrastructure); the two are independent.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include <algorithm>
#include <string>
#include <vector>

#include "../../include/sfft.h"

namespace sfft {

// ---- per-signal run state (device) -----------------------------------------------------
enum : int32_t { ST_RUN = 100 };   // final states use sfft_status values (0 OK, 1 PARTIAL, <0 error)

constexpr int kMaxFftPasses = 24;
// smallest FFT size whose passes run warp-local after the first (k_fft.cu pass_loop_w): smaller sizes run as
// many short CTAs (C4's M = 1008 at 96 threads), where block-wide passes measured faster
constexpr int kFftWlMinM = 4096;
// fft_radix[fi][kFftVwSlot]: W of a warp-local plan, whose kernel spectrum is also stored warp-blocked in VB (middle
// group g of warp region w, element k at w Mw + k G + g, G = Mw / R: lanes read consecutive entries), 0: none
constexpr int kFftVwSlot = kMaxFftPasses - 1;
inline int fft_wl_min() {   // SFFT_FFT_WL_MIN: tuning override of kFftWlMinM (host decisions: plans, launches)
  static const int v = getenv("SFFT_FFT_WL_MIN") ? atoi(getenv("SFFT_FFT_WL_MIN")) : kFftWlMinM;
  return v;
}
constexpr int kDecodeThreads = 1024;
constexpr int kLogIters = 64;
constexpr int kMaxFallbackLevels = 67;   // sfft_options.fallback_tilts: 4 fixed-stride tilt levels + 63 round-robin rounds
constexpr int kDefaultTableSlots = 512;  // per-prime table cache slots when sfft_options.table_cache_slots = 0
constexpr int kMaxPeers = 8;             // line shards of a fused record exchange (one node)
constexpr int kFusedMaxL = 8;            // lines per signal up to which FP64 plans sample inside the FFT CTAs

// Everything a kernel needs, passed by value (kernel parameter space).
struct DevParams {
  // problem
  int32_t d, k, r, L, Lp;     // L = r + 1 lines, Lp = padded line count of C rows
  int32_t kk;                  // term capacity per signal = 2k (k signal + k registry)
  int32_t H;                   // hash table slots per signal (pow2 >= 2k)
  int32_t batch;
  int64_t N, E;
  int32_t c, max_iter, stall_limit, extra, n_sched;
  int32_t literal;             // 1: registry terms sampled with the signal (K = k + |R|); 0: bin-domain g
  double tol, floor_rel, prune, round_tol;
  int32_t n_tilts;
  int32_t p_cap;               // largest prime the FFT size table supports
  int64_t p_stride, M_stride;  // line stride (>= p_cap), Bluestein buffer stride (>= M_max)
  // small tables (device)
  const int32_t* block_dims;   // [r]
  const int32_t* block_off;    // [r]
  const int64_t* lo;           // [r] image interval of every (tilted) axis
  const int64_t* hi;           // [r]
  const int64_t* tilts;        // [n_tilts][5]
  const int32_t* axis_tilt;    // [r] 2*tilt+slot of a tilted axis, -1 otherwise
  const int64_t* sched;        // [n_sched] explicit primes or null
  const int32_t* primes;       // sorted primes <= p_cap
  int32_t n_primes;
  const int32_t* pfirst;       // [n_pfirst] index of the first prime >= x (x < n_pfirst; beyond: none)
  int32_t n_pfirst;
  const int32_t* fft_M;        // [n_fft] allowed Bluestein sizes, ascending
  const int8_t* fft_radix;     // [n_fft][kMaxFftPasses]
  const int32_t* fft_npass;    // [n_fft]
  const int32_t* fft_tw_off;   // [n_fft][kMaxFftPasses] offsets of the per-pass twiddle tables
  const double2* fft_tw;       // all per-pass twiddle tables
  int32_t n_fft;
  // buffers (device)
  int64_t* v_all;              // [batch][r][kk]
  double2* C_all;              // [batch][kk][Lp]
  int2* u_all;                 // [batch][kk] (v_{j,m} mod p, 8 v_{j,m} mod p) of the current iteration
  double2* lines;              // [batch][L][p_stride]
  double2* W_tab;              // [batch][p_stride]   e^{+2 pi i q/p}
  double2* chirp;              // [batch][p_stride]   e^{-pi i (q^2 mod 2p)/p}
  double2* V;                  // [batch][M_stride]   DIF spectrum of the Bluestein kernel / M
  double2* VB;                 // [slots][M_stride]  the same, warp-blocked for the warp-local middle (kFftVwSlot)
  double2* a_reg;              // [batch][k]
  uint64_t* key_hash;          // [batch][k]
  int32_t* htab;               // [batch][H]  entry index + 1, 0 = empty
  int64_t* acc_v;              // [batch][r][k] scratch of decoded coordinates (per candidate)
  double2* acc_a;              // [batch][k]
  int32_t* wtmp;               // [batch][k][d] wrap scratch
  // state (device)
  int32_t* st_status;          // [batch]
  int32_t* st_nR;              // [batch]
  int32_t* st_p;               // [batch]
  int32_t* st_m;               // [batch]
  int32_t* st_M;               // [batch] Bluestein size index into fft tables
  int32_t* st_stall;           // [batch]
  int32_t* st_iters;           // [batch]
  int64_t* st_samples;         // [batch]
  int64_t* st_cmacs;           // [batch]
  int64_t* st_cmacs_i8;        // [batch] cMACs of the iterations whose exp-sum ran on the int8-limb kernel
  double* st_fftw;             // [batch][2] sums over iterations of L p log2(p) and L M log2(M) (Bluestein sizes)
  int32_t i8_iter;             // decode launch: this iteration's exp-sum used the int8-limb kernel
  int32_t* st_log;             // [kLogIters][2] (p, accepted) of signal 0
  int32_t* ctrl;               // [8]: n_active, max_p, max_K, fills, setup CTAs done (this iteration's block)
  int32_t* ctrl_next;          // [8]: the next iteration's block, cleared by the table prep
  int32_t* h_ctrl_map;         // host-mapped [4]: n_active, max_p, max_K, sequence ^ ctrl_mix (setup_kernel)
  int32_t* active;             // [batch] indices of the signals still running this iteration
  // per-prime tables (W_tab, chirp, V, int8 root tables) live in a cache of slots keyed by p: they depend on p
  // only, like FFT twiddles; slot n_tslots is reserved for the stage entry points
  int32_t n_tslots;
  int32_t* st_slot;            // [batch] slot of the signal's current prime
  int32_t* slot_p;             // [n_tslots] prime held by the slot, 0 = empty
  int32_t* slot_epoch;         // [n_tslots] last iteration epoch that used the slot
  int32_t* fill;               // [n_tslots] slots to (re)compute this iteration, count in ctrl[3]
  int32_t* fill_by;            // [n_tslots] active index of the CTA that refills the slot (prep_iter_kernel)
  int32_t* fill_ep;            // [n_tslots] epoch in which the slot is refilled
  int32_t* slot_ready;         // [n_tslots] epoch stamp released once the slot's tables are written
  int32_t* assign_ready;       // [1] epoch stamp released after the slot assignment
  int32_t* spin_err;           // [1] set when a stamp wait timed out (the execute fails instead of hanging)
  // stall fallback (reading R23): level 0 = the plan's own tilts and E, levels 1.. = fallback tilts
  int32_t n_levels, lvl_tmax;  // levels, tilt slots per level
  const int64_t* lvl_E;        // [n_levels]
  const int64_t* lvl_lo;       // [n_levels][r] decodable image of every axis
  const int64_t* lvl_hi;       // [n_levels][r]
  const int64_t* lvl_tilts;    // [n_levels][lvl_tmax][5] (axis0, axis1, base, height, hypo)
  const int32_t* lvl_nt;       // [n_levels] tilts per level
  const int32_t* lvl_axt;      // [n_levels][r] 2*tilt+slot of a tilted axis, -1 otherwise
  int32_t* st_lvl;             // [batch] current level
  int32_t* st_il;              // [batch] iteration counter of the current level (Alg. 3 l.5)
  int32_t* st_retilt;          // [batch] 1: switched level in the last decode, re-project before the next setup
  // int8-limb tensor-core exp-sum (k_expsum_i8.cu)
  int32_t i8_S, i8_NT, i8_NT_last, i8_ntiles, i8_nks;   // limbs, n-tile width (last tile narrower), n-tiles, K-step capacity
  int32_t i8_K;                // terms held in the B limbs (k for a solve, K for the stage entry point)
  int32_t i8_pair;             // 1: CTA pairs (cta_group::2, M = 256); B limbs stored as two column halves
  int8_t* i8_B;                // [batch][ntiles][nks][S][NT*32] B limbs in the UMMA K-major layout
  double* i8_sigma;            // [batch] coefficient scale
  // rows in discrete-log order (reading R22): f < p-1 is the sample h = g^f mod p (g a primitive root of p),
  // f = p-1 is h = 0; term j enters as its discrete log e_j = log_g(u_j) (-1 when u_j = 0), so the root of
  // (f, j) is entry (f + e_j) mod (p-1) of the table T[f] = W_p[g^f] (T[p-1] = W_p[0] = 1)
  uint2* i8_tlo;               // [batch][i8_tstride] T[f] limbs 0..3 (16 bit each: re | im << 8)
  uint32_t* i8_thi;            // [batch][i8_tstride] T[f] limbs 4..5
  int32_t* i8_pw;              // [batch][i8_tstride] h of row f: g^f mod p (f < p-1), 0 (f = p-1)
  double2* i8_chl;             // [batch][i8_tstride] Bluestein chirp in row order: chirp[pw[f]]
  int32_t* i8_dlog;            // [batch][i8_tstride] scratch: log_g(x)
  int32_t* i8_elog;            // [batch][i8_estride] e_j of the iteration's terms
  int32_t i8_estride;          // >= kk + 16, multiple of 4
  int32_t lines_log;           // launch flag: the lines hold samples in discrete-log order (int8 exp-sum)
  // fused sampling for short lines (plans whose exp-sum runs on the FP64 kernels with few lines):
  // the FFT CTA of (signal, line n) computes its own samples s_n in shared memory -- rows in discrete-log order,
  // root of (f, j) = dl_root[f + e_j] (FP64, the i8 tables' layout) -- so the lines never reach HBM
  int32_t log_tables;          // the discrete-log tables (i8_pw, i8_dlog, i8_chl, e_j in i8_elog) are built
  double2* dl_root;            // [n_tslots][i8_tstride] W_p[g^f] twice + W_p[0] (FP64), or null
  int32_t fused_sample;        // pfft launch flag: compute the samples in the FFT CTA (no exp-sum launch)
  int32_t fused_load;          // pfft launch: largest FFT size whose first DIF pass gathers its discrete-log line
  int64_t i8_tstride;          // >= p_stride + 8 (bulk copies round the table up to 16 bytes)
  // line sharding: shard line_g of line_G holds line 0 and the shifted lines of reduced axes
  // [line_lo, line_lo + L - 1); its decode is split into a local test (records) and a commit after the
  // all-gather of the records.  Unsharded plans: line_G = 1, line_lo = 0, L = r + 1, no records.
  int32_t line_lo, line_G, line_g;
  int32_t rec_words;           // int64 words per signal record: rec_fw flag words (int32 pairs) + (Lmax - 1) k coordinates
  int32_t rec_fw;              // (k + 1) / 2
  int64_t* rec_send;           // [batch][rec_words] this shard's records
  const int64_t* rec_recv;     // [line_G][batch][rec_words] all shards' records (all-gather result)
  int32_t* rec_cand;           // [batch][k] candidate bins of the local phase (identical on every shard)
  int32_t* rec_nc;             // [batch] candidate count
  double2* rec_f0;             // [batch][k] F_0 at the candidates (residual included)
  // fused FFT epilogue: line-0 CTAs select the candidates and publish them
  // (sel_ready[s] = it_epoch, release); line-n CTAs wait for it (acquire), then test + decode their line
  int32_t fuse_decode;         // launch flag of pfft_kernel (0: write the lines, stage entry point)
  int32_t it_epoch;            // iteration stamp (plan-wide counter, never repeats within a plan)
  int32_t fuse_commit;         // pfft launch flag: the last CTA of a signal to finish runs its commit (a7)
  int32_t cur_iter;            // the iteration of that launch (the commit's state / log)
  int32_t* commit_cnt;         // [batch] arrival counters of the fused commit (reset by the last CTA)
  // C rows of the entries an iteration touched, spread over the GPU (crow_kernel, k_decode.cu) instead of in the
  // commit CTA: the commit lists the touched entries and appends work items (32 entries x 16 lines) counted in
  // ctrl[5]
  int32_t crow_mode;           // launch flag of the commit kernel (0: the commit writes the rows itself)
  // multi-prime speculation (reading R26): G primes per iteration, the commit merging G record sets.  On one GPU
  // (spec_slots = G) slot s holds signal s / G with the prime of counter (i - 1) G + s % G + 1 and the sets are the
  // sibling slots'; distributed (spec_dist, spec_slots = 1) rank spec_rank holds counter (i - 1) G + spec_rank + 1
  // and the sets arrive by the all-gather of every rank's records, whose tail (word spec_tail) carries the
  // candidate count, p, m, the candidate bins and F_0 there
  int32_t spec_G;              // 1 = Alg. 2 as written
  int32_t spec_slots;          // slots per signal on this GPU (G, or 1 when distributed)
  int32_t spec_dist, spec_rank, spec_tail;
  int32_t* spec_touch;         // [slots][k] (iteration << 4) | set of the last update of entry e
  int32_t crow_nl;             // 16-line chunks per row, ceil(Lp / 16)
  int4* crow_items;            // [batch * ceil(k / 32) * crow_nl] (signal, entry chunk, line chunk, touched count)
  int32_t* crow_list;          // [batch][k] touched entry indices of the iteration, ascending b
  int32_t* sel_ready;          // [batch]
  // fused record exchange (sfft_options.line_exchange = 1): the FFT epilogue stores its record words straight into
  // the receive buffer of every shard (peer memory: CUDA IPC mappings across GPUs, plain pointers on one device)
  // and releases a per-(shard, local line, signal) stamp = peer_epoch on every shard; the commit acquires all
  // r + G stamps of its signal instead of waiting for a separate all-gather
  int32_t peer_mode;
  int32_t peer_epoch;          // iteration stamp of the exchange (the same sequence on every shard, starts at 1)
  int64_t* peer_recv[kMaxPeers];   // receive buffer [line_G][batch][rec_words] of shard h
  int32_t* peer_stamp[kMaxPeers];  // stamps [line_G][L_ref][batch] of shard h
  int32_t* stamp_local;        // this shard's own stamps (the commit waits on them)
  int32_t L_ref;               // lines of shard 0 (the largest shard; the stamp row stride)
  int32_t* bin_start;          // [batch][p_stride + 1] registry entries of bin b: bin_order[bin_start[b] .. [b+1])
  int32_t* bin_order;          // [batch][k] registry entry indices grouped by bin, ascending e within a bin
};

// reduced axes [lo, hi) of line shard g of G over r axes (contiguous, sizes differ by at most one; shard 0 largest)
__host__ __device__ inline void line_shard_range(int r, int G, int g, int* lo, int* hi) {
  const int base = r / G, extra = r % G;
  *lo = g * base + (g < extra ? g : extra);
  *hi = *lo + base + (g < extra ? 1 : 0);
}

// balanced base-256 digits of X (|X| <= 127 * 256^(S-1)), most significant first (k_expsum_i8.cu, k_fft.cu)
__device__ __forceinline__ void i8_digits(int64_t X, int S, int (&d)[8]) {
  for (int t = S - 1; t >= 0; --t) {
    const int64_t r = ((X + 128) & 255) - 128;
    d[t] = (int)r;
    X = (X - r) >> 8;
  }
}
// limb-table entry of the root (c, s) = e^{2 pi i q / p}: limb t of (re, im) as the 16-bit word re_t | im_t << 8
__device__ __forceinline__ void i8_root_entry(double c, double s, int S, uint2& lo, uint32_t& hi) {
  const double qa = 127.0 * ldexp(1.0, 8 * (S - 1));
  int dr[8], di[8];
  i8_digits(llrint(c * qa), S, dr);
  i8_digits(llrint(s * qa), S, di);
  uint32_t e[6];
#pragma unroll
  for (int i = 0; i < 6; ++i) e[i] = i < S ? ((uint32_t)(uint8_t)dr[i] | ((uint32_t)(uint8_t)di[i] << 8)) : 0u;
  lo = make_uint2(e[0] | (e[1] << 16), e[2] | (e[3] << 16));
  hi = e[4] | (e[5] << 16);
}

// int8-limb exp-sum configuration (host)
struct I8Config {
  int S, NT, NT_last, ntiles, nks;
  int small_l;   // 1: auto mode prefers the FP64 kernels (2L <= 16)
  int pair;      // 1: CTA-pair kernel (every tile width >= 32)
};

// check word of the host-mapped control block: one 16-byte store publishes (n_active, max_p, max_K,
// seq ^ ctrl_mix(n_active, max_p, max_K)) without a system-scope fence; the host accepts a 16-byte snapshot only when
// its check word matches the sequence number it waits for (a stale block carries an older sequence; a torn one
// fails the check)
__host__ __device__ inline uint32_t ctrl_mix(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t h = 0x27D4EB2Fu ^ (a * 0x9E3779B1u);
  h = (h ^ (h >> 15)) * 0x85EBCA77u + b;
  h = (h ^ (h >> 13)) * 0xC2B2AE3Du + c;
  h = (h ^ (h >> 16)) * 0x9E3779B1u;
  return h ^ (h >> 15);
}

// ---- device helpers ----------------------------------------------------------------------
__host__ __device__ inline int64_t mod_pos64(int64_t x, int64_t m) {
  int64_t q = x % m;
  return q < 0 ? q + m : q;
}
// the same for the usual case |x| < m (decodable coordinates: the plan keeps every image inside (-E/2, E/2))
// without a 64-bit division; falls back to mod_pos64 otherwise
__host__ __device__ __forceinline__ int64_t mod_near64(int64_t x, int64_t m) {
  const int64_t q = x < 0 ? x + m : x;
  return (q >= 0 && q < m) ? q : mod_pos64(x, m);
}
// e^{2 pi i (v mod E)/E} via sincospi of the exactly reduced rational 2 (v mod E) / E (line factor of a shift).
// E a power of two 2^t (every plan whose N is one): 2q / E = q * 2^(1-t) exactly, a multiply instead of the FP64
// division -- the same double bit for bit
__device__ __forceinline__ double2 line_factor_exact(int64_t v, int64_t E) {
  const int64_t q = mod_near64(v, E);
  double s, c;
  if ((E & (E - 1)) == 0) {
    const int t = 63 - __clzll((unsigned long long)E);
    sincospi((double)q * __longlong_as_double((long long)(1024 - t) << 52), &s, &c);
  } else {
    sincospi(2.0 * (double)q / (double)E, &s, &c);
  }
  return make_double2(c, s);
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) only when the kernel's limit on this device is below `bytes`
// (a host call per launch otherwise sits on the per-iteration critical path)
cudaError_t ensure_smem(const void* kern, size_t bytes);
template <class K>
inline cudaError_t ensure_smem(K* kern, size_t bytes) { return ensure_smem(reinterpret_cast<const void*>(kern), bytes); }

// Programmatic dependent launch for the per-iteration kernel chain: a kernel launched with launch_pdl may be
// scheduled while its predecessor drains; every such kernel calls pdl_wait() before touching anything the
// predecessor writes (griddepcontrol.wait returns immediately for a kernel launched without the attribute).
// SFFT_NO_PDL=1 turns the attribute off (A/B).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
inline bool pdl_enabled() {
  static const bool on = getenv("SFFT_NO_PDL") == nullptr;
  return on;
}
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// ---- launchers (each .cu file) ----------------------------------------------------------
// k_project.cu
cudaError_t launch_project(const DevParams& P, int32_t batch, const int32_t* freqs, const double* coeffs,
                           cudaStream_t st);
cudaError_t launch_line_coeffs(const DevParams& P, int32_t K, const double* c, cudaStream_t st);
// k_decode.cu
cudaError_t launch_setup(const DevParams& P, int32_t iter, cudaStream_t st, int32_t seq = 0);
// commit of an iteration: the records of the fused FFT epilogue (all line shards) -> registry update, state
cudaError_t launch_decode_commit(const DevParams& P, int32_t iter, int32_t max_p, int32_t n_active, cudaStream_t st);
// the C rows listed by this iteration's commits (P.crow_mode); grid = CTAs looping over the work items
cudaError_t launch_crow(const DevParams& P, int32_t grid, cudaStream_t st);
// re-projection of the signals that switched fallback level (reading R23); freqs = the execute's input
cudaError_t launch_retilt(const DevParams& P, int32_t batch, const int32_t* freqs, cudaStream_t st);
cudaError_t launch_stage_decode(const DevParams& P, int32_t kstar, int32_t* acc_b, int64_t* acc_v,
                                double* acc_a, int32_t* counts, cudaStream_t st);
size_t decode_smem_bytes(const DevParams& P, int32_t max_p);
// k_expsum.cu
// kind 0: vector DFMA kernel (lanes along h, TN lines per thread)
// kind 1: FP64 tensor-core kernel (mma.sync m8n8k4 f64 = DMMA; warp tile 8*MB h x 8*NB lines)
struct ExpsumShape { int kind, tn, wn, th, warps, bm, bn, nt, mb, nb; double est; };
ExpsumShape choose_expsum_shape(int L);
int expsum_blocks(const ExpsumShape& S, int32_t max_p, int32_t n_signals);
ExpsumShape expsum_for_p(const ExpsumShape& S, int32_t max_p);
int expsum_bk();
// ksplit > 1: terms split over ksplit CTAs; partial lines go to part[ks][slot][L][p_part] and are summed
// in fixed ks order by the FFT load (deterministic, no atomics)
cudaError_t launch_expsum(const DevParams& P, const ExpsumShape& S, int32_t max_p, int32_t n_signals,
                          int32_t ksplit, double2* part, int32_t p_part, cudaStream_t st, int* occ_out = nullptr);
int expsum_occupancy(const ExpsumShape& S, int32_t max_p);   // resident CTAs per SM
// k_expsum_i8.cu
int i8_limbs_for(int64_t E);
bool i8_configure(int L, int64_t E, int k, I8Config* out);
size_t i8_limb_bytes(const I8Config& c, int batch);
bool i8_fits(const I8Config& c, int p, int k, int smem_optin);
int i8_blocks(const I8Config& c, int32_t max_p, int32_t n_signals);
cudaError_t launch_i8_prepare(const DevParams& P, int32_t n_signals, int32_t K, cudaStream_t st,
                              bool only_retilted = false);
cudaError_t launch_i8_unpermute(const DevParams& P, int32_t p, double* out, cudaStream_t st);
cudaError_t launch_expsum_i8(const DevParams& P, const I8Config& c, int32_t max_p, int32_t n_signals, int32_t ksplit,
                             double2* part, int32_t p_part, int smem_optin, cudaStream_t st);
// k_fft.cu
#ifdef SFFT_FFT_PROF
cudaError_t fft_prof_read(unsigned long long* out, bool reset);   // tuning builds only
#endif
// smem_bytes: 16 * max over the sizes in use of (M + sum of the per-pass base-twiddle counts)
// per iteration: assign table slots to the active signals' primes (fills counted in ctrl[3]), compute the
// tables of new primes (grid n_signals, CTAs beyond the fill count exit; direct = stage entry point: fill the
// slot of every listed signal), then the per-signal term phases u_j / e_j and FFT size index
// the per-iteration table prep in one launch (slot assignment, fills of new primes, terms; prep_iter_kernel)
cudaError_t launch_prep_iter(const DevParams& P, int32_t n_bound, int32_t smem_bytes, cudaStream_t st, int32_t epoch);
cudaError_t launch_fft_prep(const DevParams& P, int32_t n_signals, int32_t smem_bytes, int32_t threads, int32_t big,
                            cudaStream_t st, int32_t epoch, bool direct = false);
// threads per FFT CTA for a size (more CTAs per SM for small M)
#ifndef SFFT_FFT_BIGM
#define SFFT_FFT_BIGM 8192
#endif
// sizes >= this use radices up to 16 and the 512-thread variant (128 registers, one CTA per SM); smaller sizes use
// radices <= 8 with 64 registers (SFFT_FFT_BIGM overrides, tuning)
inline int fft_big_m() {
  static const int v = getenv("SFFT_FFT_BIGM") ? atoi(getenv("SFFT_FFT_BIGM")) : SFFT_FFT_BIGM;
  return v;
}
// threads per FFT CTA: the 64-register variant fills the SM's 1024-thread register budget with as many CTAs as
// shared memory allows (1024 / CTAs per SM threads each), but no more threads than ~M/6 butterflies need
inline int fft_threads(int M, size_t smem, int64_t n_ctas) {
  if (M >= fft_big_m()) return 512;
  const size_t per_sm = 228 * 1024;
  const int ctas = smem * 4 + 4096 <= per_sm ? 4 : smem * 2 + 2048 <= per_sm ? 2 : 1;
  // (two CTAs per SM: 256 threads measured ~2 % faster than 512 on C5's M ~ 5100 lines; 768 / 1024 much slower)
  const int cap = getenv("SFFT_FFT_TCAP") ? atoi(getenv("SFFT_FFT_TCAP")) : (ctas == 2 ? 256 : 1024 / ctas);
  // ~M/6 threads; small sizes (M <= 2048) over many lines (>= 4096 CTAs) run better as more, smaller CTAs
  // per SM: ~M/12 (measured: C4 -6 %, C2 -1 %; with few CTAs, as in C5's later iterations, M/12 is slower)
  static const int tdiv_env = getenv("SFFT_FFT_TDIV") ? std::max(1, atoi(getenv("SFFT_FFT_TDIV"))) : 0;
  static const int64_t cta_min = getenv("SFFT_FFT_TDIV_CTAS") ? atoll(getenv("SFFT_FFT_TDIV_CTAS")) : 4096;
  const int tdiv = tdiv_env ? tdiv_env : (M <= 2048 && n_ctas >= cta_min ? 12 : 6);
  int t = ((M / tdiv + 31) / 32) * 32;
  return t < 64 ? 64 : (t > cap ? cap : t);
}
// wl: warp-local passes once the leading radices split the line over the warps (pfft_kernel<., true>)
cudaError_t launch_pfft(const DevParams& P, int32_t n_signals, int32_t n_lines, int32_t smem_bytes, int32_t threads, int32_t big,
                        int32_t ksplit, const double2* part, int32_t p_part, cudaStream_t st, bool wl = false);
cudaError_t launch_fft_twiddles(double2* tw, const int4* seg, int n_seg, cudaStream_t st);
// k_wrap.cu
// scratch: device int32 [n_signals * (k + 1)]
cudaError_t launch_wrap(const DevParams& P, int32_t n_signals, int32_t* out_freqs, double* out_coeffs,
                        int32_t* out_count, int32_t* out_status, int32_t* scratch, cudaStream_t st);

}  // namespace sfft
