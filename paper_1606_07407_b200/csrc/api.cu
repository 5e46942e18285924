// api.cu -- the C ABI (include/sfft.h): plan, workspace, the host-side
// iteration driver of Algorithm 2 and the stage entry points.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdarg>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <dlfcn.h>
#include <immintrin.h>
#include <functional>
#include <memory>
#include <new>
#include <nvtx3/nvToolsExt.h>

#include "sfft_internal.cuh"

// NVTX ranges around the solve, its iterations and their kernel classes (layer 8: tracing).
// Off unless SFFT_NVTX=1: the header-only NVTX3 stubs cost nothing once resolved, but the default path stays
// exactly the timed one.  Ranges bracket the host's launches (tools correlate them with the kernels).
namespace {
inline bool nvtx_on() {
  static const bool on = getenv("SFFT_NVTX") && atoi(getenv("SFFT_NVTX")) != 0;
  return on;
}
struct NvtxRange {
  bool on;
  explicit NvtxRange(const char* name) : on(nvtx_on()) { if (on) nvtxRangePushA(name); }
  NvtxRange(const char* fmt, int v) : on(nvtx_on()) {
    if (on) { char b[48]; snprintf(b, sizeof b, fmt, v); nvtxRangePushA(b); }
  }
  ~NvtxRange() { if (on) nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
}  // namespace

using namespace sfft;

#ifndef SFFT_GIT
#define SFFT_GIT "dev"
#endif

struct sfft_signal_s {
  sfft_plan_t* plan;
  int32_t batch;
  const int32_t* freqs;
  const double* coeffs;
};

namespace sfft {
cudaError_t ensure_smem(const void* kern, size_t bytes) {
  static std::vector<std::pair<std::pair<int, const void*>, size_t>> cache;   // (device, kernel) -> bytes set
  int dev = 0;
  cudaGetDevice(&dev);
  for (auto& c : cache)
    if (c.first.first == dev && c.first.second == kern) {
      if (c.second >= bytes) return cudaSuccess;
      const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
      if (e == cudaSuccess) c.second = bytes;
      return e;
    }
  const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) cache.push_back({{dev, kern}, bytes});
  return e;
}
}  // namespace sfft

namespace {

struct FftSize {
  int M;
  std::vector<int8_t> radix;
  size_t smem = 0;        // 16 * (M + sum_passes S/R): data + base twiddles
  size_t smem_upto = 0;   // max smem over all sizes <= M (launch size when max M is this one)
  int vw = 0;             // warp count of the warp-local plan (the table fill also stores V warp-blocked, k_fft.cu)
};

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

constexpr size_t kPartBytes = (size_t)512 << 20;   // exp-sum partial lines of term-split iterations

}  // namespace

struct sfft_plan_s {
  int device = 0;
  int n_sm = 148;
  cudaStream_t stream = nullptr;
  // problem
  int32_t d = 0, k = 0, r = 0, L = 0, Lp = 0, kk = 0, H = 0, batch = 1;
  int64_t N = 0, E = 0;
  std::vector<int32_t> blocks, block_off, axis_tilt;
  std::vector<int64_t> lo, hi, tilts, sched;
  // options
  int32_t c = 5, max_iter = 1000, stall_limit = 0, extra = 3;
  double tol = 1e-6, floor_rel = 1e-8, prune = 1e-8, round_tol = 0.01;
  // tables
  std::vector<int32_t> primes;
  std::vector<int32_t> prime_tab;   // device copy: the primes, then pfirst[x] = index of the first prime >= x
  int32_t p_cap = 0;
  int64_t p_stride = 0, M_stride = 0;
  std::vector<FftSize> fft;
  std::vector<int32_t> tw_off;        // [n_fft][kMaxFftPasses]
  std::vector<int4> tw_seg;           // (offset, S, R, 0) per (size, pass)
  size_t tw_total = 0;
  ExpsumShape shape{};
  I8Config i8{};
  bool i8_ok = false;          // int8-limb tensor-core exp-sum available for this plan
  bool fs_ok = false;          // fused sampling in the FFT CTA for short lines (FP64 plans, L_ref <= kFusedMaxL)
  int32_t n_fused_iters = 0;   // iterations of the current execute whose sampling ran inside the FFT (report)
  int32_t expsum_path = 0;     // sfft_options.expsum_path
  // stall fallback levels (reading R23): level 0 = the plan's own tilts / E
  int32_t n_levels = 1, lvl_tmax = 1;
  int32_t n_tslots = 0;          // per-prime table cache slots (+1 reserved for the stage entry points)
  int32_t epoch = 0;             // iteration counter across executes (table cache LRU stamp)
  std::vector<int64_t> lvl_E, lvl_lo, lvl_hi, lvl_tilts;
  std::vector<int32_t> lvl_nt, lvl_axt;
  int smem_optin = 0;
  // workspace
  size_t ws_bytes = 0;
  void* ws = nullptr;
  bool ws_owned = false;
  bool tables_ready = false;
  size_t off[128] = {0};        // workspace offsets, indexed by Buf (static_assert below)
  int32_t* h_ctrl = nullptr;   // pinned, host-mapped: setup_kernel publishes the iteration's control values here
  int32_t* h_ctrl_dev = nullptr;   // its device address
  int32_t ctrl_seq = 0;
  bool profile = false;
  int32_t literal = 0;
  std::vector<cudaEvent_t> events;
  std::string err;
  // line sharding: shard line_g of line_G (0 = unsharded) holds line 0 and the shifted lines of
  // reduced axes [line_lo, line_lo + L - 1); tile shapes / term split follow shard 0's line count L_ref so
  // that line 0 is computed identically on every shard
  int32_t line_G = 0, line_g = 0, line_lo = 0, L_ref = 0;
  int32_t rec_words = 0, rec_fw = 0;
  void* nccl_comm = nullptr;   // ncclComm_t of sfft_comm_init (shard_mode 1)
  // fused record exchange (line_exchange = 1): this shard's buffer (receive records [G][batch][rec_words] + stamps
  // [G][L_ref][batch]) and the G shards' buffers as mapped here (own one included)
  int32_t line_exchange = 0;
  void* peer_buf = nullptr;
  size_t peer_bytes = 0, peer_stamp_off = 0;
  std::vector<void*> peer_ptr;
  std::vector<bool> peer_opened;   // opened with cudaIpcOpenMemHandle (closed at destroy)
  bool peer_ready = false;
  int32_t peer_epoch = 0;
  cudaEvent_t ev_ctrl = nullptr;   // the per-iteration control read (iter_setup)
  int32_t spec_G = 1;              // multi-prime speculation (R26): primes (record sets) per iteration
  int32_t spec_slots = 1;          // slots per signal on this GPU (G, or 1 distributed); batch counts slots
  int32_t spec_dist = 0, spec_rank = 0, spec_tail = 0;
  // sfft_solve_host_batches: the second device input / output set, the H2D and D2H streams and their events
  void* pipe_buf = nullptr;
  size_t pipe_bytes = 0;
  cudaStream_t pipe_st[2] = {nullptr, nullptr};
  cudaEvent_t pipe_ev[6] = {};    // [set] inputs landed, [2 + set] solve done, [4 + set] outputs copied out
};

namespace {

enum Buf {
  B_BLOCKS, B_BOFF, B_LO, B_HI, B_TILTS, B_AXT, B_SCHED, B_PRIMES, B_FFTM, B_FFTR, B_FFTN,
  B_VALL, B_CALL, B_LINES, B_WTAB, B_CHIRP, B_V, B_AREG, B_KHASH, B_HTAB, B_ACCV, B_ACCA, B_WTMP,
  B_STATUS, B_NR, B_P, B_M, B_MI, B_STALL, B_ITERS, B_SAMPLES, B_CMACS, B_LOG, B_CTRL,
  B_IN_F, B_IN_C, B_OUT_F, B_OUT_C, B_OUT_N, B_OUT_S, B_STAGE, B_ACTIVE, B_PART, B_TWOFF, B_TW, B_TWSEG, B_UALL,
  B_WRAPS, B_I8B, B_I8SIG, B_CMACS8, B_LVLE, B_LVLLO, B_LVLHI, B_LVLT, B_LVLNT, B_LVLAXT, B_STLVL, B_STIL,
  B_STRT, B_I8PW, B_I8DLOG, B_I8ELOG, B_I8CHL, B_STSLOT, B_SLOTP, B_SLOTE, B_FILL, B_I8TLO, B_I8THI,
  B_RSEND, B_RRECV, B_RCAND, B_RNC, B_RF0, B_SELRDY, B_BINST, B_BINORD, B_FILLBY, B_FILLEP, B_SLOTRDY, B_ASGRDY, B_SPINERR,
  B_FFTW, B_DLROOT, B_CROWI, B_CROWL, B_SPECT,
  B_VB,                   // last: adding it left every other buffer's offset unchanged
  B_COUNT
};
static_assert(B_COUNT <= 128, "sfft_plan_s::off is too small for the workspace buffer list");

int fail(sfft_plan_t* P, int code, const char* fmt, ...) {
  if (P) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    P->err = buf;
  }
  return code;
}

#define CUDA_TRY(P, call)                                                                         \
  do {                                                                                            \
    cudaError_t _e = (call);                                                                      \
    if (_e != cudaSuccess) return fail((P), SFFT_ECUDA, "%s: %s", #call, cudaGetErrorString(_e)); \
  } while (0)

bool is_7smooth(int x) {
  for (int f : {2, 3, 5, 7})
    while (x % f == 0) x /= f;
  return x == 1;
}

// FP64 + shared-memory instructions of one radix-R butterfly (dft_small in registers, R - 2 twiddle powers and
// R - 1 twiddle products, R loads and stores); the fused middle has no twiddles but two DFTs and the V product
double fft_dft_cost(int R) {
  switch (R) {
    case 2: return 4; case 3: return 14; case 4: return 16; case 5: return 36; case 7: return 66; case 8: return 52;
    case 6: return 48; case 9: return 100; case 10: return 108; case 12: return 128; case 14: return 184;
    case 15: return 210; case 16: return 188;
  }
  return 16.0 * R;
}
double fft_bfly_cost(int R, bool mid) {
  return mid ? 2 * fft_dft_cost(R) + 4 * R + 3 * R : fft_dft_cost(R) + 8 * R - 12 + 2 * R;
}

FftSize radix_plan(int M) {
  // fewest passes with in-register radices {16,15,14,12,10,9,8,7,6,5,4,3,2} (DP over 2^a 3^b 5^c 7^d),
  // then descending order: the first (largest-Q) pass gets the largest radix -> fewest base twiddles
  // small sizes keep radices <= 8: with few butterflies per pass, wide radices idle most threads
  static const int kRad[] = {16, 15, 14, 12, 10, 9, 8, 7, 6, 5, 4, 3, 2};
  const int rmax = M >= fft_big_m() ? 16 : 8;
  FftSize s;
  s.M = M;
  std::vector<int> best(M + 1, 1 << 20), choice(M + 1, 0);
  best[1] = 0;
  for (int x = 2; x <= M; ++x) {
    if (M % x) continue;
    for (int R : kRad)
      if (R <= rmax && x % R == 0 && best[x / R] + 1 < best[x]) { best[x] = best[x / R] + 1; choice[x] = R; }
  }
  std::vector<int> rs;
  for (int x = M; x > 1; x /= choice[x]) rs.push_back(choice[x]);
  std::sort(rs.begin(), rs.end(), [](int a, int b) { return a > b; });
  // warp-local plans (pfft_kernel's pass_loop_w): when the launch's warp count W divides M, the first pass takes
  // radix W (one block-wide pass) and the rest of the plan -- run by each warp on its own M / W points -- is chosen
  // for lane efficiency: a radix-R pass costs ceil(Mw / R / 32) warp trips of ~fft_bfly_cost(R) instructions
  const int W = M >= fft_big_m() ? 16 : fft_threads(M, 16 * ((size_t)M + M / 4), 0) / 32;
  if (!getenv("SFFT_FFT_NO_WLPLAN") && M >= fft_wl_min() && W >= 2 && M % W == 0 && M / W > 1 &&
      std::find(std::begin(kRad), std::end(kRad), W) != std::end(kRad) && W <= rmax) {
    const int Mw = M / W;
    // cost[x][last]: cheapest plan of x points whose last (fused middle) radix is `last` (0: plan of 1)
    std::vector<double> best_w(Mw + 1, 1e30);
    std::vector<int> pick(Mw + 1, 0);
    // middle radix first: the plan of Mw = (passes) x (middle); passes run twice (DIF, DIT), the middle once
    // + ~40 instructions per warp trip (indices, loop, base twiddle) and ~150 cycles of dependent latency per pass
    auto trips = [&](int R) { return (double)((Mw / R + 31) / 32); };
    constexpr double kTrip = 40.0, kPass = 150.0;
    best_w[1] = 0.0;
    for (int x = 2; x <= Mw; ++x) {
      if (Mw % x) continue;
      for (int R : kRad)
        if (R <= rmax && x % R == 0 && best_w[x / R] < 1e29) {
          const double c = best_w[x / R] + 2.0 * (trips(R) * (fft_bfly_cost(R, false) + kTrip) + kPass);
          if (c < best_w[x]) { best_w[x] = c; pick[x] = R; }
        }
    }
    double bc = 1e30;
    int bm = 0;
    for (int R : kRad)
      if (R <= rmax && Mw % R == 0 && best_w[Mw / R] < 1e29) {
        const double c = best_w[Mw / R] + trips(R) * (fft_bfly_cost(R, true) + kTrip) + kPass;
        if (c < bc) { bc = c; bm = R; }
      }
    if (bm > 0 && (int)rs.size() > 0) {
      std::vector<int> sub;
      for (int x = Mw / bm; x > 1; x /= pick[x]) sub.push_back(pick[x]);
      std::sort(sub.begin(), sub.end(), [](int a, int b) { return a > b; });
      rs.assign(1, W);
      rs.insert(rs.end(), sub.begin(), sub.end());
      rs.push_back(bm);
      s.vw = W;
    }
  }
  // SFFT_FFT_PLAN="M:r1,r2,...;..." overrides the radices of size M (tuning experiments; order as given)
  if (const char* env = getenv("SFFT_FFT_PLAN")) {
    const std::string spec(env), key = std::to_string(M) + ":";
    size_t at = 0;
    while ((at = spec.find(key, at)) != std::string::npos && at > 0 && spec[at - 1] != ';') at += key.size();
    if (at != std::string::npos) {
      std::vector<int> ov;
      int prod = 1;
      bool ok = true;
      size_t i = at + key.size();
      while (i < spec.size() && spec[i] != ';') {
        const int R = atoi(spec.c_str() + i);
        ok = ok && R >= 2 && R <= rmax && std::find(std::begin(kRad), std::end(kRad), R) != std::end(kRad);
        ov.push_back(R);
        prod *= R;
        while (i < spec.size() && spec[i] != ',' && spec[i] != ';') ++i;
        if (i < spec.size() && spec[i] == ',') ++i;
      }
      if (ok && prod == M) {
        rs = ov;
        if (s.vw && (rs[0] % s.vw != 0 || (M / s.vw) % rs.back() != 0)) s.vw = 0;
      }
    }
  }
  for (int R : rs) s.radix.push_back((int8_t)R);
  size_t sumq = 0;
  int S = M;
  for (int8_t R : s.radix) { sumq += S / R; S /= R; }
  s.smem = 16 * ((size_t)M + sumq + 2);
  // the fused select of a line-0 CTA uses x[p ..) (p <= (M + 1) / 2): mag, cand, flag [p] + scratch[32]
  s.smem = std::max(s.smem, 32 * (size_t)((M + 1) / 2) + 128);
  return s;
}

int64_t gcd64(int64_t a, int64_t b) {
  a = a < 0 ? -a : a;
  b = b < 0 ? -b : b;
  while (b) { int64_t t = a % b; a = b; b = t; }
  return a;
}

void layout(sfft_plan_t* P) {
  const size_t S = (size_t)P->batch;
  size_t sz[B_COUNT] = {0};
  sz[B_BLOCKS] = 4 * (size_t)P->r;
  sz[B_BOFF] = 4 * (size_t)P->r;
  sz[B_LO] = 8 * (size_t)P->r;
  sz[B_HI] = 8 * (size_t)P->r;
  sz[B_TILTS] = 8 * std::max<size_t>(P->tilts.size(), 1);
  sz[B_AXT] = 4 * (size_t)P->r;
  sz[B_SCHED] = 8 * std::max<size_t>(P->sched.size(), 1);
  sz[B_PRIMES] = 4 * P->prime_tab.size();
  sz[B_FFTM] = 4 * P->fft.size();
  sz[B_FFTR] = (size_t)kMaxFftPasses * P->fft.size();
  sz[B_FFTN] = 4 * P->fft.size();
  sz[B_VALL] = 8 * S * P->r * P->kk;
  sz[B_CALL] = 16 * S * P->kk * P->Lp;
  sz[B_LINES] = 16 * S * P->L * P->p_stride;
  const size_t T = (size_t)P->n_tslots + 1;          // table slots (per prime), not per signal
  sz[B_WTAB] = 16 * T * P->p_stride;
  sz[B_CHIRP] = 16 * T * P->p_stride;
  sz[B_V] = 16 * T * P->M_stride;
  sz[B_VB] = P->fft.back().M >= kFftWlMinM ? 16 * T * P->M_stride : 0;   // V warp-blocked (k_fft.cu mid_loop)
  sz[B_AREG] = 16 * S * P->k;
  sz[B_KHASH] = 8 * S * P->k;
  sz[B_HTAB] = 4 * S * P->H;
  sz[B_ACCV] = 8 * S * P->r * P->k;
  sz[B_ACCA] = 16 * S * P->k;
  sz[B_WTMP] = 4 * S * P->k * P->d;
  for (int b : {B_STATUS, B_NR, B_P, B_M, B_MI, B_STALL, B_ITERS}) sz[b] = 4 * S;
  sz[B_SAMPLES] = 8 * S;
  sz[B_CMACS] = 8 * S;
  sz[B_LOG] = 4 * 2 * kLogIters;
  sz[B_CTRL] = 64;                              // two alternating control blocks of 8 ints
  sz[B_IN_F] = 4 * S * P->k * P->d;
  sz[B_IN_C] = 16 * S * P->k;
  sz[B_OUT_F] = 4 * S * P->k * P->d;
  sz[B_OUT_C] = 16 * S * P->k;
  sz[B_OUT_N] = 4 * S;
  sz[B_OUT_S] = 4 * S;
  sz[B_STAGE] = 64;
  sz[B_ACTIVE] = 4 * S;
  sz[B_PART] = kPartBytes;
  sz[B_TWOFF] = 4 * (size_t)kMaxFftPasses * P->fft.size();
  sz[B_TW] = 16 * P->tw_total;
  sz[B_TWSEG] = 16 * P->tw_seg.size();
  sz[B_UALL] = 8 * S * (size_t)P->kk + 256;
  sz[B_WRAPS] = 4 * S * ((size_t)P->k + 1);
  sz[B_I8B] = P->i8_ok ? i8_limb_bytes(P->i8, (int)S) : 0;
  sz[B_I8SIG] = 8 * S;
  sz[B_CMACS8] = 8 * S;
  sz[B_FFTW] = 16 * S;
  sz[B_LVLE] = 8 * (size_t)P->n_levels;
  sz[B_LVLLO] = 8 * (size_t)P->n_levels * P->r;
  sz[B_LVLHI] = 8 * (size_t)P->n_levels * P->r;
  sz[B_LVLT] = 8 * P->lvl_tilts.size();
  sz[B_LVLNT] = 4 * (size_t)P->n_levels;
  sz[B_LVLAXT] = 4 * (size_t)P->n_levels * P->r;
  for (int b : {B_STLVL, B_STIL, B_STRT}) sz[b] = 4 * S;
  const bool logt = P->i8_ok || P->fs_ok;   // discrete-log tables: the int8 exp-sum and the fused sampling
  sz[B_I8PW] = logt ? 4 * T * (2 * P->p_stride + 8) : 0;
  sz[B_I8DLOG] = logt ? 4 * T * (2 * P->p_stride + 8) : 0;
  sz[B_I8ELOG] = logt ? 4 * S * align_up((size_t)P->kk + 16, 4) : 0;
  sz[B_I8CHL] = logt ? 16 * T * (2 * P->p_stride + 8) : 0;
  sz[B_DLROOT] = P->fs_ok ? 16 * T * (2 * P->p_stride + 8) : 0;
  sz[B_CROWI] = 16 * S * (size_t)((P->k + 31) / 32) * ((P->Lp + 15) / 16);
  sz[B_CROWL] = 4 * S * (size_t)P->k;
  sz[B_SPECT] = P->spec_G > 1 ? 4 * S * (size_t)P->k : 0;
  sz[B_STSLOT] = 4 * S;
  sz[B_SLOTP] = 4 * T;
  sz[B_SLOTE] = 4 * T;
  sz[B_FILL] = 4 * T;
  sz[B_FILLBY] = 4 * T;
  sz[B_FILLEP] = 4 * T;
  sz[B_SLOTRDY] = 4 * T;
  sz[B_ASGRDY] = 4;
  sz[B_SPINERR] = 4 * (1 + S);        // [0] stamp-wait timeout flag, [1 + s] fused-commit arrival counters
  sz[B_I8TLO] = P->i8_ok ? 8 * T * (2 * P->p_stride + 8) : 0;
  sz[B_I8THI] = P->i8_ok ? 4 * T * (2 * P->p_stride + 8) : 0;
  // decode records (fused FFT epilogue -> commit); line shards also receive every shard's records
  sz[B_RSEND] = 8 * S * (size_t)P->rec_words;
  sz[B_RRECV] = P->line_G > 0 ? 8 * (size_t)P->line_G * S * (size_t)P->rec_words
                : P->spec_dist ? 8 * (size_t)P->spec_G * S * (size_t)P->rec_words : 0;
  sz[B_RCAND] = 4 * S * (size_t)P->k;
  sz[B_RNC] = 4 * S;
  sz[B_RF0] = 16 * S * (size_t)P->k;
  sz[B_SELRDY] = 4 * S;
  sz[B_BINST] = 4 * S * ((size_t)P->p_stride + 1);
  sz[B_BINORD] = 4 * S * (size_t)P->k;
  size_t o = 0;
  for (int b = 0; b < B_COUNT; ++b) {
    P->off[b] = o;
    o = align_up(o + std::max<size_t>(sz[b], 16), 256);
  }
  P->ws_bytes = o;
}

template <typename T>
T* ptr(const sfft_plan_t* P, int b) {
  return reinterpret_cast<T*>(static_cast<char*>(P->ws) + P->off[b]);
}

// warp-local FFT passes for a launch whose largest size is M (SFFT_FFT_NO_WL=1: block-wide passes only)
bool fft_wl_for(int M) {
  static const bool no_wl = getenv("SFFT_FFT_NO_WL") != nullptr;
  return !no_wl && M >= fft_wl_min();
}

DevParams dev_params(const sfft_plan_t* P, int32_t batch) {
  DevParams D;
  memset(&D, 0, sizeof D);
  D.d = P->d; D.k = P->k; D.r = P->r; D.L = P->L; D.Lp = P->Lp; D.kk = P->kk; D.H = P->H;
  D.batch = batch;
  D.N = P->N; D.E = P->E;
  D.c = P->c; D.max_iter = P->max_iter; D.stall_limit = P->stall_limit; D.extra = P->extra;
  D.n_sched = (int32_t)P->sched.size();
  D.literal = P->literal;
  D.tol = P->tol; D.floor_rel = P->floor_rel; D.prune = P->prune; D.round_tol = P->round_tol;
  D.n_tilts = (int32_t)(P->tilts.size() / 5);
  D.p_cap = P->p_cap;
  D.p_stride = P->p_stride; D.M_stride = P->M_stride;
  D.block_dims = ptr<int32_t>(P, B_BLOCKS);
  D.block_off = ptr<int32_t>(P, B_BOFF);
  D.lo = ptr<int64_t>(P, B_LO);
  D.hi = ptr<int64_t>(P, B_HI);
  D.tilts = ptr<int64_t>(P, B_TILTS);
  D.axis_tilt = ptr<int32_t>(P, B_AXT);
  D.sched = ptr<int64_t>(P, B_SCHED);
  D.primes = ptr<int32_t>(P, B_PRIMES);
  D.n_primes = (int32_t)P->primes.size();
  D.pfirst = D.primes + P->primes.size();
  D.n_pfirst = (int32_t)(P->prime_tab.size() - P->primes.size());
  D.fft_M = ptr<int32_t>(P, B_FFTM);
  D.fft_radix = ptr<int8_t>(P, B_FFTR);
  D.fft_npass = ptr<int32_t>(P, B_FFTN);
  D.fft_tw_off = ptr<int32_t>(P, B_TWOFF);
  D.fft_tw = ptr<double2>(P, B_TW);
  D.n_fft = (int32_t)P->fft.size();
  D.v_all = ptr<int64_t>(P, B_VALL);
  D.C_all = ptr<double2>(P, B_CALL);
  D.u_all = ptr<int2>(P, B_UALL);
  D.lines = ptr<double2>(P, B_LINES);
  D.W_tab = ptr<double2>(P, B_WTAB);
  D.chirp = ptr<double2>(P, B_CHIRP);
  D.V = ptr<double2>(P, B_V);
  D.VB = P->fft.back().M >= kFftWlMinM ? ptr<double2>(P, B_VB) : nullptr;
  D.a_reg = ptr<double2>(P, B_AREG);
  D.key_hash = ptr<uint64_t>(P, B_KHASH);
  D.htab = ptr<int32_t>(P, B_HTAB);
  D.acc_v = ptr<int64_t>(P, B_ACCV);
  D.acc_a = ptr<double2>(P, B_ACCA);
  D.wtmp = ptr<int32_t>(P, B_WTMP);
  D.st_status = ptr<int32_t>(P, B_STATUS);
  D.st_nR = ptr<int32_t>(P, B_NR);
  D.st_p = ptr<int32_t>(P, B_P);
  D.st_m = ptr<int32_t>(P, B_M);
  D.st_M = ptr<int32_t>(P, B_MI);
  D.st_stall = ptr<int32_t>(P, B_STALL);
  D.st_iters = ptr<int32_t>(P, B_ITERS);
  D.st_samples = ptr<int64_t>(P, B_SAMPLES);
  D.st_cmacs = ptr<int64_t>(P, B_CMACS);
  D.st_cmacs_i8 = ptr<int64_t>(P, B_CMACS8);
  D.st_fftw = ptr<double>(P, B_FFTW);
  D.st_log = ptr<int32_t>(P, B_LOG);
  D.ctrl = ptr<int32_t>(P, B_CTRL);
  D.h_ctrl_map = P->h_ctrl_dev;
  D.active = ptr<int32_t>(P, B_ACTIVE);
  D.n_levels = P->n_levels;
  D.lvl_tmax = P->lvl_tmax;
  D.lvl_E = ptr<int64_t>(P, B_LVLE);
  D.lvl_lo = ptr<int64_t>(P, B_LVLLO);
  D.lvl_hi = ptr<int64_t>(P, B_LVLHI);
  D.lvl_tilts = ptr<int64_t>(P, B_LVLT);
  D.lvl_nt = ptr<int32_t>(P, B_LVLNT);
  D.lvl_axt = ptr<int32_t>(P, B_LVLAXT);
  D.st_lvl = ptr<int32_t>(P, B_STLVL);
  D.st_il = ptr<int32_t>(P, B_STIL);
  D.st_retilt = ptr<int32_t>(P, B_STRT);
  D.n_tslots = P->n_tslots;
  D.st_slot = ptr<int32_t>(P, B_STSLOT);
  D.slot_p = ptr<int32_t>(P, B_SLOTP);
  D.slot_epoch = ptr<int32_t>(P, B_SLOTE);
  D.fill = ptr<int32_t>(P, B_FILL);
  D.fill_by = ptr<int32_t>(P, B_FILLBY);
  D.fill_ep = ptr<int32_t>(P, B_FILLEP);
  D.slot_ready = ptr<int32_t>(P, B_SLOTRDY);
  D.assign_ready = ptr<int32_t>(P, B_ASGRDY);
  D.spin_err = ptr<int32_t>(P, B_SPINERR);
  D.spec_G = 1;                              // sfft_execute sets the plan's G (stage entry points run single slots)
  D.spec_slots = 1;
  D.spec_dist = P->spec_dist;
  D.spec_rank = P->spec_rank;
  D.spec_tail = P->spec_tail;
  D.spec_touch = P->spec_G > 1 ? ptr<int32_t>(P, B_SPECT) : nullptr;
  D.commit_cnt = ptr<int32_t>(P, B_SPINERR) + 1;
  if (P->i8_ok) {
    D.i8_S = P->i8.S; D.i8_NT = P->i8.NT; D.i8_NT_last = P->i8.NT_last; D.i8_ntiles = P->i8.ntiles; D.i8_nks = P->i8.nks;
    D.i8_K = P->k;
    D.i8_pair = P->i8.pair;
    D.i8_B = ptr<int8_t>(P, B_I8B);
    D.i8_sigma = ptr<double>(P, B_I8SIG);
    D.i8_tlo = ptr<uint2>(P, B_I8TLO);
    D.i8_thi = ptr<uint32_t>(P, B_I8THI);
  }
  if (P->i8_ok || P->fs_ok) {
    D.log_tables = 1;
    D.i8_tstride = 2 * P->p_stride + 8;   // the root table holds T twice (discrete-log rows, no wrap)
    D.i8_pw = ptr<int32_t>(P, B_I8PW);
    D.i8_dlog = ptr<int32_t>(P, B_I8DLOG);
    D.i8_elog = ptr<int32_t>(P, B_I8ELOG);
    D.i8_estride = (int32_t)align_up((size_t)P->kk + 16, 4);   // rows 16-byte aligned for the bulk copies
    D.i8_chl = ptr<double2>(P, B_I8CHL);
  }
  if (P->fs_ok) D.dl_root = ptr<double2>(P, B_DLROOT);
  D.crow_nl = (P->Lp + 15) / 16;
  D.crow_items = ptr<int4>(P, B_CROWI);
  D.crow_list = ptr<int32_t>(P, B_CROWL);
  D.line_lo = P->line_lo;
  D.line_G = std::max(P->line_G, 1);
  D.line_g = P->line_g;
  D.rec_words = P->rec_words;
  D.rec_fw = P->rec_fw;
  D.rec_send = ptr<int64_t>(P, B_RSEND);
  D.rec_recv = P->line_G > 0 || P->spec_dist ? ptr<int64_t>(P, B_RRECV) : ptr<int64_t>(P, B_RSEND);   // unsharded: own
  D.L_ref = P->L_ref;
  D.peer_mode = 0;
  if (P->line_exchange == 1 && P->peer_ready) {
    D.peer_mode = 1;
    D.peer_epoch = P->peer_epoch;
    D.rec_recv = static_cast<int64_t*>(P->peer_buf);
    D.stamp_local = reinterpret_cast<int32_t*>(static_cast<char*>(P->peer_buf) + P->peer_stamp_off);
    for (int h = 0; h < P->line_G; ++h) {
      D.peer_recv[h] = static_cast<int64_t*>(P->peer_ptr[h]);
      D.peer_stamp[h] = reinterpret_cast<int32_t*>(static_cast<char*>(P->peer_ptr[h]) + P->peer_stamp_off);
    }
  }
  D.rec_cand = ptr<int32_t>(P, B_RCAND);
  D.rec_nc = ptr<int32_t>(P, B_RNC);
  D.rec_f0 = ptr<double2>(P, B_RF0);
  D.sel_ready = ptr<int32_t>(P, B_SELRDY);
  D.bin_start = ptr<int32_t>(P, B_BINST);
  D.bin_order = ptr<int32_t>(P, B_BINORD);
  return D;
}

// the fused exchange's buffer of this shard (cudaMalloc'ed separately from the workspace so that it can be shared
// through a CUDA IPC handle): receive records [G][batch][rec_words] int64, then stamps [G][L_ref][batch] int32
int ensure_peer_buf(sfft_plan_t* P) {
  if (P->peer_buf) return SFFT_OK;
  CUDA_TRY(P, cudaSetDevice(P->device));
  const size_t rec = 8 * (size_t)P->line_G * P->batch * (size_t)P->rec_words;
  P->peer_stamp_off = align_up(rec, 256);
  P->peer_bytes = P->peer_stamp_off + 4 * (size_t)P->line_G * P->L_ref * (size_t)P->batch;
  cudaError_t e = cudaMalloc(&P->peer_buf, P->peer_bytes);
  if (e != cudaSuccess) return fail(P, SFFT_ENOMEM, "cudaMalloc(%zu) for the record exchange: %s", P->peer_bytes,
                                    cudaGetErrorString(e));
  CUDA_TRY(P, cudaMemset(P->peer_buf, 0, P->peer_bytes));   // stamps 0: the exchange epochs start at 1
  return SFFT_OK;
}

int ensure_ready(sfft_plan_t* P) {
  CUDA_TRY(P, cudaSetDevice(P->device));
  {
    const cudaError_t pending = cudaGetLastError();   // a stale error of another library must not be reported as ours
    if (pending != cudaSuccess && getenv("SFFT_DEBUG"))
      fprintf(stderr, "[sfft] cleared pending CUDA error before plan setup: %s\n", cudaGetErrorString(pending));
  }
  if (!P->ws) {
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, P->ws_bytes);
    if (e != cudaSuccess) return fail(P, SFFT_ENOMEM, "cudaMalloc(%zu): %s", P->ws_bytes, cudaGetErrorString(e));
    P->ws = p;
    P->ws_owned = true;
    P->tables_ready = false;
  }
  if (!P->h_ctrl) {
    CUDA_TRY(P, cudaHostAlloc(reinterpret_cast<void**>(&P->h_ctrl), 64, cudaHostAllocMapped));
    memset(P->h_ctrl, 0, 64);
    CUDA_TRY(P, cudaHostGetDevicePointer(reinterpret_cast<void**>(&P->h_ctrl_dev), P->h_ctrl, 0));
  }
  if (!P->ev_ctrl) CUDA_TRY(P, cudaEventCreateWithFlags(&P->ev_ctrl, cudaEventDisableTiming));
  if (!P->tables_ready) {
    std::vector<int32_t> fm, fn;
    std::vector<int8_t> fr(P->fft.size() * kMaxFftPasses, 0);
    for (size_t i = 0; i < P->fft.size(); ++i) {
      fm.push_back(P->fft[i].M);
      fn.push_back((int32_t)P->fft[i].radix.size());
      for (size_t j = 0; j < P->fft[i].radix.size(); ++j) fr[i * kMaxFftPasses + j] = P->fft[i].radix[j];
      fr[i * kMaxFftPasses + kFftVwSlot] = (int8_t)P->fft[i].vw;   // after the last pass (npass < kMaxFftPasses)
    }
    auto up = [&](int b, const void* src, size_t n) -> cudaError_t {
      if (n == 0) return cudaSuccess;
      return cudaMemcpyAsync(static_cast<char*>(P->ws) + P->off[b], src, n, cudaMemcpyHostToDevice, P->stream);
    };
    CUDA_TRY(P, up(B_BLOCKS, P->blocks.data(), 4 * P->blocks.size()));
    CUDA_TRY(P, up(B_BOFF, P->block_off.data(), 4 * P->block_off.size()));
    CUDA_TRY(P, up(B_LO, P->lo.data(), 8 * P->lo.size()));
    CUDA_TRY(P, up(B_HI, P->hi.data(), 8 * P->hi.size()));
    CUDA_TRY(P, up(B_TILTS, P->tilts.data(), 8 * P->tilts.size()));
    CUDA_TRY(P, up(B_AXT, P->axis_tilt.data(), 4 * P->axis_tilt.size()));
    CUDA_TRY(P, up(B_SCHED, P->sched.data(), 8 * P->sched.size()));
    CUDA_TRY(P, up(B_PRIMES, P->prime_tab.data(), 4 * P->prime_tab.size()));
    CUDA_TRY(P, up(B_FFTM, fm.data(), 4 * fm.size()));
    CUDA_TRY(P, up(B_FFTR, fr.data(), fr.size()));
    CUDA_TRY(P, up(B_FFTN, fn.data(), 4 * fn.size()));
    CUDA_TRY(P, up(B_TWOFF, P->tw_off.data(), 4 * P->tw_off.size()));
    CUDA_TRY(P, up(B_TWSEG, P->tw_seg.data(), 16 * P->tw_seg.size()));
    CUDA_TRY(P, up(B_LVLE, P->lvl_E.data(), 8 * P->lvl_E.size()));
    CUDA_TRY(P, up(B_LVLLO, P->lvl_lo.data(), 8 * P->lvl_lo.size()));
    CUDA_TRY(P, up(B_LVLHI, P->lvl_hi.data(), 8 * P->lvl_hi.size()));
    CUDA_TRY(P, up(B_LVLT, P->lvl_tilts.data(), 8 * P->lvl_tilts.size()));
    CUDA_TRY(P, up(B_LVLNT, P->lvl_nt.data(), 4 * P->lvl_nt.size()));
    CUDA_TRY(P, up(B_LVLAXT, P->lvl_axt.data(), 4 * P->lvl_axt.size()));
    CUDA_TRY(P, launch_fft_twiddles(ptr<double2>(P, B_TW), ptr<int4>(P, B_TWSEG), (int)P->tw_seg.size(), P->stream));
    // empty per-prime table cache (slot_p = 0, slot_epoch = -1)
    CUDA_TRY(P, cudaMemsetAsync(ptr<int32_t>(P, B_SLOTP), 0, 4 * ((size_t)P->n_tslots + 1), P->stream));
    CUDA_TRY(P, cudaMemsetAsync(ptr<int32_t>(P, B_SLOTE), 0xFF, 4 * ((size_t)P->n_tslots + 1), P->stream));
    for (int b : {B_FILLEP, B_SLOTRDY})
      CUDA_TRY(P, cudaMemsetAsync(ptr<int32_t>(P, b), 0xFF, 4 * ((size_t)P->n_tslots + 1), P->stream));
    CUDA_TRY(P, cudaMemsetAsync(ptr<int32_t>(P, B_ASGRDY), 0xFF, 4, P->stream));
    // fused-decode publication stamps: never equal to an iteration stamp (those are >= 1)
    CUDA_TRY(P, cudaMemsetAsync(ptr<int32_t>(P, B_SELRDY), 0xFF, 4 * (size_t)P->batch, P->stream));
    CUDA_TRY(P, cudaStreamSynchronize(P->stream));
    P->tables_ready = true;
  }
  return SFFT_OK;
}

int fft_index_host(const sfft_plan_t* P, int p) {
  const int need = 2 * p - 1;
  for (size_t i = 0; i < P->fft.size(); ++i)
    if (P->fft[i].M >= need) return (int)i;
  return -1;
}

#define LAUNCH(P, call)                                                                          \
  do {                                                                                           \
    cudaError_t _e = (call);                                                                     \
    if (_e == cudaSuccess && g_sync_launches) _e = cudaStreamSynchronize((P)->stream);           \
    if (_e != cudaSuccess) return fail((P), SFFT_ECUDA, "%s: %s", #call, cudaGetErrorString(_e)); \
    ++launches;                                                                                  \
  } while (0)

// int8-limb exp-sum for this iteration?  Needs the limb tables in shared memory; tiny primes (late
// iterations) waste most of a 128-row MMA tile and stay on the FP64 kernels (SFFT_I8_MIN_P overrides).
bool i8_use_for(const sfft_plan_t* P, int max_p) {
  static const int min_p = getenv("SFFT_I8_MIN_P") ? atoi(getenv("SFFT_I8_MIN_P")) : 64;
  if (P->expsum_path == 2) return i8_fits(P->i8, max_p, P->k, P->smem_optin);
  return max_p >= min_p && i8_fits(P->i8, max_p, P->k, P->smem_optin);
}

// term split of the int8 kernel: same wave-quantisation model as the FP64 kernels, one CTA per SM
int i8_ksplit(const sfft_plan_t* P, int max_p, int n_active) {
  const int blocks = i8_blocks(P->i8, max_p, n_active);
  const int W = P->i8.pair ? P->n_sm / 2 : P->n_sm;                     // persistent units (CTA pairs)
  const int steps = (P->k + 15) / 16;
  const int ks_max = std::min(32, std::max(1, steps / 4));
  int ksplit = 1;
  double best = 1e30;
  for (int ks = 1; ks <= ks_max; ++ks) {
    if (ks > 1 && (size_t)ks * n_active * P->L_ref * (size_t)max_p * 16 > kPartBytes) break;
    // a tile's epilogue (accumulator drain + stores, ~10 % of a full-K tile, measured with SFFT_I8_PROF) does
    // not shrink with its K range; splits also write ks partial lines that the FFT sums
    static const double e = getenv("SFFT_I8_EPI") ? atof(getenv("SFFT_I8_EPI")) : 0.10;
    const double waves = std::ceil((double)blocks * ks / W);
    const double t = waves * (1.0 / ks + e) * (ks > 1 ? 1.03 : 1.0) + 0.02 * ks;
    if (t < best - 1e-9) { best = t; ksplit = ks; }
  }
  return ksplit;
}

// SFFT_SYNC=1: synchronise after every launch (debugging aid: pins errors to the launching call)
const bool g_sync_launches = getenv("SFFT_SYNC") != nullptr;

// ---------------------------------------------------------------- the iteration driver (Alg. 2)
// One iteration = setup (host reads n_active / max p) | front: table prep, exp-sum (a3), pfft (a4), decode
// (a5-a7; its local phase when line-sharded) | [record all-gather] | back: decode commit, fallback retilt.
struct IterPlan {
  int n_active = 0, max_p = 0, fi = 0, max_M = 0, ksplit = 1, big = 0;
  bool use_i8 = false;
  bool fused = false;         // samples computed in the FFT CTAs (no exp-sum launch), fused_smem bytes per CTA
  size_t fused_smem = 0;
  bool fuse_commit = false;   // the commit runs in the last FFT CTA of each signal (no commit launch)
};

// a1 (projection, term rows) and the int8 limbs of the signal terms, once per solve
int solve_begin(sfft_plan_t* P, DevParams& D, const sfft_signal_t* sig, int& launches) {
  cudaStream_t st = P->stream;
  CUDA_TRY(P, cudaMemsetAsync(ptr<int32_t>(P, B_CTRL), 0, 64, st));   // both control blocks
  CUDA_TRY(P, cudaMemsetAsync(ptr<int32_t>(P, B_SPINERR), 0, 4 * (1 + (size_t)P->batch), st));
  const int slots = sig->batch * D.spec_slots;   // R26: G slots per signal, the projection maps slot -> signal
  if (D.spec_G > 1)
    CUDA_TRY(P, cudaMemsetAsync(D.spec_touch, 0, 4 * (size_t)slots * P->k, st));
  LAUNCH(P, launch_project(D, slots, sig->freqs, sig->coeffs, st));
  launches += 1;   // init_state_kernel
  if (P->i8_ok) {
    LAUNCH(P, launch_i8_prepare(D, slots, P->k, st));
    launches += 1;   // sigma + limbs
  }
  return SFFT_OK;
}

int iter_setup(sfft_plan_t* P, DevParams& D, int iter, IterPlan* it, int& launches, int n_bound) {
  cudaStream_t st = P->stream;
  const int32_t seq = ++P->ctrl_seq;
  D.ctrl = ptr<int32_t>(P, B_CTRL) + 8 * (seq & 1);
  D.ctrl_next = ptr<int32_t>(P, B_CTRL) + 8 * ((seq + 1) & 1);
  LAUNCH(P, launch_setup(D, iter, st, seq));
  // the table prep needs no host decision: it is enqueued before the control read returns, sized for the
  // previous iteration's active count and the largest FFT size (CTAs beyond the device-side counts exit), so
  // the host round trip overlaps it
  {
    const FftSize& fb = P->fft.back();
    // one combined kernel while the signals fit in one wave of its (largest-FFT) shared-memory footprint;
    // beyond that the separate assign / fill / terms kernels keep the terms work at full occupancy
    if (n_bound <= P->n_sm) {
      LAUNCH(P, launch_prep_iter(D, n_bound, (int)fb.smem_upto, st, ++P->epoch));
    } else {
      LAUNCH(P, launch_fft_prep(D, n_bound, (int)fb.smem_upto, 512, 1, st, ++P->epoch));
      launches += 2;   // tables_assign, terms
    }
  }
  // poll the host-mapped control block (one 16-byte store of setup's last CTA, read as one aligned 16-byte load:
  // accepted when its check word carries this sequence number); a fault surfaces through the stream
  int32_t cv[4];
  {
    auto snap = [&]() {
      std::atomic_signal_fence(std::memory_order_seq_cst);
      const __m128i x = _mm_load_si128(reinterpret_cast<const __m128i*>(P->h_ctrl));
      _mm_storeu_si128(reinterpret_cast<__m128i*>(cv), x);
      std::atomic_signal_fence(std::memory_order_seq_cst);
      return (uint32_t)cv[3] == ((uint32_t)seq ^ ctrl_mix((uint32_t)cv[0], (uint32_t)cv[1], (uint32_t)cv[2]));
    };
    long spins = 0;
    std::chrono::steady_clock::time_point t0;
    while (!snap()) {
      if ((++spins & 1023) == 0) {
        const cudaError_t q = cudaStreamQuery(st);
        if (q != cudaSuccess && q != cudaErrorNotReady) return fail(P, SFFT_ECUDA, "setup: %s", cudaGetErrorString(q));
        if (q == cudaSuccess && !snap()) return fail(P, SFFT_ECUDA, "setup: control block not published");
        if (spins == 1024) t0 = std::chrono::steady_clock::now();
        else if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(120))
          return fail(P, SFFT_ECUDA, "setup: no control block after 120 s");
      }
    }
    std::atomic_thread_fence(std::memory_order_acquire);
  }
  it->n_active = cv[0];
  it->max_p = cv[1];
  if (it->n_active == 0) return SFFT_OK;
  it->fi = fft_index_host(P, it->max_p);
  if (it->fi < 0) return fail(P, SFFT_ENOTSUP, "p=%d beyond FFT table", it->max_p);
  it->max_M = P->fft[it->fi].M;
  const int max_K = cv[2];
  // term split when the (signal x h-tile x n-tile) grid cannot fill the GPU (late iterations); computed
  // from shard 0's line count so that every line shard sums line 0 in the same order
  const ExpsumShape shp = expsum_for_p(P->shape, it->max_p);
  it->use_i8 = P->i8_ok && i8_use_for(P, it->max_p);
  it->ksplit = 1;
  if (P->fs_ok) {
    it->fused_smem = P->fft[it->fi].smem_upto + 16 * (2 * (size_t)it->max_p + 4) + 20 * (size_t)P->k + 256;
    it->fused = it->fused_smem <= (size_t)P->smem_optin;
  }
  if (it->use_i8) {
    it->ksplit = i8_ksplit(P, it->max_p, it->n_active);
  } else {
    // wave quantisation model: time ~ ceil(B ks / W) / ks, W = resident CTAs; a split costs ~3 %
    // (partial lines written and re-read by the FFT)
    const int blocks = expsum_blocks(shp, it->max_p, it->n_active);
    const int W = P->n_sm * expsum_occupancy(shp, it->max_p);
    const int chunks = (max_K + expsum_bk() - 1) / expsum_bk();
    const int ks_max = std::min(32, std::max(1, chunks / 2));
    double best = 1e30;
    for (int ks = 1; ks <= ks_max; ++ks) {
      if (ks > 1 && (size_t)ks * it->n_active * P->L_ref * (size_t)it->max_p * 16 > kPartBytes) break;
      static const double e = getenv("SFFT_FP64_EPI") ? atof(getenv("SFFT_FP64_EPI")) : 0.0;
      const double waves = std::ceil((double)blocks * ks / W);
      const double t = waves * (1.0 / ks + e) * (ks > 1 ? 1.03 : 1.0);
      if (t < best - 1e-9) { best = t; it->ksplit = ks; }
    }
  }
  it->big = it->max_M >= fft_big_m();
  // fused commit (opt-in, SFFT_FUSE_COMMIT=1; measured slower: the commit then runs with the FFT's thread count
  // on the tail of the launch -- C3 +4 %, C4 +44 %, C5 -0.7 %): unsharded lines only (line shards commit after
  // the record all-gather), and the commit's shared memory must fit in the FFT's
  static const bool fc = getenv("SFFT_FUSE_COMMIT") && atoi(getenv("SFFT_FUSE_COMMIT")) != 0;
  it->fuse_commit = fc && P->line_G == 0 && P->spec_G == 1 && decode_smem_bytes(D, it->max_p) <= P->fft[it->fi].smem_upto;
  return SFFT_OK;
}

int iter_front(sfft_plan_t* P, DevParams& D, int iter, const IterPlan& it, int& launches,
               const std::function<int()>& mark) {
  cudaStream_t st = P->stream;
  mark();
  {
    NvtxRange nv_x(it.fused ? "sfft expsum (fused into pfft)" : it.use_i8 ? "sfft expsum_i8" : "sfft expsum_dmma");
    if (it.fused) {
      // no exp-sum launch: the FFT CTAs sample their lines (the mark pair stays for the profile's bookkeeping)
      ++P->n_fused_iters;
    } else if (it.use_i8)
      LAUNCH(P, launch_expsum_i8(D, P->i8, it.max_p, it.n_active, it.ksplit, ptr<double2>(P, B_PART), it.max_p,
                                 P->smem_optin, st));
    else
      LAUNCH(P, launch_expsum(D, expsum_for_p(P->shape, it.max_p), it.max_p, it.n_active, it.ksplit,
                              ptr<double2>(P, B_PART), it.max_p, st));
  }
  mark();
  NvtxRange nv_f("sfft pfft + select / test / decode");
  // FFT of every line with the fused select (line 0) / test + decode (lines n >= 1) epilogue -> records
  D.lines_log = it.use_i8 ? 1 : 0;
  D.fuse_decode = 1;
  D.it_epoch = P->epoch;
  D.fuse_commit = it.fuse_commit ? 1 : 0;
  D.cur_iter = iter;
  D.i8_iter = it.use_i8 ? 1 : 0;
  if (D.peer_mode) D.peer_epoch = ++P->peer_epoch;   // the same sequence on every shard (one per iteration)
  D.fused_sample = it.fused ? 1 : 0;
  if (it.fused) D.lines_log = 0;
  // first DIF pass gathering the discrete-log line (no load sweep) up to this FFT size (0: off); measured
  // (profiles/r02_experiments.md): C4's M = 1008 FFT -2 %, C3's 10080 / 2016-point lines slower (dependent gathers)
  static const int gather_max_M = getenv("SFFT_FFT_GATHER") ? atoi(getenv("SFFT_FFT_GATHER")) : 1024;
  D.fused_load = gather_max_M;
  const size_t fsm = it.fused ? it.fused_smem : P->fft[it.fi].smem_upto;
  LAUNCH(P, launch_pfft(D, it.n_active, P->L, (int)fsm, fft_threads(it.max_M, fsm, (int64_t)it.n_active * P->L), it.big,
                        it.fused ? 1 : it.ksplit, ptr<double2>(P, B_PART), it.max_p, st, fft_wl_for(it.max_M) && !it.fused));
  D.fused_sample = 0;
  D.fused_load = 0;
  D.lines_log = 0;
  D.fuse_decode = 0;
  D.fuse_commit = 0;
  D.i8_iter = 0;
  mark();
  return SFFT_OK;
}

// the C rows of the touched entries in the GPU-wide crow kernel when few signals are active (the commit grid
// leaves most SMs idle: single solves) and their rows are long: k* L >= 8192 elements per signal with k* ~ p / c
// (C3 / C4 / C5 first iterations).  Batched steps keep the rows in the commit CTAs, which already spread over the
// SMs: there the extra launch per iteration measured slower (C5 14.16 -> 14.53 ms, C4 2.59 -> 2.61 ms);
// single solves gain (C3 0.667 -> 0.632 ms, C4 0.446 -> 0.412 ms).  SFFT_CROW=0/1 forces the choice.
bool crow_on(const sfft_plan_t* P, const IterPlan& it) {
  static const int env = getenv("SFFT_CROW") ? atoi(getenv("SFFT_CROW")) : -1;
  if (env >= 0) return env != 0;
  return 4L * it.n_active <= P->n_sm && (long)(it.max_p / std::max(P->c, 1)) * P->L >= 8192;
}

int iter_back(sfft_plan_t* P, DevParams& D, int iter, const IterPlan& it, const sfft_signal_t* sig, int& launches) {
  cudaStream_t st = P->stream;
  if (!it.fuse_commit) {
    D.i8_iter = it.use_i8 ? 1 : 0;
    D.crow_mode = crow_on(P, it) ? 1 : 0;
    LAUNCH(P, launch_decode_commit(D, iter, it.max_p, it.n_active, st));
    D.i8_iter = 0;
    if (D.crow_mode) {
      // one CTA per work item of the largest iteration (every signal touching k entries), at most 8 per SM
      const long items = (long)it.n_active * ((P->k + 31) / 32) * D.crow_nl;
      LAUNCH(P, launch_crow(D, (int)std::min<long>(items, 8L * P->n_sm), st));
      D.crow_mode = 0;
    }
  }
  if (P->n_levels > 1) {                 // signals that switched fallback level (reading R23)
    LAUNCH(P, launch_retilt(D, sig->batch * D.spec_slots, sig->freqs, st));
    if (P->i8_ok) LAUNCH(P, launch_i8_prepare(D, sig->batch * D.spec_slots, P->k, st, true));
  }
  return SFFT_OK;
}

// per-signal status -> worst status; the host report (samples, cMACs, trace of signal 0)
int solve_report(sfft_plan_t* P, const DevParams& D, int32_t batch, const int32_t* ostat, sfft_report* rep,
                 int32_t last_iter, int launches, int32_t n_expsum, int32_t n_expsum_i8, int* worst_out) {
  cudaStream_t st = P->stream;
  std::vector<int32_t> hs(batch);
  int32_t spin_err = 0;
  CUDA_TRY(P, cudaMemcpyAsync(hs.data(), ostat, 4 * (size_t)batch, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(P, cudaMemcpyAsync(&spin_err, D.spin_err, 4, cudaMemcpyDeviceToHost, st));
  const int G = std::max(1, (int)D.spec_slots);
  const size_t slots = (size_t)batch * G;       // per-slot counters (R26: G slots per signal, all summed)
  std::vector<int64_t> hsamp(slots), hcm(slots), hcm8(slots);
  std::vector<double> hfw(2 * slots);
  std::vector<int32_t> hlog(2 * kLogIters), hlvl(slots);
  if (rep) {
    CUDA_TRY(P, cudaMemcpyAsync(hlvl.data(), D.st_lvl, 4 * slots, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(P, cudaMemcpyAsync(hsamp.data(), D.st_samples, 8 * slots, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(P, cudaMemcpyAsync(hcm.data(), D.st_cmacs, 8 * slots, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(P, cudaMemcpyAsync(hcm8.data(), D.st_cmacs_i8, 8 * slots, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(P, cudaMemcpyAsync(hfw.data(), D.st_fftw, 16 * slots, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(P, cudaMemcpyAsync(hlog.data(), D.st_log, 4 * 2 * kLogIters, cudaMemcpyDeviceToHost, st));
  }
  CUDA_TRY(P, cudaStreamSynchronize(st));
  if (spin_err) return fail(P, SFFT_ECUDA, "a cross-CTA stamp wait timed out (block scheduling assumption)");
  int worst = SFFT_OK, n_ok = 0, n_part = 0, n_err = 0;
  for (int s = 0; s < batch; ++s) {
    const int v = hs[s];
    if (v == SFFT_OK) ++n_ok;
    else if (v == SFFT_PARTIAL) { ++n_part; if (worst == SFFT_OK) worst = SFFT_PARTIAL; }
    else { ++n_err; if (worst >= 0) worst = v; }
  }
  *worst_out = worst;
  if (rep) {
    memset(rep, 0, sizeof *rep);
    for (size_t s = 0; s < slots; ++s) {
      rep->samples_used += hsamp[s];
      rep->cmacs += hcm[s];
      rep->cmacs_i8 += hcm8[s];
      rep->fft_plogp += hfw[2 * s];
      rep->fft_mlogm += hfw[2 * s + 1];
      rep->fallback_used += (s % G == 0) && hlvl[s] > 0;
    }
    rep->i8_limbs = P->i8_ok ? P->i8.S : 0;
    rep->n_expsum_i8 = n_expsum_i8;
    rep->iterations = last_iter;
    rep->n_ok = n_ok; rep->n_partial = n_part; rep->n_error = n_err;
    rep->status = worst;
    rep->n_iter_logged = std::min(last_iter, kLogIters);
    for (int i = 0; i < rep->n_iter_logged; ++i) { rep->primes[i] = hlog[2 * i]; rep->accepted[i] = hlog[2 * i + 1]; }
    rep->kernel_launches = launches;
    rep->n_expsum = n_expsum;
    rep->n_fused_sample = P->n_fused_iters;
  }
  return SFFT_OK;
}

// ---------------------------------------------------------------- NCCL (line sharding), loaded at run time
// Only the five entry points the record all-gather needs; types as in nccl.h (ABI-stable since 2.x).
struct NcclUid { char internal[128]; };
struct NcclApi {
  bool ok = false;
  int (*get_unique_id)(NcclUid*) = nullptr;
  int (*comm_init_rank)(void**, int, NcclUid, int) = nullptr;
  int (*all_gather)(const void*, void*, size_t, int, void*, cudaStream_t) = nullptr;
  int (*comm_destroy)(void*) = nullptr;
  const char* (*get_error_string)(int) = nullptr;
};
constexpr int kNcclInt64 = 4;   // ncclInt64

const NcclApi& nccl_api() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);   // the copy already loaded (torch)
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return a;
    a.get_unique_id = reinterpret_cast<int (*)(NcclUid*)>(dlsym(h, "ncclGetUniqueId"));
    a.comm_init_rank = reinterpret_cast<int (*)(void**, int, NcclUid, int)>(dlsym(h, "ncclCommInitRank"));
    a.all_gather = reinterpret_cast<int (*)(const void*, void*, size_t, int, void*, cudaStream_t)>(dlsym(h, "ncclAllGather"));
    a.comm_destroy = reinterpret_cast<int (*)(void*)>(dlsym(h, "ncclCommDestroy"));
    a.get_error_string = reinterpret_cast<const char* (*)(int)>(dlsym(h, "ncclGetErrorString"));
    a.ok = a.get_unique_id && a.comm_init_rank && a.all_gather && a.comm_destroy && a.get_error_string;
    return a;
  }();
  return api;
}

int nccl_allgather(sfft_plan_t* P, const int64_t* send, int64_t* recv, size_t words) {
  const NcclApi& n = nccl_api();
  const int r = n.all_gather(send, recv, words, kNcclInt64, P->nccl_comm, P->stream);
  if (r != 0) return fail(P, SFFT_ENCCL, "ncclAllGather: %s", n.get_error_string(r));
  return SFFT_OK;
}

}  // namespace

extern "C" {

const char* sfft_version(void) { return "sfft sm_100a " SFFT_GIT; }

const char* sfft_strerror(int s) {
  switch (s) {
    case SFFT_OK: return "ok";
    case SFFT_PARTIAL: return "partial result (stall or max_iter)";
    case SFFT_EINVAL: return "invalid argument";
    case SFFT_EPRECISION: return "precision budget exceeded (N^d_q > 2^40 or E > 2^42)";
    case SFFT_EDIM: return "dimension / batch mismatch";
    case SFFT_ECORRUPT: return "corrupt recovery (untilt or wrap failed)";
    case SFFT_ECUDA: return "CUDA error";
    case SFFT_ENOMEM: return "out of device memory";
    case SFFT_ENCCL: return "NCCL error";
    case SFFT_ENOTSUP: return "not supported (prime beyond the FFT size table, or more plan slots than the slot assignment holds)";
  }
  return "unknown status";
}

const char* sfft_last_error(const sfft_plan_t* plan) { return plan ? plan->err.c_str() : "null plan"; }

int sfft_plan(int32_t d, int64_t N, int32_t k, const int64_t* primes, int32_t n_primes, const sfft_tilt* tilts,
              int32_t n_tilts, double eps, const sfft_options* opt, sfft_plan_t** out) {
  if (!out) return SFFT_EINVAL;
  *out = nullptr;
  std::unique_ptr<sfft_plan_t> P(new (std::nothrow) sfft_plan_t());
  if (!P) return SFFT_ENOMEM;
  if (d < 1 || k < 1 || N < 2 || (N % 2) != 0 || N > ((int64_t)1 << 31) || n_primes < 0 || n_tilts < 0)
    return SFFT_EINVAL;
  P->d = d; P->N = N; P->k = k;
  if (opt) {
    if (opt->c > 0) P->c = opt->c;
    if (opt->tol > 0) P->tol = opt->tol;
    if (opt->bin_floor_rel > 0) P->floor_rel = opt->bin_floor_rel;
    if (opt->prune_floor > 0) P->prune = opt->prune_floor;
    if (opt->round_tol > 0) P->round_tol = opt->round_tol;
    if (opt->max_iter > 0) P->max_iter = opt->max_iter;
    if (opt->stall_limit > 0) P->stall_limit = opt->stall_limit;
    if (opt->batch > 0) P->batch = opt->batch;
    if (opt->extra_checks >= 0) P->extra = opt->extra_checks & 3;
    P->stream = (cudaStream_t)opt->stream;
    P->profile = opt->profile != 0;
    P->literal = opt->literal_residual != 0;
    P->expsum_path = opt->expsum_path;
    if (P->expsum_path < 0 || P->expsum_path > 2) return SFFT_EINVAL;
    if (opt->fallback_tilts < 0 || opt->fallback_tilts > kMaxFallbackLevels) return SFFT_EINVAL;
    if (opt->table_cache_slots < 0 || opt->table_cache_slots > (1 << 16)) return SFFT_EINVAL;
    if (opt->line_shards < 0 || (opt->line_shards > 0 && (opt->line_rank < 0 || opt->line_rank >= opt->line_shards)))
      return SFFT_EINVAL;
    P->line_G = opt->line_shards;
    P->line_g = opt->line_shards > 0 ? opt->line_rank : 0;
    if (opt->line_exchange < 0 || opt->line_exchange > 1) return SFFT_EINVAL;
    if (opt->line_exchange == 1 && (opt->line_shards < 1 || opt->line_shards > kMaxPeers)) return SFFT_EINVAL;
    P->line_exchange = opt->line_exchange;
    if (opt->spec_primes < 0 || opt->spec_primes > 16) return SFFT_EINVAL;
    if (opt->spec_distributed && (opt->spec_primes < 2 || opt->spec_rank < 0 || opt->spec_rank >= opt->spec_primes))
      return SFFT_EINVAL;
    if (opt->spec_primes > 1) {
      // R26: G slots per signal (each its own prime and registry copy) or one per rank; not with line shards (their
      // records are per line, not per prime), the literal residual or an explicit batch of slots beyond 2^20
      if (opt->line_shards > 0 || opt->literal_residual || (int64_t)P->batch * opt->spec_primes > (1 << 20))
        return SFFT_EINVAL;
      P->spec_G = opt->spec_primes;
      P->spec_dist = opt->spec_distributed ? 1 : 0;
      P->spec_rank = P->spec_dist ? opt->spec_rank : 0;
      P->spec_slots = P->spec_dist ? 1 : P->spec_G;
      P->batch *= P->spec_slots;
    }
  }
  // partition: explicit, or uniform largest d1 | d with N^d1 <= 2^40
  const double log2N = std::log2((double)N);
  if (opt && opt->n_blocks > 0 && opt->block_dims) {
    int32_t sum = 0;
    for (int q = 0; q < opt->n_blocks; ++q) {
      if (opt->block_dims[q] < 1) return SFFT_EINVAL;
      P->blocks.push_back(opt->block_dims[q]);
      sum += opt->block_dims[q];
    }
    if (sum != d) return SFFT_EINVAL;
  } else {
    int d1 = 1;
    for (int t = 1; t <= d; ++t)
      if (d % t == 0 && t * log2N <= 40.0 + 1e-9) d1 = t;
    for (int q = 0; q < d / d1; ++q) P->blocks.push_back(d1);
  }
  P->r = (int32_t)P->blocks.size();
  P->L = P->r + 1;
  P->L_ref = P->L;
  if (P->line_G > 0) {
    if (P->line_G > P->r) return SFFT_EINVAL;                 // every shard owns at least one shifted line
    int lo, hi, lo0, hi0;
    line_shard_range(P->r, P->line_G, P->line_g, &lo, &hi);
    line_shard_range(P->r, P->line_G, 0, &lo0, &hi0);
    P->line_lo = lo;
    P->L = 1 + (hi - lo);
    P->L_ref = 1 + (hi0 - lo0);
  }
  P->rec_fw = (k + 1) / 2;
  P->rec_words = P->rec_fw + (P->L_ref - 1) * k;
  if (P->spec_dist) {            // R26 distributed: + (nc, p, m) header, candidate bins, F_0 at them
    P->spec_tail = P->rec_words;
    P->rec_words += 2 + (k + 1) / 2 + 2 * k;
  }
  int64_t B = 1;
  int32_t off = 0;
  for (int q = 0; q < P->r; ++q) {
    if (P->blocks[q] * log2N > 40.0 + 1e-9) return SFFT_EPRECISION;   // reading R1
    int64_t b = 1;
    for (int t = 0; t < P->blocks[q]; ++t) b *= N;
    B = std::max(B, b);
    P->block_off.push_back(off);
    off += P->blocks[q];
  }
  // image interval of every block, tilts (Eq. (25)/(27)), E (reading R2)
  std::vector<int64_t> blo(P->r), bhi(P->r);
  for (int q = 0; q < P->r; ++q) {
    int64_t geo = 0, pw = 1;
    for (int t = 0; t < P->blocks[q]; ++t) { geo += pw; pw *= N; }
    blo[q] = -(N / 2) * geo;
    bhi[q] = (N / 2 - 1) * geo;
  }
  P->lo = blo;
  P->hi = bhi;
  P->axis_tilt.assign(P->r, -1);
  int64_t scale = 1;
  for (int t = 0; t < n_tilts; ++t) {
    const sfft_tilt& T = tilts[t];
    const int a0 = T.axis0, a1 = T.axis1;
    if (a0 < 0 || a1 < 0 || a0 >= P->r || a1 >= P->r || a0 == a1) return SFFT_EINVAL;
    if (P->axis_tilt[a0] >= 0 || P->axis_tilt[a1] >= 0) return SFFT_EINVAL;
    const int64_t b = T.base, h = T.height, c = T.hypo;
    if (b < 1 || h < 1 || b * b + h * h != c * c || gcd64(b, c) != 1 || gcd64(h, c) != 1) return SFFT_EINVAL;
    P->axis_tilt[a0] = 2 * t;
    P->axis_tilt[a1] = 2 * t + 1;
    P->tilts.insert(P->tilts.end(), {(int64_t)a0, (int64_t)a1, b, h, c});
    P->lo[a0] = b * blo[a0] - h * bhi[a1];
    P->hi[a0] = b * bhi[a0] - h * blo[a1];
    P->lo[a1] = h * blo[a0] + b * blo[a1];
    P->hi[a1] = h * bhi[a0] + b * bhi[a1];
    scale = std::max(scale, b + h);
  }
  if (eps == 0.0) {
    P->E = 2 * B * scale;
  } else {
    if (!(eps > 0.0)) return SFFT_EINVAL;
    const double Ed = std::nearbyint(1.0 / eps);
    if (std::fabs(Ed * eps - 1.0) > 1e-12) return SFFT_EINVAL;
    P->E = (int64_t)Ed;
  }
  if (P->E > ((int64_t)1 << 42)) return SFFT_EPRECISION;
  for (int q = 0; q < P->r; ++q)
    if (2 * P->hi[q] >= P->E || -2 * P->lo[q] > P->E) return SFFT_EINVAL;
  if (P->stall_limit <= 0) P->stall_limit = std::max(2 * P->r, 16);
  // fallback levels: level 0 = this plan; level l in 1..4 (reading R23) = Pythagorean triple l-1 on the disjoint
  // reduced-axis pairs (q, q + s) -- s = 1 from axis 0 (l = 1), s = 1 from axis 1 (l = 2, r >= 3), s = 2 (l = 3),
  // s = 3 (l = 4); level l >= 5 (reading R24, "randomizing the order of the dimensions") = round l - 5 of
  // the circle-method round robin over a seeded order of the axes, triple (l - 5) mod 4, so that the r - 1 (r
  // even) rounds tilt every pair of axes once; E = 2 B (base + height) (reading R2); the schedule stops at the
  // first empty level
  {
    static const int64_t kTri[4][3] = {{3, 4, 5}, {5, 12, 13}, {8, 15, 17}, {7, 24, 25}};
    const int n_fb = opt ? opt->fallback_tilts : 0;
    std::vector<std::vector<int64_t>> lt(1, P->tilts);
    std::vector<int64_t> lE(1, P->E);
    // seeded axis order (Fisher-Yates driven by a splitmix64 counter; reading R24)
    std::vector<int> order(P->r);
    for (int i = 0; i < P->r; ++i) order[i] = i;
    for (int i = P->r - 1; i >= 1; --i) {
      uint64_t z = 1ull * 0x9E3779B97F4A7C15ull + (uint64_t)(P->r - i) * 0xD1B54A32D192ED03ull;
      z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
      z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
      z ^= z >> 31;
      std::swap(order[i], order[(int)(z % (uint64_t)(i + 1))]);
    }
    for (int l = 1; l <= n_fb; ++l) {
      const int64_t* T = kTri[l <= 4 ? l - 1 : (l - 5) % 4];
      std::vector<int64_t> ts;
      if (l <= 4) {
        const int st = l <= 2 ? 1 : l - 1;
        const int off = (l == 2 && P->r >= 3) ? 1 : 0;
        for (int b = off; b < P->r; b += 2 * st)
          for (int i = 0; i < st && b + i + st < P->r; ++i) ts.insert(ts.end(), {b + i, b + i + st, T[0], T[1], T[2]});
      } else {
        const int j = l - 5, n = P->r + (P->r & 1);       // round j over n slots (one padding slot when r is odd)
        if (j < n - 1)
          for (int i = 0; i < n / 2; ++i) {
            const int x = i == 0 ? 0 : 1 + (i - 1 + j) % (n - 1);
            const int y = 1 + (n - 2 - i + j) % (n - 1);    // slot n-1-i after the rotation
            if (x < P->r && y < P->r) ts.insert(ts.end(), {order[x], order[y], T[0], T[1], T[2]});
          }
      }
      if (ts.empty()) break;
      const int64_t El = 2 * B * (T[0] + T[1]);
      if (El > ((int64_t)1 << 42)) break;
      lt.push_back(ts);
      lE.push_back(El);
    }
    P->n_levels = (int32_t)lt.size();
    size_t tmax = 1;
    for (auto& t : lt) tmax = std::max(tmax, t.size() / 5);
    P->lvl_tmax = (int32_t)tmax;
    P->lvl_E = lE;
    P->lvl_tilts.assign((size_t)P->n_levels * tmax * 5, 0);
    P->lvl_nt.assign(P->n_levels, 0);
    P->lvl_axt.assign((size_t)P->n_levels * P->r, -1);
    P->lvl_lo.assign((size_t)P->n_levels * P->r, 0);
    P->lvl_hi.assign((size_t)P->n_levels * P->r, 0);
    for (int l = 0; l < P->n_levels; ++l) {
      const std::vector<int64_t>& ts = lt[l];
      P->lvl_nt[l] = (int32_t)(ts.size() / 5);
      std::copy(ts.begin(), ts.end(), P->lvl_tilts.begin() + (size_t)l * tmax * 5);
      int64_t* lo = P->lvl_lo.data() + (size_t)l * P->r;
      int64_t* hi = P->lvl_hi.data() + (size_t)l * P->r;
      int32_t* axt = P->lvl_axt.data() + (size_t)l * P->r;
      for (int q = 0; q < P->r; ++q) { lo[q] = blo[q]; hi[q] = bhi[q]; }
      for (size_t t = 0; t < ts.size() / 5; ++t) {
        const int a0 = (int)ts[5 * t], a1 = (int)ts[5 * t + 1];
        const int64_t b = ts[5 * t + 2], h = ts[5 * t + 3];
        axt[a0] = 2 * (int)t;
        axt[a1] = 2 * (int)t + 1;
        lo[a0] = b * blo[a0] - h * bhi[a1];
        hi[a0] = b * bhi[a0] - h * blo[a1];
        lo[a1] = h * blo[a0] + b * blo[a1];
        hi[a1] = h * bhi[a0] + b * bhi[a1];
      }
    }
  }
  // device limits -> FFT sizes, p_cap, prime table
  cudaError_t ce = cudaGetDevice(&P->device);
  if (ce != cudaSuccess) return fail(nullptr, SFFT_ECUDA, "no device");
  int smem_optin = 0;
  ce = cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, P->device);
  if (ce != cudaSuccess) return SFFT_ECUDA;
  cudaDeviceGetAttribute(&P->n_sm, cudaDevAttrMultiProcessorCount, P->device);
  P->smem_optin = smem_optin;
  int M_max = 0;
  for (int M = 3; M <= 20000; ++M)
    if (is_7smooth(M)) {
      FftSize f = radix_plan(M);
      if (f.smem > (size_t)smem_optin) continue;
      if ((int)f.radix.size() + 1 > kMaxFftPasses) continue;
      f.smem_upto = std::max(f.smem, P->fft.empty() ? (size_t)0 : P->fft.back().smem_upto);
      P->fft.push_back(f);
      M_max = M;
    }
  // per-pass twiddle table layout for every FFT size
  P->tw_off.assign(P->fft.size() * kMaxFftPasses, 0);
  for (size_t i = 0; i < P->fft.size(); ++i) {
    int S = P->fft[i].M;
    for (size_t ps = 0; ps < P->fft[i].radix.size(); ++ps) {
      const int R = P->fft[i].radix[ps];
      P->tw_off[i * kMaxFftPasses + ps] = (int32_t)P->tw_total;
      P->tw_seg.push_back(make_int4((int)P->tw_total, S, R, 0));
      P->tw_total += (size_t)(S / R);
      S /= R;
    }
    P->tw_off[i * kMaxFftPasses + P->fft[i].radix.size()] = (int32_t)P->tw_total;   // end marker
  }
  P->p_cap = 0;
  {
    const int lim = (M_max + 1) / 2;
    std::vector<char> comp(lim + 1, 0);
    for (int x = 2; x <= lim; ++x) {
      if (comp[x]) continue;
      P->primes.push_back(x);
      for (long y = (long)x * x; y <= lim; y += x) comp[y] = 1;
    }
    P->p_cap = P->primes.back();
    // the setup kernel's lookup of the i-th prime >= x: two loads instead of a binary search
    P->prime_tab = P->primes;
    size_t j = 0;
    for (int x = 0; x <= lim + 1; ++x) {
      while (j < P->primes.size() && P->primes[j] < x) ++j;
      P->prime_tab.push_back((int32_t)j);
    }
  }
  if (primes && n_primes > 0) {
    for (int i = 0; i < n_primes; ++i) {
      if (primes[i] < 2 || primes[i] > P->p_cap) return SFFT_ENOTSUP;
      P->sched.push_back(primes[i]);
    }
  } else {
    // the first prime c k must be supported
    int64_t first = 0;
    for (int32_t x : P->primes)
      if (x >= std::max<int64_t>(2, (int64_t)P->c * k)) { first = x; break; }
    if (first == 0) return SFFT_ENOTSUP;
  }
  P->p_stride = align_up((size_t)P->p_cap, 32);
  P->M_stride = align_up((size_t)M_max, 32);
  P->kk = 2 * k;
  P->H = 1;
  while (P->H < 2 * k) P->H <<= 1;
  P->shape = choose_expsum_shape(P->L_ref);
  P->Lp = P->shape.nt * P->shape.bn;
  // int8-limb tensor-core exp-sum (bin-domain residual only: its B limbs are the fixed signal rows)
  if (P->expsum_path != 1 && !P->literal)
    P->i8_ok = i8_configure(P->L_ref, *std::max_element(P->lvl_E.begin(), P->lvl_E.end()), P->k, &P->i8);
  if (P->i8_ok && P->i8.small_l && P->expsum_path == 0) P->i8_ok = false;
  if (P->expsum_path == 2 && !P->i8_ok) return SFFT_ENOTSUP;
  // short lines on the FP64 path: each FFT CTA samples its own line (NEXT #3 fusion); SFFT_NO_FUSED_LINES=1 keeps
  // the separate exp-sum launch (A/B, parity)
  P->fs_ok = P->expsum_path == 0 && !P->i8_ok && !P->literal && P->L_ref <= kFusedMaxL && !getenv("SFFT_NO_FUSED_LINES");
  // shared-memory budgets of the other kernels
  if (16 * ((size_t)P->p_stride + 2) + 2 * 16 * 16 * (size_t)P->shape.bn + 256 > (size_t)smem_optin) return SFFT_ENOTSUP;
  if (8 * (size_t)P->p_stride + 4 * (2 * (size_t)P->p_stride + 2 * (size_t)k + 64) > (size_t)smem_optin)
    return SFFT_ENOTSUP;
  if (8 * (size_t)k > (size_t)smem_optin) return SFFT_ENOTSUP;
  // at most batch primes are live per iteration; the rest keeps recent primes, so that repeated executes (and later
  // iterations revisiting a prime) reuse their tables -- like FFT twiddle tables, they depend on p only (~0.8 MB
  // per slot at p_cap ~ 7056)
  P->n_tslots = std::max(P->batch + 16, kDefaultTableSlots);
  if (opt && opt->table_cache_slots > 0) P->n_tslots = std::max(P->batch + 16, (int)opt->table_cache_slots);
  {
    // the slot assignment keeps a prime -> slot hash map of >= 2 n_tslots entries in one CTA's shared memory
    // (k_fft.cu assign_slots): about 8000 slots (signals x spec_primes, or table_cache_slots) at most
    size_t hs = 2048;
    while (hs < 2 * (size_t)P->n_tslots) hs <<= 1;
    if (sizeof(int) * (2 * hs + 2 * 4096 + (size_t)P->n_tslots) > (size_t)smem_optin) return SFFT_ENOTSUP;
  }
  layout(P.get());
  *out = P.release();
  return SFFT_OK;
}

int sfft_plan_workspace_size(const sfft_plan_t* plan, size_t* bytes) {
  if (!plan || !bytes) return SFFT_EINVAL;
  *bytes = plan->ws_bytes;
  return SFFT_OK;
}

int sfft_plan_set_workspace(sfft_plan_t* plan, void* dptr, size_t bytes) {
  if (!plan || !dptr || bytes < plan->ws_bytes || ((uintptr_t)dptr & 255)) return SFFT_EINVAL;
  if (plan->ws_owned) cudaFree(plan->ws);
  plan->ws = dptr;
  plan->ws_owned = false;
  plan->tables_ready = false;
  return SFFT_OK;
}

int sfft_plan_info(const sfft_plan_t* plan, int64_t* E, int32_t* r, int32_t* L, int64_t* p_max, int32_t* tile_n) {
  if (!plan) return SFFT_EINVAL;
  if (E) *E = plan->E;
  if (r) *r = plan->r;
  if (L) *L = plan->L;
  if (p_max) *p_max = plan->p_cap;
  if (tile_n) *tile_n = plan->shape.bn;
  return SFFT_OK;
}

void sfft_plan_destroy(sfft_plan_t* plan) {
  if (!plan) return;
  if (plan->nccl_comm && nccl_api().ok) nccl_api().comm_destroy(plan->nccl_comm);
  for (size_t h = 0; h < plan->peer_opened.size(); ++h)
    if (plan->peer_opened[h] && plan->peer_ptr[h]) cudaIpcCloseMemHandle(plan->peer_ptr[h]);
  if (plan->peer_buf) cudaFree(plan->peer_buf);
  if (plan->ws_owned && plan->ws) cudaFree(plan->ws);
  if (plan->h_ctrl) cudaFreeHost(plan->h_ctrl);
  if (plan->ev_ctrl) cudaEventDestroy(plan->ev_ctrl);
  for (cudaEvent_t e : plan->events) cudaEventDestroy(e);
  if (plan->pipe_buf) cudaFree(plan->pipe_buf);
  for (cudaStream_t s : plan->pipe_st)
    if (s) cudaStreamDestroy(s);
  for (cudaEvent_t e : plan->pipe_ev)
    if (e) cudaEventDestroy(e);
  delete plan;
}

int sfft_signal_expsum(sfft_plan_t* plan, int32_t batch, const int32_t* freqs, const double* coeffs,
                       sfft_signal_t** out) {
  if (!plan || !out || !freqs || !coeffs) return SFFT_EINVAL;
  if (batch < 1 || batch > plan->batch / plan->spec_slots)
    return fail(plan, SFFT_EDIM, "batch %d outside [1, %d]", batch, plan->batch / plan->spec_slots);
  sfft_signal_t* s = new (std::nothrow) sfft_signal_t();
  if (!s) return SFFT_ENOMEM;
  s->plan = plan;
  s->batch = batch;
  s->freqs = freqs;
  s->coeffs = coeffs;
  *out = s;
  return SFFT_OK;
}

void sfft_signal_destroy(sfft_signal_t* sig) { delete sig; }

int sfft_execute(sfft_plan_t* plan, const sfft_signal_t* sig, int32_t* out_freqs, double* out_coeffs,
                 int32_t* out_count, int32_t* out_status, sfft_report* rep) {
  if (!plan || !sig || sig->plan != plan || !out_freqs || !out_coeffs || !out_count) return SFFT_EINVAL;
  if (plan->line_exchange == 1 && !plan->peer_ready)
    return fail(plan, SFFT_EINVAL, "fused record exchange needs sfft_comm_init_peers or sfft_execute_group");
  if (plan->line_exchange == 0 && plan->line_G > 1 && !plan->nccl_comm)
    return fail(plan, SFFT_EINVAL, "line-sharded plan (%d shards) needs sfft_comm_init or sfft_execute_group", plan->line_G);
  if (plan->spec_dist && !plan->nccl_comm)
    return fail(plan, SFFT_EINVAL, "distributed speculation (%d ranks) needs sfft_comm_init or sfft_execute_group",
                plan->spec_G);
  int rc = ensure_ready(plan);
  if (rc) return rc;
  sfft_plan_t* P = plan;
  cudaStream_t st = P->stream;
  NvtxRange nv_solve("sfft_execute");
  const int32_t batch = sig->batch;                 // signals; slots = batch G (R26)
  DevParams D = dev_params(P, batch * P->spec_slots);
  D.spec_G = P->spec_G;
  D.spec_slots = P->spec_slots;
  int launches = 0;
  // profiling: event marks on the stream, 5 per iteration (prep | expsum | pfft | decode)
  size_t n_ev = 0;
  auto mark = [&]() -> int {
    if (!P->profile) return 0;
    if (n_ev == P->events.size()) {
      cudaEvent_t e;
      if (cudaEventCreate(&e) != cudaSuccess) return -1;
      P->events.push_back(e);
    }
    return cudaEventRecord(P->events[n_ev++], st) == cudaSuccess ? 0 : -1;
  };
  mark();
  P->n_fused_iters = 0;
  if ((rc = solve_begin(P, D, sig, launches))) return rc;
  int iter = 1;
  int32_t last_iter = 0, n_expsum = 0, n_expsum_i8 = 0;
  std::vector<size_t> it_marks, it_i8;
  int n_bound = batch * P->spec_slots;
  for (; iter <= P->max_iter; ++iter) {
    NvtxRange nv_it("sfft iteration %d", iter);
    IterPlan it;
    if ((rc = iter_setup(P, D, iter, &it, launches, n_bound))) return rc;
    n_bound = it.n_active;
    if (it.n_active == 0) break;
    if (P->profile) it_marks.push_back(n_ev);
    mark();
    if ((rc = iter_front(P, D, iter, it, launches, mark))) return rc;
    if (P->line_G > 0 && !D.peer_mode) {
      // line sharding: all-gather of this shard's records (one rank: a device copy), then the commit
      const size_t words = (size_t)batch * P->rec_words;
      if (P->nccl_comm) {
        if ((rc = nccl_allgather(P, ptr<int64_t>(P, B_RSEND), ptr<int64_t>(P, B_RRECV), words))) return rc;
      } else {
        CUDA_TRY(P, cudaMemcpyAsync(ptr<int64_t>(P, B_RRECV), ptr<int64_t>(P, B_RSEND), 8 * words,
                                    cudaMemcpyDeviceToDevice, st));
      }
    } else if (P->spec_dist) {
      // R26 distributed: every rank's records (with their tails) to every rank; the commits merge them in rank order
      if ((rc = nccl_allgather(P, ptr<int64_t>(P, B_RSEND), ptr<int64_t>(P, B_RRECV), (size_t)batch * P->rec_words)))
        return rc;
    }
    if ((rc = iter_back(P, D, iter, it, sig, launches))) return rc;
    ++n_expsum;
    if (it.use_i8) { ++n_expsum_i8; it_i8.push_back(it_marks.empty() ? 0 : it_marks.back()); }
    mark();
    last_iter = iter;
  }
  int32_t* ostat = out_status ? out_status : ptr<int32_t>(P, B_OUT_S);
  LAUNCH(P, launch_wrap(D, batch, out_freqs, out_coeffs, out_count, ostat, ptr<int32_t>(P, B_WRAPS), st));
  launches += 2;   // digits, rank, gather
  mark();
  int worst = 0;
  if ((rc = solve_report(P, D, batch, ostat, rep, last_iter, launches, n_expsum, n_expsum_i8, &worst))) return rc;
  if (rep && P->profile && getenv("SFFT_DEBUG")) {
    for (size_t it = 0; it < it_marks.size(); ++it) {
      float a = 0, b = 0, c = 0, d = 0;
      const size_t m0 = it_marks[it];
      cudaEventElapsedTime(&a, P->events[m0], P->events[m0 + 1]);
      cudaEventElapsedTime(&b, P->events[m0 + 1], P->events[m0 + 2]);
      cudaEventElapsedTime(&c, P->events[m0 + 2], P->events[m0 + 3]);
      cudaEventElapsedTime(&d, P->events[m0 + 3], P->events[m0 + 4]);
      float g = 0;       // from the previous mark (end of the last iteration / solve start) to this prep
      cudaEventElapsedTime(&g, P->events[m0 - 1], P->events[m0]);
      fprintf(stderr, "[sfft] iter %zu gap+setup %.3f prep %.3f expsum %.3f pfft %.3f decode %.3f ms\n", it + 1, g, a, b,
              c, d);
    }
    float w = 0, b0 = 0;
    cudaEventElapsedTime(&w, P->events[n_ev - 2], P->events[n_ev - 1]);
    if (!it_marks.empty()) cudaEventElapsedTime(&b0, P->events[0], P->events[it_marks[0]]);
    fprintf(stderr, "[sfft] begin+iter1 setup %.3f wrap %.3f ms\n", b0, w);
  }
  if (rep && P->profile && n_ev >= 2) {
    auto el = [&](size_t a, size_t b) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, P->events[a], P->events[b]);
      return ms;
    };
    float tot = el(0, n_ev - 1), fx = 0.f, ff = 0.f, fd = 0.f;
    for (size_t m0 : it_marks) {
      ff += el(m0, m0 + 1) + el(m0 + 2, m0 + 3);
      fx += el(m0 + 1, m0 + 2);
      fd += el(m0 + 3, m0 + 4);
    }
    rep->ms_expsum = fx;
    for (size_t m0 : it_i8) rep->ms_expsum_i8 += el(m0 + 1, m0 + 2);
    rep->ms_fft = ff;
    rep->ms_decode = fd;
    rep->ms_other = tot - fx - ff - fd;
    rep->ms_total = tot;
  }
  return worst;
}

int sfft_execute_group(sfft_plan_t* const* plans, const sfft_signal_t* const* sigs, int32_t n_plans,
                       int32_t* out_freqs, double* out_coeffs, int32_t* out_count, int32_t* out_status,
                       sfft_report* rep) {
  if (!plans || !sigs || n_plans < 1 || !out_freqs || !out_coeffs || !out_count) return SFFT_EINVAL;
  sfft_plan_t* P0 = plans[0];
  if (!P0) return SFFT_EINVAL;
  const int G = n_plans;
  const bool spec = P0->spec_dist != 0;      // R26 distributed: plans = the G ranks of one speculation
  for (int g = 0; g < G; ++g) {
    sfft_plan_t* P = plans[g];
    if (!P || !sigs[g] || sigs[g]->plan != P) return SFFT_EINVAL;
    if (spec && (!P->spec_dist || P->spec_G != G || P->spec_rank != g))
      return fail(P0, SFFT_EINVAL, "plan %d is not speculation rank %d of %d", g, g, G);
    if (!spec && (P->line_G != G || P->line_g != g))
      return fail(P0, SFFT_EINVAL, "plan %d is not line shard %d of %d", g, g, G);
    if (P->stream != P0->stream || P->device != P0->device) return fail(P0, SFFT_EINVAL, "shards must share device and stream");
    if (P->k != P0->k || P->r != P0->r || P->d != P0->d || sigs[g]->batch != sigs[0]->batch) return SFFT_EINVAL;
    const int rc = ensure_ready(P);
    if (rc) return rc;
  }
  cudaStream_t st = P0->stream;
  const int32_t batch = sigs[0]->batch;
  // fused record exchange: every shard's FFT epilogue stores into the buffers of all shards of the group (plain
  // device pointers, the same code path as the IPC mappings across GPUs)
  const bool fused = P0->line_exchange == 1;
  for (int g = 0; g < G; ++g)
    if ((plans[g]->line_exchange == 1) != fused) return fail(P0, SFFT_EINVAL, "shards disagree on line_exchange");
  if (fused) {
    for (int g = 0; g < G; ++g) {
      const int rc0 = ensure_peer_buf(plans[g]);
      if (rc0) return rc0;
    }
    for (int g = 0; g < G; ++g) {
      plans[g]->peer_ptr.assign(G, nullptr);
      plans[g]->peer_opened.assign(G, false);
      for (int h = 0; h < G; ++h) plans[g]->peer_ptr[h] = plans[h]->peer_buf;
      plans[g]->peer_ready = true;
    }
  }
  std::vector<DevParams> D(G);
  int launches = 0, rc;
  auto nomark = []() -> int { return 0; };
  for (int g = 0; g < G; ++g) plans[g]->n_fused_iters = 0;
  for (int g = 0; g < G; ++g) {
    D[g] = dev_params(plans[g], batch);
    D[g].spec_G = plans[g]->spec_G;
    if ((rc = solve_begin(plans[g], D[g], sigs[g], launches))) return rc;
  }
  int32_t last_iter = 0, n_expsum = 0, n_expsum_i8 = 0;
  const size_t words = (size_t)batch * P0->rec_words;
  int n_bound = batch;
  for (int iter = 1; iter <= P0->max_iter; ++iter) {
    std::vector<IterPlan> it(G);
    for (int g = 0; g < G; ++g) {
      if ((rc = iter_setup(plans[g], D[g], iter, &it[g], launches, n_bound))) return rc;
      if (it[g].n_active != it[0].n_active || (!spec && it[g].max_p != it[0].max_p))   // ranks: own primes
        return fail(P0, SFFT_ECORRUPT, "shards diverged at iteration %d", iter);
    }
    if (it[0].n_active == 0) break;
    n_bound = it[0].n_active;
    for (int g = 0; g < G; ++g)
      if ((rc = iter_front(plans[g], D[g], iter, it[g], launches, nomark))) return rc;
    for (int g = 0; g < G && !fused; ++g)   // the all-gather: shard g's records into slot g of every shard
      for (int h = 0; h < G; ++h)
        CUDA_TRY(P0, cudaMemcpyAsync(ptr<int64_t>(plans[h], B_RRECV) + (size_t)g * words, ptr<int64_t>(plans[g], B_RSEND),
                                     8 * words, cudaMemcpyDeviceToDevice, st));
    for (int g = 0; g < G; ++g)
      if ((rc = iter_back(plans[g], D[g], iter, it[g], sigs[g], launches))) return rc;
    ++n_expsum;
    if (it[0].use_i8) ++n_expsum_i8;
    last_iter = iter;
  }
  // the shards' registries must be bitwise identical (same F_0, same records, same update order)
  {
    std::vector<int32_t> nR0(batch), nRg(batch);
    CUDA_TRY(P0, cudaMemcpyAsync(nR0.data(), D[0].st_nR, 4 * (size_t)batch, cudaMemcpyDeviceToHost, st));
    const size_t va = 8 * (size_t)batch * P0->r * P0->kk, aa = 16 * (size_t)batch * P0->k;
    std::vector<char> v0(va), a0(aa), vg(va), ag(aa);
    CUDA_TRY(P0, cudaMemcpyAsync(v0.data(), D[0].v_all, va, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(P0, cudaMemcpyAsync(a0.data(), D[0].a_reg, aa, cudaMemcpyDeviceToHost, st));
    for (int g = 1; g < G; ++g) {
      CUDA_TRY(P0, cudaMemcpyAsync(nRg.data(), D[g].st_nR, 4 * (size_t)batch, cudaMemcpyDeviceToHost, st));
      CUDA_TRY(P0, cudaMemcpyAsync(vg.data(), D[g].v_all, va, cudaMemcpyDeviceToHost, st));
      CUDA_TRY(P0, cudaMemcpyAsync(ag.data(), D[g].a_reg, aa, cudaMemcpyDeviceToHost, st));
      CUDA_TRY(P0, cudaStreamSynchronize(st));
      for (int s = 0; s < batch; ++s) {
        if (nRg[s] != nR0[s]) return fail(P0, SFFT_ECORRUPT, "shard %d signal %d: |R| %d vs %d", g, s, nRg[s], nR0[s]);
        for (int q = 0; q < P0->r; ++q) {
          const size_t o = 8 * (((size_t)s * P0->r + q) * P0->kk + P0->k);
          if (memcmp(v0.data() + o, vg.data() + o, 8 * (size_t)nR0[s]))
            return fail(P0, SFFT_ECORRUPT, "shard %d signal %d: registry keys differ", g, s);
        }
        if (memcmp(a0.data() + 16 * (size_t)s * P0->k, ag.data() + 16 * (size_t)s * P0->k, 16 * (size_t)nR0[s]))
          return fail(P0, SFFT_ECORRUPT, "shard %d signal %d: registry coefficients differ", g, s);
      }
    }
  }
  sfft_plan_t* P = P0;
  int32_t* ostat = out_status ? out_status : ptr<int32_t>(P, B_OUT_S);
  LAUNCH(P, launch_wrap(D[0], batch, out_freqs, out_coeffs, out_count, ostat, ptr<int32_t>(P, B_WRAPS), st));
  launches += 2;
  int worst = 0;
  if ((rc = solve_report(P, D[0], batch, ostat, rep, last_iter, launches, n_expsum, n_expsum_i8, &worst))) return rc;
  if (rep) {            // exp-sum work of every shard (and, for speculation ranks, their own primes' samples)
    for (int g = 1; g < G; ++g) {
      std::vector<int64_t> hcm(batch), hcm8(batch), hsm(batch);
      CUDA_TRY(P0, cudaMemcpyAsync(hcm.data(), D[g].st_cmacs, 8 * (size_t)batch, cudaMemcpyDeviceToHost, st));
      CUDA_TRY(P0, cudaMemcpyAsync(hcm8.data(), D[g].st_cmacs_i8, 8 * (size_t)batch, cudaMemcpyDeviceToHost, st));
      CUDA_TRY(P0, cudaMemcpyAsync(hsm.data(), D[g].st_samples, 8 * (size_t)batch, cudaMemcpyDeviceToHost, st));
      CUDA_TRY(P0, cudaStreamSynchronize(st));
      for (int s = 0; s < batch; ++s) {
        rep->cmacs += hcm[s];
        rep->cmacs_i8 += hcm8[s];
        if (spec) rep->samples_used += hsm[s];
      }
    }
  }
  return worst;
}

int sfft_solve_host(sfft_plan_t* plan, int32_t batch, const int32_t* freqs, const double* coeffs,
                    int32_t* out_freqs, double* out_coeffs, int32_t* out_count, int32_t* out_status,
                    sfft_report* rep) {
  if (!plan || !freqs || !coeffs || !out_freqs || !out_coeffs || !out_count) return SFFT_EINVAL;
  if (batch < 1 || batch > plan->batch / plan->spec_slots)
    return fail(plan, SFFT_EDIM, "batch %d outside [1, %d]", batch, plan->batch / plan->spec_slots);
  int rc = ensure_ready(plan);
  if (rc) return rc;
  sfft_plan_t* P = plan;
  const size_t nf = 4 * (size_t)batch * P->k * P->d, nc = 16 * (size_t)batch * P->k;
  CUDA_TRY(P, cudaMemcpyAsync(ptr<int32_t>(P, B_IN_F), freqs, nf, cudaMemcpyHostToDevice, P->stream));
  CUDA_TRY(P, cudaMemcpyAsync(ptr<double>(P, B_IN_C), coeffs, nc, cudaMemcpyHostToDevice, P->stream));
  sfft_signal_t sig{P, batch, ptr<int32_t>(P, B_IN_F), ptr<double>(P, B_IN_C)};
  const int st = sfft_execute(P, &sig, ptr<int32_t>(P, B_OUT_F), ptr<double>(P, B_OUT_C), ptr<int32_t>(P, B_OUT_N),
                              ptr<int32_t>(P, B_OUT_S), rep);
  if (st < 0 && st != SFFT_ENOTSUP && st != SFFT_ECORRUPT) return st;
  CUDA_TRY(P, cudaMemcpyAsync(out_freqs, ptr<int32_t>(P, B_OUT_F), nf, cudaMemcpyDeviceToHost, P->stream));
  CUDA_TRY(P, cudaMemcpyAsync(out_coeffs, ptr<double>(P, B_OUT_C), nc, cudaMemcpyDeviceToHost, P->stream));
  CUDA_TRY(P, cudaMemcpyAsync(out_count, ptr<int32_t>(P, B_OUT_N), 4 * (size_t)batch, cudaMemcpyDeviceToHost, P->stream));
  if (out_status)
    CUDA_TRY(P, cudaMemcpyAsync(out_status, ptr<int32_t>(P, B_OUT_S), 4 * (size_t)batch, cudaMemcpyDeviceToHost, P->stream));
  CUDA_TRY(P, cudaStreamSynchronize(P->stream));
  return st;
}

int sfft_solve_host_batches(sfft_plan_t* plan, int32_t n_batches, int32_t batch, const int32_t* freqs,
                            const double* coeffs, int32_t* out_freqs, double* out_coeffs, int32_t* out_count,
                            int32_t* out_status, sfft_report* rep) {
  if (!plan || n_batches < 1 || !freqs || !coeffs || !out_freqs || !out_coeffs || !out_count) return SFFT_EINVAL;
  if (batch < 1 || batch > plan->batch / plan->spec_slots)
    return fail(plan, SFFT_EDIM, "batch %d outside [1, %d]", batch, plan->batch / plan->spec_slots);
  int rc = ensure_ready(plan);
  if (rc) return rc;
  sfft_plan_t* P = plan;
  const size_t nf = 4 * (size_t)batch * P->k * P->d, nc = 16 * (size_t)batch * P->k, ns = 4 * (size_t)batch;
  // the second input / output set (the first is the workspace's, shared with sfft_solve_host), 256-B aligned parts
  const size_t a_nf = align_up(nf, 256), a_nc = align_up(nc, 256), a_ns = align_up(ns, 256);
  const size_t set_bytes = 2 * a_nf + 2 * a_nc + 2 * a_ns;
  if (P->pipe_bytes < set_bytes) {
    if (P->pipe_buf) cudaFree(P->pipe_buf);
    P->pipe_buf = nullptr;
    P->pipe_bytes = 0;
    const cudaError_t e = cudaMalloc(&P->pipe_buf, set_bytes);
    if (e != cudaSuccess) return fail(P, SFFT_ENOMEM, "cudaMalloc(%zu) for the batch pipeline: %s", set_bytes,
                                      cudaGetErrorString(e));
    P->pipe_bytes = set_bytes;
  }
  for (cudaStream_t& s : P->pipe_st)
    if (!s) CUDA_TRY(P, cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  for (cudaEvent_t& e : P->pipe_ev)
    if (!e) CUDA_TRY(P, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  struct Set { int32_t* f; double* c; int32_t* of; double* oc; int32_t* on; int32_t* os; };
  char* pb = static_cast<char*>(P->pipe_buf);
  const Set sets[2] = {
      {ptr<int32_t>(P, B_IN_F), ptr<double>(P, B_IN_C), ptr<int32_t>(P, B_OUT_F), ptr<double>(P, B_OUT_C),
       ptr<int32_t>(P, B_OUT_N), ptr<int32_t>(P, B_OUT_S)},
      {reinterpret_cast<int32_t*>(pb), reinterpret_cast<double*>(pb + a_nf), reinterpret_cast<int32_t*>(pb + a_nf + a_nc),
       reinterpret_cast<double*>(pb + 2 * a_nf + a_nc), reinterpret_cast<int32_t*>(pb + 2 * a_nf + 2 * a_nc),
       reinterpret_cast<int32_t*>(pb + 2 * a_nf + 2 * a_nc + a_ns)}};
  cudaStream_t h2d = P->pipe_st[0], d2h = P->pipe_st[1];
  // H2D of batch i into set i & 1 once the solve of batch i - 2 (the set's previous user) has finished
  auto load = [&](int i) -> int {
    const Set& s = sets[i & 1];
    if (i >= 2) CUDA_TRY(P, cudaStreamWaitEvent(h2d, P->pipe_ev[2 + (i & 1)], 0));
    CUDA_TRY(P, cudaMemcpyAsync(s.f, reinterpret_cast<const char*>(freqs) + i * nf, nf, cudaMemcpyHostToDevice, h2d));
    CUDA_TRY(P, cudaMemcpyAsync(s.c, reinterpret_cast<const char*>(coeffs) + i * nc, nc, cudaMemcpyHostToDevice, h2d));
    CUDA_TRY(P, cudaEventRecord(P->pipe_ev[i & 1], h2d));
    return SFFT_OK;
  };
  if ((rc = load(0))) return rc;
  if (n_batches > 1 && (rc = load(1))) return rc;
  int result = SFFT_OK;
  for (int i = 0; i < n_batches; ++i) {
    const Set& s = sets[i & 1];
    CUDA_TRY(P, cudaStreamWaitEvent(P->stream, P->pipe_ev[i & 1], 0));              // inputs of batch i landed
    if (i >= 2) CUDA_TRY(P, cudaStreamWaitEvent(P->stream, P->pipe_ev[4 + (i & 1)], 0));  // outputs of i - 2 read out
    sfft_signal_t sig{P, batch, s.f, s.c};
    const int st = sfft_execute(P, &sig, s.of, s.oc, s.on, s.os, rep ? rep + i : nullptr);
    if (st < 0 && st != SFFT_ENOTSUP && st != SFFT_ECORRUPT) {
      cudaStreamSynchronize(h2d);
      cudaStreamSynchronize(d2h);
      return st;
    }
    if (st < 0 && result >= 0) result = st;
    else if (st > 0 && result == SFFT_OK) result = st;
    CUDA_TRY(P, cudaEventRecord(P->pipe_ev[2 + (i & 1)], P->stream));
    CUDA_TRY(P, cudaStreamWaitEvent(d2h, P->pipe_ev[2 + (i & 1)], 0));
    CUDA_TRY(P, cudaMemcpyAsync(reinterpret_cast<char*>(out_freqs) + i * nf, s.of, nf, cudaMemcpyDeviceToHost, d2h));
    CUDA_TRY(P, cudaMemcpyAsync(reinterpret_cast<char*>(out_coeffs) + i * nc, s.oc, nc, cudaMemcpyDeviceToHost, d2h));
    CUDA_TRY(P, cudaMemcpyAsync(reinterpret_cast<char*>(out_count) + i * ns, s.on, ns, cudaMemcpyDeviceToHost, d2h));
    if (out_status)
      CUDA_TRY(P, cudaMemcpyAsync(reinterpret_cast<char*>(out_status) + i * ns, s.os, ns, cudaMemcpyDeviceToHost, d2h));
    CUDA_TRY(P, cudaEventRecord(P->pipe_ev[4 + (i & 1)], d2h));
    if (i + 2 < n_batches && (rc = load(i + 2))) return rc;
  }
  CUDA_TRY(P, cudaStreamSynchronize(d2h));
  CUDA_TRY(P, cudaStreamSynchronize(P->stream));
  return result;
}

// ---------------------------------------------------------------- stage entry points
static int set_signal0_state(sfft_plan_t* P, const DevParams& D, int p, int m, int nR) {
  int32_t h[5] = {ST_RUN, nR, p, m, 0};
  const int32_t stage_slot = P->n_tslots;             // reserved table slot of the stage entry points
  CUDA_TRY(P, cudaMemcpyAsync(D.st_slot, &stage_slot, 4, cudaMemcpyHostToDevice, P->stream));
  CUDA_TRY(P, cudaMemcpyAsync(D.active, &h[4], 4, cudaMemcpyHostToDevice, P->stream));
  CUDA_TRY(P, cudaMemcpyAsync(D.st_status, &h[0], 4, cudaMemcpyHostToDevice, P->stream));
  CUDA_TRY(P, cudaMemcpyAsync(D.st_nR, &h[1], 4, cudaMemcpyHostToDevice, P->stream));
  CUDA_TRY(P, cudaMemcpyAsync(D.st_p, &h[2], 4, cudaMemcpyHostToDevice, P->stream));
  CUDA_TRY(P, cudaMemcpyAsync(D.st_m, &h[3], 4, cudaMemcpyHostToDevice, P->stream));
  CUDA_TRY(P, cudaStreamSynchronize(P->stream));
  return SFFT_OK;
}

int sfft_stage_expsum(sfft_plan_t* plan, int32_t K, const int64_t* v, const double* c, int64_t p, int32_t m,
                      double* s_out) {
  if (!plan || !v || !c || !s_out || K < 0 || K > plan->kk || m < 0 || m >= plan->r) return SFFT_EINVAL;
  if (p < 2 || p > plan->p_cap) return SFFT_ENOTSUP;
  int rc = ensure_ready(plan);
  if (rc) return rc;
  sfft_plan_t* P = plan;
  DevParams D = dev_params(P, 1);
  D.literal = 1;                 // the stage sums exactly the K given terms
  int launches = 0;
  if (K > 0)
    CUDA_TRY(P, cudaMemcpy2DAsync(D.v_all, 8 * (size_t)P->kk, v, 8 * (size_t)K, 8 * (size_t)K, P->r,
                                  cudaMemcpyDeviceToDevice, P->stream));
  LAUNCH(P, launch_line_coeffs(D, K, c, P->stream));
  rc = set_signal0_state(P, D, (int)p, m, K - P->k);
  if (rc) return rc;
  const int fi = fft_index_host(P, (int)p);
  LAUNCH(P, launch_fft_prep(D, 1, (int)P->fft[fi].smem_upto, fft_threads(P->fft[fi].M, P->fft[fi].smem_upto, P->L), P->fft[fi].M >= fft_big_m(),
                            P->stream, 0, true));
  if (P->i8_ok && i8_use_for(P, (int)p)) {
    D.i8_K = K;
    LAUNCH(P, launch_i8_prepare(D, 1, K, P->stream));
    LAUNCH(P, launch_expsum_i8(D, P->i8, (int)p, 1, 1, nullptr, 0, P->smem_optin, P->stream));
    LAUNCH(P, launch_i8_unpermute(D, (int)p, s_out, P->stream));     // discrete-log row order -> natural
  } else {
    LAUNCH(P, launch_expsum(D, expsum_for_p(P->shape, (int)p), (int)p, 1, 1, nullptr, 0, P->stream));
    CUDA_TRY(P, cudaMemcpy2DAsync(s_out, 16 * (size_t)p, D.lines, 16 * (size_t)P->p_stride, 16 * (size_t)p, P->L,
                                  cudaMemcpyDeviceToDevice, P->stream));
  }
  CUDA_TRY(P, cudaStreamSynchronize(P->stream));
  return SFFT_OK;
}

int sfft_stage_pfft(sfft_plan_t* plan, int32_t n_lines, int64_t p, double* x) {
  if (!plan || !x || n_lines < 1) return SFFT_EINVAL;
  if (p < 2 || p > plan->p_cap) return SFFT_ENOTSUP;
  int rc = ensure_ready(plan);
  if (rc) return rc;
  sfft_plan_t* P = plan;
  DevParams D = dev_params(P, 1);
  D.lines = reinterpret_cast<double2*>(x);
  D.p_stride = p;
  D.L = n_lines;
  int launches = 0;
  rc = set_signal0_state(P, D, (int)p, 0, 0);
  if (rc) return rc;
  const int fi = fft_index_host(P, (int)p);
  const int sm = (int)P->fft[fi].smem_upto, th = fft_threads(P->fft[fi].M, P->fft[fi].smem_upto, n_lines), big = P->fft[fi].M >= fft_big_m();
  LAUNCH(P, launch_fft_prep(D, 1, sm, th, big, P->stream, 0, true));
  LAUNCH(P, launch_pfft(D, 1, n_lines, sm, th, big, 1, nullptr, 0, P->stream, fft_wl_for(P->fft[fi].M)));
  CUDA_TRY(P, cudaStreamSynchronize(P->stream));
  return SFFT_OK;
}

int sfft_stage_decode(sfft_plan_t* plan, int64_t p, int32_t m, int32_t kstar, const double* F, int32_t* acc_b,
                      int64_t* acc_v, double* acc_a, int32_t* counts) {
  if (!plan || !F || !acc_b || !acc_v || !acc_a || !counts || kstar < 1 || kstar > plan->k || m < 0 || m >= plan->r)
    return SFFT_EINVAL;
  if (p < 2 || p > plan->p_cap) return SFFT_ENOTSUP;
  int rc = ensure_ready(plan);
  if (rc) return rc;
  sfft_plan_t* P = plan;
  DevParams D = dev_params(P, 1);
  D.lines = reinterpret_cast<double2*>(const_cast<double*>(F));
  D.p_stride = p;
  int launches = 0;
  rc = set_signal0_state(P, D, (int)p, m, P->k - kstar);
  if (rc) return rc;
  LAUNCH(P, launch_stage_decode(D, kstar, acc_b, acc_v, acc_a, counts, P->stream));
  CUDA_TRY(P, cudaStreamSynchronize(P->stream));
  return SFFT_OK;
}

int sfft_stage_project(sfft_plan_t* plan, const sfft_signal_t* sig, int64_t* v_out) {
  if (!plan || !sig || !v_out) return SFFT_EINVAL;
  int rc = ensure_ready(plan);
  if (rc) return rc;
  sfft_plan_t* P = plan;
  DevParams D = dev_params(P, sig->batch);
  int launches = 0;
  LAUNCH(P, launch_project(D, sig->batch, sig->freqs, sig->coeffs, P->stream));
  CUDA_TRY(P, cudaMemcpy2DAsync(v_out, 8 * (size_t)P->k, D.v_all, 8 * (size_t)P->kk, 8 * (size_t)P->k,
                                (size_t)sig->batch * P->r, cudaMemcpyDeviceToDevice, P->stream));
  CUDA_TRY(P, cudaStreamSynchronize(P->stream));
  return SFFT_OK;
}

#ifdef SFFT_FFT_PROF
SFFT_API int sfft_debug_fft_prof(unsigned long long* out, int reset) {
  return sfft::fft_prof_read(out, reset != 0) == cudaSuccess ? SFFT_OK : SFFT_ECUDA;
}
#endif

int sfft_line_shard_range(int32_t r, int32_t G, int32_t g, int32_t* lo, int32_t* hi) {
  if (!lo || !hi || r < 1 || G < 1 || G > r || g < 0 || g >= G) return SFFT_EINVAL;
  int a, b;
  line_shard_range(r, G, g, &a, &b);
  *lo = a;
  *hi = b;
  return SFFT_OK;
}

int sfft_comm_unique_id(void* out) {
  if (!out) return SFFT_EINVAL;
  const NcclApi& n = nccl_api();
  if (!n.ok) return SFFT_ENCCL;
  NcclUid id;
  if (n.get_unique_id(&id) != 0) return SFFT_ENCCL;
  memcpy(out, id.internal, sizeof id.internal);
  return SFFT_OK;
}

int sfft_comm_peer_handle(sfft_plan_t* plan, void* out) {
  if (!plan || !out) return SFFT_EINVAL;
  if (plan->line_exchange != 1) return fail(plan, SFFT_EINVAL, "plan has line_exchange = 0");
  int rc = ensure_peer_buf(plan);
  if (rc) return rc;
  cudaIpcMemHandle_t h;
  CUDA_TRY(plan, cudaIpcGetMemHandle(&h, plan->peer_buf));
  static_assert(sizeof h == 64, "cudaIpcMemHandle_t is 64 bytes");
  memcpy(out, &h, sizeof h);
  return SFFT_OK;
}

int sfft_comm_init_peers(sfft_plan_t* plan, int32_t nranks, int32_t rank, const void* handles) {
  if (!plan || !handles || nranks < 1 || rank < 0 || rank >= nranks) return SFFT_EINVAL;
  if (plan->line_exchange != 1) return fail(plan, SFFT_EINVAL, "plan has line_exchange = 0");
  if (plan->line_G != nranks || plan->line_g != rank)
    return fail(plan, SFFT_EINVAL, "plan is line shard %d of %d, peer rank %d of %d", plan->line_g, plan->line_G, rank,
                nranks);
  if (plan->peer_ready) return fail(plan, SFFT_EINVAL, "peers already initialised");
  int rc = ensure_peer_buf(plan);
  if (rc) return rc;
  plan->peer_ptr.assign(nranks, nullptr);
  plan->peer_opened.assign(nranks, false);
  for (int h = 0; h < nranks; ++h) {
    if (h == rank) {
      plan->peer_ptr[h] = plan->peer_buf;
      continue;
    }
    cudaIpcMemHandle_t ih;
    memcpy(&ih, static_cast<const char*>(handles) + 64 * (size_t)h, sizeof ih);
    void* p = nullptr;
    const cudaError_t e = cudaIpcOpenMemHandle(&p, ih, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return fail(plan, SFFT_ECUDA, "cudaIpcOpenMemHandle(rank %d): %s", h, cudaGetErrorString(e));
    plan->peer_ptr[h] = p;
    plan->peer_opened[h] = true;
  }
  plan->peer_ready = true;
  return SFFT_OK;
}

int sfft_comm_init(sfft_plan_t* plan, int32_t nranks, int32_t rank, const void* nccl_unique_id, int32_t shard_mode) {
  if (!plan || nranks < 1 || rank < 0 || rank >= nranks) return SFFT_EINVAL;
  if (shard_mode == 0) return SFFT_OK;   // signal sharding: independent solves, no communicator
  if ((shard_mode != 1 && shard_mode != 2) || !nccl_unique_id) return SFFT_EINVAL;
  if (shard_mode == 1 && (plan->line_G != nranks || plan->line_g != rank))
    return fail(plan, SFFT_EINVAL, "plan is line shard %d of %d, communicator rank %d of %d", plan->line_g,
                plan->line_G, rank, nranks);
  if (shard_mode == 2 && (!plan->spec_dist || plan->spec_G != nranks || plan->spec_rank != rank))
    return fail(plan, SFFT_EINVAL, "plan is not speculation rank %d of %d", rank, nranks);
  if (plan->nccl_comm) return fail(plan, SFFT_EINVAL, "communicator already initialised");
  const NcclApi& n = nccl_api();
  if (!n.ok) return fail(plan, SFFT_ENCCL, "libnccl.so.2 not loadable");
  CUDA_TRY(plan, cudaSetDevice(plan->device));
  NcclUid id;
  memcpy(id.internal, nccl_unique_id, sizeof id.internal);
  void* comm = nullptr;
  const int r = n.comm_init_rank(&comm, nranks, id, rank);
  if (r != 0) return fail(plan, SFFT_ENCCL, "ncclCommInitRank: %s", n.get_error_string(r));
  plan->nccl_comm = comm;
  return SFFT_OK;
}

}  // extern "C"
