/*
 * sfft.h -- C ABI of the B200-native multidimensional phase-shift sparse FFT
 * (arXiv 1606.07407, Algorithm 2 "MultiPhaseshift").
 *
 * Library: paper_1606_07407_b200/libsfft.so (CUDA, sm_100a).  Every step of the
 * hot path runs in hand-written kernels; there is no CPU fallback.
 *
 * Conventions
 *   - "device" pointers are CUDA device memory on the plan's device; "host"
 *     pointers are ordinary (preferably pinned) host memory.
 *   - complex numbers are interleaved (re, im) doubles.
 *   - All calls are asynchronous on the plan's stream unless stated; they return
 *     an sfft_status.  Nothing is thrown across the ABI.  On error
 *     sfft_last_error(plan) holds a one-line message.
 *   - A plan is bound to one device and one stream; it is not thread-safe.
 */
#ifndef SFFT_H
#define SFFT_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define SFFT_API __attribute__((visibility("default")))
#else
#define SFFT_API
#endif

typedef enum {
  SFFT_OK = 0,
  SFFT_PARTIAL = 1,        /* max_iter or stall reached; outputs hold the current registry */
  SFFT_EINVAL = -1,        /* invalid argument (d<1, N odd or <2, sum of blocks != d, k<1, bad tilt, 1/eps not an integer, ...) */
  SFFT_EPRECISION = -2,    /* N^{d_q} > 2^40 or E > 2^42 (reading R1) */
  SFFT_EDIM = -3,          /* signal batch larger than the plan's batch */
  SFFT_ECORRUPT = -4,      /* untilt not integral / wrapped frequency outside the box (Alg. 3 l.39) */
  SFFT_ECUDA = -5,
  SFFT_ENOMEM = -6,
  SFFT_ENCCL = -7,
  SFFT_ENOTSUP = -8        /* prime larger than the FFT size table supports; or (sfft_plan) more than ~8000 slots
                              (batch x spec_primes, or table_cache_slots) for the slot assignment's hash map */
} sfft_status;

/* Eq. (25)/(27) tilt of the reduced-axis pair (axis0, axis1): sin = height/hypo, cos = base/hypo.
 * Frequencies on the pair map to (base*u0 - height*u1, height*u0 + base*u1). */
typedef struct {
  int32_t axis0, axis1;
  int64_t base, height, hypo;
} sfft_tilt;

/* Options; pass NULL to sfft_plan for the defaults in brackets. */
typedef struct {
  int32_t n_blocks;           /* partition d = d_1 + ... + d_r; 0 -> uniform largest d_1 | d with N^{d_1} <= 2^40 */
  const int32_t* block_dims;  /* host [n_blocks] */
  int32_t c;                  /* prime factor c of Alg. 2 l.8 [5, P:422] */
  double tol;                 /* collision tolerance tau [1e-6] */
  double bin_floor_rel;       /* empty-bin floor relative to p [1e-8] */
  double prune_floor;         /* registry prune floor [1e-8] (Alg. 2 l.33) */
  double round_tol;           /* max |x - round(x)| of a decoded coordinate [0.01] */
  int32_t max_iter;           /* [1000] */
  int32_t stall_limit;        /* [max(2r, 16)] */
  int32_t batch;              /* max signals per execute [1] */
  int32_t extra_checks;       /* bit0 range check, bit1 bin consistency [3] */
  void* stream;               /* cudaStream_t [legacy default stream] */
  int32_t profile;            /* 1: time every kernel class with CUDA events on the stream [0] */
  int32_t literal_residual;   /* 1: sample g (registry) on every line like f, K = k + |R| terms (Alg. 2 l.13-14
                                 verbatim); 0: sample f only and subtract g's bins p*sum c_e directly (Eq. (3)),
                                 same result up to rounding, O(|R| L) instead of O(p |R| L) [0] */
  int32_t expsum_path;        /* exp-sum arithmetic: 0 auto, 1 FP64 (DMMA / DFMA), 2 exact int8-limb products on
                                 the tcgen05 tensor cores combined in FP64 (needs
                                 literal_residual = 0 and E <= 2^36) [0: int8 limbs when available] */
  int32_t fallback_tilts;     /* stall fallback (Algorithm 3; readings R23 / R24): after
                                 stall_limit zero-accept iterations switch to the next of up to 67 tilt levels --
                                 levels 1-4: Pythagorean triples (3,4,5), (5,12,13), (8,15,17), (7,24,25) on
                                 fixed disjoint reduced-axis pairs; levels 5..: the rounds of a round robin over a
                                 seeded order of the axes (every pair tilted once after r - 1 rounds) -- keeping the
                                 modes found (mapped exactly); 0 = stop with PARTIAL; values past the last
                                 non-empty level are clamped [0] */
  int32_t line_shards;        /* line sharding: 0 = this plan holds every line [0]; G >= 1 = the
                                 plan is shard line_rank of G: it computes line 0 and the shifted lines of reduced
                                 axes [lo, hi) (contiguous, sizes differ by at most one, shard 0 the largest), and
                                 its decode exchanges per-candidate records with the other shards every iteration
                                 (sfft_comm_init, or sfft_execute_group on one device).  1 <= G <= r. */
  int32_t line_rank;          /* shard index of this plan, 0 <= line_rank < line_shards [0] */
  int32_t table_cache_slots;  /* per-prime table cache capacity (W_p roots, Bluestein chirp and kernel spectrum,
                                 int8 root limbs: ~1 MB each, they depend on p only and are kept across iterations
                                 and executes, least recently used evicted); 0 -> max(batch + 16, 512); n > 0 ->
                                 max(batch + 16, n) (batch + 16 is the minimum: every live prime has a slot) [0] */
  int32_t line_exchange;      /* how line shards exchange their per-candidate records every iteration: 0 = an
                                 all-gather after the FFT (ncclAllGather through sfft_comm_init, device copies in
                                 sfft_execute_group); 1 = fused into the FFT epilogue: every record word is stored
                                 straight into the receive buffer of every shard (peer memory over NVLink: CUDA IPC
                                 mappings from sfft_comm_peer_handle / sfft_comm_init_peers, plain pointers in
                                 sfft_execute_group) and per-(shard, line, signal) stamps released at system scope
                                 tell the commit that a shard's lines are in -- no separate collective.  At most 8
                                 shards [0] */
  int32_t spec_primes;        /* multi-prime speculation (reading R26): G primes per
                                 iteration, the prime counters (i-1) G + 1 .. i G of Alg. 2 l.8, all sampled
                                 against the same registry and merged in prime order, a key that an earlier prime of
                                 the iteration updated being skipped.  Fewer, wider iterations (single-signal
                                 latency); noiseless signals are recovered exactly, the trace differs from Alg. 2.
                                 Each signal occupies G plan slots (workspace ~G x).  0 / 1 = Alg. 2 as written;
                                 at most 16; not with line shards, fused commit or literal_residual [0] */
  int32_t spec_distributed;   /* with spec_primes = G > 1: 1 = the G primes on G ranks (GPUs), this plan being rank
                                 spec_rank with one slot per signal; every iteration the ranks all-gather their
                                 records (sfft_comm_init shard_mode 2, or sfft_execute_group on one device) and
                                 apply the same merge, so their registries stay identical [0] */
  int32_t spec_rank;          /* 0 <= spec_rank < spec_primes when spec_distributed [0] */
} sfft_options;

/* Per-execute report (host struct). Aggregates over the batch. */
typedef struct {
  int64_t samples_used;        /* sum over signals of (r+1)*p per iteration (f evaluations) */
  int64_t cmacs;               /* complex multiply-adds done by the exp-sum kernel */
  int32_t iterations;          /* iterations of the batch loop */
  int32_t n_ok, n_partial, n_error;
  int32_t status;              /* worst status over the batch */
  int32_t n_iter_logged;
  int64_t primes[64];          /* prime of signal 0 per iteration */
  int32_t accepted[64];        /* bins accepted for signal 0 per iteration */
  int32_t kernel_launches;     /* kernels launched by this execute */
  /* filled when sfft_options.profile = 1: device time per kernel class (CUDA events on the stream) */
  int32_t n_expsum;            /* exp-sum launches */
  float ms_expsum, ms_fft, ms_decode, ms_other;
  /* int8-limb tensor-core exp-sum (sfft_options.expsum_path): limbs S (0 = FP64 path only), launches, their
     complex MACs (sum over signals of L p K) and, when profiling, their device time */
  int32_t i8_limbs, n_expsum_i8;
  int64_t cmacs_i8;
  float ms_expsum_i8;
  int32_t fallback_used;       /* signals that switched to a tilt level of the stall fallback (R23) */
  float ms_total;              /* when profiling: device time of the whole execute (CUDA events) */
  double fft_plogp;            /* sum over signals and iterations of L p log2(p): the prime-length DFTs' size,
                                  5 fft_plogp = their algorithmic flops (radix-2 convention) */
  double fft_mlogm;            /* the same for the Bluestein sizes M run: 2 x 5 fft_mlogm ~ the executed FFT flops */
  int32_t n_fused_sample;      /* iterations whose sampling ran inside the FFT CTAs (no exp-sum launch; its time is
                                  in ms_fft) */
} sfft_report;

typedef struct sfft_plan_s sfft_plan_t;
typedef struct sfft_signal_s sfft_signal_t;

/*
 * sfft_plan -- validate the problem and choose partition, E, prime table, FFT sizes
 * and tile shapes (Eqs. (35)-(36) P:321-331).
 *   d, N, k      dimension, per-axis bandwidth (omega in [-N/2, N/2)^d, N even >= 2), sparsity
 *   primes       host [n_primes] explicit prime schedule p_i = primes[(i-1) mod n_primes], or NULL for
 *                the paper's rule p_i = i-th prime >= max(2, c k*) (Alg. 2 l.8)
 *   tilts        host [n_tilts] static tilts on disjoint reduced-axis pairs (Eq. (27)), or NULL
 *   eps          shift; 0 -> 1/(2 B max(base+height)) with B = max_q N^{d_q}; else 1/eps must be an integer
 *   opt          host, nullable
 *   out          receives the plan.  The plan needs workspace: either call sfft_plan_set_workspace
 *                with caller-owned device memory of sfft_plan_workspace_size() bytes, or the first
 *                execute allocates it with cudaMalloc (owned by the plan).
 */
SFFT_API int sfft_plan(int32_t d, int64_t N, int32_t k, const int64_t* primes, int32_t n_primes,
              const sfft_tilt* tilts, int32_t n_tilts, double eps, const sfft_options* opt,
              sfft_plan_t** out);
SFFT_API int sfft_plan_workspace_size(const sfft_plan_t* plan, size_t* bytes);
/* dptr: device memory of >= workspace_size bytes, 256-byte aligned, owned by the caller, must
 * outlive the plan. */
SFFT_API int sfft_plan_set_workspace(sfft_plan_t* plan, void* dptr, size_t bytes);
/* Query plan-derived values (host): E, r, number of lines L this plan computes (r+1, or 1 + its shard's
 * axes when line-sharded), p_max supported, tile shape. */
SFFT_API int sfft_plan_info(const sfft_plan_t* plan, int64_t* E, int32_t* r, int32_t* L, int64_t* p_max,
                   int32_t* tile_n);
SFFT_API void sfft_plan_destroy(sfft_plan_t* plan);

/*
 * sfft_signal_expsum -- the exponential-sum signal f(t) = sum_j a_j e^{2 pi i omega_j . t}
 * (Eq. (9)) of `batch` independent signals with k modes each.
 *   freqs   device int32 [batch][k][d]
 *   coeffs  device double [batch][k][2]
 * The handle references (does not copy) the arrays: they must stay valid until the last
 * sfft_execute using it has completed on the stream.  The product path reads them only to
 * evaluate f at sample points (SURVEY 8(a) leak rule).
 */
SFFT_API int sfft_signal_expsum(sfft_plan_t* plan, int32_t batch, const int32_t* freqs, const double* coeffs,
                       sfft_signal_t** out);
SFFT_API void sfft_signal_destroy(sfft_signal_t* sig);

/*
 * sfft_execute -- run Algorithm 2 to completion on every signal of the batch.
 *   out_freqs   device int32 [batch][k][d]  recovered frequency vectors, canonical (lexicographic) order
 *   out_coeffs  device double [batch][k][2]
 *   out_count   device int32 [batch]        number of recovered modes (<= k)
 *   out_status  device int32 [batch] or NULL  per-signal sfft_status
 *   rep         host, nullable
 * Returns SFFT_OK when every signal recovered k modes, SFFT_PARTIAL if some stalled / hit
 * max_iter (outputs hold their registries), or an error.  Synchronises the plan's stream once
 * per iteration (a 16-byte control read).
 */
SFFT_API int sfft_execute(sfft_plan_t* plan, const sfft_signal_t* sig, int32_t* out_freqs, double* out_coeffs,
                 int32_t* out_count, int32_t* out_status, sfft_report* rep);

/*
 * sfft_solve_host -- end-to-end call with HOST buffers: copies the signal to the device, runs
 * sfft_execute, copies the result back; returns after the result is on the host.
 *   freqs host int32 [batch][k][d], coeffs host double [batch][k][2] (pinned for full speed);
 *   out_* host, same shapes as sfft_execute.
 */
SFFT_API int sfft_solve_host(sfft_plan_t* plan, int32_t batch, const int32_t* freqs, const double* coeffs,
                    int32_t* out_freqs, double* out_coeffs, int32_t* out_count, int32_t* out_status,
                    sfft_report* rep);

/*
 * sfft_solve_host_batches -- n_batches consecutive batches of `batch` signals each, HOST buffers, with the
 * transfers overlapped with the solves: the H2D of batch i + 1 and the D2H of batch i - 1 run on two
 * library-owned non-blocking streams while batch i is solved on the plan's stream (two device input / output
 * sets; the second one is allocated on the first call, 2 * batch * k * (4 d + 16) + 16 * batch bytes).
 * Each batch is an independent sfft_execute (the same results as sfft_solve_host batch by batch).
 *   freqs  host int32 [n_batches][batch][k][d], coeffs host double [n_batches][batch][k][2]
 *   out_*  host [n_batches][...] with the per-batch shapes of sfft_execute; out_status nullable
 *   rep    host, nullable, [n_batches] reports
 * Pinned (page-locked) host buffers are required for the overlap (pageable ones work, serialised).  Returns after
 * the last result is on the host: a hard error of any batch at once, else the first SFFT_ENOTSUP /
 * SFFT_ECORRUPT, else SFFT_PARTIAL if any batch returned it, else SFFT_OK.
 */
SFFT_API int sfft_solve_host_batches(sfft_plan_t* plan, int32_t n_batches, int32_t batch, const int32_t* freqs,
                                     const double* coeffs, int32_t* out_freqs, double* out_coeffs, int32_t* out_count,
                                     int32_t* out_status, sfft_report* rep);

/* ---- stage entry points (teacher-forced parity of single steps; same kernels as execute) ---- */

/*
 * sfft_stage_expsum -- a3: lines of one iteration of ONE signal.
 *   v      device int64 [r][K] reduced (tilted) frequencies of the K terms (column j = term j)
 *   c      device double [K][2] term coefficients (signal a_j, registry -a_e)
 *   p, m   prime and projection axis
 *   s_out  device double [L][p][2]: line 0 unshifted, line 1+n shifted by 1/E along reduced axis n:
 *          s_n[h] = sum_j c_j exp(2 pi i v_j . ((h/p) e_m + (1/E) e_n))   (Eq. (41), exact phase)
 */
SFFT_API int sfft_stage_expsum(sfft_plan_t* plan, int32_t K, const int64_t* v, const double* c, int64_t p,
                      int32_t m, double* s_out);
/*
 * sfft_stage_pfft -- a4: n_lines unnormalised forward DFTs of length p (Eq. (3)), in place.
 *   x      device double [n_lines][p][2]
 */
SFFT_API int sfft_stage_pfft(sfft_plan_t* plan, int32_t n_lines, int64_t p, double* x);
/*
 * sfft_stage_decode -- a5+a6: select, collision-test and decode the bins of one iteration.
 *   F      device double [L][p][2]
 *   outputs (device): acc_b int32 [kstar], acc_v int64 [r][kstar], acc_a double [kstar][2],
 *   counts int32 [2] = (n_candidates, n_accepted).  Accepted bins in ascending b.
 */
SFFT_API int sfft_stage_decode(sfft_plan_t* plan, int64_t p, int32_t m, int32_t kstar, const double* F,
                      int32_t* acc_b, int64_t* acc_v, double* acc_a, int32_t* counts);
/* a1 on its own: v [batch][r][k] (device int64) of a signal (unwrap Eq. (35) + tilt Eq. (27)). */
SFFT_API int sfft_stage_project(sfft_plan_t* plan, const sfft_signal_t* sig, int64_t* v_out);

/*
 * Multi-GPU.  Signal sharding (shard_mode 0) runs independent solves per rank and needs
 * no communicator (sfft_comm_init returns SFFT_OK and does nothing).  Line sharding (shard_mode 1):
 * the plan must have been created with line_shards = nranks, line_rank = rank; every iteration each
 * rank computes line 0 (redundantly, bitwise identical on all ranks) and its own shifted lines, tests
 * and decodes the candidates of line 0 on them, all-gathers the per-candidate records (pass flag over
 * its lines, decoded coordinates of its axes: batch * ((k+1)/2 + (Lmax-1) k) int64 words per rank) with
 * ncclAllGather on the plan's stream, and applies the identical registry update (Alg. 2 l.20-33).
 * Distributed multi-prime speculation (shard_mode 2, reading R26): the plan must have been created
 * with spec_primes = nranks, spec_distributed = 1, spec_rank = rank; every iteration each rank samples, transforms
 * and decodes its own prime of the iteration, the ranks all-gather their records (flags, coordinates and a tail
 * of candidate count, p, m, candidate bins and F_0 there: batch * ((k+1)/2 + r k + 2 + (k+1)/2 + 2k) int64 words
 * per rank) and every rank merges the nranks sets in rank (prime) order into its identical registry.
 *   nccl_unique_id  host, 128 bytes from sfft_comm_unique_id on rank 0, broadcast by the caller
 * NCCL is loaded at run time (dlopen "libnccl.so.2": the copy already in the process, e.g. torch's,
 * else the system one); without it the call fails with SFFT_ENCCL.  All ranks must call it together
 * (ncclCommInitRank is collective).  The communicator is destroyed with the plan.
 */
/*
 * Fused record exchange (sfft_options.line_exchange = 1) across processes / GPUs of one node:
 *   sfft_comm_peer_handle -- allocates this shard's exchange buffer (receive records [line_shards][batch][words]
 *                            + stamps; cudaMalloc, owned by the plan) and writes its cudaIpcMemHandle_t (64 bytes)
 *                            to out (host)
 *   sfft_comm_init_peers  -- collective over the line shards: handles = host [nranks][64] bytes of every rank's
 *                            handle (all-gathered by the caller, e.g. torch.distributed); opens the peers' buffers
 *                            (cudaIpcOpenMemHandle) so that this plan's FFT epilogue stores into them.  nranks =
 *                            line_shards, rank = line_rank; one rank (nranks = 1) uses its own buffer.
 */
SFFT_API int sfft_comm_peer_handle(sfft_plan_t* plan, void* out);
SFFT_API int sfft_comm_init_peers(sfft_plan_t* plan, int32_t nranks, int32_t rank, const void* handles);
SFFT_API int sfft_comm_init(sfft_plan_t* plan, int32_t nranks, int32_t rank, const void* nccl_unique_id,
                   int32_t shard_mode);
/* Reduced axes [lo, hi) of line shard g of G over r axes (host, no device needed): contiguous, sizes
 * differ by at most one, shard 0 the largest.  The shard computes line 0 and lines 1+lo .. hi. */
SFFT_API int sfft_line_shard_range(int32_t r, int32_t G, int32_t g, int32_t* lo, int32_t* hi);
/* 128-byte NCCL unique id (ncclGetUniqueId) into host memory `out` (rank 0 of a line-sharded job). */
SFFT_API int sfft_comm_unique_id(void* out);
/*
 * sfft_execute_group -- the line-sharded solve of plans[0..n_plans) (line_shards = n_plans, line_rank g
 * = plans[g]) on ONE device: the shards' phases run one after another on plans[0]'s stream and the
 * record all-gather is a device copy into every shard's receive buffer.  Same kernels and records as the
 * multi-GPU path; used to prove the sharded protocol against the unsharded path on one GPU.  Every plan
 * needs a signal of the same arrays (sfft_signal_expsum on each plan).  Outputs are plan 0's; the call
 * fails with SFFT_ECORRUPT if the shards' registries are not bitwise identical at the end.
 */
SFFT_API int sfft_execute_group(sfft_plan_t* const* plans, const sfft_signal_t* const* sigs, int32_t n_plans,
                       int32_t* out_freqs, double* out_coeffs, int32_t* out_count, int32_t* out_status,
                       sfft_report* rep);

SFFT_API const char* sfft_strerror(int status);
SFFT_API const char* sfft_last_error(const sfft_plan_t* plan);
/* Library build identification (e.g. "sfft sm_100a <git>"). */
SFFT_API const char* sfft_version(void);

#ifdef __cplusplus
}
#endif
#endif
