/*
 * sfft_oracle.h -- TEST INFRASTRUCTURE ONLY (not the product path).
 *
 * Plain, slow, literal CPU oracle of the multidimensional phase-shift sparse FFT
 * (arXiv 1606.07407, Algorithm 2 "MultiPhaseshift").  Only
 * tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
 * --impl reference) may load this library.  It shares no code, header, table or
 * constant generator with paper_1606_07407_b200/ and never calls it.
 *
 * Every value is double / int64; no -ffast-math.  Phases are reduced exactly in
 * integers (reading R1 / SURVEY 8(c) C1): the sample point
 * t = (h/p) e_m + (1/E) e_n (reduced, possibly tilted coordinates) gives each
 * mode the phase  ((h * (v_m mod p)) mod p)/p + (v_n mod E)/E  in [0, 2).
 */
#ifndef SFFT_ORACLE_H
#define SFFT_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Solver parameters (Algorithm 2 inputs "f, c, k, N, d, d1, d2, eps", PAPER.md:377,
 * plus the readings of SURVEY 8(c) C3, C14, C15, C17-C19). */
typedef struct {
  int32_t d;
  int32_t k;
  int64_t N;
  int32_t r;                 /* number of blocks of the partition */
  const int32_t* blocks;     /* [r] d_1..d_r, sum = d */
  int32_t n_tilts;
  const int64_t* tilts;      /* [n_tilts][5]: axis0, axis1, base, height, hypo (Eq. (25)) */
  int64_t E;                 /* 1/eps; 0 -> 2 * B * max(base+height) */
  int32_t c;                 /* prime factor (5) */
  double tol;                /* collision tolerance tau, default 1e-6 */
  double bin_floor_rel;      /* |F_0[b]| < bin_floor_rel * p -> empty bin (C18), 1e-8 */
  double prune_floor;        /* prune |a| < prune_floor (C17), 1e-8 */
  double round_tol;          /* reject |x - round(x)| > round_tol (C14), 0.01 */
  int32_t max_iter;          /* 1000 */
  int32_t stall_limit;       /* 0 -> max(2r, 16) (C19) */
  int32_t extra_checks;      /* bit0 range check, bit1 bin consistency (C15) */
  int32_t n_primes;          /* explicit prime schedule p_i = primes[(i-1) mod n] */
  const int64_t* primes;     /* NULL -> i-th prime >= max(2, c k*) (Alg. 2 l.8) */
  int32_t n_fallback;        /* stall fallback (readings R23 / R24): up to ORACLE_MAX_FALLBACK levels;
                                1-4 tilt fixed axis pairs with the Pythagorean triples (3,4,5), (5,12,13),
                                (8,15,17), (7,24,25); 5.. tilt the pairs of a seeded random order of the axes */
  int32_t n_spec;            /* multi-prime speculation (reading R26): 0 / 1 = Alg. 2 as
                                written; G > 1: iteration i runs the G primes of counters (i-1) G + 1 .. i G against
                                the same residual and merges their accepted bins in prime order, a key already
                                updated by an earlier prime of the iteration being skipped */
} oracle_params;

#define ORACLE_MAX_FALLBACK 67

/* Tilts of fallback level lvl in 1..ORACLE_MAX_FALLBACK (readings R23 / R24).  Levels 1-4: triple lvl-1 on the
 * disjoint reduced-axis pairs (q, q + s): level 1 (0,1),(2,3),...; level 2 (1,2),(3,4),... (r >= 3); level 3
 * stride 2 (0,2),(1,3),(4,6),...; level 4 stride 3.  Levels 5.. ("randomizing the order of the dimensions",
 * P:293, reading R24): round j = lvl - 5 of the circle-method round robin over the seeded axis order
 * pi = oracle_axis_order(r, 1) -- n = r rounded up to even slots, slot 0 fixed, slots 1..n-1 rotated by j, pairs
 * (a[i], a[n-1-i]) for i < n/2 mapped through pi (a pair with the padding slot is skipped) -- with triple j mod 4:
 * the n - 1 rounds tilt every pair of axes exactly once.  Writes out [r/2][5]; returns the number of tilts (0 when
 * r < 2 or the level is past the last round). */
int32_t oracle_fallback_tilts(int32_t r, int32_t lvl, int64_t* out);
/* The seeded axis order: Fisher-Yates from i = r-1 down to 1, j = z_i mod (i + 1), with z_i = the splitmix64
 * finaliser of the counter c_i = seed * 0x9E3779B97F4A7C15 + (r - i) * 0xD1B54A32D192ED03 (mod 2^64). */
void oracle_axis_order(int32_t r, int32_t seed, int32_t* pi);

enum { ORACLE_OK = 0, ORACLE_PARTIAL = 1, ORACLE_EINVAL = -1, ORACLE_EPRECISION = -2,
       ORACLE_ECORRUPT = -4, ORACLE_ENOMEM = -6 };

/* ---- index maps (Eqs. (19), (27), (31), (35), (36)) ---- */
int oracle_unwrap_freq(int32_t d, int64_t N, int32_t r, const int32_t* blocks,
                       const int32_t* w /*[d]*/, int64_t* u /*[r]*/);
int oracle_wrap_freq(int32_t d, int64_t N, int32_t r, const int32_t* blocks,
                     const int64_t* u /*[r]*/, int32_t* w /*[d]*/);
void oracle_block_range(int64_t N, int32_t dq, int64_t* lo, int64_t* hi);
void oracle_tilt_freq(int64_t base, int64_t height, int64_t w1, int64_t w2, int64_t* out /*[2]*/);
int oracle_untilt_freq(int64_t base, int64_t height, int64_t hypo, int64_t v1, int64_t v2,
                       int64_t* out /*[2]*/);
/* time embedding Eq. (36): t[off_q + s] = N^s * t_red[q] */
void oracle_unwrap_time(int32_t d, int64_t N, int32_t r, const int32_t* blocks,
                        const double* t_red /*[r]*/, double* t /*[d]*/);

/* ---- primes (Alg. 2 l.8) ---- */
int64_t oracle_ith_prime_at_least(int64_t x, int32_t i);

/* ---- plan-level derived quantities ---- */
int oracle_prepare(const oracle_params* P, int64_t* E_out, int64_t* lo /*[r]*/, int64_t* hi /*[r]*/);
/* v_j = T * unwrap(w_j): reduced (tilted) frequencies of k modes, v [k][r] */
int oracle_project(const oracle_params* P, const int32_t* w /*[k][d]*/, int32_t k, int64_t* v /*[k][r]*/);

/* ---- evaluation of f at a point (Eq. (9)) ---- */
/* f(t) = sum_j a_j exp(2 pi i w_j . t) at a real point t in R^d, plain double arithmetic
 * (used only to pin the exact-phase evaluation on tiny inputs). */
void oracle_eval_point(int32_t d, int32_t K, const int32_t* w /*[K][d]*/, const double* a /*[K][2]*/,
                       const double* t /*[d]*/, double* out /*[2]*/);
/* One sample line (Eq. (41), Alg. 2 l.13-14): s[h] = sum_j c_j exp(2 pi i v_j . t_h),
 * t_h = (h/p) e_m + (1/E) e_n  (n < 0: unshifted).  Exact integer phase reduction. */
void oracle_sample_line(int32_t K, int32_t r, const int64_t* v /*[K][r]*/, const double* c /*[K][2]*/,
                        int64_t p, int32_t m, int32_t n, int64_t E, double* s /*[p][2]*/);

/* ---- DFT (Eq. (3)): F[b] = sum_h s[h] exp(-2 pi i h b / p), direct O(p^2) ---- */
void oracle_dft(int64_t p, const double* s /*[p][2]*/, double* F /*[p][2]*/);

/* ---- select + test + decode of one iteration (Alg. 2 l.18-32) ----
 * F: [(r+1)][p][2], line 0 unshifted, line 1+n shifted along reduced axis n.
 * Writes accepted bins in ascending b: acc_b [<=kstar], acc_v [<=kstar][r], acc_a [<=kstar][2].
 * Returns the number of accepted bins; *n_cand receives the number of examined bins. */
int32_t oracle_decode(const oracle_params* P, int64_t E, const int64_t* lo, const int64_t* hi,
                      int64_t p, int32_t m, int32_t kstar, const double* F,
                      int32_t* n_cand, int32_t* acc_b, int64_t* acc_v, double* acc_a);
/* the same, *n_nonempty (nullable) receiving the number of bins above the floor BEFORE the k* cap */
int32_t oracle_decode_ex(const oracle_params* P, int64_t E, const int64_t* lo, const int64_t* hi,
                         int64_t p, int32_t m, int32_t kstar, const double* F,
                         int32_t* n_cand, int32_t* n_nonempty, int32_t* acc_b, int64_t* acc_v, double* acc_a);

/* ---- the whole of Algorithm 2 for one signal ----
 * out_w [k][d] int32 (canonical lexicographic order), out_a [k][2], out_count.
 * trace [trace_cap][ORACLE_TRACE_COLS] per iteration = (i, p, m, n_candidates (after the k* cap),
 * n_accepted, n_nonempty (bins above the floor before the cap), n_accumulated (accepted keys already in R,
 * l.30 R[v] += a), n_pruned (entries removed by l.33)). */
#define ORACLE_TRACE_COLS 8
int oracle_solve(const oracle_params* P, const int32_t* w /*[k][d]*/, const double* a /*[k][2]*/,
                 int32_t* out_w, double* out_a, int32_t* out_count, int64_t* out_samples,
                 int32_t* out_iters, int32_t trace_cap, int64_t* trace);

/* The same, ns (nullable) [2] = wall ns of the solve and ns spent sampling (the "main part" of P:461-463
 * is the difference). */
int oracle_solve_timed(const oracle_params* P, const int32_t* w, const double* a, int32_t* out_w,
                       double* out_a, int32_t* out_count, int64_t* out_samples, int32_t* out_iters,
                       int32_t trace_cap, int64_t* trace, int64_t* ns);

/* Debugging aid: the registry (reduced keys raw_v [<=k][r], raw_a [<=k][2], *raw_n entries) at the end of the
 * loop, before the wrap; returns the solve status. */
int oracle_solve_raw(const oracle_params* P, const int32_t* w, const double* a, int64_t* raw_v, double* raw_a,
                     int32_t* raw_n);

/* Independent signals spread over n_threads host threads (one solve per thread at a time).
 * out_ns (nullable) [batch][2]: per-signal oracle_solve_timed times. */
int oracle_solve_batch(const oracle_params* P, int32_t batch, const int32_t* w, const double* a,
                       int32_t* out_w, double* out_a, int32_t* out_count, int64_t* out_samples,
                       int32_t* out_iters, int32_t* out_status, int32_t n_threads, int64_t* out_ns);

#ifdef __cplusplus
}
#endif
#endif
