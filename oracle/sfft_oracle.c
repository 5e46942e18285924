/*
 * sfft_oracle.c -- TEST INFRASTRUCTURE ONLY (not the product path).
 *
 * A plain, slow, literal CPU implementation of Algorithm 2 ("MultiPhaseshift",
 * PAPER.md:369-417) of arXiv 1606.07407, with the readings listed in DESIGN.md
 * (SURVEY.md 8(c) C1-C24).  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it.  It shares no code with the
 * CUDA library and does not know it exists.
 *
 * Scalar double / int64 arithmetic, direct O(p^2) DFT, linear-search registry.
 * Compiled with -O2 and WITHOUT -ffast-math.
 */
#define _POSIX_C_SOURCE 200809L
#include "sfft_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

/* ------------------------------------------------------------------------ */
/* small helpers                                                            */
/* ------------------------------------------------------------------------ */

/* non-negative residue x mod m, m > 0 */
static int64_t mod_pos(int64_t x, int64_t m) {
  int64_t q = x % m;
  return q < 0 ? q + m : q;
}

static int64_t ipow(int64_t b, int32_t e) {
  int64_t r = 1;
  for (int32_t i = 0; i < e; ++i) r *= b;
  return r;
}

static int64_t gcd64(int64_t a, int64_t b) {
  if (a < 0) a = -a;
  if (b < 0) b = -b;
  while (b) { int64_t t = a % b; a = b; b = t; }
  return a;
}

/* ------------------------------------------------------------------------ */
/* index maps                                                               */
/* ------------------------------------------------------------------------ */

/* Eq. (35): u_q = sum_{s=0}^{d_q-1} w[off_q + s] N^s  (powers 0..d_q-1, reading C9) */
int oracle_unwrap_freq(int32_t d, int64_t N, int32_t r, const int32_t* blocks,
                       const int32_t* w, int64_t* u) {
  int32_t off = 0;
  for (int32_t q = 0; q < r; ++q) {
    int64_t acc = 0, pw = 1;
    for (int32_t s = 0; s < blocks[q]; ++s) {
      int64_t x = w[off + s];
      if (x < -N / 2 || x >= N / 2) return ORACLE_EINVAL;
      acc += x * pw;
      pw *= N;
    }
    u[q] = acc;
    off += blocks[q];
  }
  return off == d ? ORACLE_OK : ORACLE_EINVAL;
}

/* image interval of one block: [-(N/2)(N^dq-1)/(N-1), (N/2-1)(N^dq-1)/(N-1)] */
void oracle_block_range(int64_t N, int32_t dq, int64_t* lo, int64_t* hi) {
  int64_t geo = 0, pw = 1;                    /* sum_{s<dq} N^s */
  for (int32_t s = 0; s < dq; ++s) { geo += pw; pw *= N; }
  *lo = -(N / 2) * geo;
  *hi = (N / 2 - 1) * geo;
}

/* inverse of Eq. (35) by balanced digits: digit = ((u + N/2) mod N) - N/2; u <- (u - digit)/N */
int oracle_wrap_freq(int32_t d, int64_t N, int32_t r, const int32_t* blocks,
                     const int64_t* u, int32_t* w) {
  int32_t off = 0;
  for (int32_t q = 0; q < r; ++q) {
    int64_t lo, hi;
    oracle_block_range(N, blocks[q], &lo, &hi);
    if (u[q] < lo || u[q] > hi) return ORACLE_EINVAL;
    int64_t x = u[q];
    for (int32_t s = 0; s < blocks[q]; ++s) {
      int64_t digit = mod_pos(x + N / 2, N) - N / 2;
      w[off + s] = (int32_t)digit;
      x = (x - digit) / N;
    }
    if (x != 0) return ORACLE_EINVAL;
    off += blocks[q];
  }
  return off == d ? ORACLE_OK : ORACLE_EINVAL;
}

/* Eq. (27): (c cos w1 - c sin w2, c sin w1 + c cos w2) with c cos = base, c sin = height */
void oracle_tilt_freq(int64_t base, int64_t height, int64_t w1, int64_t w2, int64_t* out) {
  out[0] = base * w1 - height * w2;
  out[1] = height * w1 + base * w2;
}

/* Alg. 3 l.38-39 with the scale of Eq. (27) removed (reading C20): divide by hypo^2 */
int oracle_untilt_freq(int64_t base, int64_t height, int64_t hypo, int64_t v1, int64_t v2,
                       int64_t* out) {
  int64_t c2 = hypo * hypo;
  int64_t x1 = base * v1 + height * v2;
  int64_t x2 = -height * v1 + base * v2;
  if (x1 % c2 != 0 || x2 % c2 != 0) return ORACLE_ECORRUPT;
  out[0] = x1 / c2;
  out[1] = x2 / c2;
  return ORACLE_OK;
}

/* Eq. (36): t_l = N^{R(l-1,d_q)} t~_{Q}, 0-based: t[off_q + s] = N^s t_red[q] */
void oracle_unwrap_time(int32_t d, int64_t N, int32_t r, const int32_t* blocks,
                        const double* t_red, double* t) {
  int32_t off = 0;
  (void)d;
  for (int32_t q = 0; q < r; ++q) {
    double pw = 1.0;
    for (int32_t s = 0; s < blocks[q]; ++s) {
      t[off + s] = pw * t_red[q];
      pw *= (double)N;
    }
    off += blocks[q];
  }
}

/* ------------------------------------------------------------------------ */
/* primes (Alg. 2 l.8: "p <- i-th prime number >= c k*")                     */
/* ------------------------------------------------------------------------ */

static int is_prime(int64_t x) {
  if (x < 2) return 0;
  if (x < 4) return 1;
  if (x % 2 == 0) return 0;
  for (int64_t f = 3; f * f <= x; f += 2)
    if (x % f == 0) return 0;
  return 1;
}

int64_t oracle_ith_prime_at_least(int64_t x, int32_t i) {
  int64_t c = x < 2 ? 2 : x;
  int32_t found = 0;
  for (;; ++c) {
    if (is_prime(c)) {
      ++found;
      if (found == i) return c;
    }
  }
}

/* ------------------------------------------------------------------------ */
/* plan-level quantities: E and the decodable image interval of every axis    */
/* ------------------------------------------------------------------------ */

static int tilt_of_axis(const oracle_params* P, int32_t q, int32_t* which, int32_t* slot) {
  for (int32_t t = 0; t < P->n_tilts; ++t) {
    const int64_t* T = P->tilts + 5 * t;
    if (T[0] == q) { *which = t; *slot = 0; return 1; }
    if (T[1] == q) { *which = t; *slot = 1; return 1; }
  }
  return 0;
}

int oracle_prepare(const oracle_params* P, int64_t* E_out, int64_t* lo, int64_t* hi) {
  if (P->d < 1 || P->r < 1 || P->k < 1 || P->N < 2 || (P->N % 2) != 0) return ORACLE_EINVAL;
  int32_t sum = 0;
  for (int32_t q = 0; q < P->r; ++q) {
    if (P->blocks[q] < 1) return ORACLE_EINVAL;
    sum += P->blocks[q];
  }
  if (sum != P->d) return ORACLE_EINVAL;
  /* B = max_q N^{d_q}; budget B <= 2^40 (reading C1) */
  double logB = 0.0;
  int64_t B = 1;
  for (int32_t q = 0; q < P->r; ++q) {
    double l = P->blocks[q] * log2((double)P->N);
    if (l > 40.0 + 1e-9) return ORACLE_EPRECISION;
    if (l > logB) logB = l;
    int64_t b = ipow(P->N, P->blocks[q]);
    if (b > B) B = b;
  }
  int64_t* base_lo = (int64_t*)malloc(sizeof(int64_t) * (size_t)P->r);
  int64_t* base_hi = (int64_t*)malloc(sizeof(int64_t) * (size_t)P->r);
  int rc = ORACLE_OK;
  for (int32_t q = 0; q < P->r; ++q) oracle_block_range(P->N, P->blocks[q], &base_lo[q], &base_hi[q]);
  int64_t scale = 1;
  for (int32_t t = 0; t < P->n_tilts; ++t) {
    const int64_t* T = P->tilts + 5 * t;
    int64_t a0 = T[0], a1 = T[1], b = T[2], h = T[3], c = T[4];
    if (a0 < 0 || a1 < 0 || a0 >= P->r || a1 >= P->r || a0 == a1) rc = ORACLE_EINVAL;
    if (b < 1 || h < 1 || b * b + h * h != c * c || gcd64(b, c) != 1 || gcd64(h, c) != 1) rc = ORACLE_EINVAL;
    for (int32_t u = 0; u < t; ++u) {
      const int64_t* U = P->tilts + 5 * u;
      if (U[0] == a0 || U[1] == a0 || U[0] == a1 || U[1] == a1) rc = ORACLE_EINVAL;
    }
    if (b + h > scale) scale = b + h;
  }
  for (int32_t q = 0; q < P->r && rc == ORACLE_OK; ++q) {
    int32_t t, slot;
    if (!tilt_of_axis(P, q, &t, &slot)) { lo[q] = base_lo[q]; hi[q] = base_hi[q]; continue; }
    const int64_t* T = P->tilts + 5 * t;
    int64_t a0 = T[0], a1 = T[1], b = T[2], h = T[3];
    if (slot == 0) {   /* v0 = b u0 - h u1 */
      lo[q] = b * base_lo[a0] - h * base_hi[a1];
      hi[q] = b * base_hi[a0] - h * base_lo[a1];
    } else {           /* v1 = h u0 + b u1 */
      lo[q] = h * base_lo[a0] + b * base_lo[a1];
      hi[q] = h * base_hi[a0] + b * base_hi[a1];
    }
  }
  free(base_lo);
  free(base_hi);
  if (rc) return rc;
  int64_t E = P->E ? P->E : 2 * B * scale;     /* eps = 1/(2 N^{d1}), widened by the tilt (C2) */
  if (E > ((int64_t)1 << 42)) return ORACLE_EPRECISION;
  for (int32_t q = 0; q < P->r; ++q) {
    /* decodable range of Arg/(2 pi eps) is [-E/2, E/2) (Eq. (7)) */
    if (2 * hi[q] >= E || -2 * lo[q] > E) return ORACLE_EINVAL;
  }
  *E_out = E;
  return ORACLE_OK;
}

/* v_j = T * unwrap(w_j) (Eq. (35), then Eq. (27) on every tilted axis pair) */
int oracle_project(const oracle_params* P, const int32_t* w, int32_t k, int64_t* v) {
  for (int32_t j = 0; j < k; ++j) {
    int rc = oracle_unwrap_freq(P->d, P->N, P->r, P->blocks, w + (size_t)j * P->d, v + (size_t)j * P->r);
    if (rc) return rc;
    for (int32_t t = 0; t < P->n_tilts; ++t) {
      const int64_t* T = P->tilts + 5 * t;
      int64_t out[2];
      int64_t* vj = v + (size_t)j * P->r;
      oracle_tilt_freq(T[2], T[3], vj[T[0]], vj[T[1]], out);
      vj[T[0]] = out[0];
      vj[T[1]] = out[1];
    }
  }
  return ORACLE_OK;
}

/* ------------------------------------------------------------------------ */
/* evaluation of f                                                          */
/* ------------------------------------------------------------------------ */

/* Eq. (9) at a real point, plain double (pins only) */
void oracle_eval_point(int32_t d, int32_t K, const int32_t* w, const double* a, const double* t,
                       double* out) {
  double re = 0.0, im = 0.0;
  for (int32_t j = 0; j < K; ++j) {
    double ph = 0.0;
    for (int32_t l = 0; l < d; ++l) ph += (double)w[(size_t)j * d + l] * t[l];
    double c = cos(2.0 * M_PI * ph), s = sin(2.0 * M_PI * ph);
    re += a[2 * j] * c - a[2 * j + 1] * s;
    im += a[2 * j] * s + a[2 * j + 1] * c;
  }
  out[0] = re;
  out[1] = im;
}

/* Eq. (41) / Alg. 2 l.13-14: s[h] = sum_j c_j exp(2 pi i v_j . ((h/p) e_m + (1/E) e_n)).
 * The phase v_m h/p + v_n/E is reduced exactly: ((h (v_m mod p)) mod p)/p + (v_n mod E)/E. */
void oracle_sample_line(int32_t K, int32_t r, const int64_t* v, const double* c, int64_t p,
                        int32_t m, int32_t n, int64_t E, double* s) {
  for (int64_t h = 0; h < p; ++h) {
    double re = 0.0, im = 0.0;
    for (int32_t j = 0; j < K; ++j) {
      const int64_t* vj = v + (size_t)j * r;
      int64_t num_p = mod_pos(h * mod_pos(vj[m], p), p);
      double phi = (double)num_p / (double)p;
      if (n >= 0) {
        phi += (double)mod_pos(vj[n], E) / (double)E;
        if (phi >= 1.0) phi -= 1.0;
      }
      double cs = cos(2.0 * M_PI * phi), sn = sin(2.0 * M_PI * phi);
      re += c[2 * j] * cs - c[2 * j + 1] * sn;
      im += c[2 * j] * sn + c[2 * j + 1] * cs;
    }
    s[2 * h] = re;
    s[2 * h + 1] = im;
  }
}

/* ------------------------------------------------------------------------ */
/* DFT (Eq. (3)); unnormalised forward transform, exact-index twiddle table   */
/* ------------------------------------------------------------------------ */

void oracle_dft(int64_t p, const double* s, double* F) {
  double* W = (double*)malloc(sizeof(double) * 2 * (size_t)p);
  for (int64_t q = 0; q < p; ++q) {
    W[2 * q] = cos(2.0 * M_PI * (double)q / (double)p);
    W[2 * q + 1] = -sin(2.0 * M_PI * (double)q / (double)p);
  }
  for (int64_t b = 0; b < p; ++b) {
    double re = 0.0, im = 0.0;
    for (int64_t h = 0; h < p; ++h) {
      int64_t q = (h * b) % p;
      re += s[2 * h] * W[2 * q] - s[2 * h + 1] * W[2 * q + 1];
      im += s[2 * h] * W[2 * q + 1] + s[2 * h + 1] * W[2 * q];
    }
    F[2 * b] = re;
    F[2 * b + 1] = im;
  }
  free(W);
}

/* ------------------------------------------------------------------------ */
/* select + collision test + decode (Alg. 2 l.18-32, Eqs. (41)-(42))         */
/* ------------------------------------------------------------------------ */

typedef struct { double mag; int64_t b; } cand_t;

static int cand_cmp_mag(const void* x, const void* y) {   /* |F_0|^2 descending, ties -> smaller b (C6) */
  const cand_t* a = (const cand_t*)x;
  const cand_t* b = (const cand_t*)y;
  if (a->mag > b->mag) return -1;
  if (a->mag < b->mag) return 1;
  return (a->b < b->b) ? -1 : (a->b > b->b);
}
static int cand_cmp_b(const void* x, const void* y) {
  const cand_t* a = (const cand_t*)x;
  const cand_t* b = (const cand_t*)y;
  return (a->b < b->b) ? -1 : (a->b > b->b);
}

int32_t oracle_decode(const oracle_params* P, int64_t E, const int64_t* lo, const int64_t* hi,
                      int64_t p, int32_t m, int32_t kstar, const double* F,
                      int32_t* n_cand, int32_t* acc_b, int64_t* acc_v, double* acc_a) {
  return oracle_decode_ex(P, E, lo, hi, p, m, kstar, F, n_cand, NULL, acc_b, acc_v, acc_a);
}

int32_t oracle_decode_ex(const oracle_params* P, int64_t E, const int64_t* lo, const int64_t* hi,
                         int64_t p, int32_t m, int32_t kstar, const double* F,
                         int32_t* n_cand, int32_t* n_nonempty, int32_t* acc_b, int64_t* acc_v, double* acc_a) {
  const int32_t r = P->r;
  const double* F0 = F;
  /* select (C5, C18): bins with |F_0[b]| >= floor * p, at most the k* largest.  The magnitude is |F_0|^2 =
   * Re^2 + Im^2, each operation rounded once, and the k* cap ranks it rounded to 36 significant bits (reading
   * R5): the bins carry ~1e-13 relative rounding error, so magnitudes that agree to ~1.5e-11 are ties (-> the
   * smaller b, C6) -- e.g. a false entry's bin and the collided bin it was decoded from, equal in exact
   * arithmetic -- and any implementation decides them as exact arithmetic would */
  cand_t* cand = (cand_t*)malloc(sizeof(cand_t) * (size_t)p);
  int32_t nc = 0;
  const double floor_abs = P->bin_floor_rel * (double)p;
  const double floor2 = floor_abs * floor_abs;
  for (int64_t b = 0; b < p; ++b) {
    const double re = F0[2 * b], im = F0[2 * b + 1];
    const double re2 = re * re, im2 = im * im;
    const double mag2 = re2 + im2;
    if (mag2 >= floor2) {
      int ex;
      const double fr = frexp(mag2, &ex);
      cand[nc].mag = ldexp(nearbyint(ldexp(fr, 36)), ex - 36);
      cand[nc].b = b;
      ++nc;
    }
  }
  if (n_nonempty) *n_nonempty = nc;
  if (nc > kstar) {
    qsort(cand, (size_t)nc, sizeof(cand_t), cand_cmp_mag);   /* SORT (Alg. 2 l.18) */
    nc = kstar;
    qsort(cand, (size_t)nc, sizeof(cand_t), cand_cmp_b);
  }
  *n_cand = nc;
  int32_t na = 0;
  int64_t* v = (int64_t*)malloc(sizeof(int64_t) * (size_t)r);
  for (int32_t ci = 0; ci < nc; ++ci) {
    int64_t b = cand[ci].b;
    double f0r = F0[2 * b], f0i = F0[2 * b + 1];
    double mag0 = hypot(f0r, f0i);
    /* Eq. (42): |F_n[b]| / |F_0[b]| = 1 for every n (ratio direction of Eq. (42), C4) */
    int ok = 1;
    for (int32_t n = 0; n < r && ok; ++n) {
      const double* Fn = F + (size_t)(1 + n) * 2 * p;
      double rho = hypot(Fn[2 * b], Fn[2 * b + 1]) / mag0;
      if (!(fabs(rho - 1.0) < P->tol)) ok = 0;
    }
    if (!ok) continue;
    /* Eq. (41): v_n = Arg(F_n[b] / F_0[b]) / (2 pi eps), computed as Arg(F_n conj(F_0)) E / (2 pi) */
    for (int32_t n = 0; n < r && ok; ++n) {
      const double* Fn = F + (size_t)(1 + n) * 2 * p;
      double qr = Fn[2 * b] * f0r + Fn[2 * b + 1] * f0i;
      double qi = Fn[2 * b + 1] * f0r - Fn[2 * b] * f0i;
      double x = atan2(qi, qr) * (double)E / (2.0 * M_PI);
      double xr = nearbyint(x);
      if (fabs(x - xr) > P->round_tol) ok = 0;          /* C14 */
      v[n] = (int64_t)xr;
      if ((P->extra_checks & 1) && (v[n] < lo[n] || v[n] > hi[n])) ok = 0;   /* C15 (i) */
    }
    if (!ok) continue;
    if ((P->extra_checks & 2) && mod_pos(v[m], p) != b) continue;          /* C15 (ii) */
    acc_b[na] = (int32_t)b;
    memcpy(acc_v + (size_t)na * r, v, sizeof(int64_t) * (size_t)r);
    acc_a[2 * na] = f0r / (double)p;                                         /* Eq. (7): a = F_0/p (C12) */
    acc_a[2 * na + 1] = f0i / (double)p;
    ++na;
  }
  free(v);
  free(cand);
  return na;
}

/* ------------------------------------------------------------------------ */
/* Algorithm 2                                                              */
/* ------------------------------------------------------------------------ */

typedef struct {
  int32_t n, cap, r;
  int64_t* v;     /* [cap][r] */
  double* a;      /* [cap][2] */
} registry_t;

static int32_t registry_find(const registry_t* R, const int64_t* v) {
  for (int32_t e = 0; e < R->n; ++e)
    if (memcmp(R->v + (size_t)e * R->r, v, sizeof(int64_t) * (size_t)R->r) == 0) return e;
  return -1;
}

typedef struct { const int32_t* w; int32_t d; } row_ref;
static int row_cmp(const void* x, const void* y) {
  const row_ref* a = (const row_ref*)x;
  const row_ref* b = (const row_ref*)y;
  for (int32_t l = 0; l < a->d; ++l) {
    if (a->w[l] < b->w[l]) return -1;
    if (a->w[l] > b->w[l]) return 1;
  }
  return 0;
}

/* ------------------------------------------------------------------------ */
/* stall fallback ("apply the tilting method with several angles until */
/* all k frequency pairs are found", Algorithm 3; reading R23)      */
/* ------------------------------------------------------------------------ */

static const int64_t kFallbackTriples[4][3] = {{3, 4, 5}, {5, 12, 13}, {8, 15, 17}, {7, 24, 25}};

static uint64_t splitmix64_fin(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

void oracle_axis_order(int32_t r, int32_t seed, int32_t* pi) {
  for (int32_t i = 0; i < r; ++i) pi[i] = i;
  for (int32_t i = r - 1; i >= 1; --i) {
    const uint64_t c = (uint64_t)seed * 0x9E3779B97F4A7C15ULL + (uint64_t)(r - i) * 0xD1B54A32D192ED03ULL;
    const int32_t j = (int32_t)(splitmix64_fin(c) % (uint64_t)(i + 1));
    const int32_t t = pi[i];
    pi[i] = pi[j];
    pi[j] = t;
  }
}

int32_t oracle_fallback_tilts(int32_t r, int32_t lvl, int64_t* out) {
  if (lvl < 1 || lvl > ORACLE_MAX_FALLBACK) return 0;
  if (lvl > 4) {
    /* R24: "randomizing the order of the dimensions", applied to the axes the tilt pairs up: the rounds of
     * a round robin over a seeded order of the axes, every pair tilted once over n - 1 levels */
    const int32_t j = lvl - 5;
    const int32_t n = r + (r & 1);
    if (r < 2 || j >= n - 1) return 0;
    const int64_t* T = kFallbackTriples[j % 4];
    int32_t* pi = (int32_t*)malloc(sizeof(int32_t) * (size_t)r);
    int32_t* a = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
    oracle_axis_order(r, 1, pi);
    a[0] = 0;
    for (int32_t i = 1; i < n; ++i) a[i] = 1 + (i - 1 + j) % (n - 1);   /* slots 1..n-1 rotated by j */
    int32_t cnt = 0;
    for (int32_t i = 0; i < n / 2; ++i) {
      const int32_t x = a[i], y = a[n - 1 - i];
      if (x >= r || y >= r) continue;                                  /* the padding slot of an odd r */
      int64_t* o = out + 5 * cnt++;
      o[0] = pi[x]; o[1] = pi[y]; o[2] = T[0]; o[3] = T[1]; o[4] = T[2];
    }
    free(a);
    free(pi);
    return cnt;
  }
  const int64_t* T = kFallbackTriples[lvl - 1];
  /* disjoint pairs (q, q + s): level 1 s = 1 from axis 0, level 2 s = 1 from axis 1 (r >= 3), level 3 s = 2,
   * level 4 s = 3 -- for r <= 4 every axis pair is tilted at some level ("randomizing the order
   * of the dimensions" in a fixed, reproducible form) */
  const int32_t s = lvl <= 2 ? 1 : lvl - 1;
  const int32_t off = (lvl == 2 && r >= 3) ? 1 : 0;
  int32_t n = 0;
  for (int32_t b = off; b < r; b += 2 * s)
    for (int32_t i = 0; i < s && b + i + s < r; ++i, ++n) {
      int64_t* o = out + 5 * n;
      o[0] = b + i; o[1] = b + i + s; o[2] = T[0]; o[3] = T[1]; o[4] = T[2];   /* base, height, hypo */
    }
  return n;
}

/* one level of the schedule: level 0 = the caller's own tilts and E, level >= 1 = fallback tilts with the
 * default E of that tilt (2 B (base + height), reading R2) */
static int level_params(const oracle_params* P, int32_t lvl, oracle_params* out, int64_t* tbuf) {
  *out = *P;
  if (lvl == 0) return 1;
  out->n_tilts = oracle_fallback_tilts(P->r, lvl, tbuf);
  out->tilts = tbuf;
  out->E = 0;
  return out->n_tilts > 0;
}

/* untilt v (level tilts, last pair first as in the final wrap); 0 on success, -1 if not integral */
static int untilt_all(const oracle_params* L, int64_t* u) {
  for (int32_t t = L->n_tilts - 1; t >= 0; --t) {
    const int64_t* T = L->tilts + 5 * t;
    int64_t out[2];
    if (oracle_untilt_freq(T[2], T[3], T[4], u[T[0]], u[T[1]], out)) return -1;
    u[T[0]] = out[0];
    u[T[1]] = out[1];
  }
  return 0;
}

static void tilt_all(const oracle_params* L, int64_t* u) {
  for (int32_t t = 0; t < L->n_tilts; ++t) {
    const int64_t* T = L->tilts + 5 * t;
    int64_t out[2];
    oracle_tilt_freq(T[2], T[3], u[T[0]], u[T[1]], out);
    u[T[0]] = out[0];
    u[T[1]] = out[1];
  }
}

static int64_t now_ns(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (int64_t)ts.tv_sec * 1000000000 + ts.tv_nsec;
}

int oracle_solve(const oracle_params* P, const int32_t* w, const double* a, int32_t* out_w,
                 double* out_a, int32_t* out_count, int64_t* out_samples, int32_t* out_iters,
                 int32_t trace_cap, int64_t* trace) {
  return oracle_solve_timed(P, w, a, out_w, out_a, out_count, out_samples, out_iters, trace_cap, trace, NULL);
}

/* ns[0] = wall time of the solve, ns[1] = the part spent sampling f - g (Alg. 2 l.13-14); the paper's
 * "main part" timing excludes the sampling */
static int solve_impl(const oracle_params* P, const int32_t* w, const double* a, int32_t* out_w,
                      double* out_a, int32_t* out_count, int64_t* out_samples, int32_t* out_iters,
                      int32_t trace_cap, int64_t* trace, int64_t* ns, int64_t* raw_v, double* raw_a,
                      int32_t* raw_n);

int oracle_solve_timed(const oracle_params* P, const int32_t* w, const double* a, int32_t* out_w,
                       double* out_a, int32_t* out_count, int64_t* out_samples, int32_t* out_iters,
                       int32_t trace_cap, int64_t* trace, int64_t* ns) {
  return solve_impl(P, w, a, out_w, out_a, out_count, out_samples, out_iters, trace_cap, trace, ns, NULL, NULL,
                    NULL);
}

/* debugging aid: the registry R itself (reduced keys [<=k][r] and coefficients, insertion order after prunes)
 * at the end of the loop, before the wrap */
int oracle_solve_raw(const oracle_params* P, const int32_t* w, const double* a, int64_t* raw_v, double* raw_a,
                     int32_t* raw_n) {
  int32_t* ow = (int32_t*)malloc(sizeof(int32_t) * (size_t)P->k * P->d);
  double* oa = (double*)malloc(sizeof(double) * 2 * (size_t)P->k);
  int32_t cnt = 0;
  int st = solve_impl(P, w, a, ow, oa, &cnt, NULL, NULL, 0, NULL, NULL, raw_v, raw_a, raw_n);
  free(ow);
  free(oa);
  return st;
}

static int solve_impl(const oracle_params* P, const int32_t* w, const double* a, int32_t* out_w,
                      double* out_a, int32_t* out_count, int64_t* out_samples, int32_t* out_iters,
                      int32_t trace_cap, int64_t* trace, int64_t* ns, int64_t* raw_v, double* raw_a,
                      int32_t* raw_n) {
  const int64_t t_start = now_ns();
  int64_t t_sampling = 0;
  const int32_t r = P->r, k = P->k, d = P->d;
  int64_t E;
  int64_t* lo = (int64_t*)malloc(sizeof(int64_t) * (size_t)r);
  int64_t* hi = (int64_t*)malloc(sizeof(int64_t) * (size_t)r);
  /* level 0 = the caller's plan; a stall moves to the next fallback level (reading R23) */
  int64_t* tbuf = (int64_t*)malloc(sizeof(int64_t) * 5 * (size_t)(r / 2 + 1));
  oracle_params Lv;
  int32_t lvl = 0;
  level_params(P, 0, &Lv, tbuf);
  int rc = oracle_prepare(&Lv, &E, lo, hi);
  if (rc) { free(lo); free(hi); free(tbuf); return rc; }
  const int32_t stall_limit = P->stall_limit > 0 ? P->stall_limit : (2 * r > 16 ? 2 * r : 16);

  /* the signal: reduced frequencies of its modes (only used to evaluate f, Eq. (38)) */
  int64_t* vf = (int64_t*)malloc(sizeof(int64_t) * (size_t)k * r);
  rc = oracle_project(&Lv, w, k, vf);
  if (rc) { free(lo); free(hi); free(vf); free(tbuf); return rc; }

  registry_t R;
  R.n = 0; R.cap = k; R.r = r;
  R.v = (int64_t*)malloc(sizeof(int64_t) * (size_t)k * r);
  R.a = (double*)malloc(sizeof(double) * 2 * (size_t)k);

  /* terms of the residual f - g: k signal modes then the registry with negated coefficients */
  int64_t* tv = (int64_t*)malloc(sizeof(int64_t) * (size_t)2 * k * r);
  double* tc = (double*)malloc(sizeof(double) * 2 * (size_t)2 * k);
  double* F = NULL;
  int64_t Fcap = 0;

  int64_t samples = 0;
  int32_t i = 1, it = 1, stall = 0, status = ORACLE_PARTIAL;   /* i: Alg. 2/3 counter of the level, it: total */
  const int32_t G = P->n_spec > 1 ? P->n_spec : 1;            /* reading R26: primes per iteration */
  int32_t* touch = (int32_t*)malloc(sizeof(int32_t) * (size_t)k);   /* set that last updated entry e this iteration */
  int32_t* set_b = (int32_t*)malloc(sizeof(int32_t) * (size_t)G * k);
  int64_t* set_v = (int64_t*)malloc(sizeof(int64_t) * (size_t)G * k * r);
  double* set_a = (double*)malloc(sizeof(double) * 2 * (size_t)G * k);
  int32_t* set_n = (int32_t*)malloc(sizeof(int32_t) * (size_t)G);
  while (R.n < k && it <= P->max_iter) {                        /* Alg. 2 l.6 */
    int32_t kstar = k - R.n;                                  /* l.7 */
    int64_t p0 = 0;
    int32_t m0 = 0;
    /* l.10: g from the registry; residual terms (one snapshot of R for every prime of the iteration) */
    memcpy(tv, vf, sizeof(int64_t) * (size_t)k * r);
    for (int32_t j = 0; j < k; ++j) { tc[2 * j] = a[2 * j]; tc[2 * j + 1] = a[2 * j + 1]; }
    for (int32_t e = 0; e < R.n; ++e) {
      memcpy(tv + (size_t)(k + e) * r, R.v + (size_t)e * r, sizeof(int64_t) * (size_t)r);
      tc[2 * (k + e)] = -R.a[2 * e];
      tc[2 * (k + e) + 1] = -R.a[2 * e + 1];
    }
    int32_t K = k + R.n;
    int32_t ncand = 0, nnonempty = 0, n_accum = 0, na = 0;
    for (int32_t g = 0; g < G; ++g) {
      const int32_t ig = (i - 1) * G + g + 1;                  /* prime counter of this prime (G = 1: i) */
      int64_t p = (P->n_primes > 0 && P->primes)
                      ? P->primes[(ig - 1) % P->n_primes]
                      : oracle_ith_prime_at_least((int64_t)P->c * kstar, ig);   /* l.8 (C11) */
      int32_t m = ig % r;                                      /* l.9, 0-based (C10) */
      if (g == 0) { p0 = p; m0 = m; }
      if ((r + 1) * p > Fcap) {
        Fcap = (int64_t)(r + 1) * p;
        free(F);
        F = (double*)malloc(sizeof(double) * 2 * (size_t)Fcap);
      }
      double* s = (double*)malloc(sizeof(double) * 2 * (size_t)p);
      /* l.11-17: sample the unshifted line and the r shifted lines, DFT each */
      for (int32_t line = 0; line <= r; ++line) {
        const int64_t t0 = now_ns();
        oracle_sample_line(K, r, tv, tc, p, m, line - 1, E, s);
        t_sampling += now_ns() - t0;
        oracle_dft(p, s, F + (size_t)line * 2 * p);
      }
      free(s);
      samples += (int64_t)(r + 1) * p;                        /* f evaluations only (C22) */
      /* l.18-32 */
      int32_t nc1 = 0, nn1 = 0;
      set_n[g] = oracle_decode_ex(P, E, lo, hi, p, m, kstar, F, &nc1, &nn1, set_b + (size_t)g * k,
                                  set_v + (size_t)g * k * r, set_a + (size_t)g * 2 * k);
      ncand += nc1;
      nnonempty += nn1;
      na += set_n[g];
    }
    /* l.30: R <- R u (w~, a), accumulating (C16), in ascending b; the sets in prime order, a key that an earlier
     * set of this iteration already updated is skipped (R26: that prime saw the same residual) */
    for (int32_t e = 0; e < k; ++e) touch[e] = -1;
    for (int32_t g = 0; g < G; ++g) {
      const int64_t* acc_v = set_v + (size_t)g * k * r;
      const double* acc_a = set_a + (size_t)g * 2 * k;
      for (int32_t t = 0; t < set_n[g]; ++t) {
        int32_t e = registry_find(&R, acc_v + (size_t)t * r);
        if (e >= 0) {
          if (touch[e] >= 0 && touch[e] < g) continue;
          R.a[2 * e] += acc_a[2 * t];
          R.a[2 * e + 1] += acc_a[2 * t + 1];
          touch[e] = g;
          ++n_accum;
        } else {
          if (R.n >= k) continue;         /* capacity k (only false accepts of several primes can reach it) */
          memcpy(R.v + (size_t)R.n * r, acc_v + (size_t)t * r, sizeof(int64_t) * (size_t)r);
          R.a[2 * R.n] = acc_a[2 * t];
          R.a[2 * R.n + 1] = acc_a[2 * t + 1];
          touch[R.n] = g;
          ++R.n;
        }
      }
    }
    const int64_t p = p0;
    const int32_t m = m0;
    /* l.33: prune small coefficients (C17), order-preserving */
    int32_t keep = 0;
    for (int32_t e = 0; e < R.n; ++e) {
      if (hypot(R.a[2 * e], R.a[2 * e + 1]) < P->prune_floor) continue;
      if (keep != e) {
        memmove(R.v + (size_t)keep * r, R.v + (size_t)e * r, sizeof(int64_t) * (size_t)r);
        R.a[2 * keep] = R.a[2 * e];
        R.a[2 * keep + 1] = R.a[2 * e + 1];
      }
      ++keep;
    }
    const int32_t n_pruned = R.n - keep;
    R.n = keep;
    if (trace && it <= trace_cap) {
      int64_t* T = trace + (size_t)(it - 1) * ORACLE_TRACE_COLS;
      T[0] = it; T[1] = p; T[2] = m; T[3] = ncand; T[4] = na;
      T[5] = nnonempty; T[6] = n_accum; T[7] = n_pruned;
    }
    stall = (na == 0) ? stall + 1 : 0;
    ++i;                                                        /* l.34 */
    ++it;
    if (stall >= stall_limit && R.n < k && it <= P->max_iter) {
      /* C19 / R23: no progress for stall_limit iterations -> the next tilt of the schedule (Alg. 3), keeping
       * what was found: every entry is mapped to the new coordinates exactly (untilt, which must be
       * integral, then tilt); entries that do not untilt exactly are dropped */
      oracle_params Ln;
      int64_t* tn = (int64_t*)malloc(sizeof(int64_t) * 5 * (size_t)(r / 2 + 1));
      int64_t En;
      if (lvl + 1 > P->n_fallback || lvl + 1 > ORACLE_MAX_FALLBACK || !level_params(P, lvl + 1, &Ln, tn) ||
          oracle_prepare(&Ln, &En, lo, hi) != ORACLE_OK) {
        free(tn);
        break;
      }
      int32_t keep = 0;
      int64_t* u = (int64_t*)malloc(sizeof(int64_t) * (size_t)r);
      for (int32_t e = 0; e < R.n; ++e) {
        memcpy(u, R.v + (size_t)e * r, sizeof(int64_t) * (size_t)r);
        if (untilt_all(&Lv, u)) continue;
        tilt_all(&Ln, u);
        memcpy(R.v + (size_t)keep * r, u, sizeof(int64_t) * (size_t)r);
        R.a[2 * keep] = R.a[2 * e];
        R.a[2 * keep + 1] = R.a[2 * e + 1];
        ++keep;
      }
      free(u);
      R.n = keep;
      ++lvl;
      memcpy(tbuf, tn, sizeof(int64_t) * 5 * (size_t)(r / 2 + 1));
      free(tn);
      Lv = Ln;
      Lv.tilts = tbuf;
      E = En;
      oracle_project(&Lv, w, k, vf);                            /* the signal in the new coordinates */
      i = 1;                                                    /* Alg. 3 l.5 */
      stall = 0;
    } else if (stall >= stall_limit) {
      break;
    }
  }
  if (R.n == k) status = ORACLE_OK;
  if (raw_n) {
    *raw_n = R.n;
    memcpy(raw_v, R.v, sizeof(int64_t) * (size_t)R.n * r);
    memcpy(raw_a, R.a, sizeof(double) * 2 * (size_t)R.n);
  }

  /* l.36: untilt (C20) and wrap back to d dimensions, then canonical order */
  int32_t* wt = (int32_t*)malloc(sizeof(int32_t) * (size_t)(R.n > 0 ? R.n : 1) * d);
  row_ref* refs = (row_ref*)malloc(sizeof(row_ref) * (size_t)(R.n > 0 ? R.n : 1));
  int32_t* idx_of = (int32_t*)malloc(sizeof(int32_t) * (size_t)(R.n > 0 ? R.n : 1));
  int64_t* u = (int64_t*)malloc(sizeof(int64_t) * (size_t)r);
  for (int32_t e = 0; e < R.n && status >= 0; ++e) {
    memcpy(u, R.v + (size_t)e * r, sizeof(int64_t) * (size_t)r);
    if (untilt_all(&Lv, u)) { status = ORACLE_ECORRUPT; break; }
    if (oracle_wrap_freq(d, P->N, r, P->blocks, u, wt + (size_t)e * d)) { status = ORACLE_ECORRUPT; break; }
    refs[e].w = wt + (size_t)e * d;
    refs[e].d = d;
  }
  int32_t cnt = 0;
  if (status >= 0) {
    qsort(refs, (size_t)R.n, sizeof(row_ref), row_cmp);
    for (int32_t e = 0; e < R.n; ++e) {
      int32_t src = (int32_t)((refs[e].w - wt) / d);
      idx_of[e] = src;
      memcpy(out_w + (size_t)e * d, refs[e].w, sizeof(int32_t) * (size_t)d);
      out_a[2 * e] = R.a[2 * src];
      out_a[2 * e + 1] = R.a[2 * src + 1];
    }
    cnt = R.n;
  }
  *out_count = cnt;
  if (out_samples) *out_samples = samples;
  if (out_iters) *out_iters = it - 1;

  free(u); free(idx_of); free(refs); free(wt);
  free(F); free(set_a); free(set_v); free(set_b); free(set_n); free(touch); free(tc); free(tv);
  free(R.a); free(R.v); free(vf); free(hi); free(lo); free(tbuf);
  if (ns) { ns[0] = now_ns() - t_start; ns[1] = t_sampling; }
  return status;
}

/* ------------------------------------------------------------------------ */
/* batch of independent signals over host threads                           */
/* ------------------------------------------------------------------------ */

typedef struct {
  const oracle_params* P;
  int32_t batch, next, lock_init;
  pthread_mutex_t lock;
  const int32_t* w; const double* a;
  int32_t* out_w; double* out_a; int32_t* out_count; int64_t* out_samples; int32_t* out_iters;
  int32_t* out_status;
  int64_t* out_ns;
} batch_ctx;

static void* batch_worker(void* arg) {
  batch_ctx* C = (batch_ctx*)arg;
  const int32_t k = C->P->k, d = C->P->d;
  for (;;) {
    pthread_mutex_lock(&C->lock);
    int32_t s = C->next++;
    pthread_mutex_unlock(&C->lock);
    if (s >= C->batch) break;
    int st = oracle_solve_timed(C->P, C->w + (size_t)s * k * d, C->a + (size_t)s * 2 * k,
                                C->out_w + (size_t)s * k * d, C->out_a + (size_t)s * 2 * k,
                                C->out_count + s, C->out_samples ? C->out_samples + s : NULL,
                                C->out_iters ? C->out_iters + s : NULL, 0, NULL,
                                C->out_ns ? C->out_ns + 2 * (size_t)s : NULL);
    C->out_status[s] = st;
  }
  return NULL;
}

int oracle_solve_batch(const oracle_params* P, int32_t batch, const int32_t* w, const double* a,
                       int32_t* out_w, double* out_a, int32_t* out_count, int64_t* out_samples,
                       int32_t* out_iters, int32_t* out_status, int32_t n_threads, int64_t* out_ns) {
  batch_ctx C;
  memset(&C, 0, sizeof(C));
  C.P = P; C.batch = batch; C.next = 0;
  C.w = w; C.a = a; C.out_w = out_w; C.out_a = out_a; C.out_count = out_count;
  C.out_samples = out_samples; C.out_iters = out_iters; C.out_status = out_status; C.out_ns = out_ns;
  pthread_mutex_init(&C.lock, NULL);
  if (n_threads < 1) n_threads = 1;
  if (n_threads > batch) n_threads = batch > 0 ? batch : 1;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)n_threads);
  for (int32_t t = 0; t < n_threads; ++t) pthread_create(&th[t], NULL, batch_worker, &C);
  for (int32_t t = 0; t < n_threads; ++t) pthread_join(th[t], NULL);
  free(th);
  pthread_mutex_destroy(&C.lock);
  int worst = ORACLE_OK;
  for (int32_t s = 0; s < batch; ++s)
    if (out_status[s] != ORACLE_OK && (worst == ORACLE_OK || out_status[s] < 0)) worst = out_status[s];
  return worst;
}
