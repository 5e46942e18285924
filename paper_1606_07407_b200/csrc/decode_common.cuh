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

// |F|^2 = Re^2 + Im^2, every operation rounded once (no contraction): the select's magnitude (reading R5), the
// same number as the oracle's for the same bin
__device__ __forceinline__ double mag2_rn(double2 f) {
  return __dadd_rn(__dmul_rn(f.x, f.x), __dmul_rn(f.y, f.y));
}
// the k* cap's ranking key (reading R5): |F|^2 rounded to 36 significant bits (round half to even), so that
// magnitudes equal up to the bins' rounding error are ties -> smaller b, as in the oracle
__device__ __forceinline__ double rank_key(double mag2) {
  int ex;
  const double fr = frexp(mag2, &ex);
  return ldexp(rint(ldexp(fr, 36)), ex - 36);
}

// a5 select (Alg. 2 l.18, readings R5/R6): bins b < p with |F_0[b]|^2 >= floor_abs^2 in ascending b; if more than
// kstar qualify, the kstar largest |F_0|^2 (ties -> smaller b), still ascending.  f0(b) returns F_0[b].
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
  const double floor2 = __dmul_rn(floor_abs, floor_abs);
  for (int b = b0; b < b1; ++b) {
    if (mag2_rn(f0(b)) >= floor2) mask |= 1u << (b - b0);
  }
  int pos = block_excl_scan(__popc(mask), scratch, &total);
  for (int b = b0; b < b1; ++b)
    if (mask >> (b - b0) & 1u) {
      cand[pos] = b;
      mag[pos] = rank_key(mag2_rn(f0(b)));
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

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
// registry key hash of the r-long coordinate vector: XOR over n of mix64(v_n ^ n * golden) -- order-free, so a
// warp computes it with lanes along n (key_hash_warp) and a single thread with a plain loop (same value)
__device__ __forceinline__ uint64_t key_term(int64_t v, int n) {
  return mix64((uint64_t)v ^ ((uint64_t)(n + 1) * 0x9E3779B97F4A7C15ULL));
}
__device__ __forceinline__ uint64_t key_hash_warp(const int64_t* v, int64_t stride, int r, int lane) {
  uint64_t h = 0;
  for (int n = lane; n < r; n += 32) h ^= key_term(v[(int64_t)n * stride], n);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) h ^= __shfl_xor_sync(0xffffffffu, h, o);
  return h;
}

// fused record exchange (line_exchange = 1): the FFT epilogue of shard g stores the word into every shard's copy of
// its record (receive slot g); flags are int32 words at the record start, coordinates int64 words after rec_fw
__device__ __forceinline__ int64_t peer_rec_off(const DevParams& P, int s) {
  return ((int64_t)P.line_g * P.batch + s) * P.rec_words;
}
__device__ __forceinline__ void peer_put_flag(const DevParams& P, int s, int ci, int32_t v) {
  const int64_t off = peer_rec_off(P, s);
  for (int h = 0; h < P.line_G; ++h) reinterpret_cast<int32_t*>(P.peer_recv[h] + off)[ci] = v;
}
__device__ __forceinline__ void peer_put_coord(const DevParams& P, int s, int n, int ci, int64_t v) {
  const int64_t off = peer_rec_off(P, s) + P.rec_fw + (int64_t)(n - 1) * P.k + ci;
  for (int h = 0; h < P.line_G; ++h) P.peer_recv[h][off] = v;
}
// after a CTA's record stores: system-scope release of its (shard, local line, signal) stamp on every shard
__device__ __forceinline__ void peer_release_line(const DevParams& P, int s, int n) {
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    const int64_t idx = ((int64_t)P.line_g * P.L_ref + n) * P.batch + s;
    for (int h = 0; h < P.line_G; ++h)
      asm volatile("st.release.sys.global.b32 [%0], %1;" ::"l"(P.peer_stamp[h] + idx), "r"(P.peer_epoch) : "memory");
  }
}
// the commit of signal s waits until every line of every shard released this iteration's stamp (acquire, system
// scope); a peer that never arrives flags spin_err after 2 s instead of hanging the GPU
__device__ __forceinline__ void peer_wait_lines(const DevParams& P, int s) {
  int total = 0;
  for (int g = 0; g < P.line_G; ++g) {
    int lo, hi;
    line_shard_range(P.r, P.line_G, g, &lo, &hi);
    total += 1 + (hi - lo);
  }
  for (int t = threadIdx.x; t < total; t += blockDim.x) {
    int g = 0, n = t;
    for (;; ++g) {
      int lo, hi;
      line_shard_range(P.r, P.line_G, g, &lo, &hi);
      if (n < 1 + (hi - lo)) break;
      n -= 1 + (hi - lo);
    }
    const int32_t* f = P.stamp_local + ((int64_t)g * P.L_ref + n) * P.batch + s;
    long long t0 = 0;
    for (int it = 0;; ++it) {
      int got;
      asm volatile("ld.acquire.sys.global.b32 %0, [%1];" : "=r"(got) : "l"(f) : "memory");
      if (got == P.peer_epoch) break;
      if ((it & 255) == 0) {
        long long now;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
        if (it == 0) t0 = now;
        else if (now - t0 > 2000000000ll) { atomicExch(P.spin_err, 1); break; }
      }
      __nanosleep(128);
    }
  }
  __threadfence();
  __syncthreads();
}

// multi-prime speculation (reading R26): tag of the set that updated a registry entry this iteration, and whether
// set gs must skip entry e (an earlier set of the same iteration updated it); never for G = 1
__device__ __forceinline__ int32_t spec_tag(int32_t iter, int gs) { return (iter << 4) | gs; }
__device__ __forceinline__ bool spec_skip(const DevParams& P, int s, int e, int32_t iter, int gs) {
  if (P.spec_G <= 1) return false;
  const int32_t t = P.spec_touch[(int64_t)s * P.k + e];
  return (t >> 4) == iter && (t & 15) < gs;
}

// a7 commit of one signal (steps 2-5 of decode_kernel<kDecCommit>, k_decode.cu): candidates of line 0 and the
// pass flags / coordinates of every line from the records, bin consistency, accepted list, registry update
// (hash lookup, R[v] += a, new entries and their C rows, prune) and the signal's state.  Runs in the commit
// kernel (one CTA per signal) or, fused, in the last FFT CTA of the signal to finish (k_fft.cu).
// smem: decode_smem_bytes(P, p); any blockDim that is a multiple of 32.
template <bool SPEC>   // SPEC: spec_G > 1 (R26); false compiles the single-set commit of Alg. 2
static __device__ __forceinline__ void commit_signal(const DevParams& P, int32_t iter, int s, unsigned char* smem_raw) {
  // multi-prime speculation (reading R26, spec_G > 1): slots s0 .. s0 + G - 1 hold one signal, each with its own
  // prime of the iteration and its own copy of the registry; every slot merges all G record sets in prime order
  // into its copy (so the copies stay identical), skipping keys an earlier set of the iteration updated
  const int G = SPEC ? P.spec_G : 1;
  const int s0 = SPEC && !P.spec_dist ? s - s % G : s;
  const int p_own = P.st_p[s];
  const int nR0 = P.st_nR[s];
  int nR = nR0;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int r = P.r;
  const int lvl = P.st_lvl[s];
  const int64_t Ev = P.lvl_E[lvl];
  double* mag = reinterpret_cast<double*>(smem_raw);             // arrays of >= k* entries: p >= c k* for every set
  int* cand = reinterpret_cast<int*>(mag + p_own);
  int* flag = cand + p_own;
  int* accl = flag + p_own;
  int* found = accl + P.k;
  int* scratch = found + P.k;
  int64_t* accv = P.acc_v + (int64_t)s * r * P.k;               // [r][k], column = candidate index
  int nc = 0, total = 0;
  if (P.peer_mode) peer_wait_lines(P, s);        // the records of every shard's lines are in (fused exchange)
  int na_all = 0, nR_final = nR0;
  for (int gs = 0; gs < G; ++gs) {
    // the set: this slot's own records (Alg. 2), a sibling slot's (R26 on one GPU) or rank gs's from the
    // all-gathered records with their tail (R26 distributed)
    const int sr = SPEC && !P.spec_dist ? s0 + gs : s;
    const int64_t* sbase = SPEC && P.spec_dist ? P.rec_recv + ((int64_t)gs * P.batch + s) * P.rec_words
                                               : P.rec_recv + (int64_t)sr * P.rec_words;
    const int32_t* stail = reinterpret_cast<const int32_t*>(sbase + P.spec_tail);
    const bool dist = SPEC && P.spec_dist;
    const int p = dist ? stail[1] : P.st_p[sr], m = dist ? stail[2] : P.st_m[sr];
    const int32_t* cand_src = dist ? stail + 4 : P.rec_cand + (int64_t)sr * P.k;
    const double* f0_src = dist ? reinterpret_cast<const double*>(sbase + P.spec_tail + 2 + (P.k + 1) / 2)
                                : reinterpret_cast<const double*>(P.rec_f0 + (int64_t)sr * P.k);
    // ---- commit: candidates of line 0, flags ANDed over the line shards, coordinates unpacked ----
    nc = dist ? stail[0] : P.rec_nc[sr];
    for (int ci = tid; ci < nc; ci += blockDim.x) {
      cand[ci] = cand_src[ci];
      int f = 1;
      if (SPEC) f = reinterpret_cast<const int32_t*>(sbase)[ci];
      else
        for (int g = 0; g < P.line_G; ++g)
          f &= reinterpret_cast<const int32_t*>(P.rec_recv + ((int64_t)g * P.batch + sr) * P.rec_words)[ci];
      flag[ci] = f;
    }
    __syncthreads();
    if (SPEC || P.line_G == 1) {
      // one shard holds every axis: its record already is the [r][k] coordinate array
      accv = const_cast<int64_t*>(sbase) + P.rec_fw;   // read-only below
    } else {
      for (int g = 0; g < P.line_G; ++g) {
        int glo, ghi;
        line_shard_range(r, P.line_G, g, &glo, &ghi);
        const int64_t* rv = P.rec_recv + ((int64_t)g * P.batch + sr) * P.rec_words + P.rec_fw;
        for (int nn = 0; nn < ghi - glo; ++nn)
          for (int ci = tid; ci < nc; ci += blockDim.x)
            if (flag[ci]) accv[(int64_t)(glo + nn) * P.k + ci] = rv[(int64_t)nn * P.k + ci];
      }
      __syncthreads();
    }
    if (P.extra & 2) {
      for (int ci = tid; ci < nc; ci += blockDim.x)
        if (flag[ci] && mod_pos64(accv[(int64_t)m * P.k + ci], p) != cand[ci]) flag[ci] = 0;
      __syncthreads();
    }

    // ---- 3. accepted list in ascending b ----
    {
      const int per = (nc + blockDim.x - 1) / blockDim.x;
      const int i0 = tid * per, i1 = min(nc, i0 + per);
      int c3 = 0;
      for (int i = i0; i < i1; ++i) c3 += flag[i];
      int pos3 = block_excl_scan(c3, scratch, &total);
      for (int i = i0; i < i1; ++i)
        if (flag[i]) accl[pos3++] = i;
      __syncthreads();
    }
    const int na = total;

    // ---- 4. registry update: R[v] += a ----
    int64_t* vreg = P.v_all + (int64_t)s * r * P.kk + P.k;   // column e = registry entry e
    double2* areg = P.a_reg + (int64_t)s * P.k;
    uint64_t* khash = P.key_hash + (int64_t)s * P.k;
    int* htab = P.htab + (int64_t)s * P.H;
    const int Hm = P.H - 1;
    // 4a. lookup, warp per accepted candidate: key hash with lanes along the coordinates, linear probing,
    //     full-key compare by ballot (the arrays of the select are free in the commit: mag -> hashes, flag -> new)
    //     Short keys (r < 128) go thread per candidate instead (the same hash by a plain loop).
    uint64_t* hsh = reinterpret_cast<uint64_t*>(mag);
    const int nwarps = (int)(blockDim.x >> 5);
    const bool wide = r >= 128;
    if (!wide) {
      for (int t = tid; t < na; t += blockDim.x) {
        const int ci = accl[t];
        uint64_t h = 0;
        for (int n = 0; n < r; ++n) h ^= key_term(accv[(int64_t)n * P.k + ci], n);
        int slot = (int)(h & (uint64_t)Hm);
        int fe = -1;
        for (;;) {
          const int e1 = htab[slot];
          if (e1 == 0) break;
          const int e = e1 - 1;
          if (khash[e] == h) {
            bool eq = true;
            for (int n = 0; n < r && eq; ++n) eq = vreg[(int64_t)n * P.kk + e] == accv[(int64_t)n * P.k + ci];
            if (eq) { fe = e; break; }
          }
          slot = (slot + 1) & Hm;
        }
        found[t] = fe;
        hsh[t] = h;
      }
    }
    for (int t = warp; wide && t < na; t += nwarps) {
      const int ci = accl[t];
      const uint64_t h = key_hash_warp(accv + ci, P.k, r, lane);
      int slot = (int)(h & (uint64_t)Hm);
      int fe = -1;
      for (;;) {
        const int e1 = htab[slot];
        if (e1 == 0) break;
        const int e = e1 - 1;
        if (khash[e] == h) {
          bool eq = true;
          for (int n = lane; n < r; n += 32) eq = eq && vreg[(int64_t)n * P.kk + e] == accv[(int64_t)n * P.k + ci];
          if (__all_sync(0xffffffffu, eq)) { fe = e; break; }
        }
        slot = (slot + 1) & Hm;
      }
      if (lane == 0) { found[t] = fe; hsh[t] = h; }
    }
    __syncthreads();
    // 4a'. without the bin-consistency check (extra_checks bit 1 off) two accepted candidates of one iteration can
    //      decode to the same key; Alg. 2 l.30 processes them in ascending b, so the first creates the entry and
    //      the later ones accumulate into it.  A key absent from R is marked a duplicate of the FIRST earlier
    //      accepted candidate with the same key (found = -2 - t'); so is a key of R found twice (its += a would
    //      race in 4b).  With the check on, equal keys have equal
    //      v_m mod p = b, so distinct candidates never collide and this pass is skipped.
    //      The first occurrence comes from a table of key-hash groups (open addressing over the freed cand array,
    //      slot = 1 + the smallest t of the group by atomicMin); a group whose smallest t holds a different key
    //      (a 64-bit hash collision) falls back to the scan over every earlier t.
    bool any_dup = false;
    if (!(P.extra & 2)) {
      int* gtab = cand;                                   // p_own ints; p_own >= c k* >= 2 na
      int tsz = 1;
      while (2 * tsz <= p_own) tsz *= 2;
      const int gm = tsz - 1;
      for (int i = tid; i < tsz; i += blockDim.x) gtab[i] = 0;
      __syncthreads();
      for (int t = tid; t < na; t += blockDim.x) {
        const uint64_t h = hsh[t];
        int slot = (int)((h ^ (h >> 32)) & (uint64_t)gm);
        for (;;) {
          int o = reinterpret_cast<volatile int*>(gtab)[slot];
          if (o == 0) {
            o = atomicCAS(&gtab[slot], 0, t + 1);
            if (o == 0) break;
          }
          if (hsh[o - 1] == h) {                          // every occupant of a slot has this slot's hash
            atomicMin(&gtab[slot], t + 1);
            break;
          }
          slot = (slot + 1) & gm;
        }
      }
      __syncthreads();
      int dup_local = 0;
      for (int t = tid; t < na; t += blockDim.x) {
        const uint64_t h = hsh[t];
        int slot = (int)((h ^ (h >> 32)) & (uint64_t)gm);
        while (hsh[gtab[slot] - 1] != h) slot = (slot + 1) & gm;
        const int first = gtab[slot] - 1;
        int dup = -1;
        if (first != t) {
          const int ci = accl[t], c1 = accl[first];
          bool eq = found[first] == found[t];
          if (eq && found[t] < 0)
            for (int n = 0; n < r && eq; ++n) eq = accv[(int64_t)n * P.k + c1] == accv[(int64_t)n * P.k + ci];
          if (eq) dup = first;
          else if (found[t] >= 0) {                       // hash collision: the scan (an existing key found twice)
            for (int t2 = 0; t2 < t && dup < 0; ++t2)
              if (found[t2] == found[t]) dup = t2;
          } else {
            for (int t2 = 0; t2 < t && dup < 0; ++t2) {
              if (found[t2] >= 0 || hsh[t2] != h) continue;
              const int c2 = accl[t2];
              bool e2 = true;
              for (int n = 0; n < r && e2; ++n) e2 = accv[(int64_t)n * P.k + c2] == accv[(int64_t)n * P.k + ci];
              if (e2) dup = t2;
            }
          }
        }
        flag[t] = dup;
        dup_local |= dup >= 0;
      }
      any_dup = __syncthreads_or(dup_local) != 0;
      if (any_dup) {
        for (int t = tid; t < na; t += blockDim.x)
          if (flag[t] >= 0) found[t] = -2 - flag[t];
        __syncthreads();
      }
    }
    // 4b. R[v] += a for found keys; new keys get entries nR + rank in ascending-b order (deterministic)
    int n_new;
    {
      const int per = (na + blockDim.x - 1) / blockDim.x;
      const int t0 = tid * per, t1 = min(na, t0 + per);
      int c4 = 0;
      for (int t = t0; t < t1; ++t) c4 += found[t] == -1;
      int rank = block_excl_scan(c4, scratch, &total);
      n_new = min(total, P.k - nR);
      for (int t = t0; t < t1; ++t) {
        const int ci = accl[t];
        const double2 f0 = make_double2(f0_src[2 * ci], f0_src[2 * ci + 1]);   // F_0 at the candidate (the FFT's line-0 CTA)
        const double2 a = make_double2(f0.x / (double)p, f0.y / (double)p);    // Eq. (7): a = F_0 / p
        if (found[t] >= 0) {
          const int e = found[t];
          if (!(SPEC && spec_skip(P, s, e, iter, gs))) {
            areg[e] = make_double2(areg[e].x + a.x, areg[e].y + a.y);
            if (SPEC) P.spec_touch[(int64_t)s * P.k + e] = spec_tag(iter, gs);
          }
          flag[t] = 0;
        } else if (found[t] == -1) {
          const int e = nR + rank++;
          if (e >= P.k) {                                   // capacity k (R26: several primes' false accepts)
            flag[t] = 0;
            continue;
          }
          areg[e] = a;
          khash[e] = hsh[t];
          if (SPEC) P.spec_touch[(int64_t)s * P.k + e] = spec_tag(iter, gs);
          found[t] = e;
          flag[t] = 1;
        } else {
          flag[t] = 0;                                      // duplicate: accumulated below, in ascending b
        }
      }
    }
    __syncthreads();
    if (any_dup) {
      if (tid == 0)
        for (int t = 0; t < na; ++t) {
          if (found[t] >= -1) continue;
          const int e = found[-2 - found[t]];             // the entry its first occurrence created
          found[t] = e;
          if (e < 0 || (SPEC && spec_skip(P, s, e, iter, gs))) continue;   // first occurrence dropped / key of an earlier set
          const int ci = accl[t];
          const double2 f0 = make_double2(f0_src[2 * ci], f0_src[2 * ci + 1]);
          areg[e] = make_double2(areg[e].x + f0.x / (double)p, areg[e].y + f0.y / (double)p);
          found[t] = e;
        }
      __syncthreads();
    }
    // 4c. new entries: key row and hash-table insert (warp per entry with lanes along the coordinates for long
    //     keys, thread per entry otherwise)
    if (!wide) {
      // key rows: items (entry, 8 axes) with the entries along the threads (coalesced record reads), the
      // 8 loads of an item issued before its stores
      const int rch = (r + 7) / 8;
      for (int it = tid; it < na * rch; it += blockDim.x) {
        const int t = it % na, n0 = (it / na) * 8;
        if (!flag[t]) continue;
        const int ci = accl[t], e = found[t];
        int64_t v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = n0 + u < r ? accv[(int64_t)(n0 + u) * P.k + ci] : 0;
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (n0 + u < r) vreg[(int64_t)(n0 + u) * P.kk + e] = v[u];
      }
      for (int t = tid; t < na; t += blockDim.x) {
        if (!flag[t]) continue;
        const int e = found[t];
        int slot = (int)(hsh[t] & (uint64_t)Hm);
        while (atomicCAS(&htab[slot], 0, e + 1) != 0) slot = (slot + 1) & Hm;
      }
    }
    for (int t = warp; wide && t < na; t += nwarps) {
      if (!flag[t]) continue;
      const int ci = accl[t], e = found[t];
      for (int n = lane; n < r; n += 32) vreg[(int64_t)n * P.kk + e] = accv[(int64_t)n * P.k + ci];
      if (lane == 0) {
        int slot = (int)(hsh[t] & (uint64_t)Hm);
        while (atomicCAS(&htab[slot], 0, e + 1) != 0) slot = (slot + 1) & Hm;
      }
    }
    __syncthreads();
    const int nR_new = nR + n_new;

    // prune test (only touched entries can have changed): after the last set, over every set's touched entries
    const bool last = gs == G - 1;
    int small = 0;
    for (int t = tid; !SPEC && t < na; t += blockDim.x) {
      if (found[t] < 0) continue;
      const double2 a = areg[found[t]];
      small |= hypot(a.x, a.y) < P.prune;
    }
    for (int e = tid; SPEC && last && e < nR_new; e += blockDim.x) {
      if (P.spec_touch[(int64_t)s * P.k + e] >> 4 != iter) continue;
      const double2 a = areg[e];
      small |= hypot(a.x, a.y) < P.prune;
    }
    const int any_small = __syncthreads_or(small);
    double2* Creg = P.C_all + ((int64_t)s * P.kk + P.k) * P.Lp;
    if (SPEC) {
      // R26: the rows of every set's touched entries once, after the last set, from the registry's key rows
      // (crow_kernel over a list in ascending entry order, or here when a prune follows / few rows)
      if (last) {
        const int per = (nR_new + blockDim.x - 1) / blockDim.x;
        const int e0 = tid * per, e1 = min(nR_new, e0 + per);
        int ct = 0;
        for (int e = e0; e < e1; ++e) ct += P.spec_touch[(int64_t)s * P.k + e] >> 4 == iter;
        int tt = 0;
        int pos = block_excl_scan(ct, scratch, &tt);
        __syncthreads();
        int* tl = accl;                                   // free after the last set: the touched list
        for (int e = e0; e < e1; ++e)
          if (P.spec_touch[(int64_t)s * P.k + e] >> 4 == iter) tl[pos++] = e;
        __syncthreads();
        if (P.crow_mode && !any_small) {
          for (int t = tid; t < tt; t += blockDim.x) P.crow_list[(int64_t)s * P.k + t] = tl[t];
          const int nit = ((tt + 31) / 32) * P.crow_nl;
          if (tid == 0) scratch[0] = nit > 0 ? atomicAdd(&P.ctrl[5], nit) : 0;
          __syncthreads();
          const int base = scratch[0];
          for (int i = tid; i < nit; i += blockDim.x)
            P.crow_items[base + i] = make_int4(s, i / P.crow_nl, i % P.crow_nl, tt);
        } else {
          const int64_t* vk = P.v_all + (int64_t)s * r * P.kk + P.k;
          for (int it = tid; it < tt * P.Lp; it += blockDim.x) {
            const int t = it % tt, n = it / tt;
            const int e = tl[t];
            const double2 a = areg[e];
            double2 c = make_double2(0.0, 0.0);
            if (n == 0) c = make_double2(-a.x, -a.y);
            else if (n < P.L) {
              const double2 lf = line_factor_exact(vk[(int64_t)(P.line_lo + n - 1) * P.kk + e], Ev);
              c = make_double2(-(a.x * lf.x - a.y * lf.y), -(a.x * lf.y + a.y * lf.x));
            }
            Creg[(int64_t)e * P.Lp + n] = c;
          }
        }
      }
    } else if (P.crow_mode && !any_small) {
      // the rows go to crow_kernel (GPU-wide): the touched entries in ascending b and this signal's work items
      for (int t = tid; t < na; t += blockDim.x) P.crow_list[(int64_t)s * P.k + t] = found[t];
      const int nit = ((na + 31) / 32) * P.crow_nl;
      if (tid == 0) scratch[0] = nit > 0 ? atomicAdd(&P.ctrl[5], nit) : 0;
      __syncthreads();
      const int base = scratch[0];
      for (int i = tid; i < nit; i += blockDim.x) P.crow_items[base + i] = make_int4(s, i / P.crow_nl, i % P.crow_nl, na);
    } else {
      // C rows of touched entries: C[k+e][0] = -a_e, C[k+e][1+n] = -a_e e^{2 pi i (v_{e,n} mod E)/E}.  Items
      // (entry, 8 lines) with the entries along the threads; v from the record (a touched entry's key equals
      // its candidate's coordinates), coalesced, the 8 loads of an item in flight together
      const int lch = (P.Lp + 7) / 8;
      const bool by_items = 2 * na * lch >= (int)blockDim.x;  // else too few items: warp per entry, lanes along the row
      for (int t = warp; !by_items && t < na; t += nwarps) {
        const int e = found[t], ci = accl[t];
        if (e < 0) continue;                                // dropped (capacity)
        const double2 a = areg[e];
        for (int n = lane; n < P.Lp; n += 32) {
          double2 c;
          if (n == 0) c = make_double2(-a.x, -a.y);
          else if (n < P.L) {
            const double2 lf = line_factor_exact(accv[(int64_t)(P.line_lo + n - 1) * P.k + ci], Ev);
            c = make_double2(-(a.x * lf.x - a.y * lf.y), -(a.x * lf.y + a.y * lf.x));
          } else c = make_double2(0.0, 0.0);
          Creg[(int64_t)e * P.Lp + n] = c;
        }
      }
      for (int it = tid; by_items && it < na * lch; it += blockDim.x) {
        const int t = it % na, n0 = (it / na) * 8;
        const int e = found[t], ci = accl[t];
        if (e < 0) continue;                                // dropped (capacity)
        const double2 a = areg[e];
        int64_t v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int n = n0 + u;
          v[u] = (n >= 1 && n < P.L) ? accv[(int64_t)(P.line_lo + n - 1) * P.k + ci] : 0;
        }
        double2* row = Creg + (int64_t)e * P.Lp;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int n = n0 + u;
          if (n >= P.Lp) break;
          double2 c;
          if (n == 0) c = make_double2(-a.x, -a.y);
          else if (n < P.L) {
            const double2 lf = line_factor_exact(v[u], Ev);
            c = make_double2(-(a.x * lf.x - a.y * lf.y), -(a.x * lf.y + a.y * lf.x));
          } else c = make_double2(0.0, 0.0);
          row[n] = c;
        }
      }
    }
    nR_final = nR_new;
    if (any_small) {
      // rare path: order-preserving compaction by warp 0, then rebuild the hash table
      __syncthreads();                                    // the C rows above are in before warp 0 moves them
      if (warp == 0) {
        int wpos = 0;
        for (int e = 0; e < nR_new; ++e) {
          const double2 a = areg[e];
          const bool keep = !(hypot(a.x, a.y) < P.prune);
          if (keep) {
            if (wpos != e) {
              for (int n = lane; n < r; n += 32) vreg[(int64_t)n * P.kk + wpos] = vreg[(int64_t)n * P.kk + e];
              for (int n = lane; n < P.Lp; n += 32) Creg[(int64_t)wpos * P.Lp + n] = Creg[(int64_t)e * P.Lp + n];
              if (lane == 0) { areg[wpos] = a; khash[wpos] = khash[e]; }
            }
            ++wpos;
          }
          __syncwarp();
        }
        if (lane == 0) scratch[0] = wpos;
      }
      __syncthreads();
      nR_final = scratch[0];
      for (int i = tid; i < P.H; i += blockDim.x) htab[i] = 0;
      __syncthreads();
      for (int e = tid; e < nR_final; e += blockDim.x) {
        int slot = (int)(khash[e] & (uint64_t)Hm);
        while (atomicCAS(&htab[slot], 0, e + 1) != 0) slot = (slot + 1) & Hm;
      }
      __syncthreads();
    }
    nR = nR_final;
    na_all += na;
    __syncthreads();
  }
  const int p = p_own, na = na_all;

  // ---- 5. state ----
  if (tid == 0) {
    const int K = P.k + (P.literal ? nR0 : 0);
    P.st_nR[s] = nR_final;
    int stall = na == 0 ? P.st_stall[s] + 1 : 0;
    P.st_samples[s] += (int64_t)(r + 1) * p;              // f evaluations of all shards (reading C22)
    P.st_cmacs[s] += (int64_t)P.L * p * K;
    if (P.i8_iter) P.st_cmacs_i8[s] += (int64_t)P.L * p * K;
    P.st_fftw[2 * s] += (double)P.L * p * log2((double)p);
    {
      const double Mb = (double)P.fft_M[P.st_M[s]];        // the Bluestein size the FFT ran
      P.st_fftw[2 * s + 1] += (double)P.L * Mb * log2(Mb);
    }
    P.st_iters[s] = iter;
    if (s == 0 && iter <= kLogIters) {
      P.st_log[2 * (iter - 1)] = p;
      P.st_log[2 * (iter - 1) + 1] = na;
    }
    int st = ST_RUN;
    if (nR_final >= P.k) {
      st = SFFT_OK;
    } else if (stall >= P.stall_limit) {
      // C19 / R23: no progress for stall_limit iterations -> next tilt level (Alg. 3) if another iteration may run
      if (lvl + 1 < P.n_levels && iter < P.max_iter) {
        P.st_lvl[s] = lvl + 1;
        P.st_retilt[s] = 1;
        stall = 0;
      } else {
        st = SFFT_PARTIAL;
      }
    } else if (iter >= P.max_iter) {
      st = SFFT_PARTIAL;
    }
    P.st_stall[s] = stall;
    P.st_status[s] = st;
  }
}


}  // namespace sfft
