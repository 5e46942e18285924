// k_decode.cu -- SURVEY 8(a) rows a2 (per-iteration setup), a5 (select), a6 (collision test +
// decode) and a7 (registry update), Algorithm 2 l.6-10 and l.18-34.
//
// setup_kernel  : k* = k - |R|, p = i-th prime >= max(2, c k*) (l.8, reading R10), m = i mod r (R9)
// (the select of line 0 and the per-line collision test + decode run fused in the FFT epilogue, k_fft.cu)
// decode_kernel<kDecCommit> : one CTA per signal.
//   2. records  : candidates of line 0, pass flags ANDed over the lines (and line shards), coordinates
//   2b.         : bin consistency (D_m v) = b mod p (R13)
//   3. compact  : accepted candidates in ascending b (block prefix sum)
//   4. registry : R[v] += F_0[b]/p (R14) through an open-addressing hash of the r-long key,
//                 new entries appended in ascending-b order (deterministic), their C rows
//                 (-a e^{2 pi i v_n / E}) written for the next iteration's residual; prune (R15)
//   5. state    : |R|, stall counter (R16), samples (R18), status
// decode_kernel<kDecStage> : teacher-forced stage entry point (select + test + decode of given lines).
#include <algorithm>

#include "decode_common.cuh"

namespace sfft {

// ------------------------------------------------------------------ setup
__device__ int ith_prime_at_least(const DevParams& P, int x, int i) {
  if (x < 2) x = 2;
  if (x >= P.n_pfirst) return -1;          // beyond the largest prime
  const int idx = P.pfirst[x] + i - 1;     // first index with primes[idx] >= x, then the i-th
  return idx < P.n_primes ? P.primes[idx] : -1;
}

__global__ void setup_kernel(DevParams P, int32_t iter, int32_t seq) {
  pdl_wait();
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s < P.batch && P.st_status[s] == ST_RUN) {
    const int nR = P.st_nR[s];
    const int kstar = P.k - nR;
    P.st_retilt[s] = 0;
    const int il = P.st_il[s] + 1;                         // counter of the current level (= iter without a switch)
    P.st_il[s] = il;
    // prime counter: il (Alg. 2 l.8); with G-prime speculation (R26) slot s takes counter (il - 1) G + s % G + 1
    const int ic = P.spec_G <= 1 ? il : (il - 1) * P.spec_G + (P.spec_dist ? P.spec_rank : s % P.spec_G) + 1;
    int p;
    if (P.n_sched > 0) p = (int)P.sched[(ic - 1) % P.n_sched];
    else p = ith_prime_at_least(P, P.c * kstar, ic);
    if (p < 2 || p > P.p_cap) {
      P.st_status[s] = SFFT_ENOTSUP;
    } else {
      P.st_p[s] = p;
      P.st_m[s] = ic % P.r;
      P.active[atomicAdd(&P.ctrl[0], 1)] = s;
      atomicMax(&P.ctrl[1], p);
      atomicMax(&P.ctrl[2], P.k + (P.literal ? nR : 0));  // terms the exp-sum sums
    }
  }
  // the last CTA publishes (n_active, max p, max K, check word) to the host-mapped control block in one 16-byte
  // store: the host polls it instead of a device-to-host copy and an event (ctrl_mix: no system-scope fence)
  if (P.h_ctrl_map == nullptr) return;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&P.ctrl[4], 1) == (int)gridDim.x - 1) {
      volatile int32_t* c = P.ctrl;
      const int32_t v0 = c[0], v1 = c[1], v2 = c[2];
      const int32_t chk = (int32_t)((uint32_t)seq ^ ctrl_mix((uint32_t)v0, (uint32_t)v1, (uint32_t)v2));
      asm volatile("st.volatile.global.v4.s32 [%0], {%1, %2, %3, %4};" ::"l"(P.h_ctrl_map), "r"(v0), "r"(v1), "r"(v2),
                   "r"(chk) : "memory");
    }
  }
}

// P.ctrl must be zero: it alternates between two blocks, the previous iteration's prep kernel cleared this one
cudaError_t launch_setup(const DevParams& P, int32_t iter, cudaStream_t st, int32_t seq) {
  return launch_pdl(setup_kernel, dim3((P.batch + 255) / 256), dim3(256), 0, st, P, iter, seq);
}

// ------------------------------------------------------------------ decode
// dynamic smem: cand[p] int, flag[p] int, mag[p] double, accl[k] int, found[k] int, scratch[64] int
size_t decode_smem_bytes(const DevParams& P, int32_t max_p) {
  return sizeof(double) * (size_t)max_p + sizeof(int) * (2 * (size_t)max_p + 2 * (size_t)P.k + 64);
}

// kDecStage  : teacher-forced entry point -- select, test and decode the caller's lines F, output the accepted.
// kDecCommit : execute -- the fused FFT epilogue (k_fft.cu) selected the candidates of line 0 and tested every
//              line (records: pass flag, decoded coordinates); the flags of every line shard are ANDed, the
//              coordinates unpacked, then steps 2b-5 (bin consistency, accepted list, registry, state).  With
//              line sharding the records of all shards arrive by the all-gather; line 0 is
//              computed identically on every shard, so every shard applies the same registry update.
// kDecCommitSpec : the same with multi-prime speculation (R26: G record sets merged per slot), a separate
//              instantiation so that the single-set commit keeps its register budget.
enum { kDecStage = 0, kDecCommit = 1, kDecCommitSpec = 2 };

template <int MODE>
__global__ void __launch_bounds__(kDecodeThreads)
decode_kernel(DevParams P, int32_t iter, int32_t kstar_stage, int32_t* out_b, int64_t* out_v,
              double2* out_a, int32_t* out_counts) {
  pdl_wait();
  constexpr bool STAGE = MODE == kDecStage;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int s = P.active[blockIdx.x];
  if (!STAGE) {
    commit_signal<MODE == kDecCommitSpec>(P, iter, s, smem_raw);
    return;
  }
  const int p = P.st_p[s], m = P.st_m[s];
  const int nR = P.st_nR[s];
  const int kstar = STAGE ? kstar_stage : P.k - nR;
  const int tid = threadIdx.x;
  const int r = P.r;
  const int lvl = STAGE ? 0 : P.st_lvl[s];
  const int64_t Ev = P.lvl_E[lvl];
  const int64_t* lo_v = P.lvl_lo + (int64_t)lvl * r;
  const int64_t* hi_v = P.lvl_hi + (int64_t)lvl * r;

  double* mag = reinterpret_cast<double*>(smem_raw);
  int* cand = reinterpret_cast<int*>(mag + p);
  int* flag = cand + p;
  int* accl = flag + p;
  int* found = accl + P.k;
  int* scratch = found + P.k;

  const double2* F = P.lines + (int64_t)s * P.L * P.p_stride;   // line n at F + n * p_stride
  int64_t* accv = P.acc_v + (int64_t)s * r * P.k;               // [r][k], column = candidate index
  int nc = 0, total = 0;
  if (STAGE) {
    // ---- 1. select (ascending b) ----
    nc = select_candidates([&](int b) { return F[b]; }, p, kstar, P.floor_rel * (double)p, cand, mag, flag, scratch);
    // ---- 2. collision test + decode, flat over (candidate, shifted line) pairs (4 in flight per thread);
    //      a failing pair clears its candidate's flag (benign race: all writers store 0) ----
    for (int ci = tid; ci < nc; ci += blockDim.x) flag[ci] = 1;
    __syncthreads();
    const int tot = nc * r;
    for (int t0 = tid; t0 < tot; t0 += 4 * blockDim.x) {
      double2 fv[4], f0[4];
      int ci[4], n[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int t = t0 + u * blockDim.x;
        ci[u] = t < tot ? t / r : 0;
        n[u] = t < tot ? t - ci[u] * r : -1;
        const int b = cand[ci[u]];
        f0[u] = F[b];
        fv[u] = n[u] >= 0 ? F[(int64_t)(1 + n[u]) * P.p_stride + b] : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (n[u] < 0) continue;
        int64_t v = 0;
        if (test_decode(f0[u], fv[u], P.tol, Ev, P.round_tol, P.extra & 1, lo_v[n[u]], hi_v[n[u]], &v))
          accv[(int64_t)n[u] * P.k + ci[u]] = v;
        else
          flag[ci[u]] = 0;
      }
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

  if (STAGE) {
    for (int t = tid; t < na; t += blockDim.x) {
      const int ci = accl[t];
      const int b = cand[ci];
      out_b[t] = b;
      const double2 f0 = F[b];
      out_a[t] = make_double2(f0.x / (double)p, f0.y / (double)p);
      for (int n = 0; n < r; ++n) out_v[(int64_t)n * kstar + t] = accv[(int64_t)n * P.k + ci];
    }
    if (tid == 0) { out_counts[0] = nc; out_counts[1] = na; }
    return;
  }

}

// ------------------------------------------------------------------ stall fallback (reading R23)
// One CTA per signal that switched level in the last decode: the signal terms are re-projected with the
// new level's tilts (v_j = T unwrap(omega_j), Eq. (35) + Eq. (27)) and get new line factors (its E); every
// registry entry is untilted with the old level (hypo^2 division, must be exact -- entries that are not
// are dropped) and tilted with the new one, order preserved; hashes, the hash table and the registry C
// rows are rebuilt.  The level-local iteration counter restarts (Alg. 3 l.5).
__global__ void __launch_bounds__(1024) retilt_kernel(DevParams P, const int32_t* __restrict__ freqs) {
  pdl_wait();
  const int s = blockIdx.x;
  if (!P.st_retilt[s]) return;
  __shared__ int scratch[64];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  const int r = P.r, kk = P.kk;
  const int lvl = P.st_lvl[s];
  const int64_t E = P.lvl_E[lvl];
  const int64_t* Tn = P.lvl_tilts + (int64_t)lvl * P.lvl_tmax * 5;
  const int64_t* To = P.lvl_tilts + (int64_t)(lvl - 1) * P.lvl_tmax * 5;
  const int ntn = P.lvl_nt[lvl], nto = P.lvl_nt[lvl - 1];
  int64_t* vs = P.v_all + (int64_t)s * r * kk;
  double2* Cs = P.C_all + (int64_t)s * kk * P.Lp;
  // 1. signal terms (warp per term)
  for (int j = warp; j < P.k; j += nwarps) {
    const int32_t* w = freqs + ((int64_t)(P.spec_slots > 1 ? s / P.spec_slots : s) * P.k + j) * P.d;   // slot's input
    for (int q = lane; q < r; q += 32) {
      const int off = P.block_off[q], dq = P.block_dims[q];
      int64_t acc = 0, pw = 1;
      for (int t = 0; t < dq; ++t) {
        acc += (int64_t)__ldg(w + off + t) * pw;
        pw *= P.N;
      }
      vs[(int64_t)q * kk + j] = acc;
    }
    __syncwarp();
    for (int t = lane; t < ntn; t += 32) {
      const int64_t* T = Tn + 5 * t;
      const int64_t u0 = vs[T[0] * kk + j], u1 = vs[T[1] * kk + j];
      vs[T[0] * kk + j] = T[2] * u0 - T[3] * u1;
      vs[T[1] * kk + j] = T[3] * u0 + T[2] * u1;
    }
    __syncwarp();
    const double2 a = Cs[(int64_t)j * P.Lp];                       // column 0 = a_j
    for (int n = 1 + lane; n < P.L; n += 32) {
      const double2 lf = line_factor_exact(vs[(int64_t)(P.line_lo + n - 1) * kk + j], E);
      Cs[(int64_t)j * P.Lp + n] = make_double2(a.x * lf.x - a.y * lf.y, a.x * lf.y + a.y * lf.x);
    }
  }
  // 2. registry entries (warp per entry): old untilt (exact) then new tilt, into the acc_v scratch
  const int nR = P.st_nR[s];
  int64_t* vreg = vs + P.k;                                        // column e = entry e
  int64_t* sv = P.acc_v + (int64_t)s * r * P.k;                     // [r][k]
  double2* areg = P.a_reg + (int64_t)s * P.k;
  double2* sa = P.acc_a + (int64_t)s * P.k;
  int* keep = reinterpret_cast<int*>(P.wtmp + (int64_t)s * P.k * P.d);   // [k] (wrap scratch, unused until the end)
  for (int e = warp; e < nR; e += nwarps) {
    for (int q = lane; q < r; q += 32) sv[(int64_t)q * P.k + e] = vreg[(int64_t)q * kk + e];
    __syncwarp();
    int bad = 0;
    for (int t = lane; t < nto; t += 32) {
      const int64_t* T = To + 5 * t;
      const int64_t v0 = sv[T[0] * P.k + e], v1 = sv[T[1] * P.k + e];
      const int64_t b = T[2], h = T[3], c2 = T[4] * T[4];
      const int64_t n0 = b * v0 + h * v1, n1 = -h * v0 + b * v1;
      if (n0 % c2 != 0 || n1 % c2 != 0) bad = 1;
      else { sv[T[0] * P.k + e] = n0 / c2; sv[T[1] * P.k + e] = n1 / c2; }
    }
    __syncwarp();
    for (int t = lane; t < ntn; t += 32) {
      const int64_t* T = Tn + 5 * t;
      const int64_t u0 = sv[T[0] * P.k + e], u1 = sv[T[1] * P.k + e];
      sv[T[0] * P.k + e] = T[2] * u0 - T[3] * u1;
      sv[T[1] * P.k + e] = T[3] * u0 + T[2] * u1;
    }
    bad = __any_sync(0xffffffffu, bad);
    if (lane == 0) { keep[e] = !bad; sa[e] = areg[e]; }
  }
  __syncthreads();
  // 3. order-preserving compaction (block scan over chunks of the entries)
  int total = 0;
  {
    const int per = (nR + blockDim.x - 1) / blockDim.x;
    const int e0 = tid * per, e1 = min(nR, e0 + per);
    int c = 0;
    for (int e = e0; e < e1; ++e) c += keep[e];
    int pos = block_excl_scan(c, scratch, &total);
    for (int e = e0; e < e1; ++e) {
      if (!keep[e]) continue;
      uint64_t h = 0;
      for (int n = 0; n < r; ++n) {
        const int64_t v = sv[(int64_t)n * P.k + e];
        vreg[(int64_t)n * kk + pos] = v;
        h ^= key_term(v, n);
      }
      areg[pos] = sa[e];
      P.key_hash[(int64_t)s * P.k + pos] = h;
      ++pos;
    }
  }
  __syncthreads();
  // 4. hash table and registry C rows (-a_e e^{2 pi i v_{e,n} / E})
  int* htab = P.htab + (int64_t)s * P.H;
  const int Hm = P.H - 1;
  for (int i = tid; i < P.H; i += blockDim.x) htab[i] = 0;
  __syncthreads();
  for (int e = tid; e < total; e += blockDim.x) {
    int slot = (int)(P.key_hash[(int64_t)s * P.k + e] & (uint64_t)Hm);
    while (atomicCAS(&htab[slot], 0, e + 1) != 0) slot = (slot + 1) & Hm;
  }
  double2* Creg = Cs + (int64_t)P.k * P.Lp;
  for (int e = warp; e < total; e += nwarps) {
    const double2 a = areg[e];
    for (int n = lane; n < P.Lp; n += 32) {
      double2 c;
      if (n == 0) c = make_double2(-a.x, -a.y);
      else if (n < P.L) {
        const double2 lf = line_factor_exact(vreg[(int64_t)(P.line_lo + n - 1) * kk + e], E);
        c = make_double2(-(a.x * lf.x - a.y * lf.y), -(a.x * lf.y + a.y * lf.x));
      } else c = make_double2(0.0, 0.0);
      Creg[(int64_t)e * P.Lp + n] = c;
    }
  }
  if (tid == 0) {
    P.st_nR[s] = total;
    P.st_il[s] = 0;
  }
}

cudaError_t launch_retilt(const DevParams& P, int32_t batch, const int32_t* freqs, cudaStream_t st) {
  if (P.n_levels > 1 && batch > 0) return launch_pdl(retilt_kernel, dim3(batch), dim3(1024), 0, st, P, freqs);
  return cudaGetLastError();
}

cudaError_t launch_decode_commit(const DevParams& P, int32_t iter, int32_t max_p, int32_t n_active, cudaStream_t st) {
  const size_t smem = decode_smem_bytes(P, max_p);
  const auto kern = P.spec_G > 1 ? decode_kernel<kDecCommitSpec> : decode_kernel<kDecCommit>;
  cudaError_t e = ensure_smem(kern, smem);
  if (e != cudaSuccess) return e;
  // threads: ~8 (candidate, axis) records per thread (small problems: many short CTAs, e.g. C2's 1024 signals)
  const long work = (long)P.k * (P.r + 1) / 8;
  const int threads = (int)std::min<long>(kDecodeThreads, std::max<long>(128, (work + 31) / 32 * 32));
  if (n_active > 0)
    return launch_pdl(kern, dim3(n_active), dim3(threads), smem, st, P, iter, 0, nullptr, nullptr, nullptr, nullptr);
  return cudaGetLastError();
}

// C rows of the entries this iteration's commits touched (DevParams::crow_mode): work item = 32 touched entries
// (lanes) x 16 lines (4 warps x 4 lines), C[k+e][0] = -a_e, C[k+e][n] = -a_e e^{2 pi i (v_{e,n} mod E)/E} (the
// commit's own formula, line_factor_exact), staged in shared memory and stored as 256-B row segments.  The items
// are counted in ctrl[5] of the iteration's control block (zeroed by the previous iteration's table prep, which
// clears the next block; this iteration's prep clears the other one).
__global__ void __launch_bounds__(128) crow_kernel(DevParams P) {
  pdl_wait();
  __shared__ double2 tile[32][17];
  __shared__ int ent[32];
  const int n_items = P.ctrl[5];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int w = blockIdx.x; w < n_items; w += gridDim.x) {
    const int4 item = P.crow_items[w];
    const int s = item.x, t0 = item.y * 32, n0 = item.z * 16, na = item.w;
    const int64_t Ev = P.lvl_E[P.st_lvl[s]];           // the commit's level (a level switch touches no entry)
    const int t = t0 + lane;
    const int e = t < na ? P.crow_list[(int64_t)s * P.k + t] : -1;
    if (warp == 0) ent[lane] = e;
    double2 a = make_double2(0.0, 0.0);
    if (e >= 0) a = P.a_reg[(int64_t)s * P.k + e];
    const int64_t* vreg = P.v_all + (int64_t)s * P.r * P.kk + P.k;
    for (int j = warp; j < 16; j += 4) {
      const int n = n0 + j;
      double2 c = make_double2(0.0, 0.0);
      if (e >= 0 && n == 0) c = make_double2(-a.x, -a.y);
      else if (e >= 0 && n < P.L) {
        const double2 lf = line_factor_exact(vreg[(int64_t)(P.line_lo + n - 1) * P.kk + e], Ev);
        c = make_double2(-(a.x * lf.x - a.y * lf.y), -(a.x * lf.y + a.y * lf.x));
      }
      tile[lane][j] = c;
    }
    __syncthreads();
    double2* Creg = P.C_all + ((int64_t)s * P.kk + P.k) * P.Lp;
    for (int i = threadIdx.x; i < 32 * 16; i += 128) {
      const int row = i >> 4, col = i & 15;
      const int n = n0 + col, ee = ent[row];
      if (ee >= 0 && n < P.Lp) Creg[(int64_t)ee * P.Lp + n] = tile[row][col];
    }
    __syncthreads();
  }
}

cudaError_t launch_crow(const DevParams& P, int32_t grid, cudaStream_t st) {
  if (grid < 1) return cudaGetLastError();
  return launch_pdl(crow_kernel, dim3(grid), dim3(128), 0, st, P);
}

cudaError_t launch_stage_decode(const DevParams& P, int32_t kstar, int32_t* acc_b, int64_t* acc_v,
                                double* acc_a, int32_t* counts, cudaStream_t st) {
  const int max_p = (int)P.p_stride;
  const size_t smem = decode_smem_bytes(P, max_p);
  cudaError_t e = ensure_smem(decode_kernel<kDecStage>, smem);
  if (e != cudaSuccess) return e;
  decode_kernel<kDecStage><<<1, kDecodeThreads, smem, st>>>(P, 0, kstar, acc_b, acc_v,
                                                            reinterpret_cast<double2*>(acc_a), counts);
  return cudaGetLastError();
}

}  // namespace sfft
