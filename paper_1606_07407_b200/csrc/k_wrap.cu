// k_wrap.cu -- SURVEY 8(a) row a8: back to d dimensions (Algorithm 2 l.36).
//   untilt every tilted pair: u = T^T v / hypo^2, rejecting non-integers (Alg. 3 l.38-39, reading R17)
//   wrap every block by balanced digits: digit = ((u + N/2) mod N) - N/2, u <- (u - digit)/N
//   canonical order: lexicographic by frequency vector.
// Three kernels: digits (lanes over the blocks of a registry entry), rank (one CTA per signal: a bitonic sort by
// the rows' first coordinates packed into a 64-bit key in shared memory, ties ordered by the full rows; an O(k^2)
// ranking when the keys do not fit), gather.
#include <algorithm>

#include "sfft_internal.cuh"

namespace sfft {

// floor division x / N for |x| < 2^52 via one correctly rounded FP64 division and an exact fix-up
__device__ __forceinline__ int64_t floordiv(int64_t x, int64_t N, double invN) {
  int64_t q = (int64_t)floor((double)x * invN);
  int64_t r = x - q * N;
  while (r < 0) { r += N; --q; }
  while (r >= N) { r -= N; ++q; }
  return q;
}

// G lanes (a power of two <= 32, >= r when r <= 32) per registry entry, lanes over the blocks
__global__ void wrap_digits_kernel(DevParams P, int32_t* __restrict__ bad, int G) {
  const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = (int)(gt & (G - 1));
  const int64_t gw = gt / G;
  if (gw >= (int64_t)(P.batch / P.spec_slots) * P.k) return;   // signals (R26: P.batch counts G slots each)
  const int s = (int)(gw / P.k), e = (int)(gw % P.k);
  const int sl = s * P.spec_slots;                         // the signal's (first) slot (R26: G identical copies)
  if (e >= P.st_nR[sl]) return;
  const int64_t* vreg = P.v_all + (int64_t)sl * P.r * P.kk + P.k;
  int32_t* row = P.wtmp + ((int64_t)s * P.k + e) * P.d;
  const int64_t N = P.N, h2 = N / 2;
  const double invN = 1.0 / (double)N;
  const int lgN = (N & (N - 1)) == 0 ? __ffsll(N) - 1 : -1;
  int err = 0;
  const int lvl = P.st_lvl[sl];
  const int32_t* axt = P.lvl_axt + (int64_t)lvl * P.r;
  const int64_t* tl = P.lvl_tilts + (int64_t)lvl * P.lvl_tmax * 5;
  for (int q = lane; q < P.r; q += G) {
    int64_t u = vreg[(int64_t)q * P.kk + e];
    const int at = axt[q];
    if (at >= 0) {
      const int64_t* T = tl + 5 * (at >> 1);
      const int64_t v0 = vreg[T[0] * P.kk + e], v1 = vreg[T[1] * P.kk + e];
      const int64_t b = T[2], h = T[3], c2 = T[4] * T[4];
      const int64_t num = (at & 1) ? (-h * v0 + b * v1) : (b * v0 + h * v1);
      if (num % c2 != 0) { err = 1; u = 0; }
      else u = num / c2;
    }
    const int dq = P.block_dims[q], off = P.block_off[q];
    int64_t geo = 0, pw = 1;
    for (int t = 0; t < dq; ++t) { geo += pw; pw *= N; }
    if (u < -h2 * geo || u > (h2 - 1) * geo) { err = 1; u = 0; }
    if (lgN >= 0) {
      // N = 2^lgN: floor division is an arithmetic shift, the remainder a mask (same digits)
      for (int t = 0; t < dq; ++t) {
        const int64_t x = u + h2;
        row[off + t] = (int32_t)((x & (N - 1)) - h2);  // balanced digit
        u = x >> lgN;                                  // (u - digit) / N
      }
    } else {
      for (int t = 0; t < dq; ++t) {
        const int64_t x = u + h2;
        const int64_t qn = floordiv(x, N, invN);
        row[off + t] = (int32_t)(x - qn * N - h2);    // balanced digit
        u = qn;                                        // (u - digit) / N
      }
    }
  }
  if (err) bad[s] = 1;
}

// The same digits with coalesced traffic: a CTA takes 32 entries of one signal, lanes along the entries (the reads
// vreg[q][e0 + lane] of one block q are one 256-B segment), warps along the blocks; the digit rows are staged in
// shared memory (row stride dp = d | 1 words: conflict-free) and stored as whole rows.  Used for rows up to ~380
// coordinates (48 KB of tile).
__global__ void __launch_bounds__(256) wrap_digits_tiled_kernel(DevParams P, int32_t* __restrict__ bad, int dp) {
  extern __shared__ int32_t rows[];                      // [32][dp]
  const int s = blockIdx.y, e0 = blockIdx.x * 32;
  const int sl = s * P.spec_slots;
  const int nR = P.st_nR[sl];
  if (e0 >= nR) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int e = e0 + lane;
  const bool live = e < nR;
  const int64_t* vreg = P.v_all + (int64_t)sl * P.r * P.kk + P.k;
  const int64_t N = P.N, h2 = N / 2;
  const double invN = 1.0 / (double)N;
  const int lgN = (N & (N - 1)) == 0 ? __ffsll(N) - 1 : -1;
  const int lvl = P.st_lvl[sl];
  const int32_t* axt = P.lvl_axt + (int64_t)lvl * P.r;
  const int64_t* tl = P.lvl_tilts + (int64_t)lvl * P.lvl_tmax * 5;
  int32_t* row = rows + lane * dp;
  int err = 0;
  for (int q = warp; q < P.r; q += nw) {
    int64_t u = live ? vreg[(int64_t)q * P.kk + e] : 0;
    const int at = axt[q];
    if (at >= 0 && live) {
      const int64_t* T = tl + 5 * (at >> 1);
      const int64_t v0 = vreg[T[0] * P.kk + e], v1 = vreg[T[1] * P.kk + e];
      const int64_t b = T[2], h = T[3], c2 = T[4] * T[4];
      const int64_t num = (at & 1) ? (-h * v0 + b * v1) : (b * v0 + h * v1);
      if (num % c2 != 0) { err = 1; u = 0; }
      else u = num / c2;
    }
    const int dq = P.block_dims[q], off = P.block_off[q];
    int64_t geo = 0, pw = 1;
    for (int t = 0; t < dq; ++t) { geo += pw; pw *= N; }
    if (live && (u < -h2 * geo || u > (h2 - 1) * geo)) { err = 1; u = 0; }
    for (int t = 0; t < dq; ++t) {
      const int64_t x = u + h2;
      int64_t qn;
      if (lgN >= 0) qn = x >> lgN;
      else qn = floordiv(x, N, invN);
      row[off + t] = (int32_t)(x - qn * N - h2);         // balanced digit
      u = qn;                                            // (u - digit) / N
    }
  }
  if (err) bad[s] = 1;
  __syncthreads();
  const int nrow = min(32, nR - e0);
  int32_t* out = P.wtmp + ((int64_t)s * P.k + e0) * P.d;
  for (int i = threadIdx.x; i < nrow * P.d; i += blockDim.x) {
    const int rr = i / P.d, c = i - rr * P.d;
    out[i] = rows[rr * dp + c];
  }
}

// lexicographic order of the entries -> perm[s][rank] = entry.  Rows packed into fixed-width 64-bit chunks
// (coordinate + N/2 in `bits` bits, `per` coordinates per chunk, most significant first): chunk sequences compare
// like the rows.  A bitonic sort of the entry indices (a power of two >= nR slots, padding last) first by chunk 0
// and the index -- random rows never tie there, so one chunk per row is built; when some rows tie on chunk 0
// (structured spectra, e.g. C5's collinear groups) the other chunks are built (`nchs` = nch chunks fit in shared
// memory) and the sort reruns on the whole rows; equal rows (entries flagged bad) stay by index.  Without room for
// the other chunks, runs of equal chunk 0 are insertion-sorted by the full rows from global memory.
__global__ void wrap_rank_packed_kernel(DevParams P, int32_t* __restrict__ perm, int bits, int per, int nch,
                                        int nchs) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  unsigned long long* key = reinterpret_cast<unsigned long long*>(smem_raw);    // [nchs][k]
  int* ord = reinterpret_cast<int*>(key + (size_t)nchs * P.k);                   // [power of two >= k]
  __shared__ int any_tie;
  const int s = blockIdx.x, tid = threadIdx.x;
  const int nR = P.st_nR[s * P.spec_slots];
  const int32_t* wt = P.wtmp + (int64_t)s * P.k * P.d;
  const int64_t h2 = P.N / 2;
  auto build = [&](int c0, int c1) {                         // chunks [c0, c1) of every row, chunk index fastest
    const int nc = c1 - c0;
    for (int i = tid; i < nc * nR; i += blockDim.x) {
      const int e = i / nc, c = c0 + (i - e * nc);
      const int32_t* row = wt + (int64_t)e * P.d;
      unsigned long long kv = 0;
      for (int t = 0; t < per; ++t) {
        const int l = c * per + t;
        kv = (kv << bits) | (l < P.d ? (unsigned long long)(row[l] + h2) : 0ull);
      }
      key[(int64_t)c * P.k + e] = kv;
    }
  };
  build(0, 1);
  int n = 1;
  while (n < nR) n <<= 1;
  for (int i = tid; i < n; i += blockDim.x) ord[i] = i < nR ? i : 0x7fffffff;
  if (tid == 0) any_tie = 0;
  __syncthreads();
  auto sort = [&](int ncmp) {
    auto less = [&](int a, int b) -> bool {                  // chunks [0, ncmp) then index: a before b
      if (b == 0x7fffffff) return a != 0x7fffffff;
      if (a == 0x7fffffff) return false;
      for (int c = 0; c < ncmp; ++c) {
        const unsigned long long ka = key[(int64_t)c * P.k + a], kb = key[(int64_t)c * P.k + b];
        if (ka != kb) return ka < kb;
      }
      return a < b;
    };
    for (int size = 2; size <= n; size <<= 1) {
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        for (int i = tid; i < (n >> 1); i += blockDim.x) {
          const int lo = 2 * i - (i & (stride - 1)), hi = lo + stride;
          const int a = ord[lo], b = ord[hi];
          const bool up = (lo & size) == 0;
          if (up ? less(b, a) : less(a, b)) { ord[lo] = b; ord[hi] = a; }
        }
        __syncthreads();
      }
    }
  };
  sort(1);
  if (nch > 1) {
    int tie = 0;
    for (int i = tid; i + 1 < nR; i += blockDim.x) tie |= key[ord[i]] == key[ord[i + 1]];
    if (tie) any_tie = 1;
    __syncthreads();
    if (any_tie && nchs == nch) {
      build(1, nch);
      __syncthreads();
      sort(nch);
    } else if (any_tie) {
      // a thread per run of equal chunk 0 (the run's first slot); the runs are disjoint, and a key compare
      // against a slot another thread is permuting reads the same key whichever entry it finds there
      auto row_less = [&](int a, int b) -> bool {            // full rows, then index
        const int32_t* ra = wt + (int64_t)a * P.d;
        const int32_t* rb = wt + (int64_t)b * P.d;
        for (int l = 0; l < P.d; ++l)
          if (ra[l] != rb[l]) return ra[l] < rb[l];
        return a < b;
      };
      for (int i = tid; i + 1 < nR; i += blockDim.x) {
        const unsigned long long ki = key[ord[i]];
        if ((i > 0 && key[ord[i - 1]] == ki) || key[ord[i + 1]] != ki) continue;
        int j = i + 1;
        while (j < nR && key[ord[j]] == ki) ++j;
        for (int x = i + 1; x < j; ++x) {
          const int v = ord[x];
          int y = x - 1;
          while (y >= i && row_less(v, ord[y])) { ord[y + 1] = ord[y]; --y; }
          ord[y + 1] = v;
        }
      }
    }
    __syncthreads();
  }
  for (int i = tid; i < nR; i += blockDim.x) perm[(int64_t)s * P.k + i] = ord[i];
}

// fallback when the packed rows do not fit in shared memory: keys of the first two coordinates, full
// compare from global memory on ties
__global__ void wrap_rank_kernel(DevParams P, int32_t* __restrict__ perm) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  unsigned long long* key = reinterpret_cast<unsigned long long*>(smem_raw);    // [k]
  const int s = blockIdx.x, tid = threadIdx.x;
  const int nR = P.st_nR[s * P.spec_slots];
  const int32_t* wt = P.wtmp + (int64_t)s * P.k * P.d;
  const int64_t h2 = P.N / 2;
  for (int e = tid; e < nR; e += blockDim.x) {
    const int32_t* row = wt + (int64_t)e * P.d;
    const unsigned long long k0 = (unsigned long long)(row[0] + h2);
    const unsigned long long k1 = P.d > 1 ? (unsigned long long)(row[1] + h2) : 0ull;
    key[e] = (k0 << 32) | k1;
  }
  __syncthreads();
  for (int e = tid; e < nR; e += blockDim.x) {
    const unsigned long long ke = key[e];
    const int32_t* re = wt + (int64_t)e * P.d;
    int rank = 0;
    for (int f = 0; f < nR; ++f) {
      const unsigned long long kf = key[f];
      if (kf < ke) ++rank;
      else if (kf == ke && f != e) {
        const int32_t* rf = wt + (int64_t)f * P.d;
        for (int l = 2; l < P.d; ++l)
          if (rf[l] != re[l]) { rank += rf[l] < re[l]; break; }
      }
    }
    perm[(int64_t)s * P.k + rank] = e;
  }
}

// G lanes (a power of two <= 32, >= d when d <= 32) per output row: coalesced copy of the d-vector,
// coefficient, counts and status
__global__ void wrap_gather_kernel(DevParams P, const int32_t* __restrict__ perm, const int32_t* __restrict__ bad,
                                   int32_t* __restrict__ out_freqs, double2* __restrict__ out_coeffs,
                                   int32_t* __restrict__ out_count, int32_t* __restrict__ out_status, int G,
                                   int vec) {
  const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = (int)(gt & (G - 1));
  const int64_t gw = gt / G;
  if (gw >= (int64_t)(P.batch / P.spec_slots) * P.k) return;   // signals (R26: P.batch counts G slots each)
  const int s = (int)(gw / P.k), i = (int)(gw % P.k);
  const int sl = s * P.spec_slots;
  const int nR = P.st_nR[sl];
  int32_t* of = out_freqs + ((int64_t)s * P.k + i) * P.d;
  if (i < nR) {
    const int e = perm[(int64_t)s * P.k + i];
    const int32_t* src = P.wtmp + ((int64_t)s * P.k + e) * P.d;
    if (vec) {                                          // 16-byte rows, 16-byte aligned output: int4 copies
      const int4* s4 = reinterpret_cast<const int4*>(src);
      int4* o4 = reinterpret_cast<int4*>(of);
      for (int l = lane; l < (P.d >> 2); l += G) o4[l] = s4[l];
    } else {
      for (int l = lane; l < P.d; l += G) of[l] = src[l];
    }
    if (lane == 0) out_coeffs[(int64_t)s * P.k + i] = P.a_reg[(int64_t)sl * P.k + e];
  } else {
    for (int l = lane; l < P.d; l += G) of[l] = 0;
    if (lane == 0) out_coeffs[(int64_t)s * P.k + i] = make_double2(0.0, 0.0);
  }
  if (i == 0 && lane == 0) {
    int status = P.st_status[sl];
    if (status == ST_RUN) status = SFFT_PARTIAL;
    if (bad[s]) status = SFFT_ECORRUPT;
    out_count[s] = nR;
    if (out_status) out_status[s] = status;
    P.st_status[sl] = status;
  }
}

cudaError_t launch_wrap(const DevParams& P, int32_t n_signals, int32_t* out_freqs, double* out_coeffs,
                        int32_t* out_count, int32_t* out_status, int32_t* scratch, cudaStream_t st) {
  if (n_signals <= 0) return cudaSuccess;
  int32_t* bad = scratch;                       // [n_signals]
  int32_t* perm = scratch + n_signals;          // [n_signals][k]
  cudaError_t e = cudaMemsetAsync(bad, 0, sizeof(int32_t) * n_signals, st);
  if (e != cudaSuccess) return e;
  const int64_t warps = (int64_t)n_signals * P.k;
  int G = 1;
  while (G < 32 && G < P.r) G <<= 1;
  const int dp = P.d | 1;
  const size_t tsm = sizeof(int32_t) * 32 * (size_t)dp;
  // tiles while several CTAs share an SM (C3, d = 100: wrap 0.133 -> 0.123 ms); long rows (C4, d = 1000: 128 KB
  // per tile, one CTA per SM) measured 0.12 ms slower than the lane-group kernel
  if (tsm <= 48 * 1024 && !getenv("SFFT_WRAP_LANES")) {
    e = ensure_smem(wrap_digits_tiled_kernel, tsm);
    if (e != cudaSuccess) return e;
    wrap_digits_tiled_kernel<<<dim3((unsigned)((P.k + 31) / 32), (unsigned)n_signals), 256, tsm, st>>>(P, bad, dp);
  } else {
    wrap_digits_kernel<<<(unsigned)((warps * G + 255) / 256), 256, 0, st>>>(P, bad, G);
  }
  int bits = 1;
  while (((int64_t)1 << bits) < P.N) ++bits;
  const int per = 64 / bits, nch = (P.d + per - 1) / per;
  int n2 = 1;
  while (n2 < P.k) n2 <<= 1;
  // every chunk in shared memory when it fits (the tie rerun needs them), else chunk 0 only
  const size_t full = sizeof(unsigned long long) * (size_t)nch * P.k + sizeof(int) * (size_t)n2;
  const size_t one = sizeof(unsigned long long) * (size_t)P.k + sizeof(int) * (size_t)n2;
  int optin = 0, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  const int nchs = full <= (size_t)optin ? nch : 1;
  const size_t psmem = nchs == nch ? full : one;
  if (psmem <= (size_t)optin) {
    e = ensure_smem(wrap_rank_packed_kernel, psmem);
    if (e != cudaSuccess) return e;
    // threads: the sort's n2 / 2 compare-exchanges
    const int threads = std::min(1024, std::max(64, (n2 / 2 + 31) / 32 * 32));
    wrap_rank_packed_kernel<<<n_signals, threads, psmem, st>>>(P, perm, bits, per, nch, nchs);
  } else {
    const size_t smem = sizeof(unsigned long long) * (size_t)P.k;
    e = ensure_smem(wrap_rank_kernel, smem);
    if (e != cudaSuccess) return e;
    wrap_rank_kernel<<<n_signals, 1024, smem, st>>>(P, perm);
  }
  int Gd = 1;
  // int4 copies when every row is 16-byte aligned (d % 4 == 0 and an aligned caller buffer)
  const int vec = (P.d & 3) == 0 && (reinterpret_cast<uintptr_t>(out_freqs) & 15) == 0;
  const int dw = vec ? P.d / 4 : P.d;                  // copy words per row
  while (Gd < 32 && Gd < dw) Gd <<= 1;
  wrap_gather_kernel<<<(unsigned)((warps * Gd + 255) / 256), 256, 0, st>>>(
      P, perm, bad, out_freqs, reinterpret_cast<double2*>(out_coeffs), out_count, out_status, Gd, vec);
  return cudaGetLastError();
}

}  // namespace sfft
