// Generic (any-size) device paths: Bloom rows wider than 65,536 bits for the
// builder (32,768 for the TC histogram, 16,384 for the 4-clique kernel) and
// k > 256 for the MinHash / KMV builders and estimators.  The reference
// handles any plan_budget result (sketches.py:115-138: dense graphs give
// large B and k); these kernels keep the same results there, trading the
// tuned engines' register / shared-memory layouts for warp-per-row or
// warp-per-edge loops over global memory.
//
// Builders  (sketches.py:314-396): Bloom by global 64-bit atomicOr, k-Hash
//           by a thread per (vertex, hash function), 1-Hash / KMV by a
//           warp-level radix select of the k-th smallest h_0 per vertex.
// Estimators (providers.py:137-301): warp per edge; integer statistics in
//           global memory (histograms, per-match sums), fp64 KMV sums from
//           fixed-slot partials (PartialSums).
#include "pg_generic.cuh"

namespace pg {

constexpr int kGB = 256;  // block size of the generic kernels

__device__ __forceinline__ int64_t warp_id_global() {
  return ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
}
__device__ __forceinline__ int64_t warps_total() { return ((int64_t)gridDim.x * blockDim.x) >> 5; }

__device__ __forceinline__ bool g_contains(const int32_t* __restrict__ a, int64_t len, int32_t x) {
  int64_t lo = 0, hi = len;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (a[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  return lo < len && a[lo] == x;
}
__device__ __forceinline__ int g_lower_bound64(const uint64_t* __restrict__ a, int len, uint64_t x) {
  int lo = 0, hi = len;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

static int gen_grid() { return sm_count() * 8; }

// ------------------------------------------------------------ builders --

// _build_bloom_matrix (sketches.py:314-325): bit h_i(x) mod B of row v for
// every neighbour x and function i; rows zeroed by the launcher
__global__ void __launch_bounds__(kGB) gen_bloom_kernel(const int64_t* __restrict__ off,
                                                       const int32_t* __restrict__ adj, int64_t n, int bits, int b,
                                                       const uint64_t* __restrict__ seeds,
                                                       unsigned long long* __restrict__ rows) {
  const int lane = threadIdx.x & 31;
  const int64_t words = bits / 64;
  const bool pow2 = (bits & (bits - 1)) == 0;
  for (int64_t v = warp_id_global(); v < n; v += warps_total()) {
    unsigned long long* row = rows + v * words;
    for (int64_t j = off[v] + lane; j < off[v + 1]; j += 32) {
      const int32_t x = adj[j];
      for (int h = 0; h < b; ++h) {
        const uint64_t w = hash_word(seeds[h], x);
        const uint64_t p = pow2 ? (w & (uint64_t)(bits - 1)) : (w % (uint64_t)bits);
        atomicOr(row + (p >> 6), 1ull << (p & 63));
      }
    }
  }
}

__global__ void __launch_bounds__(kGB) gen_row_popcount_kernel(const unsigned long long* __restrict__ rows,
                                                              int64_t n, int64_t words, int32_t* __restrict__ ones) {
  const int lane = threadIdx.x & 31;
  for (int64_t v = warp_id_global(); v < n; v += warps_total()) {
    int c = 0;
    for (int64_t i = lane; i < words; i += 32) c += __popcll(rows[v * words + i]);
    c = __reduce_add_sync(0xffffffffu, c);
    if (lane == 0) ones[v] = c;
  }
}

int gen_build_bloom(const int64_t* off, const int32_t* adj, int64_t n, int bits, int b, const uint64_t* seeds,
                    uint64_t* rows, int32_t* ones, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(rows, 0, sizeof(uint64_t) * (size_t)n * (bits / 64), s);
  if (e != cudaSuccess) return fail(PG_ERR_CUDA, "memset: %s", cudaGetErrorString(e));
  gen_bloom_kernel<<<gen_grid(), kGB, 0, s>>>(off, adj, n, bits, b, seeds,
                                              reinterpret_cast<unsigned long long*>(rows));
  gen_row_popcount_kernel<<<gen_grid(), kGB, 0, s>>>(reinterpret_cast<const unsigned long long*>(rows), n,
                                                     bits / 64, ones);
  return check_launch("build_bloom_generic");
}

// _build_khash_matrix (sketches.py:328-343): entry i = argmin_x h_i(x); h_i
// is a bijection of x (mix64 of seed_i ^ x), so the argmin is
// unmix64(min h_i) ^ seed_i and the smaller-ID tie-break never applies
__global__ void __launch_bounds__(kGB) gen_khash_kernel(const int64_t* __restrict__ off,
                                                       const int32_t* __restrict__ adj, int64_t n, int k,
                                                       const uint64_t* __restrict__ seeds,
                                                       int32_t* __restrict__ entries) {
  const int64_t total = n * (int64_t)k;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = t / k;
    const int i = (int)(t - v * k);
    const int64_t a = off[v], e = off[v + 1];
    if (a == e) {
      entries[t] = -1;
      continue;
    }
    const uint64_t sd = seeds[i];
    uint64_t mn = ~0ull;
    for (int64_t j = a; j < e; ++j) {
      const uint64_t h = hash_word(sd, adj[j]);
      mn = h < mn ? h : mn;
    }
    entries[t] = (int32_t)(uint32_t)(unmix64(mn) ^ sd);
  }
}

int gen_build_khash(const int64_t* off, const int32_t* adj, int64_t n, int k, const uint64_t* seeds,
                    int32_t* entries, cudaStream_t s) {
  gen_khash_kernel<<<gen_grid() * 4, kGB, 0, s>>>(off, adj, n, k, seeds, entries);
  return check_launch("build_khash_generic");
}

// k-th smallest h_0 over a vertex's neighbours by MSB radix select (8-bit
// digits, a warp-private 256-bin histogram per pass); keys are distinct
// (h_0 is a bijection), so exactly `target` keys are <= the result
__device__ uint64_t gen_select_kth(const int32_t* __restrict__ nb, int64_t d, uint64_t seed0, int64_t target,
                                   unsigned* __restrict__ hist) {
  const int lane = threadIdx.x & 31;
  uint64_t prefix = 0, pmask = 0;
  int64_t rem = target;  // rank still to find inside the current prefix class
  for (int shift = 56; shift >= 0; shift -= 8) {
    for (int i = lane; i < 256; i += 32) hist[i] = 0u;
    __syncwarp();
    for (int64_t j = lane; j < d; j += 32) {
      const uint64_t h = hash_word(seed0, nb[j]);
      if ((h & pmask) == prefix) atomicAdd(hist + ((h >> shift) & 255u), 1u);
    }
    __syncwarp();
    // the digit whose cumulative count reaches rem (one lane scans)
    unsigned dig = 0;
    int64_t before = 0;
    if (lane == 0) {
      int64_t c = 0;
      for (int i = 0; i < 256; ++i) {
        if (c + hist[i] >= (uint64_t)rem) {
          dig = i;
          before = c;
          break;
        }
        c += hist[i];
      }
    }
    dig = __shfl_sync(0xffffffffu, dig, 0);
    before = __shfl_sync(0xffffffffu, before, 0);
    rem -= before;
    prefix |= (uint64_t)dig << shift;
    pmask |= 255ull << shift;
    __syncwarp();
  }
  return prefix;
}

// Bottom-k rows for any k (warp per vertex; no sorting of whole rows):
// 1-Hash (_select_bottom_k, sketches.py:346-372): the min(d, k) members of
// smallest h_0 -- those with h_0 <= the min(d,k)-th smallest key -- taken in
// ID order from the sorted adjacency.
// KMV (_build_kmv_matrix, :375-396): the first min(k, distinct) distinct unit
// values.  unit_value is monotone in h_0, so the candidates are the t
// members of smallest h_0 with t grown past k until they hold k distinct
// values (equal doubles from distinct words are rare); the candidates are
// then placed by distinct rank (O(t^2 / 32) per vertex, in the warp's
// global scratch of `cap` slots).
template <bool kKmv>
__global__ void __launch_bounds__(kGB) gen_bottomk_kernel(
    const int64_t* __restrict__ off, const int32_t* __restrict__ adj, int64_t n, int k,
    const uint64_t* __restrict__ seeds, int32_t* __restrict__ entries, double* __restrict__ values,
    int32_t* __restrict__ ranks, const int32_t* __restrict__ rank_of, int32_t* __restrict__ lengths,
    uint64_t* __restrict__ scratch, int32_t* __restrict__ scratch_x, int32_t* __restrict__ scratch_f, int64_t cap) {
  __shared__ unsigned hist_all[kGB / 32][256];
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  unsigned* hist = hist_all[threadIdx.x >> 5];
  const uint64_t seed0 = seeds[0];
  uint64_t* U = scratch + warp_id_global() * cap;    // KMV candidate unit bits
  int32_t* X = scratch_x + warp_id_global() * cap;   // their IDs
  int32_t* F = scratch_f + warp_id_global() * cap;   // repeat flags
  for (int64_t v = warp_id_global(); v < n; v += warps_total()) {
    const int32_t* nb = adj + off[v];
    const int64_t d = off[v + 1] - off[v];
    int cnt = 0;
    if (!kKmv) {
      int32_t* row = entries + v * (int64_t)k;
      const int64_t sel = d < k ? d : k;
      const uint64_t thr = d > k ? gen_select_kth(nb, d, seed0, sel, hist) : ~0ull;
      for (int64_t j0 = 0; j0 < d && cnt < sel; j0 += 32) {
        const int64_t j = j0 + lane;
        const int32_t x = j < d ? nb[j] : 0;
        const bool take = j < d && hash_word(seed0, x) <= thr;
        const unsigned m = __ballot_sync(0xffffffffu, take);
        if (take) row[cnt + __popc(m & lt)] = x;
        cnt += __popc(m);
      }
      for (int i = cnt + lane; i < k; i += 32) row[i] = -1;
    } else {
      double* row = values + v * (int64_t)k;
      int32_t* rrow = ranks ? ranks + v * (int64_t)k : nullptr;
      int64_t t = d < k ? d : k;
      int nd = 0;
      for (;;) {  // candidates: the t members of smallest h_0
        const uint64_t thr = t < d ? gen_select_kth(nb, d, seed0, t, hist) : ~0ull;
        int c = 0;
        for (int64_t j0 = 0; j0 < d; j0 += 32) {
          const int64_t j = j0 + lane;
          const int32_t x = j < d ? nb[j] : 0;
          const uint64_t h = hash_word(seed0, x);
          const bool take = j < d && h <= thr;
          const unsigned m = __ballot_sync(0xffffffffu, take);
          if (take) {
            U[c + __popc(m & lt)] = dbits(unit_value(h));
            X[c + __popc(m & lt)] = x;
          }
          c += __popc(m);
        }
        __syncwarp();
        // distinct values among the candidates (first copy by index)
        nd = 0;
        for (int i = lane; i < c; i += 32) {
          bool dup = false;
          for (int q = 0; q < i; ++q) dup |= U[q] == U[i];
          F[i] = dup;
          nd += !dup;
        }
        nd = __reduce_add_sync(0xffffffffu, nd);
        if (nd >= k || t >= d) {
          // repeats get the sign bit (unit values are positive doubles, so
          // flagged bits compare above every value); place the first copies
          // by distinct rank and keep ranks < k
          for (int i = lane; i < c; i += 32)
            if (F[i]) U[i] |= 1ull << 63;
          __syncwarp();
          for (int i = lane; i < c; i += 32) {
            const uint64_t x = U[i];
            if (x >> 63) continue;
            int r = 0;
            for (int q = 0; q < c; ++q) r += U[q] < x;
            if (r < k) {
              row[r] = bitsd(x);
              if (rrow) rrow[r] = rank_of[X[i]];
            }
          }
          break;
        }
        __syncwarp();
        t += k - nd;  // room for the repeats
        if (t > d) t = d;
        __syncwarp();
      }
      cnt = nd < k ? nd : k;
      __syncwarp();
      for (int i = cnt + lane; i < k; i += 32) {
        row[i] = __longlong_as_double((long long)kInfBits);
        if (rrow) rrow[i] = INT32_MAX;
      }
    }
    if (lane == 0) lengths[v] = cnt;
    __syncwarp();
  }
}

int gen_build_bottomk(const int64_t* off, const int32_t* adj, int64_t n, int k, const uint64_t* seeds,
                      int32_t* entries, double* values, int32_t* ranks, const int32_t* rank_of,
                      int32_t* lengths, cudaStream_t s) {
  const bool kmv = values != nullptr;
  const int grid = gen_grid();
  if (!kmv) {
    gen_bottomk_kernel<false><<<grid, kGB, 0, s>>>(off, adj, n, k, seeds, entries, nullptr, nullptr, nullptr,
                                                   lengths, nullptr, nullptr, nullptr, 0);
    return check_launch("build_onehash_generic");
  }
  // KMV candidates: up to 2k per warp (t grows past k only by the repeats)
  const int64_t cap = 2 * (int64_t)k + 64;
  const int64_t warps = (int64_t)grid * (kGB / 32);
  retain_default_pool();
  unsigned char* ws = nullptr;
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&ws), (size_t)warps * cap * 16 + 256, s);
  if (e != cudaSuccess) return fail(PG_ERR_CUDA, "scratch: %s", cudaGetErrorString(e));
  uint64_t* U = reinterpret_cast<uint64_t*>(ws);
  int32_t* X = reinterpret_cast<int32_t*>(U + warps * cap);
  int32_t* F = X + warps * cap;
  gen_bottomk_kernel<true><<<grid, kGB, 0, s>>>(off, adj, n, k, seeds, nullptr, values, ranks, rank_of, lengths,
                                                U, X, F, cap);
  cudaFreeAsync(ws, s);
  return check_launch("build_kmv_generic");
}

// ----------------------------------------------------------- estimators --

// positional (k-Hash, providers.py:197-198) or set (1-Hash, :200-203)
// matches of two entry rows, warp-cooperative, any k; warp-uniform result
__device__ __forceinline__ int gen_matches(const int32_t* __restrict__ ent, int k, bool onehash, int32_t u,
                                           int32_t v) {
  const int lane = threadIdx.x & 31;
  const int32_t* A = ent + (int64_t)u * k;
  const int32_t* B = ent + (int64_t)v * k;
  int m = 0;
  if (!onehash) {
    for (int i = lane; i < k; i += 32) {
      const int32_t a = A[i];
      m += a >= 0 && a == B[i];
    }
  } else {
    int lb = 0;  // rows are ascending IDs followed by -1 pads
    for (int i = lane; i < k; i += 32) lb += B[i] >= 0;
    lb = __reduce_add_sync(0xffffffffu, lb);
    for (int i = lane; i < k; i += 32) {
      const int32_t a = A[i];
      if (a >= 0) m += g_contains(B, lb, a);
    }
  }
  return __reduce_add_sync(0xffffffffu, m);
}

__global__ void __launch_bounds__(kGB) gen_pairs_minhash_kernel(const int32_t* __restrict__ ent, int k,
                                                               bool onehash, const int32_t* __restrict__ sizes,
                                                               const int32_t* __restrict__ us,
                                                               const int32_t* __restrict__ vs, int64_t count,
                                                               int32_t* out_count, double* out_est) {
  const int lane = threadIdx.x & 31;
  for (int64_t e = warp_id_global(); e < count; e += warps_total()) {
    const int32_t u = us[e], v = vs[e];
    const int m = gen_matches(ent, k, onehash, u, v);
    if (lane == 0) {
      if (out_count) out_count[e] = m;
      if (out_est) {
        const int32_t su = sizes[u], sv = sizes[v];
        out_est[e] = onehash && su <= k && sv <= k ? (double)m : minhash_estimate(m, k, su, sv);
      }
    }
  }
}

int gen_pairs_minhash(const int32_t* ent, int k, bool onehash, const int32_t* sizes, const int32_t* us,
                      const int32_t* vs, int64_t count, int32_t* out_count, double* out_est, cudaStream_t s) {
  gen_pairs_minhash_kernel<<<gen_grid(), kGB, 0, s>>>(ent, k, onehash, sizes, us, vs, count, out_count, out_est);
  return check_launch("pairs_minhash_generic");
}

// per match count m: edges and sum of s_u + s_v (1-Hash pairs within
// capacity add m to the verbatim sum instead), as EpiMinhashHist /
// EpiOnehash, in global memory
__global__ void __launch_bounds__(kGB) gen_tc_minhash_kernel(const int32_t* __restrict__ ent, int k, bool onehash,
                                                            const int32_t* __restrict__ sizes,
                                                            const int32_t* __restrict__ us,
                                                            const int32_t* __restrict__ vs, int64_t b, int64_t e,
                                                            unsigned long long* out_cnt,
                                                            unsigned long long* out_ssum,
                                                            unsigned long long* out_verbatim) {
  const int lane = threadIdx.x & 31;
  unsigned long long verb = 0;
  for (int64_t j = b + warp_id_global(); j < e; j += warps_total()) {
    const int32_t v = vs[j];
    if (v < 0) continue;  // padding slot
    const int32_t u = us[j];
    const int m = gen_matches(ent, k, onehash, u, v);
    if (lane == 0) {
      const int32_t su = sizes[u], sv = sizes[v];
      if (onehash && su <= k && sv <= k) {
        verb += m;
      } else {
        atomicAdd(out_cnt + m, 1ull);
        atomicAdd(out_ssum + m, (unsigned long long)((int64_t)su + sv));
      }
    }
  }
  if (lane == 0 && verb) atomicAdd(out_verbatim, verb);
}

int gen_tc_minhash(const int32_t* ent, int k, bool onehash, const int32_t* sizes, const int32_t* us,
                   const int32_t* vs, int64_t b, int64_t e, int64_t* out_cnt, int64_t* out_ssum,
                   int64_t* out_verbatim, cudaStream_t s) {
  gen_tc_minhash_kernel<<<gen_grid(), kGB, 0, s>>>(ent, k, onehash, sizes, us, vs, b, e,
                                                   reinterpret_cast<unsigned long long*>(out_cnt),
                                                   reinterpret_cast<unsigned long long*>(out_ssum),
                                                   reinterpret_cast<unsigned long long*>(out_verbatim));
  return check_launch("tc_minhash_generic");
}

// Jaccard clustering counts (EpiJaccard): out_counts = [kept Jhat >= tau,
// kept vertex_similarity >= tau, match histogram (k+1)]
__global__ void __launch_bounds__(kGB) gen_jaccard_kernel(const int32_t* __restrict__ ent, int k,
                                                         const int32_t* __restrict__ deg,
                                                         const int32_t* __restrict__ us,
                                                         const int32_t* __restrict__ vs, int64_t b, int64_t e,
                                                         int min_matches, double tau,
                                                         unsigned long long* out_counts) {
  const int lane = threadIdx.x & 31;
  unsigned long long n_hat = 0, n_sim = 0;
  for (int64_t j = b + warp_id_global(); j < e; j += warps_total()) {
    const int32_t v = vs[j];
    if (v < 0) continue;
    const int32_t u = us[j];
    const int m = gen_matches(ent, k, false, u, v);
    if (lane == 0) {
      atomicAdd(out_counts + 2 + m, 1ull);
      n_hat += m >= min_matches;
      const int32_t du = deg[u], dv = deg[v];
      const double est = minhash_estimate(m, k, du, dv);
      const double c = fmin(fmax(est, 0.0), (double)min(du, dv));
      const double denom = __dsub_rn((double)((int64_t)du + dv), c);
      const double J = denom > 0.0 ? __ddiv_rn(c, denom) : 0.0;
      n_sim += J >= tau;
    }
  }
  if (lane == 0) {
    if (n_hat) atomicAdd(out_counts + 0, n_hat);
    if (n_sim) atomicAdd(out_counts + 1, n_sim);
  }
}

int gen_jaccard_khash(const int32_t* ent, int k, const int32_t* deg, const int32_t* us, const int32_t* vs,
                      int64_t b, int64_t e, int min_matches, double tau, int64_t* out_counts, cudaStream_t s) {
  gen_jaccard_kernel<<<gen_grid(), kGB, 0, s>>>(ent, k, deg, us, vs, b, e, min_matches, tau,
                                                reinterpret_cast<unsigned long long*>(out_counts));
  return check_launch("jaccard_khash_generic");
}

// KMV (providers.py:266-301) for one edge, warp-cooperative over global
// rows of any k: common = |A & B|, union = |A| + |B| - common, and the
// max(k_eff,1)-th smallest distinct union value from each element's rank
// (its index + the other row's elements below it + 1) -- the kmv_edge
// algorithm with global lower_bounds and 32-element rounds
struct GenKmv {
  int common, uni, k_eff;
  double kth;
};

__device__ __forceinline__ GenKmv gen_kmv_edge(const uint64_t* __restrict__ vals, int k, int32_t u, int32_t v) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  const uint64_t* A = vals + (int64_t)u * k;
  const uint64_t* B = vals + (int64_t)v * k;
  int lu = 0, lv = 0;  // finite prefix lengths (+inf pads sort last)
  for (int i = lane; i < k; i += 32) {
    lu += A[i] < kInfBits;
    lv += B[i] < kInfBits;
  }
  lu = __reduce_add_sync(0xffffffffu, lu);
  lv = __reduce_add_sync(0xffffffffu, lv);
  const int k_eff = min(lu, lv);
  const int T = max(k_eff, 1);
  int common = 0, before_u = 0, before_v = 0;
  uint64_t found = 0;
  bool have = false;
  const int rounds = (max(lu, lv) + 31) / 32;
  for (int rnd = 0; rnd < rounds; ++rnd) {
    const int idx = rnd * 32 + lane;
    uint64_t a = kInfBits, bb = kInfBits;
    int ltv = 0, ltu = 0;
    bool inv = false, inu = false;
    if (idx < lu) {
      a = A[idx];
      ltv = g_lower_bound64(B, lv, a);
      inv = ltv < lv && B[ltv] == a;
    }
    if (idx < lv) {
      bb = B[idx];
      ltu = g_lower_bound64(A, lu, bb);
      inu = ltu < lu && A[ltu] == bb;
    }
    const unsigned bu = __ballot_sync(0xffffffffu, inv);
    const unsigned bv = __ballot_sync(0xffffffffu, inu);
    const int cbu = before_u + __popc(bu & lt);
    const int cbv = before_v + __popc(bv & lt);
    if (idx < lu && idx + 1 + ltv - cbu == T) { found = a; have = true; }
    if (idx < lv && !inu && idx + 1 + ltu - cbv == T) { found = bb; have = true; }
    before_u += __popc(bu);
    before_v += __popc(bv);
    common += __popc(bu);
  }
  const unsigned hm = __ballot_sync(0xffffffffu, have);
  const uint64_t c1 = __shfl_sync(0xffffffffu, found, hm ? __ffs(hm) - 1 : 0);
  GenKmv r;
  r.common = common;
  r.uni = lu + lv - common;
  r.k_eff = k_eff;
  r.kth = bitsd(hm ? c1 : min(A[0], B[0]));  // no rank-T element: merged[0]
  return r;
}

__device__ __forceinline__ double gen_kmv_estimate(const GenKmv& r, int k, int32_t isu, int32_t isv) {
  const double su = (double)isu, sv = (double)isv;
  const double ssum = __dadd_rn(su, sv);
  double raw;
  if (isu <= k && isv <= k) raw = __dsub_rn(ssum, (double)r.uni);
  else if (r.k_eff < 2) raw = (double)r.common;
  else raw = __dsub_rn(ssum, __ddiv_rn((double)(r.k_eff - 1), r.kth));
  return fmin(fmax(raw, 0.0), fmin(su, sv));  // np.clip(raw, 0, min(su, sv))
}

__global__ void __launch_bounds__(kGB) gen_pairs_kmv_kernel(const uint64_t* __restrict__ vals, int k,
                                                           const int32_t* __restrict__ sizes,
                                                           const int32_t* __restrict__ us,
                                                           const int32_t* __restrict__ vs, int64_t count,
                                                           int32_t* out_common, int32_t* out_union,
                                                           double* out_kth, double* out_est) {
  const int lane = threadIdx.x & 31;
  for (int64_t e = warp_id_global(); e < count; e += warps_total()) {
    const int32_t u = us[e], v = vs[e];
    const GenKmv r = gen_kmv_edge(vals, k, u, v);
    if (lane == 0) {
      if (out_common) out_common[e] = r.common;
      if (out_union) out_union[e] = r.uni;
      if (out_kth) out_kth[e] = r.kth;
      if (out_est) out_est[e] = gen_kmv_estimate(r, k, sizes[u], sizes[v]);
    }
  }
}

int gen_pairs_kmv(const uint64_t* vals, int k, const int32_t* sizes, const int32_t* us, const int32_t* vs,
                  int64_t count, int32_t* out_common, int32_t* out_union, double* out_kth, double* out_est,
                  cudaStream_t s) {
  gen_pairs_kmv_kernel<<<gen_grid(), kGB, 0, s>>>(vals, k, sizes, us, vs, count, out_common, out_union, out_kth,
                                                  out_est);
  return check_launch("pairs_kmv_generic");
}

// fused KMV sum: a static warp schedule, one partial per block
__global__ void __launch_bounds__(kGB) gen_tc_kmv_kernel(const uint64_t* __restrict__ vals, int k,
                                                        const int32_t* __restrict__ sizes,
                                                        const int32_t* __restrict__ us,
                                                        const int32_t* __restrict__ vs, int64_t b, int64_t e,
                                                        double* __restrict__ part) {
  __shared__ double red[kGB / 32];
  const int lane = threadIdx.x & 31;
  double acc = 0.0;
  for (int64_t j = b + warp_id_global(); j < e; j += warps_total()) {
    const int32_t v = vs[j];
    if (v < 0) continue;
    const int32_t u = us[j];
    const GenKmv r = gen_kmv_edge(vals, k, u, v);
    if (lane == 0) acc = __dadd_rn(acc, gen_kmv_estimate(r, k, sizes[u], sizes[v]));
  }
  if (lane == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < kGB / 32; ++i) t = __dadd_rn(t, red[i]);
    part[blockIdx.x] = t;
  }
}

int gen_tc_kmv(const uint64_t* vals, int k, const int32_t* sizes, const int32_t* us, const int32_t* vs,
               int64_t b, int64_t e, double* out_sum, cudaStream_t s) {
  const int grid = gen_grid();
  PartialSums ps;
  const cudaError_t ce = ps.init(s, grid);
  if (ce != cudaSuccess) return fail(PG_ERR_CUDA, "scratch: %s", cudaGetErrorString(ce));
  gen_tc_kmv_kernel<<<grid, kGB, 0, s>>>(vals, k, sizes, us, vs, b, e, ps.p);
  ps.finish(out_sum);
  return check_launch("tc_kmv_generic");
}

// Bloom TC with a global popcount histogram (rows too wide for the
// shared-memory one): EpiBloomHist semantics
__global__ void __launch_bounds__(kGB) gen_tc_bloom_kernel(const unsigned long long* __restrict__ rows, int bits,
                                                          int op, const int32_t* __restrict__ sizes,
                                                          const double* __restrict__ lut,
                                                          const int32_t* __restrict__ us,
                                                          const int32_t* __restrict__ vs, int64_t b, int64_t e,
                                                          unsigned long long* out_hist,
                                                          unsigned long long* out_sum_pos) {
  const int lane = threadIdx.x & 31;
  const int64_t words = bits / 64;
  unsigned long long sum_pos = 0;
  for (int64_t j = b + warp_id_global(); j < e; j += warps_total()) {
    const int32_t v = vs[j];
    if (v < 0) continue;
    const int32_t u = us[j];
    const unsigned long long* A = rows + (int64_t)u * words;
    const unsigned long long* B = rows + (int64_t)v * words;
    int c = 0;
    for (int64_t i = lane; i < words; i += 32) c += __popcll(op == PG_BF_OR ? (A[i] | B[i]) : (A[i] & B[i]));
    c = __reduce_add_sync(0xffffffffu, c);
    if (lane == 0) {
      if (op == PG_BF_OR) {
        const int64_t S = (int64_t)sizes[u] + sizes[v];
        if (__dsub_rn((double)S, lut[c]) > 0.0) {
          atomicAdd(out_hist + c, 1ull);
          sum_pos += S;
        }
      } else {
        atomicAdd(out_hist + c, 1ull);
      }
    }
  }
  if (lane == 0 && sum_pos) atomicAdd(out_sum_pos, sum_pos);
}

int gen_tc_bloom(const uint64_t* rows, int bits, int op, const int32_t* sizes, const double* lut,
                 const int32_t* us, const int32_t* vs, int64_t b, int64_t e, int64_t* out_hist,
                 int64_t* out_sum_pos, cudaStream_t s) {
  gen_tc_bloom_kernel<<<gen_grid(), kGB, 0, s>>>(reinterpret_cast<const unsigned long long*>(rows), bits, op,
                                                 sizes, lut, us, vs, b, e,
                                                 reinterpret_cast<unsigned long long*>(out_hist),
                                                 reinterpret_cast<unsigned long long*>(out_sum_pos));
  return check_launch("tc_bloom_generic");
}

// 4-clique Bloom (mining.py:133-154 + BloomProvider.with_set) for rows too
// wide for the shared-memory kernels: BF(C3) of each directed edge in the
// warp's global scratch row, global histogram
__global__ void __launch_bounds__(kGB) gen_4clique_bloom_kernel(
    const int64_t* __restrict__ off, const int32_t* __restrict__ adjp, const int32_t* __restrict__ src,
    const int64_t* __restrict__ edge_ids, int64_t b, int64_t e, const unsigned long long* __restrict__ rows,
    int bits, int nh, const uint64_t* __restrict__ seeds, int op, const int32_t* __restrict__ sizes,
    const double* __restrict__ lut, unsigned long long* __restrict__ scratch, unsigned long long* out_hist,
    unsigned long long* out_sum_pos, unsigned long long* out_triples) {
  const int lane = threadIdx.x & 31;
  const int64_t words = bits / 64;
  const bool pow2 = (bits & (bits - 1)) == 0;
  unsigned long long* bf = scratch + warp_id_global() * words;
  unsigned long long triples = 0, sum_pos = 0;
  for (int64_t j = b + warp_id_global(); j < e; j += warps_total()) {
    const int64_t jj = edge_ids ? edge_ids[j] : j;
    const int32_t u = src[jj], v = adjp[jj];
    const int32_t* A = adjp + off[u];
    int64_t la = off[u + 1] - off[u];
    const int32_t* Bv = adjp + off[v];
    int64_t lb = off[v + 1] - off[v];
    if (la > lb) {
      const int32_t* t = A; A = Bv; Bv = t;
      const int64_t tl = la; la = lb; lb = tl;
    }
    if (la == 0) continue;
    for (int64_t i = lane; i < words; i += 32) bf[i] = 0ull;
    __syncwarp();
    int64_t c3 = 0;
    for (int64_t base = 0; base < la; base += 32) {  // BF(C3): build_bloom over the members
      const int64_t idx = base + lane;
      const int32_t x = idx < la ? A[idx] : -1;
      const bool hit = idx < la && g_contains(Bv, lb, x);
      if (hit) {
        for (int h = 0; h < nh; ++h) {
          const uint64_t w = hash_word(seeds[h], x);
          const uint64_t p = pow2 ? (w & (uint64_t)(bits - 1)) : (w % (uint64_t)bits);
          atomicOr(bf + (p >> 6), 1ull << (p & 63));
        }
      }
      c3 += __popc(__ballot_sync(0xffffffffu, hit));
    }
    __threadfence_block();
    __syncwarp();
    if (c3 == 0) continue;
    triples += c3;
    for (int64_t base = 0; base < la; base += 32) {  // every w in C3
      const int64_t idx = base + lane;
      const int32_t x = idx < la ? A[idx] : -1;
      unsigned mask = __ballot_sync(0xffffffffu, idx < la && g_contains(Bv, lb, x));
      while (mask) {
        const int t = __ffs(mask) - 1;
        mask &= mask - 1;
        const int32_t w = __shfl_sync(0xffffffffu, x, t);
        const unsigned long long* R = rows + (int64_t)w * words;
        int c = 0;
        for (int64_t i = lane; i < words; i += 32) {
          const unsigned long long f = __ldcg(bf + i);  // the atomics' values, from L2
          c += __popcll(op == PG_BF_OR ? (R[i] | f) : (R[i] & f));
        }
        c = __reduce_add_sync(0xffffffffu, c);
        if (lane == 0) {
          if (op == PG_BF_OR) {
            const int64_t S = (int64_t)sizes[w] + c3;
            if (__dsub_rn((double)S, lut[c]) > 0.0) {
              atomicAdd(out_hist + c, 1ull);
              sum_pos += S;
            }
          } else {
            atomicAdd(out_hist + c, 1ull);
          }
        }
      }
    }
    __syncwarp();
  }
  if (lane == 0) {
    if (triples) atomicAdd(out_triples, triples);
    if (sum_pos) atomicAdd(out_sum_pos, sum_pos);
  }
}

int gen_4clique_bloom(const int64_t* off, const int32_t* adjp, const int32_t* src, const int64_t* edge_ids,
                      int64_t b, int64_t e, const uint64_t* rows, int bits, int nh, const uint64_t* seeds, int op,
                      const int32_t* sizes, const double* lut, int64_t* out_hist, int64_t* out_sum_pos,
                      int64_t* out_triples, cudaStream_t s) {
  const int grid = gen_grid();
  const int64_t warps = (int64_t)grid * (kGB / 32);
  retain_default_pool();
  unsigned long long* scratch = nullptr;
  cudaError_t ce = cudaMallocAsync(reinterpret_cast<void**>(&scratch), sizeof(uint64_t) * warps * (bits / 64), s);
  if (ce != cudaSuccess) return fail(PG_ERR_CUDA, "scratch: %s", cudaGetErrorString(ce));
  gen_4clique_bloom_kernel<<<grid, kGB, 0, s>>>(off, adjp, src, edge_ids, b, e,
                                                reinterpret_cast<const unsigned long long*>(rows), bits, nh,
                                                seeds, op, sizes, lut, scratch,
                                                reinterpret_cast<unsigned long long*>(out_hist),
                                                reinterpret_cast<unsigned long long*>(out_sum_pos),
                                                reinterpret_cast<unsigned long long*>(out_triples));
  cudaFreeAsync(scratch, s);
  return check_launch("4clique_bloom_generic");
}

}  // namespace pg
