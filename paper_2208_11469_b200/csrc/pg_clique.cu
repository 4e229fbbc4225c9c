// 4-clique counting (mining.py:133-154 four_clique_count with
// BloomProvider.with_set / ExactProvider, providers.py:164-175).
#include "pg_generic.cuh"

namespace pg {

// ---------------------------------------------------------- 4-clique ----
// Warp per directed edge (u,v): C3 = N+u & N+v by binary search of the
// shorter row in the longer (pass 1 builds BF(C3) in shared memory with the
// reference's per-set builder semantics, sketches.py:187-198), pass 2
// re-derives the members and ANDs BF+(w) with BF(C3) for every w in C3
// (providers.py:164-175).  Histogram of popcounts per block.
__device__ __forceinline__ bool gmem_contains(const int32_t* __restrict__ a, int64_t len, int32_t x) {
  int64_t lo = 0, hi = len;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (a[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  return lo < len && a[lo] == x;
}

// One directed edge (u, v) of the 4-clique count with global-memory
// membership tests (A = the shorter out-list): BF(C3) into the warp's
// shared-memory row, then every member w's BF+(w) row against it.
__device__ __forceinline__ void clique4_edge_global(const int32_t* __restrict__ A, int64_t la,
                                                    const int32_t* __restrict__ Bv, int64_t lb,
                                                    const uint64_t* __restrict__ rows, int bits, int b,
                                                    const uint64_t* seeds, int op, const int32_t* __restrict__ sizes,
                                                    const double* __restrict__ lut, uint32_t* bf, int* hist_s,
                                                    int lane, long long& triples, long long& sum_pos) {
  const int words32 = bits >> 5, words64 = bits >> 6;
  const bool pow2 = (bits & (bits - 1)) == 0;
  const uint64_t* bf64 = reinterpret_cast<const uint64_t*>(bf);
    for (int i = lane; i < words32; i += 32) bf[i] = 0u;
    __syncwarp();
    int c3 = 0;
    for (int64_t base = 0; base < la; base += 32) {  // pass 1: BF(C3)
      const int64_t idx = base + lane;
      const int32_t x = idx < la ? A[idx] : -1;
      const bool hit = idx < la && gmem_contains(Bv, lb, x);
      if (hit) {
        for (int h = 0; h < b; ++h) {
          const uint64_t hw = hash_word(seeds[h], x);
          const uint32_t p = pow2 ? (uint32_t)(hw & (uint64_t)(bits - 1)) : (uint32_t)(hw % (uint64_t)bits);
          atomicOr(&bf[p >> 5], 1u << (p & 31));
        }
      }
      c3 += __popc(__ballot_sync(0xffffffffu, hit));
    }
    __syncwarp();
    if (c3 == 0) return;
    triples += c3;
    for (int64_t base = 0; base < la; base += 32) {  // pass 2: w in C3
      const int64_t idx = base + lane;
      const int32_t x = idx < la ? A[idx] : -1;
      const bool hit = idx < la && gmem_contains(Bv, lb, x);
      unsigned mask = __ballot_sync(0xffffffffu, hit);
      while (mask) {
        const int t = __ffs(mask) - 1;
        mask &= mask - 1;
        const int32_t wv = __shfl_sync(0xffffffffu, x, t);
        const uint64_t* rw = rows + (int64_t)wv * words64;
        int cnt = 0;
        for (int i = lane; i < words64; i += 32) {
          const uint64_t r = rw[i];
          cnt += __popcll(op == PG_BF_OR ? (r | bf64[i]) : (r & bf64[i]));
        }
        cnt = __reduce_add_sync(0xffffffffu, cnt);
        if (lane == 0) {
          if (op == PG_BF_OR) {
            const int64_t S = (int64_t)sizes[wv] + c3;
            if (__dsub_rn((double)S, lut[cnt]) > 0.0) {
              atomicAdd(hist_s + cnt, 1);
              sum_pos += S;
            }
          } else {
            atomicAdd(hist_s + cnt, 1);
          }
        }
      }
    }
    __syncwarp();
}

__global__ void __launch_bounds__(kBlock) clique4_bloom_kernel(
    const int64_t* __restrict__ off, const int32_t* __restrict__ adjp, const int32_t* __restrict__ src,
    int64_t e_begin, int64_t e_end, const uint64_t* __restrict__ rows, int bits, int b,
    const uint64_t* __restrict__ seeds_dev, int op, const int32_t* __restrict__ sizes,
    const double* __restrict__ lut, int64_t* out_hist, int64_t* out_sum_pos, int64_t* out_triples,
    const int64_t* __restrict__ edge_ids) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int words32 = bits >> 5;
  int* hist_s = reinterpret_cast<int*>(smem_raw);                                   // bits+1
  uint64_t* seeds = reinterpret_cast<uint64_t*>(smem_raw + ((bits + 1) * 4 + 15) / 16 * 16);  // 64
  uint32_t* bf_all = reinterpret_cast<uint32_t*>(seeds + 64);                       // warps * words32
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t* bf = bf_all + w * words32;
  for (int i = threadIdx.x; i <= bits; i += blockDim.x) hist_s[i] = 0;
  for (int i = threadIdx.x; i < b; i += blockDim.x) seeds[i] = seeds_dev[i];
  __syncthreads();
  long long triples = 0, sum_pos = 0;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t j = e_begin + (int64_t)blockIdx.x * (blockDim.x >> 5) + w; j < e_end; j += nwarps) {
    const int64_t jj = edge_ids ? edge_ids[j] : j;  // optional edge sample
    const int32_t u = src[jj], v = adjp[jj];
    const int32_t* A = adjp + off[u];
    int64_t la = off[u + 1] - off[u];
    const int32_t* Bv = adjp + off[v];
    int64_t lb = off[v + 1] - off[v];
    if (la > lb) {
      const int32_t* t = A; A = Bv; Bv = t;
      const int64_t tl = la; la = lb; lb = tl;
    }
    clique4_edge_global(A, la, Bv, lb, rows, bits, b, seeds, op, sizes, lut, bf, hist_s, lane, triples, sum_pos);
  }
  __syncthreads();
  for (int i = threadIdx.x; i <= bits; i += blockDim.x)
    if (hist_s[i]) atomicAdd(reinterpret_cast<unsigned long long*>(out_hist + i), (unsigned long long)hist_s[i]);
  if (lane == 0) {
    if (triples) atomicAdd(reinterpret_cast<unsigned long long*>(out_triples), (unsigned long long)triples);
    if (sum_pos) atomicAdd(reinterpret_cast<unsigned long long*>(out_sum_pos), (unsigned long long)sum_pos);
  }
}


// Staged 4-clique kernel for Bloom rows of 32*G bytes (bits = 256*G):
// warp per directed edge.  The longer out-list is staged in shared memory
// (when it fits kC4Cap) so the membership tests are shared-memory binary
// searches, and C3 = N+u & N+v is compacted once into shared memory (the
// global kernel above recomputes it).  BF(C3) is built in shared memory and
// each lane keeps its 32-byte slice in registers; the members are then
// processed 32/G at a time: G lanes per member, one 256-bit load of BF+(w)
// each, popcount of AND (OR) with the slice, G-lane reduction.  Edges whose
// shorter list exceeds kC4Cap take the global path.
#ifndef PG_C4_MINB
#define PG_C4_MINB 5  // 46 registers, no spills: 5.23 vs 5.39 ms at c5b (shared memory also caps at 5)
#endif
constexpr int kC4Cap = 512;
#ifndef PG_C4_DYNAMIC
#define PG_C4_DYNAMIC 1
#endif
#ifndef PG_C4_CHUNK
#define PG_C4_CHUNK 8
#endif
constexpr int64_t kC4Chunk = PG_C4_CHUNK;
#ifndef PG_C4_ROUNDS
#define PG_C4_ROUNDS 2  // member rows in flight per lane group
#endif

// lower bound by descending powers of two: the same trip count on every lane
// (floor(log2 len) + 1) and five instructions per step instead of the nine of
// a lo/hi loop (the C3 searches were 22 % of the kernel's instructions)
__device__ __forceinline__ bool smem_contains(const int32_t* a, int len, int32_t x) {
  int pos = 0;  // elements known to be < x
  for (int step = 1 << (31 - __clz(len | 1)); step > 0; step >>= 1) {
    const int p = pos + step;
    if (p <= len && a[p - 1] < x) pos = p;
  }
  return pos < len && a[pos] == x;
}

template <int G>
__global__ void __launch_bounds__(kBlock, PG_C4_MINB) clique4_bloom_staged_kernel(
    const int64_t* __restrict__ off, const int32_t* __restrict__ adjp, const int32_t* __restrict__ src,
    int64_t e_begin, int64_t e_end, const uint64_t* __restrict__ rows, int b,
    const uint64_t* __restrict__ seeds_dev, int op, const int32_t* __restrict__ sizes,
    const double* __restrict__ lut, int64_t* out_hist, int64_t* out_sum_pos, int64_t* out_triples,
    const int64_t* __restrict__ edge_ids, unsigned long long* ctr) {
  constexpr int bits = 256 * G, words32 = bits / 32, M = 32 / G;
  constexpr int kWarpInts = 2 * kC4Cap + words32;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  int* hist_s = reinterpret_cast<int*>(smem_raw);                                              // bits+1
  uint64_t* seeds = reinterpret_cast<uint64_t*>(smem_raw + ((bits + 1) * 4 + 15) / 16 * 16);  // 64
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int32_t* sB = reinterpret_cast<int32_t*>(seeds + 64) + w * kWarpInts;
  int32_t* sC = sB + kC4Cap;
  uint32_t* bf = reinterpret_cast<uint32_t*>(sC + kC4Cap);
  for (int i = threadIdx.x; i <= bits; i += blockDim.x) hist_s[i] = 0;
  for (int i = threadIdx.x; i < b; i += blockDim.x) seeds[i] = seeds_dev[i];
  __syncthreads();
  const int gl = lane % G, grp = lane / G;
  long long triples = 0, sum_pos = 0;
#if PG_C4_DYNAMIC
  // edges in dynamic chunks of kC4Chunk per warp (per-edge work spans two
  // orders of magnitude; a static stride left warps idle at the end)
  int64_t wb = 0, we = 0;
  for (;;) {
  if (!next_chunk(ctr, e_begin, e_end, kC4Chunk, wb, we)) break;
  for (int64_t j = wb; j < we; ++j) {
#else
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  {
  for (int64_t j = e_begin + (int64_t)blockIdx.x * (blockDim.x >> 5) + w; j < e_end; j += nwarps) {
#endif
    const int64_t jj = edge_ids ? edge_ids[j] : j;  // optional edge sample
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
    if (la > kC4Cap) {
      clique4_edge_global(A, la, Bv, lb, rows, bits, b, seeds, op, sizes, lut, bf, hist_s, lane, triples,
                          sum_pos);
      continue;
    }
    const bool staged = lb <= kC4Cap;
    if (staged) {
      for (int i = lane; i < lb; i += 32) sB[i] = Bv[i];
      __syncwarp();
    }
    int c3 = 0;  // C3 members compacted into sC, ascending
    for (int base = 0; base < la; base += 32) {
      const int idx = base + lane;
      const int32_t x = idx < la ? A[idx] : -1;
      const bool hit = idx < la && (staged ? smem_contains(sB, (int)lb, x) : gmem_contains(Bv, lb, x));
      const unsigned mask = __ballot_sync(0xffffffffu, hit);
      if (hit) sC[c3 + __popc(mask & ((1u << lane) - 1u))] = x;
      c3 += __popc(mask);
    }
    if (c3 == 0) {
      __syncwarp();
      continue;
    }
    triples += c3;
    for (int i = lane; i < words32; i += 32) bf[i] = 0u;
    __syncwarp();
    for (int t = lane; t < c3; t += 32) {  // BF(C3)
      const int32_t x = sC[t];
      for (int h = 0; h < b; ++h) {
        const uint32_t p = (uint32_t)(hash_word(seeds[h], x) & (uint64_t)(bits - 1));
        atomicOr(&bf[p >> 5], 1u << (p & 31));
      }
    }
    __syncwarp();
    uint32_t sl[8];  // this lane's 32-byte slice of BF(C3)
    {
      const uint4 a0 = reinterpret_cast<const uint4*>(bf)[2 * gl], a1 = reinterpret_cast<const uint4*>(bf)[2 * gl + 1];
      sl[0] = a0.x; sl[1] = a0.y; sl[2] = a0.z; sl[3] = a0.w;
      sl[4] = a1.x; sl[5] = a1.y; sl[6] = a1.z; sl[7] = a1.w;
    }
    // members in rounds of kRounds * M: the rows of a round are all requested
    // before the first is used (a row per iteration waited for every load)
    constexpr int kRounds = PG_C4_ROUNDS;
    for (int base = 0; base < c3; base += kRounds * M) {
      uint32_t r[kRounds][8];
      int32_t wv[kRounds];
      bool valid[kRounds];
#pragma unroll
      for (int q = 0; q < kRounds; ++q) {
        const int t = base + q * M + grp;
        valid[q] = t < c3;
        wv[q] = valid[q] ? sC[t] : sC[0];
        ldg256_keep(reinterpret_cast<const unsigned char*>(rows) + (int64_t)wv[q] * (bits / 8) + 32 * gl, r[q]);
      }
#pragma unroll
      for (int q = 0; q < kRounds; ++q) {
        if (q > 0 && base + q * M >= c3) break;  // warp-uniform
        int cnt = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) cnt += __popc(op == PG_BF_OR ? (r[q][i] | sl[i]) : (r[q][i] & sl[i]));
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        if (valid[q] && gl == 0) {
          if (op == PG_BF_OR) {
            const int64_t S = (int64_t)sizes[wv[q]] + c3;
            if (__dsub_rn((double)S, lut[cnt]) > 0.0) {
              atomicAdd(hist_s + cnt, 1);
              sum_pos += S;
            }
          } else {
            atomicAdd(hist_s + cnt, 1);
          }
        }
      }
    }
    __syncwarp();
  }
  }
  __syncthreads();
  for (int i = threadIdx.x; i <= bits; i += blockDim.x)
    if (hist_s[i]) atomicAdd(reinterpret_cast<unsigned long long*>(out_hist + i), (unsigned long long)hist_s[i]);
  for (int o = 16; o > 0; o >>= 1) sum_pos += __shfl_xor_sync(0xffffffffu, sum_pos, o);
  if (lane == 0) {
    if (triples) atomicAdd(reinterpret_cast<unsigned long long*>(out_triples), (unsigned long long)triples);
    if (sum_pos) atomicAdd(reinterpret_cast<unsigned long long*>(out_sum_pos), (unsigned long long)sum_pos);
  }
}

// Exact 4-clique: for w in C3, count x in N+w with x in N+u and x in N+v
// (two binary searches; C3 never materialised).
// one directed edge of the exact count with global binary searches
__device__ __forceinline__ long long clique4_exact_edge_global(const int64_t* __restrict__ off,
                                                              const int32_t* __restrict__ adjp,
                                                              const int32_t* __restrict__ A, int64_t la,
                                                              const int32_t* __restrict__ Bv, int64_t lb,
                                                              int lane) {
  long long total = 0;
  for (int64_t base = 0; base < la; base += 32) {
    const int64_t idx = base + lane;
    const int32_t x = idx < la ? A[idx] : -1;
    const bool hit = idx < la && gmem_contains(Bv, lb, x);
    unsigned mask = __ballot_sync(0xffffffffu, hit);
    while (mask) {
      const int t = __ffs(mask) - 1;
      mask &= mask - 1;
      const int32_t wv = __shfl_sync(0xffffffffu, x, t);
      const int32_t* Wr = adjp + off[wv];  // (the caller's w-row CSR)
      const int64_t lw = off[wv + 1] - off[wv];
      for (int64_t q = lane; q < lw; q += 32) {
        const int32_t y = Wr[q];
        total += gmem_contains(A, la, y) && gmem_contains(Bv, lb, y);
      }
    }
  }
  return total;
}

// Staged exact count: C3 compacted into shared memory (as the staged Bloom
// kernel), member out-degrees prefix-summed, and the flattened work
// sum_w |N+w| spread over the lanes (each lane: find its member by binary
// search in the prefix, test its entry against C3 in shared memory), so
// short rows do not idle the warp.  Edges whose shorter list exceeds kC4Cap
// take the global path.
// w rows (N(w) of ExactProvider.with_set, providers.py:117-118) come from
// (woff, wadj): the view's own CSR, or the provider's when it was built
// for another CSR (e.g. ExactProvider.for_graph: undirected N(w)).
__global__ void __launch_bounds__(kBlock) clique4_exact_kernel(
    const int64_t* __restrict__ off, const int32_t* __restrict__ adjp, const int32_t* __restrict__ src,
    int64_t e_begin, int64_t e_end, const int64_t* __restrict__ woff, const int32_t* __restrict__ wadj,
    int64_t* out_count, unsigned long long* ctr) {
  extern __shared__ __align__(16) int32_t smem_i[];  // (kBlock/32) * (3*kC4Cap + 1)
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int32_t* sB = smem_i + w * (3 * kC4Cap + 1);
  int32_t* sC = sB + kC4Cap;
  int32_t* sP = sC + kC4Cap;  // kC4Cap + 1 entries
  long long total = 0;
  // dynamic chunks of directed edges (as the Bloom kernel; the count is an integer)
  int64_t wb = 0, we = 0;
  while (next_chunk(ctr, e_begin, e_end, kC4Chunk, wb, we))
  for (int64_t j = wb; j < we; ++j) {
    const int32_t u = src[j], v = adjp[j];
    const int32_t* A = adjp + off[u];
    int64_t la = off[u + 1] - off[u];
    const int32_t* Bv = adjp + off[v];
    int64_t lb = off[v + 1] - off[v];
    if (la > lb) {
      const int32_t* t = A; A = Bv; Bv = t;
      const int64_t tl = la; la = lb; lb = tl;
    }
    if (la == 0) continue;
    if (la > kC4Cap) {
      total += clique4_exact_edge_global(woff, wadj, A, la, Bv, lb, lane);
      continue;
    }
    const bool staged = lb <= kC4Cap;
    if (staged) {
      for (int i = lane; i < lb; i += 32) sB[i] = Bv[i];
      __syncwarp();
    }
    int c3 = 0;
    for (int base = 0; base < la; base += 32) {
      const int idx = base + lane;
      const int32_t x = idx < la ? A[idx] : -1;
      const bool hit = idx < la && (staged ? smem_contains(sB, (int)lb, x) : gmem_contains(Bv, lb, x));
      const unsigned mask = __ballot_sync(0xffffffffu, hit);
      if (hit) sC[c3 + __popc(mask & ((1u << lane) - 1u))] = x;
      c3 += __popc(mask);
    }
    if (c3 == 0) {
      __syncwarp();
      continue;
    }
    __syncwarp();
    // exclusive prefix of the members' out-degrees (int: |N+w| < 2^31)
    int carry = 0;
    for (int base = 0; base < c3; base += 32) {
      const int t = base + lane;
      const int d = t < c3 ? (int)(woff[sC[t] + 1] - woff[sC[t]]) : 0;
      int inc = d;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
      }
      if (t < c3) sP[t] = carry + inc - d;
      carry += __shfl_sync(0xffffffffu, inc, 31);
    }
    if (lane == 0) sP[c3] = carry;
    __syncwarp();
    const int work = carry;
    for (int f = lane; f < work; f += 32) {
      int lo = 0, hi = c3 - 1;  // last member t with sP[t] <= f
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (sP[mid] <= f) lo = mid;
        else hi = mid - 1;
      }
      const int32_t y = wadj[woff[sC[lo]] + (f - sP[lo])];
      total += smem_contains(sC, c3, y);
    }
    __syncwarp();
  }
  for (int o = 16; o > 0; o >>= 1) total += __shfl_xor_sync(0xffffffffu, total, o);
  if (lane == 0 && total) atomicAdd(reinterpret_cast<unsigned long long*>(out_count), (unsigned long long)total);
}

}  // namespace pg

using namespace pg;

static int clique4_bloom(const int64_t* dir_off, const int32_t* dir_adj, const int32_t* src,
                         const int64_t* edge_ids, int64_t e_begin, int64_t e_end, const uint64_t* rows_plus,
                         int32_t bits, int32_t b, const uint64_t* seeds_dev, int32_t op, const int32_t* sizes,
                         const double* lut, int64_t* out_hist, int64_t* out_sum_pos, int64_t* out_triples,
                         void* stream) {
  PG_REQUIRE(bits >= 64 && bits % 64 == 0, "Bloom size must be a positive multiple of 64");
  PG_REQUIRE(b >= 1 && b <= 64, "Bloom hash count must be in [1, 64]");
  PG_REQUIRE(op == PG_BF_AND || op == PG_BF_L || op == PG_BF_OR, "op is not a Bloom estimator");
  PG_REQUIRE(0 <= e_begin && e_begin <= e_end, "bad edge range");
  PG_REQUIRE(out_hist && out_triples, "null output");
  PG_REQUIRE(op != PG_BF_OR || (sizes && lut && out_sum_pos), "BF_OR needs sizes, table and sum output");
  cudaStream_t s = as_stream(stream);
  cudaError_t ce = cudaMemsetAsync(out_hist, 0, sizeof(int64_t) * (bits + 1), s);
  if (ce == cudaSuccess) ce = cudaMemsetAsync(out_triples, 0, sizeof(int64_t), s);
  if (ce == cudaSuccess && out_sum_pos) ce = cudaMemsetAsync(out_sum_pos, 0, sizeof(int64_t), s);
  if (ce != cudaSuccess) return fail(PG_ERR_CUDA, "memset: %s", cudaGetErrorString(ce));
  if (e_end == e_begin) return PG_OK;
  PG_REQUIRE(dir_off && dir_adj && src && rows_plus && seeds_dev, "null pointer");
  if (bits > 16384)  // BF(C3) rows and histogram beyond the shared-memory kernels
    return gen_4clique_bloom(dir_off, dir_adj, src, edge_ids, e_begin, e_end, rows_plus, bits, b, seeds_dev, op,
                             sizes, lut, out_hist, out_sum_pos, out_triples, s);
  static const bool global_only = getenv("PG_C4_GLOBAL") != nullptr;
  const int G = bits % 256 == 0 ? bits / 256 : 0;
  if (!global_only && (G == 1 || G == 2 || G == 4 || G == 8 || G == 16 || G == 32)) {
    const size_t smem = ((size_t)(bits + 1) * 4 + 15) / 16 * 16 + 64 * 8 +
                        (size_t)(kBlock / 32) * (2 * kC4Cap * 4 + bits / 8);
#define PG_C4(GG)                                                                                              \
  if (G == GG) {                                                                                               \
    auto kern = clique4_bloom_staged_kernel<GG>;                                                               \
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);                        \
    const int grid = grid_cap(grid_for_kernel(kern, smem), e_end - e_begin, kBlock / 32);                     \
    ChunkCounter ctr;                                                                                          \
    if (ctr.init(s) != cudaSuccess) return fail(PG_ERR_CUDA, "chunk counter");                                 \
    kern<<<grid, kBlock, smem, s>>>(dir_off, dir_adj, src, e_begin, e_end, rows_plus, b, seeds_dev, op, sizes, \
                                    lut, out_hist, out_sum_pos, out_triples, edge_ids, ctr.p);                 \
    return check_launch("4clique_bloom");                                                                      \
  }
    PG_C4(1) PG_C4(2) PG_C4(4) PG_C4(8) PG_C4(16) PG_C4(32)
#undef PG_C4
  }
  const size_t smem = ((size_t)(bits + 1) * 4 + 15) / 16 * 16 + 64 * 8 + (size_t)(kBlock / 32) * (bits / 8);
  cudaFuncSetAttribute(clique4_bloom_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int grid = grid_cap(grid_for_kernel(clique4_bloom_kernel, smem), e_end - e_begin, kBlock / 32);
  clique4_bloom_kernel<<<grid, kBlock, smem, s>>>(dir_off, dir_adj, src, e_begin, e_end, rows_plus, bits, b,
                                                  seeds_dev, op, sizes, lut, out_hist, out_sum_pos,
                                                  out_triples, edge_ids);
  return check_launch("4clique_bloom");
}

extern "C" {

int pg_4clique_bloom(const int64_t* dir_off, const int32_t* dir_adj, const int32_t* src, int64_t e_begin,
                     int64_t e_end, const uint64_t* rows_plus, int32_t bits, int32_t b,
                     const uint64_t* seeds_dev, int32_t op, const int32_t* sizes, const double* lut,
                     int64_t* out_hist, int64_t* out_sum_pos, int64_t* out_triples, void* stream) {
  return clique4_bloom(dir_off, dir_adj, src, nullptr, e_begin, e_end, rows_plus, bits, b, seeds_dev, op,
                       sizes, lut, out_hist, out_sum_pos, out_triples, stream);
}

int pg_4clique_bloom_edges(const int64_t* dir_off, const int32_t* dir_adj, const int32_t* src,
                           const int64_t* edge_ids, int64_t count, const uint64_t* rows_plus, int32_t bits,
                           int32_t b, const uint64_t* seeds_dev, int32_t op, const int32_t* sizes,
                           const double* lut, int64_t* out_hist, int64_t* out_sum_pos, int64_t* out_triples,
                           void* stream) {
  PG_REQUIRE(count >= 0, "count must be >= 0");
  PG_REQUIRE(count == 0 || edge_ids, "null edge ids");
  return clique4_bloom(dir_off, dir_adj, src, edge_ids, 0, count, rows_plus, bits, b, seeds_dev, op, sizes,
                       lut, out_hist, out_sum_pos, out_triples, stream);
}

int pg_4clique_exact(const int64_t* dir_off, const int32_t* dir_adj, const int32_t* src, int64_t e_begin,
                     int64_t e_end, int64_t* out_count, void* stream) {
  return pg_4clique_exact_rows(dir_off, dir_adj, src, e_begin, e_end, dir_off, dir_adj, out_count, stream);
}

int pg_4clique_exact_rows(const int64_t* dir_off, const int32_t* dir_adj, const int32_t* src, int64_t e_begin,
                          int64_t e_end, const int64_t* w_off, const int32_t* w_adj, int64_t* out_count,
                          void* stream) {
  PG_REQUIRE(0 <= e_begin && e_begin <= e_end, "bad edge range");
  PG_REQUIRE(out_count, "null output");
  cudaStream_t s = as_stream(stream);
  cudaError_t ce = cudaMemsetAsync(out_count, 0, sizeof(int64_t), s);
  if (ce != cudaSuccess) return fail(PG_ERR_CUDA, "memset: %s", cudaGetErrorString(ce));
  if (e_end == e_begin) return PG_OK;
  PG_REQUIRE(dir_off && dir_adj && src && w_off && w_adj, "null pointer");
  const size_t smem = sizeof(int32_t) * (kBlock / 32) * (3 * kC4Cap + 1);
  cudaFuncSetAttribute(clique4_exact_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int grid = grid_cap(grid_for_kernel(clique4_exact_kernel, smem), e_end - e_begin, kBlock / 32);
  ChunkCounter ctr;
  if (ctr.init(s) != cudaSuccess) return fail(PG_ERR_CUDA, "chunk counter");
  clique4_exact_kernel<<<grid, kBlock, smem, s>>>(dir_off, dir_adj, src, e_begin, e_end, w_off, w_adj,
                                                  out_count, ctr.p);
  return check_launch("4clique_exact");
}

}  // extern "C"
