// (1) Per-vertex sketch builders.
//
// Reference semantics (paths under /root/reference/pkg/src/probgraph):
//   Bloom  : sketches.py:314-325 _build_bloom_matrix   (bit word%B of every
//            (neighbour, hash fn); ones = row popcount)
//   k-Hash : sketches.py:328-343 _build_khash_matrix   (argmin (h_i(x), x))
//   1-Hash : sketches.py:346-372 _select_bottom_k + _build_onehash_matrix
//            (k smallest (h_0(x), x), re-sorted by ID, -1 pad)
//   KMV    : sketches.py:375-396 _build_kmv_matrix     (k smallest DISTINCT
//            unit values, +inf pad)
//
// Design: one CTA of 8 warps walks chunks of 64 consecutive vertices.  A warp
// owns one vertex at a time and builds its sketch in shared memory or
// registers; vertices with more than kHub neighbours are deferred to the end
// of the chunk and built by the whole CTA, so R-MAT hubs (d up to 4e5) do not
// serialise on one warp.  The adjacency row is read once, coalesced.
#include <algorithm>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "pg_common.cuh"

namespace pg {  // generic builders (pg_generic.cu, declared in pg_generic.cuh)
int gen_build_bloom(const int64_t* off, const int32_t* adj, int64_t n, int bits, int b, const uint64_t* seeds,
                    uint64_t* rows, int32_t* ones, cudaStream_t s);
int gen_build_khash(const int64_t* off, const int32_t* adj, int64_t n, int k, const uint64_t* seeds,
                    int32_t* entries, cudaStream_t s);
int gen_build_bottomk(const int64_t* off, const int32_t* adj, int64_t n, int k, const uint64_t* seeds,
                      int32_t* entries, double* values, int32_t* ranks, const int32_t* rank_of,
                      int32_t* lengths, cudaStream_t s);
}  // namespace pg

namespace pg {

constexpr int kWarps = 8;
constexpr int kThreads = kWarps * 32;
constexpr int kChunk = 64;      // vertices per CTA chunk
constexpr int64_t kHub = 1024;  // degree above which the whole CTA builds

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ int warp_id() { return threadIdx.x >> 5; }

// ============================================================== Bloom ====
// smem: kWarps rows of bits/32 words (the CTA reuses warp 0's row for hubs),
// then up to 64 seeds, then the hub list.
template <bool kPow2>
__device__ __forceinline__ uint32_t bloom_pos(uint64_t w, uint32_t bits) {
  if (kPow2) return static_cast<uint32_t>(w & (bits - 1));
  return static_cast<uint32_t>(w % bits);
}

// pass 1: a warp builds a batch of R <= 32 consecutive vertices at once
// (R = 32 unless the rows would not fit shared memory).  Their adjacency runs
// are contiguous, so lanes stride over the batch's flattened entries
// (coalesced loads, no per-vertex latency chain), locate each entry's vertex
// in the batch's degree prefix (monotone per lane), and OR its b bits into
// that vertex's row in shared memory; the R rows are then one contiguous block
// of the output.  Vertices with d > kHubBloom are left to pass 2.
#ifndef PG_BB_MINB
#define PG_BB_MINB 6  // 40 registers: whole s20 build 327 -> 311 us
#endif
#ifndef PG_BH_MINB
#define PG_BH_MINB 4  // 62 registers (84 unbounded): whole s20 build 313 -> 257 us
#endif
#ifndef PG_MERGE_MIN
#define PG_MERGE_MIN 4
#endif
#ifndef PG_BK_HUB_KERNEL
#define PG_BK_HUB_KERNEL build_bottomk_hubs_buffered_kernel
#endif
#ifndef PG_BK_HUB
#define PG_BK_HUB 1024
#endif
#ifndef PG_BK_MINB
#define PG_BK_MINB 1
#endif
#ifndef PG_BKH_MINB
#define PG_BKH_MINB 1
#endif
#ifndef PG_KB_MINB
#define PG_KB_MINB 1
#endif
#ifndef PG_KBH_MINB
#define PG_KBH_MINB 1
#endif
constexpr int64_t kHubBloom = 1024;
constexpr int64_t kMidBloom = 64;  // rows above this take pass 1b (a warp each)

struct BloomBatchSmem {
  int64_t off[32];
  int pref[33];
};

template <bool kPow2>
__global__ void __launch_bounds__(kThreads, PG_BB_MINB) build_bloom_kernel(
    const int64_t* __restrict__ offsets, const int32_t* __restrict__ adj, int64_t n,
    uint32_t bits, int b, int R, const uint64_t* __restrict__ seeds_dev,
    uint64_t* __restrict__ rows, int32_t* __restrict__ ones, int32_t* __restrict__ hubs,
    int32_t* __restrict__ hub_count, unsigned long long* __restrict__ vtx_work, int32_t* __restrict__ mids,
    int32_t* __restrict__ mid_count) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const uint32_t words32 = bits >> 5;
  const uint32_t words64 = bits >> 6;
  BloomBatchSmem* meta = reinterpret_cast<BloomBatchSmem*>(smem_raw) + warp_id();
  uint64_t* seeds = reinterpret_cast<uint64_t*>(smem_raw + kWarps * sizeof(BloomBatchSmem));
  uint32_t* brows = reinterpret_cast<uint32_t*>(seeds + 64) + (size_t)warp_id() * R * words32;
  for (int i = threadIdx.x; i < b; i += kThreads) seeds[i] = seeds_dev[i];
  __syncthreads();
  const int lane = lane_id();
  // warps take R-vertex batches from a global counter (row costs vary
  // widely: a static split left most warps idle, 15% achieved occupancy)
  for (;;) {
    unsigned long long vbu = 0;
    if (lane == 0) vbu = atomicAdd(vtx_work, (unsigned long long)R);
    const int64_t vb = (int64_t)__shfl_sync(0xffffffffu, vbu, 0);
    if (vb >= n) break;
    const int nb = (int)((n - vb) < R ? (n - vb) : R);
    const int64_t v = vb + lane;
    const bool mine = lane < nb;
    const int64_t o = mine ? offsets[v] : 0;
    int64_t d = mine ? offsets[v + 1] - o : 0;
    const bool hub = d > kMidBloom;  // built by pass 1b (mid) or pass 2 (hub)
    if (d > kHubBloom) {
      hubs[atomicAdd(hub_count, 1)] = (int32_t)v;
      d = 0;
    } else if (hub) {
      mids[atomicAdd(mid_count, 1)] = (int32_t)v;
      d = 0;
    }
    int incl = (int)d;  // exclusive prefix of the batch's (non-hub) degrees
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, off);
      if (lane >= off) incl += y;
    }
    meta->pref[lane] = incl - (int)d;
    meta->off[lane] = o;
    if (lane == 31) meta->pref[32] = incl;
    // zero the batch rows: 64-bit granularity (R * words64 may be odd, and
    // then a warp's slot is only 8-byte aligned)
    uint64_t* brows64 = reinterpret_cast<uint64_t*>(brows);
    for (uint32_t i = lane; i < (uint32_t)R * words64; i += 32) brows64[i] = 0ull;
    __syncwarp();
    const int total = meta->pref[32];
    int j = 0;  // batch vertex of the lane's current entry (non-decreasing)
    for (int t = lane; t < total; t += 32) {
      while (meta->pref[j + 1] <= t) ++j;
      const int32_t x = adj[meta->off[j] + (t - meta->pref[j])];
      uint32_t* row = brows + j * words32;
      for (int h = 0; h < b; ++h) {
        const uint32_t p = bloom_pos<kPow2>(hash_word(seeds[h], x), bits);
        atomicOr(&row[p >> 5], 1u << (p & 31));
      }
    }
    __syncwarp();
    // the batch rows -- consecutive vertices, so one contiguous block of the
    // output, copied with 128-bit stores by all lanes (hub rows are all-zero
    // here; pass 2 ORs into them) -- and the non-hub ones (each lane its own
    // row, words read in a lane-rotated order to spread the banks)
    const uint64_t* b64 = reinterpret_cast<const uint64_t*>(brows);
    uint64_t* out = rows + vb * words64;
    const uint32_t nw = (uint32_t)nb * words64;
    if (((reinterpret_cast<uintptr_t>(out) | reinterpret_cast<uintptr_t>(b64)) & 15u) == 0) {
      const uint4* src4 = reinterpret_cast<const uint4*>(b64);
      uint4* out4 = reinterpret_cast<uint4*>(out);
      for (uint32_t i = lane; i < nw / 2; i += 32) out4[i] = src4[i];
      if ((nw & 1u) && lane == 0) out[nw - 1] = b64[nw - 1];
    } else {  // odd words64 with an odd row base (chunked builds, R == 1)
      for (uint32_t i = lane; i < nw; i += 32) out[i] = b64[i];
    }
    if (mine && !hub) {
      int c = 0;
      for (uint32_t i = 0; i < words64; ++i) c += __popcll(b64[lane * words64 + (i + lane) % words64]);
      ones[v] = c;
    }
    __syncwarp();
  }
}

// pass 1b: mid-degree vertices (kMidBloom < d <= kHubBloom), one warp each
// (the grid is sized for a warp per vertex of the range, not per batch),
// taken from a counter: a 32-vertex batch of such rows would hold up to 32K
// entries on one warp, and that tail set the duration of every chunked build
// (17% active warps).  The row is built in the warp's shared-memory slot and
// written whole (pass 1 wrote it as zeros).
template <bool kPow2>
__global__ void __launch_bounds__(kThreads, PG_BB_MINB) build_bloom_mid_kernel(
    const int64_t* __restrict__ offsets, const int32_t* __restrict__ adj, uint32_t bits, int b,
    const uint64_t* __restrict__ seeds_dev, uint64_t* __restrict__ rows, int32_t* __restrict__ ones,
    const int32_t* __restrict__ mids, const int32_t* __restrict__ mid_count, int32_t* __restrict__ mid_work) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const uint32_t words32 = bits >> 5, words64 = bits >> 6;
  uint64_t* seeds = reinterpret_cast<uint64_t*>(smem_raw);
  uint32_t* row = reinterpret_cast<uint32_t*>(seeds + 64) + (size_t)warp_id() * words32;
  for (int i = threadIdx.x; i < b; i += kThreads) seeds[i] = seeds_dev[i];
  __syncthreads();
  const int nm = *mid_count;
  const int lane = lane_id();
  for (;;) {
    int mi = 0;
    if (lane == 0) mi = atomicAdd(mid_work, 1);
    mi = __shfl_sync(0xffffffffu, mi, 0);
    if (mi >= nm) break;
    const int64_t v = mids[mi];
    const int64_t o = offsets[v], d = offsets[v + 1] - o;
    for (uint32_t i = lane; i < words32; i += 32) row[i] = 0u;
    __syncwarp();
    // four entries per lane in flight (the row is in L2/HBM: one dependent
    // load per 32 entries left the warp latency-bound)
    for (int64_t t0 = 0; t0 < d; t0 += 128) {
      int32_t x[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int64_t t = t0 + 32 * q + lane;
        x[q] = t < d ? adj[o + t] : -1;
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (x[q] < 0) continue;
        for (int h = 0; h < b; ++h) {
          const uint32_t p = bloom_pos<kPow2>(hash_word(seeds[h], x[q]), bits);
          atomicOr(&row[p >> 5], 1u << (p & 31));
        }
      }
    }
    __syncwarp();
    const uint64_t* r64 = reinterpret_cast<const uint64_t*>(row);
    int c = 0;
    for (uint32_t i = lane; i < words64; i += 32) {
      const uint64_t w = r64[i];
      rows[v * words64 + i] = w;
      c += __popcll(w);
    }
    c = __reduce_add_sync(0xffffffffu, c);
    if (lane == 0) ones[v] = c;
    __syncwarp();
  }
}

// pass 2: hub rows (zeroed by pass 1) are split into slices of
// kHubSlice entries; the grid strides over the (hub, slice) items, each CTA
// ORs its slice into a shared-memory row and then into the output row with
// 64-bit global atomics.  Pass 3 counts the hubs' ones.
constexpr int64_t kHubSlice = 2048;

template <bool kPow2>
__global__ void __launch_bounds__(kThreads, PG_BH_MINB) build_bloom_hubs_kernel(
    const int64_t* __restrict__ offsets, const int32_t* __restrict__ adj, uint32_t bits, int b,
    const uint64_t* __restrict__ seeds_dev, uint64_t* __restrict__ rows,
    const int32_t* __restrict__ hubs, const int32_t* __restrict__ hub_count) {
  extern __shared__ __align__(16) uint32_t smem[];
  __shared__ int64_t s_v[kThreads], s_o[kThreads], s_d[kThreads], s_pre[kThreads + 1];
  __shared__ int64_t s_wsum[kWarps];
  const uint32_t words32 = bits >> 5;
  const uint32_t words64 = bits >> 6;
  uint32_t* row = smem;
  uint64_t* seeds = reinterpret_cast<uint64_t*>(smem + words32 + (words32 & 1));
  for (int i = threadIdx.x; i < b; i += kThreads) seeds[i] = seeds_dev[i];
  const int nh = *hub_count;
  const int lane = lane_id(), wid = warp_id();
  int64_t item_base = 0;  // (hub, slice) items before this batch of hubs
  for (int h0 = 0; h0 < nh; h0 += kThreads) {
    // stage kThreads hubs and the exclusive prefix of their slice counts
    const int hi = h0 + threadIdx.x;
    int64_t v = 0, o = 0, d = 0;
    if (hi < nh) {
      v = hubs[hi];
      o = offsets[v];
      d = offsets[v + 1] - o;
    }
    const int64_t ns = (d + kHubSlice - 1) / kHubSlice;
    int64_t inc = ns;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, inc, off);
      if (lane >= off) inc += y;
    }
    if (lane == 31) s_wsum[wid] = inc;
    __syncthreads();
    int64_t wbase = 0;
    for (int w = 0; w < wid; ++w) wbase += s_wsum[w];
    s_v[threadIdx.x] = v;
    s_o[threadIdx.x] = o;
    s_d[threadIdx.x] = d;
    s_pre[threadIdx.x] = wbase + inc - ns;
    if (threadIdx.x == kThreads - 1) s_pre[kThreads] = wbase + inc;
    __syncthreads();
    const int64_t total = s_pre[kThreads];
    int64_t t = ((int64_t)blockIdx.x - item_base) % (int64_t)gridDim.x;
    if (t < 0) t += gridDim.x;
    for (; t < total; t += gridDim.x) {
      int lo = 0, hi2 = kThreads - 1;  // last hub j with s_pre[j] <= t
      while (lo < hi2) {
        const int mid = (lo + hi2 + 1) >> 1;
        if (s_pre[mid] <= t) lo = mid;
        else hi2 = mid - 1;
      }
      const int64_t hv = s_v[lo], ho = s_o[lo], hd = s_d[lo];
      const int64_t beg = (t - s_pre[lo]) * kHubSlice, end = min(hd, beg + kHubSlice);
      for (uint32_t i = threadIdx.x; i < words32; i += kThreads) row[i] = 0u;
      __syncthreads();
      for (int64_t j0 = beg; j0 < end; j0 += 4 * kThreads) {  // four loads in flight per thread
        int32_t x[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int64_t j = j0 + q * kThreads + threadIdx.x;
          x[q] = j < end ? adj[ho + j] : -1;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          if (x[q] < 0) continue;
          for (int h = 0; h < b; ++h) {
            const uint32_t p = bloom_pos<kPow2>(hash_word(seeds[h], x[q]), bits);
            atomicOr(&row[p >> 5], 1u << (p & 31));
          }
        }
      }
      __syncthreads();
      const uint64_t* row64 = reinterpret_cast<const uint64_t*>(row);
      for (uint32_t i = threadIdx.x; i < words64; i += kThreads) {
        const uint64_t w = row64[i];
        if (w) atomicOr(reinterpret_cast<unsigned long long*>(rows + hv * words64 + i), (unsigned long long)w);
      }
      __syncthreads();
    }
    item_base += total;
    __syncthreads();
  }
}

// pass 3: ones of the hub rows, one warp per hub
__global__ void __launch_bounds__(kThreads) bloom_hub_ones_kernel(
    const uint64_t* __restrict__ rows, uint32_t words64, int32_t* __restrict__ ones,
    const int32_t* __restrict__ hubs, const int32_t* __restrict__ hub_count) {
  const int nh = *hub_count;
  const int lane = lane_id();
  for (int hi = blockIdx.x * kWarps + warp_id(); hi < nh; hi += gridDim.x * kWarps) {
    const int64_t v = hubs[hi];
    int c = 0;
    for (uint32_t i = lane; i < words64; i += 32) c += __popcll(rows[v * words64 + i]);
    c = __reduce_add_sync(0xffffffffu, c);
    if (lane == 0) ones[v] = c;
  }
}

// ============================================================= k-Hash ====
// Lane = hash function (i = lane + 32*s).  Each lane keeps the running
// minimum of h_i(x) over the neighbour row.  For a fixed seed, h_i(x) =
// mix64(seed_i ^ x) is a bijection of x, so equal hashes mean the same ID:
// the reference's smaller-ID tie-break never fires, and the argmin is
// recovered from the minimum itself (x = unmix64(h) ^ seed_i) after the
// scan -- the loop carries one 64-bit register pair per function and a
// 64-bit compare, and IDs zero-extend so seed_i's high word stays constant.
template <int S>
__device__ __forceinline__ void khash_scan(const int32_t* __restrict__ row, int64_t beg, int64_t end,
                                           int64_t step, const uint64_t (&seed)[S],
                                           uint64_t (&best_h)[S]) {
  const int lane = lane_id();
  for (int64_t base = beg; base < end; base += step) {
    const int64_t j = base + lane;
    const uint32_t xl = j < end ? (uint32_t)row[j] : 0u;
    const int cnt = (end - base) < 32 ? (int)(end - base) : 32;
    for (int t = 0; t < cnt; ++t) {
      const uint32_t x = __shfl_sync(0xffffffffu, xl, t);
#pragma unroll
      for (int s = 0; s < S; ++s) {
        const uint64_t h = mix64(seed[s] ^ (uint64_t)x);
        best_h[s] = h < best_h[s] ? h : best_h[s];
      }
    }
  }
}

// the ID whose hash is h under `seed` (IDs are non-negative int32)
__device__ __forceinline__ int32_t khash_arg(uint64_t seed, uint64_t h) {
  return (int32_t)(uint32_t)(unmix64(h) ^ seed);
}

template <int S>
__global__ void __launch_bounds__(kThreads, PG_KB_MINB) build_khash_kernel(
    const int64_t* __restrict__ offsets, const int32_t* __restrict__ adj, int64_t n, int k,
    const uint64_t* __restrict__ seeds_dev, int32_t* __restrict__ entries, int32_t* __restrict__ hubs,
    int32_t* __restrict__ hub_count, unsigned long long* __restrict__ vtx_work) {
  const int lane = lane_id();
  uint64_t seed[S];
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const int i = lane + 32 * s;
    seed[s] = i < k ? seeds_dev[i] : 0ull;
  }
  // warps take batches of 32 consecutive vertices from a global counter
  // (degree-skewed rows make a static split leave most warps idle); the
  // batch's offsets come in with one coalesced load, broadcast by shuffles
  for (;;) {
    unsigned long long vbu = 0;
    if (lane_id() == 0) vbu = atomicAdd(vtx_work, 32ull);
    const int64_t vb = (int64_t)__shfl_sync(0xffffffffu, vbu, 0);
    if (vb >= n) break;
    const int64_t vl = vb + lane_id();
    const int64_t ol = vl < n ? offsets[vl] : 0;
    const int64_t el = vl < n ? offsets[vl + 1] : 0;
    const int nb = (int)((n - vb) < 32 ? (n - vb) : 32);
    for (int t = 0; t < nb; ++t) {
      const int64_t v = vb + t;
      const int64_t o = __shfl_sync(0xffffffffu, ol, t);
      const int64_t d = __shfl_sync(0xffffffffu, el, t) - o;
      if (d > kHub) {
        if (lane == 0) hubs[atomicAdd(hub_count, 1)] = (int32_t)v;
        continue;
      }
      uint64_t bh[S];
#pragma unroll
      for (int s = 0; s < S; ++s) bh[s] = ~0ull;
      khash_scan<S>(adj + o, 0, d, 32, seed, bh);
#pragma unroll
      for (int s = 0; s < S; ++s) {
        const int i = lane + 32 * s;
        if (i < k) entries[v * k + i] = d > 0 ? khash_arg(seed[s], bh[s]) : -1;
      }
    }
  }
}

template <int S>
__global__ void __launch_bounds__(kThreads, PG_KBH_MINB) build_khash_hubs_kernel(
    const int64_t* __restrict__ offsets, const int32_t* __restrict__ adj, int k,
    const uint64_t* __restrict__ seeds_dev, int32_t* __restrict__ entries, const int32_t* __restrict__ hubs,
    const int32_t* __restrict__ hub_count, int32_t* __restrict__ hub_work) {
  __shared__ uint64_t red_h[kWarps][32 * S];
  __shared__ int s_hi;
  const int lane = lane_id();
  uint64_t seed[S];
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const int i = lane + 32 * s;
    seed[s] = i < k ? seeds_dev[i] : 0ull;
  }
  const int nh = *hub_count;
  for (;;) {  // hubs taken from a global counter (their degrees vary widely)
    if (threadIdx.x == 0) s_hi = atomicAdd(hub_work, 1);
    __syncthreads();
    const int hi = s_hi;
    __syncthreads();
    if (hi >= nh) break;
    const int64_t v = hubs[hi];
    const int64_t o = offsets[v];
    const int64_t d = offsets[v + 1] - o;
    uint64_t bh[S];
#pragma unroll
    for (int s = 0; s < S; ++s) bh[s] = ~0ull;
    khash_scan<S>(adj + o, 32 * warp_id(), d, kThreads, seed, bh);
#pragma unroll
    for (int s = 0; s < S; ++s) red_h[warp_id()][lane + 32 * s] = bh[s];
    __syncthreads();
    for (int i = threadIdx.x; i < k; i += kThreads) {
      uint64_t h = red_h[0][i];
      for (int w = 1; w < kWarps; ++w) h = red_h[w][i] < h ? red_h[w][i] : h;
      entries[v * k + i] = khash_arg(seeds_dev[i], h);  // hubs have d > 1024
    }
    __syncthreads();
  }
}

// ===================================================== bottom-k (1-Hash, KMV)
// A warp-wide sorted list of up to 32*P 64-bit keys held in registers; lane
// L owns slots L, L+32, ...  `cnt` (warp-uniform) slots are valid.  Keys are
// unique (1-Hash: mix64 is a bijection, so distinct IDs hash apart; KMV:
// duplicates are rejected on insertion, which is the reference's dedup).
// ascending warp bitonic sort of 32 R keys; element i = lane + 32 r (R <= 2)
template <int R>
__device__ __forceinline__ void warp_bitonic_sort(uint64_t (&key)[R]) {
  const int lane = lane_id();
#pragma unroll
  for (int size = 2; size <= 32 * R; size <<= 1) {
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      uint64_t old[R];
#pragma unroll
      for (int r = 0; r < R; ++r) old[r] = key[r];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int i = lane + 32 * r;
        const bool up = (i & size) == 0;  // ascending block
        const uint64_t other = stride == 32 ? old[r ^ 1] : shfl64(old[r], lane ^ stride);
        const bool lower = (i & stride) == 0;
        const uint64_t mn = old[r] < other ? old[r] : other, mx = old[r] < other ? other : old[r];
        key[r] = (lower == up) ? mn : mx;
      }
    }
  }
}

template <int P, bool kDedup>
struct WarpBottomK {
  uint64_t key[P];
  int cnt;
  int k;

  __device__ __forceinline__ void init(int k_) {
    k = k_;
    cnt = 0;
#pragma unroll
    for (int s = 0; s < P; ++s) key[s] = ~0ull;
  }
  __device__ __forceinline__ bool full() const { return cnt >= k; }
  __device__ __forceinline__ uint64_t at(int idx) const {
    uint64_t r = 0;
#pragma unroll
    for (int s = 0; s < P; ++s) {
      const uint64_t t = shfl64(key[s], idx & 31);
      if ((idx >> 5) == s) r = t;
    }
    return r;
  }
  __device__ __forceinline__ uint64_t threshold() const { return at(k - 1); }

  __device__ __forceinline__ void insert(uint64_t c) {
    const int lane = lane_id();
    int pos = 0;
    bool dup = false;
#pragma unroll
    for (int s = 0; s < P; ++s) {
      const bool valid = lane + 32 * s < cnt;
      pos += __popc(__ballot_sync(0xffffffffu, valid && key[s] < c));
      if (kDedup) dup |= valid && key[s] == c;
    }
    if (kDedup && __any_sync(0xffffffffu, dup)) return;
    if (pos >= k) return;
    uint64_t prev[P];
#pragma unroll
    for (int s = 0; s < P; ++s) {
      const uint64_t up = shfl_up64(key[s], 1);
      const uint64_t wrap = s > 0 ? shfl64(key[s > 0 ? s - 1 : 0], 31) : 0ull;
      prev[s] = lane == 0 ? wrap : up;
    }
#pragma unroll
    for (int s = 0; s < P; ++s) {
      const int idx = lane + 32 * s;
      if (idx == pos) key[s] = c;
      else if (idx > pos) key[s] = prev[s];
    }
    cnt = min(cnt + 1, k);
  }

  // offer_merge: offer() for a full list of k = 32 P keys (P <= 2).  A
  // chunk with more than PG_MERGE_MIN keys below the threshold is merged in
  // one step instead of key by key: the chunk is warp-sorted, and with A the
  // list and C the sorted chunk padded to 32 P, min(A[i], C[32P-1-i]) holds
  // the 32 P smallest of both as a bitonic sequence, sorted by log2(32 P)
  // half-cleaner stages.  KMV lists hold distinct values: a repeat in the
  // result puts the chunk back through insert(), which rejects it.
  __device__ __forceinline__ void offer_merge(uint64_t c, bool valid) {
    const uint64_t thr = threshold();
    const bool pass = valid && c < thr;
    const unsigned mask = __ballot_sync(0xffffffffu, pass);
    if (__popc(mask) <= PG_MERGE_MIN) {
      offer_masked(c, mask);
      return;
    }
    const int lane = lane_id();
    uint64_t srt[1] = {pass ? c : ~0ull};
    warp_bitonic_sort<1>(srt);
    uint64_t old[P];
#pragma unroll
    for (int s = 0; s < P; ++s) old[s] = key[s];
    const uint64_t rev = shfl64(srt[0], 31 - lane);
    key[P - 1] = rev < key[P - 1] ? rev : key[P - 1];
    if (P == 2) {
      const uint64_t lo = key[0] < key[P - 1] ? key[0] : key[P - 1];
      const uint64_t hi = key[0] < key[P - 1] ? key[P - 1] : key[0];
      key[0] = lo;
      key[P - 1] = hi;
    }
#pragma unroll
    for (int stride = 16; stride > 0; stride >>= 1) {
#pragma unroll
      for (int s = 0; s < P; ++s) {
        const uint64_t other = shfl64(key[s], lane ^ stride);
        const bool lower = (lane & stride) == 0;
        const uint64_t mn = key[s] < other ? key[s] : other, mx = key[s] < other ? other : key[s];
        key[s] = lower ? mn : mx;
      }
    }
    if (kDedup) {
      bool dup = false;
      uint64_t carry = ~0ull;
#pragma unroll
      for (int s = 0; s < P; ++s) {
        const uint64_t prev = shfl_up64(key[s], 1);
        dup |= key[s] == (lane == 0 ? carry : prev);
        carry = shfl64(key[s], 31);
      }
      if (__any_sync(0xffffffffu, dup)) {
#pragma unroll
        for (int s = 0; s < P; ++s) key[s] = old[s];
        offer_masked(c, mask);
      }
    }
  }

  // insert the lanes of `mask` in lane order, re-filtering as the threshold drops
  __device__ __forceinline__ void offer_masked(uint64_t c, unsigned mask) {
    while (mask) {
      const int t = __ffs(mask) - 1;
      mask &= mask - 1;
      insert(shfl64(c, t));
      mask &= __ballot_sync(0xffffffffu, c < threshold());
    }
  }

  // offer one candidate per lane (valid lanes only)
  __device__ __forceinline__ void offer(uint64_t c, bool valid) {
    uint64_t thr = full() ? threshold() : ~0ull;
    bool pass_all = !full();
    unsigned mask = __ballot_sync(0xffffffffu, valid && (pass_all || c < thr));
    while (mask) {
      const int t = __ffs(mask) - 1;
      mask &= mask - 1;
      const uint64_t ct = shfl64(c, t);
      insert(ct);
      if (full()) {
        thr = threshold();
        mask &= __ballot_sync(0xffffffffu, c < thr);
      }
    }
  }
};

// Bottom-k modes: 0 1-Hash (key = hash word), 1 KMV (key = the unit value's
// IEEE bits), 2 KMV on global value ranks (key = rank_of[x], the dense rank
// of x's unit value among all vertices: same order and ties as the value
// bits, so the same selection; see pg_kmv_rank_table).
struct BottomKRank {
  const int32_t* rank_of = nullptr;       // mode 2
  const double* rank_values = nullptr;    // mode 2: value of each rank
  int32_t* ranks = nullptr;               // mode 2 output rows (INT32_MAX pad)
};

template <int kMode>
__device__ __forceinline__ uint64_t bottomk_key(uint64_t seed0, int32_t x, const BottomKRank& rk) {
  if (kMode == 2) return (uint64_t)(uint32_t)__ldg(rk.rank_of + x);
  const uint64_t w = hash_word(seed0, x);
  return kMode == 1 ? dbits(unit_value(w)) : w;
}

template <int P, int kMode>
__device__ __forceinline__ void bottomk_scan(WarpBottomK<P, kMode != 0>& L, const int32_t* __restrict__ row,
                                             int64_t beg, int64_t end, int64_t step, uint64_t seed0,
                                             const BottomKRank& rk) {
  const int lane = lane_id();
  for (int64_t base = beg; base < end; base += step) {
    const int64_t j = base + lane;
    const bool valid = j < end;
    const uint64_t c = valid ? bottomk_key<kMode>(seed0, row[j], rk) : ~0ull;
    if (P <= 2 && L.k == 32 * P && L.full()) L.offer_merge(c, valid);
    else L.offer(c, valid);
  }
}

// bottomk_scan for the CTAs that share one hub row: a warp whose list is
// full publishes its k-th key T to the CTA (shared atomicMin), and every
// warp drops candidates >= the smallest published T -- that warp already
// holds k distinct keys <= T, so none of them can reach the row's bottom-k
// (KMV: a candidate equal to T is a duplicate of a listed value).  Without
// it each warp keeps its own bottom-k of its 1/8 of the row, inserting
// ~k ln(n/8k) candidates instead of the row's ~k ln(n/k) / 8.
template <int P, int kMode>
__device__ __forceinline__ void bottomk_scan_shared(WarpBottomK<P, kMode != 0>& L,
                                                    const int32_t* __restrict__ row, int64_t beg,
                                                    int64_t end, int64_t step, uint64_t seed0,
                                                    const BottomKRank& rk, unsigned long long* s_thr) {
  const int lane = lane_id();
  uint64_t mine = ~0ull;
  for (int64_t base = beg; base < end; base += step) {
    const int64_t j = base + lane;
    const uint64_t c = j < end ? bottomk_key<kMode>(seed0, row[j], rk) : ~0ull;
    const uint64_t cta = *(volatile unsigned long long*)s_thr;
    L.offer(c, j < end && c < cta);
    if (L.full()) {
      const uint64_t t = L.threshold();
      if (t < mine) {
        mine = t;
        if (lane == 0) atomicMin(s_thr, (unsigned long long)t);
      }
    }
  }
}

// Fill a bottom-k list of k = 32 P (P <= 2) keys from k candidates at
// row[b0 + lane + stride * r] by one bitonic sort instead of k insertions.
// KMV lists hold distinct values: a repeated key (equal values of two
// neighbours) makes it return false and the caller inserts one by one.
template <int P, int kMode>
__device__ __forceinline__ bool bottomk_fill_sorted(WarpBottomK<P, kMode != 0>& L, const int32_t* __restrict__ row,
                                                    int64_t b0, int64_t stride, uint64_t seed0, const BottomKRank& rk) {
  constexpr int R = P <= 2 ? P : 1;
  const int lane = lane_id();
  uint64_t key[R];
#pragma unroll
  for (int r = 0; r < R; ++r) key[r] = bottomk_key<kMode>(seed0, row[b0 + lane + stride * r], rk);
  warp_bitonic_sort<R>(key);
  if (kMode != 0) {
    bool dup = false;
    uint64_t carry = ~0ull;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const uint64_t prev = shfl_up64(key[r], 1);
      dup |= key[r] == (lane == 0 ? carry : prev);
      carry = shfl64(key[r], 31);
    }
    if (__any_sync(0xffffffffu, dup)) return false;
  }
#pragma unroll
  for (int r = 0; r < R; ++r) L.key[r] = key[r];
  L.cnt = 32 * R;
  return true;
}

// write the final list of vertex v.  1-Hash: IDs ascending (rank sort in
// the warp's smem scratch), -1 pad; KMV: values ascending, +inf pad.
template <int P, int kMode>
__device__ __forceinline__ void bottomk_emit(const WarpBottomK<P, kMode != 0>& L, int64_t v, int k,
                                             uint64_t seed0, int32_t* scratch,
                                             int32_t* __restrict__ entries, double* __restrict__ values,
                                             int32_t* __restrict__ lengths, const BottomKRank& rk) {
  const int lane = lane_id();
  const int cnt = L.cnt;
  if (kMode == 2) {
#pragma unroll
    for (int s = 0; s < P; ++s) {
      const int idx = lane + 32 * s;
      if (idx < k) {
        const bool in = idx < cnt;
        values[v * k + idx] = in ? __ldg(rk.rank_values + (uint32_t)L.key[s]) : bitsd(kInfBits);
        rk.ranks[v * k + idx] = in ? (int32_t)L.key[s] : INT32_MAX;
      }
    }
  } else if (kMode == 1) {
#pragma unroll
    for (int s = 0; s < P; ++s) {
      const int idx = lane + 32 * s;
      if (idx < k) values[v * k + idx] = idx < cnt ? bitsd(L.key[s]) : bitsd(kInfBits);
    }
  } else {
    int32_t id[P];
#pragma unroll
    for (int s = 0; s < P; ++s) {
      const int idx = lane + 32 * s;
      id[s] = (int32_t)(unmix64(L.key[s]) ^ seed0);
      if (idx < cnt) scratch[idx] = id[s];
    }
    __syncwarp();
#pragma unroll
    for (int s = 0; s < P; ++s) {
      const int idx = lane + 32 * s;
      if (idx < cnt) {
        int rank = 0;
        for (int j = 0; j < cnt; ++j) rank += scratch[j] < id[s];
        entries[v * k + rank] = id[s];
      } else if (idx < k) {
        entries[v * k + idx] = -1;
      }
    }
    __syncwarp();
  }
  if (lane == 0) lengths[v] = cnt;
}

// KMV row of d <= 32 R neighbours (R = 1, 2): element i = lane + 32 r of a
// 32R-key warp bitonic sort (pad keys ~0 sort last), then the distinct keys
// in order (key i kept when it differs from key i-1), the first k written:
// values ascending, +inf pad; mode 2 also the rank row.  Rows shorter than
// kShortSortMin keep the list insertions (cheaper for a handful of keys).
#ifndef PG_SHORT_SORT_MIN
#define PG_SHORT_SORT_MIN 4  // c3 KMV batch pass: 12 -> 2.42 ms, 4 -> 2.27 ms, 1 -> 2.35 ms
#endif
constexpr int kShortSortMin = PG_SHORT_SORT_MIN;

template <int kMode, int R>
__device__ __forceinline__ void kmv_short_row_r(const int32_t* __restrict__ row, int d, int64_t v, int k,
                                                uint64_t seed0, double* __restrict__ values,
                                                int32_t* __restrict__ lengths, const BottomKRank& rk) {
  const int lane = lane_id();
  uint64_t key[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int i = lane + 32 * r;
    key[r] = i < d ? bottomk_key<kMode>(seed0, row[i], rk) : ~0ull;
  }
  warp_bitonic_sort<R>(key);
  const unsigned lt = (1u << lane) - 1u;
  int before = 0, total = 0;
  uint64_t carry = ~0ull;  // key 32 r - 1 (the last of the previous register)
  bool keep[R];
  int pos[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const uint64_t prev = shfl_up64(key[r], 1);
    keep[r] = key[r] != ~0ull && key[r] != (lane == 0 ? (r ? carry : ~0ull) : prev);
    const unsigned b = __ballot_sync(0xffffffffu, keep[r]);
    pos[r] = before + __popc(b & lt);
    before += __popc(b);
    carry = shfl64(key[r], 31);
  }
  total = before;
  const int cnt = min(total, k);
#pragma unroll
  for (int r = 0; r < R; ++r) {
    if (keep[r] && pos[r] < k) {
      if (kMode == 2) {
        values[v * k + pos[r]] = __ldg(rk.rank_values + (uint32_t)key[r]);
        rk.ranks[v * k + pos[r]] = (int32_t)key[r];
      } else {
        values[v * k + pos[r]] = bitsd(key[r]);
      }
    }
  }
  for (int i = cnt + lane; i < k; i += 32) {
    values[v * k + i] = bitsd(kInfBits);
    if (kMode == 2) rk.ranks[v * k + i] = INT32_MAX;
  }
  if (lane == 0) lengths[v] = cnt;
}

template <int kMode>
__device__ __forceinline__ void kmv_short_row(const int32_t* __restrict__ row, int d, int64_t v, int k,
                                              uint64_t seed0, double* __restrict__ values,
                                              int32_t* __restrict__ lengths, const BottomKRank& rk) {
  if (d <= 32) kmv_short_row_r<kMode, 1>(row, d, v, k, seed0, values, lengths, rk);
  else kmv_short_row_r<kMode, 2>(row, d, v, k, seed0, values, lengths, rk);
}

template <int P, int kMode>
__global__ void __launch_bounds__(kThreads, PG_BK_MINB) build_bottomk_kernel(
    const int64_t* __restrict__ offsets, const int32_t* __restrict__ adj, int64_t n, int k,
    const uint64_t* __restrict__ seeds_dev, int32_t* __restrict__ entries,
    double* __restrict__ values, int32_t* __restrict__ lengths, int32_t* __restrict__ hubs,
    int32_t* __restrict__ hub_count, unsigned long long* __restrict__ vtx_work, BottomKRank rk) {
  constexpr bool kKmv = kMode != 0;
  __shared__ int32_t scratch[kWarps][32 * P];
  const int lane = lane_id();
  const uint64_t seed0 = seeds_dev[0];
  // warps take batches of 32 consecutive vertices from a global counter
  // (degree-skewed rows make a static split leave most warps idle); the
  // batch's offsets come in with one coalesced load, broadcast by shuffles
  for (;;) {
    unsigned long long vbu = 0;
    if (lane_id() == 0) vbu = atomicAdd(vtx_work, 32ull);
    const int64_t vb = (int64_t)__shfl_sync(0xffffffffu, vbu, 0);
    if (vb >= n) break;
    const int64_t vl = vb + lane_id();
    const int64_t ol = vl < n ? offsets[vl] : 0;
    const int64_t el = vl < n ? offsets[vl + 1] : 0;
    const int nb = (int)((n - vb) < 32 ? (n - vb) : 32);
    for (int t = 0; t < nb; ++t) {
      const int64_t v = vb + t;
      const int64_t o = __shfl_sync(0xffffffffu, ol, t);
      const int64_t d = __shfl_sync(0xffffffffu, el, t) - o;
      if (d > PG_BK_HUB) {
        if (lane == 0) hubs[atomicAdd(hub_count, 1)] = (int32_t)v;
        continue;
      }
      if (!kKmv && d <= k) {
        // every neighbour is kept and the CSR row is already ID-sorted
        for (int j = lane; j < k; j += 32) entries[v * k + j] = j < d ? adj[o + j] : -1;
        if (lane == 0) lengths[v] = (int32_t)d;
        continue;
      }
      if (kMode != 0 && d > kShortSortMin && d <= 64) {
        // KMV rows of at most 64 neighbours: one warp bitonic sort of the
        // keys, first copies of equal keys kept (the reference's distinct
        // values), the first k written -- instead of d list insertions
        kmv_short_row<kMode>(adj + o, (int)d, v, k, seed0, values, lengths, rk);
        continue;
      }
      WarpBottomK<P, kKmv> L;
      L.init(k);
      int64_t first = 0;
      if (P <= 2 && k == 32 * P && d >= k && bottomk_fill_sorted<P, kMode>(L, adj + o, 0, 32, seed0, rk))
        first = k;  // the first k keys by one sort; the rest are offered as usual
      bottomk_scan<P, kMode>(L, adj + o, first, d, 32, seed0, rk);
      bottomk_emit<P, kMode>(L, v, k, seed0, scratch[warp_id()], entries, values, lengths, rk);
    }
  }
}

// ascending CTA bitonic sort of buf[0, n) in shared memory, n a power of two
// (>= 2); every thread of the CTA calls it; ends with a barrier
__device__ __forceinline__ void cta_bitonic_sort(uint64_t* buf, int n) {
  for (int size = 2; size <= n; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      __syncthreads();
      for (int t = threadIdx.x; t < (n >> 1); t += kThreads) {
        const int i = 2 * t - (t & (stride - 1));
        const int j = i + stride;
        const uint64_t x = buf[i], y = buf[j];
        if ((x > y) == ((i & size) == 0)) {
          buf[i] = y;
          buf[j] = x;
        }
      }
    }
  }
  __syncthreads();
}

// Hub rows (d > PG_BK_HUB) by a buffered threshold filter, one CTA per hub:
// every thread hashes kHubU entries per round and appends the keys below the
// CTA threshold T to a shared buffer (one shared atomic per warp); when the
// next round could overflow it, the CTA sorts the buffer and keeps the first
// k distinct keys, and T becomes the k-th of them.  T is the k-th distinct
// key of everything seen so far, so a later key > T cannot reach the row's
// bottom-k and a key == T is a repeat of a listed one.  A row of d entries
// costs about log_{1+B/k}(d/B) compactions and no per-key list insertions;
// the eight per-warp lists it replaces inserted ~8 k ln(d/8k) keys and were
// merged by one warp while the other seven waited (1-Hash k=64 at c3: 9.9M
// insertions for 46.5M hub entries, 1.4 ms).
#ifndef PG_HUB_U
#define PG_HUB_U 2
#endif
constexpr int kHubU = PG_HUB_U;                  // entries per thread per round
constexpr int kHubRound = kHubU * kThreads;
constexpr int kHubBuf = 2 * kHubRound;           // shared keys (8 KB)
static_assert(kHubRound >= 256, "a compaction (<= k <= 256 keys) plus one round fits");

// sort buf[0, n), keep its first min(k, distinct) distinct keys in buf[0, ..);
// returns that count (CTA-uniform via s_out)
template <bool kDedup>
__device__ __forceinline__ int hub_compact(uint64_t* buf, int n, int k, int* s_out) {
  int np = 64;
  while (np < n) np <<= 1;
  for (int i = n + threadIdx.x; i < np; i += kThreads) buf[i] = ~0ull;
  cta_bitonic_sort(buf, np);
  if (warp_id() == 0) {
    const int lane = lane_id();
    int got = 0;
    uint64_t last = 0;
    for (int base = 0; base < n && got < k; base += 32) {
      const int i = base + lane;
      const uint64_t x = i < n ? buf[i] : ~0ull;
      const uint64_t prev = shfl_up64(x, 1);
      const uint64_t before = lane == 0 ? last : prev;
      const bool isnew = i < n && (!kDedup || i == 0 || x != before);
      last = shfl64(x, 31);
      const unsigned m = __ballot_sync(0xffffffffu, isnew);
      const int pos = got + __popc(m & ((1u << lane) - 1u));
      __syncwarp();
      if (isnew && pos < k) buf[pos] = x;  // pos <= i: only slots already read
      got += __popc(m);
    }
    if (lane == 0) *s_out = got < k ? got : k;
  }
  __syncthreads();
  return *s_out;
}

template <int P, int kMode>
__global__ void __launch_bounds__(kThreads, PG_BKH_MINB) build_bottomk_hubs_buffered_kernel(
    const int64_t* __restrict__ offsets, const int32_t* __restrict__ adj, int k,
    const uint64_t* __restrict__ seeds_dev, int32_t* __restrict__ entries, double* __restrict__ values,
    int32_t* __restrict__ lengths, const int32_t* __restrict__ hubs, const int32_t* __restrict__ hub_count,
    int32_t* __restrict__ hub_work, BottomKRank rk) {
  constexpr bool kKmv = kMode != 0;
  __shared__ uint64_t buf[kHubBuf];
  __shared__ int32_t scratch[32 * P];
  __shared__ int s_hi, s_n, s_out;
  const int lane = lane_id();
  const uint64_t seed0 = seeds_dev[0];
  const int nh = *hub_count;
  for (;;) {  // hubs taken from a global counter (their degrees vary widely)
    if (threadIdx.x == 0) {
      s_hi = atomicAdd(hub_work, 1);
      s_n = 0;
    }
    __syncthreads();
    const int hi = s_hi;
    if (hi >= nh) break;
    const int64_t v = hubs[hi];
    const int64_t o = offsets[v];
    const int64_t d = offsets[v + 1] - o;
    const int32_t* __restrict__ row = adj + o;
    uint64_t T = ~0ull;  // CTA-uniform
    for (int64_t j0 = 0; j0 < d; j0 += kHubRound) {
      __syncthreads();
      int n = s_n;
      if (n >= kHubBuf - kHubRound) {  // compact as soon as a round's worth is buffered
        n = hub_compact<kKmv>(buf, n, k, &s_out);
        if (threadIdx.x == 0) s_n = n;
        T = n >= k ? buf[k - 1] : ~0ull;
        __syncthreads();
      }
      uint64_t c[kHubU];
      bool pass[kHubU];
#pragma unroll
      for (int u = 0; u < kHubU; ++u) {
        const int64_t j = j0 + u * kThreads + threadIdx.x;
        c[u] = j < d ? bottomk_key<kMode>(seed0, row[j], rk) : ~0ull;
        pass[u] = j < d && (c[u] < T || T == ~0ull);
      }
#pragma unroll
      for (int u = 0; u < kHubU; ++u) {
        const unsigned m = __ballot_sync(0xffffffffu, pass[u]);
        int base = 0;
        if (lane == 0 && m) base = atomicAdd(&s_n, __popc(m));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (pass[u]) buf[base + __popc(m & ((1u << lane) - 1u))] = c[u];
      }
    }
    __syncthreads();
    const int cnt = hub_compact<kKmv>(buf, s_n, k, &s_out);
    if (warp_id() == 0) {
      WarpBottomK<P, kKmv> M;
      M.init(k);
#pragma unroll
      for (int r = 0; r < P; ++r) {
        const int idx = lane + 32 * r;
        if (idx < cnt) M.key[r] = buf[idx];
      }
      M.cnt = cnt;
      bottomk_emit<P, kMode>(M, v, k, seed0, scratch, entries, values, lengths, rk);
    }
    __syncthreads();
  }
}

template <int P, int kMode>
__global__ void __launch_bounds__(kThreads, PG_BKH_MINB) build_bottomk_hubs_kernel(
    const int64_t* __restrict__ offsets, const int32_t* __restrict__ adj, int k,
    const uint64_t* __restrict__ seeds_dev, int32_t* __restrict__ entries, double* __restrict__ values,
    int32_t* __restrict__ lengths, const int32_t* __restrict__ hubs, const int32_t* __restrict__ hub_count,
    int32_t* __restrict__ hub_work, BottomKRank rk) {
  constexpr bool kKmv = kMode != 0;
  __shared__ int32_t scratch[32 * P];
  __shared__ uint64_t merge_keys[kWarps][32 * P];
  __shared__ int merge_cnt[kWarps];
  __shared__ int s_hi;
  __shared__ unsigned long long s_thr;
  const int lane = lane_id();
  const uint64_t seed0 = seeds_dev[0];
  const int nh = *hub_count;
  for (;;) {  // hubs taken from a global counter (their degrees vary widely)
    if (threadIdx.x == 0) {
      s_hi = atomicAdd(hub_work, 1);
      s_thr = ~0ull;
    }
    __syncthreads();
    const int hi = s_hi;
    __syncthreads();
    if (hi >= nh) break;
    const int64_t v = hubs[hi];
    const int64_t o = offsets[v];
    const int64_t d = offsets[v + 1] - o;
    WarpBottomK<P, kKmv> L;
    L.init(k);
    // each warp's first k strided candidates fill its list by one sort
    int64_t first = 32 * warp_id();
    if (P <= 2 && k == 32 * P && d >= 32 * warp_id() + (int64_t)kThreads * (P - 1) + 32 &&
        bottomk_fill_sorted<P, kMode>(L, adj + o, 32 * warp_id(), kThreads, seed0, rk))
      first += (int64_t)kThreads * P;
    bottomk_scan_shared<P, kMode>(L, adj + o, first, d, kThreads, seed0, rk, &s_thr);
#pragma unroll
    for (int s = 0; s < P; ++s) merge_keys[warp_id()][lane + 32 * s] = L.key[s];
    if (lane == 0) merge_cnt[warp_id()] = L.cnt;
    __syncthreads();
    if (warp_id() == 0) {
      WarpBottomK<P, kKmv> M;
      M.init(k);
      // warp 0's list is already a sorted, distinct bottom-k: it starts the
      // merge as is (k insertions saved per hub); the others are offered
#pragma unroll
      for (int r = 0; r < P; ++r) M.key[r] = merge_keys[0][lane + 32 * r];
      M.cnt = merge_cnt[0];
      for (int w = 1; w < kWarps; ++w) {
        const int cw = merge_cnt[w];
        for (int base = 0; base < cw; base += 32) {
          const int idx = base + lane;
          const bool valid = idx < cw;
          M.offer(valid ? merge_keys[w][idx] : ~0ull, valid);
        }
      }
      bottomk_emit<P, kMode>(M, v, k, seed0, scratch, entries, values, lengths, rk);
    }
    __syncthreads();
  }
}

// one resident wave of CTAs (each warp loops over 32-vertex batches)
template <class K>
static int grid_for(K kernel, size_t smem, int64_t n) {
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kThreads, smem) != cudaSuccess ||
      per_sm < 1)
    per_sm = 1;
  const int64_t batches = (n + 31) / 32;
  const int64_t need = (batches + kWarps - 1) / kWarps;
  return (int)std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)sm_count() * per_sm));
}

// transient device hub list: int32 count + up to n vertex IDs
struct HubList {
  int32_t* count = nullptr;
  int32_t* ids = nullptr;
  void* buf = nullptr;
  cudaStream_t s = nullptr;
  // capacity n + 1 (any vertex may be a hub): no host round trip for nnz
  // header: [hub count i32 | hub work i32 | vertex-batch work u64], then ids
  int32_t* hub_work = nullptr;
  unsigned long long* vtx_work = nullptr;
  // optional second list (Bloom: mid-degree vertices, one warp each):
  // header [mid count i32 | mid work i32], then up to n ids
  int32_t* mid_count = nullptr;
  int32_t* mid_work = nullptr;
  int32_t* mids = nullptr;
  int init(const int64_t* offsets, int64_t n, cudaStream_t st, bool with_mid = false) {
    (void)offsets;
    s = st;
    retain_default_pool();
    const size_t list = sizeof(int32_t) * (size_t)n;
    const size_t bytes = 16 + list + (with_mid ? 16 + list : 0);
    cudaError_t e = cudaMallocAsync(&buf, bytes, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(buf, 0, 16, s);
    if (e == cudaSuccess && with_mid) e = cudaMemsetAsync(static_cast<char*>(buf) + 16 + list, 0, 16, s);
    if (e != cudaSuccess) return fail(PG_ERR_CUDA, "hub list: %s", cudaGetErrorString(e));
    count = static_cast<int32_t*>(buf);
    hub_work = count + 1;
    vtx_work = reinterpret_cast<unsigned long long*>(static_cast<char*>(buf) + 8);
    ids = reinterpret_cast<int32_t*>(static_cast<char*>(buf) + 16);
    if (with_mid) {
      mid_count = reinterpret_cast<int32_t*>(static_cast<char*>(buf) + 16 + list);
      mid_work = mid_count + 1;
      mids = mid_count + 4;
    }
    return PG_OK;
  }
  ~HubList() {
    if (buf) cudaFreeAsync(buf, s);
  }
};

int hub_grid() { return sm_count() * 4; }

}  // namespace pg

using namespace pg;

template <int kMode>
static int launch_bottomk(const int64_t* offsets, const int32_t* adj, int64_t n, int32_t k,
                          const uint64_t* seeds_dev, int32_t* entries, double* values, int32_t* lengths,
                          void* stream, BottomKRank rk = BottomKRank()) {
  cudaStream_t s = as_stream(stream);
  HubList hubs;
  if (int rc = hubs.init(offsets, n, s)) return rc;
#define PG_BK(P)                                                                                          \
  {                                                                                                       \
    const int grid = grid_for(build_bottomk_kernel<P, kMode>, 0, n);                                     \
    build_bottomk_kernel<P, kMode><<<grid, kThreads, 0, s>>>(offsets, adj, n, k, seeds_dev, entries, values, \
                                                             lengths, hubs.ids, hubs.count, hubs.vtx_work, rk); \
    PG_BK_HUB_KERNEL<P, kMode><<<hub_grid(), kThreads, 0, s>>>(offsets, adj, k, seeds_dev, entries, \
                                                                         values, lengths, hubs.ids,        \
                                                                         hubs.count, hubs.hub_work, rk);   \
  }
  if (k <= 32) PG_BK(1)
  else if (k <= 64) PG_BK(2)
  else if (k <= 128) PG_BK(4)
  else PG_BK(8)
#undef PG_BK
  return check_launch(kMode == 0 ? "build_onehash" : "build_kmv");
}

// ---------------------------------------------------- KMV value ranks ----
// unit-value bits of every vertex ID (the KMV key of x as a neighbour)
__global__ void kmv_universe_kernel(int64_t n, const uint64_t* __restrict__ seeds_dev, uint64_t* __restrict__ keys,
                                    int32_t* __restrict__ ids) {
  const uint64_t seed0 = seeds_dev[0];
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n; x += (int64_t)gridDim.x * blockDim.x) {
    keys[x] = dbits(unit_value(hash_word(seed0, (int32_t)x)));
    ids[x] = (int32_t)x;
  }
}
__global__ void kmv_rank_flags_kernel(int64_t n, const uint64_t* __restrict__ keys, int32_t* __restrict__ flags) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    flags[i] = (i > 0 && keys[i] != keys[i - 1]) ? 1 : 0;
}
__global__ void kmv_rank_scatter_kernel(int64_t n, const uint64_t* __restrict__ keys,
                                        const int32_t* __restrict__ ids, const int32_t* __restrict__ dense,
                                        int32_t* __restrict__ rank_of, double* __restrict__ rank_values) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t r = dense[i];
    rank_of[ids[i]] = r;
    if (i == 0 || keys[i] != keys[i - 1]) rank_values[r] = bitsd(keys[i]);
  }
}

// ---- 1-Hash hash-rank rows (a device layout for the TC engine) ----------
// h0 is a bijection on vertex IDs (mix64 of seed ^ id), so the position of
// h0(x) among all n hash words is an exact, collision-free relabelling of
// the IDs: two 1-Hash rows share an ID iff their rank rows share a rank.
// Sorted by rank, every element of a row is at most the row's k-th smallest
// hash, so a probe of v's ranks into u's table can stop at u's largest rank.
__global__ void hash_universe_kernel(int64_t n, const uint64_t* __restrict__ seeds_dev,
                                     uint64_t* __restrict__ keys, int32_t* __restrict__ ids) {
  const uint64_t seed0 = seeds_dev[0];
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n; x += (int64_t)gridDim.x * blockDim.x) {
    keys[x] = hash_word(seed0, (int32_t)x);
    ids[x] = (int32_t)x;
  }
}
__global__ void hash_rank_scatter_kernel(int64_t n, const int32_t* __restrict__ ids, int32_t* __restrict__ rank_of) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    rank_of[ids[i]] = (int32_t)i;
}
// one warp per row: ranks of the stored IDs (INT32_MAX for the -1 pads),
// bitonic-sorted ascending across the warp's 32 * P registers
template <int P>
__global__ void __launch_bounds__(256) onehash_rank_rows_kernel(const int32_t* __restrict__ entries, int64_t n,
                                                                const int32_t* __restrict__ rank_of,
                                                                int32_t* __restrict__ out, int group) {
  constexpr int K = 32 * P;
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t v = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); v < n; v += warps) {
    int32_t x[P];
    // element index of register s on lane l: s * 32 + l
#pragma unroll
    for (int s = 0; s < P; ++s) {
      const int32_t id = entries[v * K + s * 32 + lane];
      x[s] = id < 0 ? INT32_MAX : __ldg(rank_of + id);
    }
    // bitonic network over indices i = s * 32 + lane
#pragma unroll
    for (int size = 2; size <= K; size <<= 1) {
#pragma unroll
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
#pragma unroll
        for (int s = 0; s < P; ++s) {
          const int i = s * 32 + lane;
          const bool up = (i & size) == 0;  // ascending block
          if (stride >= 32) {
            const int t = s ^ (stride >> 5);  // partner register on the same lane
            if (t > s) {
              const int32_t a = x[s], b = x[t];
              const bool sw = up ? a > b : a < b;
              x[s] = sw ? b : a;
              x[t] = sw ? a : b;
            }
          } else {
            const int32_t o = __shfl_xor_sync(0xffffffffu, x[s], stride);
            const bool low = (lane & stride) == 0;
            x[s] = (low == up) ? min(x[s], o) : max(x[s], o);
          }
        }
      }
    }
    // sorted element j goes to slot (j % group) * (K / group) + j / group:
    // with `group` lanes per row reading K / group consecutive slots each,
    // lane g's p-th register is sorted element p * group + g
    const int per = K / group;
#pragma unroll
    for (int s = 0; s < P; ++s) {
      const int j = s * 32 + lane;
      out[v * K + (j % group) * per + j / group] = x[s];
    }
  }
}

extern "C" {

int pg_hash_rank_table(int64_t n, const uint64_t* seeds_dev, int32_t* rank_of, void* stream) {
  PG_REQUIRE(n >= 0 && n <= INT32_MAX, "n must be in [0, 2^31)");
  if (n == 0) return PG_OK;
  PG_REQUIRE(seeds_dev && rank_of, "null pointer");
  cudaStream_t s = as_stream(stream);
  retain_default_pool();
  size_t t_sort = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, t_sort, (const uint64_t*)nullptr, (uint64_t*)nullptr,
                                  (const int32_t*)nullptr, (int32_t*)nullptr, n, 0, 64);
  const size_t bytes = 2 * 8 * (size_t)n + 2 * 4 * (size_t)n + t_sort + 64;
  char* buf = nullptr;
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&buf), bytes, s);
  if (e != cudaSuccess) return fail(PG_ERR_CUDA, "rank table scratch: %s", cudaGetErrorString(e));
  uint64_t* k0 = reinterpret_cast<uint64_t*>(buf);
  uint64_t* k1 = k0 + n;
  int32_t* i0 = reinterpret_cast<int32_t*>(k1 + n);
  int32_t* i1 = i0 + n;
  void* tmp = i1 + n + 8;
  const int grid = sm_count() * 8;
  hash_universe_kernel<<<grid, 256, 0, s>>>(n, seeds_dev, k0, i0);
  size_t t = t_sort;
  e = cub::DeviceRadixSort::SortPairs(tmp, t, k0, k1, i0, i1, n, 0, 64, s);
  if (e == cudaSuccess) hash_rank_scatter_kernel<<<grid, 256, 0, s>>>(n, i1, rank_of);
  cudaFreeAsync(buf, s);
  if (e != cudaSuccess) return fail(PG_ERR_CUDA, "rank table: %s", cudaGetErrorString(e));
  return check_launch("hash_rank_table");
}

int pg_onehash_rank_rows(const int32_t* entries, int64_t n, int32_t k, const int32_t* rank_of,
                         int32_t group, int32_t* rank_rows, void* stream) {
  PG_REQUIRE(n >= 0, "n must be >= 0");
  PG_REQUIRE(group >= 1 && group <= 32 && (group & (group - 1)) == 0, "group must be a power of two <= 32");
  if (k != 32 && k != 64 && k != 128)
    return fail(PG_ERR_UNSUPPORTED, "1-Hash rank rows support k = 32, 64, 128 (got %d)", k);
  if (n == 0) return PG_OK;
  PG_REQUIRE(entries && rank_of && rank_rows, "null pointer");
  cudaStream_t s = as_stream(stream);
  const int grid = (int)std::min<int64_t>((n + 7) / 8, (int64_t)sm_count() * 16);
  if (k == 32) onehash_rank_rows_kernel<1><<<grid, 256, 0, s>>>(entries, n, rank_of, rank_rows, group);
  else if (k == 64) onehash_rank_rows_kernel<2><<<grid, 256, 0, s>>>(entries, n, rank_of, rank_rows, group);
  else onehash_rank_rows_kernel<4><<<grid, 256, 0, s>>>(entries, n, rank_of, rank_rows, group);
  return check_launch("onehash_rank_rows");
}

int pg_build_bloom(const int64_t* offsets, const int32_t* adj, int64_t n, int32_t bits, int32_t b,
                   const uint64_t* seeds_dev, uint64_t* rows, int32_t* ones, void* stream) {
  PG_REQUIRE(n >= 0, "n must be >= 0");
  PG_REQUIRE(bits >= 64 && bits % 64 == 0, "Bloom size must be a positive multiple of 64");
  PG_REQUIRE(b >= 1 && b <= 64, "Bloom hash count must be in [1, 64]");
  PG_REQUIRE(offsets && seeds_dev && rows && ones, "null pointer");
  if (n == 0) return PG_OK;
  cudaStream_t s = as_stream(stream);
  if (bits > kMaxBloomBits)  // rows wider than the shared-memory batch rows
    return gen_build_bloom(offsets, adj, n, bits, b, seeds_dev, rows, ones, s);
  HubList hubs;
  if (int rc = hubs.init(offsets, n, s, true)) return rc;
  // batch size: 32 vertices per warp while the rows fit ~96 KB per CTA
  int R = 32;
  while (R > 1 && (size_t)kWarps * R * (bits / 8) > 96 * 1024) R >>= 1;
  const size_t smem = kWarps * sizeof(BloomBatchSmem) + 64 * sizeof(uint64_t) + (size_t)kWarps * R * (bits / 8);
  const size_t smem_hub = (size_t)(bits / 8) + 8 + 64 * sizeof(uint64_t);
  const size_t smem_mid = 64 * sizeof(uint64_t) + (size_t)kWarps * (bits / 8);
  const bool pow2 = (bits & (bits - 1)) == 0;
#define PG_BB(P2)                                                                                       \
  {                                                                                                     \
    cudaFuncSetAttribute(build_bloom_kernel<P2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    cudaFuncSetAttribute(build_bloom_hubs_kernel<P2>, cudaFuncAttributeMaxDynamicSharedMemorySize,        \
                         (int)smem_hub);                                                                \
    const int grid = grid_for(build_bloom_kernel<P2>, smem, (n + R - 1) / R * 32);                      \
    build_bloom_kernel<P2><<<grid, kThreads, smem, s>>>(offsets, adj, n, bits, b, R, seeds_dev, rows, ones, \
                                                        hubs.ids, hubs.count, hubs.vtx_work, hubs.mids,  \
                                                        hubs.mid_count);                                \
    cudaFuncSetAttribute(build_bloom_mid_kernel<P2>, cudaFuncAttributeMaxDynamicSharedMemorySize,         \
                         (int)smem_mid);                                                                \
    build_bloom_mid_kernel<P2><<<grid_for(build_bloom_mid_kernel<P2>, smem_mid, 32 * (int64_t)n), kThreads, smem_mid, s>>>( \
        offsets, adj, bits, b, seeds_dev, rows, ones, hubs.mids, hubs.mid_count, hubs.mid_work);        \
    build_bloom_hubs_kernel<P2><<<hub_grid(), kThreads, smem_hub, s>>>(offsets, adj, bits, b, seeds_dev,  \
                                                                       rows, hubs.ids, hubs.count);       \
    bloom_hub_ones_kernel<<<64, kThreads, 0, s>>>(rows, bits / 64, ones, hubs.ids, hubs.count);          \
  }
  if (pow2) PG_BB(true)
  else PG_BB(false)
#undef PG_BB
  return check_launch("build_bloom");
}

int pg_build_khash(const int64_t* offsets, const int32_t* adj, int64_t n, int32_t k,
                   const uint64_t* seeds_dev, int32_t* entries, void* stream) {
  PG_REQUIRE(n >= 0, "n must be >= 0");
  PG_REQUIRE(k >= 1, "k must be >= 1");
  PG_REQUIRE(offsets && seeds_dev && entries, "null pointer");
  if (n == 0) return PG_OK;
  cudaStream_t s = as_stream(stream);
  if (k > kMaxSketchK) return gen_build_khash(offsets, adj, n, k, seeds_dev, entries, s);
  HubList hubs;
  if (int rc = hubs.init(offsets, n, s)) return rc;
#define PG_KB(S)                                                                                         \
  {                                                                                                      \
    const int grid = grid_for(build_khash_kernel<S>, 0, n);                                              \
    build_khash_kernel<S><<<grid, kThreads, 0, s>>>(offsets, adj, n, k, seeds_dev, entries, hubs.ids,     \
                                                    hubs.count, hubs.vtx_work);                          \
    build_khash_hubs_kernel<S><<<hub_grid(), kThreads, 0, s>>>(offsets, adj, k, seeds_dev, entries,       \
                                                               hubs.ids, hubs.count, hubs.hub_work);     \
  }
  if (k <= 32) PG_KB(1)
  else if (k <= 64) PG_KB(2)
  else if (k <= 128) PG_KB(4)
  else PG_KB(8)
#undef PG_KB
  return check_launch("build_khash");
}

int pg_build_onehash(const int64_t* offsets, const int32_t* adj, int64_t n, int32_t k,
                     const uint64_t* seeds_dev, int32_t* entries, int32_t* lengths, void* stream) {
  PG_REQUIRE(n >= 0, "n must be >= 0");
  PG_REQUIRE(k >= 1, "k must be >= 1");
  PG_REQUIRE(offsets && seeds_dev && entries && lengths, "null pointer");
  if (n == 0) return PG_OK;
  if (k > kMaxSketchK)
    return gen_build_bottomk(offsets, adj, n, k, seeds_dev, entries, nullptr, nullptr, nullptr, lengths,
                             as_stream(stream));
  return launch_bottomk<0>(offsets, adj, n, k, seeds_dev, entries, nullptr, lengths, stream);
}

int pg_build_kmv(const int64_t* offsets, const int32_t* adj, int64_t n, int32_t k,
                 const uint64_t* seeds_dev, double* values, int32_t* lengths, void* stream) {
  PG_REQUIRE(n >= 0, "n must be >= 0");
  PG_REQUIRE(k >= 1, "k must be >= 1");
  PG_REQUIRE(offsets && seeds_dev && values && lengths, "null pointer");
  if (n == 0) return PG_OK;
  if (k > kMaxSketchK)
    return gen_build_bottomk(offsets, adj, n, k, seeds_dev, nullptr, values, nullptr, nullptr, lengths,
                             as_stream(stream));
  return launch_bottomk<1>(offsets, adj, n, k, seeds_dev, nullptr, values, lengths, stream);
}

int pg_kmv_rank_table(int64_t n, const uint64_t* seeds_dev, int32_t* rank_of, double* rank_values,
                      void* stream) {
  PG_REQUIRE(n >= 0 && n <= INT32_MAX, "n must be in [0, 2^31)");
  if (n == 0) return PG_OK;
  PG_REQUIRE(seeds_dev && rank_of && rank_values, "null pointer");
  cudaStream_t s = as_stream(stream);
  retain_default_pool();
  size_t t_sort = 0, t_scan = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, t_sort, (const uint64_t*)nullptr, (uint64_t*)nullptr,
                                  (const int32_t*)nullptr, (int32_t*)nullptr, n, 0, 64);
  cub::DeviceScan::InclusiveSum(nullptr, t_scan, (const int32_t*)nullptr, (int32_t*)nullptr, n);
  const size_t tb = std::max(t_sort, t_scan);
  const size_t bytes = 2 * 8 * (size_t)n + 3 * 4 * (size_t)n + tb + 64;
  char* buf = nullptr;
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&buf), bytes, s);
  if (e != cudaSuccess) return fail(PG_ERR_CUDA, "rank table scratch: %s", cudaGetErrorString(e));
  uint64_t* k0 = reinterpret_cast<uint64_t*>(buf);
  uint64_t* k1 = k0 + n;
  int32_t* i0 = reinterpret_cast<int32_t*>(k1 + n);
  int32_t* i1 = i0 + n;
  int32_t* fl = i1 + n;
  void* tmp = fl + n + 8;
  const int grid = sm_count() * 8;
  kmv_universe_kernel<<<grid, 256, 0, s>>>(n, seeds_dev, k0, i0);
  // unit values lie in (0, 1]: their IEEE bits are below 2^62
  size_t t = tb;
  e = cub::DeviceRadixSort::SortPairs(tmp, t, k0, k1, i0, i1, n, 0, 62, s);
  if (e == cudaSuccess) {
    kmv_rank_flags_kernel<<<grid, 256, 0, s>>>(n, k1, fl);
    t = tb;
    e = cub::DeviceScan::InclusiveSum(tmp, t, fl, i0, n, s);
  }
  if (e == cudaSuccess) kmv_rank_scatter_kernel<<<grid, 256, 0, s>>>(n, k1, i1, i0, rank_of, rank_values);
  cudaFreeAsync(buf, s);
  if (e != cudaSuccess) return fail(PG_ERR_CUDA, "rank table: %s", cudaGetErrorString(e));
  return check_launch("kmv_rank_table");
}

int pg_build_kmv_ranked(const int64_t* offsets, const int32_t* adj, int64_t n, int32_t k,
                        const uint64_t* seeds_dev, const int32_t* rank_of, const double* rank_values,
                        double* values, int32_t* ranks, int32_t* lengths, void* stream) {
  PG_REQUIRE(n >= 0, "n must be >= 0");
  PG_REQUIRE(k >= 1, "k must be >= 1");
  PG_REQUIRE(offsets && seeds_dev && rank_of && rank_values && values && ranks && lengths, "null pointer");
  if (n == 0) return PG_OK;
  if (k > kMaxSketchK)
    return gen_build_bottomk(offsets, adj, n, k, seeds_dev, nullptr, values, ranks, rank_of, lengths,
                             as_stream(stream));
  BottomKRank rk;
  rk.rank_of = rank_of;
  rk.rank_values = rank_values;
  rk.ranks = ranks;
  return launch_bottomk<2>(offsets, adj, n, k, seeds_dev, nullptr, values, lengths, stream, rk);
}

}  // extern "C"
