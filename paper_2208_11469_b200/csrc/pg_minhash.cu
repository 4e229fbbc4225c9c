// k-Hash / 1-Hash per-edge estimates (providers.py:197-232 pair_many,
// _matches_khash / _matches_onehash), their fused TC reductions and the
// Jaccard threshold count (estimators.py:123-168, mining.py:157-186).
#include <algorithm>

#include "pg_generic.cuh"

namespace pg {


template <int V, int G, bool kScalar>
__global__ void __launch_bounds__(kBlock) pairs_khash_kernel(const uint4* ent, int k, const int32_t* us,
                                                            const int32_t* vs, int64_t count,
                                                            EpiMinhashPairs epi) {
  if (kScalar) scalar_edge_loop_khash(reinterpret_cast<const int32_t*>(ent), k, us, vs, 0, count, epi);
  else group_edge_loop<V, G, OpEqPos>(ent, us, vs, 0, count, epi);
}

// CTAs/SM of the wide k-Hash engine for 128-byte rows (k = 32): 4 (64
// registers) measured 3.70 vs 4.04 ms at c4 over 3 -- the random row gathers
// are latency-bound, more warps in flight win
#ifndef PG_KHASH128_MINB
#define PG_KHASH128_MINB 4
#endif
constexpr int kKhash128Minb = PG_KHASH128_MINB;
#ifndef PG_KHASH_VCACHE
#define PG_KHASH_VCACHE 0
#endif
constexpr bool kKhashVCache = PG_KHASH_VCACHE;  // L1-allocated v rows in the wide k-Hash engine

// kEngine: 0 scalar fallback, 1 group (128-bit) engine, 2 wide padded engine
template <int V, int G, int kEngine, int MINB = 1, bool kDyn = false, int kLayout = 1>
__global__ void __launch_bounds__(kBlock, MINB) tc_khash_kernel(const uint4* ent, int k, const int32_t* sizes,
                                                               const int32_t* us, const int32_t* vs,
                                                               int64_t e_begin, int64_t e_end,
                                                               int64_t* out_cnt, int64_t* out_ssum,
                                                               unsigned long long* ctr = nullptr) {
  __shared__ int cnt_s[kMaxSketchK + 1];
  __shared__ unsigned slo_s[kMaxSketchK + 1], shi_s[kMaxSketchK + 1];
  for (int i = threadIdx.x; i <= k; i += blockDim.x) { cnt_s[i] = 0; slo_s[i] = 0; shi_s[i] = 0; }
  __syncthreads();
  EpiMinhashHist epi{sizes, cnt_s, slo_s, shi_s};
  if (kEngine == 0) scalar_edge_loop_khash(reinterpret_cast<const int32_t*>(ent), k, us, vs, e_begin, e_end, epi);
  else if (kEngine == 1) group_edge_loop<V, G, OpEqPos>(ent, us, vs, e_begin, e_end, epi);
  else wide_edge_loop<V, OpEqPos, EpiMinhashHist, kKhashVCache, kLayout, kDyn>(reinterpret_cast<const unsigned char*>(ent),
                                                                      us, vs, e_begin, e_end, epi, ctr);
  __syncthreads();
  for (int i = threadIdx.x; i <= k; i += blockDim.x) {
    if (cnt_s[i]) {
      atomicAdd(reinterpret_cast<unsigned long long*>(out_cnt + i), (unsigned long long)cnt_s[i]);
      atomicAdd(reinterpret_cast<unsigned long long*>(out_ssum + i),
                ((unsigned long long)shi_s[i] << 32) + slo_s[i]);
    }
  }
}

template <int V, int G, int kEngine, int MINB = 1, bool kDyn = false, int kLayout = 1>
__global__ void __launch_bounds__(kBlock, MINB) jaccard_khash_kernel(const uint4* ent, int k, const int32_t* deg,
                                                                    const int32_t* us, const int32_t* vs,
                                                                    int64_t e_begin, int64_t e_end,
                                                                    int min_matches, double tau,
                                                                    int64_t* out_counts,
                                                                    unsigned long long* ctr = nullptr) {
  __shared__ int hist_s[kMaxSketchK + 1];
  for (int i = threadIdx.x; i <= k; i += blockDim.x) hist_s[i] = 0;
  __syncthreads();
  EpiJaccard epi{k, min_matches, tau, deg, hist_s, 0, 0};
  if (kEngine == 0) scalar_edge_loop_khash(reinterpret_cast<const int32_t*>(ent), k, us, vs, e_begin, e_end, epi);
  else if (kEngine == 1) group_edge_loop<V, G, OpEqPos>(ent, us, vs, e_begin, e_end, epi);
  else wide_edge_loop<V, OpEqPos, EpiJaccard, kKhashVCache, kLayout, kDyn>(reinterpret_cast<const unsigned char*>(ent), us,
                                                                  vs, e_begin, e_end, epi, ctr);
  __syncthreads();
  for (int i = threadIdx.x; i <= k; i += blockDim.x)
    if (hist_s[i]) atomicAdd(reinterpret_cast<unsigned long long*>(out_counts + 2 + i), (unsigned long long)hist_s[i]);
  long long a = epi.n_hat, b = epi.n_sim;
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (a) atomicAdd(reinterpret_cast<unsigned long long*>(out_counts + 0), (unsigned long long)a);
    if (b) atomicAdd(reinterpret_cast<unsigned long long*>(out_counts + 1), (unsigned long long)b);
  }
}

// warp-per-edge match count of two ascending ID lists (-1 padded); returns
// m and the two list lengths (warp-uniform)
template <int P>
__device__ __forceinline__ int onehash_matches(const int32_t* __restrict__ ent, int k, int32_t u, int32_t v,
                                               int32_t* vbuf, int& lu, int& lv) {
  const int lane = threadIdx.x & 31;
  int32_t a[P], b[P];
  lu = 0;
  lv = 0;
#pragma unroll
  for (int s = 0; s < P; ++s) {
    const int idx = lane + 32 * s;
    a[s] = idx < k ? ent[(int64_t)u * k + idx] : -1;
    b[s] = idx < k ? ent[(int64_t)v * k + idx] : -1;
    lu += __popc(__ballot_sync(0xffffffffu, a[s] >= 0));
    lv += __popc(__ballot_sync(0xffffffffu, b[s] >= 0));
  }
#pragma unroll
  for (int s = 0; s < P; ++s) {
    const int idx = lane + 32 * s;
    if (idx < lv) vbuf[idx] = b[s];
  }
  __syncwarp();
  int m = 0;
#pragma unroll
  for (int s = 0; s < P; ++s) {
    const int idx = lane + 32 * s;
    bool hit = false;
    if (idx < lu) {
      const int p = smem_lower_bound(vbuf, lv, a[s]);
      hit = p < lv && vbuf[p] == a[s];
    }
    m += __popc(__ballot_sync(0xffffffffu, hit));
  }
  __syncwarp();
  return m;
}

template <int P, bool kFused>
__global__ void __launch_bounds__(kBlock) onehash_kernel(const int32_t* ent, int k, const int32_t* sizes,
                                                        const int32_t* us, const int32_t* vs,
                                                        int64_t e_begin, int64_t e_end,
                                                        int32_t* out_count, double* out_est,
                                                        int64_t* out_cnt, int64_t* out_ssum,
                                                        int64_t* out_verbatim) {
  __shared__ int32_t vbuf[kBlock / 32][32 * P];
  __shared__ int cnt_s[kMaxSketchK + 1];
  __shared__ unsigned slo_s[kMaxSketchK + 1], shi_s[kMaxSketchK + 1];
  if (kFused) {
    for (int i = threadIdx.x; i <= k; i += blockDim.x) { cnt_s[i] = 0; slo_s[i] = 0; shi_s[i] = 0; }
    __syncthreads();
  }
  const int lane = threadIdx.x & 31;
  long long verb = 0;
  int64_t wb, we;
  warp_slice(e_begin, e_end, wb, we);
  for (int64_t e = wb; e < we; ++e) {
    const int32_t u = us[e], v = vs[e];
    int lu, lv;
    const int m = onehash_matches<P>(ent, k, u, v, vbuf[threadIdx.x >> 5], lu, lv);
    if (lane == 0) {
      const int32_t su = sizes[u], sv = sizes[v];
      const bool verbatim = su <= k && sv <= k;
      if (kFused) {
        if (verbatim) verb += m;
        else {
          atomicAdd(cnt_s + m, 1);
          smem_add64(slo_s + m, shi_s + m, (uint64_t)((int64_t)su + sv));
        }
      } else {
        if (out_count) out_count[e] = m;
        if (out_est) out_est[e] = verbatim ? (double)m : minhash_estimate(m, k, su, sv);
      }
    }
  }
  if (kFused) {
    __syncthreads();
    for (int i = threadIdx.x; i <= k; i += blockDim.x) {
      if (cnt_s[i]) {
        atomicAdd(reinterpret_cast<unsigned long long*>(out_cnt + i), (unsigned long long)cnt_s[i]);
        atomicAdd(reinterpret_cast<unsigned long long*>(out_ssum + i),
                  ((unsigned long long)shi_s[i] << 32) + slo_s[i]);
      }
    }
    if (lane == 0 && verb) atomicAdd(reinterpret_cast<unsigned long long*>(out_verbatim), (unsigned long long)verb);
  }
}

template <int K, int P, bool kFused>
__global__ void __launch_bounds__(kBlock) onehash_htab_kernel(const int32_t* ent, const int32_t* sizes,
                                                             const int32_t* us, const int32_t* vs,
                                                             int64_t e_begin, int64_t e_end, int32_t* out_count,
                                                             double* out_est, int64_t* out_cnt, int64_t* out_ssum,
                                                             int64_t* out_verbatim, unsigned long long* ctr) {
  extern __shared__ __align__(16) int32_t htab_smem[];  // (kBlock/32) * (32/G) groups
  __shared__ int cnt_s[K + 1];
  __shared__ unsigned slo_s[K + 1], shi_s[K + 1];
  if (kFused) {
    for (int i = threadIdx.x; i <= K; i += blockDim.x) { cnt_s[i] = 0; slo_s[i] = 0; shi_s[i] = 0; }
    __syncthreads();
  }
  constexpr int kWarpInts = (32 / (K / P)) * htab_group_ints<K>();
  EpiOnehash epi{K, sizes, out_count, out_est, kFused ? cnt_s : nullptr, slo_s, shi_s, 0};
  htab_edge_loop<K, P>(ent, sizes, us, vs, e_begin, e_end, ctr, htab_smem + (threadIdx.x >> 5) * kWarpInts, epi);
  if (kFused) {
    __syncthreads();
    for (int i = threadIdx.x; i <= K; i += blockDim.x) {
      if (cnt_s[i]) {
        atomicAdd(reinterpret_cast<unsigned long long*>(out_cnt + i), (unsigned long long)cnt_s[i]);
        atomicAdd(reinterpret_cast<unsigned long long*>(out_ssum + i),
                  ((unsigned long long)shi_s[i] << 32) + slo_s[i]);
      }
    }
    long long vb = epi.verb;
    for (int o = 16; o > 0; o >>= 1) vb += __shfl_xor_sync(0xffffffffu, vb, o);
    if ((threadIdx.x & 31) == 0 && vb)
      atomicAdd(reinterpret_cast<unsigned long long*>(out_verbatim), (unsigned long long)vb);
  }
}

template <int G, int CH, bool kFused>
__global__ void __launch_bounds__(kBlock) onehash_sorted_kernel(const int32_t* ent, int k, const int32_t* sizes,
                                                               const int32_t* us, const int32_t* vs,
                                                               int64_t e_begin, int64_t e_end,
                                                               int32_t* out_count, double* out_est,
                                                               int64_t* out_cnt, int64_t* out_ssum,
                                                               int64_t* out_verbatim) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int cnt_s[kMaxSketchK + 1];
  __shared__ unsigned slo_s[kMaxSketchK + 1], shi_s[kMaxSketchK + 1];
  if (kFused) {
    for (int i = threadIdx.x; i <= k; i += blockDim.x) { cnt_s[i] = 0; slo_s[i] = 0; shi_s[i] = 0; }
    __syncthreads();
  }
  EpiOnehash epi{k, sizes, out_count, out_est, kFused ? cnt_s : nullptr, slo_s, shi_s, 0};
  sorted_edge_loop<G, CH>(ent, k, us, vs, e_begin, e_end,
                          smem_raw + (threadIdx.x >> 5) * sorted_warp_smem<G, CH>(), epi);
  if (kFused) {
    __syncthreads();
    for (int i = threadIdx.x; i <= k; i += blockDim.x) {
      if (cnt_s[i]) {
        atomicAdd(reinterpret_cast<unsigned long long*>(out_cnt + i), (unsigned long long)cnt_s[i]);
        atomicAdd(reinterpret_cast<unsigned long long*>(out_ssum + i),
                  ((unsigned long long)shi_s[i] << 32) + slo_s[i]);
      }
    }
    long long vb = epi.verb;
    for (int o = 16; o > 0; o >>= 1) vb += __shfl_xor_sync(0xffffffffu, vb, o);
    if ((threadIdx.x & 31) == 0 && vb)
      atomicAdd(reinterpret_cast<unsigned long long*>(out_verbatim), (unsigned long long)vb);
  }
}

// sorted-engine launchers; return false when k has no specialisation
// ---------------------------------- 1-Hash, per-warp table, slot blocks
// The row-padded slot layout with pad E = 256/k (pg_csr_upper_edges_padded)
// gives every warp iteration E edges of one u, so the u table is one per
// warp (built by all 32 lanes: k/32 IDs each, against k/8 per lane in the
// per-group engine, and a quarter of its shared memory) and survives across
// the whole u run.  Slot blocks as in the KMV rank engine: lane l holds slot
// l's endpoints one block ahead; after each 32-slot block every lane files
// its slot's statistics.  Same bucket table and probe as htab_edge_loop.
#ifndef PG_OH_UNROLL
#define PG_OH_UNROLL 2  // unroll of the block's iteration loop (c3: 1: 3.13 ms, 2: 2.75, 4: 5.2 with spills)
#endif
#ifndef PG_OH_PER_LANE
#define PG_OH_PER_LANE 8
#endif
constexpr int kOnehashPerLane = PG_OH_PER_LANE;  // v-row IDs per lane (pad = 32 * this / k)
#ifndef PG_OH_SLOTS
#define PG_OH_SLOTS 4
#endif
// slots per bucket of the per-warp table: 4 (K buckets, one LDS.128 per
// probe) or 2 (2K buckets, one LDS.64: half the shared-memory wavefronts)
constexpr int kOnehashSlots = PG_OH_SLOTS;

template <int K>
__device__ __forceinline__ uint32_t oh_bucket(int32_t x) {
  constexpr int kB = 4 * K / kOnehashSlots;  // buckets
  constexpr int kBits = kB == 32 ? 5 : kB == 64 ? 6 : kB == 128 ? 7 : kB == 256 ? 8 : 9;
  return ((uint32_t)x * 0x9E3779B1u) >> (32 - kBits);
}

template <int K>
struct alignas(16) OnehashWarp {
  int32_t tab[4 * K];  // K buckets x 4 slots, or 2K buckets x 2 (kOnehashSlots)
  int32_t stash[K];
  int32_t mbuf[32];    // per slot of the block: matches
  int sc;
};

// kRank: the rows are hash-rank rows (pg_onehash_rank_rows: the ranks of the
// stored IDs' h0 words, ascending, INT32_MAX pad) instead of ID rows.  Ranks
// relabel IDs one to one, so the match counts are the same integers; sorted
// by rank, nothing in v's row above u's largest rank can be in u's table, so
// those probes (44 % of them at c3; all pads) are skipped.
template <int K, bool kRank = false>
__global__ void __launch_bounds__(kBlock, 5) onehash_block_kernel(const int32_t* __restrict__ R,
                                                               const int32_t* __restrict__ sizes,
                                                               const int32_t* __restrict__ us,
                                                               const int32_t* __restrict__ vs, int64_t e_begin,
                                                               int64_t e_end, int64_t* out_cnt, int64_t* out_ssum,
                                                               int64_t* out_verbatim, unsigned long long* ctr) {
  constexpr int P = kOnehashPerLane, G = K / P, E = 32 / G, IT = 32 / E;
  constexpr int64_t kChunk = 512;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int cnt_s[K + 1];
  __shared__ unsigned slo_s[K + 1], shi_s[K + 1];
  for (int i = threadIdx.x; i <= K; i += blockDim.x) { cnt_s[i] = 0; slo_s[i] = 0; shi_s[i] = 0; }
  __syncthreads();
  OnehashWarp<K>& W = reinterpret_cast<OnehashWarp<K>*>(smem_raw)[threadIdx.x >> 5];
  const int lane = threadIdx.x & 31, gl = lane & (G - 1), grp = lane / G;
  EpiOnehash epi{K, sizes, nullptr, nullptr, cnt_s, slo_s, shi_s, 0};
  int32_t cur_u = -1;
  int sc = 0;
  int32_t tau = INT32_MAX - 1;  // kRank: the largest rank in u's table
  int64_t wb, we;
  while (next_chunk(ctr, e_begin, e_end, kChunk, wb, we)) {
    int32_t ul = 0, vl = -1;
    if (wb + lane < we) {
      ul = us[wb + lane];
      vl = vs[wb + lane];
    }
    int32_t sul = sizes[ul], svl = vl >= 0 ? sizes[vl] : 0;
    int32_t vq = __shfl_sync(0xffffffffu, vl, grp);
    uint32_t x[P];
    ldg_rowpart<P>(R + (int64_t)(vq < 0 ? 0 : vq) * K + gl * P, x);
#pragma unroll 1
    for (int64_t b0 = wb; b0 < we; b0 += 32) {
      int32_t un = 0, vn = -1, sun = 0, svn = 0;
      if (b0 + 32 + lane < we) {
        un = us[b0 + 32 + lane];
        vn = vs[b0 + 32 + lane];
      }
      constexpr int kItUnroll = PG_OH_UNROLL;
#pragma unroll kItUnroll
      for (int it = 0; it < IT; ++it) {
        const int slot = it * E + grp;
        const int32_t u = __shfl_sync(0xffffffffu, ul, it * E);
        const bool valid = b0 + slot < we && vq >= 0;
        if (it == IT / 2) {  // the next block's sizes, off the critical path
          sun = sizes[un];
          svn = vn >= 0 ? sizes[vn] : 0;
        }
        if (u != cur_u) {  // warp-uniform: rebuild the warp's table
          cur_u = u;
          int32_t y[K / 32];
#pragma unroll
          for (int q = 0; q < K / 32; ++q) y[q] = __ldg(R + (int64_t)u * K + lane + 32 * q);
          int4* T4 = reinterpret_cast<int4*>(W.tab);
#pragma unroll
          for (int i = lane; i < K; i += 32) T4[i] = make_int4(-1, -1, -1, -1);
          if (lane == 0) W.sc = 0;
          __syncwarp();
          if (kRank) {
            int32_t mx = -1;
#pragma unroll
            for (int q = 0; q < K / 32; ++q) mx = max(mx, y[q] == INT32_MAX ? -1 : y[q]);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            tau = mx;
          }
#pragma unroll
          for (int q = 0; q < K / 32; ++q) {
            if (kRank ? y[q] == INT32_MAX : y[q] < 0) continue;  // pad
            int32_t* bk = W.tab + kOnehashSlots * oh_bucket<K>(y[q]);
            bool placed = false;
#pragma unroll
            for (int sl = 0; sl < kOnehashSlots && !placed; ++sl) placed = atomicCAS(bk + sl, -1, y[q]) == -1;
            if (!placed) W.stash[atomicAdd(&W.sc, 1)] = y[q];
          }
          __syncwarp();
          sc = *reinterpret_cast<volatile int*>(&W.sc);
        }
        const int32_t vqn = __shfl_sync(0xffffffffu, it + 1 < IT ? vl : vn, it + 1 < IT ? slot + E : grp);
        uint32_t xn[P];
        ldg_rowpart<P>(R + (int64_t)(vqn < 0 ? 0 : vqn) * K + gl * P, xn);
        int m = 0;
#pragma unroll
        for (int p = 0; p < P; ++p) {
          const int32_t q = (int32_t)x[p];
          // rank rows are interleaved over the row's G lanes (register p of
          // lane g = sorted element p * G + g): once no lane of the warp has a
          // candidate, no later register has one either
          if (kRank && !__any_sync(0xffffffffu, valid && q <= tau)) break;
          if (valid && (kRank ? q <= tau : q >= 0)) {
            bool hit;
            if constexpr (kOnehashSlots == 2) {
              const int2 bk = reinterpret_cast<const int2*>(W.tab)[oh_bucket<K>(q)];
              hit = (bk.x == q) | (bk.y == q);
            } else {
              const int4 bk = reinterpret_cast<const int4*>(W.tab)[oh_bucket<K>(q)];
              hit = (bk.x == q) | (bk.y == q) | (bk.z == q) | (bk.w == q);
            }
            for (int i = 0; i < sc; ++i) hit |= W.stash[i] == q;
            m += hit;
          }
        }
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) m += __shfl_xor_sync(0xffffffffu, m, o);
        if (gl == 0) W.mbuf[slot] = m;
#pragma unroll
        for (int p = 0; p < P; ++p) x[p] = xn[p];
        vq = vqn;
      }
      __syncwarp();
      if (b0 + lane < we && vl >= 0) epi.edge_sized(b0 + lane, sul, svl, W.mbuf[lane], 0, 0);
      __syncwarp();
      ul = un;
      vl = vn;
      sul = sun;
      svl = svn;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i <= K; i += blockDim.x) {
    if (cnt_s[i]) {
      atomicAdd(reinterpret_cast<unsigned long long*>(out_cnt + i), (unsigned long long)cnt_s[i]);
      atomicAdd(reinterpret_cast<unsigned long long*>(out_ssum + i), ((unsigned long long)shi_s[i] << 32) + slo_s[i]);
    }
  }
  long long vb = epi.verb;
  for (int o = 16; o > 0; o >>= 1) vb += __shfl_xor_sync(0xffffffffu, vb, o);
  if ((threadIdx.x & 31) == 0 && vb)
    atomicAdd(reinterpret_cast<unsigned long long*>(out_verbatim), (unsigned long long)vb);
}

template <int K, bool kRank = false>
static int launch_onehash_block(cudaStream_t s, const int32_t* ent, const int32_t* sizes, const int32_t* us,
                                const int32_t* vs, int64_t b, int64_t e, int64_t* out_cnt, int64_t* out_ssum,
                                int64_t* out_verbatim) {
  auto kern = onehash_block_kernel<K, kRank>;
  const size_t sm = sizeof(OnehashWarp<K>) * (kBlock / 32);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  const int grid = grid_cap(grid_for_kernel(kern, sm), e - b, kBlock / (K / kOnehashPerLane));
  ChunkCounter ctr;
  const cudaError_t ce = ctr.init(s);
  if (ce != cudaSuccess) return fail(PG_ERR_CUDA, "chunk counter: %s", cudaGetErrorString(ce));
  kern<<<grid, kBlock, sm, s>>>(ent, sizes, us, vs, b, e, out_cnt, out_ssum, out_verbatim, ctr.p);
  return check_launch("tc_onehash_block");
}

template <int G, int CH, bool kFused>
static void launch_onehash_sorted(cudaStream_t s, const int32_t* ent, int k, const int32_t* sizes,
                                  const int32_t* us, const int32_t* vs, int64_t b, int64_t e,
                                  int32_t* out_count, double* out_est, int64_t* out_cnt,
                                  int64_t* out_ssum, int64_t* out_verbatim) {
  auto kern = onehash_sorted_kernel<G, CH, kFused>;
  const size_t sm = (size_t)(kBlock / 32) * sorted_warp_smem<G, CH>();
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  const int grid = grid_cap(grid_for_kernel(kern, sm), e - b, kBlock / G);
  kern<<<grid, kBlock, sm, s>>>(ent, k, sizes, us, vs, b, e, out_count, out_est, out_cnt, out_ssum,
                                out_verbatim);
}

template <int K, int P, bool kFused>
static void launch_onehash_htab(cudaStream_t s, const int32_t* ent, const int32_t* sizes, const int32_t* us,
                                const int32_t* vs, int64_t b, int64_t e, int32_t* out_count, double* out_est,
                                int64_t* out_cnt, int64_t* out_ssum, int64_t* out_verbatim) {
  auto kern = onehash_htab_kernel<K, P, kFused>;
  const size_t sm = sizeof(int32_t) * (kBlock / 32) * (32 / (K / P)) * htab_group_ints<K>();
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  const int grid = grid_cap(grid_for_kernel(kern, sm), e - b, kBlock / (K / P));
  ChunkCounter ctr;
  if (ctr.init(s) != cudaSuccess) return;  // reported by check_launch
  kern<<<grid, kBlock, sm, s>>>(ent, sizes, us, vs, b, e, out_count, out_est, out_cnt, out_ssum, out_verbatim,
                                ctr.p);
}

static bool onehash_sorted(cudaStream_t s, bool fused, const int32_t* ent, int k, const int32_t* sizes,
                           const int32_t* us, const int32_t* vs, int64_t b, int64_t e, int32_t* out_count,
                           double* out_est, int64_t* out_cnt, int64_t* out_ssum, int64_t* out_verbatim) {
  static const bool lookup = [] {
    const char* v = getenv("PG_ONEHASH_ENGINE");
    return v && v[0] == 'l';
  }();
  if (!lookup) {
#define PG_OT(K, P)                                                                                       \
  {                                                                                                       \
    if (fused) launch_onehash_htab<K, P, true>(s, ent, sizes, us, vs, b, e, out_count, out_est, out_cnt, \
                                               out_ssum, out_verbatim);                                   \
    else launch_onehash_htab<K, P, false>(s, ent, sizes, us, vs, b, e, out_count, out_est, out_cnt,      \
                                          out_ssum, out_verbatim);                                        \
    return true;                                                                                          \
  }
    static const int per_lane = [] {
      const char* v = getenv("PG_ONEHASH_IDS");
      return v ? atoi(v) : 8;
    }();
    if (k == 32) { if (per_lane == 16) PG_OT(32, 16) PG_OT(32, 8) }
    if (k == 64) { if (per_lane == 16) PG_OT(64, 16) PG_OT(64, 8) }
    if (k == 128) { if (per_lane == 16) PG_OT(128, 16) PG_OT(128, 8) }
#undef PG_OT
  }
#define PG_OS(G, CH)                                                                                     \
  {                                                                                                      \
    if (fused) launch_onehash_sorted<G, CH, true>(s, ent, k, sizes, us, vs, b, e, out_count, out_est,    \
                                                  out_cnt, out_ssum, out_verbatim);                      \
    else launch_onehash_sorted<G, CH, false>(s, ent, k, sizes, us, vs, b, e, out_count, out_est,        \
                                             out_cnt, out_ssum, out_verbatim);                           \
    return true;                                                                                         \
  }
  if (k == 32) PG_OS(4, 1)
  if (k == 64) PG_OS(8, 1)
  if (k == 128) PG_OS(8, 2)
#undef PG_OS
  return false;
}
// Layout helper for the hash-rank 1-Hash engine: out[e] = number of ranks of
// the probe row ps[e] that are <= the largest rank of the table row ts[e],
// i.e. the probes the engine makes for slot e (rows interleaved over `group`
// lanes as pg_onehash_rank_rows stores them).
__global__ void __launch_bounds__(256) onehash_prefix_counts_kernel(const int32_t* __restrict__ rows,
                                                                    const int32_t* __restrict__ lengths, int k,
                                                                    int group, const int32_t* __restrict__ ts,
                                                                    const int32_t* __restrict__ ps,
                                                                    int64_t count, int32_t* __restrict__ out) {
  const int per = k / group;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < count;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int32_t t = ts[e], p = ps[e];
    int c = 0;
    if (t >= 0 && p >= 0) {
      const int lt = lengths[t], lp = lengths[p];
      if (lt > 0) {
        const int jt = lt - 1;
        const int32_t tau = rows[(int64_t)t * k + (jt % group) * per + jt / group];
        int lo = 0, hi = lp;  // first sorted index of p's row above tau
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (rows[(int64_t)p * k + (mid % group) * per + mid / group] <= tau) lo = mid + 1;
          else hi = mid;
        }
        c = lo;
      }
    }
    out[e] = c;
  }
}

// Rows of an oriented CSR (table vertex t = the row, entries = the probe
// endpoints) counting-sorted by the register positions the rank-row engine
// needs for each entry, ceil(probes / group) in 0 .. k / group: a warp per
// row, two passes (bucket of every entry into `bucket`, then a stable
// scatter by warp-aggregated ranks).
__device__ __forceinline__ int onehash_probe_bucket(const int32_t* __restrict__ rows, int k, int group, int per,
                                                    int32_t tau, int32_t p, int lp) {
  int lo = 0, hi = lp;  // first sorted index of p's row above tau
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (rows[(int64_t)p * k + (mid % group) * per + mid / group] <= tau) lo = mid + 1;
    else hi = mid;
  }
  return (lo + group - 1) / group;
}
// pass 1, a thread per entry: the entry's bucket
__global__ void __launch_bounds__(256) onehash_row_buckets_kernel(const int32_t* __restrict__ src,
                                                                  const int32_t* __restrict__ adj, int64_t nnz,
                                                                  const int32_t* __restrict__ rows,
                                                                  const int32_t* __restrict__ lengths, int k,
                                                                  int group, unsigned char* __restrict__ bucket) {
  const int per = k / group;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nnz; j += (int64_t)gridDim.x * blockDim.x) {
    const int32_t t = src[j], p = adj[j];
    const int lt = lengths[t];
    int32_t tau = -1;
    if (lt > 0) tau = rows[(int64_t)t * k + ((lt - 1) % group) * per + (lt - 1) / group];
    bucket[j] = (unsigned char)onehash_probe_bucket(rows, k, group, per, tau, p, lengths[p]);
  }
}
// rows above this many entries are sorted by a whole CTA each: one warp walking
// a 500,000-entry hub row 32 entries at a time took 8 ms of the 13 ms pass
constexpr int64_t kSortLongRow = 2048;
// pass 2 for long rows, a CTA per row: bucket counts by a block reduction,
// then 256-entry rounds in order (stable), ranks from warp ballots and a
// cross-warp prefix
__global__ void __launch_bounds__(256) onehash_sort_long_rows_kernel(const int64_t* __restrict__ off,
                                                                     const int32_t* __restrict__ adj, int64_t n,
                                                                     int nb,
                                                                     const unsigned char* __restrict__ bucket,
                                                                     int32_t* __restrict__ out) {
  constexpr int kMaxB = kOnehashPerLane + 1;
  __shared__ int cnt_s[kMaxB];
  __shared__ int wcnt[8][kMaxB];
  __shared__ int64_t run_s[kMaxB];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int64_t t = blockIdx.x; t < n; t += gridDim.x) {
    const int64_t b = off[t], e = off[t + 1];
    if (e - b <= kSortLongRow) continue;  // block-uniform
    if (threadIdx.x < kMaxB) cnt_s[threadIdx.x] = 0;
    __syncthreads();
    int cnt[kMaxB];
#pragma unroll
    for (int q = 0; q < kMaxB; ++q) cnt[q] = 0;
    for (int64_t j = b + threadIdx.x; j < e; j += 256) {
      const int q = (int)bucket[j];
#pragma unroll
      for (int z = 0; z < kMaxB; ++z) cnt[z] += z == q;
    }
#pragma unroll
    for (int q = 0; q < kMaxB; ++q) {
      int c = cnt[q];
      for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
      if (lane == 0 && c) atomicAdd(&cnt_s[q], c);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int64_t run = b;
      for (int q = 0; q < kMaxB; ++q) {
        run_s[q] = run;
        run += cnt_s[q];
      }
    }
    __syncthreads();
    for (int64_t j0 = b; j0 < e; j0 += 256) {
      const int64_t j = j0 + threadIdx.x;
      const bool in = j < e;
      const int q = in ? (int)bucket[j] : -1;
      const int32_t p = in ? adj[j] : 0;
      int my_rank = 0;
      for (int z = 0; z < nb; ++z) {
        const unsigned m = __ballot_sync(0xffffffffu, q == z);
        if (lane == 0) wcnt[w][z] = __popc(m);
        if (q == z) my_rank = __popc(m & lanemask_lt());
      }
      __syncthreads();
      if (in) {
        int before = 0;
        for (int i = 0; i < w; ++i) before += wcnt[i][q];
        out[run_s[q] + before + my_rank] = p;
      }
      __syncthreads();
      if (threadIdx.x < nb) {
        int tsum = 0;
        for (int i = 0; i < 8; ++i) tsum += wcnt[i][threadIdx.x];
        run_s[threadIdx.x] += tsum;
      }
      __syncthreads();
    }
  }
}
// pass 2, a warp per row: stable counting sort of the row by bucket
__global__ void __launch_bounds__(256) onehash_sort_rows_kernel(const int64_t* __restrict__ off,
                                                                const int32_t* __restrict__ adj, int64_t n,
                                                                int nb, const unsigned char* __restrict__ bucket,
                                                                int32_t* __restrict__ out,
                                                                unsigned long long* ctr) {
  constexpr int kMaxB = kOnehashPerLane + 1;  // k / group + 1 (the engine holds kOnehashPerLane ranks per lane)
  const int lane = threadIdx.x & 31;
  for (;;) {
    unsigned long long t64 = 0;
    if (lane == 0) t64 = atomicAdd(ctr, 8ull);  // eight rows per request
    t64 = __shfl_sync(0xffffffffu, t64, 0);
    if ((int64_t)t64 >= n) return;
    const int64_t t_end = min((int64_t)t64 + 8, n);
    for (int64_t t = (int64_t)t64; t < t_end; ++t) {
      const int64_t b = off[t], e = off[t + 1];
      if (e == b || e - b > kSortLongRow) continue;  // long rows: onehash_sort_long_rows_kernel
      int64_t base[kMaxB];
      if (e - b <= 32) {  // one round: counts and positions from the same ballots
        const int64_t j = b + lane;
        const bool in = j < e;
        const int q = in ? (int)bucket[j] : -1;
        const int32_t p = in ? adj[j] : 0;
        int64_t run = b;
#pragma unroll
        for (int z = 0; z < kMaxB; ++z) {
          if (z >= nb) break;
          const unsigned m = __ballot_sync(0xffffffffu, q == z);
          if (q == z) out[run + __popc(m & lanemask_lt())] = p;
          run += __popc(m);
        }
        continue;
      }
      int cnt[kMaxB];
#pragma unroll
      for (int q = 0; q < kMaxB; ++q) cnt[q] = 0;
      for (int64_t j = b + lane; j < e; j += 32) {
        const int q = (int)bucket[j];
#pragma unroll
        for (int z = 0; z < kMaxB; ++z) cnt[z] += z == q;
      }
      int64_t run = b;
#pragma unroll
      for (int q = 0; q < kMaxB; ++q) {
        int c = cnt[q];
        for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
        base[q] = run;
        run += c;
      }
      for (int64_t j0 = b; j0 < e; j0 += 32) {
        const int64_t j = j0 + lane;
        const bool in = j < e;
        const int q = in ? (int)bucket[j] : -1;
        const int32_t p = in ? adj[j] : 0;
#pragma unroll
        for (int z = 0; z < kMaxB; ++z) {
          if (z >= nb) break;
          const unsigned m = __ballot_sync(0xffffffffu, q == z);
          if (q == z) out[base[z] + __popc(m & lanemask_lt())] = p;
          base[z] += __popc(m);
        }
      }
    }
  }
}

}  // namespace pg

using namespace pg;

extern "C" {


int pg_pairs_minhash(const int32_t* entries, int32_t k, int32_t onehash, const int32_t* sizes,
                     const int32_t* us, const int32_t* vs, int64_t count, int32_t* out_count,
                     double* out_est, void* stream) {
  PG_REQUIRE(k >= 1, "k must be >= 1");
  PG_REQUIRE(count >= 0, "count must be >= 0");
  if (count == 0) return PG_OK;
  PG_REQUIRE(entries && us && vs, "null pointer");
  PG_REQUIRE(!out_est || sizes, "estimate needs sizes");
  PG_REQUIRE(!onehash || sizes, "1-Hash needs sizes");
  cudaStream_t s = as_stream(stream);
  if (k > kMaxSketchK)
    return gen_pairs_minhash(entries, k, onehash != 0, sizes, us, vs, count, out_count, out_est, s);
  if (onehash) {
    PG_REQUIRE(sizes, "1-Hash needs sizes");
    if (onehash_sorted(s, false, entries, k, sizes, us, vs, 0, count, out_count, out_est, nullptr, nullptr,
                       nullptr))
      return check_launch("pairs_onehash_sorted");
    const int grid = grid_cap(sm_count() * 8, count, kBlock / 32);
#define PG_OH(P) onehash_kernel<P, false><<<grid, kBlock, 0, s>>>(entries, k, sizes, us, vs, 0, count, out_count, out_est, nullptr, nullptr, nullptr)
    if (k <= 32) PG_OH(1);
    else if (k <= 64) PG_OH(2);
    else if (k <= 128) PG_OH(4);
    else PG_OH(8);
#undef PG_OH
    return check_launch("pairs_onehash");
  }
  EpiMinhashPairs epi{k, sizes, out_count, out_est};
  const int grid = grid_cap(sm_count() * 8, count, kBlock);
  const int w4 = k % 4 == 0 ? k / 4 : 0;
  const uint4* e4 = reinterpret_cast<const uint4*>(entries);
  if (!fast_w4(w4)) {
    pairs_khash_kernel<1, 1, true><<<grid, kBlock, 0, s>>>(e4, k, us, vs, count, epi);
  } else {
#define PG_L(V, G) pairs_khash_kernel<V, G, false><<<grid, kBlock, 0, s>>>(e4, k, us, vs, count, epi);
    PG_ROW_DISPATCH(w4, PG_L)
#undef PG_L
  }
  return check_launch("pairs_khash");
}

int pg_onehash_prefix_counts(const int32_t* rank_rows, const int32_t* lengths, int32_t k, int32_t group,
                             const int32_t* ts, const int32_t* ps, int64_t count, int32_t* out,
                             void* stream) {
  PG_REQUIRE(k >= 1 && count >= 0, "bad sizes");
  PG_REQUIRE(group >= 1 && group <= 32 && (group & (group - 1)) == 0 && k % group == 0,
             "group must be a power of two <= 32 dividing k");
  if (count == 0) return PG_OK;
  PG_REQUIRE(rank_rows && lengths && ts && ps && out, "null pointer");
  const int grid = (int)std::min<int64_t>((count + 255) / 256, (int64_t)sm_count() * 16);
  onehash_prefix_counts_kernel<<<grid, 256, 0, as_stream(stream)>>>(rank_rows, lengths, k, group, ts, ps, count,
                                                                    out);
  return check_launch("onehash_prefix_counts");
}

int pg_onehash_sort_rows(const int64_t* off, const int32_t* adj, int64_t n, const int32_t* rank_rows,
                         const int32_t* lengths, int32_t k, int32_t group, int32_t* adj_out, void* stream) {
  PG_REQUIRE(n >= 0 && k >= 1, "bad sizes");
  PG_REQUIRE(group >= 1 && group <= 32 && (group & (group - 1)) == 0 && k % group == 0 &&
                 k / group <= kOnehashPerLane,
             "group must be a power of two <= 32 with k / group <= %d", kOnehashPerLane);
  if (n == 0) return PG_OK;
  PG_REQUIRE(off && rank_rows && lengths, "null pointer");
  cudaStream_t s = as_stream(stream);
  int64_t nnz = 0;
  cudaError_t ce = cudaMemcpyAsync(&nnz, off + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s);
  if (ce == cudaSuccess) ce = cudaStreamSynchronize(s);
  if (ce != cudaSuccess) return fail(PG_ERR_CUDA, "offsets: %s", cudaGetErrorString(ce));
  if (nnz == 0) return PG_OK;
  PG_REQUIRE(adj && adj_out && adj != adj_out, "null pointer / in place");
  unsigned char* bucket = nullptr;
  int32_t* src = nullptr;
  retain_default_pool();
  ce = cudaMallocAsync(reinterpret_cast<void**>(&bucket), (size_t)nnz, s);
  if (ce == cudaSuccess) ce = cudaMallocAsync(reinterpret_cast<void**>(&src), sizeof(int32_t) * (size_t)nnz, s);
  ChunkCounter ctr;
  if (ce == cudaSuccess) ce = ctr.init(s);
  int rc = ce == cudaSuccess ? PG_OK : fail(PG_ERR_CUDA, "scratch: %s", cudaGetErrorString(ce));
  if (rc == PG_OK) rc = pg_csr_expand_rows(off, n, nnz, src, stream);
  if (rc == PG_OK) {
    const int grid = (int)std::min<int64_t>((nnz + 255) / 256, (int64_t)sm_count() * 16);
    onehash_row_buckets_kernel<<<grid, 256, 0, s>>>(src, adj, nnz, rank_rows, lengths, k, group, bucket);
    onehash_sort_long_rows_kernel<<<sm_count() * 4, 256, 0, s>>>(off, adj, n, k / group + 1, bucket, adj_out);
    onehash_sort_rows_kernel<<<sm_count() * 8, 256, 0, s>>>(off, adj, n, k / group + 1, bucket, adj_out, ctr.p);
  }
  if (bucket) cudaFreeAsync(bucket, s);
  if (src) cudaFreeAsync(src, s);
  if (rc != PG_OK) return rc;
  return check_launch("onehash_sort_rows");
}

int pg_onehash_block_pad(int32_t k, int32_t* pad_host) {
  PG_REQUIRE(pad_host, "null output");
  *pad_host = (k == 32 || k == 64 || k == 128) ? 32 * kOnehashPerLane / k : 1;
  return PG_OK;
}

int pg_tc_minhash(const int32_t* entries, int32_t k, int32_t onehash, const int32_t* sizes,
                  const int32_t* us, const int32_t* vs, int64_t e_begin, int64_t e_end, int32_t padded,
                  int64_t* out_cnt, int64_t* out_ssum, int64_t* out_verbatim, void* stream) {
  PG_REQUIRE(k >= 1, "k must be >= 1");
  PG_REQUIRE(k <= kMaxSketchK || padded != 2, "group-u slots need k <= %d", kMaxSketchK);
  PG_REQUIRE(0 <= e_begin && e_begin <= e_end, "bad edge range");
  PG_REQUIRE(out_cnt && out_ssum && out_verbatim, "null pointer");
  if (onehash == 2 && !(padded && (k == 32 || k == 64 || k == 128)))
    return fail(PG_ERR_UNSUPPORTED, "hash-rank rows need the row-padded layout and k = 32, 64, 128 (got k = %d)", k);
  cudaStream_t s = as_stream(stream);
  // one memset when [cnt | ssum | verbatim] is one buffer
  const bool adjacent = out_ssum == out_cnt + k + 1 && out_verbatim == out_ssum + k + 1;
  cudaError_t ce = cudaMemsetAsync(out_cnt, 0, sizeof(int64_t) * (adjacent ? 2 * k + 3 : k + 1), s);
  if (ce == cudaSuccess && !adjacent) ce = cudaMemsetAsync(out_ssum, 0, sizeof(int64_t) * (k + 1), s);
  if (ce == cudaSuccess && !adjacent) ce = cudaMemsetAsync(out_verbatim, 0, sizeof(int64_t), s);
  if (ce != cudaSuccess) return fail(PG_ERR_CUDA, "memset: %s", cudaGetErrorString(ce));
  if (e_end == e_begin) return PG_OK;  // an empty range needs no inputs
  PG_REQUIRE(entries && us && vs && sizes, "null pointer");
  if (k > kMaxSketchK)
    return gen_tc_minhash(entries, k, onehash != 0, sizes, us, vs, e_begin, e_end, out_cnt, out_ssum, out_verbatim,
                          s);
  if (onehash && padded && (k == 32 || k == 64 || k == 128)) {
    // the row-padded layout of pad 32 * kOnehashPerLane / k: one u per warp iteration
    const int pad = 32 * kOnehashPerLane / k;
    PG_REQUIRE(e_begin % pad == 0, "e_begin must be a multiple of the layout pad %d", pad);
    if (onehash == 2) {  // hash-rank rows
      if (k == 32) return launch_onehash_block<32, true>(s, entries, sizes, us, vs, e_begin, e_end, out_cnt, out_ssum, out_verbatim);
      if (k == 64) return launch_onehash_block<64, true>(s, entries, sizes, us, vs, e_begin, e_end, out_cnt, out_ssum, out_verbatim);
      return launch_onehash_block<128, true>(s, entries, sizes, us, vs, e_begin, e_end, out_cnt, out_ssum, out_verbatim);
    }
    if (k == 32) return launch_onehash_block<32>(s, entries, sizes, us, vs, e_begin, e_end, out_cnt, out_ssum, out_verbatim);
    if (k == 64) return launch_onehash_block<64>(s, entries, sizes, us, vs, e_begin, e_end, out_cnt, out_ssum, out_verbatim);
    return launch_onehash_block<128>(s, entries, sizes, us, vs, e_begin, e_end, out_cnt, out_ssum, out_verbatim);
  }

  if (onehash && onehash_sorted(s, true, entries, k, sizes, us, vs, e_begin, e_end, nullptr, nullptr, out_cnt,
                                out_ssum, out_verbatim))
    return check_launch("tc_onehash_sorted");
  if (onehash) {
#define PG_OH(P)                                                                                  \
  {                                                                                               \
    auto kern = onehash_kernel<P, true>;                                                          \
    const int grid = grid_cap(grid_for_kernel(kern, 0), e_end - e_begin, kBlock / 32);            \
    kern<<<grid, kBlock, 0, s>>>(entries, k, sizes, us, vs, e_begin, e_end, nullptr, nullptr, out_cnt, out_ssum, out_verbatim); \
  }
    if (k <= 32) PG_OH(1)
    else if (k <= 64) PG_OH(2)
    else if (k <= 128) PG_OH(4)
    else PG_OH(8)
#undef PG_OH
    return check_launch("tc_onehash");
  }
  const int w4 = k % 4 == 0 ? k / 4 : 0;
  const uint4* e4 = reinterpret_cast<const uint4*>(entries);
  const int w8 = k % 8 == 0 ? k / 8 : 0;  // 32-byte chunks per row
  if (padded && (w8 == 2 || w8 == 4 || w8 == 8)) {
#define PG_KW(W8, MB)                                                                    \
  {                                                                                      \
    auto kern = tc_khash_kernel<W8, 1, 2, MB>;                                           \
    if (e_end - e_begin >= kDynamicMinSlots) kern = tc_khash_kernel<W8, 1, 2, MB, true>; \
    if (padded == 2) kern = e_end - e_begin >= kDynamicMinSlots ? tc_khash_kernel<W8, 1, 2, MB, true, 2> \
                                                                : tc_khash_kernel<W8, 1, 2, MB, false, 2>; \
    const int grid = grid_cap(grid_for_kernel(kern, 0), e_end - e_begin, kBlock);        \
    ChunkCounter ctr;                                                                    \
    if (e_end - e_begin >= kDynamicMinSlots && (ce = ctr.init(s)) != cudaSuccess) return fail(PG_ERR_CUDA, "chunk counter: %s", cudaGetErrorString(ce)); \
    kern<<<grid, kBlock, 0, s>>>(e4, k, sizes, us, vs, e_begin, e_end, out_cnt, out_ssum, ctr.p); \
  }
    if (w8 == 2) PG_KW(2, 3) else if (w8 == 4) PG_KW(4, kKhash128Minb) else PG_KW(8, 3)  // measured: 3 blocks beat the spill-free 2 (0.66 vs 0.72 ms, s20 k=64)
#undef PG_KW
  } else if (!fast_w4(w4)) {
    auto kern = tc_khash_kernel<1, 1, 0>;
    const int grid = grid_cap(grid_for_kernel(kern, 0), e_end - e_begin, kBlock);
    kern<<<grid, kBlock, 0, s>>>(e4, k, sizes, us, vs, e_begin, e_end, out_cnt, out_ssum, nullptr);
  } else {
#define PG_L(V, G)                                                                       \
  {                                                                                      \
    auto kern = tc_khash_kernel<V, G, 1>;                                                \
    const int grid = grid_cap(grid_for_kernel(kern, 0), e_end - e_begin, kBlock);        \
    kern<<<grid, kBlock, 0, s>>>(e4, k, sizes, us, vs, e_begin, e_end, out_cnt, out_ssum, nullptr); \
  }
    PG_ROW_DISPATCH(w4, PG_L)
#undef PG_L
  }
  return check_launch("tc_khash");
}

int pg_jaccard_count_khash(const int32_t* entries, int32_t k, const int32_t* degrees, const int32_t* us,
                           const int32_t* vs, int64_t e_begin, int64_t e_end, int32_t padded,
                           int32_t min_matches, double tau, int64_t* out_counts, void* stream) {
  PG_REQUIRE(k >= 1, "k must be >= 1");
  PG_REQUIRE(k <= kMaxSketchK || padded != 2, "group-u slots need k <= %d", kMaxSketchK);
  PG_REQUIRE(0 <= e_begin && e_begin <= e_end, "bad edge range");
  PG_REQUIRE(out_counts, "null pointer");
  cudaStream_t s = as_stream(stream);
  cudaError_t ce = cudaMemsetAsync(out_counts, 0, sizeof(int64_t) * (k + 3), s);
  if (ce != cudaSuccess) return fail(PG_ERR_CUDA, "memset: %s", cudaGetErrorString(ce));
  if (e_end == e_begin) return PG_OK;  // an empty range needs no inputs
  PG_REQUIRE(entries && us && vs && degrees, "null pointer");
  if (k > kMaxSketchK)
    return gen_jaccard_khash(entries, k, degrees, us, vs, e_begin, e_end, min_matches, tau, out_counts, s);
  const int w4 = k % 4 == 0 ? k / 4 : 0;
  const uint4* e4 = reinterpret_cast<const uint4*>(entries);
  const int w8 = k % 8 == 0 ? k / 8 : 0;  // 32-byte chunks per row
  if (padded && (w8 == 2 || w8 == 4 || w8 == 8)) {
#define PG_JW(W8, MB)                                                                                  \
  {                                                                                                    \
    auto kern = jaccard_khash_kernel<W8, 1, 2, MB>;                                                    \
    if (e_end - e_begin >= kDynamicMinSlots) kern = jaccard_khash_kernel<W8, 1, 2, MB, true>;          \
    if (padded == 2) kern = e_end - e_begin >= kDynamicMinSlots ? jaccard_khash_kernel<W8, 1, 2, MB, true, 2> \
                                                                : jaccard_khash_kernel<W8, 1, 2, MB, false, 2>; \
    const int grid = grid_cap(grid_for_kernel(kern, 0), e_end - e_begin, kBlock);                      \
    ChunkCounter ctr;                                                                                  \
    if (e_end - e_begin >= kDynamicMinSlots && (ce = ctr.init(s)) != cudaSuccess) return fail(PG_ERR_CUDA, "chunk counter: %s", cudaGetErrorString(ce)); \
    kern<<<grid, kBlock, 0, s>>>(e4, k, degrees, us, vs, e_begin, e_end, min_matches, tau, out_counts, ctr.p); \
  }
    if (w8 == 2) PG_JW(2, 3) else if (w8 == 4) PG_JW(4, kKhash128Minb) else PG_JW(8, 2)  // 256-B rows: 2 blocks (no spills)
#undef PG_JW
  } else if (!fast_w4(w4)) {
    auto kern = jaccard_khash_kernel<1, 1, 0>;
    const int grid = grid_cap(grid_for_kernel(kern, 0), e_end - e_begin, kBlock);
    kern<<<grid, kBlock, 0, s>>>(e4, k, degrees, us, vs, e_begin, e_end, min_matches, tau, out_counts, nullptr);
  } else {
#define PG_L(V, G)                                                                                         \
  {                                                                                                        \
    auto kern = jaccard_khash_kernel<V, G, 1>;                                                             \
    const int grid = grid_cap(grid_for_kernel(kern, 0), e_end - e_begin, kBlock);                          \
    kern<<<grid, kBlock, 0, s>>>(e4, k, degrees, us, vs, e_begin, e_end, min_matches, tau, out_counts, nullptr);    \
  }
    PG_ROW_DISPATCH(w4, PG_L)
#undef PG_L
  }
  return check_launch("jaccard_khash");
}

}  // extern "C"
