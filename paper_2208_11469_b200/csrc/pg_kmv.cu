// KMV per-edge estimates (providers.py:266-301 KmvProvider.pair_many) and
// the fused KMV TC sum.
#include "pg_generic.cuh"

namespace pg {

// --------------------------------------------------------------- KMV ----
// Warp-per-edge restatement of the merged-row logic of providers.py:266-301:
// common = |U & V|, union = |U| + |V| - common, k_eff = min(|U|,|V|), kth =
// the max(k_eff,1)-th smallest distinct value of U | V (or merged[0] when
// the union is smaller).  Ranks of union elements are computed from
// lower_bound positions in the other row and prefix counts of common
// elements, so no merge buffer is needed.
struct KmvEdge {
  int common, uni, k_eff;
  double kth;
};

template <int P>
__device__ __forceinline__ KmvEdge kmv_edge(const uint64_t* __restrict__ vals, int k, int32_t u, int32_t v,
                                            uint64_t* ubuf, uint64_t* vbuf) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = lanemask_lt();
  uint64_t a[P], b[P];
  int lu = 0, lv = 0;
#pragma unroll
  for (int s = 0; s < P; ++s) {
    const int idx = lane + 32 * s;
    a[s] = idx < k ? vals[(int64_t)u * k + idx] : kInfBits;
    b[s] = idx < k ? vals[(int64_t)v * k + idx] : kInfBits;
    lu += __popc(__ballot_sync(0xffffffffu, a[s] < kInfBits));
    lv += __popc(__ballot_sync(0xffffffffu, b[s] < kInfBits));
    if (idx < k) { ubuf[idx] = a[s]; vbuf[idx] = b[s]; }
  }
  __syncwarp();
  int ltv[P], ltu[P];
  bool inv[P], inu[P];
  int common = 0;
#pragma unroll
  for (int s = 0; s < P; ++s) {
    const int idx = lane + 32 * s;
    inv[s] = false;
    inu[s] = false;
    ltv[s] = 0;
    ltu[s] = 0;
    if (idx < lu) {
      ltv[s] = smem_lower_bound(vbuf, lv, a[s]);
      inv[s] = ltv[s] < lv && vbuf[ltv[s]] == a[s];
    }
    if (idx < lv) {
      ltu[s] = smem_lower_bound(ubuf, lu, b[s]);
      inu[s] = ltu[s] < lu && ubuf[ltu[s]] == b[s];
    }
    common += __popc(__ballot_sync(0xffffffffu, inv[s]));
  }
  KmvEdge r;
  r.common = common;
  r.uni = lu + lv - common;
  r.k_eff = min(lu, lv);
  const int T = max(r.k_eff, 1);
  // rank (1-based) of each distinct union element; find rank T
  int before_u = 0, before_v = 0;
  uint64_t found = 0;
  bool have = false;
#pragma unroll
  for (int s = 0; s < P; ++s) {
    const int idx = lane + 32 * s;
    const unsigned bu = __ballot_sync(0xffffffffu, inv[s]);
    const unsigned bv = __ballot_sync(0xffffffffu, inu[s]);
    const int cbu = before_u + __popc(bu & lt);
    const int cbv = before_v + __popc(bv & lt);
    if (idx < lu && idx + 1 + ltv[s] - cbu == T) { found = a[s]; have = true; }
    if (idx < lv && !inu[s] && idx + 1 + ltu[s] - cbv == T) { found = b[s]; have = true; }
    before_u += __popc(bu);
    before_v += __popc(bv);
  }
  const unsigned hm = __ballot_sync(0xffffffffu, have);
  const uint64_t c1 = shfl64(found, hm ? __ffs(hm) - 1 : 0);
  const uint64_t a0 = shfl64(a[0], 0), b0 = shfl64(b[0], 0);
  r.kth = bitsd(hm ? c1 : min(a0, b0));  // no rank-T element: argmax of all-False -> merged[0]
  __syncwarp();
  return r;
}

__device__ __forceinline__ double kmv_estimate(const KmvEdge& r, int k, int32_t isu, int32_t isv) {
  const double su = (double)isu, sv = (double)isv;
  const double ssum = __dadd_rn(su, sv);
  double raw;
  if (isu <= k && isv <= k) raw = __dsub_rn(ssum, (double)r.uni);
  else if (r.k_eff < 2) raw = (double)r.common;
  else raw = __dsub_rn(ssum, __ddiv_rn((double)(r.k_eff - 1), r.kth));
  return fmin(fmax(raw, 0.0), fmin(su, sv));  // np.clip(raw, 0, min(su, sv))
}

template <int P, bool kFused>
__global__ void __launch_bounds__(kBlock) kmv_kernel(const uint64_t* vals, int k, const int32_t* sizes,
                                                    const int32_t* us, const int32_t* vs, int64_t e_begin,
                                                    int64_t e_end, int32_t* out_common, int32_t* out_union,
                                                    double* out_kth, double* out_est, double* out_sum) {
  __shared__ uint64_t ubuf[kBlock / 32][32 * P];
  __shared__ uint64_t vbuf[kBlock / 32][32 * P];
  __shared__ double red[kBlock / 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double acc = 0.0;
  int64_t wb, we;
  warp_slice(e_begin, e_end, wb, we);
  for (int64_t e = wb; e < we; ++e) {
    const int32_t u = us[e], v = vs[e];
    const KmvEdge r = kmv_edge<P>(vals, k, u, v, ubuf[w], vbuf[w]);
    if (lane == 0) {
      const double est = kmv_estimate(r, k, sizes[u], sizes[v]);
      if (kFused) acc = __dadd_rn(acc, est);
      else {
        if (out_common) out_common[e] = r.common;
        if (out_union) out_union[e] = r.uni;
        if (out_kth) out_kth[e] = r.kth;
        if (out_est) out_est[e] = est;
      }
    }
  }
  if (kFused) {
    if (lane == 0) red[w] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {  // out_sum: one partial per block (PartialSums)
      double t = 0.0;
      for (int i = 0; i < kBlock / 32; ++i) t = __dadd_rn(t, red[i]);
      out_sum[blockIdx.x] = t;
    }
  }
}

struct EpiKmv {
  int k;
  const int32_t* sizes;
  int32_t* out_common;
  int32_t* out_union;
  double* out_kth;
  double* out_est;
  bool fused;
  double acc;
  __device__ __forceinline__ void edge(int64_t e, int32_t u, int32_t v, const SortedStats& st) {
    KmvEdge r;
    r.common = st.common;
    r.uni = st.lu + st.lv - st.common;
    r.k_eff = min(st.lu, st.lv);
    r.kth = st.kth;
    const double est = kmv_estimate(r, k, sizes[u], sizes[v]);
    if (fused) {
      acc = __dadd_rn(acc, est);
    } else {
      if (out_common) out_common[e] = r.common;
      if (out_union) out_union[e] = r.uni;
      if (out_kth) out_kth[e] = r.kth;
      if (out_est) out_est[e] = est;
    }
  }
};

template <int G, int CH, bool kFused>
__global__ void __launch_bounds__(kBlock, 4) kmv_sorted_kernel(const uint64_t* vals, int k, const int32_t* sizes,
                                                           const int32_t* us, const int32_t* vs,
                                                           int64_t e_begin, int64_t e_end, int32_t* out_common,
                                                           int32_t* out_union, double* out_kth,
                                                           double* out_est, double* out_sum) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ double red[kBlock / 32];
  EpiKmv epi{k, sizes, out_common, out_union, out_kth, out_est, kFused, 0.0};
  merge_edge_loop<G, CH, true>(vals, k, us, vs, e_begin, e_end,
                               smem_raw + (threadIdx.x >> 5) * merge_warp_smem<G, CH, true>(), epi);
  if (kFused) {
    double a = epi.acc;
    for (int o = 16; o > 0; o >>= 1) a = __dadd_rn(a, __shfl_xor_sync(0xffffffffu, a, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = a;
    __syncthreads();
    if (threadIdx.x == 0) {  // out_sum: one partial per block (PartialSums)
      double t = 0.0;
      for (int i = 0; i < kBlock / 32; ++i) t = __dadd_rn(t, red[i]);
      out_sum[blockIdx.x] = t;
    }
  }
}


template <int G, int CH, bool kFused>
static void launch_kmv_sorted(cudaStream_t s, const uint64_t* vals, int k, const int32_t* sizes,
                              const int32_t* us, const int32_t* vs, int64_t b, int64_t e, int32_t* out_common,
                              int32_t* out_union, double* out_kth, double* out_est, double* out_sum) {
  auto kern = kmv_sorted_kernel<G, CH, kFused>;
  const size_t sm = (size_t)(kBlock / 32) * merge_warp_smem<G, CH, true>();
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  const int grid = grid_cap(grid_for_kernel(kern, sm), e - b, kBlock / G);
  PartialSums ps;  // fused: one partial per block, summed in block order
  if (kFused && ps.init(s, grid) != cudaSuccess) return;
  kern<<<grid, kBlock, sm, s>>>(vals, k, sizes, us, vs, b, e, out_common, out_union, out_kth, out_est,
                                kFused ? ps.p : nullptr);
  if (kFused) ps.finish(out_sum);
}

static bool kmv_sorted(cudaStream_t s, bool fused, const uint64_t* vals, int k, const int32_t* sizes,
                       const int32_t* us, const int32_t* vs, int64_t b, int64_t e, int32_t* out_common,
                       int32_t* out_union, double* out_kth, double* out_est, double* out_sum) {
#define PG_KS(G, CH)                                                                                       \
  {                                                                                                        \
    if (fused) launch_kmv_sorted<G, CH, true>(s, vals, k, sizes, us, vs, b, e, out_common, out_union,     \
                                              out_kth, out_est, out_sum);                                  \
    else launch_kmv_sorted<G, CH, false>(s, vals, k, sizes, us, vs, b, e, out_common, out_union, out_kth, \
                                         out_est, out_sum);                                                \
    return true;                                                                                           \
  }
  static const int lanes = [] {
    const char* v = getenv("PG_KMV_LANES");
    return v ? atoi(v) : 0;
  }();
  // 32 merge outputs per lane (two 8-element chunks of each row per lane):
  // the two bisections per lane amortise over twice the outputs of the
  // 16-output split (measured s20 k=64: 4.80 vs 5.85 ms); PG_KMV_LANES
  // selects the 16-output split for comparison
  if (k == 32) {
    if (lanes == 4) PG_KS(4, 1)
    PG_KS(2, 2)
  }
  if (k == 64) {
    if (lanes == 8) PG_KS(8, 1)
    PG_KS(4, 2)
  }
  if (k == 128) PG_KS(8, 2)
#undef PG_KS
  return false;
}

// ------------------------------------------ KMV rank-directory engine ----
#ifndef PG_RANKED_MINB
#define PG_RANKED_MINB 3
#endif
#ifndef PG_RANKED_PER_LANE
#define PG_RANKED_PER_LANE 8
#endif
constexpr int kRankedPerLane = PG_RANKED_PER_LANE;  // v-row ranks per lane
// Rows hold global value ranks (int32 ascending, INT32_MAX pad; built by
// pg_build_kmv_ranked from pg_kmv_rank_table): the same order and ties as
// the values, in half the bytes, with 32-bit compares.  The edge slots are
// row-padded to E = 32/G (pg_csr_upper_edges_padded), so every warp
// iteration holds E edges of one u.  When u changes, the warp builds a
// directory of u's row A in shared memory: NB = 2K buckets over
// [A[0], A[lu-1]] (monotone map: one IMAD.HI), each an int4 record
// {the bucket's three smallest elements (INT32_MAX pad), first index |
// count << 8}.  A probe of x is one LDS.128: lt = |A < x|, hit = x in A (a
// bucket with more than three elements finishes from the sorted copy of A).
// For the v row B (G lanes, 8 ranks each) the reference's merged-row
// quantities (providers.py:266-301) follow without merging:
//   common = sum(hit);  dist_j = |A <= b_j| + (j+1) - C_j, the number of
//   distinct union values <= b_j (C_j = inclusive prefix of hit);  the
//   T-th distinct union value (T = k_eff) is min(A[R + T - D - 1], b_{j*+1})
//   with j* the last j with dist_j < T, R = |A <= b_j*|, D = dist_j*
//   (R = D = 0 when there is none; b_lv = +inf).
template <int K>
struct RankDir {
  static constexpr int NB = 2 * K;
  int4 rec[NB];
  int32_t a[K + 4];
  int32_t dir[NB + 4];
};

__device__ __forceinline__ uint32_t rd_bucket(int32_t x, int32_t lo, int32_t spanm1, uint32_t mul) {
  return __umulhi((uint32_t)min(max(x - lo, 0), spanm1), mul);
}

template <int K>
__device__ __forceinline__ void rd_build(RankDir<K>& W, const int32_t* __restrict__ arow, int lu, int32_t& lo,
                                         int32_t& spanm1, uint32_t& mul) {
  constexpr int NB = RankDir<K>::NB;
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int s = 0; s < K / 32; ++s) W.a[lane + 32 * s] = __ldg(arow + lane + 32 * s);
  __syncwarp();
  lo = lu > 0 ? W.a[0] : 0;
  const int32_t hi = lu > 0 ? W.a[lu - 1] : 0;
  spanm1 = hi - lo;
  const uint32_t span = (uint32_t)spanm1 + 1u;
  mul = span > (uint32_t)NB ? (uint32_t)(((uint64_t)NB << 32) / span) : 0xFFFFFFFFu;
  // dir[b] = |{i : bucket(a_i) < b}| for b in [0, NB]: element i writes i
  // over the buckets (bucket(a_{i-1}), bucket(a_i)], the last one lu over
  // (bucket(a_{lu-1}), NB]
  if (lu == 0) {
    for (int b = lane; b <= NB; b += 32) W.dir[b] = 0;
  }
#pragma unroll
  for (int s = 0; s < K / 32; ++s) {
    const int i = lane + 32 * s;
    if (i < lu) {
      const int bk = (int)rd_bucket(W.a[i], lo, spanm1, mul);
      const int bp = i == 0 ? -1 : (int)rd_bucket(W.a[i - 1], lo, spanm1, mul);
      for (int b = bp + 1; b <= bk; ++b) W.dir[b] = i;
      if (i == lu - 1)
        for (int b = bk + 1; b <= NB; ++b) W.dir[b] = lu;
    }
  }
  __syncwarp();
#pragma unroll
  for (int t = 0; t < NB / 32; ++t) {
    const int b = lane + 32 * t;
    const int d = W.dir[b], c = W.dir[b + 1] - d;
    int4 r;
    r.x = c > 0 ? W.a[d] : INT32_MAX;
    r.y = c > 1 ? W.a[d + 1] : INT32_MAX;
    r.z = c > 2 ? W.a[d + 2] : INT32_MAX;
    r.w = d | (c << 8);
    W.rec[b] = r;
  }
  __syncwarp();
}

// le = |A <= x| and hit = (x in A) from the bucket record alone (exact when
// the bucket holds at most three elements; `ovf` flags the others)
template <int K>
__device__ __forceinline__ int rd_probe(const RankDir<K>& W, int32_t x, int32_t lo, int32_t spanm1, uint32_t mul,
                                        bool ok, bool& hit, bool& ovf) {
  int4 r = make_int4(INT32_MAX, INT32_MAX, INT32_MAX, 0);
  if (ok) r = W.rec[rd_bucket(x, lo, spanm1, mul)];
  hit = (r.x == x) | (r.y == x) | (r.z == x);
  ovf = r.w >= (4 << 8);
  return (r.w & 0xff) + (r.x <= x) + (r.y <= x) + (r.z <= x);
}
// the same for an overflowing bucket, from the sorted copy of A
template <int K>
__device__ __noinline__ int rd_probe_slow(const RankDir<K>& W, int32_t x, int32_t lo, int32_t spanm1, uint32_t mul,
                                          bool& hit) {
  const int w = W.rec[rd_bucket(x, lo, spanm1, mul)].w;
  const int d = w & 0xff, c = w >> 8;
  int le = d;
  hit = false;
  for (int i = 0; i < c; ++i) {
    const int32_t y = W.a[d + i];
    le += y <= x;
    hit |= y == x;
  }
  return le;
}

// Slot blocks: a warp walks its chunk 32 slots at a time; lane l holds slot
// l's u, v, sizes and lengths (loaded one block ahead, so no iteration waits
// on an index -> row chain), the groups take E slots per iteration (v by
// shuffle), and after the block every lane finishes one slot's estimate
// (the fp64 tail runs with all 32 lanes instead of one lane per group).
template <int K>
struct RankWarp {
  RankDir<K> dir;
  int2 buf[32];  // per slot of the block: {common | (j*+1) << 8, A[R+T-D-1]}
};

// P ranks of each v row per lane (G = K/P lanes per edge, E = 32/G edges per
// iteration; the slot layout is padded to E)
template <int K, int P>
__global__ void __launch_bounds__(kBlock, PG_RANKED_MINB) kmv_ranked_kernel(const int32_t* __restrict__ R,
                                                               const double* __restrict__ rank_values,
                                                               const int32_t* __restrict__ lengths,
                                                               const int32_t* __restrict__ sizes,
                                                               const int32_t* __restrict__ us,
                                                               const int32_t* __restrict__ vs, int64_t e_begin,
                                                               int64_t e_end, double* out_sum,
                                                               unsigned long long* ctr) {
  constexpr int G = K / P, E = 32 / G, IT = 32 / E;
  constexpr int64_t kChunk = 512;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  RankWarp<K>& Wp = reinterpret_cast<RankWarp<K>*>(smem_raw)[threadIdx.x >> 5];
  RankDir<K>& W = Wp.dir;
  const int lane = threadIdx.x & 31, gl = lane & (G - 1), grp = lane / G;
  double acc = 0.0;
  int32_t cur_u = -1, lo = 0, spanm1 = 0, lu = 0;
  uint32_t mul = 0;
  int64_t wb, we;
  while (next_chunk(ctr, e_begin, e_end, kChunk, wb, we)) {
    // this block's slot of lane l (u, v) and the gathers of its endpoints
    int32_t ul = 0, vl = -1;
    if (wb + lane < we) {
      ul = us[wb + lane];
      vl = vs[wb + lane];
    }
    int32_t svl = 0, lvl = 0, sul = sizes[ul], lul = lengths[ul];
    if (vl >= 0) {
      svl = sizes[vl];
      lvl = lengths[vl];
    }
    int32_t vq = __shfl_sync(0xffffffffu, vl, grp);
    uint32_t x[P];
    ldg_rowpart<P>(R + (int64_t)(vq < 0 ? 0 : vq) * K + gl * P, x);
#pragma unroll 1
    for (int64_t b0 = wb; b0 < we; b0 += 32) {
      // next block's slots (consumed IT iterations later)
      int32_t un = 0, vn = -1, sun = 0, lun = 0, svn = 0, lvn = 0;
      if (b0 + 32 + lane < we) {
        un = us[b0 + 32 + lane];
        vn = vs[b0 + 32 + lane];
      }
#pragma unroll 1
      for (int it = 0; it < IT; ++it) {
        const int slot = it * E + grp;
        const int32_t u = __shfl_sync(0xffffffffu, ul, it * E);  // one u per padded group
        const int lv = __shfl_sync(0xffffffffu, lvl, slot);
        const bool valid = b0 + slot < we && vq >= 0;
        if (it == IT / 2) {  // the next block's endpoint gathers, off the critical path
          sun = sizes[un];
          lun = lengths[un];
          if (vn >= 0) {
            svn = sizes[vn];
            lvn = lengths[vn];
          }
        }
        if (u != cur_u) {
          cur_u = u;
          lu = __shfl_sync(0xffffffffu, lul, it * E);
          rd_build<K>(W, R + (int64_t)u * K, lu, lo, spanm1, mul);
        }
        // the next iteration's v row (the next block's first at the end)
        const int32_t vqn = __shfl_sync(0xffffffffu, it + 1 < IT ? vl : vn, it + 1 < IT ? slot + E : grp);
        uint32_t xn[P];
        ldg_rowpart<P>(R + (int64_t)(vqn < 0 ? 0 : vqn) * K + gl * P, xn);
        // le_t = |A <= b_t| (<= K <= 128) packed four per register
        int le[P];
        unsigned hits = 0, ovf = 0;
#pragma unroll
        for (int t = 0; t < P; ++t) {
          const int32_t q = (int32_t)x[t];
          const bool ok = valid && q != INT32_MAX;
          bool h, o;
          const int l = rd_probe<K>(W, q, lo, spanm1, mul, ok, h, o);
          le[t] = ok ? l : 0;
          hits |= (unsigned)(ok && h) << t;
          ovf |= (unsigned)(ok && o) << t;
        }
        if (__any_sync(0xffffffffu, ovf != 0)) {  // buckets of four or more elements
#pragma unroll
          for (int t = 0; t < P; ++t) {
            if ((ovf >> t) & 1) {
              bool h;
              const int l = rd_probe_slow<K>(W, (int32_t)x[t], lo, spanm1, mul, h);
              le[t] = l;
              hits = (hits & ~(1u << t)) | ((unsigned)h << t);
            }
          }
        }
        const int mc = __popc(hits);
        int incl = mc;
#pragma unroll
        for (int o = 1; o < G; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, incl, o);
          if (gl >= o) incl += y;
        }
        const int common = __shfl_sync(0xffffffffu, incl, (grp + 1) * G - 1);
        const int T = min(lu, lv);
        // less = #t with dist_t < T (a prefix: dist is nondecreasing);
        // cand = (|A <= b|, dist) of this lane's last such element
        int C = incl - mc, less = 0, cand = 0;
#pragma unroll
        for (int t = 0; t < P; ++t) {
          const int j = gl * P + t;
          C += (hits >> t) & 1;
          const int let = le[t];
          const int dist = let + (j + 1) - C;
          if (j < lv && dist < T) {
            ++less;
            cand = let | (dist << 16);
          }
        }
        int tot = less;
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
        const int js = tot - 1;  // last j with dist_j < T
        const int pk = __shfl_sync(0xffffffffu, cand, grp * G + (js < 0 ? 0 : js / P));
        if (valid && gl == 0) {
          int ka = 0;
          if (T >= 2) {
            const int Rr = js < 0 ? 0 : (pk & 0xffff), D = js < 0 ? 0 : (pk >> 16);
            ka = W.a[Rr + T - D - 1];
          }
          Wp.buf[slot] = make_int2(common | ((js + 1) << 8), ka);
        }
#pragma unroll
        for (int t = 0; t < P; ++t) x[t] = xn[t];
        vq = vqn;
      }
      __syncwarp();
      // every lane finishes its slot: KMV estimate (providers.py:266-301)
      if (b0 + lane < we && vl >= 0) {
        const int2 bf = Wp.buf[lane];
        const int common = bf.x & 0xff, jn = bf.x >> 8;
        KmvEdge r;
        r.common = common;
        r.uni = lul + lvl - common;
        r.k_eff = min(lul, lvl);
        r.kth = 0.0;
        if (!(sul <= K && svl <= K) && r.k_eff >= 2) {
          const int32_t kb = jn < lvl ? __ldg(R + (int64_t)vl * K + jn) : INT32_MAX;
          r.kth = __ldg(rank_values + min(bf.y, kb));
        }
        acc = __dadd_rn(acc, kmv_estimate(r, K, sul, svl));
      }
      __syncwarp();
      ul = un;
      vl = vn;
      sul = sun;
      lul = lun;
      svl = svn;
      lvl = lvn;
    }
    // one partial per dynamic chunk (fixed boundaries), whichever warp ran it
    double a = acc;
    for (int o = 16; o > 0; o >>= 1) a = __dadd_rn(a, __shfl_xor_sync(0xffffffffu, a, o));
    if (lane == 0) out_sum[(wb - e_begin) / kChunk] = a;
    acc = 0.0;
  }
}

template <int K>
static int launch_kmv_ranked(cudaStream_t s, const int32_t* ranks, const double* rank_values,
                             const int32_t* lengths, const int32_t* sizes, const int32_t* us, const int32_t* vs,
                             int64_t b, int64_t e, double* out_sum) {
  constexpr int P = kRankedPerLane;
  auto kern = kmv_ranked_kernel<K, P>;
  const size_t sm = (size_t)(kBlock / 32) * sizeof(RankWarp<K>);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  const int grid = grid_cap(grid_for_kernel(kern, sm), e - b, kBlock / (K / P));
  ChunkCounter ctr;
  PartialSums ps;  // one partial per 512-slot chunk, summed in chunk order
  cudaError_t ce = ctr.init(s);
  if (ce == cudaSuccess) ce = ps.init(s, (e - b + 511) / 512);
  if (ce != cudaSuccess) return fail(PG_ERR_CUDA, "scratch: %s", cudaGetErrorString(ce));
  kern<<<grid, kBlock, sm, s>>>(ranks, rank_values, lengths, sizes, us, vs, b, e, ps.p, ctr.p);
  ps.finish(out_sum);
  return check_launch("tc_kmv_ranked");
}

// -------------------------------------- KMV thread-per-edge merge engine ----
// One lane per edge slot over the rank rows (int32 ascending, INT32_MAX pad).
// The reference's merged-row quantities (providers.py:266-301) need, for an
// edge whose estimate is s_u + s_v - (k_eff - 1) / kth, only the T-th
// (T = k_eff = min(lu, lv)) smallest distinct value of A | B: a sequential
// two-pointer merge yields it after exactly T steps (each step consumes the
// smaller head, or both heads when they are equal), never reading past index
// T - 1 of either row.  Edges of the other two branches (both sizes <= K:
// s_u + s_v - |A | B|; k_eff < 2: |A & B|) continue the same merge until one
// row is exhausted; |A & B| = i + j - steps.  The per-lane work is ~10
// instructions per step instead of K directory probes per edge (c3: 4.6 ms
// against 10.8 ms for the rank-directory engine above).
#ifndef PG_TMERGE_NU
#define PG_TMERGE_NU 8
#endif
__device__ __forceinline__ int32_t lds_s32(uint32_t addr) {
  int32_t x;
  asm volatile("ld.shared.s32 %0, [%1];" : "=r"(x) : "r"(addr));
  return x;
}
// v rows in shared memory: element j of lane r's row at byte X = base + j*128
// + r*4 (base 128-aligned), stored at swz(X) = X ^ (sector index of j moved
// onto the top bits of the lane field).  A warp-wide load instruction then
// covers 256/K whole rows (coalesced) and its transposing stores still hit 32
// distinct banks; lanes reading the same sector index never conflict.
template <int K>
__device__ __forceinline__ uint32_t tm_swz(uint32_t x) {
  constexpr int LP = K == 32 ? 2 : K == 64 ? 3 : 4;  // log2(sectors per row)
  return x ^ ((x >> (3 + LP)) & (((1u << LP) - 1u) << (7 - LP)));
}
// one merge step: consume the smaller head (both when equal); A rows are
// contiguous, a B column's elements are 128 bytes apart before the swizzle
template <int K>
__device__ __forceinline__ void tm_step(uint32_t& pa, uint32_t& pb) {
  const int32_t a = lds_s32(pa), b = lds_s32(tm_swz<K>(pb));
  if (a <= b) pa += 4;
  if (b <= a) pb += 128;
}
#ifndef PG_TM_UNCOND
#define PG_TM_UNCOND 1
#endif
#ifndef PG_TM_STEP2
#define PG_TM_STEP2 1
#endif
#ifndef PG_TM_DEFER
#define PG_TM_DEFER 1
#endif
#ifndef PG_TM_CHUNK
#define PG_TM_CHUNK 1024
#endif
#ifndef PG_TM_REVERSE
#define PG_TM_REVERSE 1
#endif
__device__ __forceinline__ int32_t lds_s32_always(uint32_t addr) {
  int32_t x;
  asm volatile("ld.volatile.shared.s32 %0, [%1];" : "=r"(x) : "r"(addr));
  return x;
}
// two merge steps from one round of loads (both heads and their successors):
// the loop-carried chain is load -> compare -> select -> compare instead of
// two load -> compare rounds.  A successor that is out of the row is read
// but never selected: step s only ever looks at indices <= s < k_eff.
template <int K>
__device__ __forceinline__ void tm_step2(uint32_t& pa, uint32_t& pb) {
  const int32_t a0 = lds_s32(pa), b0 = lds_s32(tm_swz<K>(pb));
#if PG_TM_STEP2 == 2
  const int32_t a1 = lds_s32_always(pa + 4), b1 = lds_s32_always(tm_swz<K>(pb + 128));
#else
  const int32_t a1 = lds_s32(pa + 4), b1 = lds_s32(tm_swz<K>(pb + 128));
#endif
  const bool ta = a0 <= b0, tb = b0 <= a0;
  const int32_t a = ta ? a1 : a0, b = tb ? b1 : b0;
  const bool ta2 = a <= b, tb2 = b <= a;
  pa += (ta ? 4u : 0u) + (ta2 ? 4u : 0u);
  pb += (tb ? 128u : 0u) + (tb2 ? 128u : 0u);
}
__device__ __forceinline__ void sts_u32(uint32_t addr, uint32_t x) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(x) : "memory");
}
__device__ __forceinline__ unsigned lanemask_le() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_le;" : "=r"(m));
  return m;
}

// Shared memory per warp (one warp per CTA): the v rows word-interleaved and
// swizzled ([K][32], tm_swz above), the u rows of the block once per distinct
// u (edge slots are in u runs; a block takes the slots of at most NU runs,
// rows skewed by 32/NU banks); 10.4 KB at K = 64: 20 resident warps per SM.
// Pipeline per warp: the slots of the block after next and the lengths/sizes
// of the next block are requested before the current block's rows, and a
// block's rank -> value gather is consumed one block later.
template <int K, int NU>
struct TmergeSmem {
  static constexpr int SK = 32 / NU, AS = K + SK;
  int32_t b[K * 32];
  int32_t a[NU * AS];
  int32_t uq[NU];
};

struct TmSlots {  // a block's slots, one per lane
  int32_t u, v;
  int q;       // index of the lane's u run within the block
  bool valid;  // a real edge of one of the first NU runs
  int cons;    // slots the block consumes (a prefix of the 32)
  unsigned heads;
};
template <int NU>
__device__ __forceinline__ void tm_form(TmSlots& b, int64_t start, int64_t we) {
  const int lane = threadIdx.x;
  const bool in = start + lane < we;
  const int32_t uu = in ? b.u : -1;
  const int32_t up = __shfl_up_sync(0xffffffffu, uu, 1);
  const bool head = lane == 0 || uu != up;
  b.heads = __ballot_sync(0xffffffffu, head);
  b.q = __popc(b.heads & lanemask_le()) - 1;
  const bool act = b.q < NU;
  b.cons = __popc(__ballot_sync(0xffffffffu, act));
  b.valid = act && in && b.v >= 0;
  b.u = uu;
}

template <int K, int NU, int MINB, int CH>
__global__ void __launch_bounds__(32, MINB) kmv_tmerge_kernel(const int32_t* __restrict__ R,
                                                        const double* __restrict__ rank_values,
                                                        const int32_t* __restrict__ lengths,
                                                        const int32_t* __restrict__ sizes,
                                                        const int32_t* __restrict__ us,
                                                        const int32_t* __restrict__ vs, int64_t e_begin,
                                                        int64_t e_end, double* out_sum,
                                                        unsigned long long* ctr) {
  using SM = TmergeSmem<K, NU>;
  constexpr int64_t kChunk = CH;  // compile-time: a run-time chunk size measured 4.80 vs 4.58 ms
  constexpr int S = K / 8;   // 32-byte sectors per row
  constexpr int W = K / 32;  // words of a u row per lane
  constexpr int AS = SM::AS;
  extern __shared__ __align__(1024) unsigned char tm_raw[];
  SM& sm = *reinterpret_cast<SM*>(tm_raw);
  const int lane = threadIdx.x;
  constexpr int RP = 32 / S;  // v rows per load instruction
  const int lp = lane % S, la = lane / S;  // the lane's sector and row within a load instruction
  const uint32_t sbb = (uint32_t)__cvta_generic_to_shared(sm.b);
  const uint32_t sb0 = sbb + 4u * lane;
  const uint32_t sa00 = (uint32_t)__cvta_generic_to_shared(sm.a);
  int64_t wb, we;
#if PG_TM_REVERSE
  // chunks are handed out last to first: the full merges, which the partition
  // puts at the end of the slot list, are the long jobs and start first
  const int64_t n_chunks = (e_end - e_begin + kChunk - 1) / kChunk;
  for (;;) {
    unsigned long long c = 0;
    if (lane == 0) c = atomicAdd(ctr, 1ull);
    c = __shfl_sync(0xffffffffu, c, 0);
    if ((int64_t)c >= n_chunks) break;
    const int64_t chunk_idx = n_chunks - 1 - (int64_t)c;
    wb = e_begin + chunk_idx * kChunk;
    we = min(wb + kChunk, e_end);
#else
  while (next_chunk(ctr, e_begin, e_end, kChunk, wb, we)) {
    const int64_t chunk_idx = (wb - e_begin) / kChunk;
#endif
    double acc = 0.0;
    // pending estimate of the previous block (its kth gather is in flight)
    bool p_valid = false;
    int p_su = 0, p_sv = 0;
    KmvEdge p_r{0, 0, 0, 0.0};
    // prime: the first block's slots and metadata, the second block's slots
    int64_t start = wb;
    TmSlots cur{0, -1, 0, false, 0, 0u};
    if (start + lane < we) {
      cur.u = us[start + lane];
      cur.v = vs[start + lane];
    }
    tm_form<NU>(cur, start, we);
    int lu = 0, lv = 0, su = 0, sv = 0;
    if (cur.valid) {
      lu = lengths[cur.u];
      lv = lengths[cur.v];
      su = sizes[cur.u];
      sv = sizes[cur.v];
    }
    int64_t start_n = start + cur.cons;
    TmSlots nxt{0, -1, 0, false, 0, 0u};
    if (start_n + lane < we) {
      nxt.u = us[start_n + lane];
      nxt.v = vs[start_n + lane];
    }
#pragma unroll 1
    while (start < we) {
      // ---- next block: form it, fetch its metadata and the block after it
      tm_form<NU>(nxt, start_n, we);
      const int64_t start_nn = start_n + nxt.cons;
#if PG_TM_DEFER
      // unconditional loads (clamped indices), masked where they are used one
      // iteration later: a guarded load compiles to load + predicated move,
      // i.e. a wait for the load right where it is issued
      const int32_t mu = nxt.valid ? nxt.u : 0, mv = nxt.valid ? nxt.v : 0;
      int lun = lengths[mu], lvn = lengths[mv], sun = sizes[mu], svn = sizes[mv];
      const bool validn = nxt.valid;
      const int64_t e2 = min(start_nn + lane, e_end - 1);
      int32_t u2 = us[e2], v2 = vs[e2];
#else
      int lun = 0, lvn = 0, sun = 0, svn = 0;
      if (nxt.valid) {
        lun = lengths[nxt.u];
        lvn = lengths[nxt.v];
        sun = sizes[nxt.u];
        svn = sizes[nxt.v];
      }
      int32_t u2 = 0, v2 = -1;
      if (start_nn + lane < we) {
        u2 = us[start_nn + lane];
        v2 = vs[start_nn + lane];
      }
#endif
      // ---- current block: rows into shared memory
      const bool valid = cur.valid;
      const int T = min(lu, lv);
      // both sizes <= K (union count) or k_eff < 2 (common count): full merge
      const bool full = valid && ((su <= K && sv <= K) || T < 2);
      const int nb = valid ? (full ? lv : T) : 0;
      const int nq = min(__popc(cur.heads), NU);
      __syncwarp();  // every lane is done with the previous block's u rows
      if (cur.q < NU && ((cur.heads >> lane) & 1u)) sm.uq[cur.q] = cur.u;
      __syncwarp();
      uint32_t xa[NU][W];
#pragma unroll
      for (int r = 0; r < NU; ++r) {
        if (r < nq) {
          const int32_t ur = sm.uq[r];
          const int32_t* ra = R + (int64_t)(ur < 0 ? 0 : ur) * K + W * lane;
          if (W == 1) xa[r][0] = __ldg(reinterpret_cast<const uint32_t*>(ra));
          else if (W == 2) {
            const uint2 t = __ldg(reinterpret_cast<const uint2*>(ra));
            xa[r][0] = t.x;
            xa[r][1] = t.y;
          } else {
            const uint4 t = __ldg(reinterpret_cast<const uint4*>(ra));
            xa[r][0] = t.x;
            xa[r][1] = t.y;
            xa[r][2 % W] = t.z;
            xa[r][3 % W] = t.w;
          }
        }
      }
#pragma unroll
      for (int h = 0; h < S; h += 4) {
        // instruction i covers rows RP*i .. RP*i + RP - 1, S lanes (sectors) each
        uint32_t xb[4][8];
        bool ok[4];
#pragma unroll
        for (int s = 0; s < 4; ++s) {
          const int r = RP * (h + s) + la;
          const int32_t vr = __shfl_sync(0xffffffffu, valid ? cur.v : 0, r);
          const int nbr = __shfl_sync(0xffffffffu, nb, r);
          ok[s] = h + s < S && lp * 8 < nbr;
#if PG_TM_UNCOND
          // unconditional (a lane with nothing to fetch re-reads the first
          // sector of the matrix): a predicated asm load is followed by
          // predicated moves of its results, i.e. a wait right where it is issued
          if (h + s < S) ldg256_keep(ok[s] ? R + (int64_t)vr * K + lp * 8 : R, xb[s]);
#else
          if (ok[s]) ldg256_keep(R + (int64_t)vr * K + lp * 8, xb[s]);
#endif
        }
        if (h == 0) {
#pragma unroll
          for (int r = 0; r < NU; ++r) {
            if (r < nq) {
              int32_t* dst = sm.a + r * AS + W * lane;
              if (W == 1) dst[0] = (int32_t)xa[r][0];
              else if (W == 2) *reinterpret_cast<uint2*>(dst) = make_uint2(xa[r][0], xa[r][1]);
              else *reinterpret_cast<uint4*>(dst) = make_uint4(xa[r][0], xa[r][1], xa[r][2 % W], xa[r][3 % W]);
            }
          }
        }
#pragma unroll
        for (int s = 0; s < 4; ++s) {
          if (ok[s]) {
            const uint32_t x0 = sbb + (uint32_t)(lp * 8) * 128u + (uint32_t)(RP * (h + s) + la) * 4u;
#pragma unroll
            for (int q = 0; q < 8; ++q) sts_u32(tm_swz<K>(x0 + q * 128u), xb[s][q]);
          }
        }
      }
      // the previous block's estimates (their kth gathers have landed)
      if (p_valid) acc = __dadd_rn(acc, kmv_estimate(p_r, K, p_su, p_sv));
      __syncwarp();  // the u rows are visible to every lane
      // ---- T steps: the T-th distinct value of A | B is the last one consumed
      const uint32_t sa0 = sa00 + (uint32_t)(min(cur.q, NU - 1) * AS) * 4u;
      uint32_t pa = sa0, pb = sb0;  // shared-space byte addresses of the heads
      int s = T;
#pragma unroll 1
#if PG_TM_STEP2
      for (; s >= 2; s -= 2) tm_step2<K>(pa, pb);
#else
      for (; s >= 2; s -= 2) {
        tm_step<K>(pa, pb);
        tm_step<K>(pa, pb);
      }
#endif
      if (s) tm_step<K>(pa, pb);
      int32_t kr = 0;
      if (T >= 1) {
        const int32_t la = pa > sa0 ? lds_s32(pa - 4) : -1, lb = pb > sb0 ? lds_s32(tm_swz<K>(pb - 128)) : -1;
        kr = max(la, lb);
      }
      int steps = T;
      if (full) {
        const uint32_t ea = sa0 + lu * 4, eb = sb0 + lv * 128;
#pragma unroll 1
        while (pa < ea && pb < eb) {
          tm_step<K>(pa, pb);
          ++steps;
        }
      }
      p_valid = valid;
      p_su = su;
      p_sv = sv;
      // |A & B| is exact once a row is exhausted (used only by full merges)
      p_r.common = (int)((pa - sa0) >> 2) + (int)((pb - sb0) >> 7) - steps;
      p_r.uni = lu + lv - p_r.common;
      p_r.k_eff = T;
      p_r.kth = (valid && T >= 2) ? __ldg(rank_values + kr) : 0.0;
      // ---- rotate
      start = start_n;
      start_n = start_nn;
      cur = nxt;
#if PG_TM_DEFER
      lu = validn ? lun : 0;
      lv = validn ? lvn : 0;
      su = validn ? sun : 0;
      sv = validn ? svn : 0;
#else
      lu = lun;
      lv = lvn;
      su = sun;
      sv = svn;
#endif
      nxt.u = u2;
      nxt.v = v2;
    }
    if (p_valid) acc = __dadd_rn(acc, kmv_estimate(p_r, K, p_su, p_sv));
    // one partial per dynamic chunk (fixed boundaries), whichever warp ran it
    for (int o = 16; o > 0; o >>= 1) acc = __dadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, o));
    if (lane == 0) out_sum[chunk_idx] = acc;
  }
}

template <int K, int NU, int MINB, int CH>
static int launch_kmv_tmerge_c(cudaStream_t s, const int32_t* ranks, const double* rank_values,
                               const int32_t* lengths, const int32_t* sizes, const int32_t* us,
                               const int32_t* vs, int64_t b, int64_t e, double* out_sum, int per_sm) {
  auto kern = kmv_tmerge_kernel<K, NU, MINB, CH>;
  const size_t sm = sizeof(TmergeSmem<K, NU>);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  const int grid = grid_cap(sm_count() * per_sm, e - b, CH);
  ChunkCounter ctr;
  PartialSums ps;  // one partial per chunk, summed in chunk order
  cudaError_t ce = ctr.init(s);
  if (ce == cudaSuccess) ce = ps.init(s, (e - b + CH - 1) / CH);
  if (ce != cudaSuccess) return fail(PG_ERR_CUDA, "scratch: %s", cudaGetErrorString(ce));
  kern<<<grid, 32, sm, s>>>(ranks, rank_values, lengths, sizes, us, vs, b, e, ps.p, ctr.p);
  ps.finish(out_sum);
  return check_launch("tc_kmv_merge");
}

template <int K, int NU, int MINB>
static int launch_kmv_tmerge_v(cudaStream_t s, const int32_t* ranks, const double* rank_values,
                               const int32_t* lengths, const int32_t* sizes, const int32_t* us,
                               const int32_t* vs, int64_t b, int64_t e, double* out_sum) {
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kmv_tmerge_kernel<K, NU, MINB, PG_TM_CHUNK>, 32,
                                                    sizeof(TmergeSmem<K, NU>)) != cudaSuccess || per_sm < 1)
    per_sm = 1;
  static const int cap = [] {
    const char* v = getenv("PG_TMERGE_WARPS");
    return v ? atoi(v) : 0;
  }();
  if (cap > 0) per_sm = min(per_sm, cap);
  // dynamic chunks of PG_TM_CHUNK slots; a short range (one shard's share of
  // the full-merge part, say) takes smaller ones so that every resident warp
  // still gets about four.  The chunk size is a function of the range and the
  // device alone: sums stay reproducible for a given (e_begin, e_end).
  const int64_t want = (e - b) / ((int64_t)sm_count() * per_sm * 4);
#define PG_TMC(CH) return launch_kmv_tmerge_c<K, NU, MINB, CH>(s, ranks, rank_values, lengths, sizes, us, vs, b, e, out_sum, per_sm)
  if (want >= PG_TM_CHUNK) PG_TMC(PG_TM_CHUNK);
  if (want >= PG_TM_CHUNK / 2) PG_TMC(PG_TM_CHUNK / 2);
  if (want >= PG_TM_CHUNK / 4) PG_TMC(PG_TM_CHUNK / 4);
  PG_TMC(PG_TM_CHUNK / 8);
#undef PG_TMC
}

template <int K>
static int launch_kmv_tmerge(cudaStream_t s, const int32_t* ranks, const double* rank_values,
                             const int32_t* lengths, const int32_t* sizes, const int32_t* us, const int32_t* vs,
                             int64_t b, int64_t e, double* out_sum) {
  // resident warps (CTAs) per SM the register allocation aims at; shared
  // memory allows 20 at K = 64.  Measured at c3: 16 warps 5.0 ms, 18 4.77,
  // 20 4.64; NU = 4 (more truncated blocks) 7.2 vs 6.4 ms on an earlier version
  constexpr int M1 = K == 32 ? 24 : K == 64 ? 20 : 11, M0 = K == 32 ? 20 : K == 64 ? 16 : 8;
  static const int var = [] {
    const char* v = getenv("PG_TMERGE_VARIANT");
    return v ? atoi(v) : 0;
  }();
#define PG_TM(NU, MB) return launch_kmv_tmerge_v<K, NU, MB>(s, ranks, rank_values, lengths, sizes, us, vs, b, e, out_sum)
  if (var == 1) PG_TM(PG_TMERGE_NU, M0);
  PG_TM(PG_TMERGE_NU, M1);
#undef PG_TM
}

// Stable counting sort of edge slots for the merge engine into B + 1
// classes: the slots whose merge stops after k_eff steps by k_eff bucket
// ((k_eff - 1) * B / k, ascending; B = 1: one class), then the full-merge
// slots (both sizes <= k, or k_eff < 2) and pads, so the warps of a block of
// slots run equally long and the long merges do not hold up the short ones.
constexpr int kPartTile = 2048;
constexpr int kPartMaxClasses = 9;
__device__ __forceinline__ int tmerge_class(const int32_t* __restrict__ sizes,
                                            const int32_t* __restrict__ lengths, int k, int B, int32_t u,
                                            int32_t v) {
  if (v < 0) return B;
  const int su = sizes[u], sv = sizes[v];
  const int T = min(lengths[u], lengths[v]);
  if ((su <= k && sv <= k) || T < 2) return B;
  return (T - 1) * B / k;
}
// tile_cnt[c * tiles + tile] = slots of class c in the tile
__global__ void __launch_bounds__(256) tmerge_count_kernel(const int32_t* __restrict__ us,
                                                           const int32_t* __restrict__ vs, int64_t count,
                                                           const int32_t* __restrict__ sizes,
                                                           const int32_t* __restrict__ lengths, int k, int B,
                                                           int64_t tiles, int64_t* tile_cnt) {
  __shared__ int cnt_s[kPartMaxClasses];
  if (threadIdx.x < kPartMaxClasses) cnt_s[threadIdx.x] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * kPartTile;
  for (int i = threadIdx.x; i < kPartTile; i += 256) {
    const int64_t e = base + i;
    int c = -1;
    if (e < count) c = tmerge_class(sizes, lengths, k, B, us[e], vs[e]);
    for (int z = 0; z <= B; ++z) {
      const unsigned m = __ballot_sync(0xffffffffu, c == z);
      if ((threadIdx.x & 31) == 0 && m) atomicAdd(&cnt_s[z], __popc(m));
    }
  }
  __syncthreads();
  if (threadIdx.x <= B) tile_cnt[(int64_t)threadIdx.x * tiles + blockIdx.x] = cnt_s[threadIdx.x];
}
// exclusive scan of `len` counts in place (one block); total -> a[len]
__global__ void __launch_bounds__(1024) tmerge_scan_kernel(int64_t* a, int64_t len) {
  __shared__ int64_t part[1024];
  const int64_t per = (len + 1023) / 1024;
  const int64_t lo = min((int64_t)threadIdx.x * per, len), hi = min(lo + per, len);
  int64_t t = 0;
  for (int64_t i = lo; i < hi; ++i) t += a[i];
  part[threadIdx.x] = t;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t run = 0;
    for (int i = 0; i < 1024; ++i) {
      const int64_t x = part[i];
      part[i] = run;
      run += x;
    }
    a[len] = run;
  }
  __syncthreads();
  int64_t run = part[threadIdx.x];
  for (int64_t i = lo; i < hi; ++i) {
    const int64_t x = a[i];
    a[i] = run;
    run += x;
  }
}
__global__ void __launch_bounds__(256) tmerge_scatter_kernel(const int32_t* __restrict__ us,
                                                             const int32_t* __restrict__ vs, int64_t count,
                                                             const int32_t* __restrict__ sizes,
                                                             const int32_t* __restrict__ lengths, int k, int B,
                                                             const int64_t* __restrict__ tile_off,
                                                             int64_t tiles, int32_t* out_us, int32_t* out_vs) {
  __shared__ int wcnt[8][kPartMaxClasses];
  __shared__ int64_t run_s[kPartMaxClasses];  // next output slot of each class for this tile
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t base = (int64_t)blockIdx.x * kPartTile;
  if (threadIdx.x <= B) run_s[threadIdx.x] = tile_off[(int64_t)threadIdx.x * tiles + blockIdx.x];
  __syncthreads();
  for (int i0 = 0; i0 < kPartTile; i0 += 256) {
    const int64_t e = base + i0 + threadIdx.x;
    int32_t u = 0, v = -1;
    int c = -1;
    if (e < count) {
      u = us[e];
      v = vs[e];
      c = tmerge_class(sizes, lengths, k, B, u, v);
    }
    int my_rank = 0;
    for (int z = 0; z <= B; ++z) {
      const unsigned m = __ballot_sync(0xffffffffu, c == z);
      if (lane == 0) wcnt[w][z] = __popc(m);
      if (c == z) my_rank = __popc(m & lanemask_lt());
    }
    __syncthreads();
    if (c >= 0) {
      int before = 0;
      for (int i = 0; i < w; ++i) before += wcnt[i][c];
      const int64_t pos = run_s[c] + before + my_rank;
      out_us[pos] = u;
      out_vs[pos] = v;
    }
    __syncthreads();
    if (threadIdx.x <= B) {
      int t = 0;
      for (int i = 0; i < 8; ++i) t += wcnt[i][threadIdx.x];
      run_s[threadIdx.x] += t;
    }
    __syncthreads();
  }
}

}  // namespace pg

using namespace pg;

extern "C" {


int pg_pairs_kmv(const double* values, const int32_t* lengths, int32_t k, const int32_t* sizes,
                 const int32_t* us, const int32_t* vs, int64_t count, int32_t* out_common,
                 int32_t* out_union, double* out_kth, double* out_est, void* stream) {
  (void)lengths;  // lengths are implied by the +inf pads of each row
  PG_REQUIRE(k >= 1, "k must be >= 1");
  PG_REQUIRE(count >= 0, "count must be >= 0");
  if (count == 0) return PG_OK;
  PG_REQUIRE(values && sizes && us && vs, "null pointer");
  cudaStream_t s = as_stream(stream);
  const uint64_t* vb = reinterpret_cast<const uint64_t*>(values);
  if (k > kMaxSketchK)
    return gen_pairs_kmv(vb, k, sizes, us, vs, count, out_common, out_union, out_kth, out_est, s);
  if (kmv_sorted(s, false, vb, k, sizes, us, vs, 0, count, out_common, out_union, out_kth, out_est, nullptr))
    return check_launch("pairs_kmv_sorted");
  const int grid = grid_cap(sm_count() * 8, count, kBlock / 32);
#define PG_KM(P) kmv_kernel<P, false><<<grid, kBlock, 0, s>>>(vb, k, sizes, us, vs, 0, count, out_common, out_union, out_kth, out_est, nullptr)
  if (k <= 32) PG_KM(1);
  else if (k <= 64) PG_KM(2);
  else if (k <= 128) PG_KM(4);
  else PG_KM(8);
#undef PG_KM
  return check_launch("pairs_kmv");
}

int pg_tc_kmv(const double* values, const int32_t* lengths, int32_t k, const int32_t* sizes,
              const int32_t* us, const int32_t* vs, int64_t e_begin, int64_t e_end, double* out_sum,
              void* stream) {
  (void)lengths;
  PG_REQUIRE(k >= 1, "k must be >= 1");
  PG_REQUIRE(0 <= e_begin && e_begin <= e_end, "bad edge range");
  PG_REQUIRE(out_sum, "null pointer");
  cudaStream_t s = as_stream(stream);
  cudaError_t ce = cudaMemsetAsync(out_sum, 0, sizeof(double), s);
  if (ce != cudaSuccess) return fail(PG_ERR_CUDA, "memset: %s", cudaGetErrorString(ce));
  if (e_end == e_begin) return PG_OK;  // an empty range needs no inputs
  PG_REQUIRE(values && us && vs && sizes, "null pointer");
  const uint64_t* vb = reinterpret_cast<const uint64_t*>(values);
  if (k > kMaxSketchK) return gen_tc_kmv(vb, k, sizes, us, vs, e_begin, e_end, out_sum, s);
  if (kmv_sorted(s, true, vb, k, sizes, us, vs, e_begin, e_end, nullptr, nullptr, nullptr, nullptr, out_sum))
    return check_launch("tc_kmv_sorted");
#define PG_KM(P)                                                                                    \
  {                                                                                                 \
    auto kern = kmv_kernel<P, true>;                                                                \
    const int grid = grid_cap(grid_for_kernel(kern, 0), e_end - e_begin, kBlock / 32);              \
    PartialSums ps;                                                                                 \
    if ((ce = ps.init(s, grid)) != cudaSuccess) return fail(PG_ERR_CUDA, "scratch: %s", cudaGetErrorString(ce)); \
    kern<<<grid, kBlock, 0, s>>>(vb, k, sizes, us, vs, e_begin, e_end, nullptr, nullptr, nullptr, nullptr, ps.p); \
    ps.finish(out_sum);                                                                             \
  }
  if (k <= 32) PG_KM(1)
  else if (k <= 64) PG_KM(2)
  else if (k <= 128) PG_KM(4)
  else PG_KM(8)
#undef PG_KM
  return check_launch("tc_kmv");
}

int pg_kmv_ranked_pad(int32_t k, int32_t* pad_host) {
  PG_REQUIRE(pad_host, "null output");
  *pad_host = (k == 32 || k == 64 || k == 128) ? 32 * kRankedPerLane / k : 0;
  return PG_OK;
}

int pg_tc_kmv_ranked(const int32_t* ranks, const double* rank_values, const int32_t* lengths, int32_t k,
                     const int32_t* sizes, const int32_t* us, const int32_t* vs, int64_t e_begin, int64_t e_end,
                     double* out_sum, void* stream) {
  if (k != 32 && k != 64 && k != 128)
    return fail(PG_ERR_UNSUPPORTED, "the rank-directory KMV engine supports k = 32, 64, 128 (got %d)", k);
  const int pad = 32 * kRankedPerLane / k;
  PG_REQUIRE(0 <= e_begin && e_begin <= e_end, "bad edge range");
  PG_REQUIRE(e_begin % pad == 0, "e_begin must be a multiple of the layout pad %d", pad);
  PG_REQUIRE(out_sum, "null pointer");
  cudaStream_t s = as_stream(stream);
  cudaError_t ce = cudaMemsetAsync(out_sum, 0, sizeof(double), s);
  if (ce != cudaSuccess) return fail(PG_ERR_CUDA, "memset: %s", cudaGetErrorString(ce));
  if (e_end == e_begin) return PG_OK;  // an empty range needs no inputs
  PG_REQUIRE(ranks && rank_values && lengths && sizes && us && vs, "null pointer");
  if (k == 32) return launch_kmv_ranked<32>(s, ranks, rank_values, lengths, sizes, us, vs, e_begin, e_end, out_sum);
  if (k == 64) return launch_kmv_ranked<64>(s, ranks, rank_values, lengths, sizes, us, vs, e_begin, e_end, out_sum);
  return launch_kmv_ranked<128>(s, ranks, rank_values, lengths, sizes, us, vs, e_begin, e_end, out_sum);
}

int pg_kmv_merge_supported(int32_t k, int32_t* ok_host) {
  PG_REQUIRE(ok_host, "null output");
  *ok_host = (k == 32 || k == 64 || k == 128) ? 1 : 0;
  return PG_OK;
}

int pg_tc_kmv_merge(const int32_t* ranks, const double* rank_values, const int32_t* lengths, int32_t k,
                    const int32_t* sizes, const int32_t* us, const int32_t* vs, int64_t e_begin, int64_t e_end,
                    double* out_sum, void* stream) {
  if (k != 32 && k != 64 && k != 128)
    return fail(PG_ERR_UNSUPPORTED, "the KMV merge engine supports k = 32, 64, 128 (got %d)", k);
  PG_REQUIRE(0 <= e_begin && e_begin <= e_end, "bad edge range");
  PG_REQUIRE(out_sum, "null pointer");
  cudaStream_t s = as_stream(stream);
  cudaError_t ce = cudaMemsetAsync(out_sum, 0, sizeof(double), s);
  if (ce != cudaSuccess) return fail(PG_ERR_CUDA, "memset: %s", cudaGetErrorString(ce));
  if (e_end == e_begin) return PG_OK;  // an empty range needs no inputs
  PG_REQUIRE(ranks && rank_values && lengths && sizes && us && vs, "null pointer");
  if (k == 32) return launch_kmv_tmerge<32>(s, ranks, rank_values, lengths, sizes, us, vs, e_begin, e_end, out_sum);
  if (k == 64) return launch_kmv_tmerge<64>(s, ranks, rank_values, lengths, sizes, us, vs, e_begin, e_end, out_sum);
  return launch_kmv_tmerge<128>(s, ranks, rank_values, lengths, sizes, us, vs, e_begin, e_end, out_sum);
}

int pg_kmv_merge_partition(const int32_t* us, const int32_t* vs, int64_t count, const int32_t* sizes,
                           const int32_t* lengths, int32_t k, int32_t keff_buckets, int32_t* out_us,
                           int32_t* out_vs, int64_t* split_host, void* stream) {
  PG_REQUIRE(k >= 1, "k must be >= 1");
  PG_REQUIRE(count >= 0, "count must be >= 0");
  PG_REQUIRE(keff_buckets >= 1 && keff_buckets < kPartMaxClasses, "keff_buckets must be in [1, %d]",
             kPartMaxClasses - 1);
  PG_REQUIRE(split_host, "null output");
  *split_host = 0;
  if (count == 0) return PG_OK;
  PG_REQUIRE(us && vs && sizes && lengths && out_us && out_vs, "null pointer");
  PG_REQUIRE(us != out_us && vs != out_vs, "the partition is not in place");
  cudaStream_t s = as_stream(stream);
  const int B = keff_buckets;
  const int64_t tiles = (count + kPartTile - 1) / kPartTile, len = (int64_t)(B + 1) * tiles;
  int64_t* tile_cnt = nullptr;
  retain_default_pool();
  cudaError_t ce = cudaMallocAsync(reinterpret_cast<void**>(&tile_cnt), sizeof(int64_t) * (len + 1), s);
  if (ce != cudaSuccess) return fail(PG_ERR_CUDA, "scratch: %s", cudaGetErrorString(ce));
  tmerge_count_kernel<<<(unsigned)tiles, 256, 0, s>>>(us, vs, count, sizes, lengths, k, B, tiles, tile_cnt);
  tmerge_scan_kernel<<<1, 1024, 0, s>>>(tile_cnt, len);
  tmerge_scatter_kernel<<<(unsigned)tiles, 256, 0, s>>>(us, vs, count, sizes, lengths, k, B, tile_cnt, tiles,
                                                         out_us, out_vs);
  // the full-merge class starts where class B's first tile does
  ce = cudaMemcpyAsync(split_host, tile_cnt + (int64_t)B * tiles, sizeof(int64_t), cudaMemcpyDeviceToHost, s);
  if (ce == cudaSuccess) ce = cudaStreamSynchronize(s);
  cudaFreeAsync(tile_cnt, s);
  if (ce != cudaSuccess) return fail(PG_ERR_CUDA, "partition: %s", cudaGetErrorString(ce));
  return check_launch("kmv_merge_partition");
}

}  // extern "C"
