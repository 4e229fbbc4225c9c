// KMV per-edge estimates (providers.py:266-301 KmvProvider.pair_many) and
// the fused KMV TC sum.
#include "pg_engines.cuh"

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
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int i = 0; i < kBlock / 32; ++i) t = __dadd_rn(t, red[i]);
      if (t != 0.0) atomicAdd(out_sum, t);
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
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int i = 0; i < kBlock / 32; ++i) t = __dadd_rn(t, red[i]);
      if (t != 0.0) atomicAdd(out_sum, t);
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
  kern<<<grid, kBlock, sm, s>>>(vals, k, sizes, us, vs, b, e, out_common, out_union, out_kth, out_est, out_sum);
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
}  // namespace pg

using namespace pg;

extern "C" {


int pg_pairs_kmv(const double* values, const int32_t* lengths, int32_t k, const int32_t* sizes,
                 const int32_t* us, const int32_t* vs, int64_t count, int32_t* out_common,
                 int32_t* out_union, double* out_kth, double* out_est, void* stream) {
  (void)lengths;  // lengths are implied by the +inf pads of each row
  PG_REQUIRE(k >= 1, "k must be >= 1");
  if (k > kMaxSketchK) return fail(PG_ERR_UNSUPPORTED, "k=%d exceeds the device limit %d", k, kMaxSketchK);
  PG_REQUIRE(count >= 0, "count must be >= 0");
  if (count == 0) return PG_OK;
  PG_REQUIRE(values && sizes && us && vs, "null pointer");
  cudaStream_t s = as_stream(stream);
  const uint64_t* vb = reinterpret_cast<const uint64_t*>(values);
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
  if (k > kMaxSketchK) return fail(PG_ERR_UNSUPPORTED, "k=%d exceeds the device limit %d", k, kMaxSketchK);
  PG_REQUIRE(0 <= e_begin && e_begin <= e_end, "bad edge range");
  PG_REQUIRE(out_sum, "null pointer");
  cudaStream_t s = as_stream(stream);
  cudaError_t ce = cudaMemsetAsync(out_sum, 0, sizeof(double), s);
  if (ce != cudaSuccess) return fail(PG_ERR_CUDA, "memset: %s", cudaGetErrorString(ce));
  if (e_end == e_begin) return PG_OK;  // an empty range needs no inputs
  PG_REQUIRE(values && us && vs && sizes, "null pointer");
  const uint64_t* vb = reinterpret_cast<const uint64_t*>(values);
  if (kmv_sorted(s, true, vb, k, sizes, us, vs, e_begin, e_end, nullptr, nullptr, nullptr, nullptr, out_sum))
    return check_launch("tc_kmv_sorted");
#define PG_KM(P)                                                                                    \
  {                                                                                                 \
    auto kern = kmv_kernel<P, true>;                                                                \
    const int grid = grid_cap(grid_for_kernel(kern, 0), e_end - e_begin, kBlock / 32);              \
    kern<<<grid, kBlock, 0, s>>>(vb, k, sizes, us, vs, e_begin, e_end, nullptr, nullptr, nullptr, nullptr, out_sum); \
  }
  if (k <= 32) PG_KM(1)
  else if (k <= 64) PG_KM(2)
  else if (k <= 128) PG_KM(4)
  else PG_KM(8)
#undef PG_KM
  return check_launch("tc_kmv");
}

}  // extern "C"
