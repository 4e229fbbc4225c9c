// Bloom per-edge estimates (providers.py:137-162 pair_many, _estimate_ones;
// estimators.py:65-70 swamidass_value) and the fused Bloom TC reduction
// (mining.py:105-130 tc_estimate over _chunked_sum :63-80).
#include "pg_generic.cuh"

#ifndef PG_WIDE_MINB
#define PG_WIDE_MINB 3  // CTAs/SM of the L1-cached group-u wide kernel
#endif

namespace pg {

// ------------------------------------------------ fixed-row kernels ----
template <int V, int G, class Op>
__global__ void __launch_bounds__(kBlock) pairs_rows_kernel_bloom(const uint4* rows, const int32_t* us,
                                                                 const int32_t* vs, int64_t count,
                                                                 EpiBloomPairs epi) {
  group_edge_loop<V, G, Op>(rows, us, vs, 0, count, epi);
}
__global__ void __launch_bounds__(kBlock) pairs_scalar_kernel_bloom(const uint64_t* rows, int words,
                                                                   const int32_t* us, const int32_t* vs,
                                                                   int64_t count, EpiBloomPairs epi) {
  scalar_edge_loop_bloom(rows, words, epi.op, us, vs, 0, count, epi);
}

template <int V, int G, class Op, bool kScalar, int MINB = 1, bool kVCache = false>
__global__ void __launch_bounds__(kBlock, MINB) tc_bloom_kernel(const uint4* rows, int bits, const int32_t* us,
                                                         const int32_t* vs, int64_t e_begin,
                                                         int64_t e_end, EpiBloomHist epi,
                                                         int64_t* out_hist, int64_t* out_sum_pos) {
  extern __shared__ int hist_s[];
  for (int i = threadIdx.x; i <= bits; i += blockDim.x) hist_s[i] = 0;
  __syncthreads();
  epi.hist_s = hist_s;
  epi.sum_pos = 0;
  if (kScalar)
    scalar_edge_loop_bloom(reinterpret_cast<const uint64_t*>(rows), bits / 64, epi.op, us, vs, e_begin,
                           e_end, epi);
  else
    group_edge_loop<V, G, Op, EpiBloomHist, kVCache>(rows, us, vs, e_begin, e_end, epi);
  __syncthreads();
  for (int i = threadIdx.x; i <= bits; i += blockDim.x)
    if (hist_s[i]) atomicAdd(reinterpret_cast<unsigned long long*>(out_hist + i), (unsigned long long)hist_s[i]);
  if (epi.op == PG_BF_OR) {
    long long s = epi.sum_pos;
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0 && s) atomicAdd(reinterpret_cast<unsigned long long*>(out_sum_pos), (unsigned long long)s);
  }
}

// kSched: 0 static per-warp slices, 1 dynamic chunks (ctr), 2 static slices
// of the device-side range [range_dev[0], range_dev[1]) (appended slots)
template <int W8, class Op, int MINB, bool kVCache, int kLayout, int kSched = 0>
__global__ void __launch_bounds__(kBlock, MINB) tc_bloom_wide_kernel(const unsigned char* rows, int bits,
                                                                    const int32_t* us, const int32_t* vs,
                                                                    int64_t e_begin, int64_t e_end,
                                                                    EpiBloomHist epi, int64_t* out_hist,
                                                                    int64_t* out_sum_pos, unsigned long long* ctr,
                                                                    const int64_t* range_dev) {
  extern __shared__ int hist_s[];
  if (kSched == 2) {
    e_begin = range_dev[0];
    e_end = range_dev[1];
  }
  for (int i = threadIdx.x; i <= bits; i += blockDim.x) hist_s[i] = 0;
  __syncthreads();
  epi.hist_s = hist_s;
  epi.sum_pos = 0;
  wide_edge_loop<W8, Op, EpiBloomHist, kVCache, kLayout, kSched == 1>(rows, us, vs, e_begin, e_end, epi, ctr);
  __syncthreads();
  for (int i = threadIdx.x; i <= bits; i += blockDim.x)
    if (hist_s[i]) atomicAdd(reinterpret_cast<unsigned long long*>(out_hist + i), (unsigned long long)hist_s[i]);
  if (epi.op == PG_BF_OR) {
    long long sp = epi.sum_pos;
    for (int o = 16; o > 0; o >>= 1) sp += __shfl_xor_sync(0xffffffffu, sp, o);
    if ((threadIdx.x & 31) == 0 && sp) atomicAdd(reinterpret_cast<unsigned long long*>(out_sum_pos), (unsigned long long)sp);
  }
}
// ---------------------------------------------------------- launching ----
// Occupancy hint of the Bloom TC kernel (blocks of 256 per SM the register
// allocation must allow); PG_TC_MINB overrides it for tuning sweeps.
static int tc_minb(int w4, bool padded) {
  static int env = [] {
    const char* e = getenv("PG_TC_MINB");
    return e ? atoi(e) : 0;
  }();
  if (env >= 1 && env <= 4) return env;
  if (!padded) return 2;  // general layout: speculative u loads need ~110 regs
  if (w4 >= 16) return 2;  // 256-byte rows: 8 rows of v in flight per lane group need > 80 regs
  return 3;
}

template <int V, int G>
static auto pick_tc_bloom(int op, int minb) {
  const bool o = op == PG_BF_OR;
  static const bool vcache = getenv("PG_TC_VCACHE") != nullptr;
  if (vcache) return o ? tc_bloom_kernel<V, G, OpOr, false, 2, true> : tc_bloom_kernel<V, G, OpAnd, false, 2, true>;
  switch (minb) {
    case 2: return o ? tc_bloom_kernel<V, G, OpOr, false, 2> : tc_bloom_kernel<V, G, OpAnd, false, 2>;
    case 3: return o ? tc_bloom_kernel<V, G, OpOr, false, 3> : tc_bloom_kernel<V, G, OpAnd, false, 3>;
    case 4: return o ? tc_bloom_kernel<V, G, OpOr, false, 4> : tc_bloom_kernel<V, G, OpAnd, false, 4>;
    default: return o ? tc_bloom_kernel<V, G, OpOr, false, 1> : tc_bloom_kernel<V, G, OpAnd, false, 1>;
  }
}

}  // namespace pg

using namespace pg;

extern "C" {

int pg_pairs_bloom(const uint64_t* rows, int32_t bits, int32_t b, int32_t op, const int32_t* sizes,
                   const double* lut, const int32_t* us, const int32_t* vs, int64_t count,
                   int32_t* out_count, double* out_est, void* stream) {
  PG_REQUIRE(bits >= 64 && bits % 64 == 0, "Bloom size must be a positive multiple of 64");
  PG_REQUIRE(b >= 1, "need at least one hash function");
  PG_REQUIRE(op == PG_BF_AND || op == PG_BF_L || op == PG_BF_OR, "op is not a Bloom estimator");
  PG_REQUIRE(count >= 0, "count must be >= 0");
  if (count == 0) return PG_OK;
  PG_REQUIRE(rows && us && vs, "null pointer");
  PG_REQUIRE(!out_est || op == PG_BF_L || lut, "estimate needs the Swamidass table");
  PG_REQUIRE(!(out_est && op == PG_BF_OR) || sizes, "BF_OR needs sizes");
  EpiBloomPairs epi{op, b, sizes, lut, out_count, out_est};
  cudaStream_t s = as_stream(stream);
  const int w4 = bits % 128 == 0 ? bits / 128 : 0;
  const int grid = grid_cap(sm_count() * 8, count, kBlock);
  if (!fast_w4(w4)) {
    pairs_scalar_kernel_bloom<<<grid, kBlock, 0, s>>>(rows, bits / 64, us, vs, count, epi);
  } else {
    const uint4* r4 = reinterpret_cast<const uint4*>(rows);
#define PG_L(V, G)                                                                         \
  if (op == PG_BF_OR) pairs_rows_kernel_bloom<V, G, OpOr><<<grid, kBlock, 0, s>>>(r4, us, vs, count, epi); \
  else pairs_rows_kernel_bloom<V, G, OpAnd><<<grid, kBlock, 0, s>>>(r4, us, vs, count, epi);
    PG_ROW_DISPATCH(w4, PG_L)
#undef PG_L
  }
  return check_launch("pairs_bloom");
}

static int tc_bloom_impl(const uint64_t* rows, int32_t bits, int32_t op, const int32_t* sizes,
                         const double* lut, const int32_t* us, const int32_t* vs, int64_t e_begin,
                         int64_t e_end, int64_t* out_hist, int64_t* out_sum_pos, void* stream, int padded,
                         const int64_t* range_dev = nullptr, bool accumulate = false) {
  PG_REQUIRE(bits >= 64 && bits % 64 == 0, "Bloom size must be a positive multiple of 64");
  PG_REQUIRE(op == PG_BF_AND || op == PG_BF_L || op == PG_BF_OR, "op is not a Bloom estimator");
  PG_REQUIRE(0 <= e_begin && e_begin <= e_end, "bad edge range");
  PG_REQUIRE(out_hist, "null histogram");
  PG_REQUIRE(op != PG_BF_OR || out_sum_pos, "BF_OR needs the sum output");
  cudaStream_t s = as_stream(stream);
  // one memset when the sum slot directly follows the histogram
  const bool adjacent = out_sum_pos == out_hist + bits + 1;
  cudaError_t ce = cudaSuccess;
  if (!accumulate) {
    ce = cudaMemsetAsync(out_hist, 0, sizeof(int64_t) * (bits + 1 + (adjacent ? 1 : 0)), s);
    if (ce == cudaSuccess && out_sum_pos && !adjacent) ce = cudaMemsetAsync(out_sum_pos, 0, sizeof(int64_t), s);
  }
  if (ce != cudaSuccess) return fail(PG_ERR_CUDA, "memset: %s", cudaGetErrorString(ce));
  if (e_end == e_begin) return PG_OK;  // an empty range needs no inputs
  PG_REQUIRE(op != PG_BF_OR || (sizes && lut), "BF_OR needs sizes and the table");
  PG_REQUIRE(rows && us && vs, "null pointer");
  if (bits > kGenBloomTcBits && !range_dev)  // histogram too large for shared memory
    return gen_tc_bloom(rows, bits, op, sizes, lut, us, vs, e_begin, e_end, out_hist, out_sum_pos, s);
  PG_REQUIRE(bits <= kGenBloomTcBits, "device slot ranges support Bloom widths up to %d", kGenBloomTcBits);
  EpiBloomHist epi{op, sizes, lut, nullptr, 0};
  const size_t smem = sizeof(int) * (bits + 1);
  const int w4 = bits % 128 == 0 ? bits / 128 : 0;
  const uint4* r4 = reinterpret_cast<const uint4*>(rows);
  static const int engine = [] {
    const char* e = getenv("PG_TC_ENGINE");
    if (e && e[0] == 'r') return 0;  // 128-bit loads (group_edge_loop)
    return 2;                        // 256-bit loads (wide_edge_loop, default)
  }();
  if (engine == 2 && (w4 == 4 || w4 == 8 || w4 == 16)) {
    // measured on B200 (scripts/probe_tc.py, R-MAT s20/s22): B=1024 best with
    // 3 blocks/SM and streaming v rows; B=2048 best with L1-allocated v rows
    // (hub rows reused within an SM)
    static const char* vc_env = getenv("PG_TC_VCACHE");
    const bool vcache = vc_env ? vc_env[0] != '0' : (padded && w4 == 16);
    const int minb = tc_minb(w4, padded);
    // Harley-Seal popcount for 256-byte rows (XU-pipe bound once the row
    // stream hits L1/L2); PG_TC_CSA=0/1 overrides
    static const char* csa_env = getenv("PG_TC_CSA");
    const bool csa = csa_env ? csa_env[0] != '0' : w4 >= 16;
    const unsigned char* rb = reinterpret_cast<const unsigned char*>(rows);
    cudaError_t le = cudaSuccess;
    static const bool dyn = [] {
      const char* v = getenv("PG_TC_DYNAMIC");
      return !(v && v[0] == '0');
    }();
    // dynamic chunks pay off on large edge sets (c4/c5: 3-5%); below ~32 M
    // slots the per-launch counter costs more than the balance gains.  The
    // dynamic variant of the 256-byte-row kernel fits 3 CTAs/SM in 80
    // registers without spills (c5: 5.48 vs 6.09 ms at 2 CTAs/SM); the static
    // one spills 216 bytes there and keeps 2
    // shared-memory carveout hint (percent; PG_TC_CARVEOUT, default: driver)
    static const int carveout = [] {
      const char* v = getenv("PG_TC_CARVEOUT");
      return v ? atoi(v) : -1;
    }();
    ChunkCounter ctr;
    if (dyn && !range_dev && e_end - e_begin >= kDynamicMinSlots && (le = ctr.init(s)) != cudaSuccess) return fail(PG_ERR_CUDA, "chunk counter: %s", cudaGetErrorString(le));
#define PG_WK(W8, MB, VC, PD, SCH)                                                                    \
  (op == PG_BF_OR ? (csa ? tc_bloom_wide_kernel<W8, OpOrCsa, MB, VC, PD, SCH>                          \
                         : tc_bloom_wide_kernel<W8, OpOr, MB, VC, PD, SCH>)                            \
                  : (csa ? tc_bloom_wide_kernel<W8, OpAndCsa, MB, VC, PD, SCH>                         \
                         : tc_bloom_wide_kernel<W8, OpAnd, MB, VC, PD, SCH>))
#define PG_W(W8, MB, VC, PD)                                                                          \
  {                                                                                                  \
    auto k = PG_WK(W8, MB, VC, PD, 0);                                                               \
    if (range_dev) k = PG_WK(W8, MB, VC, PD, 2);                                                     \
    else if (ctr.p) k = PG_WK(W8, MB, VC, PD, 1);                                                    \
    le = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);            \
    if (le == cudaSuccess && carveout >= 0)                                                          \
      le = cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, carveout);        \
    if (le != cudaSuccess) return fail(PG_ERR_CUDA, "smem attribute: %s", cudaGetErrorString(le));  \
    const int grid = grid_cap(grid_for_kernel(k, smem), e_end - e_begin, kBlock);                    \
    k<<<grid, kBlock, smem, s>>>(rb, bits, us, vs, e_begin, e_end, epi, out_hist, out_sum_pos, ctr.p,  \
                                 range_dev);                                                          \
  }
#define PG_WM(W8)                                                                  \
  if (padded == 2) {                                                             \
    if (vcache) { if (minb <= 2 && !ctr.p) PG_W(W8, 2, true, 2) else PG_W(W8, PG_WIDE_MINB, true, 2) } \
    else if (minb <= 2) PG_W(W8, 2, false, 2)                                    \
    else PG_W(W8, 3, false, 2)                                                   \
  } else if (padded) {                                                           \
    if (vcache) PG_W(W8, 3, true, 1)                                             \
    else if (minb >= 4) PG_W(W8, 4, false, 1)                                    \
    else if (minb == 3) PG_W(W8, 3, false, 1)                                    \
    else PG_W(W8, 2, false, 1)                                                   \
  } else {                                                                       \
    PG_W(W8, 2, false, 0)                                                        \
  }
    if (w4 == 4) PG_WM(2)
    else if (w4 == 8) PG_WM(4)
    else PG_WM(8)
#undef PG_WM
#undef PG_W
#undef PG_WK
    return check_launch("tc_bloom_wide");
  }
  if (!fast_w4(w4)) {
    auto k = tc_bloom_kernel<1, 1, OpAnd, true>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int grid = grid_cap(grid_for_kernel(k, smem), e_end - e_begin, kBlock);
    k<<<grid, kBlock, smem, s>>>(r4, bits, us, vs, e_begin, e_end, epi, out_hist, out_sum_pos);
  } else {
#define PG_L(V, G)                                                                                   \
  {                                                                                                  \
    auto k = pick_tc_bloom<V, G>(op, tc_minb(w4, false));                                                   \
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);                 \
    const int grid = grid_cap(grid_for_kernel(k, smem), e_end - e_begin, kBlock);                    \
    k<<<grid, kBlock, smem, s>>>(r4, bits, us, vs, e_begin, e_end, epi, out_hist, out_sum_pos);      \
  }
    PG_ROW_DISPATCH(w4, PG_L)
#undef PG_L
  }
  return check_launch("tc_bloom");
}

int pg_tc_bloom(const uint64_t* rows, int32_t bits, int32_t op, const int32_t* sizes, const double* lut,
                const int32_t* us, const int32_t* vs, int64_t e_begin, int64_t e_end, int32_t padded,
                int64_t* out_hist, int64_t* out_sum_pos, void* stream) {
  int32_t pad = 1;
  if (padded) {
    pg_group_pad(bits / 8, &pad);
    PG_REQUIRE(e_begin % pad == 0, "e_begin must be a multiple of the layout pad %d", pad);
  }
  PG_REQUIRE(padded >= 0 && padded <= 2, "padded must be 0, 1 or 2");
  PG_REQUIRE(padded != 2 || pad > 1, "the group-u layout needs a padded row size");
  return tc_bloom_impl(rows, bits, op, sizes, lut, us, vs, e_begin, e_end, out_hist, out_sum_pos, stream,
                       pad > 1 ? padded : 0);
}

}  // extern "C"

extern "C" int pg_tc_bloom_range(const uint64_t* rows, int32_t bits, int32_t op, const int32_t* sizes,
                                 const double* lut, const int32_t* ug, const int32_t* vs, const int64_t* range_dev,
                                 int64_t max_slots, int32_t accumulate, int64_t* out_hist, int64_t* out_sum_pos,
                                 void* stream) {
  int32_t pad = 1;
  PG_REQUIRE(bits >= 64 && bits % 64 == 0, "Bloom size must be a positive multiple of 64");
  pg_group_pad(bits / 8, &pad);
  if (pad <= 1) return fail(PG_ERR_UNSUPPORTED, "device slot ranges need a group-u Bloom row size (got %d bits)", bits);
  PG_REQUIRE(range_dev, "null range");
  PG_REQUIRE(max_slots >= 0, "max_slots must be >= 0");
  // the wide engine's group-u layout; the launch is sized for max_slots and
  // the kernel reads the actual [begin, end) from range_dev
  return tc_bloom_impl(rows, bits, op, sizes, lut, ug, vs, 0, max_slots, out_hist, out_sum_pos, stream, 2,
                       range_dev, accumulate != 0);
}

extern "C" int pg_group_pad(int32_t row_bytes, int32_t* pad_host) {
  PG_REQUIRE(pad_host, "null output");
  PG_REQUIRE(row_bytes > 0, "row_bytes must be positive");
  const int w8 = row_bytes % 32 == 0 ? row_bytes / 32 : 0;
  *pad_host = (w8 == 2 || w8 == 4 || w8 == 8) ? w8 : 1;
  return PG_OK;
}
