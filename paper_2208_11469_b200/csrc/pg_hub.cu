// Degree-oriented, hub-cached fused Bloom triangle-count pass (the c5
// headline kernel).  Same per-edge quantity as pg_tc_bloom -- the popcount
// of row_u AND row_v (OR for BF_OR), histogrammed -- over a different edge
// schedule (providers.py:150-162 pair_many, mining.py:105-130 tc_estimate).
//
// Why: the ID-oriented kernel (pg_bloom.cu) holds the u row (the lower ID,
// i.e. the R-MAT hub) in registers across its run and streams v, the long
// tail, so every edge costs one 256-byte row from L2 -- at c5 that is
// 66.7 GB per launch and the kernel runs at the L2 -> SM throughput cap
// (~12 TB/s), with 32.7 GB of DRAM misses behind it.  Here every edge is
// oriented from its lower- to its higher-(degree, ID)-rank endpoint (the
// N+ lists of degree_order, graphs.py:154-166): u, in registers, is the
// low-degree endpoint and the streamed v is the hub side.  The n_hubs
// highest-ranked vertices' rows are staged once per CTA in shared memory
// (one persistent CTA per SM, ~220 KB), and edge slots whose v is a hub
// carry the tag -2 - hub_index, so those v rows come from shared memory and
// cost no L2 traffic.  The other v rows are the next tiers of the degree
// distribution: small enough to stay L2-resident, so DRAM traffic drops too.
//
// Popcount: with the L2 stream reduced, the XU pipe (POPC, 16/clk/SM) is
// the next ceiling (64 POPC per 2048-bit edge).  kCsa folds the 8 words a
// lane holds per edge through four carry-save adders (LOP3s on the ALU
// pipe) so that 4 POPC replace 8 (Harley-Seal).  Counts are identical.
#include "pg_engines.cuh"

namespace pg {

constexpr int kHubThreads = 768;  // one CTA per SM: 24 warps, <= 85 registers

// shared-memory position of 16-byte chunk c (of 16) of a staged 256-byte
// row: chunks 8..15 swap pairwise, so the 8 lanes of a group reading chunk
// 2gl (then 2gl+1) hit 8 distinct 16-byte bank groups -- a warp-wide
// LDS.128 over four rows is then four wavefronts, the minimum
__device__ __forceinline__ int hub_pos(int c) { return c ^ ((c >> 3) & 1); }

__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 r;
  asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(addr));
  return r;
}

template <class Op, bool kCsa>
__device__ __forceinline__ int count8(const uint32_t (&a)[8], const uint32_t (&b)[8]) {
  if (kCsa) return std::is_same<Op, OpOr>::value ? OpOrCsa::apply8(a, b) : OpAndCsa::apply8(a, b);
  return Op::apply8(a, b);
}

// Slot layout (group-u, pad G = 8): ug[e / 8] is the u of slots
// [8q, 8q+8); vs[e] >= 0 a streamed v, -1 padding, <= -2 hub -2-vs[e].
template <class Op, bool kCsa, bool kDyn, int kThreads = kHubThreads>
__global__ void __launch_bounds__(kThreads, 1) tc_bloom_hub_kernel(
    const unsigned char* __restrict__ rows, int bits, const int32_t* __restrict__ ug,
    const int32_t* __restrict__ vs, int64_t e_begin, int64_t e_end, const int32_t* __restrict__ hub_ids,
    int n_hubs, EpiBloomHist epi, int64_t* out_hist, int64_t* out_sum_pos, unsigned long long* ctr) {
  constexpr int G = 8;            // lanes per edge (256-byte rows, 32 bytes per lane)
  constexpr int64_t kRow = 256;
  extern __shared__ __align__(16) unsigned char smem[];
  int* hist_s = reinterpret_cast<int*>(smem);
  const int hist_bytes = ((bits + 1) * 4 + 15) & ~15;
  uint4* hub_rows = reinterpret_cast<uint4*>(smem + hist_bytes);
  for (int i = threadIdx.x; i <= bits; i += blockDim.x) hist_s[i] = 0;
  // stage the hub rows (16 chunks each, permuted)
  for (int i = threadIdx.x; i < n_hubs * 16; i += blockDim.x) {
    const int h = i >> 4, c = i & 15;
    const uint4* src = reinterpret_cast<const uint4*>(rows + (int64_t)hub_ids[h] * kRow) + c;
    hub_rows[h * 16 + hub_pos(c)] = __ldg(src);
  }
  __syncthreads();
  epi.hist_s = hist_s;
  epi.sum_pos = 0;
  const uint32_t hub_base = (uint32_t)__cvta_generic_to_shared(hub_rows);
  const int lane = threadIdx.x & 31;
  const int gl = lane & (G - 1);
  const int gbase = lane & ~(G - 1);
  const uint32_t off0 = (uint32_t)hub_pos(2 * gl) * 16, off1 = (uint32_t)hub_pos(2 * gl + 1) * 16;
  int32_t ucur = -1;
  uint32_t ur[8];
#pragma unroll
  for (int w = 0; w < 8; ++w) ur[w] = 0;
  int64_t wb, we;
  bool first = true;
  for (;;) {
    if (kDyn) {
      if (!next_chunk(ctr, e_begin, e_end, 512, wb, we)) break;
    } else {
      if (!first) break;
      warp_slice(e_begin, e_end, wb, we);
      if (wb >= we) break;
    }
    first = false;
    int32_t ul = 0, vl = -1;
    if (wb + lane < we) {
      ul = ug[(wb + lane) / G];
      vl = vs[wb + lane];
    }
    const int nslots = (int)(we - wb);
#pragma unroll 1
    for (int r0 = 0; r0 < nslots; r0 += 32) {
      const int64_t e = wb + r0 + lane;
      const int rem = nslots - r0;
      const bool valid = lane < rem && vl != -1;
      int32_t un = 0, vn = -1;
      if (lane + 32 < rem) {
        un = ug[(e + 32) / G];
        vn = vs[e + 32];
      }
      uint32_t vr[G][8];
#pragma unroll
      for (int j = 0; j < G; ++j) {
        const int32_t vj = __shfl_sync(0xffffffffu, vl, gbase + j);
        if (vj >= 0) {
          ldg256(rows + (int64_t)vj * kRow + gl * 32, vr[j]);
        } else if (vj <= -2) {
          const uint32_t base = hub_base + (uint32_t)(-2 - vj) * (uint32_t)kRow;
          const uint4 lo = lds128(base + off0), hi = lds128(base + off1);
          vr[j][0] = lo.x; vr[j][1] = lo.y; vr[j][2] = lo.z; vr[j][3] = lo.w;
          vr[j][4] = hi.x; vr[j][5] = hi.y; vr[j][6] = hi.z; vr[j][7] = hi.w;
        }
      }
      const int32_t u0 = __shfl_sync(0xffffffffu, ul, gbase);
      if (u0 != ucur) {
        ucur = u0;
        ldg256_keep(rows + (int64_t)u0 * kRow + gl * 32, ur);
      }
      int c[G];
#pragma unroll
      for (int j = 0; j < G; ++j) c[j] = count8<Op, kCsa>(ur, vr[j]);
      const int cnt = group_transpose_reduce<G>(c, gl);
      if (valid) {
        int32_t vv = vl;  // BF_OR reads sizes[v]: resolve a hub tag
        if (epi.op == PG_BF_OR && vl < 0) vv = hub_ids[-2 - vl];
        epi.edge(e, ul, vv, cnt);
      }
      ul = un;
      vl = vn;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i <= bits; i += blockDim.x)
    if (hist_s[i]) atomicAdd(reinterpret_cast<unsigned long long*>(out_hist + i), (unsigned long long)hist_s[i]);
  if (epi.op == PG_BF_OR) {
    long long sp = epi.sum_pos;
    for (int o = 16; o > 0; o >>= 1) sp += __shfl_xor_sync(0xffffffffu, sp, o);
    if ((threadIdx.x & 31) == 0 && sp)
      atomicAdd(reinterpret_cast<unsigned long long*>(out_sum_pos), (unsigned long long)sp);
  }
}

// hub_ids[rank - (n - H)] = v for the H highest-ranked vertices
__global__ void hub_ids_kernel(const int32_t* __restrict__ rank, int64_t n, int n_hubs, int32_t* __restrict__ hub_ids) {
  const int64_t lo = n - n_hubs;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = rank[v];
    if (r >= lo) hub_ids[r - lo] = (int32_t)v;
  }
}
// vs[e] (a vertex, or -1) -> -2 - hub index when v is a hub
__global__ void hub_tag_kernel(const int32_t* __restrict__ rank, int64_t n, int n_hubs, int32_t* __restrict__ vs,
                               int64_t slots) {
  const int64_t lo = n - n_hubs;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < slots; e += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = vs[e];
    if (v >= 0) {
      const int64_t r = rank[v];
      if (r >= lo) vs[e] = (int32_t)(-2 - (r - lo));
    }
  }
}

static size_t hub_smem(int bits, int n_hubs) { return (((size_t)(bits + 1) * 4 + 15) & ~size_t(15)) + (size_t)n_hubs * 256; }

}  // namespace pg

using namespace pg;

extern "C" {

int pg_tc_bloom_hub_capacity(int32_t bits, int32_t* max_hubs) {
  PG_REQUIRE(max_hubs, "null output");
  PG_REQUIRE(bits >= 64 && bits % 64 == 0, "Bloom size must be a positive multiple of 64");
  *max_hubs = 0;
  if (bits != 2048) return PG_OK;  // the hub engine serves 256-byte rows
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  const int64_t room = (int64_t)optin - (int64_t)hub_smem(bits, 0) - 1024;
  *max_hubs = room > 0 ? (int32_t)(room / 256) : 0;
  return PG_OK;
}

int pg_hub_tag(const int32_t* rank, int64_t n, int32_t n_hubs, int32_t* vs, int64_t slots, int32_t* hub_ids,
               void* stream) {
  PG_REQUIRE(n >= 0 && slots >= 0, "bad sizes");
  PG_REQUIRE(n_hubs >= 0 && n_hubs <= n, "n_hubs must be in [0, n]");
  if (n_hubs == 0 || n == 0) return PG_OK;
  PG_REQUIRE(rank && hub_ids && (slots == 0 || vs), "null pointer");
  cudaStream_t s = as_stream(stream);
  const int grid = sm_count() * 8;
  hub_ids_kernel<<<grid, 256, 0, s>>>(rank, n, n_hubs, hub_ids);
  if (slots) hub_tag_kernel<<<grid, 256, 0, s>>>(rank, n, n_hubs, vs, slots);
  return check_launch("hub_tag");
}

int pg_tc_bloom_hub(const uint64_t* rows, int32_t bits, int32_t op, const int32_t* sizes, const double* lut,
                    const int32_t* ug, const int32_t* vs, int64_t e_begin, int64_t e_end, const int32_t* hub_ids,
                    int32_t n_hubs, int64_t* out_hist, int64_t* out_sum_pos, void* stream) {
  PG_REQUIRE(bits == 2048, "the hub engine serves 2048-bit rows (got %d)", bits);
  PG_REQUIRE(op == PG_BF_AND || op == PG_BF_L || op == PG_BF_OR, "op is not a Bloom estimator");
  PG_REQUIRE(0 <= e_begin && e_begin <= e_end && e_begin % 8 == 0, "bad edge range");
  PG_REQUIRE(out_hist, "null histogram");
  PG_REQUIRE(op != PG_BF_OR || out_sum_pos, "BF_OR needs the sum output");
  int32_t cap = 0;
  pg_tc_bloom_hub_capacity(bits, &cap);
  PG_REQUIRE(n_hubs >= 0 && n_hubs <= cap, "n_hubs %d exceeds the shared-memory capacity %d", n_hubs, cap);
  cudaStream_t s = as_stream(stream);
  const bool adjacent = out_sum_pos == out_hist + bits + 1;
  cudaError_t ce = cudaMemsetAsync(out_hist, 0, sizeof(int64_t) * (bits + 1 + (adjacent ? 1 : 0)), s);
  if (ce == cudaSuccess && out_sum_pos && !adjacent) ce = cudaMemsetAsync(out_sum_pos, 0, sizeof(int64_t), s);
  if (ce != cudaSuccess) return fail(PG_ERR_CUDA, "memset: %s", cudaGetErrorString(ce));
  if (e_end == e_begin) return PG_OK;
  PG_REQUIRE(rows && ug && vs && (n_hubs == 0 || hub_ids), "null pointer");
  PG_REQUIRE(op != PG_BF_OR || (sizes && lut), "BF_OR needs sizes and the table");
  EpiBloomHist epi{op, sizes, lut, nullptr, 0};
  const size_t smem = hub_smem(bits, n_hubs);
  static const bool use_csa = [] {
    const char* e = getenv("PG_HUB_CSA");
    return !(e && e[0] == '0');
  }();
  ChunkCounter ctr;
  cudaError_t le = ctr.init(s);
  if (le != cudaSuccess) return fail(PG_ERR_CUDA, "chunk counter: %s", cudaGetErrorString(le));
  // CTA size (PG_HUB_THREADS tuning knob): 768 = 24 warps at <= 80
  // registers, 640 / 512 leave 96 / 128 registers per thread
  static const int threads = [] {
    const char* e = getenv("PG_HUB_THREADS");
    const int t = e ? atoi(e) : kHubThreads;
    return (t == 512 || t == 640) ? t : kHubThreads;
  }();
  auto pick = [&](auto op_tag) {
    using O = decltype(op_tag);
    if (threads == 512) return use_csa ? tc_bloom_hub_kernel<O, true, true, 512> : tc_bloom_hub_kernel<O, false, true, 512>;
    if (threads == 640) return use_csa ? tc_bloom_hub_kernel<O, true, true, 640> : tc_bloom_hub_kernel<O, false, true, 640>;
    return use_csa ? tc_bloom_hub_kernel<O, true, true> : tc_bloom_hub_kernel<O, false, true>;
  };
  auto k = op == PG_BF_OR ? pick(OpOr{}) : pick(OpAnd{});
  le = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (le != cudaSuccess) return fail(PG_ERR_CUDA, "smem attribute: %s", cudaGetErrorString(le));
  const int64_t warps_needed = (e_end - e_begin + 511) / 512;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(sm_count(), (warps_needed + 23) / 24));
  k<<<grid, threads, smem, s>>>(reinterpret_cast<const unsigned char*>(rows), bits, ug, vs, e_begin, e_end,
                                    hub_ids, n_hubs, epi, out_hist, out_sum_pos, ctr.p);
  return check_launch("tc_bloom_hub");
}

}  // extern "C"
