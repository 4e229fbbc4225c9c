// Graph generation on the device (SURVEY 8(f) "next": graph ingest and
// generation), bit-identical to the host generators in graphs.py, which
// restate the reference's generate_kronecker (graphs.py:251-276).
//
// numpy's default_rng is PCG64 (128-bit LCG, XSL-RR output); draw p of a
// stream is output(S(p+1)) where S(q) is the state after q LCG steps from the
// captured state.  Every thread jumps its LCG straight to its first draw
// (affine-map exponentiation), so any slice of the stream is generated in
// parallel and matches rng.random() element for element.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_segmented_reduce.cuh>
#include <cub/device/device_select.cuh>

#include "pg_common.cuh"

namespace pg {

typedef unsigned __int128 u128;

constexpr uint64_t kPcgMulHi = 0x2360ED051FC65DA4ull;
constexpr uint64_t kPcgMulLo = 0x4385DF649FCCF645ull;

struct Affine {  // x -> a*x + c  (mod 2^128)
  u128 a, c;
};

__host__ __device__ inline u128 mk128(uint64_t hi, uint64_t lo) { return ((u128)hi << 64) | lo; }

__host__ __device__ inline Affine compose(Affine f, Affine g) {  // g after f
  return Affine{g.a * f.a, g.a * f.c + g.c};
}

// the map that advances the stream by `delta` steps
__host__ __device__ inline Affine advance_map(u128 inc, uint64_t delta) {
  Affine result{1, 0};
  Affine base{mk128(kPcgMulHi, kPcgMulLo), inc};
  while (delta) {
    if (delta & 1) result = compose(result, base);
    base = compose(base, base);
    delta >>= 1;
  }
  return result;
}

__device__ __forceinline__ double pcg_double(u128 state) {
  const uint64_t hi = (uint64_t)(state >> 64), lo = (uint64_t)state;
  const unsigned rot = (unsigned)(state >> 122);
  const uint64_t x = hi ^ lo;
  const uint64_t r = (x >> rot) | (x << ((64 - rot) & 63));
  return (double)(r >> 11) * (1.0 / 9007199254740992.0);
}

// R-MAT: for sample i and level L the source bit uses draw 2Lc+i and the
// destination bit draw 2Lc+c+i (two rng.random(count) calls per level).
__global__ void rmat_pairs_kernel(u128 s0, u128 inc, Affine adv_c, Affine adv_2c, int scale, int64_t count,
                                  double p_ab, double thr_src0, double thr_src1, int64_t per_thread,
                                  int64_t* __restrict__ src, int64_t* __restrict__ dst) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t i0 = t * per_thread;
  if (i0 >= count) return;
  const int64_t i1 = i0 + per_thread < count ? i0 + per_thread : count;
  const Affine step{mk128(kPcgMulHi, kPcgMulLo), inc};
  const Affine to_first = advance_map(inc, (uint64_t)i0 + 1);
  u128 cur = to_first.a * s0 + to_first.c;  // S(i0 + 1)
  for (int64_t i = i0; i < i1; ++i) {
    u128 xs = cur;
    int64_t sv = 0, dv = 0;
    for (int L = 0; L < scale; ++L) {
      const u128 xd = adv_c.a * xs + adv_c.c;
      const bool sbit = pcg_double(xs) > p_ab;
      const bool dbit = pcg_double(xd) > (sbit ? thr_src1 : thr_src0);
      sv |= (int64_t)sbit << L;
      dv |= (int64_t)dbit << L;
      xs = adv_2c.a * xs + adv_2c.c;
    }
    src[i] = sv;
    dst[i] = dv;
    cur = step.a * cur + step.c;
  }
}

// uniform doubles of draws [offset, offset+count) of a stream
__global__ void pcg_uniform_kernel(u128 s0, u128 inc, int64_t offset, int64_t count, int64_t per_thread,
                                   double* __restrict__ out) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t i0 = t * per_thread;
  if (i0 >= count) return;
  const int64_t i1 = i0 + per_thread < count ? i0 + per_thread : count;
  const Affine step{mk128(kPcgMulHi, kPcgMulLo), inc};
  const Affine to_first = advance_map(inc, (uint64_t)(offset + i0) + 1);
  u128 cur = to_first.a * s0 + to_first.c;
  for (int64_t i = i0; i < i1; ++i) {
    out[i] = pcg_double(cur);
    cur = step.a * cur + step.c;
  }
}

// np.searchsorted(cdf, u, side="right"), clipped to n-1 (graphs.generate_chung_lu)
__global__ void searchsorted_right_kernel(const double* __restrict__ cdf, int64_t n, const double* __restrict__ u,
                                          int64_t count, int64_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double x = u[i];
    int64_t lo = 0, hi = n;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (cdf[mid] <= x) lo = mid + 1;
      else hi = mid;
    }
    out[i] = lo < n - 1 ? lo : n - 1;
  }
}

// canonical undirected key lo*n+hi; self loops -> n*n (sorts last, dropped)
__global__ void canonical_keys_kernel(const int64_t* __restrict__ a, const int64_t* __restrict__ b, int64_t count,
                                      uint64_t n, uint64_t* __restrict__ keys) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t x = (uint64_t)a[i], y = (uint64_t)b[i];
    keys[i] = x == y ? n * n : (x < y ? x * n + y : y * n + x);
  }
}

// both directions of every unique edge
__global__ void both_directions_kernel(const uint64_t* __restrict__ keys, int64_t m, uint64_t n,
                                       uint64_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = keys[i], lo = k / n, hi = k - lo * n;
    out[i] = k;
    out[m + i] = hi * n + lo;
  }
}

__global__ void split_keys_kernel(const uint64_t* __restrict__ keys, int64_t nnz, uint64_t n,
                                  int32_t* __restrict__ adj, int32_t* __restrict__ srcv) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nnz;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = keys[i], s = k / n;
    adj[i] = (int32_t)(k - s * n);
    srcv[i] = (int32_t)s;
  }
}

// offsets[v] = first index whose source is >= v (sources sorted)
__global__ void offsets_kernel(const int32_t* __restrict__ srcv, int64_t nnz, int64_t n, int64_t* __restrict__ off) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v <= n;
       v += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = nnz;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (srcv[mid] < v) lo = mid + 1;
      else hi = mid;
    }
    off[v] = lo;
  }
}

static int key_bits(uint64_t n) {
  const unsigned __int128 top = (unsigned __int128)n * n;  // largest key (loops)
  int bits = 1;
  while (bits < 64 && ((unsigned __int128)1 << bits) <= top) ++bits;
  return bits;
}

static size_t al256(size_t x) { return (x + 255) & ~size_t(255); }

// ---- degree ordering (graphs.py:154-166): rank by (degree, id), keep
// x in N+(v) iff rank[v] < rank[x], adjacency order preserved
__global__ void degree_keys_kernel(const int64_t* __restrict__ offsets, int64_t n, uint64_t* __restrict__ keys) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
    keys[v] = ((uint64_t)(offsets[v + 1] - offsets[v]) << 32) | (uint64_t)v;
}

__global__ void rank_scatter_kernel(const uint64_t* __restrict__ sorted, int64_t n, int32_t* __restrict__ rank) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    rank[(uint32_t)sorted[i]] = (int32_t)i;
}

__global__ void orient_flags_in_kernel(const int32_t* __restrict__ src, const int32_t* __restrict__ adj,
                                       const int32_t* __restrict__ rank, int64_t nnz, int32_t* __restrict__ flags) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nnz; j += (int64_t)gridDim.x * blockDim.x)
    flags[j] = rank[src[j]] > rank[adj[j]];
}
__global__ void orient_flags_kernel(const int32_t* __restrict__ src, const int32_t* __restrict__ adj,
                                    const int32_t* __restrict__ rank, int64_t nnz, int32_t* __restrict__ flags) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nnz; j += (int64_t)gridDim.x * blockDim.x)
    flags[j] = rank[src[j]] < rank[adj[j]];
}



}  // namespace pg

using namespace pg;

// counts[v] = sum of flags over row v, a warp per row (grid-stride)
__global__ void row_flag_count_kernel(const int64_t* __restrict__ offsets, const int32_t* __restrict__ flags,
                                      int64_t n, int64_t* __restrict__ counts) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t v = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; v < n; v += warps) {
    int64_t c = 0;
    for (int64_t j = offsets[v] + lane; j < offsets[v + 1]; j += 32) c += flags[j];
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0) counts[v] = c;
  }
}


extern "C" {

int pg_rmat_pairs(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo, int32_t scale,
                  int64_t count, double a, double b, double c, int64_t* src, int64_t* dst, void* stream) {
  PG_REQUIRE(scale >= 1 && scale <= 31, "scale must be in [1, 31]");
  PG_REQUIRE(count >= 0, "count must be >= 0");
  if (count == 0) return PG_OK;
  PG_REQUIRE(src && dst, "null pointer");
  const u128 s0 = mk128(state_hi, state_lo), inc = mk128(inc_hi, inc_lo);
  const double ab = a + b;
  const double c_norm = c / (1.0 - ab), a_norm = a / ab;
  const Affine adv_c = advance_map(inc, (uint64_t)count);
  const Affine adv_2c = advance_map(inc, 2 * (uint64_t)count);
  const int64_t per = 64;
  const int64_t threads = (count + per - 1) / per;
  const int block = 256;
  rmat_pairs_kernel<<<(unsigned)((threads + block - 1) / block), block, 0, as_stream(stream)>>>(
      s0, inc, adv_c, adv_2c, scale, count, ab, a_norm, c_norm, per, src, dst);
  return check_launch("rmat_pairs");
}

int pg_pcg64_uniform(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo, int64_t offset,
                     int64_t count, double* out, void* stream) {
  PG_REQUIRE(offset >= 0 && count >= 0, "bad range");
  if (count == 0) return PG_OK;
  PG_REQUIRE(out, "null pointer");
  const int64_t per = 64, threads = (count + per - 1) / per;
  pcg_uniform_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, as_stream(stream)>>>(
      mk128(state_hi, state_lo), mk128(inc_hi, inc_lo), offset, count, per, out);
  return check_launch("pcg64_uniform");
}

int pg_searchsorted_right(const double* cdf, int64_t n, const double* u, int64_t count, int64_t* out,
                          void* stream) {
  PG_REQUIRE(n >= 1 && count >= 0, "bad sizes");
  if (count == 0) return PG_OK;
  PG_REQUIRE(cdf && u && out, "null pointer");
  searchsorted_right_kernel<<<sm_count() * 8, 256, 0, as_stream(stream)>>>(cdf, n, u, count, out);
  return check_launch("searchsorted_right");
}

int pg_csr_from_pairs(const int64_t* a, const int64_t* b, int64_t count, int64_t n, int64_t* offsets,
                      int32_t* adj, int64_t capacity, int64_t* nnz_host, void* stream) {
  PG_REQUIRE(count >= 0 && n >= 1 && n < (int64_t)1 << 31, "bad sizes");
  PG_REQUIRE(offsets && nnz_host, "null pointer");
  cudaStream_t s = as_stream(stream);
  const int grid = sm_count() * 8;
  *nnz_host = 0;
  if (count == 0) {
    cudaError_t e = cudaMemsetAsync(offsets, 0, sizeof(int64_t) * (n + 1), s);
    return e == cudaSuccess ? PG_OK : fail(PG_ERR_CUDA, "memset: %s", cudaGetErrorString(e));
  }
  PG_REQUIRE(a && b && adj, "null pointer");
  const uint64_t un = (uint64_t)n;
  const int end_bit = key_bits(un);
  // buffers: k0, k1 (2*count keys each, for the both-directions pass), count
  size_t t_sort = 0, t_uniq = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, t_sort, (const uint64_t*)nullptr, (uint64_t*)nullptr, 2 * count, 0,
                                 end_bit);
  cub::DeviceSelect::Unique(nullptr, t_uniq, (const uint64_t*)nullptr, (uint64_t*)nullptr, (int64_t*)nullptr,
                            count);
  const size_t kb = al256(sizeof(uint64_t) * 2 * count);
  const size_t temp = al256(t_sort > t_uniq ? t_sort : t_uniq);
  void* buf = nullptr;
  cudaError_t e = cudaMallocAsync(&buf, 2 * kb + temp + 256, s);
  if (e != cudaSuccess) return fail(PG_ERR_CUDA, "cudaMallocAsync: %s", cudaGetErrorString(e));
  char* p = static_cast<char*>(buf);
  uint64_t* k0 = reinterpret_cast<uint64_t*>(p);
  uint64_t* k1 = reinterpret_cast<uint64_t*>(p + kb);
  void* tmp = p + 2 * kb;
  int64_t* d_m = reinterpret_cast<int64_t*>(p + 2 * kb + temp);
  int rc = PG_OK;
  int64_t m = 0;
  do {
    canonical_keys_kernel<<<grid, 256, 0, s>>>(a, b, count, un, k0);
    if ((rc = check_launch("canonical_keys"))) break;
    size_t tb = temp;
    e = cub::DeviceRadixSort::SortKeys(tmp, tb, k0, k1, count, 0, end_bit, s);
    if (e != cudaSuccess) { rc = fail(PG_ERR_CUDA, "sort: %s", cudaGetErrorString(e)); break; }
    tb = temp;
    e = cub::DeviceSelect::Unique(tmp, tb, k1, k0, d_m, count, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(&m, d_m, sizeof(int64_t), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) { rc = fail(PG_ERR_CUDA, "unique: %s", cudaGetErrorString(e)); break; }
    // the loop sentinel n*n sorts last
    uint64_t last = 0;
    if (m > 0) {
      e = cudaMemcpyAsync(&last, k0 + (m - 1), sizeof(uint64_t), cudaMemcpyDeviceToHost, s);
      if (e == cudaSuccess) e = cudaStreamSynchronize(s);
      if (e != cudaSuccess) { rc = fail(PG_ERR_CUDA, "unique: %s", cudaGetErrorString(e)); break; }
      if (last == un * un) --m;
    }
    *nnz_host = 2 * m;
    if (2 * m > capacity) {
      rc = fail(PG_ERR_INVALID, "adjacency capacity %lld < %lld", (long long)capacity, (long long)(2 * m));
      break;
    }
    both_directions_kernel<<<grid, 256, 0, s>>>(k0, m, un, k1);
    if ((rc = check_launch("both_directions"))) break;
    tb = temp;
    e = cub::DeviceRadixSort::SortKeys(tmp, tb, k1, k0, 2 * m, 0, end_bit, s);
    if (e != cudaSuccess) { rc = fail(PG_ERR_CUDA, "sort: %s", cudaGetErrorString(e)); break; }
    int32_t* srcv = reinterpret_cast<int32_t*>(k1);  // k1 is free again
    split_keys_kernel<<<grid, 256, 0, s>>>(k0, 2 * m, un, adj, srcv);
    if ((rc = check_launch("split_keys"))) break;
    offsets_kernel<<<grid, 256, 0, s>>>(srcv, 2 * m, n, offsets);
    rc = check_launch("offsets");
  } while (false);
  cudaFreeAsync(buf, s);
  return rc;
}

int pg_degree_order(const int64_t* offsets, const int32_t* adj, int64_t n, int64_t nnz, int32_t* rank,
                    int64_t* dir_off, int32_t* dir_adj, void* stream) {
  PG_REQUIRE(n >= 0 && nnz >= 0, "bad sizes");
  PG_REQUIRE(n < (int64_t(1) << 31), "vertex IDs must fit in int32");
  PG_REQUIRE(nnz % 2 == 0, "a symmetric CSR has an even number of entries");
  PG_REQUIRE(offsets && dir_off && (n == 0 || rank), "null pointer");
  cudaStream_t s = as_stream(stream);
  const int grid = sm_count() * 8;
  if (n == 0) {
    cudaError_t e = cudaMemsetAsync(dir_off, 0, sizeof(int64_t), s);
    return e == cudaSuccess ? PG_OK : fail(PG_ERR_CUDA, "memset: %s", cudaGetErrorString(e));
  }
  PG_REQUIRE(nnz == 0 || (adj && dir_adj), "null pointer");
  size_t t_sort = 0, t_sel = 0, t_scan = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, t_sort, (const uint64_t*)nullptr, (uint64_t*)nullptr, n);
  cub::DeviceSelect::Flagged(nullptr, t_sel, (const int32_t*)nullptr, (const int32_t*)nullptr, (int32_t*)nullptr,
                             (int64_t*)nullptr, nnz);
  cub::DeviceScan::ExclusiveSum(nullptr, t_scan, (const int64_t*)nullptr, (int64_t*)nullptr, n + 1);
  size_t temp = t_sort;
  for (size_t t : {t_sel, t_scan}) temp = t > temp ? t : temp;
  temp = al256(temp);
  // keys (2n u64) | src, flags (nnz i32 each) | counts (n+1 i64) | num | temp
  const size_t kb = al256(sizeof(uint64_t) * 2 * n), eb = al256(sizeof(int32_t) * (nnz > 0 ? nnz : 1)),
               cb = al256(sizeof(int64_t) * (n + 1));
  void* buf = nullptr;
  cudaError_t e = cudaMallocAsync(&buf, kb + 2 * eb + cb + 256 + temp, s);
  if (e != cudaSuccess) return fail(PG_ERR_CUDA, "cudaMallocAsync: %s", cudaGetErrorString(e));
  char* p = static_cast<char*>(buf);
  uint64_t* k0 = reinterpret_cast<uint64_t*>(p);
  uint64_t* k1 = k0 + n;
  int32_t* src = reinterpret_cast<int32_t*>(p + kb);
  int32_t* flags = reinterpret_cast<int32_t*>(p + kb + eb);
  int64_t* counts = reinterpret_cast<int64_t*>(p + kb + 2 * eb);
  int64_t* d_num = reinterpret_cast<int64_t*>(p + kb + 2 * eb + cb);
  void* tmp = p + kb + 2 * eb + cb + 256;
  int rc = PG_OK;
  do {
    degree_keys_kernel<<<grid, 256, 0, s>>>(offsets, n, k0);
    if ((rc = check_launch("degree_keys"))) break;
    size_t tb = temp;
    e = cub::DeviceRadixSort::SortKeys(tmp, tb, k0, k1, n, 0, 64, s);
    if (e != cudaSuccess) { rc = fail(PG_ERR_CUDA, "sort: %s", cudaGetErrorString(e)); break; }
    rank_scatter_kernel<<<grid, 256, 0, s>>>(k1, n, rank);
    if ((rc = check_launch("rank_scatter"))) break;
    e = cudaMemsetAsync(counts + n, 0, sizeof(int64_t), s);
    if (e != cudaSuccess) { rc = fail(PG_ERR_CUDA, "memset: %s", cudaGetErrorString(e)); break; }
    if (nnz > 0) {
      if ((rc = pg_csr_expand_rows(offsets, n, nnz, src, stream))) break;
      orient_flags_kernel<<<grid, 256, 0, s>>>(src, adj, rank, nnz, flags);
      if ((rc = check_launch("orient_flags"))) break;
      tb = temp;
      e = cub::DeviceSelect::Flagged(tmp, tb, adj, flags, dir_adj, d_num, nnz, s);
      if (e != cudaSuccess) { rc = fail(PG_ERR_CUDA, "select: %s", cudaGetErrorString(e)); break; }
      // d+ per row: a warp per row (CUB's segmented reduce gives each
      // segment one block, and R-MAT hub rows of 10^5 entries serialised
      // it: 41 ms at s24)
      row_flag_count_kernel<<<grid, 256, 0, s>>>(offsets, flags, n, counts);
      if ((rc = check_launch("row_flag_count"))) break;
    } else {
      e = cudaMemsetAsync(counts, 0, sizeof(int64_t) * n, s);
      if (e != cudaSuccess) { rc = fail(PG_ERR_CUDA, "memset: %s", cudaGetErrorString(e)); break; }
    }
    tb = temp;
    e = cub::DeviceScan::ExclusiveSum(tmp, tb, counts, dir_off, n + 1, s);
    if (e != cudaSuccess) { rc = fail(PG_ERR_CUDA, "scan: %s", cudaGetErrorString(e)); break; }
  } while (false);
  cudaFreeAsync(buf, s);
  return rc;
}

// The in-lists of the degree orientation: x in N-(v) iff rank[x] < rank[v]
// (the transpose of pg_degree_order's N+ lists, adjacency order preserved),
// from ranks already computed.
int pg_degree_in_lists(const int64_t* offsets, const int32_t* adj, int64_t n, int64_t nnz, const int32_t* rank,
                       int64_t* in_off, int32_t* in_adj, void* stream) {
  PG_REQUIRE(n >= 0 && nnz >= 0 && nnz % 2 == 0, "bad sizes");
  PG_REQUIRE(offsets && in_off && (n == 0 || rank), "null pointer");
  cudaStream_t s = as_stream(stream);
  const int grid = sm_count() * 8;
  if (n == 0 || nnz == 0) {
    cudaError_t e = cudaMemsetAsync(in_off, 0, sizeof(int64_t) * (n + 1), s);
    return e == cudaSuccess ? PG_OK : fail(PG_ERR_CUDA, "memset: %s", cudaGetErrorString(e));
  }
  PG_REQUIRE(adj && in_adj, "null pointer");
  size_t t_sel = 0, t_scan = 0;
  cub::DeviceSelect::Flagged(nullptr, t_sel, (const int32_t*)nullptr, (const int32_t*)nullptr, (int32_t*)nullptr,
                             (int64_t*)nullptr, nnz);
  cub::DeviceScan::ExclusiveSum(nullptr, t_scan, (const int64_t*)nullptr, (int64_t*)nullptr, n + 1);
  const size_t temp = al256(t_sel > t_scan ? t_sel : t_scan);
  const size_t eb = al256(sizeof(int32_t) * nnz), cb = al256(sizeof(int64_t) * (n + 1));
  void* buf = nullptr;
  cudaError_t e = cudaMallocAsync(&buf, 2 * eb + cb + 256 + temp, s);
  if (e != cudaSuccess) return fail(PG_ERR_CUDA, "cudaMallocAsync: %s", cudaGetErrorString(e));
  char* p = static_cast<char*>(buf);
  int32_t* src = reinterpret_cast<int32_t*>(p);
  int32_t* flags = reinterpret_cast<int32_t*>(p + eb);
  int64_t* counts = reinterpret_cast<int64_t*>(p + 2 * eb);
  int64_t* d_num = reinterpret_cast<int64_t*>(p + 2 * eb + cb);
  void* tmp = p + 2 * eb + cb + 256;
  int rc = PG_OK;
  do {
    e = cudaMemsetAsync(counts + n, 0, sizeof(int64_t), s);
    if (e != cudaSuccess) { rc = fail(PG_ERR_CUDA, "memset: %s", cudaGetErrorString(e)); break; }
    if ((rc = pg_csr_expand_rows(offsets, n, nnz, src, stream))) break;
    orient_flags_in_kernel<<<grid, 256, 0, s>>>(src, adj, rank, nnz, flags);
    if ((rc = check_launch("orient_flags_in"))) break;
    size_t tb = temp;
    e = cub::DeviceSelect::Flagged(tmp, tb, adj, flags, in_adj, d_num, nnz, s);
    if (e != cudaSuccess) { rc = fail(PG_ERR_CUDA, "select: %s", cudaGetErrorString(e)); break; }
    row_flag_count_kernel<<<grid, 256, 0, s>>>(offsets, flags, n, counts);
    if ((rc = check_launch("row_flag_count"))) break;
    tb = temp;
    e = cub::DeviceScan::ExclusiveSum(tmp, tb, counts, in_off, n + 1, s);
    if (e != cudaSuccess) { rc = fail(PG_ERR_CUDA, "scan: %s", cudaGetErrorString(e)); break; }
  } while (false);
  cudaFreeAsync(buf, s);
  return rc;
}

}  // extern "C"
