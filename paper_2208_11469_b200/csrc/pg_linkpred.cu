// Link-prediction scoring on the device (reference mining.py:248-331):
// two-hop candidate pairs of a graph, their similarity scores
// (vertex_similarity, mining.py:162-203, for a batch) and the number of
// removed edges among the top-scored candidates.
//
//  * candidates: every pair (N(w)[i], N(w)[j]), i < j, of every vertex w
//    becomes a key u*n+v (u < v); keys are radix-sorted, deduplicated and
//    pairs that are already edges (binary search in row u) dropped -- the
//    reference's _two_hop_candidates (:275-296) in ascending (u, v) order;
//  * scores: counting measures from a per-pair intersection estimate and
//    exact degrees, in the reference's order of operations; membership
//    measures sum a per-degree term table (built on the host with math.log,
//    so terms are bit-identical) sequentially in ascending member order, as
//    the reference's Python loop does;
//  * ranking: a stable radix sort by descending score over the ascending
//    keys reproduces np.lexsort((v, u, -score)); hits are counted by binary
//    search in the sorted removed-edge keys.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>

#include "pg_common.cuh"

namespace pg {

namespace {

size_t al256(size_t x) { return (x + 255) & ~size_t(255); }

int key_bits64(uint64_t n) {
  const unsigned __int128 top = (unsigned __int128)n * n;  // keys < n*n
  int b = 1;
  while (b < 64 && ((unsigned __int128)1 << b) < top) ++b;
  return b;
}

__global__ void pair_count_kernel(const int64_t* __restrict__ offsets, int64_t n, int64_t* __restrict__ cnt) {
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w <= n; w += (int64_t)gridDim.x * blockDim.x) {
    if (w == n) {
      cnt[n] = 0;
    } else {
      const int64_t d = offsets[w + 1] - offsets[w];
      cnt[w] = d * (d - 1) / 2;
    }
  }
}

// warp per vertex w: pair (i, j), i < j, of row w goes to
// base[w] + i*d - i*(i+1)/2 + (j - i - 1)
__global__ void pair_gen_kernel(const int64_t* __restrict__ offsets, const int32_t* __restrict__ adj, int64_t n,
                                const int64_t* __restrict__ base, uint64_t* __restrict__ keys) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t w = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); w < n; w += nw) {
    const int64_t o = offsets[w], d = offsets[w + 1] - o;
    const int32_t* row = adj + o;
    uint64_t* out = keys + base[w];
    for (int64_t i = 0; i + 1 < d; ++i) {
      const uint64_t u = (uint64_t)row[i];
      const int64_t start = i * d - i * (i + 1) / 2;
      for (int64_t j = i + 1 + lane; j < d; j += 32)
        out[start + (j - i - 1)] = u * (uint64_t)n + (uint64_t)row[j];  // rows ascend: u < v
    }
  }
}

__device__ __forceinline__ bool row_contains(const int32_t* __restrict__ row, int64_t len, int32_t x) {
  int64_t lo = 0, hi = len;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (row[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  return lo < len && row[lo] == x;
}

__global__ void non_edge_flags_kernel(const uint64_t* __restrict__ keys, int64_t count, int64_t n,
                                      const int64_t* __restrict__ offsets, const int32_t* __restrict__ adj,
                                      int32_t* __restrict__ flags) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < count; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t u = (int64_t)(keys[t] / (uint64_t)n), v = (int64_t)(keys[t] % (uint64_t)n);
    flags[t] = !row_contains(adj + offsets[u], offsets[u + 1] - offsets[u], (int32_t)v);
  }
}

// ---- scores
// measure: 0 JACCARD, 1 OVERLAP, 2 COMMON_NEIGHBORS, 3 TOTAL_NEIGHBORS,
//          4 ADAMIC_ADAR, 5 RESOURCE_ALLOCATION  (mining.py SimilarityMeasure)
// members: 0 exact CSR rows, 1 1-Hash rows (sorted, lengths), 2 k-Hash rows
constexpr int kMaxMembers = 256;

__device__ __forceinline__ double deg_of(const int64_t* offsets, int64_t x) {
  return (double)(offsets[x + 1] - offsets[x]);
}

__global__ void counting_scores_kernel(int measure, const uint64_t* __restrict__ keys, int64_t count, int64_t n,
                                       const int64_t* __restrict__ offsets, const double* __restrict__ est,
                                       double* __restrict__ scores) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < count; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t u = (int64_t)(keys[t] / (uint64_t)n), v = (int64_t)(keys[t] % (uint64_t)n);
    const int64_t du = offsets[u + 1] - offsets[u], dv = offsets[v + 1] - offsets[v];
    double c = est[t];
    if (measure == 2) {
      scores[t] = c;
      continue;
    }
    // _feasible_count: min(max(c, 0.0), float(min(du, dv)))
    c = fmin(fmax(c, 0.0), (double)(du < dv ? du : dv));
    double r;
    if (measure == 0) {
      const double denom = __dsub_rn((double)(du + dv), c);
      r = denom > 0.0 ? __ddiv_rn(c, denom) : 0.0;
    } else if (measure == 1) {
      const int64_t lo = du < dv ? du : dv;
      r = lo > 0 ? __ddiv_rn(c, (double)lo) : 0.0;
    } else {
      r = __dsub_rn((double)(du + dv), c);
    }
    scores[t] = r;
  }
}

__global__ void member_scores_kernel(const uint64_t* __restrict__ keys, int64_t count, int64_t n,
                                     const int64_t* __restrict__ offsets, int source,
                                     const int32_t* __restrict__ rows, int k, const int32_t* __restrict__ lengths,
                                     const double* __restrict__ term, double* __restrict__ scores) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < count; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t u = (int64_t)(keys[t] / (uint64_t)n), v = (int64_t)(keys[t] % (uint64_t)n);
    double total = 0.0;
    if (source == 0 || source == 1) {  // sorted rows: merge, ascending members
      const int32_t *a, *b;
      int64_t la, lb;
      if (source == 0) {
        a = rows + offsets[u];
        la = offsets[u + 1] - offsets[u];
        b = rows + offsets[v];
        lb = offsets[v + 1] - offsets[v];
      } else {
        a = rows + u * (int64_t)k;
        la = lengths[u];
        b = rows + v * (int64_t)k;
        lb = lengths[v];
      }
      int64_t i = 0, j = 0;
      while (i < la && j < lb) {
        const int32_t x = a[i], y = b[j];
        if (x < y) ++i;
        else if (y < x) ++j;
        else {
          total = __dadd_rn(total, term[offsets[x + 1] - offsets[x]]);
          ++i;
          ++j;
        }
      }
    } else {  // k-Hash: distinct IDs of row u present in row v, ascending
      int32_t mem[kMaxMembers];
      int cnt = 0;
      const int32_t* a = rows + u * (int64_t)k;
      const int32_t* b = rows + v * (int64_t)k;
      for (int i = 0; i < k; ++i) {
        const int32_t x = a[i];
        if (x < 0) continue;
        bool seen = false;
        for (int q = 0; q < cnt && !seen; ++q) seen = mem[q] == x;
        if (seen) continue;
        bool inb = false;
        for (int q = 0; q < k && !inb; ++q) inb = b[q] == x;
        if (!inb) continue;
        int p = cnt++;  // insertion sort
        while (p > 0 && mem[p - 1] > x) {
          mem[p] = mem[p - 1];
          --p;
        }
        mem[p] = x;
      }
      for (int q = 0; q < cnt; ++q) total = __dadd_rn(total, term[offsets[mem[q] + 1] - offsets[mem[q]]]);
    }
    scores[t] = total;
  }
}

// descending-score sort key; +0.0 and -0.0 compare equal as in numpy
__global__ void score_keys_kernel(const double* __restrict__ scores, int64_t count, uint64_t* __restrict__ out) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < count; t += (int64_t)gridDim.x * blockDim.x) {
    double s = scores[t];
    if (s == 0.0) s = 0.0;
    const uint64_t b = (uint64_t)__double_as_longlong(s);
    out[t] = (b >> 63) ? ~b : (b | 0x8000000000000000ull);
  }
}

__global__ void hits_kernel(const uint64_t* __restrict__ top_keys, int64_t top, const uint64_t* __restrict__ removed,
                            int64_t n_removed, unsigned long long* __restrict__ hits) {
  unsigned long long h = 0;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < top; t += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t x = top_keys[t];
    int64_t lo = 0, hi = n_removed;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (removed[mid] < x) lo = mid + 1;
      else hi = mid;
    }
    h += lo < n_removed && removed[lo] == x;
  }
  for (int o = 16; o > 0; o >>= 1) h += __shfl_xor_sync(0xffffffffu, h, o);
  if ((threadIdx.x & 31) == 0 && h) atomicAdd(hits, h);
}

}  // namespace

}  // namespace pg

using namespace pg;

extern "C" {

int pg_two_hop_candidates(const int64_t* offsets, const int32_t* adj, int64_t n, uint64_t* keys_out,
                          int64_t capacity, int64_t* count_host, void* stream) {
  PG_REQUIRE(n >= 0, "n must be >= 0");
  PG_REQUIRE(n < (int64_t(1) << 31), "vertex IDs must fit in int32");
  PG_REQUIRE(offsets && count_host, "null pointer");
  cudaStream_t s = as_stream(stream);
  const int grid = sm_count() * 8;
  *count_host = 0;
  if (n == 0) return PG_OK;
  // per-vertex pair counts and their exclusive scan (n+1: the total last)
  size_t t_scan = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, t_scan, (const int64_t*)nullptr, (int64_t*)nullptr, n + 1);
  const size_t cb = al256(sizeof(int64_t) * (n + 1));
  void* buf = nullptr;
  cudaError_t e = cudaMallocAsync(&buf, 2 * cb + al256(t_scan), s);
  if (e != cudaSuccess) return fail(PG_ERR_CUDA, "cudaMallocAsync: %s", cudaGetErrorString(e));
  int64_t* cnt = static_cast<int64_t*>(buf);
  int64_t* base = reinterpret_cast<int64_t*>(static_cast<char*>(buf) + cb);
  void* tmp = static_cast<char*>(buf) + 2 * cb;
  int64_t total = 0;
  pair_count_kernel<<<grid, 256, 0, s>>>(offsets, n, cnt);
  size_t tb = t_scan;
  e = cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, base, n + 1, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(&total, base + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) {
    cudaFreeAsync(buf, s);
    return fail(PG_ERR_CUDA, "two-hop counts: %s", cudaGetErrorString(e));
  }
  if (!keys_out) {  // size query: the number of (w, i<j) pairs bounds the candidates
    *count_host = total;
    cudaFreeAsync(buf, s);
    return PG_OK;
  }
  if (total == 0) {
    cudaFreeAsync(buf, s);
    return PG_OK;
  }
  if (capacity < total) {
    cudaFreeAsync(buf, s);
    return fail(PG_ERR_INVALID, "candidate capacity %lld < %lld pairs", (long long)capacity, (long long)total);
  }
  PG_REQUIRE(adj, "null pointer");
  size_t t_sort = 0, t_uniq = 0, t_sel = 0;
  const int bits = key_bits64((uint64_t)n);
  cub::DeviceRadixSort::SortKeys(nullptr, t_sort, (const uint64_t*)nullptr, (uint64_t*)nullptr, total, 0, bits);
  cub::DeviceSelect::Unique(nullptr, t_uniq, (const uint64_t*)nullptr, (uint64_t*)nullptr, (int64_t*)nullptr, total);
  cub::DeviceSelect::Flagged(nullptr, t_sel, (const uint64_t*)nullptr, (const int32_t*)nullptr, (uint64_t*)nullptr,
                             (int64_t*)nullptr, total);
  size_t temp = t_sort > t_uniq ? t_sort : t_uniq;
  temp = al256(t_sel > temp ? t_sel : temp);
  const size_t kb = al256(sizeof(uint64_t) * total), fb = al256(sizeof(int32_t) * total);
  void* buf2 = nullptr;
  e = cudaMallocAsync(&buf2, kb + fb + 256 + temp, s);
  if (e != cudaSuccess) {
    cudaFreeAsync(buf, s);
    return fail(PG_ERR_CUDA, "cudaMallocAsync: %s", cudaGetErrorString(e));
  }
  uint64_t* k1 = static_cast<uint64_t*>(buf2);
  int32_t* flags = reinterpret_cast<int32_t*>(static_cast<char*>(buf2) + kb);
  int64_t* d_num = reinterpret_cast<int64_t*>(static_cast<char*>(buf2) + kb + fb);
  void* tmp2 = static_cast<char*>(buf2) + kb + fb + 256;
  int rc = PG_OK;
  int64_t uniq = 0, out = 0;
  do {
    // generate into keys_out (capacity >= total), sort into k1, unique back
    pair_gen_kernel<<<grid, 256, 0, s>>>(offsets, adj, n, base, keys_out);
    if ((rc = check_launch("pair_gen"))) break;
    tb = temp;
    e = cub::DeviceRadixSort::SortKeys(tmp2, tb, keys_out, k1, total, 0, bits, s);
    if (e != cudaSuccess) { rc = fail(PG_ERR_CUDA, "sort: %s", cudaGetErrorString(e)); break; }
    tb = temp;
    e = cub::DeviceSelect::Unique(tmp2, tb, k1, keys_out, d_num, total, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(&uniq, d_num, sizeof(int64_t), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) { rc = fail(PG_ERR_CUDA, "unique: %s", cudaGetErrorString(e)); break; }
    non_edge_flags_kernel<<<grid, 256, 0, s>>>(keys_out, uniq, n, offsets, adj, flags);
    if ((rc = check_launch("non_edge_flags"))) break;
    tb = temp;
    e = cub::DeviceSelect::Flagged(tmp2, tb, keys_out, flags, k1, d_num, uniq, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(&out, d_num, sizeof(int64_t), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e == cudaSuccess && out > 0)
      e = cudaMemcpyAsync(keys_out, k1, sizeof(uint64_t) * out, cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) { rc = fail(PG_ERR_CUDA, "non-edge select: %s", cudaGetErrorString(e)); break; }
    *count_host = out;
  } while (false);
  cudaFreeAsync(buf2, s);
  cudaFreeAsync(buf, s);
  return rc;
}

int pg_similarity_scores(int32_t measure, const uint64_t* keys, int64_t count, int64_t n, const int64_t* offsets,
                         const double* est, int32_t member_source, const int32_t* rows, int32_t k,
                         const int32_t* lengths, const double* term, double* scores, void* stream) {
  PG_REQUIRE(measure >= 0 && measure <= 5, "unknown similarity measure");
  PG_REQUIRE(count >= 0 && n > 0, "bad sizes");
  if (count == 0) return PG_OK;
  PG_REQUIRE(keys && offsets && scores, "null pointer");
  cudaStream_t s = as_stream(stream);
  const int grid = sm_count() * 8;
  if (measure <= 3) {
    PG_REQUIRE(est, "counting measures need the per-pair estimates");
    counting_scores_kernel<<<grid, 256, 0, s>>>(measure, keys, count, n, offsets, est, scores);
    return check_launch("counting_scores");
  }
  PG_REQUIRE(member_source >= 0 && member_source <= 2, "unknown member source");
  PG_REQUIRE(rows && term, "null pointer");
  PG_REQUIRE(member_source == 0 || (k >= 1 && k <= kMaxMembers), "sketch width out of range");
  PG_REQUIRE(member_source != 1 || lengths, "1-Hash members need lengths");
  member_scores_kernel<<<grid, 128, 0, s>>>(keys, count, n, offsets, member_source, rows, k, lengths, term, scores);
  return check_launch("member_scores");
}

int pg_rank_top_hits(const uint64_t* keys, const double* scores, int64_t count, int64_t top,
                     const uint64_t* removed_sorted, int64_t n_removed, int64_t* out_hits, void* stream) {
  PG_REQUIRE(count >= 0 && top >= 0 && n_removed >= 0, "bad sizes");
  PG_REQUIRE(out_hits, "null output");
  cudaStream_t s = as_stream(stream);
  cudaError_t e = cudaMemsetAsync(out_hits, 0, sizeof(int64_t), s);
  if (e != cudaSuccess) return fail(PG_ERR_CUDA, "memset: %s", cudaGetErrorString(e));
  if (top > count) top = count;
  if (top == 0 || n_removed == 0) return PG_OK;
  PG_REQUIRE(keys && scores && removed_sorted, "null pointer");
  size_t t_sort = 0;
  cub::DeviceRadixSort::SortPairsDescending(nullptr, t_sort, (const uint64_t*)nullptr, (uint64_t*)nullptr,
                                            (const uint64_t*)nullptr, (uint64_t*)nullptr, count);
  const size_t kb = al256(sizeof(uint64_t) * count);
  void* buf = nullptr;
  e = cudaMallocAsync(&buf, 3 * kb + al256(t_sort), s);
  if (e != cudaSuccess) return fail(PG_ERR_CUDA, "cudaMallocAsync: %s", cudaGetErrorString(e));
  uint64_t* sk = static_cast<uint64_t*>(buf);
  uint64_t* sk2 = reinterpret_cast<uint64_t*>(static_cast<char*>(buf) + kb);
  uint64_t* vals = reinterpret_cast<uint64_t*>(static_cast<char*>(buf) + 2 * kb);
  void* tmp = static_cast<char*>(buf) + 3 * kb;
  const int grid = sm_count() * 8;
  int rc = PG_OK;
  do {
    score_keys_kernel<<<grid, 256, 0, s>>>(scores, count, sk);
    if ((rc = check_launch("score_keys"))) break;
    size_t tb = t_sort;
    // stable: equal scores keep the ascending (u, v) key order
    e = cub::DeviceRadixSort::SortPairsDescending(tmp, tb, sk, sk2, keys, vals, count, 0, 64, s);
    if (e != cudaSuccess) { rc = fail(PG_ERR_CUDA, "sort: %s", cudaGetErrorString(e)); break; }
    hits_kernel<<<grid, 256, 0, s>>>(vals, top, removed_sorted, n_removed,
                                     reinterpret_cast<unsigned long long*>(out_hits));
    rc = check_launch("hits");
  } while (false);
  cudaFreeAsync(buf, s);
  return rc;
}

}  // extern "C"
