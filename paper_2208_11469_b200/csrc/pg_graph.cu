// Graph preparation on the device: upper-triangular edge list (the
// reference's CsrGraph.edges(), graphs.py:101-105), CSR row expansion
// (mining.py:83-85 _directed_edge_arrays), exact pair intersection counts
// (providers.py:102-115, setops.py:23-51) and raw hash words
// (hashing.py:114-118).
#include <algorithm>

#include <cub/device/device_scan.cuh>
#include <cuda/functional>

#include "pg_common.cuh"

namespace pg {

// first index of row u holding a neighbour > u, and the row's upper count
__global__ void upper_count_kernel(const int64_t* __restrict__ offsets, const int32_t* __restrict__ adj,
                                   int64_t n, int64_t* __restrict__ first, int64_t* __restrict__ cnt,
                                   int64_t pad, bool all) {
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n;
       u += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = offsets[u], hi = offsets[u + 1];
    const int64_t end = hi;
    if (all) hi = lo;  // every entry of the row (an oriented CSR)
    while (lo < hi) {  // lower_bound of u+1
      const int64_t mid = (lo + hi) >> 1;
      if (adj[mid] <= u) lo = mid + 1;
      else hi = mid;
    }
    first[u] = lo;
    cnt[u] = (end - lo + pad - 1) / pad * pad;  // slots of row u (rounded up to pad)
  }
}

// marks[start[u]] = u for every row with slots; an inclusive max-scan of the
// marks then yields the row of every output slot (load-balanced, coalesced)
__global__ void mark_rows_kernel(const int64_t* __restrict__ start, const int64_t* __restrict__ cnt, int64_t n,
                                 int32_t* __restrict__ marks) {
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n;
       u += (int64_t)gridDim.x * blockDim.x)
    if (cnt[u] > 0) marks[start[u]] = (int32_t)u;
}

// slot o of row u: the (o - start[u])-th upper neighbour, or -1 (padding)
__global__ void upper_gather_kernel(const int64_t* __restrict__ offsets, const int32_t* __restrict__ adj,
                                    const int64_t* __restrict__ first, const int64_t* __restrict__ start,
                                    const int32_t* __restrict__ us, int64_t total, int32_t* __restrict__ vs) {
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < total;
       o += (int64_t)gridDim.x * blockDim.x) {
    const int32_t u = us[o];
    const int64_t f = first[u];
    const int64_t off = o - start[u];
    vs[o] = off < offsets[u + 1] - f ? adj[f + off] : -1;
  }
}

// ---- edge slots of a vertex range, appended on the device (no host sync) ----
// Row u of [v0, v1) contributes its lower (< u) or upper (> u) neighbours,
// padded to a multiple of `pad` with v = -1, at a running device cursor.
// The TC of an upload chunk can then run as soon as the chunk and its
// sketches are on the device (the lower triangle of chunk c needs sketches
// of chunks <= c only).
__global__ void range_slot_count_kernel(const int64_t* __restrict__ offsets, const int32_t* __restrict__ adj,
                                        int64_t v0, int64_t v1, int lower, int64_t* __restrict__ first,
                                        int64_t* __restrict__ lens, int64_t* __restrict__ cnt, int64_t pad) {
  for (int64_t u = v0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < v1;
       u += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = offsets[u], hi = offsets[u + 1];
    const int64_t beg = lo, end = hi;
    while (lo < hi) {  // first neighbour > u (the CSR is loop-free)
      const int64_t mid = (lo + hi) >> 1;
      if (adj[mid] <= u) lo = mid + 1;
      else hi = mid;
    }
    const int64_t f = lower ? beg : lo, len = lower ? lo - beg : end - lo;
    first[u - v0] = f;
    lens[u - v0] = len;
    cnt[u - v0] = (len + pad - 1) / pad * pad;
  }
}

// marks[start[r]] = r + 1 for the range's non-empty rows (0 elsewhere); the
// inclusive max-scan of the marks gives every slot its row (load-balanced:
// a thread per slot, whatever the row lengths)
__global__ void range_slot_mark_kernel(const int64_t* __restrict__ cnt, const int64_t* __restrict__ start,
                                       int64_t rows, int32_t* __restrict__ marks) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x)
    if (cnt[r] > 0) marks[start[r]] = (int32_t)(r + 1);
}

// slot o of the range (o < its device-side total): row r = rowof[o] - 1,
// the (o - start[r])-th lower/upper neighbour or -1 (padding); a group-u
// entry per `pad` slots.  Slots past `capacity` are dropped and flagged.
__global__ void range_slot_gather_kernel(const int32_t* __restrict__ adj, int64_t v0, int64_t rows,
                                         const int64_t* __restrict__ first, const int64_t* __restrict__ lens,
                                         const int64_t* __restrict__ cnt, const int64_t* __restrict__ start,
                                         const int32_t* __restrict__ rowof, int64_t max_slots, int lg_pad,
                                         int64_t capacity, const int64_t* __restrict__ cursor,
                                         int64_t* __restrict__ overflow, int32_t* __restrict__ ug,
                                         int32_t* __restrict__ vs) {
  const int64_t base = cursor[0];
  const int64_t total = start[rows - 1] + cnt[rows - 1];
  const int64_t lim = min(total, max_slots);
  if (blockIdx.x == 0 && threadIdx.x == 0 && (total > max_slots || base + total > capacity)) *overflow = 1;
  const int64_t pad_mask = (int64_t(1) << lg_pad) - 1;
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < lim; o += (int64_t)gridDim.x * blockDim.x) {
    const int64_t slot = base + o;
    if (slot >= capacity) break;
    const int32_t r = rowof[o] - 1;
    const int64_t k = o - start[r];
    vs[slot] = k < lens[r] ? adj[first[r] + k] : -1;
    if ((k & pad_mask) == 0) ug[slot >> lg_pad] = (int32_t)(v0 + r);
  }
}

// advance the cursor past the range and record [begin, end) of the slots
// actually written (clamped to max_slots and capacity, as the gather; the
// overflow flag tells the caller the range was cut short)
__global__ void range_slot_finish_kernel(const int64_t* __restrict__ cnt, const int64_t* __restrict__ start,
                                         int64_t rows, int64_t max_slots, int64_t capacity,
                                         int64_t* __restrict__ cursor, int64_t* __restrict__ range) {
  const int64_t base = cursor[0];
  int64_t total = rows > 0 ? start[rows - 1] + cnt[rows - 1] : 0;
  total = min(total, max_slots);
  total = max(int64_t(0), min(total, capacity - base));
  range[0] = base;
  range[1] = base + total;
  cursor[0] = base + total;
}

// Fused exact triangle count: sum over the edges (us[e], vs[e]) of
// |N(u) & N(v)| in the CSR (offsets, adj) -- pairs_exact_kernel plus the sum,
// without the per-edge int64 output.  Warp per edge; the longer row is staged
// in the warp's shared memory when it fits (kTcStage ints) and every element
// of the shorter row is binary-searched there.
constexpr int kTcStage = 512;

__device__ __forceinline__ bool staged_contains(const int32_t* a, int len, int32_t x) {
  int lo = 0, hi = len;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  return lo < len && a[lo] == x;
}

// G lanes per edge (32/G edges per warp iteration), each group with its
// own stage of kTcStage * G / 32 ints
template <int G>
__global__ void __launch_bounds__(256) tc_exact_kernel(const int64_t* __restrict__ offsets,
                                                       const int32_t* __restrict__ adj,
                                                       const int32_t* __restrict__ us,
                                                       const int32_t* __restrict__ vs, int64_t count,
                                                       unsigned long long* __restrict__ out) {
  constexpr int E = 32 / G, kCap = kTcStage / E;
  __shared__ int32_t stage[8][kTcStage];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, gl = lane % G, grp = lane / G;
  const unsigned gmask = (G == 32 ? 0xffffffffu : ((1u << G) - 1u)) << (grp * G);
  int32_t* sB = stage[w] + grp * kCap;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  unsigned long long hits = 0;
  for (int64_t e0 = ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5) * E; e0 < count; e0 += warps * E) {
    const int64_t e = e0 + grp;
    int64_t ab = 0, ae = 0, bb = 0, be = 0;
    if (e < count) {
      const int32_t u = us[e], v = vs[e];
      ab = offsets[u]; ae = offsets[u + 1]; bb = offsets[v]; be = offsets[v + 1];
      if (ae - ab > be - bb) {
        int64_t t = ab; ab = bb; bb = t;
        t = ae; ae = be; be = t;
      }
    }
    const int64_t la = ae - ab, lb = be - bb;
    if (lb <= kCap) {
      for (int i = gl; i < lb; i += G) sB[i] = adj[bb + i];
      __syncwarp(gmask);
      for (int64_t j = gl; j < la; j += G) hits += staged_contains(sB, (int)lb, adj[ab + j]);
      __syncwarp(gmask);
    } else {
      for (int64_t j = ab + gl; j < ae; j += G) {
        const int32_t x = adj[j];
        int64_t lo = bb, hi = be;
        while (lo < hi) {
          const int64_t mid = (lo + hi) >> 1;
          if (adj[mid] < x) lo = mid + 1;
          else hi = mid;
        }
        hits += (lo < be && adj[lo] == x);
      }
    }
  }
  for (int o = 16; o > 0; o >>= 1) hits += __shfl_xor_sync(0xffffffffu, hits, o);
  if (lane == 0 && hits) atomicAdd(out, hits);
}

__global__ void mark_csr_rows_kernel(const int64_t* __restrict__ offsets, int64_t n, int32_t* __restrict__ marks) {
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n;
       u += (int64_t)gridDim.x * blockDim.x)
    if (offsets[u + 1] > offsets[u]) marks[offsets[u]] = (int32_t)u;
}

__global__ void hash_words_kernel(const int64_t* __restrict__ keys, int64_t count, uint64_t seed,
                                  uint64_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = mix64(seed ^ static_cast<uint64_t>(keys[i]));
}

// warp per pair: every element of the shorter row is binary-searched in the
// longer row (both sorted, duplicate free)
__global__ void pairs_exact_kernel(const int64_t* __restrict__ offsets, const int32_t* __restrict__ adj,
                                   const int32_t* __restrict__ us, const int32_t* __restrict__ vs,
                                   int64_t count, int64_t* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t e = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; e < count; e += warps) {
    const int32_t u = us[e], v = vs[e];
    int64_t ab = offsets[u], ae = offsets[u + 1], bb = offsets[v], be = offsets[v + 1];
    if (ae - ab > be - bb) {
      int64_t t = ab; ab = bb; bb = t;
      t = ae; ae = be; be = t;
    }
    int64_t hits = 0;
    for (int64_t j = ab + lane; j < ae; j += 32) {
      const int32_t x = adj[j];
      int64_t lo = bb, hi = be;
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (adj[mid] < x) lo = mid + 1;
        else hi = mid;
      }
      hits += (lo < be && adj[lo] == x);
    }
    for (int o = 16; o > 0; o >>= 1) hits += __shfl_xor_sync(0xffffffffu, hits, o);
    if (lane == 0) out[e] = hits;
  }
}

static size_t scan_temp_bytes(int64_t n) {
  size_t bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, bytes, (const int64_t*)nullptr, (int64_t*)nullptr, n);
  return bytes;
}
static size_t maxscan_temp_bytes(int64_t n) {
  size_t bytes = 0;
  cub::DeviceScan::InclusiveScan(nullptr, bytes, (const int32_t*)nullptr, (int32_t*)nullptr,
                                 ::cuda::maximum<>{}, n);
  return bytes;
}

static size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

// ---- Jarvis-Patrick components (mining.py:213-245): lock-free union-find
// over the kept edges.  Roots are hooked larger-index under smaller-index
// with atomicCAS, so parent[x] <= x always and the find loop (with path
// splitting) terminates; counting runs in a separate launch after every
// union has completed.
__device__ __forceinline__ int32_t cc_find(int32_t* parent, int32_t v) {
  int32_t curr = __ldcg(parent + v);
  if (curr != v) {
    int32_t prev = v, next;
    while (curr > (next = __ldcg(parent + curr))) {
      parent[prev] = next;
      prev = curr;
      curr = next;
    }
  }
  return curr;
}

__global__ void cc_init_kernel(int32_t* __restrict__ parent, uint8_t* __restrict__ touched, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    parent[i] = (int32_t)i;
    touched[i] = 0;
  }
}

__global__ void cc_union_kernel(const int32_t* __restrict__ us, const int32_t* __restrict__ vs,
                                const double* __restrict__ scores, int64_t count, double tau,
                                int32_t* parent, uint8_t* __restrict__ touched, uint8_t* __restrict__ keep_out,
                                unsigned long long* __restrict__ kept_total) {
  unsigned long long kept = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    const bool keep = scores[i] > tau;  // strict, as the reference
    if (keep_out) keep_out[i] = keep;
    if (!keep) continue;
    ++kept;
    const int32_t a = us[i], b = vs[i];
    touched[a] = 1;
    touched[b] = 1;
    int32_t ra = cc_find(parent, a), rb = cc_find(parent, b);
    while (ra != rb) {
      if (ra < rb) {
        const int32_t t = ra;
        ra = rb;
        rb = t;
      }
      // hook root ra (the larger) under rb; on failure ra gained a parent
      const int32_t old = atomicCAS(parent + ra, ra, rb);
      if (old == ra) break;
      ra = cc_find(parent, old);
      rb = cc_find(parent, rb);
    }
  }
  for (int o = 16; o > 0; o >>= 1) kept += __shfl_xor_sync(0xffffffffu, kept, o);
  if ((threadIdx.x & 31) == 0 && kept) atomicAdd(kept_total, kept);
}

__global__ void cc_count_kernel(int32_t* parent, const uint8_t* __restrict__ touched, int64_t n,
                                unsigned long long* __restrict__ out /* [kept, clusters, touched] */) {
  unsigned long long roots = 0, tv = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (touched[i]) {
      ++tv;
      roots += cc_find(parent, (int32_t)i) == (int32_t)i;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    roots += __shfl_xor_sync(0xffffffffu, roots, o);
    tv += __shfl_xor_sync(0xffffffffu, tv, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (roots) atomicAdd(out + 1, roots);
    if (tv) atomicAdd(out + 2, tv);
  }
}

}  // namespace pg

using namespace pg;

extern "C" {

int pg_csr_upper_edges_workspace(int64_t n, int64_t capacity, size_t* out_bytes_host) {
  PG_REQUIRE(n >= 0 && capacity >= 0 && out_bytes_host, "bad arguments");
  const size_t arr = align256(sizeof(int64_t) * (size_t)(n + 1));
  const size_t t1 = scan_temp_bytes(n > 0 ? n : 1), t2 = maxscan_temp_bytes(capacity > 0 ? capacity : 1);
  *out_bytes_host = 3 * arr + align256(t1 > t2 ? t1 : t2);
  return PG_OK;
}

static int upper_edges_impl(const int64_t* offsets, const int32_t* adj, int64_t n, int32_t* us, int32_t* vs,
                            int64_t capacity, int64_t* m_host, void* workspace, size_t workspace_bytes,
                            void* stream, int64_t pad, bool all = false) {
  PG_REQUIRE(n >= 0 && capacity >= 0, "bad sizes");
  PG_REQUIRE(offsets && workspace && m_host, "null pointer");
  size_t need = 0;
  pg_csr_upper_edges_workspace(n, capacity, &need);
  PG_REQUIRE(workspace_bytes >= need, "workspace too small (%zu < %zu)", workspace_bytes, need);
  cudaStream_t s = as_stream(stream);
  *m_host = 0;
  if (n == 0) return PG_OK;
  const size_t arr = align256(sizeof(int64_t) * (size_t)(n + 1));
  char* ws = static_cast<char*>(workspace);
  int64_t* first = reinterpret_cast<int64_t*>(ws);
  int64_t* cnt = reinterpret_cast<int64_t*>(ws + arr);
  int64_t* start = reinterpret_cast<int64_t*>(ws + 2 * arr);
  void* temp = ws + 3 * arr;
  size_t temp_bytes = workspace_bytes - 3 * arr;
  const int grid = sm_count() * 8;
  upper_count_kernel<<<grid, 256, 0, s>>>(offsets, adj, n, first, cnt, pad, all);
  if (int rc = check_launch("upper_count")) return rc;
  cudaError_t e = cub::DeviceScan::ExclusiveSum(temp, temp_bytes, cnt, start, n, s);
  if (e != cudaSuccess) return fail(PG_ERR_CUDA, "scan: %s", cudaGetErrorString(e));
  int64_t last_start = 0, last_cnt = 0;
  e = cudaMemcpyAsync(&last_start, start + (n - 1), sizeof(int64_t), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(&last_cnt, cnt + (n - 1), sizeof(int64_t), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return fail(PG_ERR_CUDA, "upper edge count: %s", cudaGetErrorString(e));
  const int64_t total = last_start + last_cnt;
  *m_host = total;
  if (total > capacity)
    return fail(PG_ERR_INVALID, "%lld upper edge slots exceed capacity %lld (asymmetric adjacency?)",
                (long long)total, (long long)capacity);
  if (total == 0) return PG_OK;
  PG_REQUIRE(us && vs, "null output");
  // vs serves as the mark buffer; its max-scan is the row of each slot
  e = cudaMemsetAsync(vs, 0, sizeof(int32_t) * total, s);
  if (e != cudaSuccess) return fail(PG_ERR_CUDA, "memset: %s", cudaGetErrorString(e));
  mark_rows_kernel<<<grid, 256, 0, s>>>(start, cnt, n, vs);
  if (int rc = check_launch("mark_rows")) return rc;
  e = cub::DeviceScan::InclusiveScan(temp, temp_bytes, vs, us, ::cuda::maximum<>{}, total, s);
  if (e != cudaSuccess) return fail(PG_ERR_CUDA, "max-scan: %s", cudaGetErrorString(e));
  upper_gather_kernel<<<grid, 256, 0, s>>>(offsets, adj, first, start, us, total, vs);
  return check_launch("upper_gather");
}

int pg_csr_upper_edges(const int64_t* offsets, const int32_t* adj, int64_t n, int32_t* us, int32_t* vs,
                       int64_t capacity, int64_t* m_host, void* workspace, size_t workspace_bytes,
                       void* stream) {
  return upper_edges_impl(offsets, adj, n, us, vs, capacity, m_host, workspace, workspace_bytes, stream, 1);
}

int pg_csr_upper_edges_padded(const int64_t* offsets, const int32_t* adj, int64_t n, int32_t pad,
                              int32_t* us, int32_t* vs, int64_t capacity, int64_t* slots_host,
                              void* workspace, size_t workspace_bytes, void* stream) {
  PG_REQUIRE(pad >= 1 && pad <= 32 && (pad & (pad - 1)) == 0, "pad must be a power of two <= 32");
  return upper_edges_impl(offsets, adj, n, us, vs, capacity, slots_host, workspace, workspace_bytes, stream,
                          pad);
}

int pg_csr_row_slots_padded(const int64_t* offsets, const int32_t* adj, int64_t n, int32_t pad, int32_t* us,
                            int32_t* vs, int64_t capacity, int64_t* slots_host, void* workspace,
                            size_t workspace_bytes, void* stream) {
  PG_REQUIRE(pad >= 1 && pad <= 32 && (pad & (pad - 1)) == 0, "pad must be a power of two <= 32");
  return upper_edges_impl(offsets, adj, n, us, vs, capacity, slots_host, workspace, workspace_bytes, stream,
                          pad, true);
}

int pg_csr_range_slots_workspace(int64_t rows, int64_t max_slots, size_t* bytes) {
  PG_REQUIRE(bytes && rows >= 0 && max_slots >= 0, "bad arguments");
  size_t t1 = 0, t2 = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, t1, (const int64_t*)nullptr, (int64_t*)nullptr, rows > 0 ? rows : 1);
  cub::DeviceScan::InclusiveScan(nullptr, t2, (const int32_t*)nullptr, (int32_t*)nullptr, ::cuda::maximum<>{},
                                 max_slots > 0 ? max_slots : 1);
  *bytes = 4 * align256(sizeof(int64_t) * (size_t)(rows + 1)) + 2 * align256(sizeof(int32_t) * (size_t)(max_slots + 1)) +
           align256(t1 > t2 ? t1 : t2);
  return PG_OK;
}

int pg_csr_range_slots_append(const int64_t* offsets, const int32_t* adj, int64_t v0, int64_t v1, int32_t pad,
                              int32_t lower, int64_t max_slots, int32_t* ug, int32_t* vs, int64_t capacity,
                              int64_t* cursor_dev, int64_t* range_dev, void* workspace, size_t workspace_bytes,
                              void* stream) {
  PG_REQUIRE(0 <= v0 && v0 <= v1, "bad vertex range");
  PG_REQUIRE(pad >= 1 && pad <= 32 && (pad & (pad - 1)) == 0, "pad must be a power of two <= 32");
  PG_REQUIRE(cursor_dev && range_dev && workspace, "null pointer");
  const int64_t rows = v1 - v0;
  size_t need = 0;
  pg_csr_range_slots_workspace(rows, max_slots, &need);
  PG_REQUIRE(workspace_bytes >= need, "workspace too small (%zu < %zu)", workspace_bytes, need);
  cudaStream_t s = as_stream(stream);
  const size_t arr = align256(sizeof(int64_t) * (size_t)(rows + 1));
  const size_t sarr = align256(sizeof(int32_t) * (size_t)(max_slots + 1));
  char* ws = static_cast<char*>(workspace);
  int64_t* first = reinterpret_cast<int64_t*>(ws);
  int64_t* cnt = reinterpret_cast<int64_t*>(ws + arr);
  int64_t* start = reinterpret_cast<int64_t*>(ws + 2 * arr);
  int64_t* lens = reinterpret_cast<int64_t*>(ws + 3 * arr);
  int32_t* marks = reinterpret_cast<int32_t*>(ws + 4 * arr);
  int32_t* rowof = reinterpret_cast<int32_t*>(ws + 4 * arr + sarr);
  void* temp = ws + 4 * arr + 2 * sarr;
  size_t temp_bytes = workspace_bytes - 4 * arr - 2 * sarr;
  const int grid = sm_count() * 8;
  if (rows > 0 && max_slots > 0) {
    PG_REQUIRE(offsets && adj && ug && vs, "null pointer");
    range_slot_count_kernel<<<grid, 256, 0, s>>>(offsets, adj, v0, v1, lower, first, lens, cnt, pad);
    if (int rc = check_launch("range_slot_count")) return rc;
    cudaError_t e = cub::DeviceScan::ExclusiveSum(temp, temp_bytes, cnt, start, rows, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(marks, 0, sizeof(int32_t) * (size_t)max_slots, s);
    if (e != cudaSuccess) return fail(PG_ERR_CUDA, "scan: %s", cudaGetErrorString(e));
    range_slot_mark_kernel<<<grid, 256, 0, s>>>(cnt, start, rows, marks);
    if (int rc = check_launch("range_slot_mark")) return rc;
    size_t tb = temp_bytes;
    e = cub::DeviceScan::InclusiveScan(temp, tb, marks, rowof, ::cuda::maximum<>{}, max_slots, s);
    if (e != cudaSuccess) return fail(PG_ERR_CUDA, "max-scan: %s", cudaGetErrorString(e));
    range_slot_gather_kernel<<<grid, 256, 0, s>>>(adj, v0, rows, first, lens, cnt, start, rowof, max_slots,
                                                  __builtin_ctz(pad), capacity, cursor_dev, cursor_dev + 1, ug, vs);
    if (int rc = check_launch("range_slot_gather")) return rc;
  }
  range_slot_finish_kernel<<<1, 1, 0, s>>>(cnt, start, rows > 0 && max_slots > 0 ? rows : 0, max_slots, capacity,
                                           cursor_dev, range_dev);
  return check_launch("range_slot_finish");
}

int pg_csr_expand_rows(const int64_t* offsets, int64_t n, int64_t nnz, int32_t* src, void* stream) {
  PG_REQUIRE(n >= 0 && nnz >= 0, "bad sizes");
  if (n == 0 || nnz == 0) return PG_OK;
  PG_REQUIRE(offsets && src, "null pointer");
  cudaStream_t s = as_stream(stream);
  // row marks in a transient stream-ordered buffer, max-scanned into src
  const size_t tb = maxscan_temp_bytes(nnz);
  void* buf = nullptr;
  cudaError_t e = cudaMallocAsync(&buf, align256(sizeof(int32_t) * nnz) + tb, s);
  if (e != cudaSuccess) return fail(PG_ERR_CUDA, "cudaMallocAsync: %s", cudaGetErrorString(e));
  int32_t* marks = static_cast<int32_t*>(buf);
  void* temp = static_cast<char*>(buf) + align256(sizeof(int32_t) * nnz);
  size_t temp_bytes = tb;
  e = cudaMemsetAsync(marks, 0, sizeof(int32_t) * nnz, s);
  if (e == cudaSuccess) {
    mark_csr_rows_kernel<<<sm_count() * 8, 256, 0, s>>>(offsets, n, marks);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess)
    e = cub::DeviceScan::InclusiveScan(temp, temp_bytes, marks, src, ::cuda::maximum<>{}, nnz, s);
  const cudaError_t e2 = cudaFreeAsync(buf, s);
  if (e != cudaSuccess) return fail(PG_ERR_CUDA, "expand_rows: %s", cudaGetErrorString(e));
  if (e2 != cudaSuccess) return fail(PG_ERR_CUDA, "cudaFreeAsync: %s", cudaGetErrorString(e2));
  return PG_OK;
}

int pg_hash_words(const int64_t* keys, int64_t count, uint64_t seed, uint64_t* out, void* stream) {
  PG_REQUIRE(count >= 0, "count must be >= 0");
  if (count == 0) return PG_OK;
  PG_REQUIRE(keys && out, "null pointer");
  hash_words_kernel<<<sm_count() * 4, 256, 0, as_stream(stream)>>>(keys, count, seed, out);
  return check_launch("hash_words");
}

int pg_tc_exact(const int64_t* offsets, const int32_t* adj, const int32_t* us, const int32_t* vs, int64_t count,
                int64_t* out_sum, void* stream) {
  PG_REQUIRE(count >= 0, "count must be >= 0");
  PG_REQUIRE(out_sum, "null output");
  cudaStream_t s = as_stream(stream);
  cudaError_t e = cudaMemsetAsync(out_sum, 0, sizeof(int64_t), s);
  if (e != cudaSuccess) return fail(PG_ERR_CUDA, "memset: %s", cudaGetErrorString(e));
  if (count == 0) return PG_OK;
  PG_REQUIRE(offsets && adj && us && vs, "null pointer");
  static const int G = [] {
    const char* v = getenv("PG_TC_EXACT_LANES");
    return v ? atoi(v) : 32;
  }();
#define PG_TE(GG)                                                                                       \
  {                                                                                                     \
    int per_sm = 0;                                                                                     \
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tc_exact_kernel<GG>, 256, 0) != cudaSuccess || \
        per_sm < 1)                                                                                     \
      per_sm = 1;                                                                                       \
    const int64_t need = (count + 8 * (32 / GG) - 1) / (8 * (32 / GG));                                 \
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)sm_count() * per_sm)); \
    tc_exact_kernel<GG><<<grid, 256, 0, s>>>(offsets, adj, us, vs, count,                              \
                                             reinterpret_cast<unsigned long long*>(out_sum));           \
  }
  if (G == 8) PG_TE(8)
  else if (G == 16) PG_TE(16)
  else PG_TE(32)
#undef PG_TE
  return check_launch("tc_exact");
}

int pg_pairs_exact(const int64_t* offsets, const int32_t* adj, const int32_t* us, const int32_t* vs,
                   int64_t count, int64_t* out_count, void* stream) {
  PG_REQUIRE(count >= 0, "count must be >= 0");
  if (count == 0) return PG_OK;
  PG_REQUIRE(offsets && us && vs && out_count, "null pointer");
  pairs_exact_kernel<<<sm_count() * 8, 256, 0, as_stream(stream)>>>(offsets, adj, us, vs, count, out_count);
  return check_launch("pairs_exact");
}

int pg_jp_components(const int32_t* us, const int32_t* vs, const double* scores, int64_t count, double tau,
                     int64_t n, uint8_t* keep_out, int64_t* out, void* stream) {
  PG_REQUIRE(count >= 0 && n >= 0, "bad sizes");
  PG_REQUIRE(n < (int64_t(1) << 31), "vertex IDs must fit in int32");
  PG_REQUIRE(out, "null output");
  cudaStream_t s = as_stream(stream);
  cudaError_t e = cudaMemsetAsync(out, 0, 3 * sizeof(int64_t), s);
  if (e != cudaSuccess) return fail(PG_ERR_CUDA, "memset: %s", cudaGetErrorString(e));
  if (n == 0) return PG_OK;
  PG_REQUIRE(count == 0 || (us && vs && scores), "null pointer");
  void* buf = nullptr;
  e = cudaMallocAsync(&buf, align256(sizeof(int32_t) * n) + n, s);
  if (e != cudaSuccess) return fail(PG_ERR_CUDA, "cudaMallocAsync: %s", cudaGetErrorString(e));
  int32_t* parent = static_cast<int32_t*>(buf);
  uint8_t* touched = static_cast<uint8_t*>(buf) + align256(sizeof(int32_t) * n);
  auto* o = reinterpret_cast<unsigned long long*>(out);
  const int grid = sm_count() * 8;
  cc_init_kernel<<<grid, 256, 0, s>>>(parent, touched, n);
  if (count > 0) cc_union_kernel<<<grid, 256, 0, s>>>(us, vs, scores, count, tau, parent, touched, keep_out, o);
  cc_count_kernel<<<grid, 256, 0, s>>>(parent, touched, n, o);
  e = cudaGetLastError();
  const cudaError_t e2 = cudaFreeAsync(buf, s);
  if (e != cudaSuccess) return fail(PG_ERR_CUDA, "jp_components: %s", cudaGetErrorString(e));
  if (e2 != cudaSuccess) return fail(PG_ERR_CUDA, "cudaFreeAsync: %s", cudaGetErrorString(e2));
  return PG_OK;
}

}  // extern "C"
