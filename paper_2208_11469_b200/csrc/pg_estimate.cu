// (2)+(3) Per-edge estimator kernels and their fused whole-graph reductions.
//
// Reference semantics (paths under /root/reference/pkg/src/probgraph):
//   Bloom   providers.py:137-162 (pair_many, _estimate_ones), estimators.py:65-70
//   k-Hash  providers.py:197-198,205-232   1-Hash providers.py:200-203,205-232
//   KMV     providers.py:266-301
//   TC      mining.py:105-130 (tc_estimate) over _chunked_sum (:63-80)
//   Jaccard estimators.py:123-131,148-168; mining.py:157-186 (vertex_similarity)
//
// Fixed-width row kernels (Bloom, k-Hash) use a "group" of G lanes per edge,
// each lane issuing V 128-bit loads per row.  A warp walks a contiguous edge
// range 32 edges at a time: lane i loads edge e0+i (coalesced), the group of
// lane i streams the rows of its G edges and a G-lane transpose-reduction
// leaves the count of edge e0+i back in lane i, which runs the epilogue.  The
// u row of consecutive edges is the same CSR row, so it is loaded through L1
// (ld.global.nc) while v rows bypass L1 (L1::no_allocate).
//
// Variable-length sorted rows (1-Hash IDs, KMV values) use one warp per edge,
// rows staged in shared memory and binary searched.
//
// Reductions are exact integers (histograms / per-match sums) wherever the
// reference's per-edge value is a function of an integer count, so sharded
// runs reproduce the single-GPU result bit for bit; only KMV sums doubles.
#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "pg_common.cuh"

namespace pg {

constexpr int kBlock = 256;

// ------------------------------------------------------------ row ops ----
struct OpAnd {
  __device__ __forceinline__ static int apply(uint4 a, uint4 b) {
    return __popc(a.x & b.x) + __popc(a.y & b.y) + __popc(a.z & b.z) + __popc(a.w & b.w);
  }
  __device__ __forceinline__ static int apply8(const uint32_t (&a)[8], const uint32_t (&b)[8]) {
    int c = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) c += __popc(a[w] & b[w]);
    return c;
  }
};
struct OpOr {
  __device__ __forceinline__ static int apply(uint4 a, uint4 b) {
    return __popc(a.x | b.x) + __popc(a.y | b.y) + __popc(a.z | b.z) + __popc(a.w | b.w);
  }
  __device__ __forceinline__ static int apply8(const uint32_t (&a)[8], const uint32_t (&b)[8]) {
    int c = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) c += __popc(a[w] | b[w]);
    return c;
  }
};
// k-Hash positional matches: (eu == ev) & (eu >= 0)   (providers.py:197-198)
struct OpEqPos {
  __device__ __forceinline__ static int apply(uint4 a, uint4 b) {
    return (a.x == b.x && (int)a.x >= 0) + (a.y == b.y && (int)a.y >= 0) +
           (a.z == b.z && (int)a.z >= 0) + (a.w == b.w && (int)a.w >= 0);
  }
  __device__ __forceinline__ static int apply8(const uint32_t (&a)[8], const uint32_t (&b)[8]) {
    int c = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) c += (a[w] == b[w] && (int)a[w] >= 0);
    return c;
  }
};

// G-lane transpose-reduction: on entry c[j] is this lane's partial count of
// edge j of its group; on exit the lane with group index gl holds the full
// count of edge gl in c[0].
template <int G>
__device__ __forceinline__ int group_transpose_reduce(int (&c)[G], int gl) {
#pragma unroll
  for (int w = G / 2; w >= 1; w >>= 1) {
    const bool upper = (gl & w) != 0;
#pragma unroll
    for (int j = 0; j < w; ++j) {
      const int send = upper ? c[j] : c[j + w];
      const int keep = upper ? c[j + w] : c[j];
      c[j] = keep + __shfl_xor_sync(0xffffffffu, send, w);
    }
  }
  return c[0];
}

// contiguous per-warp slice of [e_begin, e_end), rounded to 32 edges
__device__ __forceinline__ void warp_slice(int64_t e_begin, int64_t e_end, int64_t& wb, int64_t& we) {
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int64_t total = e_end - e_begin;
  int64_t per = (total + nwarps - 1) / nwarps;
  per = (per + 31) & ~int64_t(31);
  wb = e_begin + gw * per;
  we = min(wb + per, e_end);
  if (wb > e_end) wb = e_end;
}

// Group engine: calls epi.edge(e, u, v, count) once per edge of the warp's
// slice, from the lane that loaded the edge.
//
// Latency structure (the kernel is load-latency bound): the edge indices of
// iteration i+1 are loaded while the rows of iteration i are in flight, all
// G*V v-row loads of an iteration are issued before any is consumed, and the
// u row is cached in registers across consecutive edges (edges are in CSR
// order, so u changes on average once per ~40 edges at R-MAT scale 20) and
// only reloaded when it changes.
template <int V, int G, class Op, class Epi, bool kVCache = false>
__device__ __forceinline__ void group_edge_loop(const uint4* __restrict__ rows, const int32_t* __restrict__ us,
                                                const int32_t* __restrict__ vs, int64_t e_begin,
                                                int64_t e_end, Epi& epi) {
  constexpr int W4 = V * G;
  const int lane = threadIdx.x & 31;
  const int gl = lane & (G - 1);
  const int gbase = lane & ~(G - 1);
  int64_t wb, we;
  warp_slice(e_begin, e_end, wb, we);
  if (wb >= we) return;
  int32_t ul = 0, vl = 0;
  if (wb + lane < we) {
    ul = us[wb + lane];
    vl = vs[wb + lane];
  }
  int32_t ucur = -1;
  uint4 ur[V];
#pragma unroll
  for (int i = 0; i < V; ++i) ur[i] = make_uint4(0, 0, 0, 0);
#pragma unroll 1
  for (int64_t e0 = wb; e0 < we; e0 += 32) {
    const int64_t e = e0 + lane;
    const bool valid = e < we && vl >= 0;  // v < 0: padding slot
    // prefetch the next iteration's edge indices
    int32_t un = 0, vn = 0;
    if (e + 32 < we) {
      un = us[e + 32];
      vn = vs[e + 32];
    }
    uint4 vr[G][V];
#pragma unroll
    for (int j = 0; j < G; ++j) {
      const int32_t vj = __shfl_sync(0xffffffffu, vl, gbase + j);
      const uint4* rv = rows + (int64_t)(vj < 0 ? 0 : vj) * W4 + gl;
#pragma unroll
      for (int i = 0; i < V; ++i) vr[j][i] = kVCache ? ldg_keep(rv + i * G) : ldg_stream(rv + i * G);
    }
    int c[G];
#pragma unroll
    for (int j = 0; j < G; ++j) {
      const int32_t uj = __shfl_sync(0xffffffffu, ul, gbase + j);
      if (uj != ucur) {  // group-uniform; rare
        ucur = uj;
        const uint4* ru = rows + (int64_t)uj * W4 + gl;
#pragma unroll
        for (int i = 0; i < V; ++i) ur[i] = ldg_keep(ru + i * G);
      }
      int acc = 0;
#pragma unroll
      for (int i = 0; i < V; ++i) acc += Op::apply(ur[i], vr[j][i]);
      c[j] = acc;
    }
    const int cnt = group_transpose_reduce<G>(c, gl);
    if (valid) epi.edge(e, ul, vl, cnt);
    ul = un;
    vl = vn;
  }
}

// ------------------------------------------------- wide (256-bit) engine
// sm_100 has 256-bit global loads (LDG.E.ENL2.256): a lane moves 32 bytes per
// instruction, so a 128-byte Bloom row is 4 lanes and a 256-byte row 8 lanes.
// Same warp/group/transpose structure as group_edge_loop with half the load
// instructions and twice the bytes in flight per register.
__device__ __forceinline__ void ldg256(const void* p, uint32_t (&r)[8]) {
  asm volatile("ld.global.nc.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                 "=r"(r[7])
               : "l"(p));
}
__device__ __forceinline__ void ldg256_keep(const void* p, uint32_t (&r)[8]) {
  asm volatile("ld.global.nc.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                 "=r"(r[7])
               : "l"(p));
}

// kLayout: 0 any edge list; 1 row-padded slots (every aligned group of G
// slots shares one u; us[] per slot); 2 the same with us[] holding one u per
// group (us[e / G]) -- a G-fold smaller u stream.
template <int W8, class Op, class Epi, bool kVCache = false, int kLayout = 0>
__device__ __forceinline__ void wide_edge_loop(const unsigned char* __restrict__ rows,
                                               const int32_t* __restrict__ us, const int32_t* __restrict__ vs,
                                               int64_t e_begin, int64_t e_end, Epi& epi) {
  constexpr bool kPadded = kLayout > 0;
  constexpr int G = W8 < 8 ? W8 : 8;  // lanes per edge
  constexpr int V = W8 / G;           // 32-byte chunks per lane per row
  constexpr int64_t kRowBytes = W8 * 32;
  const int lane = threadIdx.x & 31;
  const int gl = lane & (G - 1);
  const int gbase = lane & ~(G - 1);
  int64_t wb, we;
  warp_slice(e_begin, e_end, wb, we);
  if (wb >= we) return;
  int32_t ul = 0, vl = 0;
  if (wb + lane < we) {
    ul = kLayout == 2 ? us[(wb + lane) / G] : us[wb + lane];
    vl = vs[wb + lane];
  }
  int32_t ucur = -1;
  uint32_t ur[V][8];
#pragma unroll
  for (int i = 0; i < V; ++i)
#pragma unroll
    for (int w = 0; w < 8; ++w) ur[i][w] = 0;
  // 32-bit remaining-slot count instead of 64-bit bound checks (registers)
  const int nslots = (int)(we - wb);
#pragma unroll 1
  for (int r0 = 0; r0 < nslots; r0 += 32) {
    const int64_t e = wb + r0 + lane;
    const int rem = nslots - r0;
    const bool valid = lane < rem && vl >= 0;  // v < 0: padding slot
    int32_t un = 0, vn = 0;
    if (lane + 32 < rem) {
      un = kLayout == 2 ? us[(e + 32) / G] : us[e + 32];
      vn = vs[e + 32];
    }
    uint32_t vr[G][V][8];
#pragma unroll
    for (int j = 0; j < G; ++j) {
      const int32_t vj = __shfl_sync(0xffffffffu, vl, gbase + j);
      const unsigned char* rv = rows + (int64_t)(vj < 0 ? 0 : vj) * kRowBytes + gl * 32;
#pragma unroll
      for (int i = 0; i < V; ++i) {
        if (kVCache) ldg256_keep(rv + i * G * 32, vr[j][i]);
        else ldg256(rv + i * G * 32, vr[j][i]);
      }
    }
    // u rows: with the row-padded edge layout (pg_csr_upper_edges_padded)
    // all G edges of a group share one u, cached across iterations; for any
    // other input the per-edge rows are loaded speculatively in parallel.
    const int32_t u0 = __shfl_sync(0xffffffffu, ul, gbase);
    bool uniform = true;
    if (!kPadded) {
#pragma unroll
      for (int j = 1; j < G; ++j) uniform &= __shfl_sync(0xffffffffu, ul, gbase + j) == u0;
    }
    int c[G];
    if (kPadded || __all_sync(0xffffffffu, uniform)) {
      if (u0 != ucur) {
        ucur = u0;
        const unsigned char* ru = rows + (int64_t)u0 * kRowBytes + gl * 32;
#pragma unroll
        for (int i = 0; i < V; ++i) ldg256_keep(ru + i * G * 32, ur[i]);
      }
#pragma unroll
      for (int j = 0; j < G; ++j) {
        int acc = 0;
#pragma unroll
        for (int i = 0; i < V; ++i) acc += Op::apply8(ur[i], vr[j][i]);
        c[j] = acc;
      }
    } else if (!kPadded) {
#pragma unroll
      for (int j = 0; j < G; ++j) {
        const int32_t uj = __shfl_sync(0xffffffffu, ul, gbase + j);
        if (uj != ucur) {
          ucur = uj;
          const unsigned char* ru = rows + (int64_t)uj * kRowBytes + gl * 32;
#pragma unroll
          for (int i = 0; i < V; ++i) ldg256_keep(ru + i * G * 32, ur[i]);
        }
        int acc = 0;
#pragma unroll
        for (int i = 0; i < V; ++i) acc += Op::apply8(ur[i], vr[j][i]);
        c[j] = acc;
      }
    }
    const int cnt = group_transpose_reduce<G>(c, gl);
    if (valid) epi.edge(e, ul, vl, cnt);
    ul = un;
    vl = vn;
  }
}

// ------------------------------------------------ sorted-row group engine
// 1-Hash (ascending int32 IDs, -1 pad) and KMV (ascending doubles as uint64
// bits, +inf pad) rows of k = 8*G*CH elements.  G lanes per edge (32/G edges
// per warp iteration); lane gl holds the CH chunks c = s*G + gl of 8
// consecutive elements, loaded with 256-bit loads.  A membership / rank
// query for x against a row uses (1) the broadcast heads of all k/8 chunks
// held in registers to pick the chunk, then (2) a 4-probe lower_bound inside
// that 8-element chunk, read from the row's shared-memory copy.
template <class T>
struct SortedTraits;
template <>
struct SortedTraits<int32_t> {
  static constexpr int kLoads = 1;  // 256-bit loads per 8-element chunk
  __device__ static int32_t pad() { return 0x7fffffff; }
  __device__ static int32_t fix(int32_t x) { return x < 0 ? 0x7fffffff : x; }  // -1 pad sorts last
  __device__ static bool valid(int32_t x) { return x != 0x7fffffff; }
};
template <>
struct SortedTraits<uint64_t> {
  static constexpr int kLoads = 2;
  __device__ static uint64_t pad() { return kInfBits; }
  __device__ static uint64_t fix(uint64_t x) { return x; }
  __device__ static bool valid(uint64_t x) { return x < kInfBits; }
};

// KMV keys compared as doubles: the values are non-negative (or the +inf
// pad), so IEEE order equals the bit order and one DSETP replaces a 64-bit
// integer compare (two ISETPs)
template <>
struct SortedTraits<double> {
  __device__ static double pad() { return __longlong_as_double((long long)kInfBits); }
  __device__ static bool valid(double x) { return x < __longlong_as_double((long long)kInfBits); }
};

__device__ __forceinline__ double key_of(uint64_t bits) { return __longlong_as_double((long long)bits); }
__device__ __forceinline__ int32_t key_of(int32_t x) { return x; }
__device__ __forceinline__ uint64_t bits_of(double x) { return (uint64_t)__double_as_longlong(x); }
__device__ __forceinline__ uint64_t bits_of(int32_t x) { return (uint64_t)(uint32_t)x; }

template <class T, int CH, bool kKeep>
__device__ __forceinline__ void load_sorted_chunks(const T* row, int G, int gl, T (&c)[CH][8]) {
#pragma unroll
  for (int s = 0; s < CH; ++s) {
    const T* p = row + (s * G + gl) * 8;
    uint32_t r[8];
#pragma unroll
    for (int h = 0; h < SortedTraits<T>::kLoads; ++h) {
      if (kKeep) ldg256_keep(reinterpret_cast<const unsigned char*>(p) + 32 * h, r);
      else ldg256(reinterpret_cast<const unsigned char*>(p) + 32 * h, r);
      if (sizeof(T) == 4) {
#pragma unroll
        for (int w = 0; w < 8; ++w) c[s][w] = SortedTraits<T>::fix((T)r[w]);
      } else {
#pragma unroll
        for (int w = 0; w < 4; ++w)
          c[s][4 * h + w] = (T)(((uint64_t)r[2 * w + 1] << 32) | r[2 * w]);
      }
    }
  }
}

// lower_bound of x in a row: heads[i] = first element of chunk i (NC chunks),
// srow = the row in element order (shared memory).  lt = #elements < x.
template <class T, int NC>
__device__ __forceinline__ int sorted_lower_bound(T x, const T (&heads)[NC], const T* srow, bool& found) {
  int c = 0;
#pragma unroll
  for (int i = 0; i < NC; ++i) c += heads[i] <= x;
  if (c == 0) {
    found = false;
    return 0;
  }
  const T* ch = srow + (c - 1) * 8;
  int p = 0;
  if (ch[3] < x) p = 4;
  if (ch[p + 1] < x) p += 2;
  if (ch[p] < x) p += 1;
  if (p < 8 && ch[p] < x) p += 1;
  found = p < 8 && ch[p] == x;
  return (c - 1) * 8 + p;
}

// lower_bound of x in a row held in registers across the group: chunk c
// (8 sorted values) lives in lane gbase + c % G (slot c / G, CH == 1 here),
// heads[] are the broadcast chunk heads.  The chunk is fetched with 8
// register shuffles -- no shared memory, so no bank conflicts.  Every lane
// must call this (shuffles); `active` masks the result.
template <class T, int NC>
__device__ __forceinline__ int shfl_lower_bound(T x, bool active, const T (&heads)[NC], const T (&mine)[8],
                                                int gbase, bool& found) {
  int c = 0;
#pragma unroll
  for (int i = 0; i < NC; ++i) c += heads[i] <= x;
  const int chunk = c > 0 ? c - 1 : 0;
  const int src = gbase + chunk;  // CH == 1: chunk i is lane i of the group
  int lt = 0;
  bool eq = false;
#pragma unroll
  for (int w = 0; w < 8; ++w) {
    T y;
    if constexpr (sizeof(T) == 8) y = (T)shfl64((uint64_t)mine[w], src);
    else y = __shfl_sync(0xffffffffu, mine[w], src);
    lt += y < x;
    eq |= y == x;
  }
  found = active && c > 0 && eq;
  return (active && c > 0) ? chunk * 8 + lt : 0;
}

struct SortedStats {
  int common, lu, lv;
  double kth;
};

// G-lane group sums / exclusive scans (groups are aligned lane ranges)
template <int G>
__device__ __forceinline__ int group_sum(int x) {
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}
template <int G>
__device__ __forceinline__ int group_excl_scan(int x, int gl) {
  int inc = x;
#pragma unroll
  for (int o = 1; o < G; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, inc, o);
    if (gl >= o) inc += y;
  }
  return inc - x;
}

// 1-Hash lookup engine: every U element is looked up in V (chunk heads
// broadcast, the chunk itself by register shuffles for CH == 1 or from a
// shared-memory copy for CH > 1); common = number of hits.
template <int G, int CH, class Epi>
__device__ __forceinline__ void sorted_edge_loop(const int32_t* __restrict__ R, int k,
                                                 const int32_t* __restrict__ us,
                                                 const int32_t* __restrict__ vs, int64_t e_begin,
                                                 int64_t e_end, unsigned char* warp_smem, Epi& epi) {
  using T = int32_t;
  using TR = SortedTraits<T>;
  constexpr int NC = G * CH;  // chunks per row (k / 8)
  constexpr int E = 32 / G;   // edges per warp iteration
  const int lane = threadIdx.x & 31;
  const int gl = lane & (G - 1);
  const int gbase = lane & ~(G - 1);
  const int grp = lane / G;
  T* sv = reinterpret_cast<T*>(warp_smem) + grp * NC * 8;
  int64_t wb, we;
  warp_slice(e_begin, e_end, wb, we);
  if (wb >= we) return;
  int32_t ul = 0, vl = 0;
  if (wb + grp < we) {
    ul = us[wb + grp];
    vl = vs[wb + grp];
  }
#pragma unroll 1
  for (int64_t e0 = wb; e0 < we; e0 += E) {
    const int64_t e = e0 + grp;
    const bool valid = e < we;  // 1-Hash uses the unpadded edge layout
    int32_t un = 0, vn = 0;
    if (e + E < we) {
      un = us[e + E];
      vn = vs[e + E];
    }
    T a[CH][8], b[CH][8];
    load_sorted_chunks<T, CH, true>(R + (int64_t)ul * k, G, gl, a);
    load_sorted_chunks<T, CH, false>(R + (int64_t)vl * k, G, gl, b);
    int la = 0, lb = 0;
#pragma unroll
    for (int s = 0; s < CH; ++s) {
#pragma unroll
      for (int w = 0; w < 8; ++w) {
        la += TR::valid(a[s][w]);
        lb += TR::valid(b[s][w]);
      }
    }
    la = group_sum<G>(la);
    lb = group_sum<G>(lb);
    if constexpr (CH > 1) {  // shared-memory copy of V for the chunk searches
#pragma unroll
      for (int s = 0; s < CH; ++s) {
        const int c = s * G + gl;
#pragma unroll
        for (int w = 0; w < 8; ++w) sv[c * 8 + w] = b[s][w];
      }
    }
    T hb[NC];
#pragma unroll
    for (int i = 0; i < NC; ++i) hb[i] = __shfl_sync(0xffffffffu, b[i / G][0], gbase + i % G);
    __syncwarp();
    int found = 0;
#pragma unroll
    for (int s = 0; s < CH; ++s)
#pragma unroll
      for (int w = 0; w < 8; ++w) {
        bool f = false;
        if constexpr (CH == 1) {
          shfl_lower_bound<T, NC>(a[s][w], TR::valid(a[s][w]), hb, b[0], gbase, f);
        } else {
          if (TR::valid(a[s][w])) sorted_lower_bound<T, NC>(a[s][w], hb, sv, f);
        }
        found += f;
      }
    SortedStats st;
    st.common = group_sum<G>(found);
    st.lu = la;
    st.lv = lb;
    st.kth = 0.0;
    if (valid && gl == 0) epi.edge(e, ul, vl, st);
    __syncwarp();
    ul = un;
    vl = vn;
  }
}

// ------------------------------------------------ 1-Hash hash-table engine
// G = K/8 lanes per edge (8 IDs per lane), 32/G edges per warp iteration.
// The u row's IDs are inserted once per run of edges sharing u (CSR order
// keeps them consecutive) into a per-group shared-memory table of K buckets
// x 4 slots (multiplicative hash of the ID; slots claimed with atomicCAS;
// the rare fifth entry of a bucket goes to a stash).  Every v ID is then one
// 16-byte bucket load + 4 compares (+ the stash when it is non-empty): one
// LDS.128 per lookup where a binary search needs log2(K)+1 dependent loads.
// Row lengths are min(size, K); the endpoints' sizes are prefetched with
// the next edge's indices.  1-Hash needs only the number of common IDs
// (providers.py:205-232 _matches_onehash).
template <int K>
__host__ __device__ constexpr int htab_group_ints() { return 4 * K + K + 4; }  // table | stash | count

template <int K>
__device__ __forceinline__ uint32_t htab_bucket(int32_t x) {
  constexpr int kBits = K == 32 ? 5 : (K == 64 ? 6 : 7);
  return ((uint32_t)x * 0x9E3779B1u) >> (32 - kBits);
}

// P consecutive 32-bit IDs of a row (P a multiple of 8, 32-byte aligned)
template <int P>
__device__ __forceinline__ void ldg_rowpart(const int32_t* p, uint32_t (&x)[P]) {
#pragma unroll
  for (int c = 0; c < P / 8; ++c) {
    uint32_t r[8];
    ldg256_keep(p + 8 * c, r);
#pragma unroll
    for (int i = 0; i < 8; ++i) x[8 * c + i] = r[i];
  }
}

template <int K, int P, class Epi>
__device__ __forceinline__ void htab_edge_loop(const int32_t* __restrict__ R, const int32_t* __restrict__ sizes,
                                               const int32_t* __restrict__ us, const int32_t* __restrict__ vs,
                                               int64_t e_begin, int64_t e_end, int32_t* warp_smem, Epi& epi) {
  constexpr int G = K / P, E = 32 / G;
  const int lane = threadIdx.x & 31, gl = lane & (G - 1), grp = lane / G;
  const unsigned gmask = ((G == 32) ? 0xffffffffu : ((1u << G) - 1u)) << (grp * G);
  int32_t* T = warp_smem + grp * htab_group_ints<K>();  // 4K slots
  int32_t* S = T + 4 * K;                                 // stash (K)
  int* sc_p = reinterpret_cast<int*>(S + K);
  int64_t wb, we;
  warp_slice(e_begin, e_end, wb, we);
  if (wb >= we) return;
  int32_t ul = 0, vl = -1, szu = 0, szv = 0;
  if (wb + grp < we) {
    ul = us[wb + grp];
    vl = vs[wb + grp];
    szu = sizes[ul];
    szv = vl < 0 ? 0 : sizes[vl];
  }
  uint32_t x[P];
  ldg_rowpart<P>(R + (int64_t)(vl < 0 ? 0 : vl) * K + gl * P, x);
  int32_t cur_u = -1;
  int sc = 0;
#pragma unroll 1
  for (int64_t e0 = wb; e0 < we; e0 += E) {
    const int64_t e = e0 + grp;
    const bool valid = e < we && vl >= 0;
    int32_t un = 0, vn = -1;
    if (e + E < we) {
      un = us[e + E];
      vn = vs[e + E];
    }
    if (ul != cur_u) {  // uniform within the group: (re)build its table
      uint32_t y[P];
      ldg_rowpart<P>(R + (int64_t)ul * K + gl * P, y);
      int4* T4 = reinterpret_cast<int4*>(T);
#pragma unroll
      for (int i = gl; i < K; i += G) T4[i] = make_int4(-1, -1, -1, -1);
      if (gl == 0) *sc_p = 0;
      __syncwarp(gmask);
#pragma unroll
      for (int p = 0; p < P; ++p) {
        const int32_t q = (int32_t)y[p];
        if (q < 0) continue;  // -1 pad
        int32_t* bk = T + 4 * htab_bucket<K>(q);
        bool placed = false;
#pragma unroll
        for (int sl = 0; sl < 4 && !placed; ++sl) placed = atomicCAS(bk + sl, -1, q) == -1;
        if (!placed) S[atomicAdd(sc_p, 1)] = q;
      }
      __syncwarp(gmask);
      sc = *reinterpret_cast<volatile int*>(sc_p);
      cur_u = ul;
    }
    uint32_t xn[P];
    ldg_rowpart<P>(R + (int64_t)(vn < 0 ? 0 : vn) * K + gl * P, xn);
    const int32_t szun = un == ul ? szu : sizes[un];
    const int32_t szvn = vn < 0 ? 0 : sizes[vn];
    int m = 0;
#pragma unroll
    for (int p = 0; p < P; ++p) {
      const int32_t q = (int32_t)x[p];
      const int4 bk = reinterpret_cast<const int4*>(T)[htab_bucket<K>(q < 0 ? 0 : q)];
      bool hit = (bk.x == q) | (bk.y == q) | (bk.z == q) | (bk.w == q);
      for (int i = 0; i < sc; ++i) hit |= S[i] == q;
      m += hit & (q >= 0);
    }
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) m += __shfl_xor_sync(0xffffffffu, m, o);
    if (valid && gl == 0) epi.edge_sized(e, szu, szv, m, min(szu, K), min(szv, K));
#pragma unroll
    for (int p = 0; p < P; ++p) x[p] = xn[p];
    __syncwarp();
    ul = un;
    vl = vn;
    szu = szun;
    szv = szvn;
  }
}

// ------------------------------------------------ merge-path group engine
// KMV rows (k = 8*G*CH sorted elements, pads sort last).  G lanes
// per edge; the 2k-element merge of the two rows is split into G equal
// diagonals.  Each lane finds its diagonal's split point with a binary
// search over the rows' shared-memory copies (merge path) and merges its
// Q = 2k/G outputs sequentially: a value stored in both rows shows up as
// two adjacent outputs (U's copy first), which counts the common elements;
// first copies of finite values are the distinct union elements, whose group
// prefix sum locates KMV's T-th distinct value (providers.py:266-301).
// One branchless merge step: emit min(ca, cb), advance that row (index
// clamped to the sentinel pad slot at K).
template <class T, int K, class SK>
__device__ __forceinline__ T merge_step(const T* su, const T* sv, int& i, int& j, T& ca, T& cb, SK sk) {
  const bool ta = ca <= cb;
  const T x = ta ? ca : cb;
  const int nxt = min((ta ? i : j) + 1, K);
  const T y = (ta ? su : sv)[sk(nxt)];
  i = ta ? nxt : i;
  j = ta ? j : nxt;
  ca = ta ? y : ca;
  cb = ta ? cb : y;
  return x;
}

template <int G, int CH, bool kKmv, class Epi>
__device__ __forceinline__ void merge_edge_loop(const void* __restrict__ rows, int k,
                                                const int32_t* __restrict__ us,
                                                const int32_t* __restrict__ vs, int64_t e_begin,
                                                int64_t e_end, unsigned char* warp_smem, Epi& epi) {
  using TL = typename std::conditional<kKmv, uint64_t, int32_t>::type;  // stored
  using T = typename std::conditional<kKmv, double, int32_t>::type;     // compared
  using TR = SortedTraits<T>;
  constexpr int K = 8 * G * CH;  // row length
  constexpr int Q = 2 * K / G;   // merged outputs per lane
  constexpr int E = 32 / G;      // edges per warp iteration
  constexpr int LOG = 32 - __builtin_clz(K);  // bisection steps over [0, K]
  const int lane = threadIdx.x & 31;
  const int gl = lane & (G - 1);
  const int gbase = lane & ~(G - 1);
  const int grp = lane / G;
  const TL* R = reinterpret_cast<const TL*>(rows);
  // bank-skewed copies: element x at x + x/8 (lane diagonals start ~8 apart
  // in each row), a sentinel pad at K, groups offset by an odd element count
  constexpr int KP = K + K / 8 + 1;
  auto sk = [](int x) { return x + (x >> 3); };
  T* su = reinterpret_cast<T*>(warp_smem) + grp * (2 * KP + 1);
  T* sv = su + KP;
  if (gl == 0) {
    su[sk(K)] = TR::pad();
    sv[sk(K)] = TR::pad();
  }
  const unsigned gmask = ((G == 32) ? 0xffffffffu : ((1u << G) - 1u)) << gbase;
  int64_t wb, we;
  warp_slice(e_begin, e_end, wb, we);
  if (wb >= we) return;
  int32_t ul = 0, vl = 0;
  if (wb + grp < we) {
    ul = us[wb + grp];
    vl = vs[wb + grp];
  }
#pragma unroll 1
  for (int64_t e0 = wb; e0 < we; e0 += E) {
    const int64_t e = e0 + grp;
    const bool valid = e < we && vl >= 0;
    int32_t un = 0, vn = 0;
    if (e + E < we) {
      un = us[e + E];
      vn = vs[e + E];
    }
    TL a[CH][8], b[CH][8];
    load_sorted_chunks<TL, CH, true>(R + (int64_t)ul * k, G, gl, a);
    load_sorted_chunks<TL, CH, false>(R + (int64_t)(vl < 0 ? 0 : vl) * k, G, gl, b);
    int la = 0, lb = 0;
#pragma unroll
    for (int s = 0; s < CH; ++s) {
      const int c = s * G + gl;
#pragma unroll
      for (int w = 0; w < 8; ++w) {
        const T ka = key_of(a[s][w]), kb = key_of(b[s][w]);
        su[c * 9 + w] = ka;
        sv[c * 9 + w] = kb;
        la += TR::valid(ka);
        lb += TR::valid(kb);
      }
    }
    la = group_sum<G>(la);
    lb = group_sum<G>(lb);
    __syncwarp();
    // merge-path split of diagonal d0 (U-first on ties), fixed-trip bisection
    const int d0 = gl * Q;
    int lo = d0 > K ? d0 - K : 0, hi = d0 < K ? d0 : K;
#pragma unroll
    for (int it = 0; it < LOG; ++it) {
      const int mid = (lo + hi) >> 1;
      const bool go = lo < hi;
      const T x = su[sk(min(mid, K))];
      const T y = sv[sk(max(d0 - 1 - mid, 0))];
      const bool right = x <= y;
      lo = (go && right) ? mid + 1 : lo;
      hi = (go && !right) ? mid : hi;
    }
    const int i0 = lo, j0 = d0 - lo;
    T prev0 = TR::pad();
    if (d0 > 0) {
      const T pu = su[sk(max(i0 - 1, 0))], pv = sv[sk(max(j0 - 1, 0))];
      prev0 = i0 == 0 ? pv : (j0 == 0 ? pu : (pu > pv ? pu : pv));
    }
    int i = i0, j = j0;
    T ca = su[sk(i)], cb = sv[sk(j)];
    T prev = prev0;
    bool has_prev = d0 > 0;
    int dups = 0, dist = 0;
    uint32_t dmask = 0;  // bit q: output q is a distinct (first-copy) union value
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const T x = merge_step<T, K>(su, sv, i, j, ca, cb, sk);
      const bool fin = TR::valid(x);
      const bool dup = fin && has_prev && x == prev;
      dups += dup;
      if constexpr (kKmv) dmask |= (uint32_t)(fin && !dup) << q;
      else dist += fin && !dup;
      prev = x;
      has_prev = true;
    }
    SortedStats st;
    st.common = group_sum<G>(dups);
    st.lu = la;
    st.lv = lb;
    st.kth = 0.0;
    if constexpr (kKmv) {
      // T-th distinct union value: the owning lane selects the t-th set bit
      // of its mask and re-splits the merge at that position (merge path)
      dist = __popc(dmask);
      const int T_ = max(min(la, lb), 1);
      const int before = group_excl_scan<G>(dist, gl);
      const int t = T_ - before;
      const bool mine = t >= 1 && t <= dist;
      int need = mine ? t : 1, pos = 0;
      uint32_t m = dmask;
#pragma unroll
      for (int w = Q / 2; w >= 1; w >>= 1) {
        const int c = __popc(m & ((1u << w) - 1u));
        const bool up = need > c;
        need = up ? need - c : need;
        pos = up ? pos + w : pos;
        m = up ? m >> w : m;
      }
      const int d = d0 + pos;
      int lo2 = d > K ? d - K : 0, hi2 = d < K ? d : K;
#pragma unroll
      for (int it = 0; it < LOG; ++it) {
        const int mid = (lo2 + hi2) >> 1;
        const bool go = lo2 < hi2;
        const T x = su[sk(min(mid, K))];
        const T y = sv[sk(max(d - 1 - mid, 0))];
        const bool right = x <= y;
        lo2 = (go && right) ? mid + 1 : lo2;
        hi2 = (go && !right) ? mid : hi2;
      }
      const T xa = su[sk(lo2)], xb = sv[sk(d - lo2)];
      const T cand = xa <= xb ? xa : xb;
      const unsigned hm = __ballot_sync(0xffffffffu, mine) & gmask;
      const uint64_t c1 = shfl64(bits_of(cand), hm ? __ffs(hm) - 1 : gbase);
      const uint64_t u0 = shfl64(bits_of(su[0]), gbase), v0 = shfl64(bits_of(sv[0]), gbase);
      st.kth = bitsd(hm ? c1 : (u0 < v0 ? u0 : v0));  // none: argmax of all-False -> merged[0]
    }
    if (valid && gl == 0) epi.edge(e, ul, vl, st);
    __syncwarp();
    ul = un;
    vl = vn;
  }
}

// Generic fallback: one lane per edge, 64-bit words (any multiple of 64 bits,
// or any k for k-Hash).
template <class Epi>
__device__ void scalar_edge_loop_bloom(const uint64_t* __restrict__ rows, int words, int op,
                                       const int32_t* __restrict__ us, const int32_t* __restrict__ vs,
                                       int64_t e_begin, int64_t e_end, Epi& epi) {
  for (int64_t e = e_begin + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < e_end;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int32_t u = us[e], v = vs[e];
    if (v < 0) continue;  // padding slot
    const uint64_t* ru = rows + (int64_t)u * words;
    const uint64_t* rv = rows + (int64_t)v * words;
    int c = 0;
    if (op == PG_BF_OR)
      for (int i = 0; i < words; ++i) c += __popcll(ru[i] | rv[i]);
    else
      for (int i = 0; i < words; ++i) c += __popcll(ru[i] & rv[i]);
    epi.edge(e, u, v, c);
  }
}
template <class Epi>
__device__ void scalar_edge_loop_khash(const int32_t* __restrict__ ent, int k, const int32_t* __restrict__ us,
                                       const int32_t* __restrict__ vs, int64_t e_begin, int64_t e_end,
                                       Epi& epi) {
  for (int64_t e = e_begin + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < e_end;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int32_t u = us[e], v = vs[e];
    if (v < 0) continue;  // padding slot
    const int32_t* a = ent + (int64_t)u * k;
    const int32_t* b = ent + (int64_t)v * k;
    int c = 0;
    for (int i = 0; i < k; ++i) c += (a[i] == b[i] && a[i] >= 0);
    epi.edge(e, u, v, c);
  }
}

// ------------------------------------------------------ estimate math ----
// All double arithmetic below uses explicit _rn intrinsics so that no FMA
// contraction can change a per-edge value relative to numpy.
__device__ __forceinline__ double bloom_estimate(int op, int c, int b, int32_t su, int32_t sv,
                                                 const double* __restrict__ lut) {
  if (op == PG_BF_AND) return lut[c];
  if (op == PG_BF_L) return __ddiv_rn((double)c, (double)b);
  const double raw = __dsub_rn((double)((int64_t)su + sv), lut[c]);
  return raw > 0.0 ? raw : 0.0;  // np.maximum(raw, 0.0)
}
// (j/(1+j)) * (s_u+s_v), j = m/k   (providers.py:223-227)
__device__ __forceinline__ double minhash_estimate(int m, int k, int32_t su, int32_t sv) {
  const double j = __ddiv_rn((double)m, (double)k);
  return __dmul_rn(__ddiv_rn(j, __dadd_rn(1.0, j)), (double)((int64_t)su + sv));
}

// ---------------------------------------------------------- epilogues ----
struct EpiBloomPairs {
  int op, b;
  const int32_t* sizes;
  const double* lut;
  int32_t* out_count;
  double* out_est;
  __device__ __forceinline__ void edge(int64_t e, int32_t u, int32_t v, int c) {
    if (out_count) out_count[e] = c;
    if (out_est) out_est[e] = bloom_estimate(op, c, b, op == PG_BF_OR ? sizes[u] : 0, op == PG_BF_OR ? sizes[v] : 0, lut);
  }
};

struct EpiBloomHist {
  int op;
  const int32_t* sizes;
  const double* lut;
  int* hist_s;
  long long sum_pos;
  __device__ __forceinline__ void edge(int64_t, int32_t u, int32_t v, int c) {
    if (op == PG_BF_OR) {
      const int64_t S = (int64_t)sizes[u] + sizes[v];
      if (__dsub_rn((double)S, lut[c]) > 0.0) {
        atomicAdd(hist_s + c, 1);
        sum_pos += S;
      }
    } else {
      atomicAdd(hist_s + c, 1);
    }
  }
};

struct EpiMinhashPairs {
  int k;
  const int32_t* sizes;
  int32_t* out_count;
  double* out_est;
  __device__ __forceinline__ void edge(int64_t e, int32_t u, int32_t v, int m) {
    if (out_count) out_count[e] = m;
    if (out_est) out_est[e] = minhash_estimate(m, k, sizes[u], sizes[v]);
  }
};

// exact 64-bit per-bin sums in shared memory from native 32-bit atomics:
// lo accumulates mod 2^32, hi counts the wrap-arounds (a CAS-free
// replacement for 64-bit shared atomics, which compile to a spin loop)
__device__ __forceinline__ void smem_add64(unsigned* lo, unsigned* hi, uint64_t x) {
  const unsigned xl = (unsigned)x;
  const unsigned old = atomicAdd(lo, xl);
  unsigned carry = (unsigned)(x >> 32) + (old > 0xFFFFFFFFu - xl ? 1u : 0u);
  if (carry) atomicAdd(hi, carry);
}

// per match count m: number of edges and sum of (s_u+s_v)
struct EpiMinhashHist {
  const int32_t* sizes;
  int* cnt_s;
  unsigned* slo_s;
  unsigned* shi_s;
  __device__ __forceinline__ void edge(int64_t, int32_t u, int32_t v, int m) {
    atomicAdd(cnt_s + m, 1);
    smem_add64(slo_s + m, shi_s + m, (uint64_t)((int64_t)sizes[u] + sizes[v]));
  }
};

// Jaccard clustering counts (config 4)
struct EpiJaccard {
  int k, min_matches;
  double tau;
  const int32_t* deg;
  int* hist_s;
  long long n_hat, n_sim;
  __device__ __forceinline__ void edge(int64_t, int32_t u, int32_t v, int m) {
    atomicAdd(hist_s + m, 1);
    n_hat += (m >= min_matches);
    // vertex_similarity(JACCARD) over the k-Hash intersection estimate
    const int32_t du = deg[u], dv = deg[v];
    const double est = minhash_estimate(m, k, du, dv);
    const double lo = (double)min(du, dv);
    const double c = fmin(fmax(est, 0.0), lo);  // _feasible_count
    const double denom = __dsub_rn((double)((int64_t)du + dv), c);
    const double J = denom > 0.0 ? __ddiv_rn(c, denom) : 0.0;
    n_sim += (J >= tau);
  }
};

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

template <int W8, class Op, int MINB, bool kVCache, int kLayout>
__global__ void __launch_bounds__(kBlock, MINB) tc_bloom_wide_kernel(const unsigned char* rows, int bits,
                                                                    const int32_t* us, const int32_t* vs,
                                                                    int64_t e_begin, int64_t e_end,
                                                                    EpiBloomHist epi, int64_t* out_hist,
                                                                    int64_t* out_sum_pos) {
  extern __shared__ int hist_s[];
  for (int i = threadIdx.x; i <= bits; i += blockDim.x) hist_s[i] = 0;
  __syncthreads();
  epi.hist_s = hist_s;
  epi.sum_pos = 0;
  wide_edge_loop<W8, Op, EpiBloomHist, kVCache, kLayout>(rows, us, vs, e_begin, e_end, epi);
  __syncthreads();
  for (int i = threadIdx.x; i <= bits; i += blockDim.x)
    if (hist_s[i]) atomicAdd(reinterpret_cast<unsigned long long*>(out_hist + i), (unsigned long long)hist_s[i]);
  if (epi.op == PG_BF_OR) {
    long long sp = epi.sum_pos;
    for (int o = 16; o > 0; o >>= 1) sp += __shfl_xor_sync(0xffffffffu, sp, o);
    if ((threadIdx.x & 31) == 0 && sp) atomicAdd(reinterpret_cast<unsigned long long*>(out_sum_pos), (unsigned long long)sp);
  }
}

template <int V, int G, bool kScalar>
__global__ void __launch_bounds__(kBlock) pairs_khash_kernel(const uint4* ent, int k, const int32_t* us,
                                                            const int32_t* vs, int64_t count,
                                                            EpiMinhashPairs epi) {
  if (kScalar) scalar_edge_loop_khash(reinterpret_cast<const int32_t*>(ent), k, us, vs, 0, count, epi);
  else group_edge_loop<V, G, OpEqPos>(ent, us, vs, 0, count, epi);
}

// kEngine: 0 scalar fallback, 1 group (128-bit) engine, 2 wide padded engine
template <int V, int G, int kEngine, int MINB = 1>
__global__ void __launch_bounds__(kBlock, MINB) tc_khash_kernel(const uint4* ent, int k, const int32_t* sizes,
                                                               const int32_t* us, const int32_t* vs,
                                                               int64_t e_begin, int64_t e_end,
                                                               int64_t* out_cnt, int64_t* out_ssum) {
  __shared__ int cnt_s[kMaxSketchK + 1];
  __shared__ unsigned slo_s[kMaxSketchK + 1], shi_s[kMaxSketchK + 1];
  for (int i = threadIdx.x; i <= k; i += blockDim.x) { cnt_s[i] = 0; slo_s[i] = 0; shi_s[i] = 0; }
  __syncthreads();
  EpiMinhashHist epi{sizes, cnt_s, slo_s, shi_s};
  if (kEngine == 0) scalar_edge_loop_khash(reinterpret_cast<const int32_t*>(ent), k, us, vs, e_begin, e_end, epi);
  else if (kEngine == 1) group_edge_loop<V, G, OpEqPos>(ent, us, vs, e_begin, e_end, epi);
  else wide_edge_loop<V, OpEqPos, EpiMinhashHist, false, true>(reinterpret_cast<const unsigned char*>(ent), us,
                                                                vs, e_begin, e_end, epi);
  __syncthreads();
  for (int i = threadIdx.x; i <= k; i += blockDim.x) {
    if (cnt_s[i]) {
      atomicAdd(reinterpret_cast<unsigned long long*>(out_cnt + i), (unsigned long long)cnt_s[i]);
      atomicAdd(reinterpret_cast<unsigned long long*>(out_ssum + i),
                ((unsigned long long)shi_s[i] << 32) + slo_s[i]);
    }
  }
}

template <int V, int G, int kEngine, int MINB = 1>
__global__ void __launch_bounds__(kBlock, MINB) jaccard_khash_kernel(const uint4* ent, int k, const int32_t* deg,
                                                                    const int32_t* us, const int32_t* vs,
                                                                    int64_t e_begin, int64_t e_end,
                                                                    int min_matches, double tau,
                                                                    int64_t* out_counts) {
  __shared__ int hist_s[kMaxSketchK + 1];
  for (int i = threadIdx.x; i <= k; i += blockDim.x) hist_s[i] = 0;
  __syncthreads();
  EpiJaccard epi{k, min_matches, tau, deg, hist_s, 0, 0};
  if (kEngine == 0) scalar_edge_loop_khash(reinterpret_cast<const int32_t*>(ent), k, us, vs, e_begin, e_end, epi);
  else if (kEngine == 1) group_edge_loop<V, G, OpEqPos>(ent, us, vs, e_begin, e_end, epi);
  else wide_edge_loop<V, OpEqPos, EpiJaccard, false, true>(reinterpret_cast<const unsigned char*>(ent), us, vs,
                                                            e_begin, e_end, epi);
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

// ------------------------------------------------------------ 1-Hash ----
// lower_bound over a shared array of `len` ascending elements
template <class T>
__device__ __forceinline__ int smem_lower_bound(const T* a, int len, T x) {
  int lo = 0, hi = len;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
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

// ----------------------------------------- sorted-engine epilogues/kernels
struct EpiOnehash {
  int k;
  const int32_t* sizes;
  int32_t* out_count;  // pairs mode
  double* out_est;
  int* cnt_s;          // fused mode
  unsigned* slo_s;
  unsigned* shi_s;
  long long verb;
  __device__ __forceinline__ void edge(int64_t e, int32_t u, int32_t v, const SortedStats& st) {
    edge_sized(e, sizes[u], sizes[v], st.common, st.lu, st.lv);
  }
  // the same with the endpoints' sizes already loaded (lengths unused)
  __device__ __forceinline__ void edge_sized(int64_t e, int32_t su, int32_t sv, int m, int, int) {
    const bool verbatim = su <= k && sv <= k;
    if (cnt_s) {
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
};

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

template <int G, int CH>
__host__ __device__ constexpr int sorted_warp_smem() {
  // V-row copies for the shared-memory chunk search (CH > 1 only)
  return CH == 1 ? 16 : (32 / G) * G * CH * 8 * 4;
}

template <int G, int CH, bool kKmv>
__host__ __device__ constexpr int merge_warp_smem() {
  // both (bank-skewed) rows of every edge of the warp's iteration
  return (32 / G) * (2 * (G * CH * 9 + 1) + 1) * (kKmv ? 8 : 4);
}

template <int K, int P, bool kFused>
__global__ void __launch_bounds__(kBlock) onehash_htab_kernel(const int32_t* ent, const int32_t* sizes,
                                                             const int32_t* us, const int32_t* vs,
                                                             int64_t e_begin, int64_t e_end, int32_t* out_count,
                                                             double* out_est, int64_t* out_cnt, int64_t* out_ssum,
                                                             int64_t* out_verbatim) {
  extern __shared__ __align__(16) int32_t htab_smem[];  // (kBlock/32) * (32/G) groups
  __shared__ int cnt_s[K + 1];
  __shared__ unsigned slo_s[K + 1], shi_s[K + 1];
  if (kFused) {
    for (int i = threadIdx.x; i <= K; i += blockDim.x) { cnt_s[i] = 0; slo_s[i] = 0; shi_s[i] = 0; }
    __syncthreads();
  }
  constexpr int kWarpInts = (32 / (K / P)) * htab_group_ints<K>();
  EpiOnehash epi{K, sizes, out_count, out_est, kFused ? cnt_s : nullptr, slo_s, shi_s, 0};
  htab_edge_loop<K, P>(ent, sizes, us, vs, e_begin, e_end, htab_smem + (threadIdx.x >> 5) * kWarpInts, epi);
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
constexpr int kC4Cap = 512;

__device__ __forceinline__ bool smem_contains(const int32_t* a, int len, int32_t x) {
  int lo = 0, hi = len;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  return lo < len && a[lo] == x;
}

template <int G>
__global__ void __launch_bounds__(kBlock) clique4_bloom_staged_kernel(
    const int64_t* __restrict__ off, const int32_t* __restrict__ adjp, const int32_t* __restrict__ src,
    int64_t e_begin, int64_t e_end, const uint64_t* __restrict__ rows, int b,
    const uint64_t* __restrict__ seeds_dev, int op, const int32_t* __restrict__ sizes,
    const double* __restrict__ lut, int64_t* out_hist, int64_t* out_sum_pos, int64_t* out_triples,
    const int64_t* __restrict__ edge_ids) {
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
    for (int base = 0; base < c3; base += M) {
      const int t = base + grp;
      const bool valid = t < c3;
      const int32_t wv = valid ? sC[t] : sC[0];
      uint32_t r[8];
      ldg256_keep(reinterpret_cast<const unsigned char*>(rows) + (int64_t)wv * (bits / 8) + 32 * gl, r);
      int cnt = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) cnt += __popc(op == PG_BF_OR ? (r[i] | sl[i]) : (r[i] & sl[i]));
#pragma unroll
      for (int o = G / 2; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
      if (valid && gl == 0) {
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
    __syncwarp();
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
      const int32_t* Wr = adjp + off[wv];
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
__global__ void __launch_bounds__(kBlock) clique4_exact_kernel(
    const int64_t* __restrict__ off, const int32_t* __restrict__ adjp, const int32_t* __restrict__ src,
    int64_t e_begin, int64_t e_end, int64_t* out_count) {
  extern __shared__ __align__(16) int32_t smem_i[];  // (kBlock/32) * (3*kC4Cap + 1)
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int32_t* sB = smem_i + w * (3 * kC4Cap + 1);
  int32_t* sC = sB + kC4Cap;
  int32_t* sP = sC + kC4Cap;  // kC4Cap + 1 entries
  long long total = 0;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t j = e_begin + (int64_t)blockIdx.x * (blockDim.x >> 5) + w; j < e_end; j += nwarps) {
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
      total += clique4_exact_edge_global(off, adjp, A, la, Bv, lb, lane);
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
      const int d = t < c3 ? (int)(off[sC[t] + 1] - off[sC[t]]) : 0;
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
      const int32_t y = adjp[off[sC[lo]] + (f - sP[lo])];
      total += smem_contains(sC, c3, y);
    }
    __syncwarp();
  }
  for (int o = 16; o > 0; o >>= 1) total += __shfl_xor_sync(0xffffffffu, total, o);
  if (lane == 0 && total) atomicAdd(reinterpret_cast<unsigned long long*>(out_count), (unsigned long long)total);
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

template <class K>
static int grid_for_kernel(K kernel, size_t smem) {
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kBlock, smem) != cudaSuccess || per_sm < 1)
    per_sm = 1;
  return sm_count() * per_sm;
}

static int grid_cap(int grid, int64_t items, int per_block) {
  const int64_t need = (items + per_block - 1) / per_block;
  return (int)std::max<int64_t>(1, std::min<int64_t>(grid, need));
}

// sorted-engine launchers; return false when k has no specialisation
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
  kern<<<grid, kBlock, sm, s>>>(ent, sizes, us, vs, b, e, out_count, out_est, out_cnt, out_ssum, out_verbatim);
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

// dispatch helpers: (W4 = row bytes / 16) -> (V, G)
#define PG_ROW_DISPATCH(W4, MACRO) \
  switch (W4) {                    \
    case 1: MACRO(1, 1); break;    \
    case 2: MACRO(1, 2); break;    \
    case 4: MACRO(1, 4); break;    \
    case 8: MACRO(1, 8); break;    \
    case 16: MACRO(2, 8); break;   \
    case 32: MACRO(4, 8); break;   \
    default: MACRO(1, 1); break;   \
  }

extern "C" int pg_group_pad(int32_t row_bytes, int32_t* pad_host);

static bool fast_w4(int w4) { return w4 == 1 || w4 == 2 || w4 == 4 || w4 == 8 || w4 == 16 || w4 == 32; }

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
                         int64_t e_end, int64_t* out_hist, int64_t* out_sum_pos, void* stream, int padded) {
  PG_REQUIRE(bits >= 64 && bits % 64 == 0, "Bloom size must be a positive multiple of 64");
  PG_REQUIRE(op == PG_BF_AND || op == PG_BF_L || op == PG_BF_OR, "op is not a Bloom estimator");
  PG_REQUIRE(0 <= e_begin && e_begin <= e_end, "bad edge range");
  PG_REQUIRE(out_hist, "null histogram");
  PG_REQUIRE(op != PG_BF_OR || out_sum_pos, "BF_OR needs the sum output");
  cudaStream_t s = as_stream(stream);
  // one memset when the sum slot directly follows the histogram
  const bool adjacent = out_sum_pos == out_hist + bits + 1;
  cudaError_t ce = cudaMemsetAsync(out_hist, 0, sizeof(int64_t) * (bits + 1 + (adjacent ? 1 : 0)), s);
  if (ce == cudaSuccess && out_sum_pos && !adjacent) ce = cudaMemsetAsync(out_sum_pos, 0, sizeof(int64_t), s);
  if (ce != cudaSuccess) return fail(PG_ERR_CUDA, "memset: %s", cudaGetErrorString(ce));
  if (e_end == e_begin) return PG_OK;  // an empty range needs no inputs
  PG_REQUIRE(op != PG_BF_OR || (sizes && lut), "BF_OR needs sizes and the table");
  PG_REQUIRE(rows && us && vs, "null pointer");
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
    // measured on B200 (scripts/sweep_tc.py, R-MAT s20/s22): B=1024 best with
    // 3 blocks/SM and streaming v rows; B=2048 best with L1-allocated v rows
    // (hub rows reused within an SM)
    static const char* vc_env = getenv("PG_TC_VCACHE");
    const bool vcache = vc_env ? vc_env[0] != '0' : (padded && w4 == 16);
    const int minb = tc_minb(w4, padded);
    const unsigned char* rb = reinterpret_cast<const unsigned char*>(rows);
    cudaError_t le = cudaSuccess;
#define PG_W(W8, MB, VC, PD)                                                                          \
  {                                                                                                  \
    auto k = op == PG_BF_OR ? tc_bloom_wide_kernel<W8, OpOr, MB, VC, PD>                             \
                            : tc_bloom_wide_kernel<W8, OpAnd, MB, VC, PD>;                           \
    le = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);            \
    if (le != cudaSuccess) return fail(PG_ERR_CUDA, "smem attribute: %s", cudaGetErrorString(le));  \
    const int grid = grid_cap(grid_for_kernel(k, smem), e_end - e_begin, kBlock);                    \
    k<<<grid, kBlock, smem, s>>>(rb, bits, us, vs, e_begin, e_end, epi, out_hist, out_sum_pos);      \
  }
#define PG_WM(W8)                                                                  \
  if (padded == 2) {                                                             \
    if (vcache) { if (minb <= 2) PG_W(W8, 2, true, 2) else PG_W(W8, 3, true, 2) } \
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

int pg_pairs_minhash(const int32_t* entries, int32_t k, int32_t onehash, const int32_t* sizes,
                     const int32_t* us, const int32_t* vs, int64_t count, int32_t* out_count,
                     double* out_est, void* stream) {
  PG_REQUIRE(k >= 1, "k must be >= 1");
  if (k > kMaxSketchK) return fail(PG_ERR_UNSUPPORTED, "k=%d exceeds the device limit %d", k, kMaxSketchK);
  PG_REQUIRE(count >= 0, "count must be >= 0");
  if (count == 0) return PG_OK;
  PG_REQUIRE(entries && us && vs, "null pointer");
  PG_REQUIRE(!out_est || sizes, "estimate needs sizes");
  cudaStream_t s = as_stream(stream);
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

int pg_tc_minhash(const int32_t* entries, int32_t k, int32_t onehash, const int32_t* sizes,
                  const int32_t* us, const int32_t* vs, int64_t e_begin, int64_t e_end, int32_t padded,
                  int64_t* out_cnt, int64_t* out_ssum, int64_t* out_verbatim, void* stream) {
  PG_REQUIRE(k >= 1, "k must be >= 1");
  if (k > kMaxSketchK) return fail(PG_ERR_UNSUPPORTED, "k=%d exceeds the device limit %d", k, kMaxSketchK);
  PG_REQUIRE(0 <= e_begin && e_begin <= e_end, "bad edge range");
  PG_REQUIRE(out_cnt && out_ssum && out_verbatim, "null pointer");
  cudaStream_t s = as_stream(stream);
  // one memset when [cnt | ssum | verbatim] is one buffer
  const bool adjacent = out_ssum == out_cnt + k + 1 && out_verbatim == out_ssum + k + 1;
  cudaError_t ce = cudaMemsetAsync(out_cnt, 0, sizeof(int64_t) * (adjacent ? 2 * k + 3 : k + 1), s);
  if (ce == cudaSuccess && !adjacent) ce = cudaMemsetAsync(out_ssum, 0, sizeof(int64_t) * (k + 1), s);
  if (ce == cudaSuccess && !adjacent) ce = cudaMemsetAsync(out_verbatim, 0, sizeof(int64_t), s);
  if (ce != cudaSuccess) return fail(PG_ERR_CUDA, "memset: %s", cudaGetErrorString(ce));
  if (e_end == e_begin) return PG_OK;  // an empty range needs no inputs
  PG_REQUIRE(entries && us && vs && sizes, "null pointer");
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
    const int grid = grid_cap(grid_for_kernel(kern, 0), e_end - e_begin, kBlock);        \
    kern<<<grid, kBlock, 0, s>>>(e4, k, sizes, us, vs, e_begin, e_end, out_cnt, out_ssum); \
  }
    if (w8 == 2) PG_KW(2, 3) else if (w8 == 4) PG_KW(4, 3) else PG_KW(8, 3)  // measured: 3 blocks beat the spill-free 2 (0.66 vs 0.72 ms, s20 k=64)
#undef PG_KW
  } else if (!fast_w4(w4)) {
    auto kern = tc_khash_kernel<1, 1, 0>;
    const int grid = grid_cap(grid_for_kernel(kern, 0), e_end - e_begin, kBlock);
    kern<<<grid, kBlock, 0, s>>>(e4, k, sizes, us, vs, e_begin, e_end, out_cnt, out_ssum);
  } else {
#define PG_L(V, G)                                                                       \
  {                                                                                      \
    auto kern = tc_khash_kernel<V, G, 1>;                                                \
    const int grid = grid_cap(grid_for_kernel(kern, 0), e_end - e_begin, kBlock);        \
    kern<<<grid, kBlock, 0, s>>>(e4, k, sizes, us, vs, e_begin, e_end, out_cnt, out_ssum); \
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
  if (k > kMaxSketchK) return fail(PG_ERR_UNSUPPORTED, "k=%d exceeds the device limit %d", k, kMaxSketchK);
  PG_REQUIRE(0 <= e_begin && e_begin <= e_end, "bad edge range");
  PG_REQUIRE(out_counts, "null pointer");
  cudaStream_t s = as_stream(stream);
  cudaError_t ce = cudaMemsetAsync(out_counts, 0, sizeof(int64_t) * (k + 3), s);
  if (ce != cudaSuccess) return fail(PG_ERR_CUDA, "memset: %s", cudaGetErrorString(ce));
  if (e_end == e_begin) return PG_OK;  // an empty range needs no inputs
  PG_REQUIRE(entries && us && vs && degrees, "null pointer");
  const int w4 = k % 4 == 0 ? k / 4 : 0;
  const uint4* e4 = reinterpret_cast<const uint4*>(entries);
  const int w8 = k % 8 == 0 ? k / 8 : 0;  // 32-byte chunks per row
  if (padded && (w8 == 2 || w8 == 4 || w8 == 8)) {
#define PG_JW(W8, MB)                                                                                  \
  {                                                                                                    \
    auto kern = jaccard_khash_kernel<W8, 1, 2, MB>;                                                    \
    const int grid = grid_cap(grid_for_kernel(kern, 0), e_end - e_begin, kBlock);                      \
    kern<<<grid, kBlock, 0, s>>>(e4, k, degrees, us, vs, e_begin, e_end, min_matches, tau, out_counts); \
  }
    if (w8 == 2) PG_JW(2, 3) else if (w8 == 4) PG_JW(4, 3) else PG_JW(8, 2)  // 256-B rows: 2 blocks (no spills)
#undef PG_JW
  } else if (!fast_w4(w4)) {
    auto kern = jaccard_khash_kernel<1, 1, 0>;
    const int grid = grid_cap(grid_for_kernel(kern, 0), e_end - e_begin, kBlock);
    kern<<<grid, kBlock, 0, s>>>(e4, k, degrees, us, vs, e_begin, e_end, min_matches, tau, out_counts);
  } else {
#define PG_L(V, G)                                                                                         \
  {                                                                                                        \
    auto kern = jaccard_khash_kernel<V, G, 1>;                                                             \
    const int grid = grid_cap(grid_for_kernel(kern, 0), e_end - e_begin, kBlock);                          \
    kern<<<grid, kBlock, 0, s>>>(e4, k, degrees, us, vs, e_begin, e_end, min_matches, tau, out_counts);    \
  }
    PG_ROW_DISPATCH(w4, PG_L)
#undef PG_L
  }
  return check_launch("jaccard_khash");
}

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

static int clique4_bloom(const int64_t* dir_off, const int32_t* dir_adj, const int32_t* src,
                         const int64_t* edge_ids, int64_t e_begin, int64_t e_end, const uint64_t* rows_plus,
                         int32_t bits, int32_t b, const uint64_t* seeds_dev, int32_t op, const int32_t* sizes,
                         const double* lut, int64_t* out_hist, int64_t* out_sum_pos, int64_t* out_triples,
                         void* stream) {
  PG_REQUIRE(bits >= 64 && bits % 64 == 0, "Bloom size must be a positive multiple of 64");
  if (bits > 16384) return fail(PG_ERR_UNSUPPORTED, "4-clique kernel supports Bloom widths up to 16384");
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
    kern<<<grid, kBlock, smem, s>>>(dir_off, dir_adj, src, e_begin, e_end, rows_plus, b, seeds_dev, op, sizes, \
                                    lut, out_hist, out_sum_pos, out_triples, edge_ids);                        \
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
  PG_REQUIRE(0 <= e_begin && e_begin <= e_end, "bad edge range");
  PG_REQUIRE(out_count, "null output");
  cudaStream_t s = as_stream(stream);
  cudaError_t ce = cudaMemsetAsync(out_count, 0, sizeof(int64_t), s);
  if (ce != cudaSuccess) return fail(PG_ERR_CUDA, "memset: %s", cudaGetErrorString(ce));
  if (e_end == e_begin) return PG_OK;
  PG_REQUIRE(dir_off && dir_adj && src, "null pointer");
  const size_t smem = sizeof(int32_t) * (kBlock / 32) * (3 * kC4Cap + 1);
  cudaFuncSetAttribute(clique4_exact_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int grid = grid_cap(grid_for_kernel(clique4_exact_kernel, smem), e_end - e_begin, kBlock / 32);
  clique4_exact_kernel<<<grid, kBlock, smem, s>>>(dir_off, dir_adj, src, e_begin, e_end, out_count);
  return check_launch("4clique_exact");
}

}  // extern "C"

extern "C" int pg_group_pad(int32_t row_bytes, int32_t* pad_host) {
  PG_REQUIRE(pad_host, "null output");
  PG_REQUIRE(row_bytes > 0, "row_bytes must be positive");
  const int w8 = row_bytes % 32 == 0 ? row_bytes / 32 : 0;
  *pad_host = (w8 == 2 || w8 == 4 || w8 == 8) ? w8 : 1;
  return PG_OK;
}
