#pragma once
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
//
// This header holds the shared device engines, row ops and epilogues; the
// kernels and C entry points live in pg_bloom.cu (Bloom pairs / TC),
// pg_minhash.cu (k-Hash / 1-Hash pairs, TC, Jaccard), pg_kmv.cu and
// pg_clique.cu (4-clique).
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
// Integer adds steered onto the FMA pipe: a * kImadW[i] + b with the
// multiplier read from constant memory is an IMAD (FMA pipe) rather than an
// IADD3 / LEA (ALU pipe).  The Bloom kernels at 2048 bits are ALU-bound
// (LOP3 for AND and the carry-save adders), the FMA pipe idles.
#ifndef PG_IMAD_ADDS
#define PG_IMAD_ADDS 1
#endif
#ifndef PG_WIDE_SUB
#define PG_WIDE_SUB 8  // v rows in flight per sub-step of the padded wide engine
#endif
static __constant__ int kImadW[4] = {1, 2, 4, 8};
static __constant__ int kImadHi = 65536;  // packs a second 16-bit count into a register on the FMA pipe
#ifndef PG_WIDE_PACK
#define PG_WIDE_PACK 1  // packed transpose-reduce in the 8-lane wide engine
#endif
#ifndef PG_WIDE_CLAMP1
#define PG_WIDE_CLAMP1 1  // pad slots (v < 0) clamped once by the loading lane
#endif
__device__ __forceinline__ int imad(int a, int b, int c) { return a * b + c; }

// Harley-Seal variants: the 8 words a lane holds per edge pass through four
// carry-save adders (LOP3s, ALU pipe) so 4 POPC replace 8 -- POPC issues on
// the XU pipe (16/clk/SM), the ceiling of the 2048-bit rows once the row
// stream is cached.  Same counts.
__device__ __forceinline__ void csa3(uint32_t& carry, uint32_t& s, uint32_t a, uint32_t b, uint32_t c) {
  const uint32_t u = a ^ b;
  carry = (a & b) | (u & c);
  s = u ^ c;
}
#ifndef PG_CSA_LEVEL
#define PG_CSA_LEVEL 4
#endif
__device__ __forceinline__ int popc8_csa(const uint32_t (&x)[8]) {
  uint32_t s1, c1, s2, c2, s3, c3, s4, c4;
  csa3(c1, s1, x[0], x[1], x[2]);
  csa3(c2, s2, x[3], x[4], x[5]);
  csa3(c3, s3, s1, s2, x[6]);
#if PG_CSA_LEVEL == 3
  // three adders, five POPC: one LOP3 pair fewer per 8 words, one POPC more
  return imad(__popc(c1) + __popc(c2) + __popc(c3), kImadW[1], imad(__popc(s3), kImadW[0], __popc(x[7])));
#endif
  csa3(c4, s4, c1, c2, c3);
#if PG_IMAD_ADDS
  // ones + 2*twos + 4*fours as two IMADs on the FMA pipe (the multipliers
  // come from constant memory, so ptxas cannot turn them into ALU LEAs):
  // the ALU pipe is the 2048-bit kernel's binding resource
  return imad(__popc(c4), kImadW[2], imad(__popc(s4), kImadW[1], imad(__popc(s3), kImadW[0], __popc(x[7]))));
#else
  return __popc(s3) + __popc(x[7]) + 2 * __popc(s4) + 4 * __popc(c4);  // ones, twos, fours
#endif
}
struct OpAndCsa : OpAnd {
  __device__ __forceinline__ static int apply8(const uint32_t (&a)[8], const uint32_t (&b)[8]) {
    uint32_t x[8];
#pragma unroll
    for (int w = 0; w < 8; ++w) x[w] = a[w] & b[w];
    return popc8_csa(x);
  }
};
struct OpOrCsa : OpOr {
  __device__ __forceinline__ static int apply8(const uint32_t (&a)[8], const uint32_t (&b)[8]) {
    uint32_t x[8];
#pragma unroll
    for (int w = 0; w < 8; ++w) x[w] = a[w] | b[w];
    return popc8_csa(x);
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
#if PG_IMAD_ADDS
      c[j] = imad(__shfl_xor_sync(0xffffffffu, send, w), kImadW[0], keep);
#else
      c[j] = keep + __shfl_xor_sync(0xffffffffu, send, w);
#endif
    }
  }
  return c[0];
}

// The same for G = 8 with two 16-bit counts per register (p[i] = c[2i] |
// c[2i+1] << 16; each count <= 2048): the w = 4 and w = 2 rounds move half the
// registers (6 SEL + 3 SHFL instead of 12 + 6), the last round adds the
// shuffled pair and picks the lane's half.  ALU-pipe diet for the 2048-bit
// Bloom kernel.
__device__ __forceinline__ int group_transpose_reduce_packed8(uint32_t (&p)[4], int gl) {
  {
    const bool upper = (gl & 4) != 0;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const uint32_t send = upper ? p[j] : p[j + 2];
      const uint32_t keep = upper ? p[j + 2] : p[j];
      p[j] = (uint32_t)imad((int)__shfl_xor_sync(0xffffffffu, send, 4), kImadW[0], (int)keep);
    }
  }
  {
    const bool upper = (gl & 2) != 0;
    const uint32_t send = upper ? p[0] : p[1];
    const uint32_t keep = upper ? p[1] : p[0];
    p[0] = (uint32_t)imad((int)__shfl_xor_sync(0xffffffffu, send, 2), kImadW[0], (int)keep);
  }
  const uint32_t t = (uint32_t)imad((int)__shfl_xor_sync(0xffffffffu, p[0], 1), kImadW[0], (int)p[0]);
  return (gl & 1) ? (int)(t >> 16) : (int)(t & 0xffffu);
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

// Dynamic edge chunks: a warp takes the next `chunk`-edge range of
// [e_begin, e_end) from a per-launch global counter (zeroed by the launcher).
// Per-edge cost varies (row lengths, u-run rebuilds), and a static split
// left warps idle at the block's final barrier.
__device__ __forceinline__ bool next_chunk(unsigned long long* ctr, int64_t e_begin, int64_t e_end,
                                           int64_t chunk, int64_t& wb, int64_t& we) {
  unsigned long long c = 0;
  if ((threadIdx.x & 31) == 0) c = atomicAdd(ctr, 1ull);
  c = __shfl_sync(0xffffffffu, c, 0);
  wb = e_begin + (int64_t)c * chunk;
  if (wb >= e_end) return false;
  we = min(wb + chunk, e_end);
  return true;
}

// edge sets from which the fixed-row engines take dynamic chunks
constexpr int64_t kDynamicMinSlots = int64_t(1) << 25;

// host: one zeroed 64-bit chunk counter per launch (stream-ordered scratch)
struct ChunkCounter {
  unsigned long long* p = nullptr;
  cudaStream_t s = nullptr;
  cudaError_t init(cudaStream_t st) {
    s = st;
    retain_default_pool();
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&p), sizeof(unsigned long long), s);
    if (e == cudaSuccess) e = cudaMemsetAsync(p, 0, sizeof(unsigned long long), s);
    return e;
  }
  ~ChunkCounter() {
    if (p) cudaFreeAsync(p, s);
  }
};

// Reproducible fp64 sums: kernels write partial sums to fixed slots (one
// per block of a fixed grid, or one per dynamic edge chunk), and
// fixed_order_sum_kernel adds them in index order (a strided pass per thread,
// then a fixed tree), so a sum does not depend on scheduling or atomics.
__global__ void fixed_order_sum_kernel(const double* __restrict__ part, int64_t n, double* out);

struct PartialSums {
  double* p = nullptr;
  int64_t n = 0;
  cudaStream_t s = nullptr;
  cudaError_t init(cudaStream_t st, int64_t count) {
    s = st;
    n = count;
    retain_default_pool();
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&p), sizeof(double) * (count > 0 ? count : 1), s);
    if (e == cudaSuccess) e = cudaMemsetAsync(p, 0, sizeof(double) * (count > 0 ? count : 1), s);
    return e;
  }
  void finish(double* out) { fixed_order_sum_kernel<<<1, 256, 0, s>>>(p, n, out); }
  ~PartialSums() {
    if (p) cudaFreeAsync(p, s);
  }
};

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

// base + r * bytes as one mad.wide.u32 (IMAD.WIDE.U32, FMA pipe); written in
// PTX so the compiler cannot re-split it into multiply + OR + 64-bit add on
// the ALU pipe
// Row sizes in constant memory: a multiplier ptxas cannot see keeps the
// product on IMAD.WIDE (a known power of two becomes LEA + LEA.HI.X, ALU).
static __constant__ uint32_t kRowBytesC[17] = {0, 32, 64, 96, 128, 160, 192, 224, 256,
                                               288, 320, 352, 384, 416, 448, 480, 512};
__device__ __forceinline__ const unsigned char* row_addr(const unsigned char* base, uint32_t r, uint32_t bytes) {
  uint64_t out;

  asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(out) : "r"(r), "r"(bytes), "l"(base));
  return reinterpret_cast<const unsigned char*>(out);
}

// kLayout: 0 any edge list; 1 row-padded slots (every aligned group of G
// slots shares one u; us[] per slot); 2 the same with us[] holding one u per
// group (us[e / G]) -- a G-fold smaller u stream.
template <int W8, class Op, class Epi, bool kVCache = false, int kLayout = 0, bool kDyn = false>
__device__ __forceinline__ void wide_edge_loop(const unsigned char* __restrict__ rows,
                                               const int32_t* __restrict__ us, const int32_t* __restrict__ vs,
                                               int64_t e_begin, int64_t e_end, Epi& epi,
                                               unsigned long long* ctr = nullptr) {
  constexpr bool kPadded = kLayout > 0;
  constexpr int G = W8 < 8 ? W8 : 8;  // lanes per edge
  constexpr int V = W8 / G;           // 32-byte chunks per lane per row
  constexpr int64_t kRowBytes = W8 * 32;
  const int lane = threadIdx.x & 31;
  const int gl = lane & (G - 1);
  const int gbase = lane & ~(G - 1);
  const unsigned char* rows_gl = rows + gl * 32;
  int32_t ucur = -1;
  uint32_t ur[V][8];
#pragma unroll
  for (int i = 0; i < V; ++i)
#pragma unroll
    for (int w = 0; w < 8; ++w) ur[i][w] = 0;
  const uint32_t row_bytes_r = kRowBytesC[W8];
  // ranges: dynamic 512-slot chunks (kDyn: the launcher passes a counter),
  // else one static per-warp slice (the cached u row survives chunk ends)
  int64_t wb, we;
  bool first = true;
  for (;;) {
  if (kDyn) {
    if (!next_chunk(ctr, e_begin, e_end, 512, wb, we)) return;
  } else {
    if (!first) return;
    warp_slice(e_begin, e_end, wb, we);
    if (wb >= we) return;
  }
  first = false;
  // 32-bit slot indices relative to the range start (wb is a multiple of G
  // for the padded layouts), so the index arithmetic of the prefetch is one
  // shift and two IMAD.WIDE instead of 64-bit divides and adds
  const int32_t* __restrict__ usb = kLayout == 2 ? us + wb / G : us + wb;
  const int32_t* __restrict__ vsb = vs + wb;
  int32_t ul = 0, vl = 0;
  if (wb + lane < we) {
    ul = kLayout == 2 ? usb[(unsigned)lane / G] : usb[lane];
    vl = vsb[lane];
  }
  // 32-bit remaining-slot count instead of 64-bit bound checks (registers)
  const int nslots = (int)(we - wb);
#pragma unroll 1
  for (int r0 = 0; r0 < nslots; r0 += 32) {
    const unsigned i = (unsigned)(r0 + lane);
    const int64_t e = wb + i;
    const int rem = nslots - r0;
    const bool valid = lane < rem && vl >= 0;  // v < 0: padding slot
    int32_t un = 0, vn = 0;
    if (lane + 32 < rem) {
      un = kLayout == 2 ? usb[(i + 32) / G] : usb[i + 32];
      vn = vsb[i + 32];
    }
    // rows in flight per sub-step: all G (default), or kSub at a time so
    // fewer registers hold rows (more CTAs per SM)
    constexpr int kSub = (kPadded && PG_WIDE_SUB < G) ? PG_WIDE_SUB : G;
    constexpr bool kPack = PG_WIDE_PACK && kPadded && G == 8 && V == 1 && kSub == G;
    int c[G];
    uint32_t cp[4];
#if PG_WIDE_CLAMP1
    const int32_t vls = vl < 0 ? 0 : vl;
#endif
#pragma unroll
    for (int j0 = 0; j0 < G; j0 += kSub) {
    uint32_t vr[kSub][V][8];
#pragma unroll
    for (int jj = 0; jj < kSub; ++jj) {
      const int j = j0 + jj;
#if PG_WIDE_CLAMP1
      // pad slots were clamped to row 0 by the loading lane (vls)
      const uint32_t vrow = (uint32_t)__shfl_sync(0xffffffffu, vls, j, G);
#else
      const int32_t vj = __shfl_sync(0xffffffffu, vl, j, G);
      const uint32_t vrow = (uint32_t)(vj < 0 ? 0 : vj);
#endif
      // lane base + row * bytes: one IMAD.WIDE.U32 (FMA pipe) per row
      // instead of multiply, OR and a 64-bit add on the ALU pipe
      const unsigned char* rv = row_addr(rows_gl, vrow, row_bytes_r);
#pragma unroll
      for (int i = 0; i < V; ++i) {
        if (kVCache) ldg256_keep(rv + i * G * 32, vr[jj][i]);
        else ldg256(rv + i * G * 32, vr[jj][i]);
      }
    }
    // u rows: with the row-padded edge layout (pg_csr_upper_edges_padded)
    // all G edges of a group share one u, cached across iterations; for any
    // other input the per-edge rows are loaded speculatively in parallel.
    const int32_t u0 = __shfl_sync(0xffffffffu, ul, 0, G);
    bool uniform = true;
    if (!kPadded) {
#pragma unroll
      for (int j = 1; j < G; ++j) uniform &= __shfl_sync(0xffffffffu, ul, j, G) == u0;
    }
    if (kPadded || __all_sync(0xffffffffu, uniform)) {
      if (u0 != ucur) {
        ucur = u0;
        const unsigned char* ru = row_addr(rows_gl, (uint32_t)u0, row_bytes_r);
#pragma unroll
        for (int i = 0; i < V; ++i) ldg256_keep(ru + i * G * 32, ur[i]);
      }
#pragma unroll
      for (int jj = 0; jj < kSub; ++jj) {
        int acc = 0;
#pragma unroll
        for (int i = 0; i < V; ++i) acc += Op::apply8(ur[i], vr[jj][i]);
        if (kPack) {
          // two 16-bit counts per register: the odd edge joins on the FMA pipe
          if (jj & 1) cp[jj >> 1] = (uint32_t)imad(acc, kImadHi, (int)cp[jj >> 1]);
          else cp[jj >> 1] = (uint32_t)acc;
        } else {
          c[j0 + jj] = acc;
        }
      }
    } else if (!kPadded) {
#pragma unroll
      for (int j = 0; j < G; ++j) {
        const int32_t uj = __shfl_sync(0xffffffffu, ul, j, G);
        if (uj != ucur) {
          ucur = uj;
          const unsigned char* ru = row_addr(rows_gl, (uint32_t)uj, row_bytes_r);
#pragma unroll
          for (int i = 0; i < V; ++i) ldg256_keep(ru + i * G * 32, ur[i]);
        }
        int acc = 0;
#pragma unroll
        for (int i = 0; i < V; ++i) acc += Op::apply8(ur[i], vr[j][i]);
        c[j] = acc;
      }
    }
    }  // sub-steps
    int cnt;
    if constexpr (kPack) cnt = group_transpose_reduce_packed8(cp, gl);
    else cnt = group_transpose_reduce<G>(c, gl);
    if (valid) epi.edge(e, ul, vl, cnt);
    ul = un;
    vl = vn;
  }
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
                                               int64_t e_begin, int64_t e_end, unsigned long long* ctr,
                                               int32_t* warp_smem, Epi& epi) {
  constexpr int G = K / P, E = 32 / G;
  constexpr int64_t kChunk = 64 * E;
  const int lane = threadIdx.x & 31, gl = lane & (G - 1), grp = lane / G;
  const unsigned gmask = ((G == 32) ? 0xffffffffu : ((1u << G) - 1u)) << (grp * G);
  int32_t* T = warp_smem + grp * htab_group_ints<K>();  // 4K slots
  int32_t* S = T + 4 * K;                                 // stash (K)
  int* sc_p = reinterpret_cast<int*>(S + K);
  int32_t cur_u = -1;  // the group's table survives chunk boundaries
  int sc = 0;
  int64_t wb, we;
  while (next_chunk(ctr, e_begin, e_end, kChunk, wb, we)) {
    int32_t ul = 0, vl = -1, szu = 0, szv = 0;
    if (wb + grp < we) {
      ul = us[wb + grp];
      vl = vs[wb + grp];
      szu = sizes[ul];
      szv = vl < 0 ? 0 : sizes[vl];
    }
    uint32_t x[P];
    ldg_rowpart<P>(R + (int64_t)(vl < 0 ? 0 : vl) * K + gl * P, x);
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
        if (q >= 0) {  // pads (-1) cost no shared-memory wavefront
          const int4 bk = reinterpret_cast<const int4*>(T)[htab_bucket<K>(q)];
          bool hit = (bk.x == q) | (bk.y == q) | (bk.z == q) | (bk.w == q);
          for (int i = 0; i < sc; ++i) hit |= S[i] == q;
          m += hit;
        }
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

template <class K>
inline int grid_for_kernel(K kernel, size_t smem) {
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kBlock, smem) != cudaSuccess || per_sm < 1)
    per_sm = 1;
  return sm_count() * per_sm;
}

inline int grid_cap(int grid, int64_t items, int per_block) {
  const int64_t need = (items + per_block - 1) / per_block;
  return (int)std::max<int64_t>(1, std::min<int64_t>(grid, need));
}

}  // namespace pg

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

inline bool fast_w4(int w4) { return w4 == 1 || w4 == 2 || w4 == 4 || w4 == 8 || w4 == 16 || w4 == 32; }
