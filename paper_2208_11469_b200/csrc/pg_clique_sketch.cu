// 4-clique counting with MinHash / KMV providers (mining.py:133-154
// four_clique_count driving MinHashProvider.with_set / KmvProvider.with_set,
// providers.py:234-241 and :303-307).
//
// For every directed edge (u, v) the reference materialises C3 = N+u & N+v,
// then for every w in C3 builds the member sketch of C3 (build_khash /
// build_onehash / build_kmv, sketches.py:201-237) and estimates |S_w & C3|
// with est_intersection_minhash / est_intersection_kmv (estimators.py:
// 157-200).  The member sketch depends only on (u, v), so here one warp per
// directed edge builds it once in shared memory and its lanes then evaluate
// the members w in parallel, one member per lane:
//   k-Hash : mem[i] = argmin_{x in C3} h_i(x).  h_i is a bijection of x
//            (mix64 of seed_i ^ x), so ties never happen and the argmin is
//            unmix64(min h_i) ^ seed_i.  Estimate from positional matches
//            with w's entry row (an empty sketch when |S_w| = 0).
//   1-Hash : the min(k, |C3|) members of smallest h_0 (distinct keys: h_0 is
//            a bijection), found as the threshold thr = the k-th smallest
//            h_0 by rank counting; |entries_w & mem| counts w's stored IDs
//            that are in C3 (binary search) with h_0 <= thr.
//   KMV    : the min(k, distinct) smallest distinct unit values of C3,
//            placed by distinct rank; w's stored values are merged with them
//            for the union / k_eff-th union value / common count.
// Per-triple estimates are summed in fp64 per lane; the sum is reduced in a
// fixed order (lanes by xor tree, warps then blocks by index) and the edge
// schedule is static, so the result is reproducible run to run.  Edges whose
// shorter out-list exceeds kC4Cap keep C3 (and its keys) in a per-warp
// global scratch sized by the caller (pg_4clique_sketch_workspace_size).
#include <cstdlib>
#include <type_traits>

#include "pg_engines.cuh"

namespace pg {

constexpr int kCSCap = 256;  // C3 entries held in shared memory per warp
constexpr int kCSBlock = 256;
#ifndef PG_C4S_CHUNK
#define PG_C4S_CHUNK 8
#endif
constexpr int64_t kC4SChunk = PG_C4S_CHUNK;  // directed edges per dynamic chunk

__device__ __forceinline__ bool contains_sorted(const int32_t* a, int len, int32_t x) {
  int lo = 0, hi = len;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  return lo < len && a[lo] == x;
}
__device__ __forceinline__ bool contains_sorted64(const int32_t* a, int64_t len, int32_t x) {
  int64_t lo = 0, hi = len;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (a[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  return lo < len && a[lo] == x;
}

// slot of a KMV value (IEEE bits of a unit value) in a 2^tb-slot table
__device__ __forceinline__ uint32_t kmv_slot(uint64_t x, int tb) {
  return ((uint32_t)(x ^ (x >> 29)) * 0x9E3779B1u) >> (32 - tb);
}

// (j / (1 + j)) * S with j = m / d, the reference's order of operations
__device__ __forceinline__ double jaccard_scaled(double j, int64_t S) {
  return __dmul_rn(__ddiv_rn(j, __dadd_rn(1.0, j)), (double)S);
}

struct C4SketchArgs {
  const int32_t* ent;     // k-Hash / 1-Hash entry rows (int32[n][k])
  const double* vals;     // KMV value rows (double[n][k])
  const int32_t* lengths; // 1-Hash / KMV stored lengths
  const int32_t* sizes;   // |S_w| (degrees of the sketched source)
  const uint64_t* seeds;  // k (k-Hash) or 1 seeds
  int k;
  // k > kMaxSketchK: the member sketch and the 1-Hash member table live in
  // per-warp global scratch (gM: k values, gT: tcap slots); else nullptr
  uint64_t* gM;
  int32_t* gT;
  int tcap;
};

// kBig (k > kMaxSketchK): member sketch and 1-Hash table in the global
// scratch of C4SketchArgs; resolved at compile time so the common case keeps
// shared-memory (LDS) addressing
template <int KIND, bool kBig>
__global__ void __launch_bounds__(kCSBlock, 3) clique4_sketch_kernel(
    const int64_t* __restrict__ off, const int32_t* __restrict__ adjp, const int32_t* __restrict__ src,
    const int64_t* __restrict__ edge_ids, int64_t e_begin, int64_t e_end, C4SketchArgs a,
    int32_t* __restrict__ gC, int32_t* __restrict__ gF, uint64_t* __restrict__ gH, int64_t scratch_per_warp,
    int cap, double* __restrict__ part, unsigned long long* __restrict__ out_triples,
    unsigned long long* __restrict__ ctr) {
  constexpr int kWarps = kCSBlock / 32;
  // dynamic shared memory (c4s_smem): per warp the staged longer list /
  // repeat flags, C3, its keys and the member sketch; then the seeds
  extern __shared__ __align__(16) unsigned char smem_cs[];
  uint64_t* sH_all = reinterpret_cast<uint64_t*>(smem_cs);         // [kWarps][kCSCap]
  uint64_t* sM_all = sH_all + kWarps * kCSCap;                      // [kWarps][kMaxSketchK]
  uint64_t* seeds_s = sM_all + kWarps * kMaxSketchK;                // [kMaxSketchK]
  int32_t* sB_all = reinterpret_cast<int32_t*>(seeds_s + kMaxSketchK);  // [kWarps][kCSCap]
  int32_t* sC_all = sB_all + kWarps * kCSCap;                       // [kWarps][kCSCap]
  __shared__ uint64_t thr_s[kWarps];
  const int k = a.k;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nseeds = KIND == PG_KHASH ? min(k, kMaxSketchK) : 1;
  for (int i = threadIdx.x; i < nseeds; i += blockDim.x) seeds_s[i] = a.seeds[i];
  __syncthreads();
  int32_t* sB = sB_all + wid * kCSCap;
  const int64_t gw = (int64_t)blockIdx.x * kWarps + wid;
  int32_t* gCw = gC + gw * scratch_per_warp;
  int32_t* gFw = gF + gw * scratch_per_warp;
  uint64_t* gHw = gH + gw * scratch_per_warp;
  long long triples = 0;
  // directed edges in dynamic chunks of kC4SChunk per warp (per-edge work
  // spans orders of magnitude); one fp64 partial per chunk, summed in chunk
  // order afterwards, so the total does not depend on which warp ran what
  int64_t wb = 0, we = 0;
  while (next_chunk(ctr, e_begin, e_end, kC4SChunk, wb, we)) {
  double acc = 0.0;
  for (int64_t j = wb; j < we; ++j) {
    const int64_t jj = edge_ids ? edge_ids[j] : j;
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
    // C3 and its keys in the warp's shared arrays (kS) or its global
    // scratch; a compile-time choice keeps shared-memory addressing
    auto edge = [&](auto small_tag) {
      constexpr bool kS = decltype(small_tag)::value;
      int32_t* C = kS ? sC_all + wid * kCSCap : gCw;
      uint64_t* H = kS ? sH_all + wid * kCSCap : gHw;
      int32_t* F = kS ? sB : gFw;  // KMV repeat flags (sB is free once C3 is built)
      const bool staged = lb <= cap;
      if (staged) {
        for (int i = lane; i < lb; i += 32) sB[i] = Bv[i];
        __syncwarp();
      }
      int c3 = 0;
      for (int64_t base = 0; base < la; base += 32) {
        const int64_t idx = base + lane;
        const int32_t x = idx < la ? A[idx] : -1;
        const bool hit = idx < la && (staged ? contains_sorted(sB, (int)lb, x) : contains_sorted64(Bv, lb, x));
        const unsigned mask = __ballot_sync(0xffffffffu, hit);
        if (hit) C[c3 + __popc(mask & ((1u << lane) - 1u))] = x;
        c3 += __popc(mask);
      }
      __syncwarp();
      if (c3 == 0) return;
      triples += c3;
      uint64_t* M = kBig ? a.gM + gw * k : sM_all + wid * kMaxSketchK;
      const uint64_t s0 = seeds_s[0];
      int lm = 0;          // KMV: stored member values
      int ktb = 0;         // KMV: log2 of the member-set table size (0: none)
      uint64_t thr = ~0ull;  // 1-Hash: largest selected h_0
      int tb = 5;          // 1-Hash: log2 of the member-set table size
      if (KIND == PG_KHASH) {
        for (int i = lane; i < k; i += 32) {
          const uint64_t s = (!kBig || i < kMaxSketchK) ? seeds_s[i] : a.seeds[i];
          uint64_t mn = ~0ull;
          for (int t = 0; t < c3; ++t) {
            const uint64_t h = hash_word(s, C[t]);
            mn = h < mn ? h : mn;
          }
          M[i] = (uint64_t)(uint32_t)(unmix64(mn) ^ s);  // the argmin's ID (low 32 bits)
        }
      } else {
        for (int t = lane; t < c3; t += 32) {
          const uint64_t h = hash_word(s0, C[t]);
          H[t] = KIND == PG_KMV ? dbits(unit_value(h)) : h;
        }
        __syncwarp();
        if (KIND == PG_ONEHASH) {
          if (c3 > k) {  // thr = the k-th smallest key (keys are distinct)
            for (int t = lane; t < c3; t += 32) {
              const uint64_t x = H[t];
              int r = 0;
              for (int q = 0; q < c3; ++q) r += H[q] < x;
              if (r == k - 1) thr_s[wid] = x;
            }
            __syncwarp();
            thr = thr_s[wid];
          }
          // the selected members in an open-addressing set (T = 2^tb >= 2 *
          // selected slots, linear probing, -1 empty) over the warp's key
          // array, which is free once thr is known (in the global-scratch
          // case the keys live in gH and the shared region is unused)
          const int sel = c3 < k ? c3 : k;
          tb = 5;
          while ((1 << tb) < 2 * sel) ++tb;
          int32_t* tab = kBig ? a.gT + gw * a.tcap : reinterpret_cast<int32_t*>(sH_all + wid * kCSCap);
          for (int i = lane; i < (1 << tb); i += 32) tab[i] = -1;
          __syncwarp();
          for (int t = lane; t < c3; t += 32) {
            const int32_t x = C[t];
            if (thr != ~0ull && hash_word(s0, x) > thr) continue;
            uint32_t h = ((uint32_t)x * 0x9E3779B1u) >> (32 - tb);
            while (atomicCAS(tab + h, -1, x) != -1) h = (h + 1) & ((1u << tb) - 1);
          }
          __syncwarp();
        } else {
          // KMV: units are positive doubles, so their bits order like the
          // values; mark repeats (a smaller index holds the same value) with
          // the sign bit, then place every first copy at its distinct rank
          for (int t = lane; t < c3; t += 32) {
            const uint64_t x = H[t];
            bool dup = false;
            for (int q = 0; q < t; ++q) dup |= H[q] == x;
            F[t] = dup;
          }
          __syncwarp();
          for (int t = lane; t < c3; t += 32)
            if (F[t]) H[t] |= 1ull << 63;
          __syncwarp();
          int nd = 0;
          for (int t = lane; t < c3; t += 32) {
            const uint64_t x = H[t];
            if (x >> 63) continue;
            ++nd;
            int r = 0;
            for (int q = 0; q < c3; ++q) r += H[q] < x;  // flagged repeats compare larger
            if (r < k) M[r] = x;
          }
          nd = __reduce_add_sync(0xffffffffu, nd);
          lm = nd < k ? nd : k;
          // M as an open-addressing set over the (now free) key array: when
          // only |W & M| is needed (both sets within capacity, or k_eff < 2)
          // each member's lw values are independent probes instead of a
          // serial merge
          if (!kBig && 2 * lm <= kCSCap) {
            __syncwarp();
            ktb = 5;
            while ((1 << ktb) < 2 * lm) ++ktb;
            unsigned long long* kt = reinterpret_cast<unsigned long long*>(sH_all + wid * kCSCap);
            for (int i = lane; i < (1 << ktb); i += 32) kt[i] = ~0ull;
            __syncwarp();
            for (int i = lane; i < lm; i += 32) {
              const uint64_t x = M[i];
              uint32_t h = kmv_slot(x, ktb);
              while (atomicCAS(kt + h, ~0ull, (unsigned long long)x) != ~0ull) h = (h + 1) & ((1u << ktb) - 1);
            }
          }
        }
      }
      __syncwarp();
      // every member w of C3, one lane each
      for (int t = lane; t < c3; t += 32) {
        const int32_t w = C[t];
        const int64_t sw = a.sizes[w];
        double est;
        if (KIND == PG_KHASH) {
          if (sw == 0) {
            est = 0.0;
          } else {
            int m = 0;
            const int k4 = (k & 3) == 0 ? k / 4 : 0;  // 16-byte rows only when k % 4 == 0
            const int4* row = reinterpret_cast<const int4*>(a.ent + (int64_t)w * k);
            for (int i = 0; i < k4; ++i) {
              const int4 r = __ldg(row + i);
              m += (r.x == (int32_t)M[4 * i]) + (r.y == (int32_t)M[4 * i + 1]) + (r.z == (int32_t)M[4 * i + 2]) +
                   (r.w == (int32_t)M[4 * i + 3]);
            }
            for (int i = 4 * k4; i < k; ++i) m += __ldg(a.ent + (int64_t)w * k + i) == (int32_t)M[i];
            est = jaccard_scaled(__ddiv_rn((double)m, (double)k), sw + c3);
          }
        } else if (KIND == PG_ONEHASH) {
          const int lw = a.lengths[w];
          const int32_t* row = a.ent + (int64_t)w * k;
          const int32_t* tab = kBig ? a.gT + gw * a.tcap : reinterpret_cast<const int32_t*>(sH_all + wid * kCSCap);
          const uint32_t tmask = (1u << tb) - 1;
          int common = 0;
          // 8 entries per 32-byte load (rows of k % 8 == 0 are 32-byte
          // aligned); the 8 probes are independent
          for (int base = 0; base < lw; base += 8) {
            uint32_t y8[8];
            if ((k & 7) == 0) {
              ldg256_keep(row + base, y8);
            } else {
#pragma unroll
              for (int t = 0; t < 8; ++t) y8[t] = base + t < lw ? (uint32_t)__ldg(row + base + t) : 0u;
            }
#pragma unroll
            for (int t = 0; t < 8; ++t) {
              if (base + t >= lw) break;
              const int32_t y = (int32_t)y8[t];
              uint32_t h = (y8[t] * 0x9E3779B1u) >> (32 - tb);
              int32_t c;
              // (global table: read through L2, where the atomicCAS claims landed)
              while ((c = kBig ? __ldcg(tab + h) : tab[h]) != y && c != -1) h = (h + 1) & tmask;
              common += c == y;
            }
          }
          if (sw <= k && c3 <= k) {
            est = (double)common;
          } else {
            const int ly = c3 < k ? c3 : k;
            int denom = lw + ly - common;
            denom = denom < k ? denom : k;
            const double jj2 = denom ? __ddiv_rn((double)common, (double)denom) : 0.0;
            est = jaccard_scaled(jj2, sw + c3);
          }
        } else {  // KMV
          const int lw = a.lengths[w];
          const uint64_t* W = reinterpret_cast<const uint64_t*>(a.vals) + (int64_t)w * k;
          const bool both_small = sw <= k && c3 <= k;
          const int k_eff = lw < lm ? lw : lm;
          const bool full = both_small || k_eff < 2;
          int i = 0, q = 0, cnt = 0, inter = 0;
          uint64_t kth = 0;
          if (full && ktb) {  // |W & M| by probes; the merge below is skipped
            const unsigned long long* kt = reinterpret_cast<const unsigned long long*>(sH_all + wid * kCSCap);
            const uint32_t km = (1u << ktb) - 1;
            for (int b = 0; b < lw; b += 4) {
              uint64_t x4[4];
              if ((k & 3) == 0) {
                uint32_t r8[8];
                ldg256_keep(W + b, r8);
#pragma unroll
                for (int t2 = 0; t2 < 4; ++t2) x4[t2] = ((uint64_t)r8[2 * t2 + 1] << 32) | r8[2 * t2];
              } else {
#pragma unroll
                for (int t2 = 0; t2 < 4; ++t2) x4[t2] = b + t2 < lw ? __ldg(W + b + t2) : ~0ull;
              }
#pragma unroll
              for (int t2 = 0; t2 < 4; ++t2) {
                if (b + t2 >= lw) break;
                uint32_t h = kmv_slot(x4[t2], ktb);
                uint64_t c;
                while ((c = kt[h]) != x4[t2] && c != ~0ull) h = (h + 1) & km;
                inter += c == x4[t2];
              }
            }
            i = lw;
            q = lm;
          }
          // W in 4-value (32-byte) chunks: rows of k % 4 == 0 are aligned
          const bool vec = (k & 3) == 0;
          uint32_t w8[8];
          auto load4 = [&](int at) {
            if (vec) {
              ldg256_keep(W + at, w8);
            } else {
#pragma unroll
              for (int t = 0; t < 4; ++t) {
                const uint64_t x = at + t < lw ? __ldg(W + at + t) : ~0ull;
                w8[2 * t] = (uint32_t)x;
                w8[2 * t + 1] = (uint32_t)(x >> 32);
              }
            }
          };
          auto wat = [&](int at) {  // register selects, no local-memory indexing
            const int t = at & 3;
            const uint32_t lo = t == 0 ? w8[0] : t == 1 ? w8[2] : t == 2 ? w8[4] : w8[6];
            const uint32_t hi = t == 0 ? w8[1] : t == 1 ? w8[3] : t == 2 ? w8[5] : w8[7];
            return ((uint64_t)hi << 32) | lo;
          };
          if (i < lw) load4(0);
          uint64_t wa = i < lw ? wat(0) : ~0ull;
          auto advance = [&]() {
            if (++i < lw) {
              if ((i & 3) == 0) load4(i);
              wa = wat(i);
            }
          };
          while (i < lw || q < lm) {
            const uint64_t xa = i < lw ? wa : ~0ull;
            const uint64_t xb = q < lm ? M[q] : ~0ull;
            uint64_t x;
            if (xa < xb) {
              x = xa;
              advance();
            } else if (xb < xa) {
              x = xb;
              ++q;
            } else {
              x = xa;
              ++inter;
              ++q;
              advance();
            }
            ++cnt;
            if (!full && cnt == k_eff) {
              kth = x;
              break;
            }
          }
          double raw;
          if (both_small) {
            raw = (double)(sw + c3 - (int64_t)(lw + lm - inter));
          } else if (k_eff < 2) {
            raw = (double)inter;
          } else {
            const double est_union = __ddiv_rn((double)(k_eff - 1), bitsd(kth));
            raw = __dsub_rn((double)(sw + c3), est_union);
          }
          const double hi = (double)(sw < c3 ? sw : c3);
          raw = raw > 0.0 ? raw : 0.0;
          est = raw < hi ? raw : hi;
        }
        acc = __dadd_rn(acc, est);
      }
      __syncwarp();
    };
    if (la <= cap) edge(std::true_type{});
    else edge(std::false_type{});
  }
  for (int o = 16; o > 0; o >>= 1) acc = __dadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, o));
  if (lane == 0) part[(wb - e_begin) / kC4SChunk] = acc;
  }
  // (triples is warp-uniform: every lane added the same c3)
  if (lane == 0 && triples) atomicAdd(out_triples, (unsigned long long)triples);
}

// shared-memory C3 capacity; PG_C4S_CAP (1..512) lowers it so tests can
// drive the global-scratch path on small graphs
static int c4s_cap() {
  const char* e = getenv("PG_C4S_CAP");
  const int c = e ? atoi(e) : kCSCap;
  return c >= 1 && c <= kCSCap ? c : kCSCap;
}

// 1-Hash member-table slots for k > kMaxSketchK (>= 2 * min(|C3|, k))
static int c4s_tcap(int k) {
  int t = 32;
  while (t < 2 * k) t <<= 1;
  return t;
}

constexpr size_t c4s_smem() {
  return (size_t)(kCSBlock / 32) * (kCSCap * 8 + kMaxSketchK * 8 + 2 * kCSCap * 4) + kMaxSketchK * 8;
}

template <int KIND>
static int c4s_grid() {
  auto kern = clique4_sketch_kernel<KIND, false>;
  cudaFuncSetAttribute(clique4_sketch_kernel<KIND, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)c4s_smem());
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c4s_smem());
  return grid_for_kernel(kern, c4s_smem());
}

static int c4s_grid_for(int kind) {
  // kCSBlock == kBlock, so grid_for_kernel's occupancy query applies
  static_assert(kCSBlock == kBlock, "occupancy helper assumes kBlock threads");
  if (kind == PG_KHASH) return c4s_grid<PG_KHASH>();
  if (kind == PG_ONEHASH) return c4s_grid<PG_ONEHASH>();
  return c4s_grid<PG_KMV>();
}

}  // namespace pg

using namespace pg;

extern "C" {

int pg_4clique_sketch_workspace_size(int32_t kind, int32_t k, int64_t max_out_degree, size_t* bytes) {
  PG_REQUIRE(bytes, "null output");
  PG_REQUIRE(kind == PG_KHASH || kind == PG_ONEHASH || kind == PG_KMV, "kind must be PG_KHASH/ONEHASH/KMV");
  PG_REQUIRE(max_out_degree >= 0, "max_out_degree must be >= 0");
  PG_REQUIRE(k >= 1, "k must be >= 1");
  const int64_t grid = c4s_grid_for(kind);
  const int64_t per_warp = max_out_degree > c4s_cap() ? max_out_degree : 0;
  const int64_t warps = grid * (kCSBlock / 32);
  *bytes = (size_t)(grid * 8 + 16) + (size_t)(warps * per_warp) * 16 + 16;
  if (k > kMaxSketchK) *bytes += (size_t)warps * ((size_t)k * 8 + (size_t)c4s_tcap(k) * 4) + 16;
  return PG_OK;
}

int pg_4clique_sketch(int32_t kind, const int64_t* dir_off, const int32_t* dir_adj, const int32_t* src,
                      const int64_t* edge_ids, int64_t e_begin, int64_t e_end, const void* rows,
                      const int32_t* lengths, const int32_t* sizes, int32_t k, const uint64_t* seeds_dev,
                      int64_t max_out_degree, void* workspace, size_t workspace_bytes, double* out_sum,
                      int64_t* out_triples, void* stream) {
  PG_REQUIRE(kind == PG_KHASH || kind == PG_ONEHASH || kind == PG_KMV, "kind must be PG_KHASH/ONEHASH/KMV");
  PG_REQUIRE(k >= 1, "k must be >= 1");
  PG_REQUIRE(0 <= e_begin && e_begin <= e_end, "bad edge range");
  PG_REQUIRE(out_sum && out_triples, "null output");
  size_t need = 0;
  int rc = pg_4clique_sketch_workspace_size(kind, k, max_out_degree, &need);
  if (rc) return rc;
  PG_REQUIRE(workspace && workspace_bytes >= need, "workspace too small (%zu < %zu bytes)", workspace_bytes, need);
  cudaStream_t s = as_stream(stream);
  cudaError_t ce = cudaMemsetAsync(out_sum, 0, sizeof(double), s);
  if (ce == cudaSuccess) ce = cudaMemsetAsync(out_triples, 0, sizeof(int64_t), s);
  if (ce != cudaSuccess) return fail(PG_ERR_CUDA, "memset: %s", cudaGetErrorString(ce));
  if (e_end == e_begin) return PG_OK;
  PG_REQUIRE(dir_off && dir_adj && src && rows && sizes && seeds_dev, "null pointer");
  PG_REQUIRE(kind == PG_KHASH || lengths, "1-Hash / KMV need lengths");
  const int grid = c4s_grid_for(kind);
  const int cap = c4s_cap();
  const int64_t per_warp = max_out_degree > cap ? max_out_degree : 0;
  const int64_t warps = (int64_t)grid * (kCSBlock / 32);
  unsigned char* ws = static_cast<unsigned char*>(workspace);
  double* part = reinterpret_cast<double*>(ws);
  uint64_t* gH = reinterpret_cast<uint64_t*>(ws + (((size_t)grid * 8 + 15) & ~size_t(15)));
  int32_t* gC = reinterpret_cast<int32_t*>(gH + warps * per_warp);
  int32_t* gF = gC + warps * per_warp;
  uint64_t* gM = nullptr;
  int32_t* gT = nullptr;
  const int tcap = c4s_tcap(k);
  if (k > kMaxSketchK) {
    gM = reinterpret_cast<uint64_t*>(
        (reinterpret_cast<uintptr_t>(gF + warps * per_warp) + 15) & ~uintptr_t(15));
    gT = reinterpret_cast<int32_t*>(gM + warps * (int64_t)k);
  }
  C4SketchArgs args{kind == PG_KMV ? nullptr : static_cast<const int32_t*>(rows),
                    kind == PG_KMV ? static_cast<const double*>(rows) : nullptr, lengths, sizes, seeds_dev, k,
                    gM, gT, tcap};
  auto* trip = reinterpret_cast<unsigned long long*>(out_triples);
  ChunkCounter ctr;
  PartialSums ps;  // one partial per chunk of directed edges, summed in chunk order
  cudaError_t se = ctr.init(s);
  if (se == cudaSuccess) se = ps.init(s, (e_end - e_begin + kC4SChunk - 1) / kC4SChunk);
  if (se != cudaSuccess) return fail(PG_ERR_CUDA, "scratch: %s", cudaGetErrorString(se));
  (void)part;
#define PG_C4S(KK)                                                                                       \
  (k > kMaxSketchK ? clique4_sketch_kernel<KK, true> : clique4_sketch_kernel<KK, false>)                \
      <<<grid, kCSBlock, c4s_smem(), s>>>(dir_off, dir_adj, src, edge_ids, e_begin, e_end, \
                                                               args, gC, gF, gH, per_warp, cap, ps.p, trip, ctr.p)
  if (kind == PG_KHASH) PG_C4S(PG_KHASH);
  else if (kind == PG_ONEHASH) PG_C4S(PG_ONEHASH);
  else PG_C4S(PG_KMV);
#undef PG_C4S
  ps.finish(out_sum);
  return check_launch("4clique_sketch");
}

}  // extern "C"
