// Scalar with_set (providers.py:164-175 BloomProvider.with_set, :234-241
// MinHashProvider.with_set, :303-307 KmvProvider.with_set): the estimate of
// |S_w & members| for one vertex w and one explicit member set, in a single
// one-warp launch.  The member sketch is built in shared memory with the
// reference's per-set builders' semantics (sketches.py:187-237) and
// compared with w's stored row; members and the result may live in pinned
// mapped host memory, so a call is one launch and one stream synchronisation.
//
// `members` is the caller's argument sorted (np.sort: repeats kept, as the
// reference's builders see them; its length enters the estimates as
// len(members)); at most kScalarCap of them (PG_ERR_UNSUPPORTED otherwise:
// the caller then builds the member sketch with the whole-graph builders).
#include "pg_engines.cuh"

namespace pg {

constexpr int kScalarCap = 2048;  // members held in shared memory
constexpr int kScalarBits = 65536;  // Bloom rows built in shared memory

struct ScalarSmem {
  uint64_t key[kScalarCap];   // h_0 (1-Hash) / unit bits (KMV) of the members
  int32_t mem[kScalarCap];    // the distinct members, ascending
  int32_t flag[kScalarCap];  // KMV repeat flags
  uint64_t M[kMaxSketchK];    // member sketch (k-Hash IDs, KMV values)
  int32_t tab[2 * kMaxSketchK];
  unsigned hist[256];
  int cnt;
};

__device__ __forceinline__ int warp_sum_i(int x) { return __reduce_add_sync(0xffffffffu, x); }

// k-th smallest (1-based) of n distinct 64-bit keys by MSB radix select
__device__ uint64_t scalar_select(const uint64_t* key, int n, int target, unsigned* hist) {
  const int lane = threadIdx.x & 31;
  uint64_t prefix = 0, pmask = 0;
  int rem = target;
  for (int shift = 56; shift >= 0; shift -= 8) {
    for (int i = lane; i < 256; i += 32) hist[i] = 0u;
    __syncwarp();
    for (int j = lane; j < n; j += 32)
      if ((key[j] & pmask) == prefix) atomicAdd(hist + ((key[j] >> shift) & 255u), 1u);
    __syncwarp();
    int dig = 0, before = 0;
    if (lane == 0) {
      int c = 0;
      for (int i = 0; i < 256; ++i) {
        if (c + (int)hist[i] >= rem) {
          dig = i;
          before = c;
          break;
        }
        c += hist[i];
      }
    }
    dig = __shfl_sync(0xffffffffu, dig, 0);
    before = __shfl_sync(0xffffffffu, before, 0);
    rem -= before;
    prefix |= (uint64_t)dig << shift;
    pmask |= 255ull << shift;
    __syncwarp();
  }
  return prefix;
}

__global__ void __launch_bounds__(32) with_set_kernel(int kind, const void* __restrict__ rows,
                                                      const int32_t* __restrict__ lengths,
                                                      const int32_t* __restrict__ sizes, int width, int nh,
                                                      const uint64_t* __restrict__ seeds, const double* __restrict__ lut,
                                                      int32_t w, const int32_t* __restrict__ members_in, int ncount,
                                                      double* __restrict__ out) {
  const int64_t nraw = ncount;  // len(members) as the reference passes it
  extern __shared__ __align__(16) unsigned char smem_raw[];
  ScalarSmem& S = *reinterpret_cast<ScalarSmem*>(smem_raw);
  uint32_t* bf = reinterpret_cast<uint32_t*>(smem_raw + sizeof(ScalarSmem));  // Bloom: width/32 words
  const int lane = threadIdx.x;
  const int64_t sw = sizes[w];
  // members_in: the sorted multiset (np.sort of the argument).  The per-set
  // builders see repeats only in 1-Hash (build_onehash keeps them, and
  // intersect_merge then counts a repeated member as shared); the distinct
  // members, in order, go to S.mem
  int nm = 0;
  for (int base = 0; base < ncount; base += 32) {
    const int i = base + lane;
    const int32_t x = i < ncount ? members_in[i] : 0;
    const bool first = i < ncount && (i == 0 || members_in[i - 1] != x);
    const unsigned m = __ballot_sync(0xffffffffu, first);
    if (first) S.mem[nm + __popc(m & ((1u << lane) - 1u))] = x;
    nm += __popc(m);
  }
  __syncwarp();
  double est = 0.0;
  if (kind == PG_BF_AND || kind == PG_BF_L || kind == PG_BF_OR) {
    const int words32 = width >> 5;
    const bool pow2 = (width & (width - 1)) == 0;
    for (int i = lane; i < words32; i += 32) bf[i] = 0u;
    __syncwarp();
    for (int i = lane; i < nm; i += 32) {
      const int32_t x = S.mem[i];
      for (int h = 0; h < nh; ++h) {
        const uint64_t hw = hash_word(seeds[h], x);
        const uint32_t p = pow2 ? (uint32_t)(hw & (uint64_t)(width - 1)) : (uint32_t)(hw % (uint64_t)width);
        atomicOr(bf + (p >> 5), 1u << (p & 31));
      }
    }
    __syncwarp();
    const uint32_t* rw = reinterpret_cast<const uint32_t*>(rows) + (int64_t)w * words32;
    int ones = 0;
    for (int i = lane; i < words32; i += 32) ones += __popc(kind == PG_BF_OR ? (rw[i] | bf[i]) : (rw[i] & bf[i]));
    ones = warp_sum_i(ones);
    if (kind == PG_BF_OR) {
      const double raw = __dsub_rn((double)(sw + nraw), lut[ones]);
      est = raw > 0.0 ? raw : 0.0;
    } else if (kind == PG_BF_L) {
      est = __ddiv_rn((double)ones, (double)nh);
    } else {
      est = lut[ones];
    }
  } else if (kind == PG_KHASH) {
    const int k = width;
    const int32_t* ent = reinterpret_cast<const int32_t*>(rows) + (int64_t)w * k;
    int m = 0;
    if (sw > 0 && nm > 0) {
      for (int i = lane; i < k; i += 32) {
        const uint64_t sd = seeds[i];
        uint64_t mn = ~0ull;
        for (int q = 0; q < nm; ++q) {
          const uint64_t h = hash_word(sd, S.mem[q]);
          mn = h < mn ? h : mn;
        }
        m += ent[i] == (int32_t)(uint32_t)(unmix64(mn) ^ sd);
      }
    }
    m = warp_sum_i(m);
    if (sw > 0 && nm > 0) {
      const double j = __ddiv_rn((double)m, (double)k);
      est = __dmul_rn(__ddiv_rn(j, __dadd_rn(1.0, j)), (double)(sw + nraw));
    }
  } else if (kind == PG_ONEHASH) {
    // build_onehash (sketches.py:217-226) on the multiset: the min(k, n)
    // entries of smallest (h_0, x), repeats kept; key equality <=> same x
    const int k = width;
    const int32_t* ent = reinterpret_cast<const int32_t*>(rows) + (int64_t)w * k;
    const int lw = lengths[w];
    const uint64_t s0 = seeds[0];
    for (int i = lane; i < ncount; i += 32) S.key[i] = hash_word(s0, members_in[i]);
    __syncwarp();
    const int ly = ncount < k ? ncount : k;  // stored entries, repeats counted
    const uint64_t thr = ncount > k ? scalar_select(S.key, ncount, k, S.hist) : ~0ull;
    // distinct selected members (key <= thr) as an open-addressing set
    int nsel = 0;
    for (int i = lane; i < nm; i += 32) nsel += hash_word(s0, S.mem[i]) <= thr;
    nsel = warp_sum_i(nsel);
    int tb = 5;
    while ((1 << tb) < 2 * nsel) ++tb;
    for (int i = lane; i < (1 << tb); i += 32) S.tab[i] = -1;
    __syncwarp();
    for (int i = lane; i < nm; i += 32) {
      const int32_t x = S.mem[i];
      if (hash_word(s0, x) > thr) continue;
      uint32_t h = ((uint32_t)x * 0x9E3779B1u) >> (32 - tb);
      while (atomicCAS(S.tab + h, -1, x) != -1) h = (h + 1) & ((1u << tb) - 1);
    }
    __syncwarp();
    int hits = 0;
    for (int i = lane; i < lw; i += 32) {
      const int32_t y = ent[i];
      uint32_t h = ((uint32_t)y * 0x9E3779B1u) >> (32 - tb);
      int32_t c;
      while ((c = S.tab[h]) != y && c != -1) h = (h + 1) & ((1u << tb) - 1);
      hits += c == y;
    }
    hits = warp_sum_i(hits);
    // intersect_merge (setops.py) counts adjacent equal pairs of the merged
    // entries: every repeat of a stored member pairs with its first copy
    const int common = (lw > 0 && ly > 0) ? ly - nsel + hits : 0;
    // est_intersection_minhash (estimators.py:157-168) over
    // _jaccard_onehash (:134-145)
    if (sw <= k && nraw <= k) {
      est = (double)common;
    } else if (lw + ly > 0) {
      int denom = lw + ly - common;
      denom = denom < k ? denom : k;
      const double j = denom ? __ddiv_rn((double)common, (double)denom) : 0.0;
      est = __dmul_rn(__ddiv_rn(j, __dadd_rn(1.0, j)), (double)(sw + nraw));
    }
  } else {  // KMV: est_intersection_kmv (estimators.py:171-200)
    const int k = width;
    const uint64_t* W = reinterpret_cast<const uint64_t*>(rows) + (int64_t)w * k;
    const int lw = lengths[w];
    const uint64_t s0 = seeds[0];
    for (int i = lane; i < nm; i += 32) S.key[i] = dbits(unit_value(hash_word(s0, S.mem[i])));
    __syncwarp();
    // distinct values: repeats flagged with the sign bit (units are positive)
    for (int i = lane; i < nm; i += 32) {
      bool dup = false;
      for (int q = 0; q < i; ++q) dup |= S.key[q] == S.key[i];
      S.flag[i] = dup;
    }
    __syncwarp();
    for (int i = lane; i < nm; i += 32)
      if (S.flag[i]) S.key[i] |= 1ull << 63;
    __syncwarp();
    int nd = 0;
    for (int i = lane; i < nm; i += 32) {
      const uint64_t x = S.key[i];
      if (x >> 63) continue;
      ++nd;
      int r = 0;
      for (int q = 0; q < nm; ++q) r += S.key[q] < x;
      if (r < k) S.M[r] = x;
    }
    nd = warp_sum_i(nd);
    __syncwarp();
    const int lm = nd < k ? nd : k;
    const bool both_small = sw <= k && nraw <= k;
    const int k_eff = lw < lm ? lw : lm;
    if (lane == 0) {
      // the merge of the two ascending value lists
      int i = 0, q = 0, cnt = 0, inter = 0;
      uint64_t kth = 0;
      const bool full = both_small || k_eff < 2;
      while (i < lw || q < lm) {
        const uint64_t xa = i < lw ? (uint64_t)__double_as_longlong(((const double*)W)[i]) : ~0ull;
        const uint64_t xb = q < lm ? S.M[q] : ~0ull;
        uint64_t x;
        if (xa < xb) {
          x = xa;
          ++i;
        } else if (xb < xa) {
          x = xb;
          ++q;
        } else {
          x = xa;
          ++inter;
          ++i;
          ++q;
        }
        ++cnt;
        if (!full && cnt == k_eff) {
          kth = x;
          break;
        }
      }
      double raw;
      if (both_small) {
        raw = (double)(sw + nraw - (int64_t)(lw + lm - inter));
      } else if (k_eff < 2) {
        raw = (double)inter;
      } else {
        raw = __dsub_rn((double)(sw + nraw), __ddiv_rn((double)(k_eff - 1), bitsd(kth)));
      }
      const double hi = (double)(sw < nraw ? sw : nraw);
      raw = raw > 0.0 ? raw : 0.0;
      est = raw < hi ? raw : hi;
    }
  }
  if (lane == 0) out[0] = est;
}

}  // namespace pg

using namespace pg;

extern "C" {

int pg_with_set(int32_t kind, const void* rows, const int32_t* lengths, const int32_t* sizes, int32_t width,
                int32_t hash_count, const uint64_t* seeds_dev, const double* lut, int32_t w,
                const int32_t* members, int32_t count, double* out, void* stream) {
  PG_REQUIRE(kind >= PG_BF_AND && kind <= PG_KMV, "unknown estimator kind %d", kind);
  PG_REQUIRE(count >= 0 && w >= 0, "bad arguments");
  PG_REQUIRE(rows && sizes && seeds_dev && out && (count == 0 || members), "null pointer");
  const bool bloom = kind <= PG_BF_OR;
  if (count > kScalarCap) return fail(PG_ERR_UNSUPPORTED, "with_set holds up to %d members", kScalarCap);
  if (bloom) {
    PG_REQUIRE(width >= 64 && width % 64 == 0, "Bloom size must be a positive multiple of 64");
    if (width > kScalarBits) return fail(PG_ERR_UNSUPPORTED, "with_set builds Bloom rows up to %d bits", kScalarBits);
    PG_REQUIRE(kind == PG_BF_L || lut, "the estimate needs the Swamidass table");
    PG_REQUIRE(hash_count >= 1 && hash_count <= 64, "bad hash count");
  } else {
    PG_REQUIRE(width >= 1, "k must be >= 1");
    if (width > kMaxSketchK) return fail(PG_ERR_UNSUPPORTED, "with_set sketches up to k = %d", kMaxSketchK);
    PG_REQUIRE(kind == PG_KHASH || lengths, "1-Hash / KMV need lengths");
  }
  const size_t smem = sizeof(ScalarSmem) + (bloom ? (size_t)width / 8 : 0);
  cudaStream_t s = as_stream(stream);
  cudaFuncSetAttribute(with_set_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  with_set_kernel<<<1, 32, smem, s>>>(kind, rows, lengths, sizes, width, hash_count, seeds_dev, lut, w, members,
                                      count, out);
  return check_launch("with_set");
}

}  // extern "C"
