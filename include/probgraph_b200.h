/*
 * probgraph_b200.h -- C ABI of the B200-native per-edge sketch-intersection
 * engine (ProbGraph, arxiv 2208.11469).
 *
 * This is the drop-in boundary that sits under the reference's Python
 * provider/plugin API (`make_provider`, `IntersectionProvider.pair_many`,
 * `build_sketched_graph`, `tc_estimate`, `four_clique_count`,
 * `jarvis_patrick_cluster`).  Every entry point names the reference
 * interface it replaces (paths relative to /root/reference/pkg/src/probgraph).
 *
 * Conventions (all functions):
 *   - return 0 on success, a negative PG_ERR_* code on failure; the message
 *     of the last failure on the calling thread is read with pg_last_error;
 *   - every array argument is a DEVICE pointer owned by the caller (torch
 *     tensors or cudaMalloc), unless the name ends in `_host`;
 *   - `stream` is a cudaStream_t passed as void*; NULL means the legacy
 *     default stream.  Calls are asynchronous and stream-ordered; none of
 *     them synchronises the host except where stated;
 *   - scratch: the large, input-sized scratch is caller-allocated with a
 *     size query (pg_csr_upper_edges_workspace, pg_csr_range_slots_workspace,
 *     pg_4clique_sketch_workspace_size); small or launch-shaped scratch
 *     (dynamic-chunk counters, per-block fp64 partial sums, hub lists, the
 *     generic kernels' per-warp rows) is taken stream-ordered from the
 *     device's default memory pool (cudaMallocAsync / cudaFreeAsync on the
 *     call's stream; the pool's release threshold is raised once so repeated
 *     calls reuse it) -- no call allocates persistently;
 *   - vertex IDs are int32 (n < 2^31), CSR offsets are int64;
 *   - sketch layouts in HBM (row-major, one row per vertex):
 *       Bloom : uint64 rows[n][bits/64], little-endian bit p of the row is
 *               word p>>6, bit p&63; ones int32[n]
 *       k-Hash: int32 entries[n][k], -1 for an empty neighbourhood
 *       1-Hash: int32 entries[n][k] ascending IDs, -1 pad; lengths int32[n]
 *       KMV   : double values[n][k] ascending, +inf pad; lengths int32[n]
 */
#ifndef PROBGRAPH_B200_H
#define PROBGRAPH_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define PG_API __attribute__((visibility("default")))
#else
#define PG_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define PG_ABI_VERSION 1

#define PG_OK 0
#define PG_ERR_INVALID (-1)     /* bad argument            -> ValueError     */
#define PG_ERR_CUDA (-2)        /* CUDA runtime failure    -> RuntimeError   */
#define PG_ERR_UNSUPPORTED (-3) /* parameter outside an engine's range (e.g.
                                   the rank-directory KMV engine's k in
                                   {32, 64, 128}); the library's public paths
                                   fall back to a general engine            */

/* estimator / op selectors (reference EstimatorKind, estimators.py:54-62) */
#define PG_BF_AND 0
#define PG_BF_L 1
#define PG_BF_OR 2
#define PG_KHASH 3
#define PG_ONEHASH 4
#define PG_KMV 5

/* ---- runtime -------------------------------------------------------- */
PG_API int pg_abi_version(void);
/* copies the calling thread's last error message (NUL terminated) */
PG_API int pg_last_error(char* buf, size_t len);
/* SM count of the current device */
PG_API int pg_device_sm_count(int* out_host);

/* ---- a2: hash family  (hashing.py:78-111 HashFamily.__post_init__) --- */
/* seed_i = mix64(base ^ mix64(i+1)), i < count; host-only, no device use */
PG_API int pg_family_seeds(uint64_t base, int32_t count, uint64_t* out_host);
/* the same seeds written to device memory on `stream` (no host transfer) */
PG_API int pg_family_seeds_device(uint64_t base, int32_t count, uint64_t* out_dev,
                                  void* stream);
/* a1/a3 words: out[j] = mix64(seed ^ (uint64)keys[j])  (hashing.py:114-118) */
PG_API int pg_hash_words(const int64_t* keys, int64_t count, uint64_t seed,
                  uint64_t* out, void* stream);

/* ---- graph preparation (graphs.py:101-105 CsrGraph.edges,
 *      mining.py:83-85 _directed_edge_arrays) ----------------------------- */
/* bytes of scratch pg_csr_upper_edges(_padded) needs for n vertices and
 * `capacity` output slots */
PG_API int pg_csr_upper_edges_workspace(int64_t n, int64_t capacity,
                                        size_t* out_bytes_host);
/* Writes every undirected edge once, u < v, in CSR order (== graph.edges()).
 * us/vs hold `capacity` entries (m = nnz/2 for a symmetric CSR); m_host
 * receives the count (host sync); a count above capacity is an error. */
PG_API int pg_csr_upper_edges(const int64_t* offsets, const int32_t* adj, int64_t n,
                       int32_t* us, int32_t* vs, int64_t capacity, int64_t* m_host,
                       void* workspace, size_t workspace_bytes, void* stream);
/* Same edge list with every CSR row's run of upper edges padded to a
 * multiple of `pad` (power of two <= 32) with (u, -1) slots, so groups of
 * `pad` consecutive slots never straddle two u rows -- the layout the fused
 * row kernels consume (pad = their lanes-per-edge group size, see
 * pg_group_pad).  slots_host receives the slot count (host sync). */
PG_API int pg_csr_upper_edges_padded(const int64_t* offsets, const int32_t* adj, int64_t n,
                              int32_t pad, int32_t* us, int32_t* vs, int64_t capacity,
                              int64_t* slots_host, void* workspace, size_t workspace_bytes,
                              void* stream);
/* The same padded slots for the rows of [v0, v1) only -- their lower
 * (lower = 1: neighbours < u) or upper (0: > u) entries -- appended at the
 * device cursor cursor_dev[0] with no host sync; range_dev receives the
 * appended [begin, end) and cursor_dev[0] advances to end; us is the
 * group-u array (one u per pad slots, padded mode 2).  cursor_dev[1] is set
 * to 1 if the range's slots exceed max_slots (a host bound on them, e.g.
 * its entries + (pad-1) rows) or `capacity` (they are then dropped).  Used
 * to lay out each upload chunk as it lands (CsrGraph.edges(),
 * graphs.py:101-105, restricted to a vertex range; the lower triangle holds
 * every undirected edge once as well). */
PG_API int pg_csr_range_slots_workspace(int64_t rows, int64_t max_slots, size_t* bytes);
PG_API int pg_csr_range_slots_append(const int64_t* offsets, const int32_t* adj, int64_t v0,
                              int64_t v1, int32_t pad, int32_t lower, int64_t max_slots,
                              int32_t* ug, int32_t* vs, int64_t capacity, int64_t* cursor_dev,
                              int64_t* range_dev, void* workspace, size_t workspace_bytes,
                              void* stream);
/* lanes-per-edge group size of the fused kernels for rows of `row_bytes`
 * (Bloom: bits/8, k-Hash: 4k) = the pad of the layout above (1: no pad) */
PG_API int pg_group_pad(int32_t row_bytes, int32_t* pad_host);
/* src[j] = row of adjacency entry j (np.repeat(arange(n), degrees)) */
PG_API int pg_csr_expand_rows(const int64_t* offsets, int64_t n, int64_t nnz,
                       int32_t* src, void* stream);

/* ---- (1) sketch builders  (sketches.py:314-396 _build_*_matrix,
 *      :399-451 build_sketched_graph) ------------------------------------
 * Every size plan_budget produces is served: Bloom rows up to 65,536 bits and
 * k <= 256 by the tuned kernels; wider rows / larger k by generic kernels
 * (pg_generic.cu: global atomics, a thread per (vertex, function), a
 * warp-level radix select per vertex).  The estimators below likewise fall
 * back to warp-per-edge kernels with global statistics for k > 256 and
 * Bloom rows over 32,768 bits (16,384 for the 4-clique count). */
/* seeds_dev: the HashFamily seeds (count = b, k, 1, 1 respectively) */
PG_API int pg_build_bloom(const int64_t* offsets, const int32_t* adj, int64_t n,
                   int32_t bits, int32_t b, const uint64_t* seeds_dev,
                   uint64_t* rows, int32_t* ones, void* stream);
PG_API int pg_build_khash(const int64_t* offsets, const int32_t* adj, int64_t n,
                   int32_t k, const uint64_t* seeds_dev, int32_t* entries,
                   void* stream);
PG_API int pg_build_onehash(const int64_t* offsets, const int32_t* adj, int64_t n,
                     int32_t k, const uint64_t* seeds_dev, int32_t* entries,
                     int32_t* lengths, void* stream);
PG_API int pg_build_kmv(const int64_t* offsets, const int32_t* adj, int64_t n,
                 int32_t k, const uint64_t* seeds_dev, double* values,
                 int32_t* lengths, void* stream);
/* KMV value ranks (a device layout of sketches.py:375-396, not a reference
 * interface): rank_of[x] = dense rank of unit_value(h_0(x)) among all x in
 * [0, n) (hashing.py:146-153), rank_values[r] = the value of rank r.  Equal
 * values share a rank, so ranks order and compare exactly like the values. */
PG_API int pg_kmv_rank_table(int64_t n, const uint64_t* seeds_dev, int32_t* rank_of,
                      double* rank_values, void* stream);
/* pg_build_kmv plus ranks[n][k] (int32 ascending, INT32_MAX pad): the same
 * selection made on ranks; values = rank_values[ranks] (bit-identical). */
PG_API int pg_build_kmv_ranked(const int64_t* offsets, const int32_t* adj, int64_t n,
                        int32_t k, const uint64_t* seeds_dev, const int32_t* rank_of,
                        const double* rank_values, double* values, int32_t* ranks,
                        int32_t* lengths, void* stream);

/* ---- (2) per-edge estimators, parity path
 *      (providers.py:150-162 BloomProvider.pair_many,
 *       :205-232 MinHashProvider.pair_many, :266-301 KmvProvider.pair_many) */
/* op: PG_BF_AND | PG_BF_L | PG_BF_OR.  lut: double[bits+1] =
 * swamidass_value(bits, b, 0..bits) (estimators.py:65-70).  out_count
 * (popcount of AND / OR) and out_est are each nullable. */
PG_API int pg_pairs_bloom(const uint64_t* rows, int32_t bits, int32_t b, int32_t op,
                   const int32_t* sizes, const double* lut,
                   const int32_t* us, const int32_t* vs, int64_t count,
                   int32_t* out_count, double* out_est, void* stream);
/* onehash != 0 selects 1-Hash semantics; out_count = match count */
PG_API int pg_pairs_minhash(const int32_t* entries, int32_t k, int32_t onehash,
                     const int32_t* sizes, const int32_t* us,
                     const int32_t* vs, int64_t count, int32_t* out_count,
                     double* out_est, void* stream);
/* out_common / out_union: common and distinct-union counts; out_kth: the
 * max(k_eff,1)-th smallest distinct union value (all nullable) */
PG_API int pg_pairs_kmv(const double* values, const int32_t* lengths, int32_t k,
                 const int32_t* sizes, const int32_t* us, const int32_t* vs,
                 int64_t count, int32_t* out_common, int32_t* out_union,
                 double* out_kth, double* out_est, void* stream);

/* ---- (2)+(3) fused whole-graph passes over edges [e_begin, e_end) -------
 *      mining.py:105-130 tc_estimate, :63-80 _chunked_sum                */
/* Fused passes take `padded`: 0 = any (us, vs) edge list, 1 = the
 * row-padded layout of pg_csr_upper_edges_padded with pad =
 * pg_group_pad(row bytes) and e_begin a multiple of pad (precondition, not
 * checked: every aligned group of pad slots holds one u).  Slots with
 * vs[j] < 0 are padding and skipped.  pg_tc_bloom, and pg_tc_minhash /
 * pg_jaccard_count_khash for k-Hash rows of 64/128/256 bytes, also take 2 =
 * the same layout with us[] holding one u per pad-slot group (us[j / pad], a
 * pad-fold smaller u stream).  Any orientation of an edge gives the same
 * per-edge count (every estimator is symmetric in (u, v)), so the slots may
 * run from the lower- to the higher-(degree, ID)-rank endpoint (the N+ lists
 * of degree_order) -- the layout the library picks for matrices that stream
 * from HBM.
 * Bloom TC.
 * out_hist: int64[bits+1] histogram of per-edge popcounts
 * (for PG_BF_OR only edges with raw > 0 are counted, and out_sum_pos
 * receives the int64 sum of (s_u+s_v) over those edges).  Overwrites
 * the outputs.  Final estimate is formed on the host from the integers. */
PG_API int pg_tc_bloom(const uint64_t* rows, int32_t bits, int32_t op,
                const int32_t* sizes, const double* lut, const int32_t* us,
                const int32_t* vs, int64_t e_begin, int64_t e_end, int32_t padded,
                int64_t* out_hist, int64_t* out_sum_pos, void* stream);
/* pg_tc_bloom (padded mode 2) over the slots [range_dev[0], range_dev[1])
 * read on the device (a pg_csr_range_slots_append range); the launch is
 * sized for max_slots.  accumulate = 1 adds into out_hist / out_sum_pos
 * instead of overwriting them (one histogram over several ranges). */
PG_API int pg_tc_bloom_range(const uint64_t* rows, int32_t bits, int32_t op,
                      const int32_t* sizes, const double* lut, const int32_t* ug,
                      const int32_t* vs, const int64_t* range_dev, int64_t max_slots,
                      int32_t accumulate, int64_t* out_hist, int64_t* out_sum_pos,
                      void* stream);
/* ---- degree-oriented, hub-cached Bloom TC (2048-bit rows) ---------------
 *      same per-edge popcounts as pg_tc_bloom (providers.py:150-162,
 *      mining.py:105-130), every edge oriented low -> high (degree, ID)
 *      rank (graphs.py:154-166 degree_order).                             */
/* Every entry of an oriented CSR (e.g. the N+ lists of pg_degree_order) as
 * row-padded slots (pad a power of two <= 32, (u, -1) padding): the
 * pg_csr_upper_edges_padded layout without the v > u filter.  Workspace
 * from pg_csr_upper_edges_workspace; slots_host receives the count. */
PG_API int pg_csr_row_slots_padded(const int64_t* offsets, const int32_t* adj, int64_t n,
                            int32_t pad, int32_t* us, int32_t* vs, int64_t capacity,
                            int64_t* slots_host, void* workspace, size_t workspace_bytes,
                            void* stream);
/* hub_ids[i] = the vertex of rank n - n_hubs + i (rank from
 * pg_degree_order), and every slot vs[e] >= 0 naming such a vertex becomes
 * the tag -2 - i (in place). */
PG_API int pg_hub_tag(const int32_t* rank, int64_t n, int32_t n_hubs, int32_t* vs,
               int64_t slots, int32_t* hub_ids, void* stream);
/* most hub rows the engine can stage in one CTA's shared memory (0 when
 * `bits` has no hub engine) */
PG_API int pg_tc_bloom_hub_capacity(int32_t bits, int32_t* max_hubs);
/* pg_tc_bloom over hub-tagged group-u slots (ug[e / 8] = u of slots
 * [8q, 8q+8), e_begin a multiple of 8): hub v rows read from shared memory.
 * Same outputs and overwrite semantics as pg_tc_bloom. */
PG_API int pg_tc_bloom_hub(const uint64_t* rows, int32_t bits, int32_t op,
                    const int32_t* sizes, const double* lut, const int32_t* ug,
                    const int32_t* vs, int64_t e_begin, int64_t e_end,
                    const int32_t* hub_ids, int32_t n_hubs, int64_t* out_hist,
                    int64_t* out_sum_pos, void* stream);
/* slot pad of the 1-Hash per-warp-table TC engine for k (the layout pad
 * pg_tc_minhash expects with onehash = 1 and padded = 1; 1 = no such engine
 * for k, padded slots are then not needed) */
PG_API int pg_onehash_block_pad(int32_t k, int32_t* pad_host);
/* 1-Hash hash-rank rows, a device layout for the TC engine with no reference
 * counterpart: rank_of[x] = position of h0(x) = mix64(seed_0 ^ x) among the
 * hash words of all n vertices (h0 is a bijection on IDs: an exact
 * relabelling), and rank_rows[v] = the ranks of entries[v] ascending,
 * INT32_MAX pad (k = 32, 64, 128), stored interleaved for `group` lanes per
 * row (sorted element j at slot (j % group) * (k / group) + j / group; group
 * = 32 / pg_onehash_block_pad(k) for the TC engine, 1 = plain ascending).  Two rows share an ID iff their rank rows
 * share a rank (providers.py:200-203 _matches_onehash counts the same
 * integer), and no rank of v above u's largest can be in u's row, so the
 * engine stops probing there.  pg_tc_minhash takes them with onehash = 2. */
PG_API int pg_hash_rank_table(int64_t n, const uint64_t* seeds_dev, int32_t* rank_of,
                       void* stream);
PG_API int pg_onehash_rank_rows(const int32_t* entries, int64_t n, int32_t k,
                         const int32_t* rank_of, int32_t group, int32_t* rank_rows,
                         void* stream);
/* out[e] = the number of probes the rank-row engine makes for a slot with
 * table row ts[e] and probe row ps[e] (ranks of ps[e] <= the largest rank of
 * ts[e]; 0 for pads): a layout helper -- slots of one table row sorted by it
 * keep the edges a warp processes together equally long. */
PG_API int pg_onehash_prefix_counts(const int32_t* rank_rows, const int32_t* lengths, int32_t k,
                             int32_t group, const int32_t* ts, const int32_t* ps,
                             int64_t count, int32_t* out, void* stream);
/* adj_out = the rows of the oriented CSR (off, adj) (row = table vertex,
 * entries = probe endpoints) counting-sorted (stable) by the register
 * positions the rank-row engine needs per entry, ceil(probes / group)
 * (probes as pg_onehash_prefix_counts).  Synchronises the stream once. */
PG_API int pg_onehash_sort_rows(const int64_t* off, const int32_t* adj, int64_t n,
                         const int32_t* rank_rows, const int32_t* lengths, int32_t k,
                         int32_t group, int32_t* adj_out, void* stream);
/* k-/1-Hash TC: out_cnt[m], out_ssum[m] (m = 0..k): number of edges and
 * int64 sum of (s_u+s_v) of non-verbatim edges with m matches;
 * out_verbatim[0] = sum of matches over verbatim 1-Hash edges. */
PG_API int pg_tc_minhash(const int32_t* entries, int32_t k, int32_t onehash,
                  const int32_t* sizes, const int32_t* us, const int32_t* vs,
                  int64_t e_begin, int64_t e_end, int32_t padded, int64_t* out_cnt,
                  int64_t* out_ssum, int64_t* out_verbatim, void* stream);
/* KMV TC: out_sum[0] = sum of per-edge estimates (fp64; block sums added
 * atomically, so the last bits depend on the order) */
PG_API int pg_tc_kmv(const double* values, const int32_t* lengths, int32_t k,
              const int32_t* sizes, const int32_t* us, const int32_t* vs,
              int64_t e_begin, int64_t e_end, double* out_sum, void* stream);
/* KMV TC over rank rows (pg_build_kmv_ranked) and the row-padded edge slots
 * of pad = pg_kmv_ranked_pad(k) (256/k for k = 32, 64, 128; 0 = no
 * rank-directory engine for k): the same per-edge estimates as pg_tc_kmv
 * (providers.py:266-301), out_sum[0] = their sum. */
PG_API int pg_kmv_ranked_pad(int32_t k, int32_t* pad_host);
PG_API int pg_tc_kmv_ranked(const int32_t* ranks, const double* rank_values,
                     const int32_t* lengths, int32_t k, const int32_t* sizes,
                     const int32_t* us, const int32_t* vs, int64_t e_begin,
                     int64_t e_end, double* out_sum, void* stream);
/* KMV TC over rank rows with one lane per edge slot (any slot layout; slots
 * with vs < 0 are pads): a two-pointer merge that stops after k_eff steps
 * where the estimate only needs the k_eff-th distinct union value
 * (providers.py:266-301; same per-edge estimates as pg_tc_kmv), k = 32, 64,
 * 128 (pg_kmv_merge_supported).  out_sum[0] = the sum, reproducible for a
 * given (e_begin, e_end).  pg_kmv_merge_partition reorders a slot list
 * (stable counting sort) into [slots whose merge stops after k_eff steps,
 * by k_eff bucket (k_eff - 1) * keff_buckets / k ascending (1..8 buckets) |
 * full-merge slots and pads], *split_host = size of the first part: the
 * layout the engine runs fastest on (synchronises the stream). */
PG_API int pg_kmv_merge_supported(int32_t k, int32_t* ok_host);
PG_API int pg_tc_kmv_merge(const int32_t* ranks, const double* rank_values,
                    const int32_t* lengths, int32_t k, const int32_t* sizes,
                    const int32_t* us, const int32_t* vs, int64_t e_begin,
                    int64_t e_end, double* out_sum, void* stream);
PG_API int pg_kmv_merge_partition(const int32_t* us, const int32_t* vs, int64_t count,
                    const int32_t* sizes, const int32_t* lengths, int32_t k,
                    int32_t keff_buckets, int32_t* out_us, int32_t* out_vs,
                    int64_t* split_host, void* stream);
/* Jaccard clustering count (config 4; estimators.py:123-131 + 148-154 and
 * mining.py:157-186).  out_counts[0] = #edges with matches >= min_matches
 * (J-hat = m/k >= tau), out_counts[1] = #edges whose vertex_similarity
 * JACCARD reading (clamped intersection) is >= tau, out_counts[2..k+2] =
 * histogram of matches. */
PG_API int pg_jaccard_count_khash(const int32_t* entries, int32_t k,
                           const int32_t* degrees, const int32_t* us,
                           const int32_t* vs, int64_t e_begin, int64_t e_end,
                           int32_t padded, int32_t min_matches, double tau,
                           int64_t* out_counts, void* stream);
/* 4-clique, Bloom over N+ (mining.py:133-154 + providers.py:164-175):
 * for each directed edge j in [e_begin,e_end) with src[j]=u, dir_adj[j]=v:
 * C3 = N+u & N+v exactly, then for w in C3 histogram
 * popcount(rows_plus[w] op BF(C3)).  op = PG_BF_AND | PG_BF_L | PG_BF_OR
 * (OR: out_hist counts positive edges, out_sum_pos gets sum(s_w + |C3|)).
 * out_triples[0] = number of (u,v,w) triples. */
PG_API int pg_4clique_bloom(const int64_t* dir_off, const int32_t* dir_adj,
                     const int32_t* src, int64_t e_begin, int64_t e_end,
                     const uint64_t* rows_plus, int32_t bits, int32_t b,
                     const uint64_t* seeds_dev, int32_t op,
                     const int32_t* sizes, const double* lut,
                     int64_t* out_hist, int64_t* out_sum_pos,
                     int64_t* out_triples, void* stream);

/* the same over a list of directed-edge indices (an edge sample): edge
 * j = edge_ids[i] is (src[j], dir_adj[j]) */
PG_API int pg_4clique_bloom_edges(const int64_t* dir_off, const int32_t* dir_adj,
                     const int32_t* src, const int64_t* edge_ids, int64_t count,
                     const uint64_t* rows_plus, int32_t bits, int32_t b,
                     const uint64_t* seeds_dev, int32_t op,
                     const int32_t* sizes, const double* lut,
                     int64_t* out_hist, int64_t* out_sum_pos,
                     int64_t* out_triples, void* stream);

/* exact 4-clique count over N+ (mining.py:133-154 with ExactProvider):
 * out_count[0] = sum over directed edges (u,v) and w in C3 of |N+w & C3| */
PG_API int pg_4clique_exact(const int64_t* dir_off, const int32_t* dir_adj,
                     const int32_t* src, int64_t e_begin, int64_t e_end,
                     int64_t* out_count, void* stream);

/* the same with the w rows N(w) taken from a second CSR (w_off, w_adj): the
 * ExactProvider's own rows (providers.py:117-118 with_set over
 * ExactProvider._slice), e.g. a provider built for_graph (undirected N(w))
 * while C3 comes from the view's N+ lists.  pg_4clique_exact is this with
 * w_off = dir_off, w_adj = dir_adj. */
PG_API int pg_4clique_exact_rows(const int64_t* dir_off, const int32_t* dir_adj,
                     const int32_t* src, int64_t e_begin, int64_t e_end,
                     const int64_t* w_off, const int32_t* w_adj,
                     int64_t* out_count, void* stream);

/* 4-clique with MinHash / KMV providers (mining.py:133-154 driving
 * MinHashProvider.with_set / KmvProvider.with_set, providers.py:234-241,
 * 303-307): for each directed edge j (edge_ids[j] when edge_ids is not
 * NULL) C3 = N+u & N+v exactly; the member sketch of C3 (build_khash /
 * build_onehash / build_kmv, sketches.py:201-237) is built once per edge and
 * every w in C3 adds est_intersection_minhash / est_intersection_kmv
 * (estimators.py:157-200) of (sketch(w), member sketch, sizes[w], |C3|).
 * kind = PG_KHASH | PG_ONEHASH | PG_KMV; rows = int32 entries (k-Hash /
 * 1-Hash) or double values (KMV), k columns; lengths: 1-Hash / KMV stored
 * lengths (NULL for k-Hash); seeds_dev: k (k-Hash) or 1 seeds.
 * out_sum[0] = sum of the per-triple estimates (fp64, fixed reduction
 * order: reproducible), out_triples[0] = number of (u,v,w) triples.
 * max_out_degree bounds |N+| over the view (C3 scratch for long lists);
 * the caller allocates `workspace` of pg_4clique_sketch_workspace_size
 * bytes (k > 256: the member sketch and the 1-Hash member table are in the
 * workspace too). */
PG_API int pg_4clique_sketch_workspace_size(int32_t kind, int32_t k,
                     int64_t max_out_degree, size_t* bytes);
PG_API int pg_4clique_sketch(int32_t kind, const int64_t* dir_off,
                     const int32_t* dir_adj, const int32_t* src,
                     const int64_t* edge_ids, int64_t e_begin, int64_t e_end,
                     const void* rows, const int32_t* lengths,
                     const int32_t* sizes, int32_t k, const uint64_t* seeds_dev,
                     int64_t max_out_degree, void* workspace,
                     size_t workspace_bytes, double* out_sum,
                     int64_t* out_triples, void* stream);

/* Scalar with_set (providers.py:164-175, 234-241, 303-307): the estimate
 * of |S_w & members| for vertex w and an explicit member set in one
 * one-warp launch (the member sketch is built in shared memory with the
 * per-set builders' semantics, sketches.py:187-237).  kind = PG_BF_AND |
 * PG_BF_L | PG_BF_OR (rows: uint64 Bloom rows of `width` bits, hash_count
 * functions, lut: the Swamidass table; NULL for BF_L) or PG_KHASH |
 * PG_ONEHASH (int32 entry rows) | PG_KMV (double value rows), width = k;
 * lengths: 1-Hash / KMV stored lengths.  members: the caller's `count`
 * IDs sorted ascending, repeats kept (the reference builders see them:
 * build_onehash keeps repeats and intersect_merge counts them; `count` is
 * len(members) in the estimates).  out[0] = the estimate.  members and out may be pinned mapped host
 * memory.  PG_ERR_UNSUPPORTED beyond 2048 members, 65,536 bits or k = 256
 * (callers then build the member sketch with the batch builders). */
PG_API int pg_with_set(int32_t kind, const void* rows, const int32_t* lengths,
                     const int32_t* sizes, int32_t width, int32_t hash_count,
                     const uint64_t* seeds_dev, const double* lut, int32_t w,
                     const int32_t* members, int32_t count, double* out,
                     void* stream);

/* Jarvis-Patrick clustering tail (mining.py:213-245): edge i = (us[i],
 * vs[i]) is kept iff scores[i] > tau; out[0] = kept edges, out[1] =
 * connected components of the kept-edge graph (ClusterResult.cluster_count),
 * out[2] = vertices touched by a kept edge (singleton_count = n - out[2]);
 * keep_out (nullable) receives each edge's 0/1 keep flag */
PG_API int pg_jp_components(const int32_t* us, const int32_t* vs,
                     const double* scores, int64_t count, double tau,
                     int64_t n, uint8_t* keep_out, int64_t* out, void* stream);

/* degree ordering (graphs.py:154-166 degree_order): rank[v] = position of
 * (degree(v), v) in ascending order; the directed CSR keeps x in N+(v) iff
 * rank[v] < rank[x], adjacency order preserved.  dir_off: n+1 entries,
 * dir_adj: nnz/2 entries (each undirected edge once; nnz must be even). */
PG_API int pg_degree_order(const int64_t* offsets, const int32_t* adj, int64_t n,
                     int64_t nnz, int32_t* rank, int64_t* dir_off,
                     int32_t* dir_adj, void* stream);
/* The transpose of pg_degree_order's lists from its ranks: x in N-(v) iff
 * rank[x] < rank[v]; in_off n+1 entries, in_adj nnz/2 entries. */
PG_API int pg_degree_in_lists(const int64_t* offsets, const int32_t* adj, int64_t n,
                     int64_t nnz, const int32_t* rank, int64_t* in_off,
                     int32_t* in_adj, void* stream);

/* ---- link prediction (mining.py:248-331) ---------
 * two-hop candidates (_two_hop_candidates, :275-296): keys u*n+v (u < v),
 * ascending, of non-adjacent pairs with a common neighbour.  keys_out NULL:
 * *count_host = sum over w of C(deg w, 2), the capacity keys_out needs. */
PG_API int pg_two_hop_candidates(const int64_t* offsets, const int32_t* adj,
                     int64_t n, uint64_t* keys_out, int64_t capacity,
                     int64_t* count_host, void* stream);
/* vertex_similarity (:162-203) of every candidate.  measure: 0 JACCARD,
 * 1 OVERLAP, 2 COMMON_NEIGHBORS, 3 TOTAL_NEIGHBORS (from est[i], the
 * provider's pair estimate), 4 ADAMIC_ADAR, 5 RESOURCE_ALLOCATION (members
 * from member_source 0 = CSR rows (rows = adj), 1 = 1-Hash entries [n][k]
 * + lengths, 2 = k-Hash entries [n][k]; term[d] = the per-member term of a
 * degree-d member, summed in ascending member order) */
PG_API int pg_similarity_scores(int32_t measure, const uint64_t* keys,
                     int64_t count, int64_t n, const int64_t* offsets,
                     const double* est, int32_t member_source,
                     const int32_t* rows, int32_t k, const int32_t* lengths,
                     const double* term, double* scores, void* stream);
/* link_prediction_eval's tail (:320-331): rank by (-score, u, v), take the
 * first min(top, count), count those in removed_sorted -> out_hits[0] */
PG_API int pg_rank_top_hits(const uint64_t* keys, const double* scores,
                     int64_t count, int64_t top,
                     const uint64_t* removed_sorted, int64_t n_removed,
                     int64_t* out_hits, void* stream);

/* exact |N(u) & N(v)| per pair over a sorted CSR (providers.py:102-115
 * ExactProvider.pair_many; setops.py:23-51) */
/* sum over the edges (us[e], vs[e]) of |N(u) & N(v)| in the CSR -- the
 * exact triangle count of a degree-ordered view (mining.py:88-102
 * triangle_count with the exact provider) without per-edge outputs */
PG_API int pg_tc_exact(const int64_t* offsets, const int32_t* adj, const int32_t* us,
                const int32_t* vs, int64_t count, int64_t* out_sum, void* stream);
PG_API int pg_pairs_exact(const int64_t* offsets, const int32_t* adj,
                   const int32_t* us, const int32_t* vs, int64_t count,
                   int64_t* out_count, void* stream);

/* ---- graph generation (SURVEY 8(f) "next"; graphs.py:251-276) -------
 * numpy default_rng(seed) == PCG64; (state, inc) are the 128-bit values of
 * rng.bit_generator.state captured before the first draw. */
/* R-MAT pairs, bit-identical to generate_kronecker's two rng.random(count)
 * draws per level (a, b, c = initiator probabilities) */
PG_API int pg_rmat_pairs(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi,
                  uint64_t inc_lo, int32_t scale, int64_t count, double a,
                  double b, double c, int64_t* src, int64_t* dst, void* stream);
/* draws [offset, offset+count) of rng.random() */
PG_API int pg_pcg64_uniform(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi,
                     uint64_t inc_lo, int64_t offset, int64_t count,
                     double* out, void* stream);
/* np.searchsorted(cdf, u, "right") clipped to n-1 */
PG_API int pg_searchsorted_right(const double* cdf, int64_t n, const double* u,
                          int64_t count, int64_t* out, void* stream);
/* CsrGraph.from_edges on the device (graphs.py:57-89): drop loops,
 * deduplicate, symmetrise; offsets int64[n+1], adj int32[capacity];
 * nnz_host receives 2m (host sync) */
PG_API int pg_csr_from_pairs(const int64_t* a, const int64_t* b, int64_t count,
                      int64_t n, int64_t* offsets, int32_t* adj,
                      int64_t capacity, int64_t* nnz_host, void* stream);

/* ---- utilities ------------------------------------------------------- */
/* writes `bytes` bytes to a scratch buffer (L2 flush between timed runs) */
PG_API int pg_l2_flush(void* buf, size_t bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* PROBGRAPH_B200_H */
