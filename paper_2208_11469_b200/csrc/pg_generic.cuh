// Generic device paths for sketch sizes outside the tuned engines' ranges
// (Bloom rows wider than the shared-memory builders / histograms, k > 256):
// plan_budget (sketches.py:115-138) sizes B = s*(n+2m)/n*64 bits and
// k = s*2m/n, so dense graphs reach them.  Simpler and slower than the
// tuned kernels, same integers and the same IEEE expressions.
#pragma once
#include "pg_engines.cuh"

namespace pg {

constexpr int kGenBloomTcBits = 32768;  // wider rows: global histogram

int gen_build_bloom(const int64_t* off, const int32_t* adj, int64_t n, int bits, int b, const uint64_t* seeds,
                    uint64_t* rows, int32_t* ones, cudaStream_t s);
int gen_build_khash(const int64_t* off, const int32_t* adj, int64_t n, int k, const uint64_t* seeds,
                    int32_t* entries, cudaStream_t s);
// 1-Hash (values == nullptr) or KMV (entries == nullptr; ranks / rank_of
// nullable) bottom-k rows for any k, by a warp radix select of h_0(x)
int gen_build_bottomk(const int64_t* off, const int32_t* adj, int64_t n, int k, const uint64_t* seeds,
                      int32_t* entries, double* values, int32_t* ranks, const int32_t* rank_of,
                      int32_t* lengths, cudaStream_t s);

int gen_pairs_minhash(const int32_t* ent, int k, bool onehash, const int32_t* sizes, const int32_t* us,
                      const int32_t* vs, int64_t count, int32_t* out_count, double* out_est, cudaStream_t s);
// outputs zeroed by the caller; slots with vs < 0 are padding
int gen_tc_minhash(const int32_t* ent, int k, bool onehash, const int32_t* sizes, const int32_t* us,
                   const int32_t* vs, int64_t b, int64_t e, int64_t* out_cnt, int64_t* out_ssum,
                   int64_t* out_verbatim, cudaStream_t s);
int gen_jaccard_khash(const int32_t* ent, int k, const int32_t* deg, const int32_t* us, const int32_t* vs,
                      int64_t b, int64_t e, int min_matches, double tau, int64_t* out_counts, cudaStream_t s);
int gen_pairs_kmv(const uint64_t* vals, int k, const int32_t* sizes, const int32_t* us, const int32_t* vs,
                  int64_t count, int32_t* out_common, int32_t* out_union, double* out_kth, double* out_est,
                  cudaStream_t s);
int gen_tc_kmv(const uint64_t* vals, int k, const int32_t* sizes, const int32_t* us, const int32_t* vs,
               int64_t b, int64_t e, double* out_sum, cudaStream_t s);
int gen_tc_bloom(const uint64_t* rows, int bits, int op, const int32_t* sizes, const double* lut,
                 const int32_t* us, const int32_t* vs, int64_t b, int64_t e, int64_t* out_hist,
                 int64_t* out_sum_pos, cudaStream_t s);
int gen_4clique_bloom(const int64_t* off, const int32_t* adjp, const int32_t* src, const int64_t* edge_ids,
                      int64_t b, int64_t e, const uint64_t* rows, int bits, int nh, const uint64_t* seeds, int op,
                      const int32_t* sizes, const double* lut, int64_t* out_hist, int64_t* out_sum_pos,
                      int64_t* out_triples, cudaStream_t s);

}  // namespace pg
