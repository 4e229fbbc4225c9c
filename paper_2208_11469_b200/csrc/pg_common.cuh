// Shared device helpers for the per-edge sketch-intersection engine.
// Hash family: reference hashing.py:43-75 (mix64 constants and finalizer).
#pragma once
#include <cstdint>
#include <cstddef>
#include <cuda_runtime.h>

#include "../../include/probgraph_b200.h"

namespace pg {

constexpr uint64_t kC1 = 0xFF51AFD7ED558CCDull;
constexpr uint64_t kC2 = 0xC4CEB9FE1A85EC53ull;

// multiplicative inverse of an odd 64-bit constant (Newton iteration)
__host__ __device__ constexpr uint64_t inv_odd(uint64_t a) {
  uint64_t x = a;  // correct to 3 bits for odd a
  x *= 2 - a * x;
  x *= 2 - a * x;
  x *= 2 - a * x;
  x *= 2 - a * x;
  x *= 2 - a * x;
  return x;
}
constexpr uint64_t kC1inv = inv_odd(kC1);
constexpr uint64_t kC2inv = inv_odd(kC2);
static_assert(kC1 * kC1inv == 1ull, "inverse");
static_assert(kC2 * kC2inv == 1ull, "inverse");

// 64-bit avalanche finalizer (hashing.py:56-75)
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x ^= x >> 33;
  x *= kC1;
  x ^= x >> 33;
  x *= kC2;
  x ^= x >> 33;
  return x;
}
// inverse of mix64 (x ^= x>>33 is an involution because 33 >= 32)
__host__ __device__ __forceinline__ uint64_t unmix64(uint64_t x) {
  x ^= x >> 33;
  x *= kC2inv;
  x ^= x >> 33;
  x *= kC1inv;
  x ^= x >> 33;
  return x;
}

// word(i, key) = mix64(seed_i ^ uint64(key))  (hashing.py:114-118);
// keys are vertex IDs (non-negative int32), whose int64 -> uint64 cast is a
// zero extension: the high word of seed_i ^ key is seed_i's, which the
// compiler hoists out of the neighbour loops
__device__ __forceinline__ uint64_t hash_word(uint64_t seed, int32_t key) {
  return mix64(seed ^ static_cast<uint64_t>(static_cast<uint32_t>(key)));
}

// unit value (word+1)*2^-64 in (0,1]; all-ones word -> 1.0 (hashing.py:148-153).
// __ull2double_rn rounds to nearest-even like numpy's uint64->float64 cast.
__device__ __forceinline__ double unit_value(uint64_t w) {
  if (w == ~0ull) return 1.0;
  return __dmul_rn(__ull2double_rn(w + 1ull), 0x1p-64);
}

__device__ __forceinline__ uint64_t dbits(double d) {
  return static_cast<uint64_t>(__double_as_longlong(d));
}
__device__ __forceinline__ double bitsd(uint64_t b) {
  return __longlong_as_double(static_cast<long long>(b));
}

constexpr uint64_t kInfBits = 0x7FF0000000000000ull;

__device__ __forceinline__ uint64_t shfl64(uint64_t v, int src, unsigned mask = 0xffffffffu) {
  return __shfl_sync(mask, v, src);
}
__device__ __forceinline__ uint64_t shfl_up64(uint64_t v, int d) {
  return __shfl_up_sync(0xffffffffu, v, d);
}

// streaming 128-bit read-only load that does not allocate in L1
__device__ __forceinline__ uint4 ldg_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ uint4 ldg_keep(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// ------------------------------------------------------------------ errors
void set_error(const char* fmt, ...);
int fail(int code, const char* fmt, ...);
int check_launch(const char* what);
int sm_count();
void retain_default_pool();

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

constexpr int kMaxSketchK = 256;       // device 1-Hash/KMV/k-Hash capacity limit
constexpr int kMaxBloomBits = 65536;   // Bloom width limit (smem row per warp)

}  // namespace pg

#define PG_REQUIRE(cond, ...)                                  \
  do {                                                         \
    if (!(cond)) return ::pg::fail(PG_ERR_INVALID, __VA_ARGS__); \
  } while (0)
