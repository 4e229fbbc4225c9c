// Error plumbing, device queries and small utilities of the C ABI.
#include <cstdarg>
#include <cstdio>
#include <cstring>

#include "pg_common.cuh"

namespace pg {

__global__ void fixed_order_sum_kernel(const double* __restrict__ part, int64_t n, double* out) {
  __shared__ double red[256];
  double a = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) a = __dadd_rn(a, part[i]);
  red[threadIdx.x] = a;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) red[threadIdx.x] = __dadd_rn(red[threadIdx.x], red[threadIdx.x + w]);
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = red[0];
}


static thread_local char g_err[512] = {0};

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(PG_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
  return PG_OK;
}

int sm_count() {
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms > 0 ? sms : 148;
}

__global__ void l2_flush_kernel(uint4* buf, size_t n16, uint32_t salt) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i < n16; i += stride) buf[i] = make_uint4(salt, (uint32_t)i, salt, 0u);
}

__global__ void family_seeds_kernel(uint64_t base, int32_t count, uint64_t* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < count) out[i] = mix64(base ^ mix64(static_cast<uint64_t>(i) + 1ull));
}

// Scratch allocations (cudaMallocAsync) come from the device's default pool;
// keep its memory across synchronisations instead of releasing it at every
// sync point and mapping it again on the next call.
void retain_default_pool() {
  static bool done[64] = {false};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64 || done[dev]) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t keep = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  done[dev] = true;
}

}  // namespace pg

extern "C" {

int pg_abi_version(void) { return PG_ABI_VERSION; }

int pg_last_error(char* buf, size_t len) {
  if (!buf || len == 0) return PG_ERR_INVALID;
  strncpy(buf, pg::g_err, len - 1);
  buf[len - 1] = 0;
  return PG_OK;
}

int pg_device_sm_count(int* out_host) {
  if (!out_host) return pg::fail(PG_ERR_INVALID, "null output");
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return pg::fail(PG_ERR_CUDA, "cudaGetDevice: %s", cudaGetErrorString(e));
  e = cudaDeviceGetAttribute(out_host, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return pg::fail(PG_ERR_CUDA, "attribute: %s", cudaGetErrorString(e));
  return PG_OK;
}

int pg_family_seeds(uint64_t base, int32_t count, uint64_t* out_host) {
  if (count < 1) return pg::fail(PG_ERR_INVALID, "hash family needs at least one function");
  if (!out_host) return pg::fail(PG_ERR_INVALID, "null output");
  for (int32_t i = 0; i < count; ++i)
    out_host[i] = pg::mix64(base ^ pg::mix64(static_cast<uint64_t>(i) + 1ull));
  return PG_OK;
}

int pg_family_seeds_device(uint64_t base, int32_t count, uint64_t* out_dev, void* stream) {
  if (count < 1) return pg::fail(PG_ERR_INVALID, "hash family needs at least one function");
  if (!out_dev) return pg::fail(PG_ERR_INVALID, "null output");
  pg::family_seeds_kernel<<<(count + 127) / 128, 128, 0, pg::as_stream(stream)>>>(base, count, out_dev);
  return pg::check_launch("family_seeds");
}

int pg_l2_flush(void* buf, size_t bytes, void* stream) {
  if (!buf) return pg::fail(PG_ERR_INVALID, "null buffer");
  static uint32_t salt = 1;
  size_t n16 = bytes / 16;
  if (n16 == 0) return PG_OK;
  pg::l2_flush_kernel<<<pg::sm_count() * 4, 512, 0, pg::as_stream(stream)>>>(
      reinterpret_cast<uint4*>(buf), n16, salt++);
  return pg::check_launch("l2_flush");
}

}  // extern "C"
