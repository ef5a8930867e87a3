// Library-level C ABI: version, thread-local error text, device queries and
// the small elementwise helper used by the multi-GPU K-split path.
#include "common.cuh"

#include <mutex>
#include <string.h>

namespace bgx {

static thread_local char g_last_error[512] = "";

void set_error(const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
  va_end(ap);
}

int sm_count_current() {
  static std::mutex mu;
  static int cache[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return BGX_ERR_NO_DEVICE;
  if (dev < 0 || dev >= 64) return BGX_ERR_NO_DEVICE;
  std::lock_guard<std::mutex> lk(mu);
  if (cache[dev] == 0) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
      return BGX_ERR_NO_DEVICE;
    cache[dev] = n;
  }
  return cache[dev];
}

template <typename OutT>
__global__ void cast_f32_kernel(const float *__restrict__ src, const OutT *__restrict__ c0,
                                OutT *__restrict__ out, int64_t n) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t step = (int64_t)gridDim.x * blockDim.x;
  for (; i < n; i += step) {
    float v = src[i];
    if (c0) v = __fadd_rn(v, Conv<OutT>::to_f(c0[i]));
    out[i] = Conv<OutT>::from_f(v);
  }
}

// One CTA per SM (the dynamic shared memory request forces it): record
// (smid, %clock64, %globaltimer).  Two samples around a timed region give
// each SM's average clock over it — the in-band measurement of the clock the
// work actually ran at (NVML's clock reading is refreshed too slowly for a
// region of ~100 ms).
__global__ void clock_sample_kernel(uint64_t *out) {
  if (threadIdx.x != 0) return;
  uint32_t smid;
  uint64_t clk, ns;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(clk));
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns));
  out[blockIdx.x * 3 + 0] = smid;
  out[blockIdx.x * 3 + 1] = clk;
  out[blockIdx.x * 3 + 2] = ns;
}

}  // namespace bgx

using namespace bgx;

extern "C" {

int bgx_version(void) { return BGX_VERSION; }

const char *bgx_last_error(void) { return g_last_error; }

int bgx_sm_count(void) {
  int n = sm_count_current();
  if (n < 0) set_error("no CUDA device");
  return n;
}

int bgx_cast_f32(const float *src, const void *c0, void *out, int32_t out_dtype, int64_t n,
                 void *stream) {
  BGX_CHECK_ARG(n >= 0, "bgx_cast_f32: negative n");
  if (n == 0) return BGX_OK;
  BGX_CHECK_ARG(src && out, "bgx_cast_f32: null pointer");
  int sms = sm_count_current();
  if (sms <= 0) { set_error("bgx_cast_f32: no device"); return BGX_ERR_NO_DEVICE; }
  int64_t blocks = (n + 255) / 256;
  if (blocks > (int64_t)sms * 16) blocks = (int64_t)sms * 16;
  cudaStream_t s = (cudaStream_t)stream;
  switch (out_dtype) {
    case BGX_F32:
      cast_f32_kernel<float><<<(unsigned)blocks, 256, 0, s>>>(src, (const float *)c0,
                                                               (float *)out, n);
      break;
    case BGX_BF16:
      cast_f32_kernel<__nv_bfloat16><<<(unsigned)blocks, 256, 0, s>>>(
          src, (const __nv_bfloat16 *)c0, (__nv_bfloat16 *)out, n);
      break;
    case BGX_F16:
      cast_f32_kernel<__half><<<(unsigned)blocks, 256, 0, s>>>(src, (const __half *)c0,
                                                                (__half *)out, n);
      break;
    default:
      set_error("bgx_cast_f32: unsupported out dtype %d", out_dtype);
      return BGX_ERR_UNSUPPORTED;
  }
  return check_launch("cast_f32_kernel");
}

int bgx_clock_sample(uint64_t *out, void *stream) {
  BGX_CHECK_ARG(out != nullptr, "bgx_clock_sample: null output");
  const int sms = sm_count_current();
  if (sms <= 0) { set_error("bgx_clock_sample: no device"); return BGX_ERR_NO_DEVICE; }
  constexpr int SMEM = 200 * 1024;   // > half an SM's shared memory: one CTA per SM
  set_max_smem_once(reinterpret_cast<const void *>(clock_sample_kernel), SMEM);
  clock_sample_kernel<<<(unsigned)sms, 32, SMEM, (cudaStream_t)stream>>>(out);
  return check_launch("clock_sample_kernel");
}

}  // extern "C"
