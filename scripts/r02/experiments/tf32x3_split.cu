// bgx_tf32_split — operands for f32-accurate GEMMs on the tf32 tensor cores
// ("3xTF32", mode "tf32x3" of the Python API).  Each f32 value x is split
// into hi = tf32(x) and lo = tf32(x - hi) (x - hi is exact in f32), and the
// K axis is tripled so that ONE tcgen05 kind::tf32 GEMM of the split operands
// sums hi*hi + hi*lo + lo*hi for every k:
//   A' = [ hi | hi | lo ]  (segments along K of A)
//   B' = [ hi ; lo ; hi ]  (segments along K of B)
// The dropped lo*lo term is ~2^-22 of the product, so the result carries f32
// accuracy (relative error ~1e-6 against the reference's f32 loop nest,
// within the FFMA tolerance of 1e-5) at tensor-core speed.  Not the
// reference's summation order: a tolerance mode, like FFMA.
#include "common.cuh"

namespace bgx {
namespace {

__device__ __forceinline__ float to_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// k_rows = 0: K runs along the columns of src (A: rows = M, cols = K) and the
//             destination rows hold [hi | hi | lo], each segment `seg` wide;
// k_rows = 1: K runs along the rows of src (B: rows = K, cols = N) and the
//             destination holds [hi ; lo ; hi] row blocks of `seg` rows.
// Segment positions past K are zero (they pad K to 16-byte multiples).
__global__ void __launch_bounds__(256)
tf32_split_kernel(const float *__restrict__ src, int64_t batch, int64_t rows, int64_t cols,
                  int64_t sb, int64_t sr, int64_t sc, float *__restrict__ dst, int64_t db,
                  int64_t dld, int k_rows, int64_t seg) {
  const int64_t drows = k_rows ? 3 * seg : rows;
  const int64_t dcols = k_rows ? cols : 3 * seg;
  const int64_t total = batch * drows * dcols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = e % dcols;
    const int64_t t = e / dcols;
    const int64_t r = t % drows;
    const int64_t b = t / drows;
    int64_t sr_i, sc_i;
    int part;
    bool live;
    if (k_rows) {
      part = (int)(r / seg);
      const int64_t k = r - part * seg;
      sr_i = k; sc_i = c;
      live = k < rows;
      part = part == 1 ? 1 : 0;          // rows: hi, lo, hi
    } else {
      part = (int)(c / seg);
      const int64_t k = c - part * seg;
      sr_i = r; sc_i = k;
      live = k < cols;
      part = part == 2 ? 1 : 0;          // cols: hi, hi, lo
    }
    float v = 0.f;
    if (live) {
      const float x = src[b * sb + sr_i * sr + sc_i * sc];
      const float hi = to_tf32(x);
      v = part ? to_tf32(x - hi) : hi;
    }
    dst[b * db + r * dld + c] = v;
  }
}

}  // namespace
}  // namespace bgx

using namespace bgx;

extern "C" int bgx_tf32_split(const float *src, int64_t batch, int64_t rows, int64_t cols,
                              const int64_t *src_stride, float *dst, int64_t dst_batch_stride,
                              int64_t dst_ld, int32_t k_rows, int64_t seg, void *stream) {
  BGX_CHECK_ARG(src != nullptr && dst != nullptr && src_stride != nullptr,
                "bgx_tf32_split: null pointer");
  BGX_CHECK_ARG(batch >= 0 && rows >= 0 && cols >= 0, "bgx_tf32_split: negative extent");
  BGX_CHECK_ARG(k_rows == 0 || k_rows == 1, "bgx_tf32_split: k_rows must be 0 or 1");
  BGX_CHECK_ARG(seg >= (k_rows ? rows : cols), "bgx_tf32_split: segment shorter than K");
  BGX_CHECK_ARG(dst_ld >= (k_rows ? cols : 3 * seg), "bgx_tf32_split: destination row too short");
  const int64_t total = batch * (k_rows ? 3 * seg * cols : rows * 3 * seg);
  if (total == 0) return BGX_OK;
  const int sms = sm_count_current();
  if (sms <= 0) {
    set_error("bgx_tf32_split: no device");
    return BGX_ERR_NO_DEVICE;
  }
  int64_t blocks = (total + 255) / 256;
  if (blocks > (int64_t)sms * 32) blocks = (int64_t)sms * 32;
  tf32_split_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(
      src, batch, rows, cols, src_stride[0], src_stride[1], src_stride[2], dst, dst_batch_stride,
      dst_ld, k_rows, seg);
  return check_launch("tf32_split_kernel");
}
