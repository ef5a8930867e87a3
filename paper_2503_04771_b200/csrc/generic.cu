// bgx_generic — the reference's linalg.generic loop nest on the GPU with the
// reference's exact arithmetic (bridgegen interp.py:372-424, body from
// einsum.py:100-118, scalar semantics interp.py:260-274).
//
// One thread owns one output element (the parallel axes come first in the
// reference's axis order, einsum.py:81, so each output element is produced by
// one contiguous run of the reduction sub-space).  The thread walks that
// sub-space in the same lexicographic order with an odometer, forms
// p = x1 * x2 * ... (left fold) and acc = p + acc with __fmul_rn/__fadd_rn
// (no FMA contraction, no flush-to-zero), so every output is bit-identical to
// the reference.  bf16/f16 operands (the DSL extension)
// use the tensor-core path's semantics: values are widened to f32, the same
// loop runs in f32 with per-op rounding, and the result is rounded once to the
// storage type (round-to-nearest-even).  This is the kernel for bodies the GEMM planner does not map
// (single-input reductions, Hadamard/outer products, 3+-operand patterns,
// rank-0 outputs) and for fp32 parity runs.
#include "common.cuh"

namespace bgx {
namespace {

template <typename T> __device__ __forceinline__ T mul_rn(T a, T b);
template <> __device__ __forceinline__ float mul_rn<float>(float a, float b) { return __fmul_rn(a, b); }
template <> __device__ __forceinline__ double mul_rn<double>(double a, double b) { return __dmul_rn(a, b); }
template <typename T> __device__ __forceinline__ T add_rn(T a, T b);
template <> __device__ __forceinline__ float add_rn<float>(float a, float b) { return __fadd_rn(a, b); }
template <> __device__ __forceinline__ double add_rn<double>(double a, double b) { return __dadd_rn(a, b); }

// storage type S, arithmetic type T (T = S for f32/f64, float for bf16/f16)
template <typename S, typename T> __device__ __forceinline__ T ld_as(const S *p) {
  return Conv<S>::to_f(*p);
}
template <> __device__ __forceinline__ float ld_as<float, float>(const float *p) { return *p; }
template <> __device__ __forceinline__ double ld_as<double, double>(const double *p) { return *p; }
template <typename S, typename T> __device__ __forceinline__ S st_as(T v) {
  return Conv<S>::from_f(v);
}
template <> __device__ __forceinline__ float st_as<float, float>(float v) { return v; }
template <> __device__ __forceinline__ double st_as<double, double>(double v) { return v; }

// DENSE: every input is laid out exactly like the (row-major) output over the
// parallel axes and there is no reduction — the offsets are the output index.
template <typename S, typename T, int NIN, bool DENSE>
__global__ void __launch_bounds__(128)
generic_kernel(const bgx_generic_desc d, int64_t n_out, int64_t red_points) {
  const int n_in = NIN > 0 ? NIN : d.n_in;
  const int n_par = d.n_par, n_axes = d.n_axes, n_red = n_axes - n_par;
  const bool passthrough = (n_in == 1 && n_red == 0);
  const bool idx32 = n_out <= 0x7fffffffLL;
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < n_out;
       o += (int64_t)gridDim.x * blockDim.x) {
    int64_t off[BGX_MAX_OPERANDS];
#pragma unroll
    for (int k = 0; k < BGX_MAX_OPERANDS; ++k) off[k] = DENSE ? o : 0;
    if (!DENSE) {
      if (idx32) {   // 32-bit index arithmetic: the divisions dominate elementwise bodies
        uint32_t rem = (uint32_t)o;
        for (int a = n_par - 1; a >= 0; --a) {
          const uint32_t e = (uint32_t)d.extents[a];
          const uint32_t q = rem / e, i = rem - q * e;
          rem = q;
          for (int k = 0; k < n_in; ++k) off[k] += (int64_t)i * d.strides[k][a];
        }
      } else {
        int64_t rem = o;
        for (int a = n_par - 1; a >= 0; --a) {
          const int64_t e = d.extents[a];
          const int64_t i = rem % e;
          rem /= e;
          for (int k = 0; k < n_in; ++k) off[k] += i * d.strides[k][a];
        }
      }
    }
    const S *const *ins = reinterpret_cast<const S *const *>(d.ins);
    S *out = static_cast<S *>(d.out);
    if (passthrough) {
      out[o] = ins[0][off[0]];
      continue;
    }
    // c0 == NULL: zero initial output (+0.0, as the reference's zeros array)
    T acc = d.c0 ? ld_as<S, T>(static_cast<const S *>(d.c0) + o) : T(0);
    if (red_points == 0) {
      out[o] = st_as<S, T>(acc);
      continue;
    }
    if (n_red == 0) {  // elementwise body (Hadamard / outer product): one point
      T p = ld_as<S, T>(ins[0] + off[0]);
      for (int k = 1; k < n_in; ++k) p = mul_rn<T>(p, ld_as<S, T>(ins[k] + off[k]));
      out[o] = st_as<S, T>(add_rn<T>(p, acc));
      continue;
    }
    // Innermost reduction axis: U points of every operand are loaded ahead
    // (independent loads in flight), then folded into the running sum in the
    // reference's order — same arithmetic sequence, latency hidden.
    constexpr int U = 8;
    const int ax_in = n_axes - 1;
    const int64_t E = d.extents[ax_in];
    int64_t sin[BGX_MAX_OPERANDS];
    for (int k = 0; k < n_in; ++k) sin[k] = d.strides[k][ax_in];
    const int64_t outer = red_points / E;
    int64_t idx[BGX_MAX_AXES];
    for (int a = 0; a < n_red - 1; ++a) idx[a] = 0;
    for (int64_t r = 0; r < outer; ++r) {
      int64_t j = 0;
      for (; j + U <= E; j += U) {
        T v[NIN > 0 ? NIN : BGX_MAX_OPERANDS][U];
#pragma unroll
        for (int k = 0; k < (NIN > 0 ? NIN : BGX_MAX_OPERANDS); ++k) {
          if (k >= n_in) break;
          const S *base = ins[k] + off[k] + j * sin[k];
#pragma unroll
          for (int u = 0; u < U; ++u) v[k][u] = ld_as<S, T>(base + u * sin[k]);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          T p = v[0][u];
          for (int k = 1; k < n_in; ++k) p = mul_rn<T>(p, v[k][u]);
          acc = add_rn<T>(p, acc);
        }
      }
      for (; j < E; ++j) {
        T p = ld_as<S, T>(ins[0] + off[0] + j * sin[0]);
        for (int k = 1; k < n_in; ++k) p = mul_rn<T>(p, ld_as<S, T>(ins[k] + off[k] + j * sin[k]));
        acc = add_rn<T>(p, acc);
      }
      // odometer over the outer reduction axes (last of them fastest)
      for (int a = n_red - 2; a >= 0; --a) {
        const int ax = n_par + a;
        if (++idx[a] < d.extents[ax]) {
          for (int k = 0; k < n_in; ++k) off[k] += d.strides[k][ax];
          break;
        }
        for (int k = 0; k < n_in; ++k) off[k] -= (d.extents[ax] - 1) * d.strides[k][ax];
        idx[a] = 0;
      }
    }
    out[o] = st_as<S, T>(acc);
  }
}

template <typename S, typename T, bool DENSE>
void launch_generic_n(const bgx_generic_desc &d, int64_t n_out, int64_t red, unsigned blocks,
                      cudaStream_t s) {
  switch (d.n_in) {
    case 1: generic_kernel<S, T, 1, DENSE><<<blocks, 128, 0, s>>>(d, n_out, red); break;
    case 2: generic_kernel<S, T, 2, DENSE><<<blocks, 128, 0, s>>>(d, n_out, red); break;
    case 3: generic_kernel<S, T, 3, DENSE><<<blocks, 128, 0, s>>>(d, n_out, red); break;
    default: generic_kernel<S, T, 0, DENSE><<<blocks, 128, 0, s>>>(d, n_out, red); break;
  }
}

template <typename S, typename T>
int launch_generic(const bgx_generic_desc &d, int64_t n_out, int64_t red, cudaStream_t s) {
  const int sms = sm_count_current();
  if (sms <= 0) { set_error("bgx_generic: no device"); return BGX_ERR_NO_DEVICE; }
  int64_t blocks = (n_out + 127) / 128;
  if (blocks > (int64_t)sms * 64) blocks = (int64_t)sms * 64;
  // dense elementwise: no reduction and every input strided like the
  // row-major output over the parallel axes
  bool dense = d.n_axes == d.n_par;
  for (int k = 0; k < d.n_in && dense; ++k) {
    int64_t st = 1;
    for (int a = d.n_par - 1; a >= 0 && dense; --a) {
      if (d.extents[a] != 1 && d.strides[k][a] != st) dense = false;
      st *= d.extents[a];
    }
  }
  if (dense) launch_generic_n<S, T, true>(d, n_out, red, (unsigned)blocks, s);
  else launch_generic_n<S, T, false>(d, n_out, red, (unsigned)blocks, s);
  return check_launch("generic_kernel");
}

}  // namespace
}  // namespace bgx

using namespace bgx;

extern "C" int bgx_generic(const bgx_generic_desc *d, void *stream) {
  BGX_CHECK_ARG(d != nullptr, "bgx_generic: null descriptor");
  BGX_CHECK_ARG(d->n_in >= 1 && d->n_in <= BGX_MAX_OPERANDS, "bgx_generic: n_in %d", d->n_in);
  BGX_CHECK_ARG(d->n_axes >= 0 && d->n_axes <= BGX_MAX_AXES && d->n_par >= 0 &&
                    d->n_par <= d->n_axes,
                "bgx_generic: axes %d / parallel %d", d->n_axes, d->n_par);
  BGX_CHECK_ARG(d->dtype == BGX_F32 || d->dtype == BGX_F64 || d->dtype == BGX_BF16 ||
                    d->dtype == BGX_F16,
                "bgx_generic: dtype %d", d->dtype);
  int64_t n_out = 1, red = 1;
  for (int a = 0; a < d->n_axes; ++a) {
    BGX_CHECK_ARG(d->extents[a] >= 0, "bgx_generic: negative extent");
    if (a < d->n_par) n_out *= d->extents[a]; else red *= d->extents[a];
  }
  if (n_out == 0) return BGX_OK;
  BGX_CHECK_ARG(d->out != nullptr, "bgx_generic: null out");
  // c0 == NULL means a zero initial output
  const bool passthrough = d->n_in == 1 && d->n_axes == d->n_par;
  if (red > 0 || passthrough)
    for (int k = 0; k < d->n_in; ++k) BGX_CHECK_ARG(d->ins[k] != nullptr, "bgx_generic: null input");
  cudaStream_t s = (cudaStream_t)stream;
  switch (d->dtype) {
    case BGX_F32: return launch_generic<float, float>(*d, n_out, red, s);
    case BGX_F64: return launch_generic<double, double>(*d, n_out, red, s);
    case BGX_BF16: return launch_generic<__nv_bfloat16, float>(*d, n_out, red, s);
    default: return launch_generic<__half, float>(*d, n_out, red, s);
  }
}
