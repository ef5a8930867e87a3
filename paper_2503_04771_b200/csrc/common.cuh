// Shared helpers for libbgx.so: error reporting, dtype utilities and the
// sm_100a PTX wrappers (mbarrier, TMA, tcgen05/TMEM) used by the kernels.
#pragma once

#include <cuda_runtime.h>
#include <mutex>
#include <set>
#include <utility>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdint.h>
#include <stdio.h>
#include <stdarg.h>

#include "../../include/bgx.h"

namespace bgx {

// ---------------------------------------------------------------------------
// Errors: thread-local last message, negative status codes (bgx.h)

void set_error(const char *fmt, ...);

#define BGX_CHECK_ARG(cond, ...)                                              \
  do {                                                                        \
    if (!(cond)) { ::bgx::set_error(__VA_ARGS__); return BGX_ERR_INVALID; }   \
  } while (0)

#define BGX_CUDA_TRY(expr)                                                    \
  do {                                                                        \
    cudaError_t _e = (expr);                                                  \
    if (_e != cudaSuccess) {                                                  \
      ::bgx::set_error("%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e), \
                       __FILE__, __LINE__);                                   \
      return BGX_ERR_CUDA;                                                    \
    }                                                                         \
  } while (0)

// Launch-error check (asynchronous faults surface at the caller's sync).
inline int check_launch(const char *what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s launch failed: %s", what, cudaGetErrorString(e));
    return BGX_ERR_CUDA;
  }
  return BGX_OK;
}

inline int dtype_size(int32_t dt) {
  switch (dt) {
    case BGX_F32: return 4;
    case BGX_F64: return 8;
    case BGX_BF16: return 2;
    case BGX_F16: return 2;
    default: return 0;
  }
}

int sm_count_current();  // cached per device

// ---------------------------------------------------------------------------
// Scalar conversions (device)

template <typename T> struct Conv;
template <> struct Conv<float> {
  __device__ static float to_f(float v) { return v; }
  __device__ static float from_f(float v) { return v; }
};
template <> struct Conv<double> {
  __device__ static float to_f(double v) { return (float)v; }
  __device__ static double from_f(float v) { return (double)v; }
};
template <> struct Conv<__nv_bfloat16> {
  __device__ static float to_f(__nv_bfloat16 v) { return __bfloat162float(v); }
  __device__ static __nv_bfloat16 from_f(float v) { return __float2bfloat16_rn(v); }
};
template <> struct Conv<__half> {
  __device__ static float to_f(__half v) { return __half2float(v); }
  __device__ static __half from_f(float v) { return __float2half_rn(v); }
};

// Two f32 -> packed 16-bit pair (lo in bits 0-15), round-to-nearest-even.
template <typename H> __device__ __forceinline__ uint32_t pack2(float lo, float hi);
template <> __device__ __forceinline__ uint32_t pack2<__nv_bfloat16>(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
template <> __device__ __forceinline__ uint32_t pack2<__half>(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

// ---------------------------------------------------------------------------
// PTX wrappers (sm_100a)

// One-time kernel setup (cudaFuncSetAttribute, occupancy queries) may first
// run while the caller's stream is being captured into a CUDA graph; those
// calls are not stream work, so switch this thread to relaxed capture mode
// around them instead of invalidating the caller's capture.
struct RelaxedCaptureScope {
  cudaStreamCaptureMode mode = cudaStreamCaptureModeRelaxed;
  RelaxedCaptureScope() { cudaThreadExchangeStreamCaptureMode(&mode); }
  ~RelaxedCaptureScope() { cudaThreadExchangeStreamCaptureMode(&mode); }
};

// cudaFuncAttributeMaxDynamicSharedMemorySize = `bytes` for `kern` on the
// current device, set once per (kernel, device) (capture-safe).
inline void set_max_smem_once(const void *kern, int bytes) {
  static std::mutex mu;
  static std::set<std::pair<const void *, int>> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  if (done.insert({kern, dev}).second) {
    RelaxedCaptureScope relaxed;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  }
}

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Arrive on the barrier at the same smem offset in CTA `cta` of the cluster.
__device__ __forceinline__ void mbar_arrive_cluster(uint64_t *bar, uint32_t cta) {
  asm volatile(
      "{\n\t.reg .b32 remAddr32;\n\t"
      "mapa.shared::cluster.u32  remAddr32, %0, %1;\n\t"
      "mbarrier.arrive.release.cluster.shared::cluster.b64  _, [remAddr32];\n\t}"
      ::"r"(smem_u32(bar)), "r"(cta) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
               ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

// The suspend-time hint lets a waiting warp sleep in hardware until the
// phase completes (bounded by the hint, in ns) instead of re-polling: fewer
// issued instructions while the pipeline is full, i.e. less power for the
// same work on a power-capped part.
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "BGX_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
      "@!P1 bra BGX_WAIT_%=;\n\t}"
      ::"r"(smem_u32(bar)), "r"(parity), "r"(0x989680u) : "memory");
}

__device__ __forceinline__ void prefetch_tmap(const void *tmap) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(tmap) : "memory");
}

// 3-D tiled TMA load global -> shared, completing bytes on `bar`.
__device__ __forceinline__ void tma_load_3d(void *dst, const void *tmap, uint64_t *bar,
                                            int32_t c0, int32_t c1, int32_t c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];"
      ::"r"(smem_u32(dst)), "l"(tmap), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

// 2-CTA variant: the completion is signalled on the barrier of the leader CTA
// (peer-bit cleared address); used with cta_group::2 so both CTAs' halves
// land on one barrier.
__device__ __forceinline__ void tma_load_3d_cg2(void *dst, const void *tmap, uint64_t *bar,
                                                int32_t c0, int32_t c1, int32_t c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];"
      ::"r"(smem_u32(dst)), "l"(tmap), "r"(smem_u32(bar) & 0xFEFFFFFFu), "r"(c0), "r"(c1),
        "r"(c2)
      : "memory");
}

// 2-CTA load multicast to the CTAs in `mask` (same smem offset in each);
// the mbarrier address has the peer bit cleared, so every destination's
// transaction bytes land on ITS pair leader's barrier.
__device__ __forceinline__ void tma_load_3d_cg2_mc(void *dst, const void *tmap, uint64_t *bar,
                                                   int32_t c0, int32_t c1, int32_t c2,
                                                   uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      ".multicast::cluster [%0], [%1, {%3, %4, %5}], [%2], %6;"
      ::"r"(smem_u32(dst)), "l"(tmap), "r"(smem_u32(bar) & 0xFEFFFFFFu), "r"(c0), "r"(c1),
        "r"(c2), "h"(mask)
      : "memory");
}

// One lane of the (fully active) warp returns true; warp-uniform control flow
// around it lets ptxas keep loop state in uniform registers.
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}"
      : "=r"(pred));
  return pred != 0;
}

// 3-D tiled TMA store shared -> global (bulk-group completion).
__device__ __forceinline__ void tma_store_3d(const void *tmap, const void *src, int32_t c0,
                                             int32_t c1, int32_t c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];"
      ::"l"(tmap), "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2) : "memory");
}
__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
// Wait until at most N committed bulk groups still READ shared memory.
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\t"
               "barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// Named barrier over a subset of the CTA's warps (id 0 is __syncthreads).
__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Loads of data another CTA / another GPU wrote in this kernel: relaxed at
// system scope (never served from a stale L1 line; peer addresses go over
// NVLink).
__device__ __forceinline__ float4 ld_sys_v4(const float *p) {
  float4 v;
  asm volatile("ld.relaxed.sys.global.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p)
               : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ float ld_sys(const float *p) {
  float v;
  asm volatile("ld.relaxed.sys.global.f32 %0, [%1];" : "=f"(v) : "l"(p) : "memory");
  return v;
}

// ---- tcgen05 / TMEM ---------------------------------------------------------

template <int CG>
__device__ __forceinline__ void tmem_alloc(uint32_t *slot, uint32_t ncols) {
  if constexpr (CG == 1)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 ::"r"(smem_u32(slot)), "r"(ncols));
  else
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;"
                 ::"r"(smem_u32(slot)), "r"(ncols));
}
template <int CG>
__device__ __forceinline__ void tmem_relinquish() {
  if constexpr (CG == 1)
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  else
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
}
template <int CG>
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  if constexpr (CG == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols));
  else
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols));
}

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// D[tmem] (+)= A[smem] * B[smem], kind::f16 (bf16/f16 in, f32 accumulate).
template <int CG>
__device__ __forceinline__ void umma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                         uint32_t idesc, uint32_t accumulate) {
  if constexpr (CG == 1)
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
        ::"r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
  else
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}"
        ::"r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// kind::tf32 (fp32 storage, tf32 multiply, f32 accumulate); K = 8 per MMA.
template <int CG>
__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                          uint32_t idesc, uint32_t accumulate) {
  if constexpr (CG == 1)
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
        ::"r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
  else
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
        ::"r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

template <int CG, int IN_BYTES>
__device__ __forceinline__ void umma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                     uint32_t idesc, uint32_t accumulate) {
  if constexpr (IN_BYTES == 4) umma_tf32<CG>(tmem_d, adesc, bdesc, idesc, accumulate);
  else umma_f16<CG>(tmem_d, adesc, bdesc, idesc, accumulate);
}

// Signal `bar` when all previously issued tcgen05.mma of this thread retire.
__device__ __forceinline__ void umma_commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
               ::"r"(smem_u32(bar)) : "memory");
}
// 2-CTA: arrive on the barrier at this smem offset in every CTA of `mask`.
__device__ __forceinline__ void umma_commit_mc(uint64_t *bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)), "h"(mask) : "memory");
}

// 32 lanes x 32 bit, 32 consecutive columns per thread.
__device__ __forceinline__ void tmem_ld_32x32b_x32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
        "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
        "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// ---- UMMA descriptors -------------------------------------------------------
// Shared-memory matrix descriptor (sm_100): start>>4 [0,14), LBO>>4 [16,30),
// SBO>>4 [32,46), version=1 [46,48), base_offset [49,52), layout [61,64)
// with SWIZZLE_128B = 2.  Unit-tested on the host by tests/test_descriptors.py.
__host__ __device__ __forceinline__ uint64_t make_sdesc_sw128(uint32_t saddr, uint32_t lbo,
                                                              uint32_t sbo, uint32_t layout = 2) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)(layout & 7u) << 61;   // 2 = SWIZZLE_128B, 1 = SWIZZLE_128B_BASE32B
  return d;
}

// Instruction descriptor, kind::f16: c_format F32 [4,6)=1; a/b format [7,10)
// [10,13) (0 = F16, 1 = BF16); a_major [15], b_major [16] (1 = MN-major);
// N>>3 [17,23); M>>4 [24,29).
__host__ __device__ __forceinline__ uint32_t make_idesc_f16(bool bf16, bool a_mn_major,
                                                            bool b_mn_major, uint32_t M,
                                                            uint32_t N) {
  uint32_t fmt = bf16 ? 1u : 0u;
  uint32_t d = 0;
  d |= 1u << 4;
  d |= fmt << 7;
  d |= fmt << 10;
  d |= (a_mn_major ? 1u : 0u) << 15;
  d |= (b_mn_major ? 1u : 0u) << 16;
  d |= ((N >> 3) & 0x3Fu) << 17;
  d |= ((M >> 4) & 0x1Fu) << 24;
  return d;
}

// kind::tf32 instruction descriptor: a/b format TF32 = 2, otherwise as f16.
__host__ __device__ __forceinline__ uint32_t make_idesc_tf32(bool a_mn_major, bool b_mn_major,
                                                             uint32_t M, uint32_t N) {
  uint32_t d = 0;
  d |= 1u << 4;
  d |= 2u << 7;
  d |= 2u << 10;
  d |= (a_mn_major ? 1u : 0u) << 15;
  d |= (b_mn_major ? 1u : 0u) << 16;
  d |= ((N >> 3) & 0x3Fu) << 17;
  d |= ((M >> 4) & 0x1Fu) << 24;
  return d;
}

// Drop extent-1 axes and merge neighbouring axes of the same kind (parallel
// with parallel, reduction with reduction) that every input walks as one:
// stride[a] == extent[a+1] * stride[a+1].  The output is dense row-major over
// the parallel axes, so merging them never changes an output address, and a
// merged reduction axis visits the points in the same order — the reference's
// loop nest, bit for bit.  (d,b,a)->(a) with (d,b) contiguous becomes a
// single-axis column reduction and takes colchain_kernel (exact) or the
// column tree layout (tolerance mode); BGX_NO_COALESCE=1 for A/B.
inline bgx_generic_desc coalesce_axes(const bgx_generic_desc &d) {
  static const bool off = getenv("BGX_NO_COALESCE") != nullptr;
  if (off) return d;
  for (int a = 0; a < d.n_axes; ++a)
    if (d.extents[a] == 0) return d;
  bgx_generic_desc w = d;
  int n = 0, n_par = 0;
  for (int a = 0; a < d.n_axes; ++a) {
    const bool par = a < d.n_par;
    if (d.extents[a] == 1) continue;
    // merge into the previous kept axis when it is the same kind and contiguous with this one
    if (n > 0 && (par == (n - 1 < n_par))) {
      bool ok = true;
      for (int k = 0; k < d.n_in && ok; ++k) ok = w.strides[k][n - 1] == d.extents[a] * d.strides[k][a];
      if (ok) {
        w.extents[n - 1] *= d.extents[a];
        for (int k = 0; k < d.n_in; ++k) w.strides[k][n - 1] = d.strides[k][a];
        continue;
      }
    }
    w.extents[n] = d.extents[a];
    for (int k = 0; k < d.n_in; ++k) w.strides[k][n] = d.strides[k][a];
    ++n;
    if (par) ++n_par;
  }
  if (n == 0) return d;
  if (n == n_par && d.n_axes > d.n_par) {
    // every reduction axis had extent 1: keep one, so the body still adds
    // its single point to c0 (a one-input body without reduction axes is a
    // plain copy)
    w.extents[n] = 1;
    for (int k = 0; k < d.n_in; ++k) w.strides[k][n] = 0;
    ++n;
  }
  w.n_axes = n;
  w.n_par = n_par;
  return w;
}

}  // namespace bgx
