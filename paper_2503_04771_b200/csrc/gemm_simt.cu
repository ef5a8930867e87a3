// CUDA-core batched strided contraction (bgx_contract modes EXACT / FFMA /
// SIMT).  Shared-memory tiled, register-blocked; any element strides.
//
// EXACT (f32/f64): each output element starts from c0 and accumulates
// fl(fl(a*b) + acc) in increasing k — precisely the reference's per-point
// body (bridgegen einsum.py:111-117 evaluated by interp.py:407-420) — so the
// result is bit-identical to the reference for 2-operand contractions with
// one (flattened, lexicographically ordered) reduction group.
// FFMA (f32): fused fma(a, b, acc); <= 1e-5 relative vs the reference.
// SIMT (bf16/f16 in, f32 accumulate): products of 16-bit values are exact in
// f32, so fma == separate rounding here: bit-identical to the reference's f32
// arithmetic on the upcast inputs; one final rounding to the output dtype.
#include "common.cuh"

#include <stdlib.h>
#include <type_traits>

namespace bgx {
namespace {

template <typename Acc> struct Arith;
template <> struct Arith<float> {
  template <bool FUSED>
  __device__ static float mac(float a, float b, float c) {
    if constexpr (FUSED) return __fmaf_rn(a, b, c);
    else return __fadd_rn(__fmul_rn(a, b), c);
  }
};
template <> struct Arith<double> {
  template <bool FUSED>
  __device__ static double mac(double a, double b, double c) {
    if constexpr (FUSED) return __fma_rn(a, b, c);
    else return __dadd_rn(__dmul_rn(a, b), c);
  }
};

template <typename T> __device__ __forceinline__ float ld_f(const T *p) { return Conv<T>::to_f(*p); }

template <typename In, typename Acc> __device__ __forceinline__ Acc to_acc(In v) {
  if constexpr (sizeof(In) == 2) return (Acc)Conv<In>::to_f(v);
  else return (Acc)v;
}
template <typename Out, typename Acc> __device__ __forceinline__ Out from_acc(Acc v) {
  if constexpr (sizeof(Out) == 2) return Conv<Out>::from_f((float)v);
  else return (Out)v;
}

struct Params {
  int64_t batch, M, N, K;
  const void *a; int64_t sa[3];
  const void *b; int64_t sb[3];
  const void *c0; int64_t sc[3];
  void *out; int64_t so[3];
  int64_t tiles_m, tiles_n;
};

constexpr int BK = 16;

// BM x BN tile, TM x TN outputs per thread, K staged through shared memory
// in KT-deep tiles; the next tile's elements are loaded into registers while
// the current one is multiplied (one round trip of global-load latency per
// tile is otherwise exposed — it dominated small, latency-bound problems).
// Each output accumulates its products in increasing k from c0, so EXACT
// mode stays bit-identical to the reference.
template <typename In, typename Out, typename Acc, bool FUSED, int BM, int BN, int TM = 4,
          int TN = 4, int KT = BK>
__global__ void __launch_bounds__((BM / TM) * (BN / TN))
simt_gemm_kernel(const Params p) {
  constexpr int NT = (BM / TM) * (BN / TN);
  constexpr int LA = BM * KT / NT, LB = BN * KT / NT;   // elements per thread per tile
  static_assert(LA * NT == BM * KT && LB * NT == BN * KT, "tile / thread mismatch");
  // B rows unpadded when each thread reads 4 consecutive f32 columns: one
  // 16-byte shared load instead of four (8 lanes cover a 128-byte row, no
  // bank conflict); padded otherwise
  constexpr int BPAD = (TN % 4 == 0 && sizeof(Acc) == 4) ? 0 : 1;
  __shared__ Acc As[KT][BM + 1];
  __shared__ __align__(16) Acc Bs[KT][BN + BPAD];
  const int tid = threadIdx.x;
  const int tx = tid % (BN / TN), ty = tid / (BN / TN);
  int64_t t = blockIdx.x;
  const int64_t tn = t % p.tiles_n;
  t /= p.tiles_n;
  const int64_t tm = t % p.tiles_m;
  const int64_t b = t / p.tiles_m;
  const int64_t m0 = tm * BM, n0 = tn * BN;
  const In *A = static_cast<const In *>(p.a) + b * p.sa[0];
  const In *B = static_cast<const In *>(p.b) + b * p.sb[0];

  Acc acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int64_t m = m0 + ty * TM + i, n = n0 + tx * TN + j;
      Acc v = (Acc)0;
      if (p.c0 && m < p.M && n < p.N)
        v = to_acc<Out, Acc>(static_cast<const Out *>(p.c0)[b * p.sc[0] + m * p.sc[1] + n * p.sc[2]]);
      acc[i][j] = v;
    }

  // load mapping: run threads along whichever global dim has unit stride
  const bool a_k_inner = p.sa[2] == 1;
  const bool b_n_inner = p.sb[2] == 1 || p.sb[1] != 1;
  Acc ra[LA], rb[LB];
  auto load = [&](int64_t k0) {
#pragma unroll
    for (int l = 0; l < LA; ++l) {
      const int e = tid + l * NT;
      int mm, kk;
      if (a_k_inner) { kk = e % KT; mm = e / KT; } else { mm = e % BM; kk = e / BM; }
      const int64_t m = m0 + mm, k = k0 + kk;
      ra[l] = (m < p.M && k < p.K) ? to_acc<In, Acc>(A[m * p.sa[1] + k * p.sa[2]]) : (Acc)0;
    }
#pragma unroll
    for (int l = 0; l < LB; ++l) {
      const int e = tid + l * NT;
      int nn, kk;
      if (b_n_inner) { nn = e % BN; kk = e / BN; } else { kk = e % KT; nn = e / KT; }
      const int64_t n = n0 + nn, k = k0 + kk;
      rb[l] = (n < p.N && k < p.K) ? to_acc<In, Acc>(B[k * p.sb[1] + n * p.sb[2]]) : (Acc)0;
    }
  };
  auto stash = [&]() {
#pragma unroll
    for (int l = 0; l < LA; ++l) {
      const int e = tid + l * NT;
      int mm, kk;
      if (a_k_inner) { kk = e % KT; mm = e / KT; } else { mm = e % BM; kk = e / BM; }
      As[kk][mm] = ra[l];
    }
#pragma unroll
    for (int l = 0; l < LB; ++l) {
      const int e = tid + l * NT;
      int nn, kk;
      if (b_n_inner) { nn = e % BN; kk = e / BN; } else { kk = e % KT; nn = e / KT; }
      Bs[kk][nn] = rb[l];
    }
  };
  if (p.K > 0) load(0);
  for (int64_t k0 = 0; k0 < p.K; k0 += KT) {
    stash();
    __syncthreads();
    if (k0 + KT < p.K) load(k0 + KT);    // in flight while this tile is multiplied
    const int kmax = (p.K - k0) < KT ? (int)(p.K - k0) : KT;
#pragma unroll 8
    for (int kk = 0; kk < kmax; ++kk) {
      Acc av[TM], bv[TN];
#pragma unroll
      for (int i = 0; i < TM; ++i) av[i] = As[kk][ty * TM + i];
      if constexpr (BPAD == 0) {
#pragma unroll
        for (int j = 0; j < TN; j += 4) {
          const float4 q = *reinterpret_cast<const float4 *>(&Bs[kk][tx * TN + j]);
          bv[j] = q.x; bv[j + 1] = q.y; bv[j + 2] = q.z; bv[j + 3] = q.w;
        }
      } else {
#pragma unroll
        for (int j = 0; j < TN; ++j) bv[j] = Bs[kk][tx * TN + j];
      }
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = Arith<Acc>::template mac<FUSED>(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
  Out *O = static_cast<Out *>(p.out) + b * p.so[0];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int64_t m = m0 + ty * TM + i, n = n0 + tx * TN + j;
      if (m < p.M && n < p.N) O[m * p.so[1] + n * p.so[2]] = from_acc<Out, Acc>(acc[i][j]);
    }
}

// 128 x 128 tile, 256 threads, 8 x 8 outputs per thread (two 4-wide groups in
// each dimension so shared-memory fragment reads are broadcast / 16-byte),
// BK = 8, double-buffered shared memory with register prefetch of the next
// k-tile.  Each output still accumulates its products in increasing k from
// c0, so EXACT mode stays bit-identical to the reference.
constexpr int BT = 128, BKB = 8;

template <typename In, typename Out, typename Acc, bool FUSED>
__global__ void __launch_bounds__(256, sizeof(Acc) == 4 ? 2 : 1)
simt_gemm_big_kernel(const Params p) {
  __shared__ __align__(16) Acc As[2][BKB][BT];
  __shared__ __align__(16) Acc Bs[2][BKB][BT];
  const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
  int64_t t = blockIdx.x;
  const int64_t tn = t % p.tiles_n;
  t /= p.tiles_n;
  const int64_t tm = t % p.tiles_m;
  const int64_t b = t / p.tiles_m;
  const int64_t m0 = tm * BT, n0 = tn * BT;
  const In *A = static_cast<const In *>(p.a) + b * p.sa[0];
  const In *B = static_cast<const In *>(p.b) + b * p.sb[0];
  // load mappings: 4 elements per thread per operand per k-tile
  const bool a_k = p.sa[2] == 1;
  const bool b_n = p.sb[2] == 1 || p.sb[1] != 1;
  const int a_r = a_k ? tid / 2 : (tid % 32) * 4, a_c = a_k ? (tid % 2) * 4 : tid / 32;
  const int b_r = b_n ? tid / 32 : (tid % 2) * 4, b_c = b_n ? (tid % 32) * 4 : tid / 2;
  Acc ra[4], rb[4];
  // 16-byte vector loads when the 4 elements a thread fetches are contiguous
  // and aligned (f32 operands with unit inner stride); scalar otherwise
  const bool vec_a = sizeof(In) == 4 && sizeof(Acc) == 4 &&
                     (a_k ? (p.sa[1] % 4 == 0 && p.K % 4 == 0) : (p.sa[2] % 4 == 0 && p.M % 4 == 0)) &&
                     p.sa[0] % 4 == 0 && ((uintptr_t)p.a % 16) == 0;
  const bool vec_b = sizeof(In) == 4 && sizeof(Acc) == 4 &&
                     (b_n ? (p.sb[1] % 4 == 0 && p.N % 4 == 0) : (p.sb[2] % 4 == 0 && p.K % 4 == 0)) &&
                     p.sb[0] % 4 == 0 && ((uintptr_t)p.b % 16) == 0 &&
                     (b_n ? p.sb[2] == 1 : p.sb[1] == 1);
  // per-thread operand pointers at k = 0; each k-tile advances them by BKB * k-stride
  const In *pa = A + (int64_t)(m0 + (a_k ? a_r : a_r)) * p.sa[1] + (int64_t)a_c * p.sa[2];
  const In *pb = B + (int64_t)(b_r) * p.sb[1] + (int64_t)(n0 + b_c) * p.sb[2];
  const int64_t a_kstep = (int64_t)BKB * p.sa[2], b_kstep = (int64_t)BKB * p.sb[1];
  const int64_t a_qstep = a_k ? p.sa[2] : p.sa[1];   // between the 4 elements of a thread
  const int64_t b_qstep = b_n ? p.sb[2] : p.sb[1];
  const int64_t a_m = m0 + a_r, b_n0 = n0 + b_c;
  auto load_tiles = [&](int64_t k0) {
    const int64_t ak = k0 + a_c, bk = k0 + b_r;
    if (vec_a) {
      if (a_m < p.M && ak < p.K) {
        const float4 v = *reinterpret_cast<const float4 *>(pa);
        ra[0] = v.x; ra[1] = v.y; ra[2] = v.z; ra[3] = v.w;
      } else {
        ra[0] = ra[1] = ra[2] = ra[3] = (Acc)0;
      }
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const bool ok = a_k ? (a_m < p.M && ak + q < p.K) : (a_m + q < p.M && ak < p.K);
        ra[q] = ok ? to_acc<In, Acc>(pa[q * a_qstep]) : (Acc)0;
      }
    }
    if (vec_b) {
      if (bk < p.K && b_n0 < p.N) {
        const float4 v = *reinterpret_cast<const float4 *>(pb);
        rb[0] = v.x; rb[1] = v.y; rb[2] = v.z; rb[3] = v.w;
      } else {
        rb[0] = rb[1] = rb[2] = rb[3] = (Acc)0;
      }
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const bool ok = b_n ? (bk < p.K && b_n0 + q < p.N) : (bk + q < p.K && b_n0 < p.N);
        rb[q] = ok ? to_acc<In, Acc>(pb[q * b_qstep]) : (Acc)0;
      }
    }
    pa += a_kstep;
    pb += b_kstep;
  };
  auto store_tiles = [&](int buf) {
    // contiguous-in-tile fragments go out as one 16-byte store (no conflicts)
    if constexpr (sizeof(Acc) == 4) {
      if (!a_k) {
        *reinterpret_cast<float4 *>(&As[buf][a_c][a_r]) = make_float4(ra[0], ra[1], ra[2], ra[3]);
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) As[buf][a_c + q][a_r] = ra[q];
      }
      if (b_n) {
        *reinterpret_cast<float4 *>(&Bs[buf][b_r][b_c]) = make_float4(rb[0], rb[1], rb[2], rb[3]);
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) Bs[buf][b_r + q][b_c] = rb[q];
      }
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (a_k) As[buf][a_c + q][a_r] = ra[q]; else As[buf][a_c][a_r + q] = ra[q];
        if (b_n) Bs[buf][b_r][b_c + q] = rb[q]; else Bs[buf][b_r + q][b_c] = rb[q];
      }
    }
  };
  Acc acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int64_t m = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + i - 4);
      const int64_t n = n0 + (j < 4 ? tx * 4 + j : 64 + tx * 4 + j - 4);
      Acc v = (Acc)0;
      if (p.c0 && m < p.M && n < p.N)
        v = to_acc<Out, Acc>(static_cast<const Out *>(p.c0)[b * p.sc[0] + m * p.sc[1] + n * p.sc[2]]);
      acc[i][j] = v;
    }
  const int64_t ktiles = (p.K + BKB - 1) / BKB;
  if (ktiles > 0) {
    load_tiles(0);
    store_tiles(0);
  }
  __syncthreads();
  for (int64_t kt = 0; kt < ktiles; ++kt) {
    const int buf = kt & 1;
    if (kt + 1 < ktiles) load_tiles((kt + 1) * BKB);   // in flight during the math
    const int kmax = (p.K - kt * BKB) < BKB ? (int)(p.K - kt * BKB) : BKB;
    auto kstep = [&](int kk) {
      Acc av[8], bv[8];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        av[i] = As[buf][kk][ty * 4 + i];
        av[4 + i] = As[buf][kk][64 + ty * 4 + i];
        bv[i] = Bs[buf][kk][tx * 4 + i];
        bv[4 + i] = Bs[buf][kk][64 + tx * 4 + i];
      }
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = Arith<Acc>::template mac<FUSED>(av[i], bv[j], acc[i][j]);
    };
    if (kmax == BKB) {
      // full k-tile: straight-line code, so the compiler can issue the next
      // step's shared loads under the current step's FMAs
#pragma unroll
      for (int kk = 0; kk < BKB; ++kk) kstep(kk);
    } else {
      for (int kk = 0; kk < kmax; ++kk) kstep(kk);
    }
    if (kt + 1 < ktiles) store_tiles(buf ^ 1);
    __syncthreads();
  }
  Out *O = static_cast<Out *>(p.out) + b * p.so[0];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int64_t m = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + i - 4);
      const int64_t n = n0 + (j < 4 ? tx * 4 + j : 64 + tx * 4 + j - 4);
      if (m < p.M && n < p.N) O[m * p.so[1] + n * p.so[2]] = from_acc<Out, Acc>(acc[i][j]);
    }
}


// ---- f32, A K-major + B N-major: cp.async multi-stage pipeline ------------------
// The common row-major case.  Operand tiles go global -> shared with 16-byte
// cp.async (zero fill at the edges), CP_STAGES k-tiles in flight, so no
// registers are spent on staging and the 128-register budget of two CTAs per
// SM holds the 8x8 accumulators plus both fragments.  Each output still
// accumulates in increasing k from c0 (the k loop stops at K exactly), so
// EXACT mode stays bit-identical to the reference.
constexpr int CP_BK = 16, CP_APAD = 4;

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem, int bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(smem)), "l"(gmem),
               "r"(bytes) : "memory");
}

template <int CP_STAGES>
constexpr size_t cp_smem_bytes() { return sizeof(float) * CP_STAGES * (BT * (CP_BK + CP_APAD) + CP_BK * BT); }

template <bool FUSED, int CP_STAGES>
__global__ void __launch_bounds__(256, 2) simt_f32_cp_kernel(const Params p) {
  extern __shared__ __align__(16) float cp_smem[];
  auto As = reinterpret_cast<float (*)[BT][CP_BK + CP_APAD]>(cp_smem);                 // [s][m][k]
  auto Bs = reinterpret_cast<float (*)[CP_BK][BT]>(cp_smem + CP_STAGES * BT * (CP_BK + CP_APAD));
  const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
  int64_t t = blockIdx.x;
  const int64_t tn = t % p.tiles_n;
  t /= p.tiles_n;
  const int64_t tm = t % p.tiles_m;
  const int64_t b = t / p.tiles_m;
  const int64_t m0 = tm * BT, n0 = tn * BT;
  const float *A = static_cast<const float *>(p.a) + b * p.sa[0];
  const float *B = static_cast<const float *>(p.b) + b * p.sb[0];
  const int64_t lda = p.sa[1], ldb = p.sb[1];
  const int64_t ktiles = (p.K + CP_BK - 1) / CP_BK;
  // interior tiles (all 128 rows / columns live): per-thread source pointers
  // computed once, one pointer add and one unpredicated cp.async per chunk
  const bool interior_mn = m0 + BT <= p.M && n0 + BT <= p.N;
  const float *a_src[2], *b_src[2];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int ca = tid + q * 256, cb = tid + q * 256;
    a_src[q] = A + (m0 + ca / 4) * lda + (ca % 4) * 4;
    b_src[q] = B + (int64_t)(cb / 32) * ldb + n0 + (cb % 32) * 4;
  }
  auto issue = [&](int64_t kt) {
    const int st = (int)(kt % CP_STAGES);
    const int64_t k0 = kt * CP_BK;
    if (interior_mn && k0 + CP_BK <= p.K) {
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int c = tid + q * 256;
        cp_async16(&As[st][c / 4][(c % 4) * 4], a_src[q] + k0, 16);
        cp_async16(&Bs[st][c / 32][(c % 32) * 4], b_src[q] + k0 * ldb, 16);
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
      return;
    }
#pragma unroll
    for (int q = 0; q < 2; ++q) {           // A: 128 rows x 4 chunks
      const int c = tid + q * 256, row = c / 4, kq = (c % 4) * 4;
      const int64_t m = m0 + row, k = k0 + kq;
      int bytes = 0;
      if (m < p.M && k < p.K) bytes = (int)((p.K - k) >= 4 ? 16 : (p.K - k) * 4);
      cp_async16(&As[st][row][kq], bytes ? A + m * lda + k : A, bytes);
    }
#pragma unroll
    for (int q = 0; q < 2; ++q) {           // B: 16 rows x 32 chunks
      const int c = tid + q * 256, row = c / 32, nq = (c % 32) * 4;
      const int64_t k = k0 + row, n = n0 + nq;
      int bytes = 0;
      if (k < p.K && n < p.N) bytes = (int)((p.N - n) >= 4 ? 16 : (p.N - n) * 4);
      cp_async16(&Bs[st][row][nq], bytes ? B + k * ldb + n : B, bytes);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  float acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int64_t m = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + i - 4);
      const int64_t n = n0 + (j < 4 ? tx * 4 + j : 64 + tx * 4 + j - 4);
      float v = 0.f;
      if (p.c0 && m < p.M && n < p.N)
        v = static_cast<const float *>(p.c0)[b * p.sc[0] + m * p.sc[1] + n * p.sc[2]];
      acc[i][j] = v;
    }
#pragma unroll
  for (int s = 0; s < CP_STAGES - 1; ++s) {
    if (s < ktiles) issue(s);
    else asm volatile("cp.async.commit_group;" ::: "memory");
  }
  for (int64_t kt = 0; kt < ktiles; ++kt) {
    asm volatile("cp.async.wait_group %0;" ::"n"(CP_STAGES - 2) : "memory");
    __syncthreads();                         // tile kt landed; slot kt-1 is free
    if (kt + CP_STAGES - 1 < ktiles) issue(kt + CP_STAGES - 1);
    else asm volatile("cp.async.commit_group;" ::: "memory");
    const int st = (int)(kt % CP_STAGES);
    const int kmax = (p.K - kt * CP_BK) < CP_BK ? (int)(p.K - kt * CP_BK) : CP_BK;
    auto kstep = [&](int kk) {
      float av[8], bv[8];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        av[i] = As[st][ty * 4 + i][kk];
        av[4 + i] = As[st][64 + ty * 4 + i][kk];
      }
      const float4 b0 = *reinterpret_cast<const float4 *>(&Bs[st][kk][tx * 4]);
      const float4 b1 = *reinterpret_cast<const float4 *>(&Bs[st][kk][64 + tx * 4]);
      bv[0] = b0.x; bv[1] = b0.y; bv[2] = b0.z; bv[3] = b0.w;
      bv[4] = b1.x; bv[5] = b1.y; bv[6] = b1.z; bv[7] = b1.w;
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = Arith<float>::template mac<FUSED>(av[i], bv[j], acc[i][j]);
    };
    if (kmax == CP_BK) {
      // A fragments two k at a time (LDS.64): 4 A + 2 B loads per k step
#pragma unroll
      for (int kk = 0; kk < CP_BK; kk += 2) {
        float2 a2[8];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          a2[i] = *reinterpret_cast<const float2 *>(&As[st][ty * 4 + i][kk]);
          a2[4 + i] = *reinterpret_cast<const float2 *>(&As[st][64 + ty * 4 + i][kk]);
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          float bv[8];
          const float4 b0 = *reinterpret_cast<const float4 *>(&Bs[st][kk + h][tx * 4]);
          const float4 b1 = *reinterpret_cast<const float4 *>(&Bs[st][kk + h][64 + tx * 4]);
          bv[0] = b0.x; bv[1] = b0.y; bv[2] = b0.z; bv[3] = b0.w;
          bv[4] = b1.x; bv[5] = b1.y; bv[6] = b1.z; bv[7] = b1.w;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float av = h ? a2[i].y : a2[i].x;
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[i][j] = Arith<float>::template mac<FUSED>(av, bv[j], acc[i][j]);
          }
        }
      }
    } else {
      for (int kk = 0; kk < kmax; ++kk) kstep(kk);
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  float *O = static_cast<float *>(p.out) + b * p.so[0];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int64_t m = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + i - 4);
      const int64_t n = n0 + (j < 4 ? tx * 4 + j : 64 + tx * 4 + j - 4);
      if (m < p.M && n < p.N) O[m * p.so[1] + n * p.so[2]] = acc[i][j];
    }
}

// ---- f32, latency-bound sizes, row-major operands: cp.async ring ------------------
// The small-problem kernel above spends as many instructions on its generic
// strided, bounds-checked register staging as on the arithmetic; with one warp
// per scheduler (the problem has too few outputs for more) those instructions
// are the kernel time.  Here A (K-major) and B (N-major) tiles go global ->
// shared with one or two 16-byte cp.async per thread per stage (zero fill at
// the edges), SM_STAGES KT-deep stages in flight, and A fragments are read
// four k at a time.  Each output still accumulates fl(fl(a*b) + acc) in
// increasing k from c0 and the k loop stops at K exactly: EXACT mode stays
// bit-identical to the reference.
constexpr int SM_KT = 32, SM_STAGES = 4, SM_APAD = 4;

template <bool FUSED, int TM, int TN>
__global__ void __launch_bounds__(128) simt_f32_small_cp_kernel(const Params p) {
  constexpr int NT = 128;
  constexpr int TX = 32 / TN;              // threads along N: BN = 32
  constexpr int BN = 32, BM = (NT / TX) * TM;
  __shared__ __align__(16) float As[SM_STAGES][BM][SM_KT + SM_APAD];   // [s][m][k]
  __shared__ __align__(16) float Bs[SM_STAGES][SM_KT][BN];             // [s][k][n]
  const int tid = threadIdx.x, tx = tid % TX, ty = tid / TX;
  int64_t t = blockIdx.x;
  const int64_t tn = t % p.tiles_n;
  t /= p.tiles_n;
  const int64_t tm = t % p.tiles_m;
  const int64_t b = t / p.tiles_m;
  const int64_t m0 = tm * BM, n0 = tn * BN;
  const float *A = static_cast<const float *>(p.a) + b * p.sa[0];
  const float *B = static_cast<const float *>(p.b) + b * p.sb[0];
  const int64_t lda = p.sa[1], ldb = p.sb[1];
  const int64_t ktiles = (p.K + SM_KT - 1) / SM_KT;
  auto issue = [&](int64_t kt) {
    const int st = (int)(kt % SM_STAGES);
    const int64_t k0 = kt * SM_KT;
#pragma unroll
    for (int c = tid; c < BM * (SM_KT / 4); c += NT) {   // A: BM rows x 8 chunks
      const int row = c / (SM_KT / 4), kq = (c % (SM_KT / 4)) * 4;
      const int64_t m = m0 + row, k = k0 + kq;
      int bytes = 0;
      if (m < p.M && k < p.K) bytes = (int)((p.K - k) >= 4 ? 16 : (p.K - k) * 4);
      cp_async16(&As[st][row][kq], bytes ? A + m * lda + k : A, bytes);
    }
#pragma unroll
    for (int c = tid; c < SM_KT * (BN / 4); c += NT) {   // B: KT rows x 8 chunks
      const int row = c / (BN / 4), nq = (c % (BN / 4)) * 4;
      const int64_t k = k0 + row, n = n0 + nq;
      int bytes = 0;
      if (k < p.K && n < p.N) bytes = (int)((p.N - n) >= 4 ? 16 : (p.N - n) * 4);
      cp_async16(&Bs[st][row][nq], bytes ? B + k * ldb + n : B, bytes);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
#pragma unroll
  for (int s = 0; s < SM_STAGES - 1; ++s) {
    if (s < ktiles) issue(s);
    else asm volatile("cp.async.commit_group;" ::: "memory");
  }
  float acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int64_t m = m0 + ty * TM + i, n = n0 + tx * TN + j;
      acc[i][j] = (p.c0 && m < p.M && n < p.N)
                      ? static_cast<const float *>(p.c0)[b * p.sc[0] + m * p.sc[1] + n * p.sc[2]]
                      : 0.f;
    }
  for (int64_t kt = 0; kt < ktiles; ++kt) {
    asm volatile("cp.async.wait_group %0;" ::"n"(SM_STAGES - 2) : "memory");
    __syncthreads();                         // tile kt landed; slot kt-1 is free
    if (kt + SM_STAGES - 1 < ktiles) issue(kt + SM_STAGES - 1);
    else asm volatile("cp.async.commit_group;" ::: "memory");
    const int st = (int)(kt % SM_STAGES);
    const int kmax = (p.K - kt * SM_KT) < SM_KT ? (int)(p.K - kt * SM_KT) : SM_KT;
    auto kstep = [&](const float (&av)[TM], int kk) {
      float bv[TN];
      if constexpr (TN == 4) {
        const float4 q = *reinterpret_cast<const float4 *>(&Bs[st][kk][tx * 4]);
        bv[0] = q.x; bv[1] = q.y; bv[2] = q.z; bv[3] = q.w;
      } else {
        const float2 q = *reinterpret_cast<const float2 *>(&Bs[st][kk][tx * 2]);
        bv[0] = q.x; bv[1] = q.y;
      }
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = Arith<float>::template mac<FUSED>(av[i], bv[j], acc[i][j]);
    };
    if (kmax == SM_KT) {
#pragma unroll
      for (int kk = 0; kk < SM_KT; kk += 4) {
        float4 a4[TM];
#pragma unroll
        for (int i = 0; i < TM; ++i) a4[i] = *reinterpret_cast<const float4 *>(&As[st][ty * TM + i][kk]);
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          float av[TM];
#pragma unroll
          for (int i = 0; i < TM; ++i) av[i] = h == 0 ? a4[i].x : h == 1 ? a4[i].y : h == 2 ? a4[i].z : a4[i].w;
          kstep(av, kk + h);
        }
      }
    } else {
      for (int kk = 0; kk < kmax; ++kk) {
        float av[TM];
#pragma unroll
        for (int i = 0; i < TM; ++i) av[i] = As[st][ty * TM + i][kk];
        kstep(av, kk);
      }
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  float *O = static_cast<float *>(p.out) + b * p.so[0];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int64_t m = m0 + ty * TM + i, n = n0 + tx * TN + j;
      if (m < p.M && n < p.N) O[m * p.so[1] + n * p.so[2]] = acc[i][j];
    }
}

template <typename In, typename Out, typename Acc, bool FUSED>
int launch(const bgx_contract_desc &d, cudaStream_t s) {
  Params p;
  p.batch = d.batch; p.M = d.M; p.N = d.N; p.K = d.K;
  p.a = d.a; p.b = d.b; p.c0 = d.c0; p.out = d.out;
  for (int i = 0; i < 3; ++i) {
    p.sa[i] = d.a_stride[i]; p.sb[i] = d.b_stride[i];
    p.sc[i] = d.c_stride[i]; p.so[i] = d.o_stride[i];
  }
  const int sms = sm_count_current();
  const int64_t outs = d.M * d.N * d.batch;
  const bool small = outs < (int64_t)sms * 64 * 64 * 2;
  // BGX_SIMT_SMALL (A/B only): 0 = one output per thread, 1 = four chains per thread,
  // 2/3/4 = f32 row-major cp.async ring with 1x4 / 1x2 / 2x2 outputs per thread
  static const int small_variant = getenv("BGX_SIMT_SMALL") ? atoi(getenv("BGX_SIMT_SMALL")) : 4;
  const int64_t tiles_16x32 = ((d.M + 15) / 16) * ((d.N + 31) / 32) * d.batch;
  const bool rowmajor_f32 = std::is_same<In, float>::value && std::is_same<Out, float>::value &&
                            d.a_stride[2] == 1 && d.b_stride[2] == 1 && d.a_stride[1] % 4 == 0 &&
                            d.b_stride[1] % 4 == 0 && (d.batch <= 1 || (d.a_stride[0] % 4 == 0 &&
                            d.b_stride[0] % 4 == 0)) && ((uintptr_t)d.a % 16) == 0 &&
                            ((uintptr_t)d.b % 16) == 0;
  if (outs <= (int64_t)sms * 2048 && small_variant >= 2 && rowmajor_f32 && tiles_16x32 >= sms / 2) {
    // latency-bound f32 row-major: cp.async ring, no register staging
    if (small_variant == 3) {
      p.tiles_m = (d.M + 7) / 8; p.tiles_n = (d.N + 31) / 32;
      simt_f32_small_cp_kernel<FUSED, 1, 2><<<(unsigned)(p.tiles_m * p.tiles_n * d.batch), 128, 0, s>>>(p);
    } else if (small_variant == 4) {
      p.tiles_m = (d.M + 15) / 16; p.tiles_n = (d.N + 31) / 32;
      simt_f32_small_cp_kernel<FUSED, 2, 2><<<(unsigned)tiles_16x32, 128, 0, s>>>(p);
    } else {
      p.tiles_m = (d.M + 15) / 16; p.tiles_n = (d.N + 31) / 32;
      simt_f32_small_cp_kernel<FUSED, 1, 4><<<(unsigned)tiles_16x32, 128, 0, s>>>(p);
    }
  } else if (outs <= (int64_t)sms * 2048 && small_variant >= 1 && tiles_16x32 >= sms / 2) {
    // latency-bound sizes: the per-output k-sequential chain is the floor;
    // four independent chains per thread (1 x 4 outputs) hide the add
    // latency and amortise the shared-memory reads, 16 x 32 tiles of 128
    // threads keep one block on (almost) every SM
    p.tiles_m = (d.M + 15) / 16; p.tiles_n = (d.N + 31) / 32;
    simt_gemm_kernel<In, Out, Acc, FUSED, 16, 32, 1, 4, 64><<<(unsigned)tiles_16x32, 128, 0, s>>>(p);
  } else if (outs <= (int64_t)sms * 2048) {
    // latency-bound sizes: one output per thread, 16 x 16 tiles (the per-output
    // k-sequential chain is the floor, so maximise the number of chains)
    p.tiles_m = (d.M + 15) / 16; p.tiles_n = (d.N + 15) / 16;
    int64_t blocks = p.tiles_m * p.tiles_n * d.batch;
    simt_gemm_kernel<In, Out, Acc, FUSED, 16, 16, 1, 1, 64><<<(unsigned)blocks, 256, 0, s>>>(p);
  } else if (small) {
    p.tiles_m = (d.M + 31) / 32; p.tiles_n = (d.N + 31) / 32;
    int64_t blocks = p.tiles_m * p.tiles_n * d.batch;
    simt_gemm_kernel<In, Out, Acc, FUSED, 32, 32><<<(unsigned)blocks, 64, 0, s>>>(p);
  } else if ((d.M * d.N * d.batch) < (int64_t)sms * BT * BT) {
    p.tiles_m = (d.M + 63) / 64; p.tiles_n = (d.N + 63) / 64;
    int64_t blocks = p.tiles_m * p.tiles_n * d.batch;
    if (blocks > 0x7fffffffLL) { set_error("simt gemm: grid too large"); return BGX_ERR_UNSUPPORTED; }
    simt_gemm_kernel<In, Out, Acc, FUSED, 64, 64><<<(unsigned)blocks, 256, 0, s>>>(p);
  } else {
    p.tiles_m = (d.M + BT - 1) / BT; p.tiles_n = (d.N + BT - 1) / BT;
    int64_t blocks = p.tiles_m * p.tiles_n * d.batch;
    if (blocks > 0x7fffffffLL) { set_error("simt gemm: grid too large"); return BGX_ERR_UNSUPPORTED; }
    // f32 row-major operands (A K-major, B N-major, 16-byte rows): cp.async pipeline
    // (BGX_NO_SIMT_CP, read once per process: the register-staged kernel, for A/B)
    static const bool no_cp = getenv("BGX_NO_SIMT_CP") != nullptr;
    const bool cp_ok = std::is_same<In, float>::value && std::is_same<Out, float>::value &&
                       d.a_stride[2] == 1 && d.b_stride[2] == 1 && d.a_stride[1] % 4 == 0 &&
                       d.b_stride[1] % 4 == 0 && (d.batch <= 1 || (d.a_stride[0] % 4 == 0 &&
                       d.b_stride[0] % 4 == 0)) && ((uintptr_t)d.a % 16) == 0 &&
                       ((uintptr_t)d.b % 16) == 0 && !no_cp;
    // 2 stages: a third (measured, 55 KB dynamic smem) was 2-3% slower
    if (cp_ok) simt_f32_cp_kernel<FUSED, 2><<<(unsigned)blocks, 256, cp_smem_bytes<2>(), s>>>(p);
    else simt_gemm_big_kernel<In, Out, Acc, FUSED><<<(unsigned)blocks, 256, 0, s>>>(p);
  }
  return check_launch("simt_gemm_kernel");
}

}  // namespace

// Entry used by bgx_contract (contract.cu).  kind: 2 exact, 3 ffma, 4 16-bit.
int contract_simt(const bgx_contract_desc &d, int kind, cudaStream_t s) {
  const int in = d.in_dtype, out = d.out_dtype;
  if (in == BGX_F32 && out == BGX_F32)
    return kind == 3 ? launch<float, float, float, true>(d, s) : launch<float, float, float, false>(d, s);
  if (in == BGX_F64 && out == BGX_F64)
    return kind == 3 ? launch<double, double, double, true>(d, s) : launch<double, double, double, false>(d, s);
  if (in == BGX_BF16 && out == BGX_BF16) return launch<__nv_bfloat16, __nv_bfloat16, float, true>(d, s);
  if (in == BGX_BF16 && out == BGX_F32) return launch<__nv_bfloat16, float, float, true>(d, s);
  if (in == BGX_F16 && out == BGX_F16) return launch<__half, __half, float, true>(d, s);
  if (in == BGX_F16 && out == BGX_F32) return launch<__half, float, float, true>(d, s);
  set_error("simt gemm: unsupported dtype pair in=%d out=%d", in, out);
  return BGX_ERR_UNSUPPORTED;
}

}  // namespace bgx
