// Tensor-core batched contraction for sm_100a: TMA -> shared memory (128B
// swizzle) -> tcgen05.mma (kind::f16, bf16/f16 in, f32 accumulate in TMEM)
// -> tcgen05.ld epilogue -> global.  Replaces bridgegen's per-point
// multiply-accumulate loop (interp.py:407-420 with the einsum.py:111-117 body)
// for two-input contractions whose axes group into batch / M / N / K.
//
// Structure (one CTA per SM, persistent, warp-specialised, 256 threads):
//   warp 0      TMA producer (one lane): fills a STAGES-deep ring of A/B
//               k-blocks, signalling `full[s]` with transaction bytes;
//   warp 1      MMA issuer (one lane): waits `full[s]`, issues 4 x
//               tcgen05.mma (K = 16 each) per 64-wide k-block into one of two
//               TMEM accumulators, frees the slot with tcgen05.commit ->
//               `empty[s]`, and signals `tmem_full[acc]` after the last k-block;
//   warp 2      TMEM allocator (2 x BN columns);
//   warps 4..7  epilogue: wait `tmem_full[acc]`, tcgen05.ld 32 lanes x 32
//               columns per step, add c0 (beta = 1 semantics of
//               interp.py:399), convert, store; then arrive `tmem_empty[acc]`
//               so the MMA warp can reuse the accumulator — the epilogue of
//               tile i overlaps the main loop of tile i+1.
// Tiles: 128 (M) x BN (N) x 64 (K); batch folded into the tile index; tile
// order is rasterised in groups of `raster` M-tiles for L2 reuse.
// Operand layouts: A K-major or M-major, B K-major or N-major — the major-ness
// goes into the instruction descriptor, no transposing copy is made.
#include "common.cuh"

#include <cudaTypedefs.h>
#include <mutex>

namespace bgx {

namespace {

constexpr int BM = 128;
constexpr int BK = 64;                 // 64 x 16-bit = 128 B = one swizzle row
constexpr int A_STAGE_BYTES = BM * BK * 2;  // 16 KB
constexpr int NUM_THREADS = 256;

struct TcParams {
  int64_t batch, M, N, K;
  int32_t tiles_m, tiles_n, k_blocks, raster;
  int64_t num_tiles;
  uint32_t idesc;
  int32_t a_mn, b_mn;            // 1 = MN-major operand
  const void *c0; int64_t sc[3];
  void *out; int64_t so[3];
};

template <int BN> struct Cfg {
  static constexpr int B_STAGE_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_STAGE_BYTES + B_STAGE_BYTES;
  static constexpr int STAGES = BN == 256 ? 4 : (BN == 128 ? 6 : 8);
  static constexpr int TMEM_COLS = 2 * BN < 32 ? 32 : 2 * BN;
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
};

__device__ __forceinline__ void tile_coords(const TcParams &p, int64_t t, int64_t &b, int64_t &tm,
                                            int64_t &tn) {
  const int64_t per_batch = (int64_t)p.tiles_m * p.tiles_n;
  b = t / per_batch;
  int64_t r = t % per_batch;
  const int64_t G = p.raster;
  const int64_t group = r / (G * p.tiles_n);
  const int64_t in_group = r % (G * p.tiles_n);
  const int64_t first_m = group * G;
  const int64_t gm = (p.tiles_m - first_m) < G ? (p.tiles_m - first_m) : G;
  tm = first_m + in_group % gm;
  tn = in_group / gm;
}

template <typename OutT> struct Store;
template <> struct Store<float> {
  __device__ static void row32(float *dst, const float *v, bool full, int64_t valid) {
    if (full && ((uintptr_t)dst & 15) == 0) {
#pragma unroll
      for (int j = 0; j < 32; j += 4)
        *reinterpret_cast<float4 *>(dst + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
    } else {
      for (int j = 0; j < 32; ++j) if (j < valid) dst[j] = v[j];
    }
  }
};
template <typename H> struct Store16 {
  __device__ static void row32(H *dst, const float *v, bool full, int64_t valid) {
    if (full && ((uintptr_t)dst & 15) == 0) {
#pragma unroll
      for (int j = 0; j < 32; j += 8) {
        uint4 pk;
        uint32_t *w = reinterpret_cast<uint32_t *>(&pk);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          H lo = Conv<H>::from_f(v[j + 2 * q]), hi = Conv<H>::from_f(v[j + 2 * q + 1]);
          w[q] = (uint32_t)(*reinterpret_cast<uint16_t *>(&lo)) |
                 ((uint32_t)(*reinterpret_cast<uint16_t *>(&hi)) << 16);
        }
        *reinterpret_cast<uint4 *>(dst + j) = pk;
      }
    } else {
      for (int j = 0; j < 32; ++j) if (j < valid) dst[j] = Conv<H>::from_f(v[j]);
    }
  }
};
template <> struct Store<__nv_bfloat16> : Store16<__nv_bfloat16> {};
template <> struct Store<__half> : Store16<__half> {};

template <int BN, typename OutT>
__global__ void __launch_bounds__(NUM_THREADS, 1)
tc_gemm_kernel(const __grid_constant__ CUtensorMap tmap_a,
               const __grid_constant__ CUtensorMap tmap_b, const TcParams p) {
  using C = Cfg<BN>;
  constexpr int STAGES = C::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t *smem_a = smem;
  uint8_t *smem_b = smem + STAGES * A_STAGE_BYTES;
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + STAGES * C::STAGE_BYTES);
  uint64_t *full = bars;
  uint64_t *empty = bars + STAGES;
  uint64_t *tmem_full = bars + 2 * STAGES;
  uint64_t *tmem_empty = bars + 2 * STAGES + 2;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 2 * STAGES + 4);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmap_a);
    prefetch_tmap(&tmap_b);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tmem_full[a], 1);
      mbar_init(&tmem_empty[a], 128);
    }
    fence_barrier_init();
  }
  if (warp == 2) {
    tmem_alloc<1>(tmem_slot, C::TMEM_COLS);
    tmem_relinquish<1>();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ===== TMA producer =====
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
        int64_t b, tm, tn;
        tile_coords(p, t, b, tm, tn);
        const int32_t m0 = (int32_t)(tm * BM), n0 = (int32_t)(tn * BN), bb = (int32_t)b;
        for (int kb = 0; kb < p.k_blocks; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_expect_tx(&full[stage], C::STAGE_BYTES);
          const int32_t k0 = kb * BK;
          uint8_t *sa = smem_a + stage * A_STAGE_BYTES;
          uint8_t *sb = smem_b + stage * C::B_STAGE_BYTES;
          if (p.a_mn) {
            tma_load_3d(sa, &tmap_a, &full[stage], m0, k0, bb);
            tma_load_3d(sa + 8192, &tmap_a, &full[stage], m0 + 64, k0, bb);
          } else {
            tma_load_3d(sa, &tmap_a, &full[stage], k0, m0, bb);
          }
          if (p.b_mn) {
#pragma unroll
            for (int j = 0; j < BN / 64; ++j)
              tma_load_3d(sb + j * 8192, &tmap_b, &full[stage], n0 + 64 * j, k0, bb);
          } else {
            tma_load_3d(sb, &tmap_b, &full[stage], k0, n0, bb);
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ===== MMA issuer =====
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      // per-k16 descriptor advance and fixed LBO/SBO per operand layout
      const uint32_t a_step = p.a_mn ? 2048u : 32u, b_step = p.b_mn ? 2048u : 32u;
      const uint32_t a_lbo = p.a_mn ? 8192u : 16u, b_lbo = p.b_mn ? 8192u : 16u;
      for (int64_t t = blockIdx.x; t < p.num_tiles; t += gridDim.x, ++it) {
        const int acc = it & 1;
        const uint32_t acc_phase = (it >> 1) & 1;
        mbar_wait(&tmem_empty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < p.k_blocks; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem_a + stage * A_STAGE_BYTES);
          const uint32_t sb = smem_u32(smem_b + stage * C::B_STAGE_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t ad = make_sdesc_sw128(sa + k * a_step, a_lbo, 1024);
            const uint64_t bd = make_sdesc_sw128(sb + k * b_step, b_lbo, 1024);
            umma_f16<1>(d_tmem, ad, bd, p.idesc, (kb | k) != 0);
          }
          umma_commit(&empty[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        umma_commit(&tmem_full[acc]);
      }
    }
  } else if (warp >= 4) {
    // ===== epilogue =====
    const int ew = warp - 4;  // TMEM lanes [32*ew, 32*ew + 32)
    int it = 0;
    for (int64_t t = blockIdx.x; t < p.num_tiles; t += gridDim.x, ++it) {
      int64_t b, tm, tn;
      tile_coords(p, t, b, tm, tn);
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      mbar_wait(&tmem_full[acc], acc_phase);
      tc_fence_after();
      const int64_t m = tm * BM + ew * 32 + lane;
      const bool row_ok = m < p.M;
      OutT *orow = static_cast<OutT *>(p.out) + b * p.so[0] + m * p.so[1];
      const OutT *crow = p.c0 ? static_cast<const OutT *>(p.c0) + b * p.sc[0] + m * p.sc[1] : nullptr;
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(ew * 32) << 16) + acc * BN + c * 32, r);
        tmem_ld_wait();
        const int64_t n = tn * BN + c * 32;
        if (row_ok && n < p.N) {
          float v[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
          const int64_t valid = p.N - n;
          if (crow) {
            for (int j = 0; j < 32; ++j)
              if (j < valid) v[j] = __fadd_rn(v[j], Conv<OutT>::to_f(crow[n + j]));
          }
          Store<OutT>::row32(orow + n, v, valid >= 32, valid);
        }
      }
      tc_fence_before();
      mbar_arrive(&tmem_empty[acc]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<1>(tmem_base, C::TMEM_COLS);
  }
}

// ---- host: tensor maps ------------------------------------------------------

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault,
                                         &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// 3-D map over a 16-bit tensor: dims (inner, outer, batch) with element
// strides (1, s_outer, s_batch); box (box_inner, box_outer, 1), 128B swizzle.
int make_map(CUtensorMap *map, const void *base, CUtensorMapDataType dt, int64_t inner,
             int64_t outer, int64_t batch, int64_t s_outer, int64_t s_batch, uint32_t box_inner,
             uint32_t box_outer) {
  auto enc = get_encode();
  if (!enc) { set_error("cuTensorMapEncodeTiled unavailable"); return BGX_ERR_CUDA; }
  cuuint64_t dims[3] = {(cuuint64_t)inner, (cuuint64_t)outer, (cuuint64_t)batch};
  if (batch <= 1) s_batch = s_outer * outer;  // any legal value; never stepped
  cuuint64_t strides[2] = {(cuuint64_t)(s_outer * 2), (cuuint64_t)(s_batch * 2)};
  cuuint32_t box[3] = {box_inner, box_outer, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, dt, 3, const_cast<void *>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d): dims %lld x %lld x %lld strides %lld/%lld",
              (int)r, (long long)inner, (long long)outer, (long long)batch,
              (long long)s_outer, (long long)s_batch);
    return BGX_ERR_INVALID;
  }
  return BGX_OK;
}

template <int BN, typename OutT>
int launch_tc(const bgx_contract_desc &d, const TcParams &p0, cudaStream_t s) {
  using C = Cfg<BN>;
  TcParams p = p0;
  const CUtensorMapDataType dt =
      d.in_dtype == BGX_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  CUtensorMap ma, mb;
  int rc;
  if (p.a_mn)
    rc = make_map(&ma, d.a, dt, d.M, d.K, d.batch, d.a_stride[2], d.a_stride[0], 64, 64);
  else
    rc = make_map(&ma, d.a, dt, d.K, d.M, d.batch, d.a_stride[1], d.a_stride[0], 64, BM);
  if (rc) return rc;
  if (p.b_mn)
    rc = make_map(&mb, d.b, dt, d.N, d.K, d.batch, d.b_stride[1], d.b_stride[0], 64, 64);
  else
    rc = make_map(&mb, d.b, dt, d.K, d.N, d.batch, d.b_stride[2], d.b_stride[0], 64, BN);
  if (rc) return rc;
  p.idesc = make_idesc_f16(d.in_dtype == BGX_BF16, p.a_mn, p.b_mn, BM, BN);
  p.tiles_n = (int32_t)((d.N + BN - 1) / BN);
  p.num_tiles = (int64_t)p.tiles_m * p.tiles_n * d.batch;
  auto kern = tc_gemm_kernel<BN, OutT>;
  static thread_local int configured[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!configured[dev & 63]) {
    BGX_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      C::SMEM_BYTES));
    configured[dev & 63] = 1;
  }
  int sms = sm_count_current();
  int64_t grid = p.num_tiles < sms ? p.num_tiles : sms;
  if (d.sched.max_ctas > 0 && grid > d.sched.max_ctas) grid = d.sched.max_ctas;
  kern<<<(unsigned)grid, NUM_THREADS, C::SMEM_BYTES, s>>>(ma, mb, p);
  return check_launch("tc_gemm_kernel");
}

template <typename OutT>
int dispatch_bn(const bgx_contract_desc &d, int bn, const TcParams &p, cudaStream_t s) {
  switch (bn) {
    case 64: return launch_tc<64, OutT>(d, p, s);
    case 128: return launch_tc<128, OutT>(d, p, s);
    default: return launch_tc<256, OutT>(d, p, s);
  }
}

}  // namespace

// Legality of the TMA/tcgen05 path for a descriptor (see bgx.h).
bool tc_legal(const bgx_contract_desc &d, const char **why) {
  auto fail = [&](const char *w) { if (why) *why = w; return false; };
  if (!(d.in_dtype == BGX_BF16 || d.in_dtype == BGX_F16)) return fail("inputs not bf16/f16");
  if (!(d.out_dtype == d.in_dtype || d.out_dtype == BGX_F32)) return fail("out dtype");
  if (d.M <= 0 || d.N <= 0 || d.K <= 0 || d.batch <= 0) return fail("empty extent");
  if (d.M >= (1ll << 31) || d.N >= (1ll << 31) || d.K >= (1ll << 31)) return fail("extent >= 2^31");
  const bool a_mn = d.a_stride[2] != 1 && d.a_stride[1] == 1;
  const bool a_k = d.a_stride[2] == 1;
  if (!a_mn && !a_k) return fail("A has no unit stride in m or k");
  const bool b_mn = d.b_stride[2] == 1;
  const bool b_k = !b_mn && d.b_stride[1] == 1;
  if (!b_mn && !b_k) return fail("B has no unit stride in k or n");
  auto al16 = [](int64_t elems) { return (elems * 2) % 16 == 0; };
  if (((uintptr_t)d.a % 16) || ((uintptr_t)d.b % 16)) return fail("A/B base not 16B aligned");
  if (a_k && (!al16(d.a_stride[1]) || (d.batch > 1 && !al16(d.a_stride[0])))) return fail("A strides");
  if (a_mn && (!al16(d.a_stride[2]) || (d.batch > 1 && !al16(d.a_stride[0])))) return fail("A strides");
  if (b_mn && (!al16(d.b_stride[1]) || (d.batch > 1 && !al16(d.b_stride[0])))) return fail("B strides");
  if (b_k && (!al16(d.b_stride[2]) || (d.batch > 1 && !al16(d.b_stride[0])))) return fail("B strides");
  if (d.o_stride[2] != 1) return fail("out n-stride != 1");
  if (d.c0 && d.c_stride[2] != 1) return fail("c0 n-stride != 1");
  return true;
}

int contract_tc(const bgx_contract_desc &d, cudaStream_t s) {
  const char *why = nullptr;
  if (!tc_legal(d, &why)) {
    set_error("tensor-core path not legal: %s", why);
    return BGX_ERR_UNSUPPORTED;
  }
  TcParams p{};
  p.batch = d.batch; p.M = d.M; p.N = d.N; p.K = d.K;
  p.a_mn = d.a_stride[2] != 1 ? 1 : 0;
  p.b_mn = d.b_stride[2] == 1 ? 1 : 0;
  p.tiles_m = (int32_t)((d.M + BM - 1) / BM);
  p.k_blocks = (int32_t)((d.K + BK - 1) / BK);
  p.raster = d.sched.raster > 0 ? d.sched.raster : 16;
  p.c0 = d.c0; p.out = d.out;
  for (int i = 0; i < 3; ++i) { p.sc[i] = d.c_stride[i]; p.so[i] = d.o_stride[i]; }
  int bn = d.sched.tile_n;
  if (bn != 64 && bn != 128 && bn != 256) bn = d.N <= 64 ? 64 : (d.N <= 128 ? 128 : 256);
  if (d.out_dtype == BGX_F32) return dispatch_bn<float>(d, bn, p, s);
  if (d.out_dtype == BGX_BF16) return dispatch_bn<__nv_bfloat16>(d, bn, p, s);
  return dispatch_bn<__half>(d, bn, p, s);
}

}  // namespace bgx
