// Tensor-core batched contraction for sm_100a: TMA -> shared memory (128B
// swizzle) -> tcgen05.mma (kind::f16, bf16/f16 in, f32 accumulate in TMEM)
// -> tcgen05.ld epilogue -> global.  Replaces bridgegen's per-point
// multiply-accumulate loop (interp.py:407-420 with the einsum.py:111-117 body)
// for two-input contractions whose axes group into batch / M / N / K.
//
// Structure (persistent, warp-specialised, 256 threads per CTA):
//   warp 0      TMA producer (one lane): fills a STAGES-deep ring of A/B
//               k-blocks, signalling `full[s]` with transaction bytes;
//   warp 1      MMA issuer (one lane, leader CTA only): waits `full[s]`,
//               issues 4 x tcgen05.mma (K = 16 each) per 64-wide k-block into
//               one of two TMEM accumulators, frees the slot with
//               tcgen05.commit -> `empty[s]`, and signals `tmem_full[acc]`
//               after the last k-block;
//   warp 2      TMEM allocator (2 x BN columns: double-buffered accumulator);
//   warps 4..7  epilogue: wait `tmem_full[acc]`, tcgen05.ld 32 lanes x 32
//               columns per step, add c0 (beta = 1 semantics of
//               interp.py:399), convert, store; then arrive `tmem_empty[acc]`
//               so the MMA warp can reuse the accumulator — the epilogue of
//               tile i overlaps the main loop of tile i+1.
// CG = 1: one CTA per SM computes 128 x BN tiles (tcgen05.mma cta_group::1).
// CG = 2: a cluster of 2 CTAs on one TPC computes 256 x BN tiles with
//   tcgen05.mma.cta_group::2 (M = 256): each CTA stages its 128 rows of A and
//   its BN/2 columns of B (TMA .cta_group::2 signals the leader's barrier), the
//   leader issues the MMAs, each CTA's TMEM holds its 128 accumulator rows.
//   Per SM this halves the shared-memory and L2->SM bytes of B per flop.
// Tiles: BK = 64; batch folded into the tile index; tile order rasterised in
// groups of `raster` M-tiles for L2 reuse.  Operand layouts: A K- or M-major,
// B K- or N-major — the major-ness goes into the instruction descriptor, no
// transposing copy is made.
#include "common.cuh"

#include <cudaTypedefs.h>
#include <mutex>
#include <string.h>

// 512-wide pair tiles: read both TMEM halves into packed registers before any
// store (0 = read, release and store one half at a time).  A/B on B200:
// 4096^3 forced to 512 tiles +1.8 % burst, other shapes neutral.
#ifndef BGX_EPI_DRAIN_BOTH
#define BGX_EPI_DRAIN_BOTH 1
#endif
// 1 (default): staged 32 x 32 output chunks leave shared memory through the
// LSU — coalesced 16-byte st.global, whole sectors of 8 (16-bit) or 4 (f32)
// rows per warp instruction — instead of a TMA bulk store, which keeps the
// SM's TMA unit for operand loads.  B200 A/B (profiles/r02_epilogue_stores.txt):
// C3 64 x 1024^3 104.4 -> 102.4 us, 4096^3 96.3 -> 95.2 us, chain neutral.
#ifndef BGX_EPI_LSU
#define BGX_EPI_LSU 1
#endif

namespace bgx {

namespace {

// Timeline probe (schedule debug bit 4096): %globaltimer when each CTA's
// producer starts each of its first TR_UNITS units, read back with
// bgxdbg_trace_read (A/B tooling, not part of the C ABI).
constexpr int TR_CTAS = 160, TR_UNITS = 64;
__device__ unsigned long long g_trace[TR_CTAS * TR_UNITS];

constexpr int BM = 128;                     // rows of A per CTA
constexpr int ROW_BYTES = 128;              // one 128B-swizzle row of K per k-block
constexpr int A_STAGE_BYTES = BM * ROW_BYTES;  // 16 KB
// K elements per k-block: 64 for 16-bit inputs, 32 for tf32 (fp32 storage)
template <int IN_BYTES> struct Elem {
  static constexpr int BK = ROW_BYTES / IN_BYTES;
  static constexpr int MMA_K = 32 / IN_BYTES;        // K per tcgen05.mma (16 / 8)
  static constexpr int MN_ATOM = ROW_BYTES / IN_BYTES;  // MN elements per swizzle row
  static constexpr int BOX_BYTES = MN_ATOM * BK * IN_BYTES;  // one MN-major box (8 / 4 KB)
};
constexpr int EPI_WARPS = 8;                // 2 warps per TMEM lane quadrant
// 512-wide tiles: resident stages whose first halves are issued ahead of
// their second halves at a tile end (the epilogue drains columns [0,256)
// behind them); each held stage delays its refill.
#ifndef LATE_STAGES
#define LATE_STAGES 4
#endif
constexpr int NUM_THREADS = 128 + 32 * EPI_WARPS;
constexpr int SMEM_BUDGET = 227 * 1024;

struct TcParams {
  int64_t batch, M, N, K;
  int32_t tiles_m, tiles_n, k_blocks, raster;
  int64_t num_tiles;
  int32_t k_splits, kb_per_split;  // split-K: unit u -> tile u % num_tiles, K slice u / num_tiles
  int64_t num_units;
  // tail split (stream-K style): tiles >= tail_start are split into
  // tail_splits K slices; slices 0..S-2 store f32 partials to `ws` (one
  // TILE_M x BN block per slice) and count themselves in tail_counters; the
  // last slice (the finisher) waits for that count — every CTA of the
  // persistent grid is resident and every tile's other slices come earlier
  // in each CTA's unit order, so the wait cannot deadlock — and adds the
  // partials, in slice order, to its own accumulator before storing
  int64_t tail_start;
  int32_t tail_splits, kb_per_tail;
  float *ws;
  uint32_t *tail_counters;
  int64_t ws_bytes;
  uint32_t idesc;
  int32_t a_mn, b_mn;            // 1 = MN-major operand
  int32_t stages;                // ring depth actually used (<= Cfg::STAGES)
  int32_t tma_store;             // 1: epilogue stores through TMA (out map legal)
  int32_t debug;                 // bit 0: skip the epilogue stores (timing probe)
  const void *c0; int64_t sc[3];
  void *out; int64_t so[3];
  // fused K-split reduce-scatter epilogue (RS kernels only, bgx.h)
  int32_t rs_world, rs_rank, rs_out_dtype;
  int32_t rs_defer;                     // BGX_RS_DEFERRED: deliver only (bgx_rs_reduce sums)
  int64_t rs_rpo;                       // output rows per owner
  float *rs_slots[BGX_MAX_RANKS];
  uint32_t *rs_counters[BGX_MAX_RANKS];
  void *rs_out[BGX_MAX_RANKS];
  const void *rs_c0[BGX_MAX_RANKS];
  uint32_t *rs_ws_counters;
};

template <int BN, int CG, int OUT_BYTES, int IN_BYTES = 2> struct Cfg {
  using E = Elem<IN_BYTES>;
  static constexpr int BN_CTA = BN / CG;                 // B columns staged per CTA
  // one tcgen05.mma covers at most N = 256: wider tiles issue NSPLIT MMAs per
  // K-step into adjacent TMEM column ranges
  static constexpr int MMA_N = BN > 256 ? 256 : BN;
  static constexpr int NSPLIT = BN / MMA_N;
  static constexpr int B_BOX_N = MMA_N / CG;             // B columns per CTA per MMA
  static constexpr int B_HALF_BYTES = B_BOX_N * ROW_BYTES;
  static constexpr int B_STAGE_BYTES = BN_CTA * ROW_BYTES;
  static constexpr int ACC_BUFS = 2 * BN <= 512 ? 2 : 1; // double-buffered accumulator?
  static constexpr int STAGE_BYTES = A_STAGE_BYTES + B_STAGE_BYTES;
  // epilogue staging: 4 warps x 2 buffers x (32 rows x 32 cols) of the output
  static constexpr int EPI_BUF_BYTES = 32 * 32 * OUT_BYTES;
  static constexpr int EPI_BYTES = EPI_WARPS * 2 * EPI_BUF_BYTES;
  static constexpr int STAGES_RAW = (SMEM_BUDGET - 2048 - EPI_BYTES) / STAGE_BYTES;
  static constexpr int STAGES = STAGES_RAW > 8 ? 8 : STAGES_RAW;
  static constexpr int TMEM_COLS = ACC_BUFS * BN < 32 ? 32 : ACC_BUFS * BN;
  static constexpr int SMEM_BYTES =
      STAGES * STAGE_BYTES + EPI_BYTES + 1024 /*align*/ + 256 /*barriers*/;
  static constexpr int TILE_M = BM * CG;
};

__device__ __forceinline__ void tile_coords(const TcParams &p, int64_t t, int64_t &b, int64_t &tm,
                                            int64_t &tn) {
  const int64_t per_batch = (int64_t)p.tiles_m * p.tiles_n;
  b = t / per_batch;
  int64_t r = t % per_batch;
  if (p.raster > 0) {
    // groups of G M-tiles; inside a group M fastest, then N (A slab resident)
    const int64_t G = p.raster;
    const int64_t group = r / (G * p.tiles_n);
    const int64_t in_group = r % (G * p.tiles_n);
    const int64_t first_m = group * G;
    const int64_t gm = (p.tiles_m - first_m) < G ? (p.tiles_m - first_m) : G;
    tm = first_m + in_group % gm;
    tn = in_group / gm;
  } else {
    // groups of G N-tiles; inside a group N fastest, then M (B slab resident
    // in L2 while A streams through once per group)
    const int64_t G = -p.raster;
    const int64_t group = r / (G * p.tiles_m);
    const int64_t in_group = r % (G * p.tiles_m);
    const int64_t first_n = group * G;
    const int64_t gn = (p.tiles_n - first_n) < G ? (p.tiles_n - first_n) : G;
    tn = first_n + in_group % gn;
    tm = in_group / gn;
  }
}

// Write one thread's row of 32 output values into the warp's swizzled staging
// buffer (32 rows x 32 cols) in the layout the output tensor map's swizzle
// expects: SW64 for 16-bit outputs (64-byte rows), SW128 for f32 (128-byte
// rows): 16-byte chunk j of row r lands at chunk j ^ f(r).
template <typename OutT>
__device__ __forceinline__ void stage_row32(uint8_t *buf, int r, const float *v) {
  if constexpr (sizeof(OutT) == 4) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      float4 q = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
      *reinterpret_cast<float4 *>(buf + r * 128 + ((j ^ (r & 7)) << 4)) = q;
    }
  } else {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      uint4 pk;
      uint32_t *w = reinterpret_cast<uint32_t *>(&pk);
#pragma unroll
      for (int q = 0; q < 4; ++q) w[q] = pack2<OutT>(v[8 * j + 2 * q], v[8 * j + 2 * q + 1]);
      *reinterpret_cast<uint4 *>(buf + r * 64 + ((j ^ ((r >> 1) & 3)) << 4)) = pk;
    }
  }
}

// LSU store of one staged 32 x 32 chunk (the stage_row32 layout): lane l
// moves 16-byte group l % CPR of row l / CPR (+ RPI rows per step), so each
// warp instruction writes whole sectors of RPI consecutive rows.
template <typename OutT>
__device__ __forceinline__ void lsu_store_chunk(const uint8_t *buf, OutT *row0, int64_t row_stride,
                                                int64_t rows_valid, int64_t cols_valid, int lane) {
  constexpr int RB = 32 * (int)sizeof(OutT);   // staged bytes per row (64 or 128)
  constexpr int CPR = RB / 16;                 // 16-byte groups per row
  constexpr int RPI = 32 / CPR;                // rows per warp instruction
  constexpr int EPG = 16 / (int)sizeof(OutT);  // elements per group
  const int j = lane % CPR;
#pragma unroll
  for (int i = 0; i < 32 / RPI; ++i) {
    const int r = i * RPI + lane / CPR;
    const int sw = sizeof(OutT) == 4 ? (r & 7) : ((r >> 1) & 3);
    const uint4 v = *reinterpret_cast<const uint4 *>(buf + r * RB + ((j ^ sw) << 4));
    if (r < rows_valid) {
      OutT *dst = row0 + r * row_stride + j * EPG;
      if ((j + 1) * EPG <= cols_valid) {
        *reinterpret_cast<uint4 *>(dst) = v;
      } else {
        const OutT *e = reinterpret_cast<const OutT *>(&v);
        for (int q = 0; q < EPG; ++q)
          if (j * EPG + q < cols_valid) dst[q] = e[q];
      }
    }
  }
}

struct UnitInfo {
  int64_t t;       // tile index
  int kb_lo, nkb;  // K-block range
  int64_t slot;    // >= 0: tail-split partial slot in ws; -1: regular output
  int64_t kslice;  // uniform split-K slice (extra output batch), else 0
};
__device__ __forceinline__ UnitInfo unit_info(const TcParams &p, int64_t u) {
  UnitInfo r;
  r.slot = -1;
  r.kslice = 0;
  if (p.tail_splits > 1 && u >= p.tail_start) {
    const int64_t tt = p.num_tiles - p.tail_start;
    const int64_t v = u - p.tail_start;
    r.t = p.tail_start + v % tt;
    const int s = (int)(v / tt);
    r.kb_lo = s * p.kb_per_tail;
    const int hi = r.kb_lo + p.kb_per_tail < p.k_blocks ? r.kb_lo + p.kb_per_tail : p.k_blocks;
    r.nkb = hi - r.kb_lo;
    r.slot = s * tt + (r.t - p.tail_start);
    return r;
  }
  r.t = u % p.num_tiles;
  r.kslice = u / p.num_tiles;
  if (p.kb_per_split == 0) {
    // balanced partition (fused reduce-scatter): exactly k_splits non-empty
    // slices (k_splits <= k_blocks)
    r.kb_lo = (int)(r.kslice * p.k_blocks / p.k_splits);
    r.nkb = (int)((r.kslice + 1) * p.k_blocks / p.k_splits) - r.kb_lo;
    return r;
  }
  r.kb_lo = (int)r.kslice * p.kb_per_split;
  const int hi = r.kb_lo + p.kb_per_split < p.k_blocks ? r.kb_lo + p.kb_per_split : p.k_blocks;
  r.nkb = hi - r.kb_lo;
  return r;
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

// ---- fused K-split reduce-scatter epilogue helpers --------------------------

// 32 f32 values of a row written by another CTA or GPU in this kernel.
__device__ __forceinline__ void load_row32_sys(const float *src, float *v, int64_t valid) {
  if (valid >= 32 && ((uintptr_t)src & 15) == 0) {
#pragma unroll
    for (int j = 0; j < 32; j += 4) {
      const float4 q = ld_sys_v4(src + j);
      v[j] = q.x; v[j + 1] = q.y; v[j + 2] = q.z; v[j + 3] = q.w;
    }
  } else {
    for (int j = 0; j < 32; ++j) v[j] = j < valid ? ld_sys(src + j) : 0.f;
  }
}

// Publish this CTA's stores for one tile and count the arrival on `counter`
// (system scope when the counter and the data may live on another GPU).
// Returns true in every epilogue thread of the unit that completes the
// count (it resets the counter for the next call).  No thread ever waits for
// another CTA or GPU: the last arriver does the reduction.
template <bool SYS>
__device__ __forceinline__ bool rs_arrive(uint32_t *counter, uint32_t target, int *flag,
                                          int nthreads) {
  if (SYS) __threadfence_system(); else __threadfence();
  named_bar_sync(1, nthreads);
  if (threadIdx.x == 128) {   // first epilogue thread
    const uint32_t old = SYS ? atomicAdd_system(counter, 1u) : atomicAdd(counter, 1u);
    const int last = old == target - 1;
    if (last) {
      if (SYS) atomicExch_system(counter, 0u); else atomicExch(counter, 0u);
    }
    *flag = last;
  }
  named_bar_sync(1, nthreads);
  const bool last = *(volatile int *)flag != 0;
  if (last) {
    if (SYS) __threadfence_system(); else __threadfence();
  }
  return last;
}

template <int CG>
__device__ __forceinline__ void tma_load(void *dst, const void *tmap, uint64_t *bar, int32_t c0,
                                         int32_t c1, int32_t c2) {
  if constexpr (CG == 1) tma_load_3d(dst, tmap, bar, c0, c1, c2);
  else tma_load_3d_cg2(dst, tmap, bar, c0, c1, c2);
}

// CN = 2 (CTA pairs only): a cluster of two pairs computes the two tiles
// (tm, 2j) and (tm, 2j+1) of one schedule unit; both need the same A rows,
// so each CTA loads HALF of its A k-block and multicasts it to its
// counterpart in the other pair — L2->SM bytes per flop drop by 1/4 (1/6 for
// 512-wide tiles), which on the power-capped B200 buys clock.  The A halves
// are 2-CTA multicast loads whose bytes complete on each destination pair's
// leader barrier, so full[s] still expects the pair's whole stage.  A stage
// is refilled only after BOTH pairs' MMAs released it (empty[] counts CN
// commits, multicast to all four CTAs).
template <int BN, int CG, typename OutT, int IN_BYTES, bool RS = false, int CN = 1>
__global__ void __launch_bounds__(NUM_THREADS, 1)
tc_gemm_kernel(const __grid_constant__ CUtensorMap tmap_a,
               const __grid_constant__ CUtensorMap tmap_b,
               const __grid_constant__ CUtensorMap tmap_o, const TcParams p) {
  using C = Cfg<BN, CG, (int)sizeof(OutT), IN_BYTES>;
  using E = typename C::E;
  constexpr int BK = E::BK;
  constexpr int MAX_STAGES = C::STAGES;
  const int STAGES = p.stages;
  constexpr int BN_CTA = C::BN_CTA;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t *smem_a = smem;
  uint8_t *smem_b = smem + MAX_STAGES * A_STAGE_BYTES;
  uint8_t *smem_epi = smem + MAX_STAGES * C::STAGE_BYTES;   // 1024-B aligned
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem_epi + C::EPI_BYTES);
  uint64_t *full = bars;
  uint64_t *empty = bars + MAX_STAGES;
  uint64_t *tmem_full = bars + 2 * MAX_STAGES;
  uint64_t *tmem_empty = bars + 2 * MAX_STAGES + 2;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 2 * MAX_STAGES + 4);
  int *rs_flag = reinterpret_cast<int *>(tmem_slot + 1);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  static_assert(CN == 1 || (CG == 2 && IN_BYTES == 2 && !RS), "A multicast: CTA pairs, 16-bit");
  constexpr int CL = CG * CN;                       // CTAs per cluster
  const uint32_t crank = CL == 1 ? 0 : cluster_ctarank();
  const uint32_t rank = crank & (uint32_t)(CG - 1); // rank inside the CTA pair
  const uint32_t pair = CN == 1 ? 0 : crank >> 1;   // which pair of the cluster
  const uint16_t pair_mask = (uint16_t)(0x3u << (2 * pair));
  const bool leader = rank == 0;
  const int64_t cluster_id = blockIdx.x / CL;
  const int64_t num_clusters = gridDim.x / CL;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmap_a);
    prefetch_tmap(&tmap_b);
    if (p.tma_store && !BGX_EPI_LSU) prefetch_tmap(&tmap_o);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CN);   // one commit per pair of the cluster
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tmem_full[a], 1);
      mbar_init(&tmem_empty[a], EPI_WARPS * CG);  // one arrive per epilogue warp per CTA
    }
    fence_barrier_init();
  }
  if (warp == 2) {
    tmem_alloc<CG>(tmem_slot, C::TMEM_COLS);
    tmem_relinquish<CG>();
  }
  tc_fence_before();
  if constexpr (CL == 1) __syncthreads(); else cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ===== TMA producer (every CTA loads its own A rows / B columns) =====
    // Warp-uniform loop; one elected lane issues the barrier ops and copies.
    // Clusters start staggered (a few hundred ns apart) so that the epilogue
    // store bursts of different SMs do not coincide: with equal tile times the
    // offset persists for the whole persistent loop.
    if (C::ACC_BUFS == 1 && !(p.debug & 8)) {
      const unsigned delay = (unsigned)(cluster_id % 16) * 256u;
      if (delay) __nanosleep(delay);
    }
    int stage = 0;
    uint32_t phase = 0;
    int trace_i = 0;
    for (int64_t u = cluster_id; u < p.num_units; u += num_clusters) {
      if ((p.debug & 4096) && lane == 0 && blockIdx.x < TR_CTAS && trace_i < TR_UNITS) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_trace[blockIdx.x * TR_UNITS + trace_i] = t;
      }
      ++trace_i;
      const UnitInfo ui = unit_info(p, u);
      const int64_t t = ui.t;
      const int kb_lo = ui.kb_lo, kb_hi = ui.kb_lo + ui.nkb;
      int64_t b, tm, tn;
      tile_coords(p, t, b, tm, tn);
      tn = tn * CN + pair;
      const int32_t m0 = (int32_t)(tm * C::TILE_M + rank * BM);
      // B columns of this CTA: for each MMA split h, [h*MMA_N + rank*B_BOX_N, +B_BOX_N)
      const int32_t n0 = (int32_t)(tn * BN + rank * C::B_BOX_N);
      const int32_t bb = (int32_t)b;
      for (int kb = kb_lo; kb < kb_hi; ++kb) {
        mbar_wait(&empty[stage], phase ^ 1);
        if (elect_one()) {
          if (leader) mbar_expect_tx(&full[stage], CG * C::STAGE_BYTES);
          const int32_t k0 = kb * BK;  // in elements
          uint8_t *sa = smem_a + stage * A_STAGE_BYTES;
          uint8_t *sb = smem_b + stage * C::B_STAGE_BYTES;
          if constexpr (CN == 2) {
            // my half of the A rows, multicast to me and my counterpart
            const uint16_t amask = (uint16_t)((1u << rank) | (1u << (rank + 2)));
            if (p.a_mn)
              tma_load_3d_cg2_mc(sa + pair * E::BOX_BYTES, &tmap_a, &full[stage],
                                 m0 + E::MN_ATOM * (int32_t)pair, k0, bb, amask);
            else
              tma_load_3d_cg2_mc(sa + pair * (A_STAGE_BYTES / 2), &tmap_a, &full[stage], k0,
                                 m0 + (BM / 2) * (int32_t)pair, bb, amask);
          } else if (p.a_mn) {
#pragma unroll
            for (int j = 0; j < BM / E::MN_ATOM; ++j)
              tma_load<CG>(sa + j * E::BOX_BYTES, &tmap_a, &full[stage], m0 + E::MN_ATOM * j, k0, bb);
          } else {
            tma_load<CG>(sa, &tmap_a, &full[stage], k0, m0, bb);
          }
#pragma unroll
          for (int h = 0; h < C::NSPLIT; ++h) {
            uint8_t *sbh = sb + h * C::B_HALF_BYTES;
            const int32_t nh = n0 + h * C::MMA_N;
            if (p.b_mn) {
#pragma unroll
              for (int j = 0; j < C::B_BOX_N / E::MN_ATOM; ++j)
                tma_load<CG>(sbh + j * E::BOX_BYTES, &tmap_b, &full[stage], nh + E::MN_ATOM * j,
                             k0, bb);
            } else {
              tma_load<CG>(sbh, &tmap_b, &full[stage], k0, nh, bb);
            }
          }
        }
        __syncwarp();
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    if (leader) {
      // ===== MMA issuer: warp-uniform loop, one elected lane issues =====
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      // Descriptor = {lo: start>>4 | LBO>>4 << 16, hi: SBO>>4 | version | SW128}:
      // only the start-address field moves along K, so precompute the rest.
      // per-MMA K advance: 32 bytes along a K-major row, or MMA_K rows of 128 B
      // for MN-major; MN-major LBO = one box (MN_ATOM x BK), SBO = 8 rows
      // 32-bit MN-major operands use the SWIZZLE_128B_BASE32B layout (32-byte
      // chunks swizzled within 128 B, 4-row atoms: SBO = 512 B) — the TMA map
      // of such operands uses CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B to match.
      constexpr uint32_t MN_STEP = E::MMA_K * ROW_BYTES;
      constexpr uint32_t MN_LAYOUT = IN_BYTES == 4 ? 1u : 2u;
      constexpr uint32_t MN_SBO = IN_BYTES == 4 ? 512u : 1024u;
      const uint32_t a_step = (p.a_mn ? MN_STEP : 32u) >> 4, b_step = (p.b_mn ? MN_STEP : 32u) >> 4;
      const uint64_t a_fixed = p.a_mn ? make_sdesc_sw128(0, E::BOX_BYTES, MN_SBO, MN_LAYOUT)
                                      : make_sdesc_sw128(0, 16u, 1024);
      const uint64_t b_fixed = p.b_mn ? make_sdesc_sw128(0, E::BOX_BYTES, MN_SBO, MN_LAYOUT)
                                      : make_sdesc_sw128(0, 16u, 1024);
      // the descriptor's start-address field holds bits [4,18) of the CTA-local
      // shared address; inside a cluster the shared::cta address also carries
      // the CTA rank in its upper bits (bit 24+), which must not spill into
      // the LBO field (it did for the second pair of a 4-CTA cluster)
      const uint32_t sa0 = (smem_u32(smem_a) & 0x3FFFFu) >> 4;
      const uint32_t sb0 = (smem_u32(smem_b) & 0x3FFFFu) >> 4;
      // With a single 512-column accumulator (BN = 512) the two N = 256 halves
      // are released separately by the epilogue (tmem_empty[0] = columns
      // [0,256), tmem_empty[1] = [256,512)): the next tile's first-half MMAs
      // run over every resident stage while the second half still drains.
      constexpr bool SPLIT_RELEASE = C::ACC_BUFS == 1 && C::NSPLIT == 2;
      auto issue = [&](int st, int kb, int h_lo, int h_hi, uint32_t d_tmem) {
        const uint64_t ad0 = a_fixed | (uint64_t)(sa0 + st * (A_STAGE_BYTES >> 4));
        const uint64_t bd0 = b_fixed | (uint64_t)(sb0 + st * (C::B_STAGE_BYTES >> 4));
#pragma unroll
        for (int k = 0; k < BK / E::MMA_K; ++k)
#pragma unroll
          for (int h = 0; h < C::NSPLIT; ++h)
            if (h >= h_lo && h < h_hi)
              umma<CG, IN_BYTES>(d_tmem + h * C::MMA_N, ad0 + k * a_step,
                                 bd0 + h * (C::B_HALF_BYTES >> 4) + k * b_step, p.idesc,
                                 (kb | k) != 0);
      };
      auto release = [&](int st) {
        if constexpr (CG == 1) umma_commit(&empty[st]);
        else umma_commit_mc(&empty[st], CN == 2 ? (uint16_t)0xF : (uint16_t)0x3);
      };
      for (int64_t u = cluster_id; u < p.num_units; u += num_clusters, ++it) {
        const int nkb = unit_info(p, u).nkb;
        const int acc = it % C::ACC_BUFS;
        const uint32_t acc_phase = (it / C::ACC_BUFS) & 1;
        const uint32_t d_tmem = tmem_base + acc * BN;
        int kb = 0;
        auto commit_full = [&](int which) {
          if (elect_one()) {
            if constexpr (CG == 1) umma_commit(&tmem_full[which]);
            else umma_commit_mc(&tmem_full[which], pair_mask);
          }
          __syncwarp();
        };
        // resident stages [kb, kb + n): every first-half MMA, then (after
        // `between`) every second-half MMA, releasing each stage
        auto split_pass = [&](int kb0, int n, auto &&between) {
          const int stage0 = stage;
          const uint32_t phase0 = phase;
          for (int e = 0; e < n; ++e) {
            mbar_wait(&full[stage], phase);
            tc_fence_after();
            if (elect_one()) issue(stage, kb0 + e, 0, 1, d_tmem);
            __syncwarp();
            if (++stage == STAGES) { stage = 0; phase ^= 1; }
          }
          between();
          stage = stage0;
          phase = phase0;
          for (int e = 0; e < n; ++e) {
            if (elect_one()) {
              issue(stage, kb0 + e, 1, 2, d_tmem);
              release(stage);
            }
            __syncwarp();
            if (++stage == STAGES) { stage = 0; phase ^= 1; }
          }
        };
        if constexpr (SPLIT_RELEASE) {
          // Tile start: the first half runs over the resident stages while
          // the epilogue still drains the previous tile's second half.  Tile
          // end: the last resident stages issue every first-half MMA, commit
          // the first half (tmem_full[0]), then the second halves (tmem_full[1])
          // — the epilogue reads columns [0,256) while the tensor core is
          // still busy on [256,512), so the single accumulator never idles it.
          const int early_max = (p.debug >> 20) & 7 ? (p.debug >> 20) & 7 : STAGES;   // A/B knob
          const int early_cap = early_max < STAGES ? early_max : STAGES;
          const int early = nkb < early_cap ? nkb : early_cap;
          const int late_max = (p.debug >> 16) & 7 ? (p.debug >> 16) & 7 : LATE_STAGES;
          const int late_cap = late_max < STAGES ? late_max : STAGES;
          const int late = (nkb - early) < late_cap ? (nkb - early) : late_cap;
          mbar_wait(&tmem_empty[0], acc_phase ^ 1);
          tc_fence_after();
          split_pass(0, early, [&] {
            if (late == 0) commit_full(0);            // all of the first half issued
            mbar_wait(&tmem_empty[1], acc_phase ^ 1);
            tc_fence_after();
          });
          for (kb = early; kb < nkb - late; ++kb) {
            mbar_wait(&full[stage], phase);
            tc_fence_after();
            if (elect_one()) {
              issue(stage, kb, 0, 2, d_tmem);
              release(stage);
            }
            __syncwarp();
            if (++stage == STAGES) { stage = 0; phase ^= 1; }
          }
          if (late > 0) split_pass(nkb - late, late, [&] { commit_full(0); });
          commit_full(1);
        } else {
          mbar_wait(&tmem_empty[acc], acc_phase ^ 1);
          tc_fence_after();
          for (; kb < nkb; ++kb) {
            mbar_wait(&full[stage], phase);
            tc_fence_after();
            if (elect_one()) {
              issue(stage, kb, 0, C::NSPLIT, d_tmem);
              release(stage);
            }
            __syncwarp();
            if (++stage == STAGES) { stage = 0; phase ^= 1; }
          }
          commit_full(acc);
        }
      }
    }
  } else if (warp >= 4) {
    // ===== epilogue (every CTA drains its own 128 TMEM lanes) =====
    // 8 warps: warp w reads TMEM lane quadrant w % 4 (hardware rule) and the
    // column chunks c = g, g + 2, ... of it (g = which of the two warps on that
    // quadrant); the next chunk's tcgen05.ld is in flight while the current
    // one is converted, staged and stored.
    const int ew = warp - 4;
    const int quad = warp % 4;  // TMEM lanes [32*quad, 32*quad + 32)
    const int g = ew / 4;
    uint8_t *ebuf = smem_epi + ew * 2 * C::EPI_BUF_BYTES;
    int it = 0, chunk = 0;
    for (int64_t u = cluster_id; u < p.num_units; u += num_clusters, ++it) {
      const UnitInfo ui = unit_info(p, u);
      const int64_t t = ui.t;
      int64_t b, tm, tn;
      tile_coords(p, t, b, tm, tn);
      tn = tn * CN + pair;
      b += ui.kslice * p.batch;  // uniform split-K slices are extra output batches
      // tail-split partial: f32 block of the workspace for this slice, stored
      // column-major inside each 32-column chunk ([c][j][row]) so that a
      // warp's 32 rows of one column are one coalesced 128-byte line
      const int row_in_tile = (int)(rank * BM + quad * 32 + lane);
      const bool tail = ui.slot >= 0;
      const int64_t tt = p.num_tiles - p.tail_start;
      const bool finisher = tail && ui.slot / tt == p.tail_splits - 1;
      float *wsrow = tail && !finisher
                         ? p.ws + ui.slot * (int64_t)C::TILE_M * BN + row_in_tile : nullptr;
      uint32_t *tcount = tail ? p.tail_counters + (t - p.tail_start) * CG + rank : nullptr;
      const int acc = it % C::ACC_BUFS;
      const uint32_t acc_phase = (it / C::ACC_BUFS) & 1;
      // One epilogue warp polls the accumulator barrier; the other seven wait
      // in a named barrier, which issues nothing (ncu: with all eight warps
      // polling, the wait loop was half of the kernel's instructions — issue
      // energy on a power-capped part)
      if (ew == 0) mbar_wait(&tmem_full[acc], acc_phase);
      named_bar_sync(2, 32 * EPI_WARPS);
      tc_fence_after();
      constexpr bool SPLIT_RELEASE = C::ACC_BUFS == 1 && C::NSPLIT == 2;
      // SPLIT_RELEASE: tmem_full[0] signals columns [0,256), tmem_full[1]
      // the whole tile.  Only the two-phase drain reads the first half early;
      // every other path waits for the whole tile here.
      auto wait_second_half = [&] {
        if (ew == 0) mbar_wait(&tmem_full[1], acc_phase);
        named_bar_sync(2, 32 * EPI_WARPS);
        tc_fence_after();
      };
      if constexpr (SPLIT_RELEASE) {
        const bool two_phase = !RS && sizeof(OutT) == 2 && p.tma_store && p.c0 == nullptr &&
                               !(p.debug & 5) && !tail;
        if (!two_phase) wait_second_half();
      }
      auto arrive_empty = [&](int which) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if constexpr (CG == 1) mbar_arrive(&tmem_empty[which]);
          else mbar_arrive_cluster(&tmem_empty[which], 2 * pair);   // own pair's leader
        }
      };
      if (p.debug & 4) {  // timing probe: release the accumulator without reading it
        arrive_empty(acc);
        if (SPLIT_RELEASE) arrive_empty(1);
        continue;
      }
      const int64_t m_warp = tm * C::TILE_M + rank * BM + quad * 32;
      const int64_t m = m_warp + lane;
      const bool row_ok = m < p.M;
      const uint32_t taddr = tmem_base + ((uint32_t)(quad * 32) << 16) + acc * BN;
      constexpr int NCHUNK = BN / 32;
      if constexpr (RS) {
        // ===== fused K-split reduce-scatter (bgx_contract_reduce_scatter) =====
        // owner of this CTA's 128 rows (rows_per_owner is a multiple of 128,
        // so the two CTAs of a pair may deliver to different owners) and the
        // row inside the owner's slab
        const int owner = (int)((tm * C::TILE_M + rank * BM) / p.rs_rpo);
        const int64_t lrow = m - (int64_t)owner * p.rs_rpo;
        const int64_t cidx = t * CG + rank;   // one counter per CTA half of a tile
        const int S = p.k_splits;
        float *slot_row = p.rs_slots[owner] + ((int64_t)p.rs_rank * p.rs_rpo + lrow) * p.N;
        float *dst = p.rs_defer
            ? p.rs_slots[owner] + (((int64_t)p.rs_rank * S + ui.kslice) * p.rs_rpo + lrow) * p.N
            : (S > 1 ? p.ws + (ui.kslice * p.M + m) * p.N : slot_row);
        // (1) TMEM -> f32 partial rows (local split slice, or straight into
        //     the owner's slot over NVLink)
        uint32_t rbuf[2][32];
        tmem_ld_32x32b_x32(taddr + g * 32, rbuf[0]);
#pragma unroll 1
        for (int c = g, k = 0; c < NCHUNK; c += 2, ++k) {
          tmem_ld_wait();
          uint32_t (&r)[32] = rbuf[k & 1];
          if (c + 2 < NCHUNK) tmem_ld_32x32b_x32(taddr + (c + 2) * 32, rbuf[(k + 1) & 1]);
          const int64_t n = tn * BN + c * 32;
          if (n >= p.N || !row_ok) continue;
          float v[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
          Store<float>::row32(dst + n, v, p.N - n >= 32, p.N - n);
        }
        tmem_ld_wait();
        arrive_empty(acc);
        if (p.rs_defer) {
          // delivered; the owner's bgx_rs_reduce sums after the caller's
          // barrier — make this thread's peer stores visible system-wide
          // before the kernel can be seen as finished
          __threadfence_system();
          continue;
        }
        // a CTA half entirely below the last output row has no owner (its
        // rows do not exist): nothing to deliver, no counter to bump
        if (tm * C::TILE_M + rank * BM >= p.M) continue;
        constexpr int NT = 32 * EPI_WARPS;
        // (2) local split-K: the last slice of this tile sums the slices in
        //     slice order and forwards the rank's partial to the owner
        if (S > 1) {
          if (!rs_arrive<false>(p.rs_ws_counters + cidx, (uint32_t)S, rs_flag, NT)) continue;
          if (row_ok) {
#pragma unroll 1
            for (int c = g; c < NCHUNK; c += 2) {
              const int64_t n = tn * BN + c * 32;
              if (n >= p.N) continue;
              const int64_t valid = p.N - n;
              float v[32], w[32];
              load_row32_sys(p.ws + m * p.N + n, v, valid);
              for (int sl = 1; sl < S; ++sl) {
                load_row32_sys(p.ws + ((int64_t)sl * p.M + m) * p.N + n, w, valid);
#pragma unroll
                for (int j = 0; j < 32; ++j) v[j] = __fadd_rn(v[j], w[j]);
              }
              Store<float>::row32(slot_row + n, v, valid >= 32, valid);
            }
          }
        }
        // (3) cross-rank: the last rank to deliver this tile reduces the
        //     owner's slots in rank order, adds c0 and writes the output
        if (!rs_arrive<true>(p.rs_counters[owner] + cidx, (uint32_t)p.rs_world, rs_flag, NT))
          continue;
        if (row_ok) {
          const float *slot0 = p.rs_slots[owner] + lrow * p.N;
          const int64_t slot_stride = p.rs_rpo * p.N;
          const int oes = p.rs_out_dtype == BGX_F32 ? 4 : 2;
          uint8_t *orow_rs = static_cast<uint8_t *>(p.rs_out[owner]) + lrow * p.so[1] * oes;
          const uint8_t *crow_rs = p.rs_c0[owner]
              ? static_cast<const uint8_t *>(p.rs_c0[owner]) + lrow * p.sc[1] * oes : nullptr;
#pragma unroll 1
          for (int c = g; c < NCHUNK; c += 2) {
            const int64_t n = tn * BN + c * 32;
            if (n >= p.N) continue;
            const int64_t valid = p.N - n;
            float v[32], w[32];
            load_row32_sys(slot0 + n, v, valid);
            for (int rk = 1; rk < p.rs_world; ++rk) {
              load_row32_sys(slot0 + rk * slot_stride + n, w, valid);
#pragma unroll
              for (int j = 0; j < 32; ++j) v[j] = __fadd_rn(v[j], w[j]);
            }
            if (p.rs_out_dtype == BGX_F32) {
              if (crow_rs)
                for (int j = 0; j < 32; ++j)
                  if (j < valid) v[j] = __fadd_rn(v[j], ld_sys((const float *)crow_rs + n + j));
              Store<float>::row32((float *)orow_rs + n, v, valid >= 32, valid);
            } else if (p.rs_out_dtype == BGX_BF16) {
              if (crow_rs)
                for (int j = 0; j < 32; ++j)
                  if (j < valid)
                    v[j] = __fadd_rn(v[j], Conv<__nv_bfloat16>::to_f(
                                               ((const __nv_bfloat16 *)crow_rs)[n + j]));
              Store<__nv_bfloat16>::row32((__nv_bfloat16 *)orow_rs + n, v, valid >= 32, valid);
            } else {
              if (crow_rs)
                for (int j = 0; j < 32; ++j)
                  if (j < valid)
                    v[j] = __fadd_rn(v[j], Conv<__half>::to_f(((const __half *)crow_rs)[n + j]));
              Store<__half>::row32((__half *)orow_rs + n, v, valid >= 32, valid);
            }
          }
        }
        continue;
      } else {
      OutT *orow = static_cast<OutT *>(p.out) + b * p.so[0] + m * p.so[1];
      const OutT *crow = p.c0 ? static_cast<const OutT *>(p.c0) + b * p.sc[0] + m * p.sc[1] : nullptr;
      if constexpr (SPLIT_RELEASE && sizeof(OutT) == 2) {
        if (p.tma_store && crow == nullptr && !(p.debug & 1) && !tail) {
          // Two-phase drain: read this warp's chunks of each accumulator half
          // into packed 16-bit registers, release that half of TMEM to the MMA
          // warp, and only then stage + TMA-store — the stores (and their
          // buffer waits) leave the MMA critical path.
          constexpr int PER_HALF = NCHUNK / 2 / 2;  // chunks per warp per half
#if BGX_EPI_DRAIN_BOTH
          // drain BOTH halves into registers before any store: the next
          // tile's second-half MMAs wait only for the TMEM reads
          uint32_t pk2[2][PER_HALF][16];
#pragma unroll
          for (int half = 0; half < 2; ++half) {
            if (half == 1) wait_second_half();
#pragma unroll
            for (int j = 0; j < PER_HALF; ++j) {
              const int c = half * (NCHUNK / 2) + g + 2 * j;
              uint32_t r[32];
              tmem_ld_32x32b_x32(taddr + c * 32, r);
              tmem_ld_wait();
#pragma unroll
              for (int q = 0; q < 16; ++q)
                pk2[half][j][q] = pack2<OutT>(__uint_as_float(r[2 * q]), __uint_as_float(r[2 * q + 1]));
            }
            arrive_empty(half);
          }
#pragma unroll
          for (int half = 0; half < 2; ++half) {
            uint32_t (&pk)[PER_HALF][16] = pk2[half];
#else
#pragma unroll 1
          for (int half = 0; half < 2; ++half) {
            if (half == 1) wait_second_half();
            uint32_t pk[PER_HALF][16];
#pragma unroll
            for (int j = 0; j < PER_HALF; ++j) {
              const int c = half * (NCHUNK / 2) + g + 2 * j;
              uint32_t r[32];
              tmem_ld_32x32b_x32(taddr + c * 32, r);
              tmem_ld_wait();
#pragma unroll
              for (int q = 0; q < 16; ++q)
                pk[j][q] = pack2<OutT>(__uint_as_float(r[2 * q]), __uint_as_float(r[2 * q + 1]));
            }
            arrive_empty(half);   // this half of TMEM is free for the next tile
#endif
#pragma unroll
            for (int j = 0; j < PER_HALF; ++j) {
              const int c = half * (NCHUNK / 2) + g + 2 * j;
              const int64_t n = tn * BN + c * 32;
              if (n >= p.N) continue;
              uint8_t *buf = ebuf + (chunk & 1) * C::EPI_BUF_BYTES;
              ++chunk;
              if (!BGX_EPI_LSU && lane == 0) bulk_wait_read<1>();
              __syncwarp();
#pragma unroll
              for (int v4 = 0; v4 < 4; ++v4) {
                uint4 w = make_uint4(pk[j][4 * v4], pk[j][4 * v4 + 1], pk[j][4 * v4 + 2],
                                     pk[j][4 * v4 + 3]);
                *reinterpret_cast<uint4 *>(buf + lane * 64 + ((v4 ^ ((lane >> 1) & 3)) << 4)) = w;
              }
#if BGX_EPI_LSU
              __syncwarp();
              lsu_store_chunk<OutT>(buf, static_cast<OutT *>(p.out) + b * p.so[0] + m_warp * p.so[1] + n,
                                    p.so[1], p.M - m_warp, p.N - n, lane);
#else
              fence_proxy_async_smem();
              __syncwarp();
              if (lane == 0) {
                tma_store_3d(&tmap_o, buf, (int32_t)n, (int32_t)m_warp, (int32_t)b);
                bulk_commit();
              }
#endif
            }
          }
          continue;
        }
      }
      // one 32-column chunk of this thread's output row: TMA store through the
      // warp's swizzled staging buffer, or direct stores
      auto store_out = [&](const float *v, int64_t n, int64_t valid) {
        if (p.tma_store) {
          uint8_t *buf = ebuf + (chunk & 1) * C::EPI_BUF_BYTES;
          ++chunk;
          if (!BGX_EPI_LSU && lane == 0) bulk_wait_read<1>();   // the buffer used two chunks ago is free
          __syncwarp();
          stage_row32<OutT>(buf, lane, v);
#if BGX_EPI_LSU
          __syncwarp();
          lsu_store_chunk<OutT>(buf, static_cast<OutT *>(p.out) + b * p.so[0] + m_warp * p.so[1] + n,
                                p.so[1], p.M - m_warp, p.N - n, lane);
#else
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_3d(&tmap_o, buf, (int32_t)n, (int32_t)m_warp, (int32_t)b);
            bulk_commit();
          }
#endif
        } else if (row_ok) {
          Store<OutT>::row32(orow + n, v, valid >= 32, valid);
        }
      };
      if (finisher) {   // wait until the tile's other K slices stored their partials
        if (threadIdx.x == 128)
          while (ld_acquire_gpu(tcount) < (uint32_t)(p.tail_splits - 1)) __nanosleep(64);
        named_bar_sync(1, 32 * EPI_WARPS);
        __threadfence();
      }
      if (finisher) {
        // (((0 + p_0) + p_1) + ...) + own slice: fixed order whatever the timing
        const float *part0 = p.ws + (t - p.tail_start) * (int64_t)C::TILE_M * BN + row_in_tile;
#pragma unroll 1
        for (int c = g; c < NCHUNK; c += 2) {
          uint32_t r[32];
          tmem_ld_32x32b_x32(taddr + c * 32, r);
          tmem_ld_wait();
          if (SPLIT_RELEASE && c >= NCHUNK / 2 && c - 2 < NCHUNK / 2)
            arrive_empty(0);  // every chunk of columns [0, BN/2) has been read
          const int64_t n = tn * BN + c * 32;
          if (n >= p.N) continue;
          const int64_t valid = p.N - n;
          float v[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = 0.f;
          for (int sl = 0; sl < p.tail_splits - 1; ++sl) {
            const float *wc = part0 + sl * tt * (int64_t)C::TILE_M * BN +
                              (int64_t)(c * 32) * C::TILE_M;
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = __fadd_rn(v[j], __ldcg(wc + j * C::TILE_M));
          }
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = __fadd_rn(v[j], __uint_as_float(r[j]));
          if (crow && row_ok)
            for (int j = 0; j < 32; ++j)
              if (j < valid) v[j] = __fadd_rn(v[j], Conv<OutT>::to_f(crow[n + j]));
          store_out(v, n, valid);
        }
        arrive_empty(SPLIT_RELEASE ? 1 : acc);
        continue;
      }
      uint32_t rbuf[2][32];
      tmem_ld_32x32b_x32(taddr + g * 32, rbuf[0]);
#pragma unroll 2
      for (int c = g, k = 0; c < NCHUNK; c += 2, ++k) {
        tmem_ld_wait();
        uint32_t (&r)[32] = rbuf[k & 1];
        if (SPLIT_RELEASE && c >= NCHUNK / 2 && c - 2 < NCHUNK / 2)
          arrive_empty(0);  // every chunk of columns [0, BN/2) has been read
        if (c + 2 < NCHUNK) tmem_ld_32x32b_x32(taddr + (c + 2) * 32, rbuf[(k + 1) & 1]);
        const int64_t n = tn * BN + c * 32;
        if (n >= p.N || (p.debug & 1)) continue;  // warp-uniform
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
        const int64_t valid = p.N - n;
        if (crow && row_ok && wsrow == nullptr) {
          for (int j = 0; j < 32; ++j)
            if (j < valid) v[j] = __fadd_rn(v[j], Conv<OutT>::to_f(crow[n + j]));
        }
        if (wsrow != nullptr) {
          float *wc = wsrow + (int64_t)(c * 32) * C::TILE_M;
#pragma unroll
          for (int j = 0; j < 32; ++j) __stcg(wc + j * C::TILE_M, v[j]);
        } else {
          store_out(v, n, valid);
        }
      }
      tmem_ld_wait();
      arrive_empty(SPLIT_RELEASE ? 1 : acc);
      if (wsrow != nullptr) {   // publish this slice's partial to the finisher
        __threadfence();
        named_bar_sync(1, 32 * EPI_WARPS);
        if (threadIdx.x == 128) atomicAdd(tcount, 1u);
      }
      }  // !RS
    }
    if (lane == 0) bulk_wait_all();
    __syncwarp();
  }
  tc_fence_before();
  if constexpr (CL == 1) __syncthreads(); else cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<CG>(tmem_base, C::TMEM_COLS);
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

// 3-D map: dims (inner, outer, batch) with element strides (1, s_outer,
// s_batch); box (box_inner, box_outer, 1); 128B swizzle unless given.
int make_map(CUtensorMap *map, const void *base, CUtensorMapDataType dt, int64_t inner,
             int64_t outer, int64_t batch, int64_t s_outer, int64_t s_batch, uint32_t box_inner,
             uint32_t box_outer, int esize = 2,
             CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
  auto enc = get_encode();
  if (!enc) { set_error("cuTensorMapEncodeTiled unavailable"); return BGX_ERR_CUDA; }
  cuuint64_t dims[3] = {(cuuint64_t)inner, (cuuint64_t)outer, (cuuint64_t)batch};
  if (batch <= 1) s_batch = s_outer * outer;  // any legal value; never stepped
  cuuint64_t strides[2] = {(cuuint64_t)(s_outer * esize), (cuuint64_t)(s_batch * esize)};
  cuuint32_t box[3] = {box_inner, box_outer, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, dt, 3, const_cast<void *>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d): dims %lld x %lld x %lld strides %lld/%lld",
              (int)r, (long long)inner, (long long)outer, (long long)batch,
              (long long)s_outer, (long long)s_batch);
    return BGX_ERR_INVALID;
  }
  return BGX_OK;
}

// Max co-resident clusters for a kernel config, cached per (device, kernel).
template <typename K>
int max_clusters(K kern, int smem, int cg) {
  int n = 0;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2 * 148);
  cfg.blockDim = dim3(NUM_THREADS);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cg;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

template <int BN, int CG, typename OutT, int IN_BYTES, bool RS = false, int CN = 1>
int launch_tc(const bgx_contract_desc &d, const TcParams &p0, cudaStream_t s) {
  using C = Cfg<BN, CG, (int)sizeof(OutT), IN_BYTES>;
  using E = typename C::E;
  TcParams p = p0;
  const CUtensorMapDataType dt = IN_BYTES == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                 : d.in_dtype == BGX_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                                          : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  CUtensorMap ma, mb;
  int rc;
  constexpr uint32_t AT = E::MN_ATOM, KB = E::BK;
  const CUtensorMapSwizzle mn_swz =
      IN_BYTES == 4 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B;
  if (p.a_mn)
    rc = make_map(&ma, d.a, dt, d.M, d.K, d.batch, d.a_stride[2], d.a_stride[0], AT, KB, IN_BYTES,
                  mn_swz);
  else
    rc = make_map(&ma, d.a, dt, d.K, d.M, d.batch, d.a_stride[1], d.a_stride[0], KB, BM / CN,
                  IN_BYTES);
  if (rc) return rc;
  if (p.b_mn)
    rc = make_map(&mb, d.b, dt, d.N, d.K, d.batch, d.b_stride[1], d.b_stride[0], AT, KB, IN_BYTES,
                  mn_swz);
  else
    rc = make_map(&mb, d.b, dt, d.K, d.N, d.batch, d.b_stride[2], d.b_stride[0], KB, C::B_BOX_N,
                  IN_BYTES);
  if (rc) return rc;
  // output map for the TMA-store epilogue (falls back to direct stores when
  // the output's row/batch strides are not 16-byte multiples)
  CUtensorMap mo;
  memset(&mo, 0, sizeof(mo));
  const int oes = (int)sizeof(OutT);
  p.tma_store = ((uintptr_t)d.out % 16 == 0) && (d.o_stride[1] * oes) % 16 == 0 &&
                (d.batch * (p.k_splits > 1 ? p.k_splits : 1) <= 1 ||
                 (d.o_stride[0] * oes) % 16 == 0) && !(p.debug & 2) && !RS;
  // (tma_store: the output allows the staged, coalesced epilogue; the map is
  // only needed when the chunks leave through TMA)
  if (p.tma_store && !BGX_EPI_LSU) {
    const CUtensorMapDataType odt = oes == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                   : (d.out_dtype == BGX_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                                              : CU_TENSOR_MAP_DATA_TYPE_FLOAT16);
    rc = make_map(&mo, d.out, odt, d.N, d.M, d.batch * p.k_splits, d.o_stride[1], d.o_stride[0],
                  32, 32, oes,
                  oes == 4 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B);
    if (rc) return rc;
  }
  p.idesc = IN_BYTES == 4 ? make_idesc_tf32(p.a_mn, p.b_mn, C::TILE_M, C::MMA_N)
                          : make_idesc_f16(d.in_dtype == BGX_BF16, p.a_mn, p.b_mn, C::TILE_M, C::MMA_N);
  p.stages = (d.sched.stages >= 2 && d.sched.stages <= C::STAGES) ? d.sched.stages : C::STAGES;
  p.tiles_m = (int32_t)((d.M + C::TILE_M - 1) / C::TILE_M);
  p.tiles_n = (int32_t)(((d.N + BN - 1) / BN + CN - 1) / CN);   // schedule units along N
  p.num_tiles = (int64_t)p.tiles_m * p.tiles_n * d.batch;
  if (p.k_splits < 1) p.k_splits = 1;
  if (RS) {
    // fused reduce-scatter: balanced slices, count kept (unit_info), so both
    // reduction placements sum the same slices and every rank fills the
    // same number of deferred slots
    p.kb_per_split = 0;
  } else {
    p.kb_per_split = (p.k_blocks + p.k_splits - 1) / p.k_splits;
    p.k_splits = (p.k_blocks + p.kb_per_split - 1) / p.kb_per_split;
  }
  p.num_units = p.num_tiles * p.k_splits;
  auto kern = tc_gemm_kernel<BN, CG, OutT, IN_BYTES, RS, CN>;
  constexpr int CL = CG * CN;
  static thread_local int configured[64] = {0};
  static thread_local int clusters[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!configured[dev & 63]) {
    RelaxedCaptureScope relaxed;
    BGX_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      C::SMEM_BYTES));
    configured[dev & 63] = 1;
    clusters[dev & 63] = CL == 1 ? sm_count_current() : max_clusters(kern, C::SMEM_BYTES, CL);
    if (clusters[dev & 63] <= 0) clusters[dev & 63] = sm_count_current() / CL;
  }
  int64_t nclusters = clusters[dev & 63];
  // tail split: only the tiles of the last, partial wave are split in K
  if (p.tail_splits > 1 && p.k_splits == 1 && p.ws != nullptr && CN == 1) {
    const int64_t slots = nclusters;
    p.tail_start = (p.num_tiles / slots) * slots;
    const int64_t tt = p.num_tiles - p.tail_start;
    p.kb_per_tail = (p.k_blocks + p.tail_splits - 1) / p.tail_splits;
    p.tail_splits = (p.k_blocks + p.kb_per_tail - 1) / p.kb_per_tail;
    const int64_t part = (tt * p.tail_splits * (int64_t)C::TILE_M * BN * 4 + 255) / 256 * 256;
    const int64_t need = part + tt * CG * 4;
    if (tt == 0 || p.tail_splits < 2 || need > p.ws_bytes) {
      p.tail_splits = 1;
      p.tail_start = p.num_tiles;
    } else {
      p.num_units = p.tail_start + tt * p.tail_splits;
      p.tail_counters = reinterpret_cast<uint32_t *>(reinterpret_cast<uint8_t *>(p.ws) + part);
      BGX_CUDA_TRY(cudaMemsetAsync(p.tail_counters, 0, tt * CG * 4, s));
    }
  } else {
    p.tail_splits = 1;
    p.tail_start = p.num_tiles;
  }
  if (p.num_units < nclusters) nclusters = p.num_units;
  if (d.sched.max_ctas > 0 && nclusters * CL > d.sched.max_ctas) nclusters = d.sched.max_ctas / CL;
  if (nclusters < 1) nclusters = 1;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)(nclusters * CL));
  cfg.blockDim = dim3(NUM_THREADS);
  cfg.dynamicSmemBytes = C::SMEM_BYTES;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  BGX_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, ma, mb, mo, p));
  return check_launch("tc_gemm_kernel");
}

// Co-resident 4-CTA clusters of the A-multicast kernel (a 4-CTA cluster must
// fit in one GPC: 33 on a 148-SM B200, i.e. 132 SMs busy), cached per device.
template <int BN, typename OutT>
int cn2_slots() {
  using C = Cfg<BN, 2, (int)sizeof(OutT), 2>;
  static thread_local int cache[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!cache[dev & 63]) {
    RelaxedCaptureScope relaxed;
    auto kern = tc_gemm_kernel<BN, 2, OutT, 2, false, 2>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_BYTES) !=
        cudaSuccess) {
      cudaGetLastError();
      cache[dev & 63] = -1;
    } else {
      const int n = max_clusters(kern, C::SMEM_BYTES, 4);
      cache[dev & 63] = n > 0 ? n : -1;
    }
  }
  return cache[dev & 63];
}

template <int CG, typename OutT, int IB = 2>
int dispatch_bn(const bgx_contract_desc &d, int bn, const TcParams &p, cudaStream_t s,
                int cn = 1) {
  if constexpr (CG == 2 && IB == 2) {
    // automatic A multicast: only when the 4-CTA clusters (fewer SMs, but a
    // quarter less L2->SM traffic per flop, hence higher clocks under the
    // power cap) need no more waves than CTA pairs do — e.g. 4096^3
    if (cn == 0 && (bn == 256 || bn == 512) && p.k_splits <= 1 && p.tail_splits <= 1) {
      const int64_t tm = (d.M + 255) / 256, tn = (d.N + bn - 1) / bn;
      const int64_t tiles = tm * tn * d.batch, units = tm * ((tn + 1) / 2) * d.batch;
      const int64_t slots2 = sm_count_current() / 2;
      const int64_t slots4 = bn == 512 ? cn2_slots<512, OutT>() : cn2_slots<256, OutT>();
      if (slots4 > 0 && (units + slots4 - 1) / slots4 <= (tiles + slots2 - 1) / slots2 &&
          tiles >= slots2)
        cn = 2;
    }
    if (cn == 2 && bn == 512) return launch_tc<512, 2, OutT, 2, false, 2>(d, p, s);
    if (cn == 2 && bn == 256) return launch_tc<256, 2, OutT, 2, false, 2>(d, p, s);
  }
  switch (bn) {
    case 64:
      return CG == 1 ? launch_tc<64, 1, OutT, IB>(d, p, s) : launch_tc<128, CG, OutT, IB>(d, p, s);
    case 128: return launch_tc<128, CG, OutT, IB>(d, p, s);
    case 512:
      return CG == 2 ? launch_tc<512, 2, OutT, IB>(d, p, s) : launch_tc<256, CG, OutT, IB>(d, p, s);
    default: return launch_tc<256, CG, OutT, IB>(d, p, s);
  }
}

// Uniform split-K count for `tiles` output tiles on `slots` persistent
// clusters: only when the tiles leave most clusters idle and every slice
// keeps >= 8 k-blocks (shared by the tile choice and tc_splitk_plan).
int64_t uniform_splits(int64_t tiles, int64_t slots, int64_t k_blocks) {
  if (tiles * 2 > slots || k_blocks < 16) return 1;
  int64_t sp = slots / tiles;
  if (sp > k_blocks / 8) sp = k_blocks / 8;
  if (sp > 32) sp = 32;
  return sp < 2 ? 1 : sp;
}

// Tile choice: minimise waves x per-CTA tile area / efficiency over the
// candidate (CG, BN) shapes.  A CTA's time per tile is proportional to its
// tile area at the full per-SM MMA rate, scaled by the shape's measured
// efficiency (round-1 sweeps on B200, scripts/sweep_gemm.py: narrower tiles
// pay relatively more epilogue / A-operand traffic per flop, single CTAs more
// L2->SM bytes of B).  Small outputs are costed with the split-K they would
// get (a unit is then 1/S of a tile's K, +10 % for the partial stores and
// the reduction pass), so wide tiles split in K beat narrow unsplit ones.
// A later candidate must be >3 % cheaper to win.
void choose_tile(const bgx_contract_desc &d, int sms, int &cg, int &bn) {
  struct Cand { int cg, bn; double eff; };
  const Cand cands[] = {{2, 512, 1.06}, {2, 256, 1.00}, {2, 128, 0.85}, {1, 256, 0.88},
                        {1, 128, 0.80}, {1, 64, 0.60}};
  const int BKe = d.in_dtype == BGX_F32 ? Elem<4>::BK : Elem<2>::BK;
  const int64_t k_blocks = (d.K + BKe - 1) / BKe;
  double best = -1.0;
  for (const Cand &c : cands) {
    if (c.bn > 64 && d.N <= c.bn / 2) continue;  // tiles would be mostly empty
    const int64_t tm = (d.M + 128 * c.cg - 1) / (128 * c.cg);
    const int64_t tn = (d.N + c.bn - 1) / c.bn;
    const int64_t slots = sms / c.cg;
    const int64_t tiles = tm * tn * d.batch;
    const int64_t sp = uniform_splits(tiles, slots, k_blocks);
    const int64_t waves = (tiles + slots - 1) / slots;
    const int64_t split_waves = (tiles * sp + slots - 1) / slots;
    double eff_waves = (double)split_waves / (double)sp * (sp > 1 ? 1.1 : 1.0);
    // a last wave at most half full gets the 2-way tail split (tc_splitk_plan)
    const int64_t tail = tiles % slots;
    if (sp == 1 && tiles >= slots && tail > 0 && tail * 2 <= slots && k_blocks >= 128)
      eff_waves = (double)(tiles / slots) + 0.55;
    // the 512-wide tile's single accumulator drains the MMA pipe at every
    // tile boundary: with few tiles per pair (<= 6 waves) that costs more
    // than its operand economy buys (rows x 8192 x 8192, round 2: 4096 rows
    // 352.8 -> 340.8 us, 6144 rows 546.7 -> 530.6 us with 256-wide tiles;
    // 8192 rows and up keep 512, profiles/r02_slab_tiles.txt)
    const double eff = (c.bn == 512 && waves <= 6) ? 0.97 : c.eff;
    const double cost = eff_waves * (double)(128 * c.bn) / eff;
    // single 512-column accumulator: its drain is amortised only over long K
    // and several waves (4096^3 measured faster with 256-wide tiles; 8192^3,
    // 7 waves, 5 % faster with 512: profiles/r01_tile512_8192.txt)
    if (c.bn == 512 && (d.N < 1024 || d.K < 8192 || waves < 4)) continue;
    if (best < 0 || cost < best * 0.97) {
      best = cost;
      cg = c.cg;
      bn = c.bn;
    }
  }
}

}  // namespace

// Legality of the TMA/tcgen05 path for a descriptor (see bgx.h).
bool tc_legal(const bgx_contract_desc &d, const char **why) {
  auto fail = [&](const char *w) { if (why) *why = w; return false; };
  const bool tf32 = d.in_dtype == BGX_F32 && d.mode == BGX_MODE_TF32;
  if (!(d.in_dtype == BGX_BF16 || d.in_dtype == BGX_F16 || tf32))
    return fail("inputs not bf16/f16 (or f32 with BGX_MODE_TF32)");
  if (!(d.out_dtype == d.in_dtype || d.out_dtype == BGX_F32)) return fail("out dtype");
  const int es = tf32 ? 4 : 2;

  if (d.M <= 0 || d.N <= 0 || d.K <= 0 || d.batch <= 0) return fail("empty extent");
  if (d.M >= (1ll << 31) || d.N >= (1ll << 31) || d.K >= (1ll << 31)) return fail("extent >= 2^31");
  const bool a_mn = d.a_stride[2] != 1 && d.a_stride[1] == 1;
  const bool a_k = d.a_stride[2] == 1;
  if (!a_mn && !a_k) return fail("A has no unit stride in m or k");
  const bool b_mn = d.b_stride[2] == 1;
  const bool b_k = !b_mn && d.b_stride[1] == 1;
  if (!b_mn && !b_k) return fail("B has no unit stride in k or n");
  auto al16 = [es](int64_t elems) { return (elems * es) % 16 == 0; };
  if (((uintptr_t)d.a % 16) || ((uintptr_t)d.b % 16)) return fail("A/B base not 16B aligned");
  if (a_k && (!al16(d.a_stride[1]) || (d.batch > 1 && !al16(d.a_stride[0])))) return fail("A strides");
  if (a_mn && (!al16(d.a_stride[2]) || (d.batch > 1 && !al16(d.a_stride[0])))) return fail("A strides");
  if (b_mn && (!al16(d.b_stride[1]) || (d.batch > 1 && !al16(d.b_stride[0])))) return fail("B strides");
  if (b_k && (!al16(d.b_stride[2]) || (d.batch > 1 && !al16(d.b_stride[0])))) return fail("B strides");
  if (d.o_stride[2] != 1) return fail("out n-stride != 1");
  if (d.c0 && d.c_stride[2] != 1) return fail("c0 n-stride != 1");
  return true;
}

void tc_tile_choice(const bgx_contract_desc &d, int *cg_out, int *bn_out);

namespace {
int contract_tc_impl(const bgx_contract_desc &d, int splits, cudaStream_t s, int tail_splits = 1,
                     void *ws = nullptr, int64_t ws_bytes = 0) {
  const char *why = nullptr;
  if (!tc_legal(d, &why)) {
    set_error("tensor-core path not legal: %s", why);
    return BGX_ERR_UNSUPPORTED;
  }
  TcParams p{};
  p.k_splits = splits;
  p.tail_splits = tail_splits;
  p.ws = static_cast<float *>(ws);
  p.ws_bytes = ws_bytes;
  p.batch = d.batch; p.M = d.M; p.N = d.N; p.K = d.K;
  p.a_mn = d.a_stride[2] != 1 ? 1 : 0;
  p.b_mn = d.b_stride[2] == 1 ? 1 : 0;
  const int BKe = d.in_dtype == BGX_F32 ? Elem<4>::BK : Elem<2>::BK;
  p.k_blocks = (int32_t)((d.K + BKe - 1) / BKe);
  if (p.k_splits > p.k_blocks) p.k_splits = p.k_blocks;
  if (p.k_splits < 1) p.k_splits = 1;
  p.c0 = d.c0; p.out = d.out;
  for (int i = 0; i < 3; ++i) { p.sc[i] = d.c_stride[i]; p.so[i] = d.o_stride[i]; }
  int cg = 0, bn = 0;
  tc_tile_choice(d, &cg, &bn);
  // default raster: 512-wide pair tiles keep an 8-N-tile slab of B (8 x 512
  // columns) L2-resident while A streams (-8); otherwise M-groups.
  p.raster = d.sched.raster != 0 ? d.sched.raster : (bn == 512 ? -8 : (cg == 2 ? 8 : 16));
  p.debug = d.sched.reserved[0];
  // two CTA pairs per cluster sharing A by multicast (schedule reserved[1]
  // = cluster_n: 0 automatic, 1 off, 2 on; never with the tail split, whose
  // workspace slots are per unit)
  const int cn = (cg != 2 || tail_splits > 1 || d.sched.reserved[1] == 1) ? 1
                 : d.sched.reserved[1] == 2 ? 2 : 0;
  if (d.in_dtype == BGX_F32)  // tf32 tensor cores (opt-in BGX_MODE_TF32)
    return cg == 2 ? dispatch_bn<2, float, 4>(d, bn, p, s) : dispatch_bn<1, float, 4>(d, bn, p, s);
  if (d.out_dtype == BGX_F32)
    return cg == 2 ? dispatch_bn<2, float>(d, bn, p, s, cn) : dispatch_bn<1, float>(d, bn, p, s);
  if (d.out_dtype == BGX_BF16)
    return cg == 2 ? dispatch_bn<2, __nv_bfloat16>(d, bn, p, s, cn)
                   : dispatch_bn<1, __nv_bfloat16>(d, bn, p, s);
  return cg == 2 ? dispatch_bn<2, __half>(d, bn, p, s, cn) : dispatch_bn<1, __half>(d, bn, p, s);
}

// out[b,m,n] = (c0) + sum_s ws[s][b][m][n], summed in increasing s (deterministic).
template <typename OutT>
__global__ void __launch_bounds__(256)
splitk_reduce_kernel(const float *__restrict__ ws, int splits, int64_t batch, int64_t M,
                     int64_t N, const OutT *__restrict__ c0, int64_t sc0, int64_t sc1,
                     int64_t sc2, OutT *__restrict__ out, int64_t so0, int64_t so1, int64_t so2) {
  const int64_t total = batch * M * N, slice = total;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t n = i % N, m = (i / N) % M, b = i / (M * N);
    float v = 0.f;
    for (int sp = 0; sp < splits; ++sp) v = __fadd_rn(v, ws[sp * slice + i]);
    if (c0) v = __fadd_rn(v, Conv<OutT>::to_f(c0[b * sc0 + m * sc1 + n * sc2]));
    out[b * so0 + m * so1 + n * so2] = Conv<OutT>::from_f(v);
  }
}
}  // namespace

int contract_tc(const bgx_contract_desc &d, cudaStream_t s) { return contract_tc_impl(d, 1, s); }

// Split-K plan: only when the (batch x M x N) tiles leave most SMs idle and K
// is long enough to give every slice >= 8 k-blocks.
void tc_splitk_plan(const bgx_contract_desc &d, int *splits, int64_t *ws_bytes) {
  *splits = 1;
  *ws_bytes = 0;
  if (!tc_legal(d, nullptr)) return;
  int cg = 0, bn = 0;
  tc_tile_choice(d, &cg, &bn);
  const int64_t tiles = ((d.M + 128 * cg - 1) / (128 * cg)) * ((d.N + bn - 1) / bn) * d.batch;
  const int64_t slots = sm_count_current() / cg;
  const int BKe = d.in_dtype == BGX_F32 ? Elem<4>::BK : Elem<2>::BK;
  const int64_t k_blocks = (d.K + BKe - 1) / BKe;
  const int64_t sp = uniform_splits(tiles, slots, k_blocks);
  if (sp == 1) {
    // tail split: when the last wave is at most half full, split only its
    // tiles in two K halves (reported as a negative split count); the second
    // half finishes the tile inside the kernel.  Measured on B200
    // (profiles/r01_tail_split.txt): +2-18 % for K >= 8192, break-even at
    // 4096^3 (the partial exchange costs about the half wave it saves),
    // slower for K = 2048; 3- and 4-way splits never beat 2.
    const int64_t tail = tiles % slots;
    if (tiles < slots || tail == 0 || tail * 2 > slots || k_blocks < 128) return;
    const int64_t ts = 2;
    *splits = -(int)ts;
    *ws_bytes = (slots - 1) * ts * (int64_t)(128 * cg) * bn * 4 + 256 + slots * cg * 4;
    return;
  }
  *splits = (int)sp;
  *ws_bytes = sp * d.batch * d.M * d.N * 4;
}

int contract_tc_splitk(const bgx_contract_desc &d, int splits, void *ws, int64_t ws_bytes,
                       cudaStream_t s) {
  if (splits < -1) {  // tail split of the last partial wave
    BGX_CHECK_ARG(ws != nullptr && ((uintptr_t)ws % 16) == 0, "tail split: workspace must be 16B aligned");
    return contract_tc_impl(d, 1, s, -splits, ws, ws_bytes);
  }
  if (splits <= 1) return contract_tc(d, s);
  BGX_CHECK_ARG(ws != nullptr && ((uintptr_t)ws % 16) == 0, "split-K: workspace must be 16B aligned");
  BGX_CHECK_ARG(ws_bytes >= (int64_t)splits * d.batch * d.M * d.N * 4,
                "split-K: workspace too small (%lld bytes for %d splits)", (long long)ws_bytes, splits);
  bgx_contract_desc dp = d;
  dp.out = ws;
  dp.out_dtype = BGX_F32;
  dp.c0 = nullptr;
  dp.o_stride[0] = d.M * d.N;
  dp.o_stride[1] = d.N;
  dp.o_stride[2] = 1;
  const int BKe = d.in_dtype == BGX_F32 ? Elem<4>::BK : Elem<2>::BK;
  const int64_t k_blocks = (d.K + BKe - 1) / BKe;
  const int64_t per = (k_blocks + splits - 1) / splits;
  splits = (int)((k_blocks + per - 1) / per);   // the kernel normalises the same way
  int rc = contract_tc_impl(dp, splits, s);
  if (rc) return rc;
  const int64_t total = d.batch * d.M * d.N;
  int64_t blocks = (total + 255) / 256;
  const int64_t cap = (int64_t)sm_count_current() * 16;
  if (blocks > cap) blocks = cap;
  switch (d.out_dtype) {
    case BGX_F32:
      splitk_reduce_kernel<float><<<(unsigned)blocks, 256, 0, s>>>(
          (const float *)ws, splits, d.batch, d.M, d.N, (const float *)d.c0, d.c_stride[0],
          d.c_stride[1], d.c_stride[2], (float *)d.out, d.o_stride[0], d.o_stride[1], d.o_stride[2]);
      break;
    case BGX_BF16:
      splitk_reduce_kernel<__nv_bfloat16><<<(unsigned)blocks, 256, 0, s>>>(
          (const float *)ws, splits, d.batch, d.M, d.N, (const __nv_bfloat16 *)d.c0,
          d.c_stride[0], d.c_stride[1], d.c_stride[2], (__nv_bfloat16 *)d.out, d.o_stride[0],
          d.o_stride[1], d.o_stride[2]);
      break;
    default:
      splitk_reduce_kernel<__half><<<(unsigned)blocks, 256, 0, s>>>(
          (const float *)ws, splits, d.batch, d.M, d.N, (const __half *)d.c0, d.c_stride[0],
          d.c_stride[1], d.c_stride[2], (__half *)d.out, d.o_stride[0], d.o_stride[1],
          d.o_stride[2]);
  }
  return check_launch("splitk_reduce_kernel");
}

// ---- fused K-split reduce-scatter (bgx_contract_rs_plan / _reduce_scatter) ----

int tc_rs_plan(const bgx_contract_desc &d, int world, bgx_rs_plan *pl) {
  const char *why = nullptr;
  BGX_CHECK_ARG(world >= 1 && world <= BGX_MAX_RANKS, "reduce-scatter: world %d", world);
  BGX_CHECK_ARG(d.batch == 1, "reduce-scatter: batch must be 1 (got %lld)", (long long)d.batch);
  BGX_CHECK_ARG(d.in_dtype == BGX_BF16 || d.in_dtype == BGX_F16,
                "reduce-scatter: inputs must be bf16/f16");
  BGX_CHECK_ARG(d.out_dtype == d.in_dtype || d.out_dtype == BGX_F32, "reduce-scatter: out dtype");
  if (!tc_legal(d, &why)) {
    set_error("tensor-core path not legal: %s", why);
    return BGX_ERR_UNSUPPORTED;
  }
  memset(pl, 0, sizeof(*pl));
  pl->world = world;
  const int64_t rows = (d.M + world - 1) / world;
  // CTA pairs (256-row tiles); ownership is per CTA (128 rows), so each
  // owner's slab only has to be a multiple of 128 rows
  // instantiated fused variants: (1, 128), (1, 256), (2, 256)
  const int bn = d.N > 128 ? 256 : 128;
  const int cg = (d.M > 128 && bn == 256) ? 2 : 1;
  const int64_t tile_m = 128 * cg;
  pl->cta_group = cg;
  pl->tile_n = bn;
  pl->rows_per_owner = (rows + BM - 1) / BM * BM;
  const int64_t tiles = ((d.M + tile_m - 1) / tile_m) * ((d.N + bn - 1) / bn);
  const int64_t slots = sm_count_current() / cg;
  const int64_t k_blocks = (d.K + Elem<2>::BK - 1) / Elem<2>::BK;
  int64_t sp = slots / (tiles > 0 ? tiles : 1);
  if (sp > k_blocks / 8) sp = k_blocks / 8;
  if (sp > 32) sp = 32;
  if (sp < 1) sp = 1;
  pl->local_splits = (int32_t)sp;
  pl->out_dtype = d.out_dtype;
  pl->mode = BGX_RS_DEFERRED;
  pl->slot_bytes = (int64_t)world * sp * pl->rows_per_owner * d.N * 4;
  pl->counter_bytes = (tiles * cg * 4 + 15) / 16 * 16;
  pl->ws_bytes = 0;
  return BGX_OK;
}

// ---- deferred reduce-scatter: the owner's all-SM reduction ------------------
// out[r][j] = cast( (((sum_s slot[0][s]) + sum_s slot[1][s]) + ...) + c0 ),
// every inner sum slice-ordered from slice 0 — the order of the in-kernel mode.
template <typename OutT>
__global__ void rs_reduce_kernel(const float *__restrict__ slots, const OutT *__restrict__ c0,
                                 OutT *__restrict__ out, int64_t rows, int64_t N, int64_t rpo,
                                 int world, int S, int64_t so, int64_t sc) {
  const int64_t total = rows * N;
  const int64_t plane = rpo * N;           // one (rank, slice) partial
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / N, j = i - r * N;
    const float *src = slots + r * N + j;
    float acc = 0.f;
    for (int rk = 0; rk < world; ++rk) {
      float part = __ldg(src + (int64_t)rk * S * plane);
      for (int sl = 1; sl < S; ++sl) part = __fadd_rn(part, __ldg(src + ((int64_t)rk * S + sl) * plane));
      acc = rk == 0 ? part : __fadd_rn(acc, part);
    }
    if (c0) acc = __fadd_rn(acc, Conv<OutT>::to_f(c0[r * sc + j]));
    out[r * so + j] = Conv<OutT>::from_f(acc);
  }
}

// Vector form (N % 4 == 0, 16-byte aligned slots): thread (x, y) sums rank y's
// S slices of 4 columns (loads batched four slices at a time, so every
// thread keeps 64 bytes in flight), the ranks' partials meet in shared memory
// and lane y = 0 adds them in rank order, adds c0, casts and stores.
constexpr int RSR_X = 64;
__device__ __forceinline__ float4 f4_add(float4 a, float4 b) {
  return make_float4(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y), __fadd_rn(a.z, b.z),
                     __fadd_rn(a.w, b.w));
}
template <typename OutT>
__global__ void __launch_bounds__(RSR_X * BGX_MAX_RANKS)
rs_reduce_vec_kernel(const float *__restrict__ slots, const OutT *__restrict__ c0,
                     OutT *__restrict__ out, int64_t rows, int64_t N, int64_t rpo, int S,
                     int64_t so, int64_t sc) {
  __shared__ float4 part[BGX_MAX_RANKS][RSR_X];
  const int64_t nq = N / 4;
  const int64_t q = blockIdx.x * (int64_t)RSR_X + threadIdx.x;
  const int rk = threadIdx.y, world = blockDim.y;
  const int64_t r = q / nq, j = (q - r * nq) * 4;
  const bool ok = r < rows;
  if (ok) {
    const int64_t plane = rpo * N;
    const float4 *src = reinterpret_cast<const float4 *>(slots + ((int64_t)rk * S * rpo + r) * N + j);
    const int64_t pstep = plane / 4;   // float4s per slice plane
    float4 p = make_float4(0.f, 0.f, 0.f, 0.f);
    int sl = 0;
    for (; sl + 4 <= S; sl += 4) {            // four slices' loads in flight
      const float4 x0 = __ldg(src + sl * pstep), x1 = __ldg(src + (sl + 1) * pstep);
      const float4 x2 = __ldg(src + (sl + 2) * pstep), x3 = __ldg(src + (sl + 3) * pstep);
      p = f4_add(f4_add(f4_add(sl == 0 ? x0 : f4_add(p, x0), x1), x2), x3);
    }
    for (; sl < S; ++sl) {
      const float4 x = __ldg(src + sl * pstep);
      p = sl == 0 ? x : f4_add(p, x);
    }
    part[rk][threadIdx.x] = p;
  }
  __syncthreads();
  if (!ok || rk != 0) return;
  float4 acc = part[0][threadIdx.x];
  for (int k = 1; k < world; ++k) acc = f4_add(acc, part[k][threadIdx.x]);
  float v[4] = {acc.x, acc.y, acc.z, acc.w};
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    if (c0) v[e] = __fadd_rn(v[e], Conv<OutT>::to_f(c0[r * sc + j + e]));
    out[r * so + j + e] = Conv<OutT>::from_f(v[e]);
  }
}

int rs_reduce(const bgx_contract_desc &d, const bgx_reduce_scatter &rs, cudaStream_t s) {
  const bgx_rs_plan &pl = rs.plan;
  BGX_CHECK_ARG(pl.mode == BGX_RS_DEFERRED, "bgx_rs_reduce: plan mode %d is not deferred", pl.mode);
  BGX_CHECK_ARG(pl.world >= 1 && pl.world <= BGX_MAX_RANKS && pl.rank >= 0 && pl.rank < pl.world,
                "bgx_rs_reduce: rank %d of %d", pl.rank, pl.world);
  BGX_CHECK_ARG(pl.local_splits >= 1 && pl.rows_per_owner > 0, "bgx_rs_reduce: bad plan");
  const int S = pl.local_splits;        // every rank delivered exactly S slices
  const int r = pl.rank;
  BGX_CHECK_ARG(rs.slots[r] && rs.out[r], "bgx_rs_reduce: null slot/out for owner %d", r);
  int64_t rows = d.M - (int64_t)r * pl.rows_per_owner;
  if (rows > pl.rows_per_owner) rows = pl.rows_per_owner;
  if (rows <= 0) return BGX_OK;          // an owner past the last row has nothing
  const int64_t total = rows * d.N;
  int64_t blocks = (total + 255) / 256;
  const int64_t cap = (int64_t)sm_count_current() * 8;
  if (blocks > cap) blocks = cap;
  const int64_t so = d.o_stride[1], sc = d.c_stride[1];
  if (d.N % 4 == 0 && ((uintptr_t)rs.slots[r] & 15) == 0) {
    const dim3 blk(RSR_X, pl.world);
    const unsigned grid = (unsigned)((total / 4 + RSR_X - 1) / RSR_X);
    const int64_t rpo = pl.rows_per_owner;
    switch (pl.out_dtype) {
      case BGX_F32:
        rs_reduce_vec_kernel<float><<<grid, blk, 0, s>>>(rs.slots[r], (const float *)rs.c0[r],
                                                         (float *)rs.out[r], rows, d.N, rpo, S, so, sc);
        return check_launch("rs_reduce_vec_kernel");
      case BGX_BF16:
        rs_reduce_vec_kernel<__nv_bfloat16><<<grid, blk, 0, s>>>(
            rs.slots[r], (const __nv_bfloat16 *)rs.c0[r], (__nv_bfloat16 *)rs.out[r], rows, d.N,
            rpo, S, so, sc);
        return check_launch("rs_reduce_vec_kernel");
      case BGX_F16:
        rs_reduce_vec_kernel<__half><<<grid, blk, 0, s>>>(rs.slots[r], (const __half *)rs.c0[r],
                                                          (__half *)rs.out[r], rows, d.N, rpo, S,
                                                          so, sc);
        return check_launch("rs_reduce_vec_kernel");
      default:
        break;
    }
  }
  switch (pl.out_dtype) {
    case BGX_F32:
      rs_reduce_kernel<float><<<(unsigned)blocks, 256, 0, s>>>(
          rs.slots[r], (const float *)rs.c0[r], (float *)rs.out[r], rows, d.N, pl.rows_per_owner,
          pl.world, S, so, sc);
      break;
    case BGX_BF16:
      rs_reduce_kernel<__nv_bfloat16><<<(unsigned)blocks, 256, 0, s>>>(
          rs.slots[r], (const __nv_bfloat16 *)rs.c0[r], (__nv_bfloat16 *)rs.out[r], rows, d.N,
          pl.rows_per_owner, pl.world, S, so, sc);
      break;
    case BGX_F16:
      rs_reduce_kernel<__half><<<(unsigned)blocks, 256, 0, s>>>(
          rs.slots[r], (const __half *)rs.c0[r], (__half *)rs.out[r], rows, d.N, pl.rows_per_owner,
          pl.world, S, so, sc);
      break;
    default:
      set_error("bgx_rs_reduce: out dtype %d", pl.out_dtype);
      return BGX_ERR_INVALID;
  }
  return check_launch("rs_reduce_kernel");
}

int contract_tc_rs(const bgx_contract_desc &d, const bgx_reduce_scatter &rs, cudaStream_t s) {
  const bgx_rs_plan &pl = rs.plan;
  const char *why = nullptr;
  BGX_CHECK_ARG(pl.world >= 1 && pl.world <= BGX_MAX_RANKS && pl.rank >= 0 && pl.rank < pl.world,
                "reduce-scatter: rank %d of %d", pl.rank, pl.world);
  BGX_CHECK_ARG(d.batch == 1, "reduce-scatter: batch must be 1");
  BGX_CHECK_ARG(d.in_dtype == BGX_BF16 || d.in_dtype == BGX_F16,
                "reduce-scatter: inputs must be bf16/f16");
  BGX_CHECK_ARG(pl.out_dtype == BGX_F32 || pl.out_dtype == d.in_dtype, "reduce-scatter: out dtype");
  BGX_CHECK_ARG((pl.cta_group == 1 && (pl.tile_n == 128 || pl.tile_n == 256)) ||
                    (pl.cta_group == 2 && pl.tile_n == 256),
                "reduce-scatter: tile %d x %d", 128 * pl.cta_group, pl.tile_n);
  BGX_CHECK_ARG(pl.rows_per_owner > 0 && pl.rows_per_owner % BM == 0 &&
                    pl.rows_per_owner * pl.world >= d.M,
                "reduce-scatter: rows_per_owner %lld", (long long)pl.rows_per_owner);
  BGX_CHECK_ARG(pl.mode == BGX_RS_IN_KERNEL || pl.mode == BGX_RS_DEFERRED,
                "reduce-scatter: mode %d", pl.mode);
  BGX_CHECK_ARG(pl.local_splits >= 1 && (pl.local_splits == 1 || pl.mode == BGX_RS_DEFERRED ||
                                         (rs.ws && rs.ws_counters)),
                "reduce-scatter: local split workspace missing");
  for (int r = 0; r < pl.world; ++r)
    BGX_CHECK_ARG(rs.slots[r] && rs.counters[r] && rs.out[r],
                  "reduce-scatter: null slot/counter/out pointer for owner %d", r);
  bgx_contract_desc dd = d;
  dd.out = nullptr;
  dd.c0 = nullptr;
  dd.sched.cta_group = pl.cta_group;
  dd.sched.tile_n = pl.tile_n;
  if (!tc_legal(dd, &why)) {
    set_error("tensor-core path not legal: %s", why);
    return BGX_ERR_UNSUPPORTED;
  }
  TcParams p{};
  p.batch = 1; p.M = d.M; p.N = d.N; p.K = d.K;
  p.a_mn = d.a_stride[2] != 1 ? 1 : 0;
  p.b_mn = d.b_stride[2] == 1 ? 1 : 0;
  p.k_blocks = (int32_t)((d.K + Elem<2>::BK - 1) / Elem<2>::BK);
  // deferred mode: the owners' reduction reads exactly local_splits slices
  // from every rank, so every rank must be able to fill them
  BGX_CHECK_ARG(pl.mode != BGX_RS_DEFERRED || pl.local_splits <= p.k_blocks,
                "reduce-scatter: local_splits %d > %d k-blocks of this rank's slab (deferred "
                "mode needs local_splits <= every rank's k-blocks)", pl.local_splits, p.k_blocks);
  p.k_splits = pl.local_splits > p.k_blocks ? p.k_blocks : pl.local_splits;
  p.tail_splits = 1;
  p.ws = rs.ws;
  for (int i = 0; i < 3; ++i) { p.sc[i] = d.c_stride[i]; p.so[i] = d.o_stride[i]; }
  p.raster = d.sched.raster != 0 ? d.sched.raster : (pl.cta_group == 2 ? 8 : 16);
  p.debug = d.sched.reserved[0];
  p.rs_world = pl.world;
  p.rs_rank = pl.rank;
  p.rs_defer = pl.mode == BGX_RS_DEFERRED ? 1 : 0;
  p.rs_out_dtype = pl.out_dtype;
  p.rs_rpo = pl.rows_per_owner;
  for (int r = 0; r < BGX_MAX_RANKS; ++r) {
    p.rs_slots[r] = r < pl.world ? rs.slots[r] : nullptr;
    p.rs_counters[r] = r < pl.world ? rs.counters[r] : nullptr;
    p.rs_out[r] = r < pl.world ? rs.out[r] : nullptr;
    p.rs_c0[r] = r < pl.world ? rs.c0[r] : nullptr;
  }
  p.rs_ws_counters = rs.ws_counters;
  if (pl.cta_group == 2) return launch_tc<256, 2, float, 2, true>(dd, p, s);
  if (pl.tile_n == 128) return launch_tc<128, 1, float, 2, true>(dd, p, s);
  return launch_tc<256, 1, float, 2, true>(dd, p, s);
}

// Tile shape the TC path would use (bgx_contract_tile).
void tc_tile_choice(const bgx_contract_desc &d, int *cg_out, int *bn_out) {
  int cg = 0, bn = 0;
  choose_tile(d, sm_count_current(), cg, bn);
  if (d.sched.cta_group == 1 || d.sched.cta_group == 2) cg = d.sched.cta_group;
  if (d.sched.tile_n == 64 || d.sched.tile_n == 128 || d.sched.tile_n == 256 ||
      d.sched.tile_n == 512)
    bn = d.sched.tile_n;
  if (cg == 2 && bn == 64) bn = 128;
  if (cg == 1 && bn == 512) bn = 256;
  *cg_out = cg;
  *bn_out = bn;
}

}  // namespace bgx

extern "C" __attribute__((visibility("default"))) int bgxdbg_trace_read(void *host, int64_t bytes) {
  const int64_t n = (int64_t)sizeof(bgx::g_trace) < bytes ? (int64_t)sizeof(bgx::g_trace) : bytes;
  return cudaMemcpyFromSymbol(host, bgx::g_trace, (size_t)n) == cudaSuccess ? 0 : -3;
}
