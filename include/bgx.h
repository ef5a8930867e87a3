/*
 * bgx.h — C ABI of libbgx.so, the B200 (sm_100a) execution backend for the
 * einsum / linalg.generic hot path of arXiv 2503.04771 (reference package
 * `bridgegen`, pure Python).
 *
 * The reference has no native boundary: its only compute engine is
 * `interp._Machine._generic` (/root/reference/pkg/src/bridgegen/interp.py:372-424),
 * dispatched from `_Machine.execute` (interp.py:351-352).  Every entry point
 * below replaces one piece of that loop nest; the Python mirror of the
 * reference API (paper_2503_04771_b200/interp.py, .../compat.py) classifies a
 * generic op and calls exactly one of them.  INTEGRATION.md shows the ctypes
 * binding a bridgegen maintainer would add at interp.py:351.
 *
 * Conventions
 *   - Plain C types only; no torch/CUDA types in signatures.  `stream` is a
 *     cudaStream_t passed as void* (NULL = legacy default stream).
 *   - All pointers are DEVICE pointers on the current CUDA device, except the
 *     descriptor structs themselves (host memory, read during the call only).
 *   - Strides are in ELEMENTS, may be any non-negative value (views allowed).
 *   - Return 0 (BGX_OK) or a negative bgx_status; bgx_last_error() returns a
 *     thread-local message for the last failure on the calling thread.
 *   - The library never allocates user-visible memory and never frees caller
 *     memory.  Calls are stream-ordered and asynchronous; thread-safe across
 *     threads/devices/streams.
 *   - There is no CPU fallback: an unsupported case returns
 *     BGX_ERR_UNSUPPORTED and the caller must pick another entry point.
 */
#ifndef BGX_H_
#define BGX_H_

#include <stdint.h>

#if defined(__GNUC__)
#define BGX_API __attribute__((visibility("default")))
#else
#define BGX_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define BGX_VERSION 1
#define BGX_MAX_RANK 8        /* permute operand rank */
#define BGX_MAX_AXES 12       /* generic iteration axes */
#define BGX_MAX_OPERANDS 6    /* generic inputs */

typedef enum {
  BGX_OK = 0,
  BGX_ERR_INVALID = -1,      /* bad arguments (shapes, strides, dtypes)       */
  BGX_ERR_UNSUPPORTED = -2,  /* valid but not handled by this entry point     */
  BGX_ERR_CUDA = -3,         /* CUDA runtime / driver failure                 */
  BGX_ERR_NO_DEVICE = -4     /* no sm_100 device visible                      */
} bgx_status;

/* Element types.  The reference knows only f32/f64 (bridgegen ir.py:71-78);
 * bf16/f16 are the tensor-core input types of the B200 path. */
typedef enum { BGX_F32 = 0, BGX_F64 = 1, BGX_BF16 = 2, BGX_F16 = 3 } bgx_dtype;

typedef struct {
  void *data;                    /* device pointer                              */
  int32_t dtype;                 /* bgx_dtype                                   */
  int32_t rank;                  /* 0..BGX_MAX_RANK                             */
  int64_t shape[BGX_MAX_RANK];
  int64_t stride[BGX_MAX_RANK];  /* elements                                    */
} bgx_tensor;

/* ---- library ------------------------------------------------------------ */
BGX_API int bgx_version(void);
BGX_API const char *bgx_last_error(void);
/* Number of SMs of the current device (148 on B200), or a negative status. */
BGX_API int bgx_sm_count(void);

/* ---- permutation ---------------------------------------------------------
 * Replaces _generic for a passthrough body (einsum.py:105-108 `return x1`):
 *   out[i_0..i_{r-1}] = in[j] with j[perm[d]] = i_d, i.e. output dim d reads
 *   input dim perm[d].  Bit-exact (bytes are moved, never converted).
 * in/out: same dtype, same rank r, out->shape[d] == in->shape[perm[d]].     */
BGX_API int bgx_permute(const bgx_tensor *in, const bgx_tensor *out,
                const int32_t *perm, void *stream);

/* ---- generic loop nest ---------------------------------------------------
 * Replaces _generic for ANY einsum body (interp.py:372-424 + einsum.py:100-118)
 * with the reference's exact rounding: one device thread per output element
 * walks that element's reduction sub-space in the reference's lexicographic
 * order, p = x1; p = p*xk (k = 2..n); acc = p + acc, each op separately
 * rounded (no FMA).  Bit-identical to the reference for f32 and f64.
 * bf16/f16 (DSL extension): operands widened to f32, the same loop in f32,
 * one final round-to-nearest-even to the storage type.
 * Axes: [0, n_par) are the output (parallel) axes in output order, then the
 * reduction axes (einsum.py:81).  c0 and out are dense row-major over the
 * parallel axes; c0 may equal out or be NULL (zero initial output, i.e. +0.0 —
 * what the reference computes from a zeros array).  passthrough = (n_in == 1
 * && no reduction). */
typedef struct {
  int32_t n_in;
  int32_t n_axes;
  int32_t n_par;
  int32_t dtype;                       /* BGX_F32, BGX_F64, BGX_BF16, BGX_F16 */
  int64_t extents[BGX_MAX_AXES];
  const void *ins[BGX_MAX_OPERANDS];
  int64_t strides[BGX_MAX_OPERANDS][BGX_MAX_AXES]; /* 0 = axis not indexed */
  const void *c0;
  void *out;
} bgx_generic_desc;
BGX_API int bgx_generic(const bgx_generic_desc *d, void *stream);

/* Tolerance mode for bodies WITH a reduction (BGX_MODE_FFMA callers): each
 * output element's reduction sub-space is cut into chunks summed by
 * 256-thread blocks (strided partial sums + shuffle tree), then the chunk
 * sums are added in chunk order with c0.  Deterministic; f32 accumulation
 * (f64 for f64), one final rounding; NOT the reference's summation order
 * (relative error ~1e-7 f32).  bgx_generic_tree_plan gives the workspace the
 * call needs (0 when one chunk per output suffices).                       */
BGX_API int bgx_generic_tree_plan(const bgx_generic_desc *d, int64_t *workspace_bytes);
BGX_API int bgx_generic_tree(const bgx_generic_desc *d, void *workspace, int64_t workspace_bytes,
                             void *stream);

/* ---- batched strided contraction (GEMM) ----------------------------------
 * Replaces _generic for a two-input multiply-accumulate body whose axes
 * group into batch / M / N / K (each group flattened to one extent by the
 * caller):
 *   out[b,m,n] = (c0 ? c0[b,m,n] : 0) + sum_k a[b,m,k] * b[b,k,n]
 * Kernel selection (bgx_contract_desc.mode):
 *   BGX_MODE_AUTO    bf16/f16 -> tensor cores (tcgen05) when TMA-legal, else
 *                    SIMT; f32/f64 -> BGX_MODE_EXACT.
 *   BGX_MODE_EXACT   f32/f64 CUDA-core tiles, products and sums separately
 *                    rounded in increasing k: bit-identical to the reference.
 *   BGX_MODE_FFMA    f32/f64 CUDA-core tiles with fused multiply-add (rel.
 *                    err <= 1e-5 vs the reference, faster); 16-bit inputs as
 *                    BGX_MODE_AUTO.
 *   BGX_MODE_TC      tcgen05/TMEM/TMA tensor-core path (bf16/f16 inputs, f32
 *                    accumulate); BGX_ERR_UNSUPPORTED if not TMA-legal.
 *   BGX_MODE_SIMT    CUDA-core path for any dtype (f32 accumulate for 16-bit).
 *   BGX_MODE_TF32    f32 inputs on the tensor cores (tcgen05 kind::tf32, f32
 *                    accumulate; 10-bit mantissa products, rel. err ~1e-3);
 *                    any operand majorness (MN-major via SWIZZLE_128B_BASE32B).
 * Output dtype may be the input dtype or f32 (out_dtype).  The TC path needs
 * one unit stride in each of a (k or m) and b (k or n), 16-byte aligned base
 * pointers and 16-byte multiple non-unit strides, and out/c0 n-stride 1.    */
typedef enum {
  BGX_MODE_AUTO = 0, BGX_MODE_EXACT = 1, BGX_MODE_FFMA = 2, BGX_MODE_TC = 3,
  BGX_MODE_SIMT = 4, BGX_MODE_TF32 = 5
} bgx_mode;

typedef struct {
  int32_t tile_n;     /* 0 = auto; TC: 64/128/256, 512 (CTA pair only: two
                         N=256 MMAs per K-step, single TMEM accumulator)      */
  int32_t stages;     /* 0 = auto; TC smem pipeline depth                   */
  int32_t cta_group;  /* 0 = auto; TC: 1 or 2 (CTA pair, M = 256)           */
  int32_t max_ctas;   /* 0 = auto (persistent: one CTA per SM)              */
  int32_t raster;     /* 0 = auto; >0: groups of this many M-tiles (A slab
                         L2-resident), <0: groups of |raster| N-tiles         */
  int32_t reserved[3]; /* reserved[0]: timing-probe bits (1 skip epilogue
                          stores — the output is NOT written; 2 direct stores;
                          4 skip the epilogue; 8 no start stagger).
                          reserved[1] = cluster_n: 0 automatic, 1 one
                          CTA pair per cluster, 2 two pairs sharing A by TMA
                          multicast (4-CTA clusters).                         */
} bgx_schedule;

typedef struct {
  int64_t batch, M, N, K;
  const void *a; int64_t a_stride[3];   /* (batch, m, k) */
  const void *b; int64_t b_stride[3];   /* (batch, k, n) */
  const void *c0; int64_t c_stride[3];  /* (batch, m, n); NULL => zero init */
  void *out; int64_t o_stride[3];       /* (batch, m, n) */
  int32_t in_dtype;                     /* bgx_dtype of a and b             */
  int32_t out_dtype;                    /* bgx_dtype of out and c0          */
  int32_t mode;                         /* bgx_mode                         */
  int32_t flags;                        /* reserved, 0                      */
  bgx_schedule sched;
} bgx_contract_desc;
BGX_API int bgx_contract(const bgx_contract_desc *d, void *stream);
/* Which kernel bgx_contract would launch: 1 = tcgen05, 2 = SIMT exact,
 * 3 = SIMT ffma, 4 = SIMT 16-bit, negative = error. */
BGX_API int bgx_contract_kernel(const bgx_contract_desc *d);
/* Tile shape of the tcgen05 path for this descriptor: cta_group (1 = one CTA,
 * 128-row tiles; 2 = CTA pair, 256-row tiles) and tile_n; both 0 when the
 * descriptor would not run on tensor cores. */
BGX_API int bgx_contract_tile(const bgx_contract_desc *d, int32_t *cta_group, int32_t *tile_n);

/* ---- split-K on one GPU --------------------------------------------------
 * For contractions whose batch x M x N tiles leave most SMs idle (small
 * output, long K): `splits` persistent units per tile each contract a K slice
 * on the tensor cores into f32 partials in `workspace` (splits x batch x M x N
 * floats), then one reduction kernel sums the slices in order, adds c0 and
 * casts.  splits < -1 selects the TAIL split instead (stream-K style): full
 * waves of tiles run unsplit and only the tiles of the last, partial wave are
 * split into -splits K slices (f32 partials in `workspace`; the last slice of
 * each tile to finish sums the slices in slice order inside the same kernel —
 * deterministic — and writes the output).  bgx_contract_splitk_plan returns the split count the library
 * would use (1 = neither is worth it) and the workspace size in bytes.     */
BGX_API int bgx_contract_splitk_plan(const bgx_contract_desc *d, int32_t *splits,
                                     int64_t *workspace_bytes);
BGX_API int bgx_contract_splitk(const bgx_contract_desc *d, int32_t splits, void *workspace,
                                int64_t workspace_bytes, void *stream);

/* ---- multi-GPU K-split: GEMM fused with the reduce-scatter ----------------
 * Replaces the K-split exchange (per-rank K slab -> f32 partials
 * -> ncclReduceScatter -> cast) by ONE tcgen05 kernel per rank whose
 * epilogue moves the partial tiles over NVLink as they finish:
 *   level 1 (only when local_splits > 1): the rank's K slab is split again
 *     over its SMs; each unit stores its f32 tile to the local `ws`
 *     (local_splits x M x N) and bumps ws_counters[tile]; the last local
 *     unit sums the slices in slice order and carries on with level 2;
 *   level 2: the rank's f32 partial tile is stored straight into the owner's
 *     slot  slots[owner] + (rank * rows_per_owner + local_row) * N  (peer
 *     memory: plain st.global over NVLink) and, after a system-scope fence,
 *     counters[owner][tile] is bumped with a system-scope atomic; the unit
 *     that brings it to `world` sums the world slots IN RANK ORDER (bitwise
 *     deterministic, independent of arrival order), adds c0[owner], casts to
 *     out_dtype and stores the owner's output rows.
 * Output row r belongs to owner r / rows_per_owner (a multiple of 128: a
 * CTA pair's two 128-row halves may go to different owners); out[owner]/c0[owner] point at that owner's rows_per_owner x N
 * slab (row strides desc.o_stride[1] / desc.c_stride[1]).  No rank ever waits
 * for another inside the kernel (the last arriver does the work), so the
 * kernel cannot deadlock; the caller orders consecutive calls with a barrier
 * (slots are reused).  Counters must be zero before the first call; each call
 * leaves them zero.  desc.a/b are the rank's K slab (M x K_r, K_r x N);
 * desc.out/c0 are ignored; batch must be 1.  On one GPU, `world` launches
 * with local buffers (rank 0..world-1 in stream order) compute exactly what
 * `world` GPUs would.  bgx_contract_rs_plan fills tile shape, rows_per_owner,
 * local_splits and the buffer sizes for a (M, N, K_r, world) problem; every
 * rank must use the same plan.
 *
 * plan.mode selects where the sums happen:
 *   BGX_RS_IN_KERNEL (0): as above — the last arriver reduces inside the
 *     kernel (levels 1 and 2);
 *   BGX_RS_DEFERRED (1, the planner's choice): the kernel only delivers —
 *     every (rank, local slice) unit stores its f32 partial tile straight
 *     into  slots[owner] + ((rank * local_splits + slice) * rows_per_owner
 *     + local_row) * N  (no counters, no ws); after the caller's barrier
 *     each owner runs bgx_rs_reduce, one all-SM kernel that sums its slots
 *     slice-major inside each rank, ranks in rank order (the same order as
 *     mode 0, so both modes are bit-identical), adds c0, casts and stores
 *     its out rows.  The serial tail of the last arrivers (latency-bound
 *     remote reads by a few CTAs) becomes one bandwidth-bound local pass.
 *     slot_bytes = world * local_splits * rows_per_owner * N * 4, ws_bytes 0.
 * bgx_rs_reduce(d, rs, stream) reduces owner rs->plan.rank (mode 1 only).  */
#define BGX_RS_IN_KERNEL 0
#define BGX_RS_DEFERRED 1
#define BGX_MAX_RANKS 8
typedef struct {
  int32_t world, rank;
  int32_t cta_group, tile_n;     /* tile shape (from the plan)               */
  int32_t local_splits;          /* >= 1                                     */
  int32_t out_dtype;             /* bgx_dtype of out / c0                    */
  int32_t mode;                  /* BGX_RS_IN_KERNEL / BGX_RS_DEFERRED       */
  int32_t reserved0;
  int64_t rows_per_owner;
  int64_t slot_bytes;            /* per owner: world * rows_per_owner * N * 4
                                    (mode 1: x local_splits)                 */
  int64_t counter_bytes;         /* per owner and for ws_counters            */
  int64_t ws_bytes;              /* local: local_splits * M * N * 4 (or 0)   */
} bgx_rs_plan;
typedef struct {
  bgx_rs_plan plan;
  float *slots[BGX_MAX_RANKS];            /* per owner, peer-mapped         */
  uint32_t *counters[BGX_MAX_RANKS];      /* per owner, peer-mapped         */
  void *out[BGX_MAX_RANKS];               /* per owner, peer-mapped         */
  const void *c0[BGX_MAX_RANKS];          /* per owner or NULL              */
  float *ws;                              /* local (local_splits > 1)       */
  uint32_t *ws_counters;                  /* local                          */
} bgx_reduce_scatter;
BGX_API int bgx_contract_rs_plan(const bgx_contract_desc *d, int32_t world, bgx_rs_plan *plan);
BGX_API int bgx_contract_reduce_scatter(const bgx_contract_desc *d, const bgx_reduce_scatter *rs,
                                        void *stream);
BGX_API int bgx_rs_reduce(const bgx_contract_desc *d, const bgx_reduce_scatter *rs, void *stream);

/* ---- one process, several devices: the M-shard -------------
 * The contraction's output rows (or batches) are split into n independent
 * slabs; descs[i] describes slab i with pointers on device devices[i] (A's
 * rows / batches of that slab, B whole, that slab of c0 and out) and
 * streams[i] is a stream on that device (NULL: its legacy default stream;
 * `streams` itself may be NULL).  Each slab is launched with bgx_contract on
 * its own device — launches are asynchronous, so the devices run
 * concurrently — and the caller's current device is restored.  No data moves
 * between devices (there is no exchange in the M-shard); slabs are computed
 * exactly as one device would compute those rows.  Stops at the first
 * failing slab (bgx_last_error names it). */
BGX_API int bgx_contract_sharded(const bgx_contract_desc *descs, const int32_t *devices,
                                 void *const *streams, int32_t n);

/* ---- the K-split exchange over NCCL ------------------------
 * NCCL is loaded at run time (the copy already in the process, else
 * libnccl.so.2); BGX_ERR_UNSUPPORTED without it.  One communicator per rank
 * (one process per GPU, or one thread per GPU), created collectively:
 *   rank 0: bgx_nccl_unique_id(id) -> share the 128 bytes with every rank ->
 *   every rank on its device: bgx_nccl_comm_init(&comm, world, rank, id).
 * bgx_ksplit_reduce(partial, out, c0, out_dtype, rows, cols, scatter, ws,
 * comm, stream): `partial` is this rank's rows x cols f32 partial sum (its K
 * slab's contribution, e.g. from bgx_contract with out_dtype f32); the
 * partials are summed over the ranks with ncclReduceScatter (scatter != 0:
 * rows % world == 0, this rank receives rows [rank*rows/world, ...) into
 * `out`) or ncclAllReduce (every rank receives all rows), in f32, then c0
 * (same rows, out_dtype) is added and the result cast to out_dtype
 * (bgx_cast_f32).  `ws` is an f32 workspace of the received size, needed
 * unless out_dtype is f32 and c0 is NULL (then NCCL writes `out` directly).
 * Stream-ordered; the summation order across ranks is NCCL's. */
BGX_API int bgx_nccl_unique_id(void *id_out /* 128 bytes */);
BGX_API int bgx_nccl_comm_init(void **comm, int32_t world, int32_t rank, const void *id);
BGX_API int bgx_nccl_comm_destroy(void *comm);
BGX_API int bgx_ksplit_reduce(const float *partial, void *out, const void *c0, int32_t out_dtype,
                              int64_t rows, int64_t cols, int32_t scatter, float *ws, void *comm,
                              void *stream);
/* Releases the library's per-process state (unloads NCCL once every
 * communicator is destroyed).  The library holds no device memory of its
 * own: workspaces are always the caller's. */
BGX_API int bgx_shutdown(void);

/* ---- elementwise helpers for multi-GPU K-split -------------------------
 * out[i] = (dtype_out) src[i] for n elements, src f32 (the reduced partials),
 * out f32/bf16/f16; with c0 != NULL adds c0[i] first (in f32).           */
BGX_API int bgx_cast_f32(const float *src, const void *c0, void *out, int32_t out_dtype,
                 int64_t n, void *stream);

/* ---- measurement -----------------------------------------------------------
 * One CTA per SM writes (smid, %clock64, %globaltimer) to out[3 * sm_count]
 * (device memory).  Two samples around a timed region give every SM's
 * average clock over it (bench.py's in-band clocks figure).                */
BGX_API int bgx_clock_sample(uint64_t *out, void *stream);

/* ---- runtime-compiled kernels (GPU case study) ---------
 * Replaces the simulated sequential thread grid of bridgegen run_kernel
 * (interp.py:434-461): CUDA C generated from an IR kernel is compiled with
 * NVRTC for sm_100a (no FMA contraction, no FTZ) and launched as a 1-D grid of
 * `grid` blocks x `block` threads; `args` is the cudaLaunchKernel argument
 * array.  `log` (optional) receives the compiler log.                      */
BGX_API int bgx_rtc_compile(const char *src, const char *name, void **handle, char *log,
                            int64_t log_len);
BGX_API int bgx_rtc_launch(void *handle, uint64_t grid, uint32_t block, void **args,
                           void *stream);
BGX_API int bgx_rtc_free(void *handle);

#ifdef __cplusplus
}
#endif
#endif /* BGX_H_ */
