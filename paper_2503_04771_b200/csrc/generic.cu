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

#include <stdlib.h>
#include <type_traits>

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

// Thread -> output mapping when the parallel axes are walked in another
// order than the output's (launch_generic: the innermost walked axis is the
// one the streamed operands are contiguous along, so warp loads coalesce;
// the output, written once, takes the strided side): row-major strides of
// the output for each walked axis.
struct OutMap {
  int64_t stride[BGX_MAX_AXES];
};

// DENSE: every input is laid out exactly like the (row-major) output over the
// parallel axes and there is no reduction — the offsets are the output index.
// PERM: the parallel axes of `d` are in walk order; om maps them to the output.
template <typename S, typename T, int NIN, bool DENSE, bool PERM = false>
__global__ void __launch_bounds__(128)
generic_kernel(const bgx_generic_desc d, int64_t n_out, int64_t red_points, const OutMap om) {
  const int n_in = NIN > 0 ? NIN : d.n_in;
  const int n_par = d.n_par, n_axes = d.n_axes, n_red = n_axes - n_par;
  const bool passthrough = (n_in == 1 && n_red == 0);
  const bool idx32 = n_out <= 0x7fffffffLL;
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < n_out;
       o += (int64_t)gridDim.x * blockDim.x) {
    int64_t off[BGX_MAX_OPERANDS];
#pragma unroll
    for (int k = 0; k < BGX_MAX_OPERANDS; ++k) off[k] = DENSE ? o : 0;
    int64_t oo = PERM ? 0 : o;   // this output's element offset
    if (!DENSE) {
      if (idx32) {   // 32-bit index arithmetic: the divisions dominate elementwise bodies
        uint32_t rem = (uint32_t)o;
        for (int a = n_par - 1; a >= 0; --a) {
          const uint32_t e = (uint32_t)d.extents[a];
          const uint32_t q = rem / e, i = rem - q * e;
          rem = q;
          for (int k = 0; k < n_in; ++k) off[k] += (int64_t)i * d.strides[k][a];
          if (PERM) oo += (int64_t)i * om.stride[a];
        }
      } else {
        int64_t rem = o;
        for (int a = n_par - 1; a >= 0; --a) {
          const int64_t e = d.extents[a];
          const int64_t i = rem % e;
          rem /= e;
          for (int k = 0; k < n_in; ++k) off[k] += i * d.strides[k][a];
          if (PERM) oo += i * om.stride[a];
        }
      }
    }
    const S *const *ins = reinterpret_cast<const S *const *>(d.ins);
    S *out = static_cast<S *>(d.out);
    if (passthrough) {
      out[oo] = ins[0][off[0]];
      continue;
    }
    // c0 == NULL: zero initial output (+0.0, as the reference's zeros array)
    T acc = d.c0 ? ld_as<S, T>(static_cast<const S *>(d.c0) + oo) : T(0);
    if (red_points == 0) {
      out[oo] = st_as<S, T>(acc);
      continue;
    }
    if (n_red == 0) {  // elementwise body (Hadamard / outer product): one point
      T p = ld_as<S, T>(ins[0] + off[0]);
      for (int k = 1; k < n_in; ++k) p = mul_rn<T>(p, ld_as<S, T>(ins[k] + off[k]));
      out[oo] = st_as<S, T>(add_rn<T>(p, acc));
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
    // operands that do not move along any reduction axis: one load per
    // output, kept in a register (a warp-divergent re-load per point was the
    // whole cost of bodies like (d,a,c),(c,d,b)->(b,c,d))
    uint32_t inv = 0;
    T fixedv[NIN > 0 ? NIN : BGX_MAX_OPERANDS];
#pragma unroll
    for (int k = 0; k < (NIN > 0 ? NIN : BGX_MAX_OPERANDS); ++k) {
      if (k >= n_in) break;
      bool moves = false;
      for (int a = n_par; a < n_axes; ++a) moves = moves || (d.strides[k][a] != 0 && d.extents[a] > 1);
      if (!moves) {
        inv |= 1u << k;
        fixedv[k] = ld_as<S, T>(ins[k] + off[k]);
      }
    }
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
          if (inv >> k & 1) {
#pragma unroll
            for (int u = 0; u < U; ++u) v[k][u] = fixedv[k];
            continue;
          }
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
    out[oo] = st_as<S, T>(acc);
  }
}

// Dense elementwise bodies (Hadamard products: every input strided like the
// row-major output, no reduction): 16-byte vectors of every operand per
// thread, the same per-element arithmetic as generic_kernel (left-fold
// product, + c0 or +0.0, separately rounded) — bit-identical, HBM-bound.
template <typename S, typename T, int NIN>
__global__ void __launch_bounds__(256)
dense_ew_kernel(const bgx_generic_desc d, int64_t n_out) {
  constexpr int V = 16 / (int)sizeof(S);
  const S *const *ins = reinterpret_cast<const S *const *>(d.ins);
  const S *c0 = static_cast<const S *>(d.c0);
  S *out = static_cast<S *>(d.out);
  const int64_t nv = n_out / V;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv; i += stride) {
    uint4 q[NIN + 1];
#pragma unroll
    for (int k = 0; k < NIN; ++k) q[k] = __ldcs(reinterpret_cast<const uint4 *>(ins[k]) + i);
    q[NIN] = c0 ? __ldcs(reinterpret_cast<const uint4 *>(c0) + i) : make_uint4(0, 0, 0, 0);
    uint4 r;
    S *re = reinterpret_cast<S *>(&r);
#pragma unroll
    for (int e = 0; e < V; ++e) {
      T p = ld_as<S, T>(reinterpret_cast<const S *>(&q[0]) + e);
#pragma unroll
      for (int k = 1; k < NIN; ++k) p = mul_rn<T>(p, ld_as<S, T>(reinterpret_cast<const S *>(&q[k]) + e));
      const T acc = c0 ? ld_as<S, T>(reinterpret_cast<const S *>(&q[NIN]) + e) : T(0);
      re[e] = st_as<S, T>(add_rn<T>(p, acc));
    }
    __stcs(reinterpret_cast<uint4 *>(out) + i, r);
  }
  for (int64_t o = nv * V + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < n_out; o += stride) {
    T p = ld_as<S, T>(ins[0] + o);
#pragma unroll
    for (int k = 1; k < NIN; ++k) p = mul_rn<T>(p, ld_as<S, T>(ins[k] + o));
    out[o] = st_as<S, T>(add_rn<T>(p, c0 ? ld_as<S, T>(c0 + o) : T(0)));
  }
}

// Elementwise bodies with broadcast or strided operands (outer products,
// scalings, (c),(a,c),(b)->(c,a,b)): the output is dense, so a thread takes V
// consecutive outputs along the innermost output axis (one 16-byte store),
// decodes their row once, and loads each operand as one 16-byte vector (unit
// stride, aligned), one broadcast scalar (stride 0) or V strided scalars.
// The per-output index decode of generic_kernel (a division per axis per
// output) was the cost: 33.5M-output outer product 229 us ~ 0.6 TB/s.
// Same per-element arithmetic as generic_kernel: p = left fold of products,
// out = p + c0 (or + 0).
// one 16-byte vector of outputs: operand loads (bcast_ew_load) kept apart
// from the product / c0 / store (bcast_ew_store) so several vectors' loads
// can be in flight before the first store (stores may alias the inputs as
// far as the compiler knows)
template <typename S, typename T, int NIN>
__device__ __forceinline__ void bcast_ew_load(const bgx_generic_desc &d, const int64_t (&off)[NIN],
                                              const int64_t (&sin)[NIN], T (&v)[NIN][16 / sizeof(S)]) {
  constexpr int V = 16 / (int)sizeof(S);
  const S *const *ins = reinterpret_cast<const S *const *>(d.ins);
#pragma unroll
  for (int k = 0; k < NIN; ++k) {
    const S *src = ins[k] + off[k];
    if (sin[k] == 0) {
      const T x = ld_as<S, T>(src);
#pragma unroll
      for (int e = 0; e < V; ++e) v[k][e] = x;
    } else if (sin[k] == 1 && ((uintptr_t)src & 15) == 0) {
      const uint4 q = *reinterpret_cast<const uint4 *>(src);   // may be reused across rows
#pragma unroll
      for (int e = 0; e < V; ++e) v[k][e] = ld_as<S, T>(reinterpret_cast<const S *>(&q) + e);
    } else {
#pragma unroll
      for (int e = 0; e < V; ++e) v[k][e] = ld_as<S, T>(src + e * sin[k]);
    }
  }
}

template <typename S, typename T, int NIN>
__device__ __forceinline__ void bcast_ew_store(const bgx_generic_desc &d, const T (&v)[NIN][16 / sizeof(S)],
                                               int64_t o) {
  constexpr int V = 16 / (int)sizeof(S);
  const S *c0 = static_cast<const S *>(d.c0);
  const uint4 cq = c0 ? __ldcs(reinterpret_cast<const uint4 *>(c0 + o)) : make_uint4(0, 0, 0, 0);
  uint4 r;
  S *re = reinterpret_cast<S *>(&r);
#pragma unroll
  for (int e = 0; e < V; ++e) {
    T p = v[0][e];
#pragma unroll
    for (int k = 1; k < NIN; ++k) p = mul_rn<T>(p, v[k][e]);
    const T acc = c0 ? ld_as<S, T>(reinterpret_cast<const S *>(&cq) + e) : T(0);
    re[e] = st_as<S, T>(add_rn<T>(p, acc));
  }
  __stcs(reinterpret_cast<uint4 *>(static_cast<S *>(d.out) + o), r);
}

// Elementwise bodies with broadcast or strided operands (outer products,
// scalings, (c),(a,c),(b)->(c,a,b)): the output is dense, so work goes by
// 16-byte vectors of consecutive outputs along the innermost output axis.
// ROWS (rows of >= 32 vectors): a warp walks whole rows, decoding each row
// once; otherwise a thread decodes every vector.  Operands load as one 16-byte vector (unit stride, aligned), one
// broadcast scalar (stride 0) or V strided scalars.  The per-output decode
// of generic_kernel (a division per axis per output) was the cost:
// 33.5M-output outer product 229 us ~ 0.6 TB/s.  Same per-element
// arithmetic as generic_kernel: p = left fold of products, out = p + c0 (or + 0).
template <typename S, typename T, int NIN, bool ROWS>
__global__ void __launch_bounds__(256) bcast_ew_kernel(const bgx_generic_desc d, int64_t n_out) {
  constexpr int V = 16 / (int)sizeof(S);
  const int np = d.n_par;
  const int64_t E = d.extents[np - 1];
  int64_t sin[NIN];
#pragma unroll
  for (int k = 0; k < NIN; ++k) sin[k] = d.strides[k][np - 1];
  const bool idx32 = n_out <= 0x7fffffffLL;
  auto decode_row = [&](int64_t row, int64_t (&off)[NIN]) {
#pragma unroll
    for (int k = 0; k < NIN; ++k) off[k] = 0;
    if (idx32) {
      uint32_t rem = (uint32_t)row;
      for (int a = np - 2; a >= 0; --a) {
        const uint32_t e = (uint32_t)d.extents[a], q = rem / e, x = rem - q * e;
        rem = q;
#pragma unroll
        for (int k = 0; k < NIN; ++k) off[k] += (int64_t)x * d.strides[k][a];
      }
    } else {
      int64_t rem = row;
      for (int a = np - 2; a >= 0; --a) {
        const int64_t e = d.extents[a], x = rem % e;
        rem /= e;
#pragma unroll
        for (int k = 0; k < NIN; ++k) off[k] += x * d.strides[k][a];
      }
    }
  };
  if constexpr (ROWS) {
    // a warp walks whole rows (one decode per row); each lane issues the
    // operand loads of U vectors before their stores
    constexpr int U = sizeof(S) == 2 ? 2 : 4;
    const int lane = threadIdx.x % 32;
    const int64_t nrows = n_out / E, vpr = E / V;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x / 32);
    for (int64_t row = blockIdx.x * (int64_t)(blockDim.x / 32) + threadIdx.x / 32; row < nrows;
         row += warps) {
      int64_t base[NIN];
      decode_row(row, base);
      for (int64_t j0 = lane; j0 < vpr; j0 += 32 * U) {
        T v[U][NIN][V];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t jv = j0 + 32 * u;
          if (jv < vpr) {
            int64_t off[NIN];
#pragma unroll
            for (int k = 0; k < NIN; ++k) off[k] = base[k] + jv * V * sin[k];
            bcast_ew_load<S, T, NIN>(d, off, sin, v[u]);
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t jv = j0 + 32 * u;
          if (jv < vpr) bcast_ew_store<S, T, NIN>(d, v[u], row * E + jv * V);
        }
      }
    }
  } else {
    const int64_t nv = n_out / V;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv;
         i += (int64_t)gridDim.x * blockDim.x) {
      const int64_t o = i * V;
      int64_t row, j;
      if (idx32) { row = (uint32_t)o / (uint32_t)E; j = (uint32_t)o - (uint32_t)row * (uint32_t)E; }
      else { row = o / E; j = o - row * E; }
      int64_t off[NIN];
      decode_row(row, off);
#pragma unroll
      for (int k = 0; k < NIN; ++k) off[k] += j * sin[k];
      T v[NIN][V];
      bcast_ew_load<S, T, NIN>(d, off, sin, v);
      bcast_ew_store<S, T, NIN>(d, v, o);
    }
  }
}

template <typename S, typename T, bool DENSE>
void launch_generic_n(const bgx_generic_desc &d, int64_t n_out, int64_t red, unsigned blocks,
                      cudaStream_t s, const OutMap *om = nullptr) {
  OutMap m{};
  if (om) m = *om;
  if (!DENSE && om) {
    switch (d.n_in) {
      case 1: generic_kernel<S, T, 1, false, true><<<blocks, 128, 0, s>>>(d, n_out, red, m); break;
      case 2: generic_kernel<S, T, 2, false, true><<<blocks, 128, 0, s>>>(d, n_out, red, m); break;
      case 3: generic_kernel<S, T, 3, false, true><<<blocks, 128, 0, s>>>(d, n_out, red, m); break;
      default: generic_kernel<S, T, 0, false, true><<<blocks, 128, 0, s>>>(d, n_out, red, m); break;
    }
    return;
  }
  switch (d.n_in) {
    case 1: generic_kernel<S, T, 1, DENSE><<<blocks, 128, 0, s>>>(d, n_out, red, m); break;
    case 2: generic_kernel<S, T, 2, DENSE><<<blocks, 128, 0, s>>>(d, n_out, red, m); break;
    case 3: generic_kernel<S, T, 3, DENSE><<<blocks, 128, 0, s>>>(d, n_out, red, m); break;
    default: generic_kernel<S, T, 0, DENSE><<<blocks, 128, 0, s>>>(d, n_out, red, m); break;
  }
}

// Walk order of the parallel axes for the per-thread loop nest: the axis
// along which the most streamed operands (those that move along the
// reduction, read red_points times per output) are contiguous goes
// innermost, so a warp's loads coalesce; operands fixed along the reduction
// and the output (written once) count less.  Returns true and fills `w` / `om`
// when the order differs from the output's.
bool walk_order(const bgx_generic_desc &d, bgx_generic_desc &w, OutMap &om) {
  const int n_par = d.n_par;
  if (n_par < 2 || d.n_axes == n_par) return false;
  auto score = [&](int a) {
    if (d.extents[a] == 1) return -1.0;
    double sc = a == n_par - 1 ? 0.25 : 0.0;       // the output's contiguous axis
    for (int k = 0; k < d.n_in; ++k) {
      if (d.strides[k][a] != 1) continue;
      bool streamed = false;
      for (int r = n_par; r < d.n_axes; ++r) streamed = streamed || (d.strides[k][r] != 0 && d.extents[r] > 1);
      sc += streamed ? 1.0 : 0.1;
    }
    return sc;
  };
  int best = n_par - 1;
  double bs = score(best);
  for (int a = 0; a < n_par - 1; ++a)
    if (score(a) > bs + 0.5) { bs = score(a); best = a; }
  // then, just outside it, the axes the streamed operands do not move along
  // (consecutive warps re-read the same operand lines from cache)
  auto reuse = [&](int a) {
    int r = 0;
    for (int k = 0; k < d.n_in; ++k) {
      bool streamed = false;
      for (int x = n_par; x < d.n_axes; ++x) streamed = streamed || (d.strides[k][x] != 0 && d.extents[x] > 1);
      if (streamed && d.strides[k][a] == 0 && d.extents[a] > 1) ++r;
    }
    return r;
  };
  int order[BGX_MAX_AXES], n = 0;
  for (int pass = 0; pass < 2; ++pass)        // outer: moved-along axes, inner: reused ones
    for (int a = 0; a < n_par; ++a)
      if (a != best && (reuse(a) > 0) == (pass == 1)) order[n++] = a;
  order[n++] = best;
  bool same = true;
  for (int a = 0; a < n_par; ++a) same = same && order[a] == a;
  if (same) return false;
  int64_t ost[BGX_MAX_AXES];
  int64_t st = 1;
  for (int a = n_par - 1; a >= 0; --a) { ost[a] = st; st *= d.extents[a]; }
  w = d;
  for (int pos = 0; pos < n_par; ++pos) {
    const int a = order[pos];
    w.extents[pos] = d.extents[a];
    for (int k = 0; k < d.n_in; ++k) w.strides[k][pos] = d.strides[k][a];
    om.stride[pos] = ost[a];
  }
  return true;
}

// ---- row reductions: one reduction axis, contiguous in every input ---------
// (i,j)->(i), (i,j),(i,j)->(i), (i,j),(j)->(i) (GEMV), ...: each output is a
// sequential chain over j (the reference order), so only the outputs give
// parallelism.  The per-thread row walk of generic_kernel makes every warp
// load touch 32 different rows; here a warp owns 32 consecutive outputs and
// stages 32 x RT tiles of its 32 rows through shared memory with 4-byte
// cp.async (each row segment is one coalesced 128-byte line), STAGES tiles in
// flight; every lane then folds its own row from shared memory in order —
// the same arithmetic sequence, bit-identical to the reference.
constexpr int RR_TJ = 32;      // columns per tile
constexpr int RR_STAGES = 4;   // tiles in flight per warp
constexpr int RR_WARPS = 4;    // warps per block

__device__ __forceinline__ void cp_async4(void *smem, const void *gmem, bool pred) {
  const int sz = pred ? 4 : 0;   // src-size 0: zero fill, no global access
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(smem_u32(smem)),
               "l"(gmem), "r"(sz) : "memory");
}
__device__ __forceinline__ void cp_async8(void *smem, const void *gmem, bool pred) {
  const int sz = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_u32(smem)),
               "l"(gmem), "r"(sz) : "memory");
}
// 16-byte copy of the first `bytes` (0..16) bytes, the rest zero-filled.
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem, int bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(smem)),
               "l"(gmem), "r"(bytes) : "memory");
}
// full 16-byte copy (no zero-fill operand)
__device__ __forceinline__ void cp_async16_full(void *smem, const void *gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem)), "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N> __device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// COLS: the reduction axis is NOT contiguous but consecutive outputs are
// (column sums, vector-matrix products): tile[step][lane] is then loaded
// straight along the outputs — one coalesced line per reduction step.
// VEC (row layout, 16-byte aligned rows): tiles are staged with 16-byte
// cp.async — 32 / (row bytes / 16) rows per instruction instead of one — into
// rows padded to a 16-byte multiple, and each lane folds its row from
// 16-byte shared loads (conflict-free: 8 lanes per phase hit 8 distinct
// 4-bank groups).  Same element order, same arithmetic.
template <typename T> constexpr int rr_stride(bool vec, int tj = RR_TJ) {
  return vec ? tj + 16 / (int)sizeof(T) : tj + 1;
}

// NW warps per block, ST tiles in flight per warp, TJ columns per tile.
template <typename T, int NIN, bool COLS, bool VEC = false, int NW = RR_WARPS, int ST = RR_STAGES,
          int TJ = RR_TJ, typename S = T>
__global__ void __launch_bounds__(32 * NW)
rowreduce_kernel(const bgx_generic_desc d, int64_t n_out, uint32_t shared_mask) {
  // shared_mask bit k: input k does not depend on the output index (e.g. the
  // vector of a GEMV): its tile row is loaded once and read by every lane
  // tile[stage][input][row][col], +1 column of padding against bank conflicts
  extern __shared__ __align__(16) uint8_t rr_smem_raw[];
  S *tiles = reinterpret_cast<S *>(rr_smem_raw);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  constexpr int RS = rr_stride<S>(VEC, TJ);          // tile row stride (elements)
  constexpr int TSZ = 32 * RS;                    // one tile
  S *wtiles = tiles + (size_t)warp * ST * NIN * TSZ;
  const int n_par = d.n_par;
  const int64_t E = d.extents[d.n_axes - 1];
  const int64_t o0 = ((int64_t)blockIdx.x * NW + warp) * 32;
  if (o0 >= n_out) return;
  const int64_t o = o0 + lane;
  const bool row_ok = o < n_out;
  const bool all_rows = o0 + 32 <= n_out;
  // this lane's row bases
  int64_t off[NIN];
#pragma unroll
  for (int k = 0; k < NIN; ++k) off[k] = 0;
  if (row_ok) {
    int64_t rem = o;
    for (int a = n_par - 1; a >= 0; --a) {
      const int64_t e = d.extents[a];
      const int64_t i = rem % e;
      rem /= e;
#pragma unroll
      for (int k = 0; k < NIN; ++k) off[k] += i * d.strides[k][a];
    }
  }
  const S *const *ins = reinterpret_cast<const S *const *>(d.ins);
  const int64_t ntiles = (E + TJ - 1) / TJ;
  // VEC staging: the source of each (row group i, vector) this lane copies
  constexpr int VE16 = 16 / (int)sizeof(S);
  constexpr int VRPI = VEC ? 32 / (TJ / VE16) : 1;
  constexpr int VG = VEC ? 32 / VRPI : 1;            // row groups per tile
  const S *vsrc[NIN][VG];
  bool vrow_ok[VG];
  if constexpr (VEC) {
    const int v = lane % (TJ / VE16);
#pragma unroll
    for (int i = 0; i < VG; ++i) {
      const int rr = i * VRPI + lane / (TJ / VE16);
      vrow_ok[i] = o0 + rr < n_out;
#pragma unroll
      for (int k = 0; k < NIN; ++k) {
        const int64_t base = __shfl_sync(0xffffffffu, off[k], rr);
        vsrc[k][i] = ins[k] + base + v * VE16;
      }
    }
  }
  auto issue = [&](int64_t t) {
    const int stage = (int)(t % ST);
    const int64_t j = t * TJ + lane;          // this lane's column of the tile
#pragma unroll
    for (int k = 0; k < NIN; ++k) {
      S *tile = wtiles + (stage * NIN + k) * TSZ;
      if ((shared_mask >> (8 + k)) & 1) {
        // constant along the reduction (a per-output factor): never staged
      } else if (COLS && ((shared_mask >> k) & 1)) {
        // shared operand (e.g. the vector of a vector-matrix product): one
        // element per reduction step, lane l loads step l of the tile
        const int64_t sk = d.strides[k][d.n_axes - 1];
        const int64_t jj = t * TJ + lane;
        const bool ok = jj < E;
        const S *src = ins[k] + (ok ? off[k] + jj * sk : 0);
        if constexpr (sizeof(S) == 4) cp_async4(tile + lane, src, ok);
        else cp_async8(tile + lane, src, ok);
      } else if constexpr (VEC) {
        // rows of the tile as 16-byte vectors: lane -> (row, vector) pairs
        constexpr int E16 = 16 / (int)sizeof(S);
        constexpr int VPR = TJ / E16;           // vectors per tile row
        static_assert(VPR <= 32 && 32 % VPR == 0, "a tile row must fit one warp instruction");
        constexpr int RPI = 32 / VPR;              // rows per instruction
        const int v = lane % VPR;
        if ((shared_mask >> k) & 1) {
          // shared operand: one row, VPR lanes
          const int64_t jj = t * TJ + v * E16;
          const int64_t left = E - jj;
          const int bytes = left >= E16 ? 16 : (left > 0 ? (int)left * (int)sizeof(S) : 0);
          if (lane < VPR) cp_async16(tile + v * E16, ins[k] + (bytes ? off[k] + jj : 0), bytes);
        } else {
          // per-lane source pointers precomputed once (vsrc); a full tile of
          // 32 live rows is one pointer add + one cp.async per row group
          const bool full = (t + 1) * TJ <= E;
          if (full && all_rows) {
            S *dst0 = tile + (lane / VPR) * RS + v * E16;
#pragma unroll
            for (int i = 0; i < 32 / RPI; ++i)
              cp_async16_full(dst0 + i * RPI * RS, vsrc[k][i] + t * TJ);
          } else {
            const int64_t jj = t * TJ + v * E16;
            const int64_t left = E - jj;
            const int tail = left >= E16 ? 16 : (left > 0 ? (int)left * (int)sizeof(S) : 0);
#pragma unroll
            for (int i = 0; i < 32 / RPI; ++i) {
              const int rr = i * RPI + lane / VPR;
              const int bytes = !vrow_ok[i] ? 0 : (full ? 16 : tail);
              cp_async16(tile + rr * RS + v * E16, bytes ? vsrc[k][i] + t * TJ : ins[k], bytes);
            }
          }
        }
      } else if constexpr (COLS) {
        const int64_t sk = d.strides[k][d.n_axes - 1];
        for (int rr = 0; rr < 32; ++rr) {
          const int64_t jj = t * TJ + rr;       // reduction step of this tile row
          const bool ok = row_ok && jj < E;
          const S *src = ins[k] + (ok ? off[k] + jj * sk : 0);
          if constexpr (sizeof(S) == 4) cp_async4(tile + rr * RS + lane, src, ok);
          else cp_async8(tile + rr * RS + lane, src, ok);
        }
      } else {
        auto copy_row = [&](int rr) {
          const int64_t base = __shfl_sync(0xffffffffu, off[k], rr);
          const bool ok = (o0 + rr < n_out) && j < E;
          const S *src = ins[k] + (ok ? base + j : 0);
          if constexpr (sizeof(S) == 4) cp_async4(tile + rr * RS + lane, src, ok);
          else cp_async8(tile + rr * RS + lane, src, ok);
        };
        if ((shared_mask >> k) & 1) {
          copy_row(0);
        } else {
          for (int rr = 0; rr < 32; ++rr) copy_row(rr);
        }
      }
    }
    cp_async_commit();
  };
  T acc = (row_ok && d.c0) ? ld_as<S, T>(static_cast<const S *>(d.c0) + o) : T(0);
  // operands constant along the reduction (shared_mask bits 8..15): one
  // value per lane, multiplied in at their place in the left fold
  T invv[NIN];
#pragma unroll
  for (int k = 0; k < NIN; ++k)
    invv[k] = (((shared_mask >> (8 + k)) & 1) && row_ok) ? ld_as<S, T>(ins[k] + off[k]) : T(0);
  for (int64_t t = 0; t < ST - 1; ++t) {
    if (t < ntiles) issue(t); else cp_async_commit();
  }
  for (int64_t t = 0; t < ntiles; ++t) {
    if (t + ST - 1 < ntiles) issue(t + ST - 1); else cp_async_commit();
    cp_async_wait<ST - 1>();              // tile t has landed (this lane's copies)
    __syncwarp();                                // ... and every lane's
    const int stage = (int)(t % ST);
    const int jmax = (E - t * TJ) < TJ ? (int)(E - t * TJ) : TJ;
    // element c of this lane's chain: row layout tile[lane][c], column layout tile[c][lane]
    const S *row[NIN];
    int cstep[NIN];
#pragma unroll
    for (int k = 0; k < NIN; ++k) {
      const bool sh = (shared_mask >> k) & 1;
      row[k] = wtiles + (stage * NIN + k) * TSZ + (sh ? 0 : (COLS ? lane : lane * RS));
      cstep[k] = (COLS && !sh) ? RS : 1;
    }
    if (VEC && jmax == TJ) {
      constexpr int E16 = 16 / (int)sizeof(S);
#pragma unroll 2
      for (int c4 = 0; c4 < TJ; c4 += E16) {
        T v[NIN][E16];
#pragma unroll
        for (int k = 0; k < NIN; ++k) {
          if ((shared_mask >> (8 + k)) & 1) {
#pragma unroll
            for (int i = 0; i < E16; ++i) v[k][i] = invv[k];
            continue;
          }
          const uint4 q = *reinterpret_cast<const uint4 *>(row[k] + c4);
          const S *e = reinterpret_cast<const S *>(&q);
#pragma unroll
          for (int i = 0; i < E16; ++i) v[k][i] = ld_as<S, T>(e + i);
        }
#pragma unroll
        for (int i = 0; i < E16; ++i) {
          T p = v[0][i];
#pragma unroll
          for (int k = 1; k < NIN; ++k) p = mul_rn<T>(p, v[k][i]);
          acc = add_rn<T>(p, acc);
        }
      }
    } else if (jmax == TJ) {
#pragma unroll 8
      for (int c = 0; c < TJ; ++c) {
        T p = ((shared_mask >> 8) & 1) ? invv[0] : ld_as<S, T>(row[0] + c * cstep[0]);
#pragma unroll
        for (int k = 1; k < NIN; ++k)
          p = mul_rn<T>(p, ((shared_mask >> (8 + k)) & 1) ? invv[k] : ld_as<S, T>(row[k] + c * cstep[k]));
        acc = add_rn<T>(p, acc);
      }
    } else {
      for (int c = 0; c < jmax; ++c) {
        T p = ((shared_mask >> 8) & 1) ? invv[0] : ld_as<S, T>(row[0] + c * cstep[0]);
#pragma unroll
        for (int k = 1; k < NIN; ++k)
          p = mul_rn<T>(p, ((shared_mask >> (8 + k)) & 1) ? invv[k] : ld_as<S, T>(row[k] + c * cstep[k]));
        acc = add_rn<T>(p, acc);
      }
    }
    __syncwarp();                                // stage free before it is refilled
  }
  cp_async_wait<0>();
  if (row_ok) static_cast<S *>(d.out)[o] = st_as<S, T>(acc);
}

// ---- exact column chains, 16-byte staged ----------------------------------
// Column sums and vector-matrix products in the reference order: output
// column i is the sequential chain over the reduction rows.  One warp owns 32
// adjacent columns (lane = column); each 32-row x 32-column tile of every
// per-column operand is staged with 16-byte cp.async (8 rows per instruction
// for f32) from source pointers computed once, and the fold is fully unrolled
// with compile-time shared-memory offsets — the general rowreduce column mode
// spends ~4x more instructions per element on runtime addressing (ncu: 2.5
// cycles per issued instruction, 17 % issue-busy, 1.5 TB/s).  SHM bit k:
// operand k is shared by the 32 columns (the vector of a GEMV): one element
// per lane per tile, read back as a broadcast.

template <typename T, int NIN, int SHM, int ST, int CPW, typename S = T>
__global__ void __launch_bounds__(32)
colchain_kernel(const bgx_generic_desc d, int64_t n_out) {
  constexpr int E16 = 16 / (int)sizeof(S);
  constexpr int GPR = CPW / E16;             // 16-byte groups per tile row
  static_assert(GPR >= 1 && 32 % GPR == 0, "a tile row is whole 16-byte groups");
  constexpr int RPI = 32 / GPR;              // tile rows per copy instruction
  constexpr int RS = CPW + E16;              // tile row stride (elements)
  constexpr int TSZ = 32 * RS;
  constexpr int NPC = NIN - __builtin_popcount(SHM);   // per-column operands
  constexpr int SSZ = NPC * TSZ + (NIN - NPC) * 32;    // one stage
  extern __shared__ __align__(16) uint8_t cc_smem_raw[];
  const int lane = threadIdx.x;
  S *wst = reinterpret_cast<S *>(cc_smem_raw);
  const int64_t o0 = (int64_t)blockIdx.x * CPW;
  if (o0 >= n_out) return;
  const int64_t o = o0 + lane % CPW;   // lanes >= CPW fold a duplicate chain, never stored
  const int ax = d.n_axes - 1;
  const int64_t E = d.extents[ax];
  // the column group's bases (its CPW outputs are adjacent columns)
  int64_t base[NIN];
#pragma unroll
  for (int k = 0; k < NIN; ++k) base[k] = 0;
  {
    int64_t rem = o0;
    for (int a = d.n_par - 1; a >= 0; --a) {
      const int64_t e = d.extents[a], i = rem % e;
      rem /= e;
#pragma unroll
      for (int k = 0; k < NIN; ++k) base[k] += i * d.strides[k][a];
    }
  }
  const S *const *ins = reinterpret_cast<const S *const *>(d.ins);
  const S *src[NIN];
  int64_t step[NIN];   // source advance per tile
  const int q = lane % GPR, r0 = lane / GPR;
#pragma unroll
  for (int k = 0; k < NIN; ++k) {
    const int64_t sk = d.strides[k][ax];
    if ((SHM >> k) & 1) src[k] = ins[k] + base[k] + lane * sk;
    else src[k] = ins[k] + base[k] + r0 * sk + q * E16;
    step[k] = 32 * sk;
  }
  const int64_t ntiles = (E + 31) / 32;
  auto issue = [&](int64_t t) {
    S *stg = wst + (int)(t % ST) * SSZ;
    const bool full = (t + 1) * 32 <= E;
    int pc = 0, sc = 0;
#pragma unroll
    for (int k = 0; k < NIN; ++k) {
      const S *g = src[k] + t * step[k];
      if ((SHM >> k) & 1) {
        if constexpr (sizeof(S) == 2) {
          // 16-bit shared operand (unit stride, 16-byte aligned: host-checked):
          // lanes 0-3 copy the tile's 32 values as 4 x 16 bytes
          S *dst = stg + NPC * TSZ + sc * 32 + lane * 8;
          const int64_t left = E - t * 32 - lane * 8;
          const int bytes = left >= 8 ? 16 : (left > 0 ? (int)left * 2 : 0);
          if (lane < 4) cp_async16(dst, bytes ? g + 7 * lane : ins[k], bytes);
        } else {
          S *dst = stg + NPC * TSZ + sc * 32 + lane;
          const bool ok = full || t * 32 + lane < E;
          if constexpr (sizeof(S) == 4) cp_async4(dst, ok ? g : ins[k], ok);
          else cp_async8(dst, ok ? g : ins[k], ok);
        }
        ++sc;
      } else {
        S *dst = stg + pc * TSZ + r0 * RS + q * E16;
        const int64_t rstep = RPI * d.strides[k][ax];
        if (full) {
#pragma unroll
          for (int i = 0; i < 32 / RPI; ++i) cp_async16_full(dst + i * RPI * RS, g + i * rstep);
        } else {
#pragma unroll
          for (int i = 0; i < 32 / RPI; ++i) {
            const bool ok = t * 32 + i * RPI + r0 < E;
            cp_async16(dst + i * RPI * RS, ok ? g + i * rstep : ins[k], ok ? 16 : 0);
          }
        }
        ++pc;
      }
    }
    cp_async_commit();
  };
  T acc = d.c0 ? ld_as<S, T>(static_cast<const S *>(d.c0) + o) : T(0);
  // (reading a full tile into registers and refilling its stage before the
  // add chain, to issue in the chain's shadow, was 10-15 % slower)
  for (int64_t t = 0; t < ST - 1; ++t) {
    if (t < ntiles) issue(t); else cp_async_commit();
  }
  for (int64_t t = 0; t < ntiles; ++t) {
    if (t + ST - 1 < ntiles) issue(t + ST - 1); else cp_async_commit();
    cp_async_wait<ST - 1>();
    __syncwarp();
    const S *stg = wst + (int)(t % ST) * SSZ;
    const S *col[NIN];
    {
      int pc = 0, sc = 0;
#pragma unroll
      for (int k = 0; k < NIN; ++k) {
        if ((SHM >> k) & 1) col[k] = stg + NPC * TSZ + 32 * sc++;
        else col[k] = stg + (pc++) * TSZ + lane % CPW;
      }
    }
    auto elem = [&](int k, int c) {
      return ld_as<S, T>(((SHM >> k) & 1) ? col[k] + c : col[k] + c * RS);
    };
    if ((t + 1) * 32 <= E) {
#pragma unroll
      for (int c = 0; c < 32; ++c) {
        T p = elem(0, c);
#pragma unroll
        for (int k = 1; k < NIN; ++k) p = mul_rn<T>(p, elem(k, c));
        acc = add_rn<T>(p, acc);
      }
    } else {
      const int jmax = (int)(E - t * 32);
      for (int c = 0; c < jmax; ++c) {
        T p = elem(0, c);
#pragma unroll
        for (int k = 1; k < NIN; ++k) p = mul_rn<T>(p, elem(k, c));
        acc = add_rn<T>(p, acc);
      }
    }
    __syncwarp();
  }
  cp_async_wait<0>();
  if (lane < CPW) static_cast<S *>(d.out)[o] = st_as<S, T>(acc);
}

// Column chains (colchain_kernel) when every warp's 32 (or 8) outputs are
// adjacent columns (output count and innermost output extent multiples of the
// group) and every
// operand either moves with the innermost output axis at unit stride, 16-byte
// aligned rows (staged), or ignores it (warp-uniform: staged once per step).
// Fewer than CC_MIN_OUT outputs leave too few warps to stream HBM; those keep
// the block-per-output chain kernels.  BGX_NO_COLCHAIN=1 for A/B.
constexpr int64_t CC_MIN_OUT = 512;

template <typename T, typename S = T>
bool try_colchain(const bgx_generic_desc &d, int64_t n_out, cudaStream_t s, int *rc) {
  static const bool off = getenv("BGX_NO_COLCHAIN") != nullptr;
  const int ax = d.n_axes - 1, inner = d.n_par - 1;
  if (off || n_out < CC_MIN_OUT || n_out % 8 || d.extents[inner] % 8 || d.extents[ax] < 64 ||
      n_out / 8 > 0x7fffffffLL)
    return false;
  int shm = 0;
  for (int k = 0; k < d.n_in; ++k) {
    if (d.strides[k][inner] == 0) { shm |= 1 << k; continue; }
    if (d.strides[k][inner] != 1 || ((uintptr_t)d.ins[k] % 16) != 0 ||
        (d.strides[k][ax] * (int64_t)sizeof(S)) % 16 != 0)
      return false;
    for (int a = 0; a < inner; ++a)
      if (d.extents[a] > 1 && (d.strides[k][a] * (int64_t)sizeof(S)) % 16 != 0) return false;
  }
  if (shm == (1 << d.n_in) - 1) return false;
  if (sizeof(S) == 2) {
    // 16-bit shared operands are staged 16 bytes at a time: unit stride along
    // the reduction, 16-byte aligned for every warp
    for (int k = 0; k < d.n_in; ++k) {
      if (!((shm >> k) & 1)) continue;
      if (d.strides[k][ax] != 1 || ((uintptr_t)d.ins[k] % 16) != 0) return false;
      for (int a = 0; a < inner; ++a)
        if (d.extents[a] > 1 && (d.strides[k][a] * 2) % 16 != 0) return false;
    }
  }
  // one warp per block (4-warp blocks: 10-40 % slower, scripts/r02/rr_vcols_ab.sh).
  // A warp's chains advance one tile per ~500 cycles whatever the pipeline
  // depth, so with fewer 32-column groups than SMs the columns are split 8 per
  // warp — 4x the warps — and the 8-column tiles keep 8 in flight
  const int sms = sm_count_current() > 0 ? sm_count_current() : 148;
  static const int cpw_env = getenv("BGX_CC_CPW") ? atoi(getenv("BGX_CC_CPW")) : 0;
  int cpw = cpw_env == 8 || cpw_env == 32 ? cpw_env : (n_out / 32 >= sms ? 32 : 8);
  if (n_out % cpw || d.extents[inner] % cpw) return false;
  const int64_t warps = n_out / cpw;
  const int st = warps >= 2 * sms ? 4 : 8;
  constexpr int E16 = 16 / (int)sizeof(S);
  const int npc = d.n_in - __builtin_popcount(shm);
  const size_t smem = (size_t)st * (npc * 32 * (cpw + E16) + (d.n_in - npc) * 32) * sizeof(S);
  auto go = [&](auto kern) {
    set_max_smem_once(reinterpret_cast<const void *>(kern), 200 * 1024);
    kern<<<(unsigned)warps, 32, smem, s>>>(d, n_out);
  };
  auto pick = [&](auto stc, auto cpwc) {
    constexpr int ST = decltype(stc)::value, CPW = decltype(cpwc)::value;
    if (d.n_in == 1) go(colchain_kernel<T, 1, 0, ST, CPW, S>);
    else if (shm == 0) go(colchain_kernel<T, 2, 0, ST, CPW, S>);
    else if (shm == 1) go(colchain_kernel<T, 2, 1, ST, CPW, S>);
    else go(colchain_kernel<T, 2, 2, ST, CPW, S>);
  };
  using I4 = std::integral_constant<int, 4>;
  using I8 = std::integral_constant<int, 8>;
  using I32 = std::integral_constant<int, 32>;
  if (cpw == 32) { if (st == 4) pick(I4{}, I32{}); else pick(I8{}, I32{}); }
  else { if (st == 4) pick(I4{}, I8{}); else pick(I8{}, I8{}); }
  *rc = check_launch("colchain_kernel");
  return true;
}

// S: storage type (f32/f64, or bf16/f16 folded in f32: 16-byte staged rows
// only — cp.async has no 2-byte copies)
template <typename T, typename S = T>
bool try_rowreduce(const bgx_generic_desc &d, int64_t n_out, cudaStream_t s, int *rc) {
  constexpr bool same = std::is_same<S, T>::value;
  if (d.n_axes != d.n_par + 1 || d.n_in < 1 || d.n_in > 2 || d.n_par < 1) return false;
  const int ax = d.n_axes - 1, inner = d.n_par - 1;
  if (try_colchain<T, S>(d, n_out, s, rc)) return true;
  bool rows = true, cols = true;
  // rows mode may carry operands constant along the reduction (a per-output
  // factor, loaded once per lane) as long as one operand streams the row
  uint32_t inv_mask = 0;
  bool streamed = false;
  for (int k = 0; k < d.n_in; ++k) {
    if (d.strides[k][ax] == 0 && d.extents[ax] > 1) inv_mask |= 1u << k;
    else streamed = streamed || d.strides[k][ax] == 1;
  }
  if (!streamed || inv_mask == (1u << d.n_in) - 1) inv_mask = 0;
  for (int k = 0; k < d.n_in; ++k) {
    rows = rows && (d.strides[k][ax] == 1 || ((inv_mask >> k) & 1));
    // consecutive outputs at consecutive addresses (or the input ignores the
    // output index entirely)
    bool shared = true;
    for (int a = 0; a < d.n_par; ++a) shared = shared && (d.strides[k][a] == 0 || d.extents[a] == 1);
    cols = cols && (d.strides[k][inner] == 1 || shared);
  }
  if (inv_mask) cols = false;
  if (!rows && !cols) return false;
  if (d.extents[ax] < 64 || n_out < 32) return false;
  if (!rows && d.extents[inner] < 32) return false;   // warps would straddle short rows
  // 16-byte staging: rows mode, every per-row operand 16-byte aligned with
  // its row strides in whole vectors (any reduction extent: tails are
  // zero-filled copies)
  bool vec = rows;
  for (int k = 0; k < d.n_in && vec; ++k) {
    if ((inv_mask >> k) & 1) continue;
    vec = ((uintptr_t)d.ins[k] % 16) == 0;
    for (int a = 0; a < d.n_par && vec; ++a)
      vec = d.extents[a] == 1 || (d.strides[k][a] * (int64_t)sizeof(S)) % 16 == 0;
  }
  if constexpr (!same) {
    if (!rows || !vec) return false;   // 16-bit storage: 16-byte staged rows only
  }
  // fewer outputs than 4 warps per SM: one-warp blocks, so every SM streams
  // (a warp's chains cannot be split across SMs)
  const int sms = sm_count_current();
  const bool few = n_out <= (int64_t)(sms > 0 ? sms : 148) * 32 * 4;
  // column mode: the per-thread loop nest keeps every SM full (this
  // kernel's staging holds one or two blocks per SM) — 1.2-4.7x faster with
  // many outputs and for one input; two inputs over few long columns keep
  // the staged kernel in one-warp blocks (profiles/r02_rowreduce_cols.txt)
  if (!rows && (!few || d.n_in == 1)) return false;
  const bool thin = (vec || !rows) && few;
  // thin rows: wide tiles (128 f32 / 64 f64 columns = one 16-byte vector per
  // lane per row, 2-3 in flight) — the per-tile issue and wait overhead,
  // not the bytes in flight, bounded these chains (GEMV 8192^2 123 -> 90 us,
  // profiles/r02_rowreduce_cols.txt); BGX_RR_THIN_TJ=32/64/128 for A/B
  static const int thin_tj_env = getenv("BGX_RR_THIN_TJ") ? atoi(getenv("BGX_RR_THIN_TJ")) : 0;
  const int nw = thin ? 1 : RR_WARPS;
  const bool thin_rows = thin && rows && vec;
  int tj = RR_TJ;
  if (thin_rows) {
    tj = thin_tj_env ? thin_tj_env : (sizeof(S) <= 4 ? 128 : 64);
    if (tj != 32 && tj != 64 && tj != 128) tj = RR_TJ;
    if (sizeof(S) == 8 && tj == 128) tj = 64;
  }
  int st = thin_rows ? (tj == 128 ? 2 : tj == 64 ? 3 : RR_STAGES) : RR_STAGES;
  // many outputs, one f32 input: 64-column tiles, 2 in flight (5-12 % faster
  // than 32 x 4: fewer tile iterations per element; BGX_RR_NARROW=1 for A/B)
  static const bool narrow_env = getenv("BGX_RR_NARROW") != nullptr;
  const bool wide4 = !narrow_env && !thin && rows && vec && d.n_in == 1 && sizeof(S) <= 4;
  if (wide4) { tj = 64; st = 2; }
  const int64_t blocks = (n_out + 32 * nw - 1) / (32 * nw);
  if (blocks > 0x7fffffffLL) return false;
  const size_t smem = (size_t)nw * st * d.n_in * 32 * rr_stride<S>(vec, tj) * sizeof(S);
  if (smem > 200 * 1024) return false;
  uint32_t shared_mask = 0;
  for (int k = 0; k < d.n_in; ++k) {
    bool shared = true;
    for (int a = 0; a < d.n_par; ++a) shared = shared && (d.strides[k][a] == 0 || d.extents[a] == 1);
    if (shared && !((inv_mask >> k) & 1)) shared_mask |= 1u << k;
  }
  shared_mask |= inv_mask << 8;
  auto go = [&](auto kern) {
    // once per (kernel, device), at the largest staging this path allows
    set_max_smem_once(reinterpret_cast<const void *>(kern), 200 * 1024);
    kern<<<(unsigned)blocks, 32 * nw, smem, s>>>(d, n_out, shared_mask);
  };
  constexpr bool f32 = sizeof(S) <= 4;   // 128-column tiles: f32 and 16-bit storage
  if (f32 && thin_rows && tj == 128) {
    if constexpr (f32) {
      if (d.n_in == 1) go(rowreduce_kernel<T, 1, false, true, 1, 2, 128, S>);
      else go(rowreduce_kernel<T, 2, false, true, 1, 2, 128, S>);
    }
  } else if (thin_rows && tj == 64) {
    if (d.n_in == 1) go(rowreduce_kernel<T, 1, false, true, 1, 3, 64, S>);
    else go(rowreduce_kernel<T, 2, false, true, 1, 3, 64, S>);
  } else if (thin_rows) {
    if (d.n_in == 1) go(rowreduce_kernel<T, 1, false, true, 1, RR_STAGES, RR_TJ, S>);
    else go(rowreduce_kernel<T, 2, false, true, 1, RR_STAGES, RR_TJ, S>);
  } else if (rows && vec && wide4) {
    if constexpr (f32) go(rowreduce_kernel<T, 1, false, true, RR_WARPS, 2, 64, S>);
  } else if (rows && vec) {
    if (d.n_in == 1) go(rowreduce_kernel<T, 1, false, true, RR_WARPS, RR_STAGES, RR_TJ, S>);
    else go(rowreduce_kernel<T, 2, false, true, RR_WARPS, RR_STAGES, RR_TJ, S>);
  } else if (rows) {
    if constexpr (same) {
      if (d.n_in == 1) go(rowreduce_kernel<T, 1, false>); else go(rowreduce_kernel<T, 2, false>);
    }
  } else {   // columns (few outputs: one-warp blocks over every SM)
    if constexpr (same) {
      if (d.n_in == 1) go(rowreduce_kernel<T, 1, true, false, 1>);
      else go(rowreduce_kernel<T, 2, true, false, 1>);
    }
  }
  *rc = check_launch("rowreduce_kernel");
  return true;
}

// ---- rank-0 outputs: ONE sequential chain (full reductions, dot products) ---
// Fold nvec 16-byte vectors of x (times y when NIN == 2: per-point products)
// into acc in order.  The shared loads run one group of G vectors ahead of the
// dependent adds: an unrolled loop without the carry-over waited a shared-load
// latency (~30 cycles) at the top of every group, ~5 instead of 4 cycles per
// point.  nvec must be a multiple of G.
template <typename T, int NIN, int G = 4>
__device__ __forceinline__ T fold16(const T *x, const T *y, int nvec, T acc) {
  constexpr int EV = 16 / (int)sizeof(T);
  const uint4 *xv = reinterpret_cast<const uint4 *>(x);
  const uint4 *yv = reinterpret_cast<const uint4 *>(NIN > 1 ? y : x);
  uint4 cx[G], cy[G];
#pragma unroll
  for (int i = 0; i < G; ++i) {
    cx[i] = xv[i];
    if constexpr (NIN > 1) cy[i] = yv[i];
  }
  const int ng = nvec / G;
  for (int g = 0; g < ng; ++g) {
    const int nb = (g + 1 < ng ? g + 1 : g) * G;
    uint4 nx[G], ny[G];
#pragma unroll
    for (int i = 0; i < G; ++i) {
      nx[i] = xv[nb + i];
      if constexpr (NIN > 1) ny[i] = yv[nb + i];
    }
#pragma unroll
    for (int i = 0; i < G; ++i) {
      const T *a = reinterpret_cast<const T *>(&cx[i]);
      const T *b = reinterpret_cast<const T *>(&cy[i]);
#pragma unroll
      for (int e = 0; e < EV; ++e) {
        T p = a[e];
        if constexpr (NIN > 1) p = mul_rn<T>(p, b[e]);
        acc = add_rn<T>(p, acc);
      }
    }
#pragma unroll
    for (int i = 0; i < G; ++i) {
      cx[i] = nx[i];
      if constexpr (NIN > 1) cy[i] = ny[i];
    }
  }
  return acc;
}

// The reference order makes the whole reduction one dependent chain of adds;
// only memory latency can be removed.  When every input is dense in the
// reduction order (row-major over the reduction axes), the block's threads
// stage the next tile of every input into shared memory (cp.async, coalesced)
// while thread 0 folds the current one from shared memory — the fold runs at
// the add latency instead of a global round trip per few elements.
constexpr int CH_TILE = 4096;   // elements per input per stage
constexpr int CH_THREADS = 256;

template <typename T, int NIN>
__global__ void __launch_bounds__(CH_THREADS) chain_kernel(const bgx_generic_desc d, int64_t total) {
  extern __shared__ __align__(16) uint8_t ch_smem_raw[];
  T *buf = reinterpret_cast<T *>(ch_smem_raw);     // [2][NIN][CH_TILE]
  const T *const *ins = reinterpret_cast<const T *const *>(d.ins);
  const int64_t ntiles = (total + CH_TILE - 1) / CH_TILE;
  auto issue = [&](int64_t t) {
    const int st = (int)(t & 1);
#pragma unroll
    for (int k = 0; k < NIN; ++k) {
      T *dst = buf + (st * NIN + k) * CH_TILE;
      for (int e = threadIdx.x; e < CH_TILE; e += CH_THREADS) {
        const int64_t g = t * CH_TILE + e;
        const bool ok = g < total;
        if constexpr (sizeof(T) == 4) cp_async4(dst + e, ins[k] + (ok ? g : 0), ok);
        else cp_async8(dst + e, ins[k] + (ok ? g : 0), ok);
      }
    }
    cp_async_commit();
  };
  T acc = d.c0 ? static_cast<const T *>(d.c0)[0] : T(0);
  issue(0);
  for (int64_t t = 0; t < ntiles; ++t) {
    if (t + 1 < ntiles) issue(t + 1); else cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    if (threadIdx.x == 0) {
      const int st = (int)(t & 1);
      const int64_t n = total - t * CH_TILE < CH_TILE ? total - t * CH_TILE : CH_TILE;
      const T *x0 = buf + (st * NIN + 0) * CH_TILE;
      const T *x1 = NIN > 1 ? buf + (st * NIN + 1) * CH_TILE : nullptr;
      int64_t e = 0;
      if (n == CH_TILE) {
        acc = fold16<T, NIN>(x0, x1, CH_TILE * (int)sizeof(T) / 16, acc);
        e = CH_TILE;
      }
      for (; e < n; ++e) {
        T p = x0[e];
        if constexpr (NIN > 1) p = mul_rn<T>(p, x1[e]);
        acc = add_rn<T>(p, acc);
      }
    }
    __syncthreads();                   // stage free before it is refilled
  }
  cp_async_wait<0>();
  if (threadIdx.x == 0) static_cast<T *>(d.out)[0] = acc;
}

template <typename T>
bool try_chain(const bgx_generic_desc &d, int64_t n_out, int64_t red, cudaStream_t s, int *rc) {
  if (n_out != 1 || d.n_par != 0 || d.n_in < 1 || d.n_in > 2 || red < 2 * CH_TILE) return false;
  for (int k = 0; k < d.n_in; ++k) {   // dense in the reduction order
    int64_t st = 1;
    for (int a = d.n_axes - 1; a >= 0; --a) {
      if (d.extents[a] != 1 && d.strides[k][a] != st) return false;
      st *= d.extents[a];
    }
  }
  const size_t smem = (size_t)2 * d.n_in * CH_TILE * sizeof(T);
  // smem is fixed per (T, n_in): set once per kernel and device (thread-safe)
  if (d.n_in == 1)
    set_max_smem_once(reinterpret_cast<const void *>(chain_kernel<T, 1>), (int)smem);
  else
    set_max_smem_once(reinterpret_cast<const void *>(chain_kernel<T, 2>), (int)smem);
  if (d.n_in == 1)
    chain_kernel<T, 1><<<1, CH_THREADS, smem, s>>>(d, red);
  else
    chain_kernel<T, 2><<<1, CH_THREADS, smem, s>>>(d, red);
  *rc = check_launch("chain_kernel");
  return true;
}

// ---- few outputs, long reductions, any operand layout ---------------------
// One block per output element.  Each output is still ONE dependent chain of
// adds in the reference's point order, but the per-point products
// p = ((x1*x2)*x3)... (per-op rounding; which thread forms a product does not
// change its bits) are formed by warps 1..7 into a shared-memory tile, each
// thread a contiguous run of points walked with an odometer, while thread 0
// folds the previous tile: the fold runs at the add latency whatever the
// operand strides (broadcast operands, transposed walks, 3+ inputs).
// points per producer thread (16 f32 / 8 f64) and per stage (3584 / 1792)
template <typename T> constexpr int cg_per() { return sizeof(T) == 4 ? 16 : 8; }
template <typename T> constexpr int cg_tile() { return (CH_THREADS - 32) * cg_per<T>(); }

template <typename T>
__global__ void __launch_bounds__(CH_THREADS) chain_general_kernel(const bgx_generic_desc d,
                                                                   int64_t red) {
  constexpr int CG_PER = cg_per<T>(), CG_TILE = cg_tile<T>();
  __shared__ __align__(16) T buf[2][CG_TILE];
  const T *const *ins = reinterpret_cast<const T *const *>(d.ins);
  const int n_in = d.n_in, n_par = d.n_par, n_axes = d.n_axes;
  // this block's output element and its operand base offsets
  int64_t base[BGX_MAX_OPERANDS];
  for (int k = 0; k < BGX_MAX_OPERANDS; ++k) base[k] = 0;
  {
    int64_t rem = blockIdx.x;
    for (int a = n_par - 1; a >= 0; --a) {
      const int64_t i = rem % d.extents[a];
      rem /= d.extents[a];
      for (int k = 0; k < n_in; ++k) base[k] += i * d.strides[k][a];
    }
  }
  const int64_t ntiles = (red + CG_TILE - 1) / CG_TILE;
  auto produce = [&](int64_t t) {
    if (threadIdx.x < 32) return;                  // warp 0 folds
    const int64_t e0 = t * CG_TILE + (int64_t)(threadIdx.x - 32) * CG_PER;
    if (e0 >= red) return;
    int64_t idx[BGX_MAX_AXES], off[BGX_MAX_OPERANDS];
    for (int k = 0; k < n_in; ++k) off[k] = base[k];
    int64_t rem = e0;
    for (int a = n_axes - 1; a >= n_par; --a) {
      idx[a] = rem % d.extents[a];
      rem /= d.extents[a];
      for (int k = 0; k < n_in; ++k) off[k] += idx[a] * d.strides[k][a];
    }
    T *dst = buf[t & 1] + (threadIdx.x - 32) * CG_PER;
    const int n = red - e0 < CG_PER ? (int)(red - e0) : CG_PER;
    const int ai = n_axes - 1;
    if (n == CG_PER && ai >= n_par && idx[ai] + CG_PER <= d.extents[ai]) {
      // the run stays on the innermost reduction axis: CG_PER independent
      // loads per operand in flight (the odometer loop below waits a memory
      // round trip per point — the producers, not the fold, bounded
      // gathers like (a,c,b),(b,a),(b)->(b))
      T v[CG_PER];
      const int64_t s0 = d.strides[0][ai];
#pragma unroll
      for (int j = 0; j < CG_PER; ++j) v[j] = ins[0][off[0] + j * s0];
      for (int k = 1; k < n_in; ++k) {
        const int64_t sk = d.strides[k][ai];
        T w[CG_PER];
#pragma unroll
        for (int j = 0; j < CG_PER; ++j) w[j] = ins[k][off[k] + j * sk];
#pragma unroll
        for (int j = 0; j < CG_PER; ++j) v[j] = mul_rn<T>(v[j], w[j]);
      }
#pragma unroll
      for (int j = 0; j < CG_PER; ++j) dst[j] = v[j];
      return;
    }
    for (int j = 0; j < n; ++j) {
      T p = ins[0][off[0]];
      for (int k = 1; k < n_in; ++k) p = mul_rn<T>(p, ins[k][off[k]]);
      dst[j] = p;
      for (int a = n_axes - 1; a >= n_par; --a) {     // odometer, innermost fastest
        for (int k = 0; k < n_in; ++k) off[k] += d.strides[k][a];
        if (++idx[a] < d.extents[a]) break;
        for (int k = 0; k < n_in; ++k) off[k] -= d.extents[a] * d.strides[k][a];
        idx[a] = 0;
      }
    }
  };
  T acc = d.c0 ? static_cast<const T *>(d.c0)[blockIdx.x] : T(0);
  produce(0);
  __syncthreads();
  for (int64_t t = 0; t < ntiles; ++t) {
    if (t + 1 < ntiles) produce(t + 1);
    if (threadIdx.x == 0) {
      const T *x = buf[t & 1];
      const int64_t n = red - t * CG_TILE < CG_TILE ? red - t * CG_TILE : CG_TILE;
      int64_t e = 0;
      // whole groups of 4 16-byte vectors pipelined, the rest one by one
      const int nv = (int)(n * (int64_t)sizeof(T) / 16) / 4 * 4;
      if (nv > 0) {
        acc = fold16<T, 1>(x, nullptr, nv, acc);
        e = (int64_t)nv * (16 / (int)sizeof(T));
      }
      for (; e < n; ++e) acc = add_rn<T>(x[e], acc);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) static_cast<T *>(d.out)[blockIdx.x] = acc;
}

// Few outputs (<= 4 per SM) over long reductions (>= 2 tiles each): the
// one-thread-per-output loop nest would leave almost every SM idle and wait a
// memory round trip every few points.
template <typename T>
bool try_chain_general(const bgx_generic_desc &d, int64_t n_out, int64_t red, cudaStream_t s,
                       int *rc) {
  const int sms = sm_count_current();
  if (n_out < 1 || n_out > 4 * (int64_t)(sms > 0 ? sms : 148) || red < 2 * cg_tile<T>() ||
      d.n_in < 1 || d.n_axes <= d.n_par)
    return false;
  chain_general_kernel<T><<<(unsigned)n_out, CH_THREADS, 0, s>>>(d, red);
  *rc = check_launch("chain_general_kernel");
  return true;
}

// What the row / column kernels left for the per-thread loop nest, when that
// walk cannot coalesce (no parallel axis moves the largest operand at unit
// stride: each thread streams its own run, a warp load touches 32 lines):
// block-per-output chains for up to 32 outputs per SM and reductions of at
// least 1024 points, whose producer warps read each output's points
// contiguously: (b,a,c),(c,a)->(b) 2048 x 4096 points 291 -> 104 us,
// (d,a,c),(c,a),(c)->(d) 4096 x 2048 159 -> 138 us; with more outputs or
// shorter chains the per-block cost loses to the loop nest (8192 x 2048:
// 151 -> 225 us, scripts/r02/cg_wide_ab.sh).  BGX_NO_CG_WIDE=1 for A/B.
template <typename T>
bool try_chain_general_wide(const bgx_generic_desc &d, int64_t n_out, int64_t red, cudaStream_t s,
                            int *rc) {
  static const bool off = getenv("BGX_NO_CG_WIDE") != nullptr;
  const int sms = sm_count_current();
  if (off || n_out < 1 || n_out > 32 * (int64_t)(sms > 0 ? sms : 148) || red < 1024 || d.n_in < 1 ||
      d.n_axes <= d.n_par || n_out > 0x7fffffffLL)
    return false;
  int big = 0;
  int64_t bigsz = -1;
  for (int k = 0; k < d.n_in; ++k) {
    int64_t sz = 1;   // elements the operand spans (product of the extents it moves along)
    for (int a = 0; a < d.n_axes; ++a)
      if (d.strides[k][a] != 0) sz *= d.extents[a];
    if (sz > bigsz) { bigsz = sz; big = k; }
  }
  for (int a = 0; a < d.n_par; ++a)
    if (d.extents[a] > 1 && (d.strides[big][a] == 1 || d.strides[big][a] == -1)) return false;
  chain_general_kernel<T><<<(unsigned)n_out, CH_THREADS, 0, s>>>(d, red);
  *rc = check_launch("chain_general_kernel");
  return true;
}

template <typename S, typename T>
int launch_generic(const bgx_generic_desc &d0, int64_t n_out, int64_t red, cudaStream_t s) {
  const bgx_generic_desc d = coalesce_axes(d0);
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
  if constexpr (std::is_same<S, T>::value) {   // f32 / f64 storage
    int rc = 0;
    // BGX_NO_ROWREDUCE=1: force the per-thread loop nest (A/B timing only)
    static const bool no_rr = getenv("BGX_NO_ROWREDUCE") != nullptr;
    // few outputs over long reductions first: a block per output folds at the
    // add latency, where the row / column kernels' few warps pay a tile
    // pipeline per 32 points ((d,b,a)->(d) 256 x 16384: 127 -> 58 us)
    if (!no_rr && try_chain<T>(d, n_out, red, s, &rc)) return rc;
    if (!no_rr && try_chain_general<T>(d, n_out, red, s, &rc)) return rc;
    if (!no_rr && try_rowreduce<T>(d, n_out, s, &rc)) return rc;
    if (!no_rr && try_chain_general_wide<T>(d, n_out, red, s, &rc)) return rc;
  } else {
    // bf16 / f16 storage folded in f32: the staged row kernel (16-byte rows)
    int rc = 0;
    static const bool no_rr = getenv("BGX_NO_ROWREDUCE") != nullptr;
    if (!no_rr && try_rowreduce<T, S>(d, n_out, s, &rc)) return rc;
  }
  if (dense && d.n_in >= 2 && d.n_in <= 3 && red == 1) {
    bool aligned = ((uintptr_t)d.out % 16 == 0) && ((uintptr_t)d.c0 % 16 == 0);
    for (int k = 0; k < d.n_in; ++k) aligned = aligned && ((uintptr_t)d.ins[k] % 16 == 0);
    if (aligned) {
      int64_t vb = (n_out / (16 / (int64_t)sizeof(S)) + 255) / 256;
      if (vb > (int64_t)sms * 16) vb = (int64_t)sms * 16;
      if (vb < 1) vb = 1;
      if (d.n_in == 2) dense_ew_kernel<S, T, 2><<<(unsigned)vb, 256, 0, s>>>(d, n_out);
      else dense_ew_kernel<S, T, 3><<<(unsigned)vb, 256, 0, s>>>(d, n_out);
      return check_launch("dense_ew_kernel");
    }
  }
  // broadcast / strided elementwise bodies: V outputs per thread along the
  // innermost output axis (BGX_NO_BCAST_EW=1 for A/B)
  static const bool no_bcast = getenv("BGX_NO_BCAST_EW") != nullptr;
  if (!no_bcast && !dense && d.n_axes == d.n_par && d.n_par >= 1 && d.n_in >= 2 && d.n_in <= 3 &&
      red == 1 && d.extents[d.n_par - 1] % (16 / (int64_t)sizeof(S)) == 0 &&
      (uintptr_t)d.out % 16 == 0 && (uintptr_t)d.c0 % 16 == 0) {
    int64_t vb = (n_out / (16 / (int64_t)sizeof(S)) + 255) / 256;
    if (vb > (int64_t)sms * 16) vb = (int64_t)sms * 16;
    if (vb < 1) vb = 1;
    static const bool no_rows = getenv("BGX_BCAST_NO_ROWS") != nullptr;   // A/B only
    // rows of at least 32 x U vectors (U = 4, 2 for 16-bit; shorter rows idle
    // lanes) and enough rows for 16 warps per SM (256 rows of 65536: 2.6x
    // slower than one decode per vector)
    const bool rows = !no_rows &&
                      d.extents[d.n_par - 1] / (16 / (int64_t)sizeof(S)) >= (sizeof(S) == 2 ? 64 : 128) &&
                      n_out / d.extents[d.n_par - 1] >= 16 * (int64_t)sms;
    if (rows) {
      const int64_t nrows = n_out / d.extents[d.n_par - 1];
      int64_t rb = (nrows + 7) / 8;   // 8 warps per block, a row per warp
      if (rb > (int64_t)sms * 16) rb = (int64_t)sms * 16;
      if (rb < 1) rb = 1;
      if (d.n_in == 2) bcast_ew_kernel<S, T, 2, true><<<(unsigned)rb, 256, 0, s>>>(d, n_out);
      else bcast_ew_kernel<S, T, 3, true><<<(unsigned)rb, 256, 0, s>>>(d, n_out);
    } else if (d.n_in == 2) {
      bcast_ew_kernel<S, T, 2, false><<<(unsigned)vb, 256, 0, s>>>(d, n_out);
    } else {
      bcast_ew_kernel<S, T, 3, false><<<(unsigned)vb, 256, 0, s>>>(d, n_out);
    }
    return check_launch("bcast_ew_kernel");
  }
  if (dense) {
    launch_generic_n<S, T, true>(d, n_out, red, (unsigned)blocks, s);
  } else {
    static const bool no_walk = getenv("BGX_NO_WALK_ORDER") != nullptr;   // A/B only
    bgx_generic_desc w;
    OutMap om{};
    if (!no_walk && walk_order(d, w, om))
      launch_generic_n<S, T, false>(w, n_out, red, (unsigned)blocks, s, &om);
    else
      launch_generic_n<S, T, false>(d, n_out, red, (unsigned)blocks, s);
  }
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
