// bgx_generic_tree — tolerance-mode reductions for einsum bodies
// (bridgegen interp.py:372-424 with the einsum.py:111-117 body, minus the
// reference's summation ORDER).
//
// The exact kernels (generic.cu) keep the reference's bits, which forces one
// sequential chain per output element: a 4096^2 full sum is one chain of 16.7 M
// dependent adds (59 ms).  Callers that accept a bounded rounding difference
// (BGX_MODE_FFMA / contract(mode="ffma")) get this instead: the reduction
// sub-space of each output element is cut into `splits` chunks, each chunk is
// summed by one 256-thread block (strided per-thread partial sums, then a
// warp-shuffle / shared-memory tree), and a second pass adds the chunk sums
// in chunk order plus c0.  Deterministic (fixed order everywhere), f32
// accumulation for f32/bf16/f16 (f64 for f64), one final rounding to the
// storage type.  Relative error ~ sqrt(log2 n) * eps typical vs the exact
// sum.  Memory-bound: n_in * elem bytes per point.
#include "common.cuh"

namespace bgx {
namespace {

constexpr int TR_THREADS = 256;
constexpr int64_t TR_MIN_CHUNK = 2048;   // points per block at least

template <typename S, typename T> __device__ __forceinline__ T ld_t(const S *p) {
  return (T)Conv<S>::to_f(*p);
}
template <> __device__ __forceinline__ double ld_t<double, double>(const double *p) { return *p; }
template <typename S, typename T> __device__ __forceinline__ S st_t(T v) {
  return Conv<S>::from_f((float)v);
}
template <> __device__ __forceinline__ double st_t<double, double>(double v) { return v; }

// Offsets of output element o over the parallel axes.
__device__ __forceinline__ void par_offsets(const bgx_generic_desc &d, int64_t o, int n_in,
                                            int64_t *off) {
  for (int k = 0; k < n_in; ++k) off[k] = 0;
  int64_t rem = o;
  for (int a = d.n_par - 1; a >= 0; --a) {
    const int64_t e = d.extents[a];
    const int64_t i = rem % e;
    rem /= e;
    for (int k = 0; k < n_in; ++k) off[k] += i * d.strides[k][a];
  }
}

template <typename T> __device__ __forceinline__ T block_sum(T v, T *red) {
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) v += __shfl_xor_sync(0xffffffffu, v, s);
  const int w = threadIdx.x / 32, l = threadIdx.x % 32;
  if (l == 0) red[w] = v;
  __syncthreads();
  T t = 0;
  if (w == 0) {
    t = l < TR_THREADS / 32 ? red[l] : T(0);
#pragma unroll
    for (int s = 4; s > 0; s >>= 1) t += __shfl_xor_sync(0xffffffffu, t, s);
  }
  __syncthreads();   // red reusable by the next block iteration
  return t;          // valid in thread 0
}

// Block b -> (output o = b / splits, chunk s = b % splits) over points
// [s * chunk, min(red, (s + 1) * chunk)) of o's reduction sub-space (the
// reduction axes in the reference's order, last fastest: consecutive
// threads take consecutive points, coalesced when that axis is contiguous).
template <typename S, typename T, int NIN>
__global__ void __launch_bounds__(TR_THREADS)
tree_partial_kernel(const bgx_generic_desc d, int64_t n_out, int64_t red, int splits,
                    int64_t chunk, T *ws) {
  __shared__ T sred[TR_THREADS / 32];
  const int n_in = NIN > 0 ? NIN : d.n_in;
  const int n_red = d.n_axes - d.n_par;
  const S *const *ins = reinterpret_cast<const S *const *>(d.ins);
  for (int64_t blk = blockIdx.x; blk < n_out * splits; blk += gridDim.x) {
    const int64_t o = blk / splits;
    const int s = (int)(blk % splits);
    int64_t base[BGX_MAX_OPERANDS];
    par_offsets(d, o, n_in, base);
    const int64_t lo = (int64_t)s * chunk;
    const int64_t hi = lo + chunk < red ? lo + chunk : red;
    T acc = 0;
    const bool one_axis = n_red == 1, idx32 = red <= 0x7fffffffLL;
    for (int64_t r = lo + threadIdx.x; r < hi; r += TR_THREADS) {
      int64_t off[BGX_MAX_OPERANDS];
#pragma unroll
      for (int k = 0; k < BGX_MAX_OPERANDS; ++k)
        if (k < n_in) off[k] = base[k] + (one_axis ? r * d.strides[k][d.n_par] : 0);
      if (!one_axis) {   // reduction coordinates of point r (last axis fastest)
        if (idx32) {
          uint32_t rem = (uint32_t)r;
          for (int a = n_red - 1; a >= 0; --a) {
            const int ax = d.n_par + a;
            const uint32_t e = (uint32_t)d.extents[ax];
            const uint32_t q = rem / e, i = rem - q * e;
            rem = q;
#pragma unroll
            for (int k = 0; k < BGX_MAX_OPERANDS; ++k)
              if (k < n_in) off[k] += (int64_t)i * d.strides[k][ax];
          }
        } else {
          int64_t rem = r;
          for (int a = n_red - 1; a >= 0; --a) {
            const int ax = d.n_par + a;
            const int64_t e = d.extents[ax];
            const int64_t i = rem % e;
            rem /= e;
#pragma unroll
            for (int k = 0; k < BGX_MAX_OPERANDS; ++k)
              if (k < n_in) off[k] += i * d.strides[k][ax];
          }
        }
      }
      T p = ld_t<S, T>(ins[0] + off[0]);
#pragma unroll
      for (int k = 1; k < BGX_MAX_OPERANDS; ++k)
        if (k < n_in) p *= ld_t<S, T>(ins[k] + off[k]);
      acc += p;
    }
    acc = block_sum<T>(acc, sred);
    if (threadIdx.x == 0) {
      if (splits == 1) {
        if (d.c0) acc += ld_t<S, T>(static_cast<const S *>(d.c0) + o);
        static_cast<S *>(d.out)[o] = st_t<S, T>(acc);
      } else {
        ws[o * splits + s] = acc;
      }
    }
  }
}

// VEC consecutive storage elements as T (one 16-byte load).
template <typename S, typename T> struct Vec {
  static constexpr int N = 16 / (int)sizeof(S);
  __device__ static void load(const S *p, T *v) {
    const uint4 q = *reinterpret_cast<const uint4 *>(p);
    const S *e = reinterpret_cast<const S *>(&q);
#pragma unroll
    for (int i = 0; i < N; ++i) v[i] = ld_t<S, T>(e + i);
  }
};

// CONTIG layout: every input's reduction sub-space is one dense run (the
// reduction axes row-major with unit innermost stride), so point r of output
// o sits at base + r: 16-byte vector loads, several in flight per thread.
template <typename S, typename T, int NIN>
__global__ void __launch_bounds__(TR_THREADS)
tree_contig_kernel(const bgx_generic_desc d, int64_t n_out, int64_t red, int splits,
                   int64_t chunk, T *ws) {
  __shared__ T sred[TR_THREADS / 32];
  constexpr int V = Vec<S, T>::N;
  constexpr int U = 4;
  const S *const *ins = reinterpret_cast<const S *const *>(d.ins);
  for (int64_t blk = blockIdx.x; blk < n_out * splits; blk += gridDim.x) {
    const int64_t o = blk / splits;
    const int s = (int)(blk % splits);
    int64_t base[BGX_MAX_OPERANDS];
    par_offsets(d, o, NIN, base);
    const int64_t lo = (int64_t)s * chunk;
    const int64_t n = (lo + chunk < red ? lo + chunk : red) - lo;
    const S *p[NIN];
    bool aligned = true;
#pragma unroll
    for (int k = 0; k < NIN; ++k) {
      p[k] = ins[k] + base[k] + lo;
      aligned = aligned && ((uintptr_t)p[k] % 16 == 0);
    }
    T acc = 0;
    int64_t done = 0;
    if (aligned) {
      const int64_t nv = n / V;
      int64_t i = threadIdx.x;
      for (; i + (U - 1) * TR_THREADS < nv; i += U * TR_THREADS) {
        T v[U][NIN][V];
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int k = 0; k < NIN; ++k) Vec<S, T>::load(p[k] + (i + u * TR_THREADS) * V, v[u][k]);
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int e = 0; e < V; ++e) {
            T q = v[u][0][e];
#pragma unroll
            for (int k = 1; k < NIN; ++k) q *= v[u][k][e];
            acc += q;
          }
      }
      for (; i < nv; i += TR_THREADS) {
        T v[NIN][V];
#pragma unroll
        for (int k = 0; k < NIN; ++k) Vec<S, T>::load(p[k] + i * V, v[k]);
#pragma unroll
        for (int e = 0; e < V; ++e) {
          T q = v[0][e];
#pragma unroll
          for (int k = 1; k < NIN; ++k) q *= v[k][e];
          acc += q;
        }
      }
      done = nv * V;
    }
    for (int64_t i = done + threadIdx.x; i < n; i += TR_THREADS) {
      T q = ld_t<S, T>(p[0] + i);
#pragma unroll
      for (int k = 1; k < NIN; ++k) q *= ld_t<S, T>(p[k] + i);
      acc += q;
    }
    acc = block_sum<T>(acc, sred);
    if (threadIdx.x == 0) {
      if (splits == 1) {
        if (d.c0) acc += ld_t<S, T>(static_cast<const S *>(d.c0) + o);
        static_cast<S *>(d.out)[o] = st_t<S, T>(acc);
      } else {
        ws[o * splits + s] = acc;
      }
    }
  }
}

// COLUMN layout: the innermost OUTPUT axis has unit stride (or is broadcast)
// in every input and the reduction runs across it (column sums, x^T A): a
// block owns 32 consecutive outputs along that axis — one per lane, so each
// warp load is one 128-byte line — and its 8 warps split the reduction
// points of its chunk; the 8 partials per output are added in warp order.
template <typename S, typename T, int NIN>
__global__ void __launch_bounds__(TR_THREADS)
tree_column_kernel(const bgx_generic_desc d, int64_t n_tiles, int64_t red, int splits,
                   int64_t chunk, T *ws) {
  __shared__ T part[TR_THREADS / 32][32];
  const int pl = d.n_par - 1;
  const int64_t E = d.extents[pl];
  const int64_t ctiles = (E + 31) / 32;
  const int n_red = d.n_axes - d.n_par;
  const int w = threadIdx.x / 32, lane = threadIdx.x % 32;
  const S *const *ins = reinterpret_cast<const S *const *>(d.ins);
  for (int64_t blk = blockIdx.x; blk < n_tiles * splits; blk += gridDim.x) {
    const int64_t t = blk / splits;
    const int s = (int)(blk % splits);
    const int64_t q = t / ctiles, c = (t % ctiles) * 32 + lane;
    const bool live = c < E;
    int64_t base[BGX_MAX_OPERANDS];
#pragma unroll
    for (int k = 0; k < NIN; ++k) base[k] = (live ? c : 0) * d.strides[k][pl];
    int64_t rem = q;
    for (int a = pl - 1; a >= 0; --a) {
      const int64_t e = d.extents[a];
      const int64_t i = rem % e;
      rem /= e;
#pragma unroll
      for (int k = 0; k < NIN; ++k) base[k] += i * d.strides[k][a];
    }
    const int64_t lo = (int64_t)s * chunk;
    const int64_t hi = lo + chunk < red ? lo + chunk : red;
    T acc = 0;
    constexpr int W = TR_THREADS / 32;
    if (n_red == 1) {
      // one reduction axis: point r at base + r * stride; U points of every
      // warp in flight at once
      constexpr int U = 8;
      int64_t st[NIN];
#pragma unroll
      for (int k = 0; k < NIN; ++k) st[k] = d.strides[k][d.n_par];
      int64_t r = lo + w;
      if (live) {
        for (; r + (U - 1) * W < hi; r += U * W) {
          T v[U];
#pragma unroll
          for (int u = 0; u < U; ++u) v[u] = ld_t<S, T>(ins[0] + base[0] + (r + u * W) * st[0]);
#pragma unroll
          for (int k = 1; k < NIN; ++k)
#pragma unroll
            for (int u = 0; u < U; ++u) v[u] *= ld_t<S, T>(ins[k] + base[k] + (r + u * W) * st[k]);
#pragma unroll
          for (int u = 0; u < U; ++u) acc += v[u];
        }
        for (; r < hi; r += W) {
          T v = ld_t<S, T>(ins[0] + base[0] + r * st[0]);
#pragma unroll
          for (int k = 1; k < NIN; ++k) v *= ld_t<S, T>(ins[k] + base[k] + r * st[k]);
          acc += v;
        }
      }
    } else {
      for (int64_t r = lo + w; r < hi; r += W) {
        int64_t off[NIN];
#pragma unroll
        for (int k = 0; k < NIN; ++k) off[k] = base[k];
        int64_t rr = r;
        for (int a = n_red - 1; a >= 0; --a) {   // warp-uniform
          const int ax = d.n_par + a;
          const int64_t e = d.extents[ax];
          const int64_t i = rr % e;
          rr /= e;
#pragma unroll
          for (int k = 0; k < NIN; ++k) off[k] += i * d.strides[k][ax];
        }
        if (live) {
          T v = ld_t<S, T>(ins[0] + off[0]);
#pragma unroll
          for (int k = 1; k < NIN; ++k) v *= ld_t<S, T>(ins[k] + off[k]);
          acc += v;
        }
      }
    }
    part[w][lane] = acc;
    __syncthreads();
    if (w == 0 && live) {
      T sum = 0;
#pragma unroll
      for (int j = 0; j < TR_THREADS / 32; ++j) sum += part[j][lane];
      const int64_t o = q * E + c;
      if (splits == 1) {
        if (d.c0) sum += ld_t<S, T>(static_cast<const S *>(d.c0) + o);
        static_cast<S *>(d.out)[o] = st_t<S, T>(sum);
      } else {
        ws[o * splits + s] = sum;
      }
    }
    __syncthreads();
  }
}

// out[o] = c0[o] + sum over chunks in chunk order.
template <typename S, typename T>
__global__ void __launch_bounds__(TR_THREADS)
tree_finish_kernel(const bgx_generic_desc d, int64_t n_out, int splits, const T *ws) {
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < n_out;
       o += (int64_t)gridDim.x * blockDim.x) {
    T acc = 0;
    for (int s = 0; s < splits; ++s) acc += ws[o * splits + s];
    if (d.c0) acc += ld_t<S, T>(static_cast<const S *>(d.c0) + o);
    static_cast<S *>(d.out)[o] = st_t<S, T>(acc);
  }
}

enum class TreeLayout { General, Contig, Column };

// Which kernel fits the operand layout (see the kernels above).
TreeLayout tree_layout(const bgx_generic_desc &d) {
  bool contig = true;
  for (int k = 0; k < d.n_in && contig; ++k) {
    int64_t st = 1;
    for (int a = d.n_axes - 1; a >= d.n_par && contig; --a) {
      if (d.extents[a] != 1 && d.strides[k][a] != st) contig = false;
      st *= d.extents[a];
    }
  }
  if (contig) return TreeLayout::Contig;
  if (d.n_par >= 1 && d.extents[d.n_par - 1] >= 32) {
    const int pl = d.n_par - 1;
    bool col = false, ok = true;
    for (int k = 0; k < d.n_in; ++k) {
      if (d.strides[k][pl] == 1) col = true;
      else if (d.strides[k][pl] != 0) ok = false;
    }
    if (ok && col) return TreeLayout::Column;
  }
  return TreeLayout::General;
}

// Independent units the layout's kernel distributes (outputs, or 32-wide
// column tiles), and the chunk count per unit: enough blocks to fill the
// GPU (8 per SM), each chunk at least TR_MIN_CHUNK points.
int64_t tree_units(const bgx_generic_desc &d, TreeLayout lay, int64_t n_out) {
  if (lay != TreeLayout::Column) return n_out;
  const int64_t E = d.extents[d.n_par - 1];
  return (n_out / E) * ((E + 31) / 32);
}

int tree_splits(int64_t units, int64_t red, TreeLayout lay) {
  const int sms = sm_count_current();
  const int64_t target = (int64_t)(sms > 0 ? sms : 148) * 8;   // 8 blocks of 256 per SM
  int64_t sp = (target + units - 1) / units;
  const int64_t min_chunk = lay == TreeLayout::Column ? 256 : TR_MIN_CHUNK;
  const int64_t by_size = (red + min_chunk - 1) / min_chunk;
  if (sp > by_size) sp = by_size;
  if (sp > 65536) sp = 65536;
  return sp < 1 ? 1 : (int)sp;
}

template <typename S, typename T>
int launch_tree(const bgx_generic_desc &d, int64_t n_out, int64_t red, void *ws,
                int64_t ws_bytes, cudaStream_t s) {
  TreeLayout lay = tree_layout(d);
  if (d.n_in > 3 && lay != TreeLayout::General) lay = TreeLayout::General;
  const int64_t units = tree_units(d, lay, n_out);
  const int splits = tree_splits(units, red, lay);
  int64_t chunk = (red + splits - 1) / splits;
  if (lay == TreeLayout::Contig) chunk = (chunk + 63) / 64 * 64;   // keeps 16-byte vector runs aligned
  if (splits > 1 && (ws == nullptr || ws_bytes < n_out * splits * (int64_t)sizeof(T))) {
    set_error("bgx_generic_tree: workspace of %lld bytes needed",
              (long long)(n_out * splits * (int64_t)sizeof(T)));
    return BGX_ERR_INVALID;
  }
  const int sms = sm_count_current();
  int64_t blocks = units * splits;
  const int64_t cap = (int64_t)(sms > 0 ? sms : 148) * 32;
  if (blocks > cap) blocks = cap;
  T *w = static_cast<T *>(ws);
  const unsigned g = (unsigned)blocks;
#define BGX_TREE_LAUNCH(KERN, ARG0)                                                        \
  switch (d.n_in) {                                                                        \
    case 1: KERN<S, T, 1><<<g, TR_THREADS, 0, s>>>(d, ARG0, red, splits, chunk, w); break;  \
    case 2: KERN<S, T, 2><<<g, TR_THREADS, 0, s>>>(d, ARG0, red, splits, chunk, w); break;  \
    default: KERN<S, T, 3><<<g, TR_THREADS, 0, s>>>(d, ARG0, red, splits, chunk, w); break; \
  }
  if (lay == TreeLayout::Contig) {
    BGX_TREE_LAUNCH(tree_contig_kernel, n_out)
  } else if (lay == TreeLayout::Column) {
    BGX_TREE_LAUNCH(tree_column_kernel, units)
  } else {
    switch (d.n_in) {
      case 1: tree_partial_kernel<S, T, 1><<<g, TR_THREADS, 0, s>>>(d, n_out, red, splits, chunk, w); break;
      case 2: tree_partial_kernel<S, T, 2><<<g, TR_THREADS, 0, s>>>(d, n_out, red, splits, chunk, w); break;
      case 3: tree_partial_kernel<S, T, 3><<<g, TR_THREADS, 0, s>>>(d, n_out, red, splits, chunk, w); break;
      default: tree_partial_kernel<S, T, 0><<<g, TR_THREADS, 0, s>>>(d, n_out, red, splits, chunk, w); break;
    }
  }
#undef BGX_TREE_LAUNCH
  int rc = check_launch("tree_partial_kernel");
  if (rc != BGX_OK || splits == 1) return rc;
  int64_t fb = (n_out + TR_THREADS - 1) / TR_THREADS;
  if (fb > cap) fb = cap;
  tree_finish_kernel<S, T><<<(unsigned)fb, TR_THREADS, 0, s>>>(d, n_out, splits, w);
  return check_launch("tree_finish_kernel");
}

int tree_check(const bgx_generic_desc *d, int64_t *n_out, int64_t *red) {
  BGX_CHECK_ARG(d != nullptr, "bgx_generic_tree: null descriptor");
  BGX_CHECK_ARG(d->n_in >= 1 && d->n_in <= BGX_MAX_OPERANDS, "bgx_generic_tree: n_in %d", d->n_in);
  BGX_CHECK_ARG(d->n_axes >= 0 && d->n_axes <= BGX_MAX_AXES && d->n_par >= 0 &&
                    d->n_par < d->n_axes,
                "bgx_generic_tree: needs at least one reduction axis (axes %d / parallel %d)",
                d->n_axes, d->n_par);
  BGX_CHECK_ARG(d->dtype == BGX_F32 || d->dtype == BGX_F64 || d->dtype == BGX_BF16 ||
                    d->dtype == BGX_F16,
                "bgx_generic_tree: dtype %d", d->dtype);
  *n_out = 1;
  *red = 1;
  for (int a = 0; a < d->n_axes; ++a) {
    BGX_CHECK_ARG(d->extents[a] >= 0, "bgx_generic_tree: negative extent");
    if (a < d->n_par) *n_out *= d->extents[a]; else *red *= d->extents[a];
  }
  return BGX_OK;
}

}  // namespace
}  // namespace bgx

using namespace bgx;

extern "C" int bgx_generic_tree_plan(const bgx_generic_desc *d, int64_t *workspace_bytes) {
  BGX_CHECK_ARG(workspace_bytes != nullptr, "bgx_generic_tree_plan: null output");
  int64_t n_out, red;
  const int rc = tree_check(d, &n_out, &red);
  if (rc != BGX_OK) return rc;
  TreeLayout lay = tree_layout(*d);
  if (d->n_in > 3 && lay != TreeLayout::General) lay = TreeLayout::General;
  const int splits =
      (n_out > 0 && red > 0) ? tree_splits(tree_units(*d, lay, n_out), red, lay) : 1;
  const int64_t esz = d->dtype == BGX_F64 ? 8 : 4;
  *workspace_bytes = splits > 1 ? n_out * splits * esz : 0;
  return BGX_OK;
}

extern "C" int bgx_generic_tree(const bgx_generic_desc *d, void *workspace,
                                int64_t workspace_bytes, void *stream) {
  int64_t n_out, red;
  const int rc = tree_check(d, &n_out, &red);
  if (rc != BGX_OK) return rc;
  if (n_out == 0) return BGX_OK;
  if (red == 0) return bgx_generic(d, stream);   // nothing to sum: c0 (or +0) is the result
  BGX_CHECK_ARG(d->out != nullptr, "bgx_generic_tree: null out");
  for (int k = 0; k < d->n_in; ++k)
    BGX_CHECK_ARG(d->ins[k] != nullptr, "bgx_generic_tree: null input");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  switch (d->dtype) {
    case BGX_F32: return launch_tree<float, float>(*d, n_out, red, workspace, workspace_bytes, s);
    case BGX_F64: return launch_tree<double, double>(*d, n_out, red, workspace, workspace_bytes, s);
    case BGX_BF16:
      return launch_tree<__nv_bfloat16, float>(*d, n_out, red, workspace, workspace_bytes, s);
    default: return launch_tree<__half, float>(*d, n_out, red, workspace, workspace_bytes, s);
  }
}
