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
constexpr int64_t TR_WARP_MAX = 8192;    // contiguous runs up to this: one warp per output

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
    const int ax_in = d.n_par + n_red - 1;
    if (!one_axis && d.extents[ax_in] >= TR_THREADS) {
      // innermost reduction axis at least a block wide: decode point r once,
      // then walk it with an odometer (one carry into the outer axes at most
      // per step) instead of a full mixed-radix decode per point
      const int64_t E = d.extents[ax_in];
      int64_t r = lo + threadIdx.x;
      if (r < hi) {
        int64_t idx[BGX_MAX_AXES];
        int64_t off[BGX_MAX_OPERANDS];
#pragma unroll
        for (int k = 0; k < BGX_MAX_OPERANDS; ++k)
          if (k < n_in) off[k] = base[k];
        int64_t rem = r;
        for (int a = n_red - 1; a >= 0; --a) {
          const int ax = d.n_par + a;
          idx[a] = rem % d.extents[ax];
          rem /= d.extents[ax];
#pragma unroll
          for (int k = 0; k < BGX_MAX_OPERANDS; ++k)
            if (k < n_in) off[k] += idx[a] * d.strides[k][ax];
        }
        auto step_odometer = [&]() {
          // advance by TR_THREADS points: inner axis, then at most one carry
          idx[n_red - 1] += TR_THREADS;
#pragma unroll
          for (int k = 0; k < BGX_MAX_OPERANDS; ++k)
            if (k < n_in) off[k] += (int64_t)TR_THREADS * d.strides[k][ax_in];
          if (idx[n_red - 1] >= E) {
            idx[n_red - 1] -= E;
#pragma unroll
            for (int k = 0; k < BGX_MAX_OPERANDS; ++k)
              if (k < n_in) off[k] -= E * d.strides[k][ax_in];
            for (int a = n_red - 2; a >= 0; --a) {
              const int ax = d.n_par + a;
#pragma unroll
              for (int k = 0; k < BGX_MAX_OPERANDS; ++k)
                if (k < n_in) off[k] += d.strides[k][ax];
              if (++idx[a] < d.extents[ax]) break;
#pragma unroll
              for (int k = 0; k < BGX_MAX_OPERANDS; ++k)
                if (k < n_in) off[k] -= d.extents[ax] * d.strides[k][ax];
              idx[a] = 0;
            }
          }
        };
        // the odometer position after each step; up to GU points gathered
        // and loaded together (independent loads in flight per thread)
        constexpr int GU = 4;
        while (r < hi) {
          int64_t offs[GU][BGX_MAX_OPERANDS];
          int nu = 0;
          for (; nu < GU && r < hi; ++nu, r += TR_THREADS) {
#pragma unroll
            for (int k = 0; k < BGX_MAX_OPERANDS; ++k)
              if (k < n_in) offs[nu][k] = off[k];
            step_odometer();
          }
          T pv[GU];
#pragma unroll
          for (int u = 0; u < GU; ++u) {
            if (u >= nu) break;
            T p = ld_t<S, T>(ins[0] + offs[u][0]);
#pragma unroll
            for (int k = 1; k < BGX_MAX_OPERANDS; ++k)
              if (k < n_in) p *= ld_t<S, T>(ins[k] + offs[u][k]);
            pv[u] = p;
          }
#pragma unroll
          for (int u = 0; u < GU; ++u)
            if (u < nu) acc += pv[u];
        }
      }
    } else
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

// CONTIG layout with short runs (a block per output would leave most of its
// threads idle): one WARP per output, 16-byte vectors per lane, shuffle sum.
template <typename S, typename T, int NIN>
__global__ void __launch_bounds__(TR_THREADS)
tree_contig_warp_kernel(const bgx_generic_desc d, int64_t n_out, int64_t red) {
  constexpr int V = Vec<S, T>::N;
  const S *const *ins = reinterpret_cast<const S *const *>(d.ins);
  const int lane = threadIdx.x % 32;
  const int64_t warps = (int64_t)gridDim.x * (TR_THREADS / 32);
  for (int64_t o = (int64_t)blockIdx.x * (TR_THREADS / 32) + threadIdx.x / 32; o < n_out;
       o += warps) {
    int64_t base[BGX_MAX_OPERANDS];
    par_offsets(d, o, NIN, base);
    const S *p[NIN];
    bool aligned = true;
#pragma unroll
    for (int k = 0; k < NIN; ++k) {
      p[k] = ins[k] + base[k];
      aligned = aligned && ((uintptr_t)p[k] % 16 == 0);
    }
    T acc = 0;
    int64_t done = 0;
    if (aligned) {
      const int64_t nv = red / V;
      for (int64_t i = lane; i < nv; i += 32) {
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
    for (int64_t i = done + lane; i < red; i += 32) {
      T q = ld_t<S, T>(p[0] + i);
#pragma unroll
      for (int k = 1; k < NIN; ++k) q *= ld_t<S, T>(p[k] + i);
      acc += q;
    }
#pragma unroll
    for (int sh = 16; sh > 0; sh >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, sh);
    if (lane == 0) {
      if (d.c0) acc += ld_t<S, T>(static_cast<const S *>(d.c0) + o);
      static_cast<S *>(d.out)[o] = st_t<S, T>(acc);
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
    // tile fastest: the blocks in flight read adjacent 128-byte segments of
    // the same rows (DRAM row locality), chunk by chunk
    const int64_t t = blk % n_tiles;
    const int s = (int)(blk / n_tiles);
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
    T acc = 0;
    constexpr int W = TR_THREADS / 32;
    // chunks s, s + splits, ...: the blocks in flight move down the rows
    // together (a narrow window of rows, i.e. of DRAM pages and TLB entries)
    for (int64_t cb = (int64_t)s * chunk; cb < red; cb += (int64_t)splits * chunk) {
    const int64_t lo = cb;
    const int64_t hi = lo + chunk < red ? lo + chunk : red;
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
    }   // chunks
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

// COLUMN layout, 16-bit storage, one reduction axis, even column count:
// each lane owns TWO adjacent columns (one 4-byte load per input per point),
// so a warp row is 64 columns = one 128-byte line, as for f32.  BCM: bit k
// set = input k is broadcast along the columns (stride 0, one scalar per
// point) — a template parameter, so the unrolled loads stay branch-free.
template <typename S, int NIN, int BCM>
__global__ void __launch_bounds__(TR_THREADS)
tree_column2_kernel(const bgx_generic_desc d, int64_t n_tiles, int64_t red, int splits,
                    int64_t chunk, float *ws) {
  __shared__ float part[TR_THREADS / 32][64];
  const int pl = d.n_par - 1;
  const int64_t E = d.extents[pl];
  const int64_t ctiles = (E + 63) / 64;
  const int w = threadIdx.x / 32, lane = threadIdx.x % 32;
  constexpr int W = TR_THREADS / 32;
  const S *const *ins = reinterpret_cast<const S *const *>(d.ins);
  for (int64_t blk = blockIdx.x; blk < n_tiles * splits; blk += gridDim.x) {
    const int64_t t = blk % n_tiles;
    const int s = (int)(blk / n_tiles);
    const int64_t q = t / ctiles, c = (t % ctiles) * 64 + 2 * lane;
    const bool live = c < E;                   // E even: c + 1 < E too
    const S *ptr[NIN];
    int64_t st[NIN];
#pragma unroll
    for (int k = 0; k < NIN; ++k) {
      int64_t off = ((BCM >> k) & 1) ? 0 : (live ? c : 0);
      int64_t rem = q;
      for (int a = pl - 1; a >= 0; --a) {
        const int64_t e = d.extents[a];
        off += (rem % e) * d.strides[k][a];
        rem /= e;
      }
      ptr[k] = ins[k] + off;
      st[k] = d.strides[k][d.n_par];
    }
    float a0 = 0.f, a1 = 0.f;
    for (int64_t cb = (int64_t)s * chunk; cb < red && live; cb += (int64_t)splits * chunk) {
      const int64_t hi = cb + chunk < red ? cb + chunk : red;
      constexpr int U = 8;
      int64_t r = cb + w;
      for (; r + (U - 1) * W < hi; r += U * W) {
        float x0[U], x1[U];
#pragma unroll
        for (int k = 0; k < NIN; ++k) {
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const S *pp = ptr[k] + (r + u * W) * st[k];
            float v0, v1;
            if ((BCM >> k) & 1) {   // folded after unrolling
              v0 = v1 = Conv<S>::to_f(*pp);
            } else {
              const uint32_t two = *reinterpret_cast<const uint32_t *>(pp);
              const S *e = reinterpret_cast<const S *>(&two);
              v0 = Conv<S>::to_f(e[0]);
              v1 = Conv<S>::to_f(e[1]);
            }
            if (k == 0) { x0[u] = v0; x1[u] = v1; } else { x0[u] *= v0; x1[u] *= v1; }
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) { a0 += x0[u]; a1 += x1[u]; }
      }
      for (; r < hi; r += W) {
        float x0 = 1.f, x1 = 1.f;
#pragma unroll
        for (int k = 0; k < NIN; ++k) {
          const S *pp = ptr[k] + r * st[k];
          float v0, v1;
          if ((BCM >> k) & 1) {   // folded after unrolling
            v0 = v1 = Conv<S>::to_f(*pp);
          } else {
            const uint32_t two = *reinterpret_cast<const uint32_t *>(pp);
            const S *e = reinterpret_cast<const S *>(&two);
            v0 = Conv<S>::to_f(e[0]);
            v1 = Conv<S>::to_f(e[1]);
          }
          if (k == 0) { x0 = v0; x1 = v1; } else { x0 *= v0; x1 *= v1; }
        }
        a0 += x0;
        a1 += x1;
      }
    }
    part[w][2 * lane] = a0;
    part[w][2 * lane + 1] = a1;
    __syncthreads();
    if (w < 2) {
      const int col = w * 32 + lane;           // 64 columns over two warps
      const int64_t cc = (t % ctiles) * 64 + col;
      if (cc < E) {
        float sum = 0.f;
#pragma unroll
        for (int j = 0; j < W; ++j) sum += part[j][col];
        const int64_t o = q * E + cc;
        if (splits == 1) {
          if (d.c0) sum += Conv<S>::to_f(static_cast<const S *>(d.c0)[o]);
          static_cast<S *>(d.out)[o] = Conv<S>::from_f(sum);
        } else {
          ws[o * splits + s] = sum;
        }
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

enum class TreeLayout { General, Contig, Column, Column2 };

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
    if (ok && col) {
      // 16-bit, one reduction axis, every unit-stride input 4-byte aligned
      // at even columns: two columns per lane
      bool two = dtype_size(d.dtype) == 2 && d.n_axes - d.n_par == 1 && d.n_in <= 2 &&
                 d.extents[pl] % 2 == 0;
      for (int k = 0; k < d.n_in && two; ++k) {
        if (d.strides[k][pl] == 0) continue;
        two = ((uintptr_t)d.ins[k] % 4 == 0);
        for (int a = 0; a < d.n_axes && two; ++a)
          if (a != pl && d.extents[a] != 1) two = d.strides[k][a] % 2 == 0;
      }
      return two ? TreeLayout::Column2 : TreeLayout::Column;
    }
  }
  return TreeLayout::General;
}

// Independent units the layout's kernel distributes (outputs, or 32-wide
// column tiles), and the chunk count per unit: enough blocks to fill the
// GPU (8 per SM), each chunk at least TR_MIN_CHUNK points.
int64_t tree_units(const bgx_generic_desc &d, TreeLayout lay, int64_t n_out) {
  if (lay != TreeLayout::Column && lay != TreeLayout::Column2) return n_out;
  const int64_t E = d.extents[d.n_par - 1];
  const int64_t cw = lay == TreeLayout::Column2 ? 64 : 32;
  return (n_out / E) * ((E + cw - 1) / cw);
}

int tree_splits(int64_t units, int64_t red, TreeLayout lay) {
  const int sms = sm_count_current();
  const int64_t target = (int64_t)(sms > 0 ? sms : 148) * 8;   // 8 blocks of 256 per SM
  int64_t sp = (target + units - 1) / units;
  const int64_t min_chunk =
      (lay == TreeLayout::Column || lay == TreeLayout::Column2) ? 256 : TR_MIN_CHUNK;
  const int64_t by_size = (red + min_chunk - 1) / min_chunk;
  if (sp > by_size) sp = by_size;
  if (sp > 65536) sp = 65536;
  return sp < 1 ? 1 : (int)sp;
}

template <typename S, typename T>
int launch_tree(const bgx_generic_desc &d0, int64_t n_out, int64_t red, void *ws,
                int64_t ws_bytes, cudaStream_t s) {
  const bgx_generic_desc d = coalesce_axes(d0);   // same merge as the workspace plan
  TreeLayout lay = tree_layout(d);
  if (d.n_in > 3 && lay != TreeLayout::General) lay = TreeLayout::General;
  const int64_t units = tree_units(d, lay, n_out);
  const int splits = tree_splits(units, red, lay);
  int64_t chunk = (red + splits - 1) / splits;
  if (lay == TreeLayout::Contig) chunk = (chunk + 63) / 64 * 64;   // keeps 16-byte vector runs aligned
  // column layouts: `splits` partial sums per output, each over the
  // interleaved 256-row chunks s, s + splits, ...
  if (lay == TreeLayout::Column || lay == TreeLayout::Column2) chunk = 256;
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
  if (lay == TreeLayout::Contig && splits == 1 && red <= TR_WARP_MAX) {
    int64_t wb = (n_out + TR_THREADS / 32 - 1) / (TR_THREADS / 32);
    if (wb > cap) wb = cap;
    switch (d.n_in) {
      case 1: tree_contig_warp_kernel<S, T, 1><<<(unsigned)wb, TR_THREADS, 0, s>>>(d, n_out, red); break;
      case 2: tree_contig_warp_kernel<S, T, 2><<<(unsigned)wb, TR_THREADS, 0, s>>>(d, n_out, red); break;
      default: tree_contig_warp_kernel<S, T, 3><<<(unsigned)wb, TR_THREADS, 0, s>>>(d, n_out, red); break;
    }
    return check_launch("tree_contig_warp_kernel");
  }
  if (lay == TreeLayout::Contig) {
    BGX_TREE_LAUNCH(tree_contig_kernel, n_out)
  } else if (lay == TreeLayout::Column2) {
    if constexpr (sizeof(S) == 2) {
      float *wf = reinterpret_cast<float *>(w);
      const int pl = d.n_par - 1;
      const int bcm = (d.strides[0][pl] == 0 ? 1 : 0) | (d.n_in > 1 && d.strides[1][pl] == 0 ? 2 : 0);
      if (d.n_in == 1)
        tree_column2_kernel<S, 1, 0><<<g, TR_THREADS, 0, s>>>(d, units, red, splits, chunk, wf);
      else if (bcm == 1)
        tree_column2_kernel<S, 2, 1><<<g, TR_THREADS, 0, s>>>(d, units, red, splits, chunk, wf);
      else if (bcm == 2)
        tree_column2_kernel<S, 2, 2><<<g, TR_THREADS, 0, s>>>(d, units, red, splits, chunk, wf);
      else
        tree_column2_kernel<S, 2, 0><<<g, TR_THREADS, 0, s>>>(d, units, red, splits, chunk, wf);
    }
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
  const bgx_generic_desc c = coalesce_axes(*d);
  TreeLayout lay = tree_layout(c);
  if (c.n_in > 3 && lay != TreeLayout::General) lay = TreeLayout::General;
  const int splits =
      (n_out > 0 && red > 0) ? tree_splits(tree_units(c, lay, n_out), red, lay) : 1;
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
