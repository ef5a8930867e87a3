// bgx_permute — pure permutation / copy contractions (passthrough body,
// bridgegen einsum.py:105-108), bit-exact: bytes are moved, never converted.
//
// Host side canonicalises the (in, out, perm) triple: drops extent-1 dims and
// merges output dims whose input and output strides compose, so e.g.
// (i,j,k)->(i,j,k) becomes one contiguous run and (i,j,k)->(k,j,i) keeps three
// dims.  Then one of two HBM-bound kernels runs:
//   * row copy   — the output's unit-stride dim is also the input's: each
//                  block streams rows with 16-byte vector accesses when aligned;
//   * tiled transpose — the two unit-stride dims differ: a TILE x TILE tile is
//                  read coalesced along the input's inner dim into padded
//                  shared memory and written coalesced along the output's
//                  inner dim; the remaining dims fold into the grid.
// Roofline: 2 * numel * elem_size bytes of HBM traffic per call.
#include "common.cuh"

#include <algorithm>
#include <vector>

namespace bgx {
namespace {

constexpr int kMaxBatchDims = BGX_MAX_RANK;

struct BatchDims {
  int n;
  int64_t extent[kMaxBatchDims];
  int64_t in_stride[kMaxBatchDims];
  int64_t out_stride[kMaxBatchDims];
};

__device__ __forceinline__ void decode_batch(const BatchDims &bd, int64_t idx, int64_t &in_off,
                                             int64_t &out_off) {
  in_off = 0;
  out_off = 0;
  for (int d = bd.n - 1; d >= 0; --d) {
    int64_t e = bd.extent[d];
    int64_t i = idx % e;
    idx /= e;
    in_off += i * bd.in_stride[d];
    out_off += i * bd.out_stride[d];
  }
}

// ---- tiled transpose --------------------------------------------------------
// X = input's inner dim (stride sx_in, usually 1), Y = output's inner dim.
// Tile of TILE (x) by TILE (y); block = (32, 8) threads.
constexpr int TILE = 64;
constexpr int BLK_Y = 8;

template <typename T>
__global__ void __launch_bounds__(32 * BLK_Y)
transpose_kernel(const T *__restrict__ in, T *__restrict__ out, int64_t nx, int64_t ny,
                 int64_t in_sx, int64_t in_sy, int64_t out_sx, int64_t out_sy,
                 int64_t tiles_x, int64_t tiles_y, BatchDims bd) {
  __shared__ T tile[TILE][TILE + 1];
  int64_t t = blockIdx.x;
  const int64_t tx = t % tiles_x;
  t /= tiles_x;
  const int64_t ty = t % tiles_y;
  t /= tiles_y;
  int64_t in_off, out_off;
  decode_batch(bd, t, in_off, out_off);
  const int64_t x0 = tx * TILE, y0 = ty * TILE;
  // read: threadIdx.x runs along X (coalesced in the input)
#pragma unroll
  for (int j = 0; j < TILE / BLK_Y; ++j) {
    const int ly = threadIdx.y + j * BLK_Y;
    const int64_t y = y0 + ly;
#pragma unroll
    for (int i = 0; i < TILE / 32; ++i) {
      const int lx = threadIdx.x + i * 32;
      const int64_t x = x0 + lx;
      if (x < nx && y < ny) tile[ly][lx] = in[in_off + x * in_sx + y * in_sy];
    }
  }
  __syncthreads();
  // write: threadIdx.x runs along Y (coalesced in the output)
#pragma unroll
  for (int j = 0; j < TILE / BLK_Y; ++j) {
    const int lx = threadIdx.y + j * BLK_Y;
    const int64_t x = x0 + lx;
#pragma unroll
    for (int i = 0; i < TILE / 32; ++i) {
      const int ly = threadIdx.x + i * 32;
      const int64_t y = y0 + ly;
      if (x < nx && y < ny) out[out_off + x * out_sx + y * out_sy] = tile[ly][lx];
    }
  }
}

// ---- vectorised transpose (fast path) ------------------------------------
// Both unit-stride dims (input's X, output's Y) are contiguous and every other
// stride is a multiple of the 16-byte vector: threads move 16-byte vectors on
// both sides, the tile is staged in padded shared memory, the grid is 3-D
// (x tile, y tile, batch) so no per-element division is needed.  Extents of X
// and Y are multiples of VEC, so vectors never straddle an edge.
template <typename T>
__global__ void __launch_bounds__(256)
transpose_vec_kernel(const T *__restrict__ in, T *__restrict__ out, int64_t nx, int64_t ny,
                     int64_t in_sy, int64_t out_sx, BatchDims bd) {
  constexpr int VEC = 16 / sizeof(T);
  constexpr int TPR = TILE / VEC;          // threads per tile row (vectors per row)
  constexpr int RPP = 256 / TPR;           // rows per pass
  __shared__ T tile[TILE][TILE + 1];
  int64_t in_off, out_off;
  decode_batch(bd, blockIdx.z, in_off, out_off);
  const int64_t x0 = (int64_t)blockIdx.x * TILE, y0 = (int64_t)blockIdx.y * TILE;
  const int tv = threadIdx.x % TPR, tr = threadIdx.x / TPR;
  // read: rows of the input (fixed y), 16-byte vectors along x
  const T *src = in + in_off + x0 + (int64_t)tv * VEC;
#pragma unroll
  for (int r = tr; r < TILE; r += RPP) {
    const int64_t y = y0 + r;
    if (y < ny && x0 + tv * VEC < nx) {
      uint4 v = __ldcs(reinterpret_cast<const uint4 *>(src + y * in_sy));
      const T *e = reinterpret_cast<const T *>(&v);
#pragma unroll
      for (int q = 0; q < VEC; ++q) tile[r][tv * VEC + q] = e[q];
    }
  }
  __syncthreads();
  // write: rows of the output (fixed x), 16-byte vectors along y
  T *dst = out + out_off + y0 + (int64_t)tv * VEC;
#pragma unroll
  for (int c = tr; c < TILE; c += RPP) {
    const int64_t x = x0 + c;
    if (x < nx && y0 + tv * VEC < ny) {
      uint4 v;
      T *e = reinterpret_cast<T *>(&v);
#pragma unroll
      for (int q = 0; q < VEC; ++q) e[q] = tile[tv * VEC + q][c];
      __stcs(reinterpret_cast<uint4 *>(dst + x * out_sx), v);
    }
  }
}

// ---- row copy ---------------------------------------------------------------
// Rows of length n along a dim that is inner in both tensors.  Long rows are
// cut into `nchunk` pieces of `chunk` elements, one per block, so a single
// contiguous run (an identity permutation, or any copy whose dims all merge)
// still spreads over every SM.
template <typename T>
__global__ void __launch_bounds__(256)
copy_rows_kernel(const T *__restrict__ in, T *__restrict__ out, int64_t n, int64_t in_s,
                 int64_t out_s, int64_t rows, int64_t chunk, int64_t nchunk, BatchDims bd) {
  for (int64_t blk = blockIdx.x; blk < rows * nchunk; blk += gridDim.x) {
    const int64_t r = blk / nchunk, c0 = (blk % nchunk) * chunk;
    const int64_t c1 = c0 + chunk < n ? c0 + chunk : n;
    int64_t in_off, out_off;
    decode_batch(bd, r, in_off, out_off);
    for (int64_t x = c0 + threadIdx.x; x < c1; x += blockDim.x)
      out[out_off + x * out_s] = in[in_off + x * in_s];
  }
}

// Contiguous rows, 16-byte vectors (rows and bases 16B aligned).
__global__ void __launch_bounds__(256)
copy_rows_vec_kernel(const uint4 *__restrict__ in, uint4 *__restrict__ out, int64_t nvec,
                     int64_t rows, int64_t chunk, int64_t nchunk, BatchDims bd) {
  for (int64_t blk = blockIdx.x; blk < rows * nchunk; blk += gridDim.x) {
    const int64_t r = blk / nchunk, c0 = (blk % nchunk) * chunk;
    const int64_t c1 = c0 + chunk < nvec ? c0 + chunk : nvec;
    int64_t in_off, out_off;
    decode_batch(bd, r, in_off, out_off);  // in uint4 units (host pre-divides)
    const uint4 *src = in + in_off;
    uint4 *dst = out + out_off;
    int64_t x = c0 + threadIdx.x;
    constexpr int U = 8;   // 8 independent 16-byte loads in flight per thread
    for (; x + (U - 1) * 256 < c1; x += U * 256) {
      uint4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = __ldcs(src + x + u * 256);
#pragma unroll
      for (int u = 0; u < U; ++u) __stcs(dst + x + u * 256, v[u]);
    }
    for (; x < c1; x += 256) __stcs(dst + x, __ldcs(src + x));
  }
}

// Contiguous rows SHORTER than a block's worth of vectors (a permutation
// that keeps a short inner dim in place, e.g. (c,a,b)->(a,c,b) with b = 64):
// the flat (row, vector) index space is spread over all threads, 32-bit
// index arithmetic.
__global__ void __launch_bounds__(256)
copy_short_rows_vec_kernel(const uint4 *__restrict__ in, uint4 *__restrict__ out, uint32_t nvec,
                           uint32_t total, BatchDims bd) {
  for (uint32_t g = blockIdx.x * 256u + threadIdx.x; g < total; g += gridDim.x * 256u) {
    uint32_t r = g / nvec;
    const uint32_t x = g - r * nvec;
    int64_t in_off = x, out_off = x;
    for (int d = bd.n - 1; d >= 0; --d) {
      const uint32_t e = (uint32_t)bd.extent[d];
      const uint32_t q = r / e, i = r - q * e;
      r = q;
      in_off += (int64_t)i * bd.in_stride[d];
      out_off += (int64_t)i * bd.out_stride[d];
    }
    __stcs(out + out_off, __ldcs(in + in_off));
  }
}

struct Dim {
  int64_t extent, in_stride, out_stride;
};

template <typename T>
int launch_permute(const void *in, void *out, std::vector<Dim> dims, cudaStream_t s) {
  const int sms = sm_count_current();
  if (sms <= 0) { set_error("bgx_permute: no device"); return BGX_ERR_NO_DEVICE; }
  // output-inner dim = last; input-inner dim = smallest input stride
  int yi = (int)dims.size() - 1;
  int xi = 0;
  for (int d = 0; d < (int)dims.size(); ++d)
    if (dims[d].in_stride < dims[xi].in_stride) xi = d;
  BatchDims bd{};
  if (xi == yi || dims[yi].in_stride == 1 || dims[xi].in_stride == dims[yi].in_stride) {
    // row copy along the output's inner dim
    const Dim row = dims[yi];
    int64_t rows = 1;
    for (int d = 0; d < yi; ++d) {
      bd.extent[bd.n] = dims[d].extent;
      bd.in_stride[bd.n] = dims[d].in_stride;
      bd.out_stride[bd.n] = dims[d].out_stride;
      ++bd.n;
      rows *= dims[d].extent;
    }
    const int64_t vec = 16 / (int64_t)sizeof(T);
    bool vec_ok = row.in_stride == 1 && row.out_stride == 1 && row.extent % vec == 0 &&
                  ((uintptr_t)in % 16 == 0) && ((uintptr_t)out % 16 == 0);
    for (int d = 0; d < bd.n && vec_ok; ++d)
      vec_ok = bd.in_stride[d] % vec == 0 && bd.out_stride[d] % vec == 0;
    // rows cut into 2048-element (vector) pieces handed out grid-stride, so
    // the blocks in flight stream one contiguous window of memory
    const int64_t len = vec_ok ? row.extent / vec : row.extent;
    const int64_t chunk = len < 2048 ? (len > 0 ? len : 1) : 2048;
    const int64_t nchunk = (len + chunk - 1) / chunk;
    int64_t grid = std::min<int64_t>(rows * nchunk, (int64_t)sms * 32);
    if (vec_ok) {
      for (int d = 0; d < bd.n; ++d) {
        bd.in_stride[d] /= vec;
        bd.out_stride[d] /= vec;
      }
      bool small32 = len < 256 && rows * len < 0x7fffffffLL;
      for (int d = 0; d < bd.n && small32; ++d) small32 = bd.extent[d] < 0x7fffffffLL;
      if (small32) {
        const int64_t total = rows * len;
        const int64_t g2 = std::min<int64_t>((total + 255) / 256, (int64_t)sms * 32);
        copy_short_rows_vec_kernel<<<(unsigned)g2, 256, 0, s>>>(
            (const uint4 *)in, (uint4 *)out, (uint32_t)len, (uint32_t)total, bd);
        return check_launch("permute copy (short rows)");
      }
      copy_rows_vec_kernel<<<(unsigned)grid, 256, 0, s>>>((const uint4 *)in, (uint4 *)out,
                                                         len, rows, chunk, nchunk, bd);
    } else {
      copy_rows_kernel<T><<<(unsigned)grid, 256, 0, s>>>((const T *)in, (T *)out, row.extent,
                                                         row.in_stride, row.out_stride, rows,
                                                         chunk, nchunk, bd);
    }
    return check_launch("permute copy");
  }
  const Dim X = dims[xi], Y = dims[yi];
  int64_t batch = 1;
  for (int d = 0; d < (int)dims.size(); ++d) {
    if (d == xi || d == yi) continue;
    bd.extent[bd.n] = dims[d].extent;
    bd.in_stride[bd.n] = dims[d].in_stride;
    bd.out_stride[bd.n] = dims[d].out_stride;
    ++bd.n;
    batch *= dims[d].extent;
  }
  const int64_t tiles_x = (X.extent + TILE - 1) / TILE;
  const int64_t tiles_y = (Y.extent + TILE - 1) / TILE;
  const int64_t blocks = tiles_x * tiles_y * batch;
  {
    constexpr int64_t VEC = 16 / (int64_t)sizeof(T);
    bool fast = X.in_stride == 1 && Y.out_stride == 1 && X.extent % VEC == 0 &&
                Y.extent % VEC == 0 && Y.in_stride % VEC == 0 && X.out_stride % VEC == 0 &&
                ((uintptr_t)in % 16 == 0) && ((uintptr_t)out % 16 == 0) &&
                tiles_x < 0x7fffffffLL && tiles_y < 65536 && batch < 65536;
    for (int d = 0; d < bd.n && fast; ++d)
      fast = bd.in_stride[d] % VEC == 0 && bd.out_stride[d] % VEC == 0;
    if (fast) {
      dim3 grid((unsigned)tiles_x, (unsigned)tiles_y, (unsigned)batch);
      transpose_vec_kernel<T><<<grid, 256, 0, s>>>((const T *)in, (T *)out, X.extent, Y.extent,
                                                    Y.in_stride, X.out_stride, bd);
      return check_launch("permute transpose (vec)");
    }
  }
  if (blocks > 0x7fffffffLL) { set_error("bgx_permute: too many tiles"); return BGX_ERR_UNSUPPORTED; }
  dim3 block(32, BLK_Y);
  transpose_kernel<T><<<(unsigned)blocks, block, 0, s>>>(
      (const T *)in, (T *)out, X.extent, Y.extent, X.in_stride, Y.in_stride, X.out_stride,
      Y.out_stride, tiles_x, tiles_y, bd);
  return check_launch("permute transpose");
}

}  // namespace
}  // namespace bgx

using namespace bgx;

extern "C" int bgx_permute(const bgx_tensor *in, const bgx_tensor *out, const int32_t *perm,
                           void *stream) {
  BGX_CHECK_ARG(in && out && (perm || in->rank == 0), "bgx_permute: null argument");
  BGX_CHECK_ARG(in->rank == out->rank, "bgx_permute: rank mismatch %d vs %d", in->rank,
                out->rank);
  BGX_CHECK_ARG(in->rank >= 0 && in->rank <= BGX_MAX_RANK, "bgx_permute: rank %d", in->rank);
  BGX_CHECK_ARG(in->dtype == out->dtype, "bgx_permute: dtype mismatch");
  const int esz = dtype_size(in->dtype);
  BGX_CHECK_ARG(esz > 0, "bgx_permute: bad dtype %d", in->dtype);
  const int r = in->rank;
  bool seen[BGX_MAX_RANK] = {false};
  int64_t numel = 1;
  for (int d = 0; d < r; ++d) {
    BGX_CHECK_ARG(perm[d] >= 0 && perm[d] < r && !seen[perm[d]], "bgx_permute: bad perm");
    seen[perm[d]] = true;
    BGX_CHECK_ARG(out->shape[d] == in->shape[perm[d]],
                  "bgx_permute: out dim %d extent %lld != in dim %d extent %lld", d,
                  (long long)out->shape[d], perm[d], (long long)in->shape[perm[d]]);
    BGX_CHECK_ARG(out->shape[d] >= 0 && in->stride[perm[d]] >= 0 && out->stride[d] >= 0,
                  "bgx_permute: negative extent/stride");
    numel *= out->shape[d];
  }
  if (numel == 0) return BGX_OK;
  BGX_CHECK_ARG(in->data && out->data, "bgx_permute: null data");
  // canonicalise: output-ordered dims, drop extent 1, merge composable pairs
  std::vector<Dim> dims;
  for (int d = 0; d < r; ++d) {
    if (out->shape[d] == 1) continue;
    Dim cur{out->shape[d], in->stride[perm[d]], out->stride[d]};
    if (!dims.empty()) {
      Dim &p = dims.back();
      if (p.in_stride == cur.in_stride * cur.extent && p.out_stride == cur.out_stride * cur.extent) {
        p.extent *= cur.extent;
        p.in_stride = cur.in_stride;
        p.out_stride = cur.out_stride;
        continue;
      }
    }
    dims.push_back(cur);
  }
  if (dims.empty()) dims.push_back(Dim{1, 1, 1});
  cudaStream_t s = (cudaStream_t)stream;
  switch (esz) {
    case 1: return launch_permute<uint8_t>(in->data, out->data, dims, s);
    case 2: return launch_permute<uint16_t>(in->data, out->data, dims, s);
    case 4: return launch_permute<uint32_t>(in->data, out->data, dims, s);
    default: return launch_permute<uint64_t>(in->data, out->data, dims, s);
  }
}
