// Stand-alone probe: is the 64x64-tile transpose (bgx permute.cu) limited by
// the transpose access pattern or by its one-tile-per-block structure?
// Times, on 8192^2 f32 (256 MiB each way): the tile transpose, the same
// tiling as a plain copy, a grid-stride float4 copy, and cudaMemcpy D2D.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a tile_probe.cu -o tile_probe
#include <cstdio>
#include <cuda_runtime.h>

constexpr int TILE = 64;

template <bool TRANSPOSE>
__global__ void __launch_bounds__(256) tile_kernel(const float *__restrict__ in, float *__restrict__ out,
                                                   int n) {
  __shared__ float tile[TILE][TILE + 1];
  const int x0 = blockIdx.x * TILE, y0 = blockIdx.y * TILE;
  const int tv = threadIdx.x % 16, tr = threadIdx.x / 16;
  for (int r = tr; r < TILE; r += 16) {
    float4 v = __ldcs(reinterpret_cast<const float4 *>(in + (size_t)(y0 + r) * n + x0 + tv * 4));
    tile[r][tv * 4] = v.x; tile[r][tv * 4 + 1] = v.y; tile[r][tv * 4 + 2] = v.z; tile[r][tv * 4 + 3] = v.w;
  }
  __syncthreads();
  for (int c = tr; c < TILE; c += 16) {
    float4 v;
    if (TRANSPOSE) {
      v.x = tile[tv * 4][c]; v.y = tile[tv * 4 + 1][c]; v.z = tile[tv * 4 + 2][c]; v.w = tile[tv * 4 + 3][c];
      __stcs(reinterpret_cast<float4 *>(out + (size_t)(x0 + c) * n + y0 + tv * 4), v);
    } else {
      v.x = tile[c][tv * 4]; v.y = tile[c][tv * 4 + 1]; v.z = tile[c][tv * 4 + 2]; v.w = tile[c][tv * 4 + 3];
      __stcs(reinterpret_cast<float4 *>(out + (size_t)(y0 + c) * n + x0 + tv * 4), v);
    }
  }
}

__global__ void copy4(const float4 *__restrict__ in, float4 *__restrict__ out, size_t n4) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x)
    __stcs(out + i, __ldcs(in + i));
}

template <typename F> float timeit(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) f();
  float best = 1e9;
  for (int rep = 0; rep < 20; ++rep) {
    cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  const int n = 8192;
  const size_t bytes = (size_t)n * n * 4;
  float *in, *out;
  cudaMalloc(&in, bytes); cudaMalloc(&out, bytes);
  cudaMemset(in, 1, bytes);
  dim3 grid(n / TILE, n / TILE);
  auto rep = [&](const char *name, float ms) {
    printf("%-28s %8.1f us  %7.1f GB/s\n", name, ms * 1e3, 2.0 * bytes / (ms * 1e-3) / 1e9);
  };
  rep("tile transpose 64x64", timeit([&] { tile_kernel<true><<<grid, 256>>>(in, out, n); }));
  rep("tile copy 64x64", timeit([&] { tile_kernel<false><<<grid, 256>>>(in, out, n); }));
  rep("grid-stride float4 copy", timeit([&] { copy4<<<148 * 8, 256>>>((const float4 *)in, (float4 *)out, bytes / 16); }));
  rep("cudaMemcpy D2D", timeit([&] { cudaMemcpyAsync(out, in, bytes, cudaMemcpyDeviceToDevice); }));
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
