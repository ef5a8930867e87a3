/*
 * Plain-C consumer of libbgx.so through include/bgx.h only (no torch, no
 * Python): what a non-Python host of the einsum path (e.g. a C/C++ runtime
 * next to bridgegen) links against.  Runs three entry points on device
 * buffers it allocates itself and checks them on the CPU:
 *   1. bgx_contract   (i,k),(k,j)->(i,j) f32, mode EXACT: bit-identical to
 *                     the reference's per-point order (acc = fl(fl(a*b) + acc),
 *                     k increasing, interp.py:398-416);
 *   2. bgx_permute    (i,j)->(j,i) f32: bytes moved unchanged;
 *   3. bgx_generic    (i,j)->(i) f32 row sums, reference order.
 * Build: gcc -O2 -I include examples/c_abi_demo.c -L paper_2503_04771_b200 -lbgx \
 *            -L /usr/local/cuda/lib64 -lcudart -Wl,-rpath,paper_2503_04771_b200 -o c_abi_demo
 * (tests/test_c_abi_demo.py compiles it on CPU and runs it on the B200.)
 */
#include <cuda_runtime_api.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include "bgx.h"

#define CHECK(x)                                                               \
  do {                                                                         \
    int rc_ = (x);                                                             \
    if (rc_ != 0) {                                                            \
      fprintf(stderr, "%s failed (%d): %s\n", #x, rc_, bgx_last_error());     \
      return 1;                                                                \
    }                                                                          \
  } while (0)

static float lcg(uint32_t *s) {
  *s = *s * 1664525u + 1013904223u;
  return (float)((*s >> 8) & 0xffff) / 32768.0f - 1.0f;
}

int main(void) {
  enum { M = 96, N = 80, K = 64 };
  static float a[M * K], b[K * N], c[M * N], want[M * N], t[N * M], rs[M];
  uint32_t seed = 7;
  for (int i = 0; i < M * K; ++i) a[i] = lcg(&seed);
  for (int i = 0; i < K * N; ++i) b[i] = lcg(&seed);
  /* reference arithmetic, volatile so the compiler keeps mul and add separate */
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < N; ++j) {
      volatile float acc = 0.0f;
      for (int k = 0; k < K; ++k) {
        volatile float p = a[i * K + k] * b[k * N + j];
        acc = p + acc;
      }
      want[i * N + j] = acc;
    }
  float *da, *db, *dc, *dt, *drs;
  if (cudaMalloc((void **)&da, sizeof a) || cudaMalloc((void **)&db, sizeof b) ||
      cudaMalloc((void **)&dc, sizeof c) || cudaMalloc((void **)&dt, sizeof t) ||
      cudaMalloc((void **)&drs, sizeof rs)) {
    fprintf(stderr, "cudaMalloc failed\n");
    return 1;
  }
  cudaMemcpy(da, a, sizeof a, cudaMemcpyHostToDevice);
  cudaMemcpy(db, b, sizeof b, cudaMemcpyHostToDevice);

  /* 1. GEMM through the contraction descriptor */
  bgx_contract_desc d;
  memset(&d, 0, sizeof d);
  d.batch = 1; d.M = M; d.N = N; d.K = K;
  d.a = da; d.a_stride[1] = K; d.a_stride[2] = 1;
  d.b = db; d.b_stride[1] = N; d.b_stride[2] = 1;
  d.out = dc; d.o_stride[1] = N; d.o_stride[2] = 1;
  d.in_dtype = d.out_dtype = BGX_F32;
  d.mode = BGX_MODE_EXACT;
  CHECK(bgx_contract(&d, NULL));
  cudaMemcpy(c, dc, sizeof c, cudaMemcpyDeviceToHost);
  if (memcmp(c, want, sizeof c) != 0) {
    fprintf(stderr, "contract: not bit-identical to the reference order\n");
    return 1;
  }

  /* 2. transpose of the result */
  bgx_tensor tin, tout;
  memset(&tin, 0, sizeof tin);
  memset(&tout, 0, sizeof tout);
  tin.data = dc; tin.dtype = BGX_F32; tin.rank = 2;
  tin.shape[0] = M; tin.shape[1] = N; tin.stride[0] = N; tin.stride[1] = 1;
  tout.data = dt; tout.dtype = BGX_F32; tout.rank = 2;
  tout.shape[0] = N; tout.shape[1] = M; tout.stride[0] = M; tout.stride[1] = 1;
  const int32_t perm[2] = {1, 0};
  CHECK(bgx_permute(&tin, &tout, perm, NULL));
  cudaMemcpy(t, dt, sizeof t, cudaMemcpyDeviceToHost);
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < N; ++j)
      if (memcmp(&t[j * M + i], &c[i * N + j], sizeof(float)) != 0) {
        fprintf(stderr, "permute: element (%d,%d) differs\n", i, j);
        return 1;
      }

  /* 3. row sums with the generic loop nest (axes: i parallel, j reduced) */
  bgx_generic_desc g;
  memset(&g, 0, sizeof g);
  g.n_in = 1; g.n_axes = 2; g.n_par = 1; g.dtype = BGX_F32;
  g.extents[0] = M; g.extents[1] = N;
  g.ins[0] = dc; g.strides[0][0] = N; g.strides[0][1] = 1;
  g.c0 = NULL; g.out = drs;
  CHECK(bgx_generic(&g, NULL));
  cudaMemcpy(rs, drs, sizeof rs, cudaMemcpyDeviceToHost);
  for (int i = 0; i < M; ++i) {
    volatile float acc = 0.0f;
    for (int j = 0; j < N; ++j) acc = c[i * N + j] + acc;
    if (memcmp(&rs[i], (const void *)&acc, sizeof(float)) != 0) {
      fprintf(stderr, "generic: row %d differs\n", i);
      return 1;
    }
  }
  cudaFree(da); cudaFree(db); cudaFree(dc); cudaFree(dt); cudaFree(drs);
  CHECK(bgx_shutdown());
  printf("c_abi_demo ok: bgx_version %d, %d SMs\n", bgx_version(), bgx_sm_count());
  return 0;
}
