// Host-only probe compiled by tests/test_abi.py (nvcc, no GPU needed):
// prints the C layout of the include/bgx.h structs and sample UMMA
// descriptor encodings so the Python side can check them.
#include <cstddef>
#include <cstdio>
#include "../paper_2503_04771_b200/csrc/common.cuh"

int main() {
  printf("bgx_tensor %zu %zu %zu\n", sizeof(bgx_tensor), offsetof(bgx_tensor, shape),
         offsetof(bgx_tensor, stride));
  printf("bgx_generic_desc %zu %zu %zu %zu\n", sizeof(bgx_generic_desc),
         offsetof(bgx_generic_desc, ins), offsetof(bgx_generic_desc, c0),
         offsetof(bgx_generic_desc, out));
  printf("bgx_contract_desc %zu %zu %zu %zu\n", sizeof(bgx_contract_desc),
         offsetof(bgx_contract_desc, c0), offsetof(bgx_contract_desc, in_dtype),
         offsetof(bgx_contract_desc, sched));
  printf("bgx_rs_plan %zu %zu %zu\n", sizeof(bgx_rs_plan), offsetof(bgx_rs_plan, rows_per_owner),
         offsetof(bgx_rs_plan, ws_bytes));
  printf("bgx_reduce_scatter %zu %zu %zu %zu %zu\n", sizeof(bgx_reduce_scatter),
         offsetof(bgx_reduce_scatter, slots), offsetof(bgx_reduce_scatter, out),
         offsetof(bgx_reduce_scatter, ws), offsetof(bgx_reduce_scatter, ws_counters));
  printf("sdesc %llu %llu\n", (unsigned long long)bgx::make_sdesc_sw128(0x12400, 16, 1024),
         (unsigned long long)bgx::make_sdesc_sw128(0x3f800, 8192, 1024));
  printf("idesc %u %u %u\n", bgx::make_idesc_f16(true, false, true, 128, 256),
         bgx::make_idesc_f16(false, true, false, 128, 64),
         bgx::make_idesc_f16(true, true, true, 256, 128));
  return 0;
}
