// bgx_contract — kernel selection for two-input contractions (see bgx.h).
#include "common.cuh"

namespace bgx {
bool tc_legal(const bgx_contract_desc &d, const char **why);
int contract_tc(const bgx_contract_desc &d, cudaStream_t s);
int contract_simt(const bgx_contract_desc &d, int kind, cudaStream_t s);
void tc_tile_choice(const bgx_contract_desc &d, int *cg_out, int *bn_out);
void tc_splitk_plan(const bgx_contract_desc &d, int *splits, int64_t *ws_bytes);
int contract_tc_splitk(const bgx_contract_desc &d, int splits, void *ws, int64_t ws_bytes,
                       cudaStream_t s);
int tc_rs_plan(const bgx_contract_desc &d, int world, bgx_rs_plan *pl);
int contract_tc_rs(const bgx_contract_desc &d, const bgx_reduce_scatter &rs, cudaStream_t s);
int rs_reduce(const bgx_contract_desc &d, const bgx_reduce_scatter &rs, cudaStream_t s);

namespace {

enum { KIND_TC = 1, KIND_EXACT = 2, KIND_FFMA = 3, KIND_SIMT16 = 4 };

int select_kind(const bgx_contract_desc &d) {
  const bool half_in = d.in_dtype == BGX_BF16 || d.in_dtype == BGX_F16;
  switch (d.mode) {
    case BGX_MODE_AUTO:
      if (half_in) return tc_legal(d, nullptr) ? KIND_TC : KIND_SIMT16;
      return KIND_EXACT;
    case BGX_MODE_EXACT:
      if (half_in) return KIND_SIMT16;  // exact products in f32 (see gemm_simt.cu)
      return KIND_EXACT;
    case BGX_MODE_FFMA:
      // tolerance mode: fused multiply-add for f32 and f64; 16-bit inputs
      // take the auto path (tensor cores when legal: products exact in f32)
      if (half_in) return tc_legal(d, nullptr) ? KIND_TC : KIND_SIMT16;
      return KIND_FFMA;
    case BGX_MODE_TC: {
      const char *why = nullptr;
      if (!tc_legal(d, &why)) {
        set_error("bgx_contract: tensor-core path not legal: %s", why);
        return BGX_ERR_UNSUPPORTED;
      }
      return KIND_TC;
    }
    case BGX_MODE_SIMT:
      return half_in ? KIND_SIMT16 : KIND_EXACT;
    case BGX_MODE_TF32: {
      const char *why = nullptr;
      if (d.in_dtype != BGX_F32) {
        set_error("bgx_contract: TF32 mode needs f32 inputs");
        return BGX_ERR_UNSUPPORTED;
      }
      if (!tc_legal(d, &why)) {
        set_error("bgx_contract: tf32 tensor-core path not legal: %s", why);
        return BGX_ERR_UNSUPPORTED;
      }
      return KIND_TC;
    }
    default:
      set_error("bgx_contract: bad mode %d", d.mode);
      return BGX_ERR_INVALID;
  }
}

int validate(const bgx_contract_desc &d) {
  BGX_CHECK_ARG(d.batch >= 0 && d.M >= 0 && d.N >= 0 && d.K >= 0, "bgx_contract: negative extent");
  BGX_CHECK_ARG(dtype_size(d.in_dtype) > 0 && dtype_size(d.out_dtype) > 0, "bgx_contract: bad dtype");
  const bool half_in = d.in_dtype == BGX_BF16 || d.in_dtype == BGX_F16;
  if (half_in)
    BGX_CHECK_ARG(d.out_dtype == d.in_dtype || d.out_dtype == BGX_F32,
                  "bgx_contract: out dtype must equal in dtype or be f32");
  else
    BGX_CHECK_ARG(d.out_dtype == d.in_dtype, "bgx_contract: f32/f64 out dtype must equal in dtype");
  for (int i = 0; i < 3; ++i)
    BGX_CHECK_ARG(d.a_stride[i] >= 0 && d.b_stride[i] >= 0 && d.c_stride[i] >= 0 && d.o_stride[i] >= 0,
                  "bgx_contract: negative stride");
  return BGX_OK;
}

}  // namespace
}  // namespace bgx

using namespace bgx;

extern "C" int bgx_contract_kernel(const bgx_contract_desc *d) {
  BGX_CHECK_ARG(d != nullptr, "bgx_contract_kernel: null descriptor");
  int rc = validate(*d);
  if (rc) return rc;
  return select_kind(*d);
}

extern "C" int bgx_contract(const bgx_contract_desc *d, void *stream) {
  BGX_CHECK_ARG(d != nullptr, "bgx_contract: null descriptor");
  int rc = validate(*d);
  if (rc) return rc;
  if (d->batch == 0 || d->M == 0 || d->N == 0) return BGX_OK;
  BGX_CHECK_ARG(d->out != nullptr, "bgx_contract: null out");
  const int kind = select_kind(*d);
  if (kind < 0) return kind;
  cudaStream_t s = (cudaStream_t)stream;
  if (d->K == 0) {
    // empty reduction: out = c0 (or 0).  Handled by the SIMT kernel's init.
    return contract_simt(*d, KIND_EXACT, s);
  }
  BGX_CHECK_ARG(d->a != nullptr && d->b != nullptr, "bgx_contract: null operand");
  if (kind == KIND_TC) return contract_tc(*d, s);
  return contract_simt(*d, kind, s);
}

extern "C" int bgx_contract_tile(const bgx_contract_desc *d, int32_t *cta_group, int32_t *tile_n) {
  BGX_CHECK_ARG(d != nullptr && cta_group != nullptr && tile_n != nullptr,
                "bgx_contract_tile: null argument");
  int rc = validate(*d);
  if (rc) return rc;
  if (select_kind(*d) != KIND_TC) {
    *cta_group = 0;
    *tile_n = 0;
    return BGX_OK;
  }
  int cg = 0, bn = 0;
  tc_tile_choice(*d, &cg, &bn);
  *cta_group = cg;
  *tile_n = bn;
  return BGX_OK;
}

extern "C" int bgx_contract_splitk_plan(const bgx_contract_desc *d, int32_t *splits,
                                        int64_t *workspace_bytes) {
  BGX_CHECK_ARG(d && splits && workspace_bytes, "bgx_contract_splitk_plan: null argument");
  int rc = validate(*d);
  if (rc) return rc;
  int sp = 1;
  int64_t ws = 0;
  if (select_kind(*d) == KIND_TC) tc_splitk_plan(*d, &sp, &ws);
  *splits = sp;
  *workspace_bytes = ws;
  return BGX_OK;
}

extern "C" int bgx_contract_splitk(const bgx_contract_desc *d, int32_t splits, void *workspace,
                                   int64_t workspace_bytes, void *stream) {
  BGX_CHECK_ARG(d != nullptr, "bgx_contract_splitk: null descriptor");
  int rc = validate(*d);
  if (rc) return rc;
  if (d->batch == 0 || d->M == 0 || d->N == 0) return BGX_OK;
  if ((splits <= 1 && splits >= -1) || d->K == 0) return bgx_contract(d, stream);
  const int kind = select_kind(*d);
  if (kind != KIND_TC) {
    set_error("bgx_contract_splitk: split-K runs on the tensor-core path only");
    return kind < 0 ? kind : BGX_ERR_UNSUPPORTED;
  }
  BGX_CHECK_ARG(d->a != nullptr && d->b != nullptr && d->out != nullptr,
                "bgx_contract_splitk: null operand");
  return contract_tc_splitk(*d, splits, workspace, workspace_bytes, (cudaStream_t)stream);
}

extern "C" int bgx_contract_rs_plan(const bgx_contract_desc *d, int32_t world, bgx_rs_plan *plan) {
  BGX_CHECK_ARG(d && plan, "bgx_contract_rs_plan: null argument");
  int rc = validate(*d);
  if (rc) return rc;
  return tc_rs_plan(*d, world, plan);
}

extern "C" int bgx_contract_reduce_scatter(const bgx_contract_desc *d, const bgx_reduce_scatter *rs,
                                           void *stream) {
  BGX_CHECK_ARG(d && rs, "bgx_contract_reduce_scatter: null argument");
  int rc = validate(*d);
  if (rc) return rc;
  BGX_CHECK_ARG(d->M > 0 && d->N > 0 && d->K > 0, "bgx_contract_reduce_scatter: empty extent");
  BGX_CHECK_ARG(d->a != nullptr && d->b != nullptr, "bgx_contract_reduce_scatter: null operand");
  return contract_tc_rs(*d, *rs, (cudaStream_t)stream);
}

extern "C" int bgx_rs_reduce(const bgx_contract_desc *d, const bgx_reduce_scatter *rs, void *stream) {
  BGX_CHECK_ARG(d && rs, "bgx_rs_reduce: null argument");
  BGX_CHECK_ARG(d->M > 0 && d->N > 0 && d->K > 0, "bgx_rs_reduce: empty extent");
  return rs_reduce(*d, *rs, (cudaStream_t)stream);
}
