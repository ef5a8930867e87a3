"""Small-output / long-K GEMM shapes through contract(): tile, split and
TFLOP/s (CUDA events, median of 20 after warm-up)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_04771_b200 import _lib, executor  # noqa: E402
from paper_2503_04771_b200.api import contract  # noqa: E402

SHAPES = [(256, 256, 1 << 20), (512, 512, 1 << 18), (1024, 1024, 1 << 18), (1024, 1024, 1 << 16),
          (2048, 2048, 1 << 16), (768, 1536, 1 << 17), (4096, 4096, 4096), (8192, 8192, 8192)]


def main():
    dev = torch.device("cuda", 0)
    lib = _lib.load()
    for M, N, K in SHAPES:
        a = torch.randn(M, K, device=dev).bfloat16()
        b = torch.randn(K, N, device=dev).bfloat16()
        out = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
        d = _lib.BgxContractDesc()
        d.batch, d.M, d.N, d.K = 1, M, N, K
        d.a_stride[1], d.a_stride[2], d.b_stride[1], d.b_stride[2] = K, 1, N, 1
        d.o_stride[1], d.o_stride[2] = N, 1
        d.in_dtype = d.out_dtype = _lib.BF16
        d.a, d.b, d.out = a.data_ptr(), b.data_ptr(), out.data_ptr()
        cg, bn, sp, ws = _lib._i32(), _lib._i32(), _lib._i32(), _lib._i64()
        lib.bgx_contract_tile(d, cg, bn)
        lib.bgx_contract_splitk_plan(d, sp, ws)
        for _ in range(5):
            contract("(i,k),(k,j)->(i,j)", a, b, out=out)
        torch.cuda.synchronize()
        ts = []
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for _ in range(20):
            s.record()
            contract("(i,k),(k,j)->(i,j)", a, b, out=out)
            e.record()
            e.synchronize()
            ts.append(s.elapsed_time(e))
        ts.sort()
        ms = ts[10]
        err = float((out.double() - a.double() @ b.double()).norm() / (a.double() @ b.double()).norm())
        print(json.dumps({"M": M, "N": N, "K": K, "cta_group": cg.value, "tile_n": bn.value,
                          "splits": sp.value, "ms": round(ms, 4),
                          "tflops": round(2 * M * N * K / ms / 1e9, 1), "relF": err}), flush=True)
        del a, b, out
        executor.reset_launch_log()


if __name__ == "__main__":
    main()
