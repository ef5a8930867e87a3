"""Timing of the fused K-split reduce-scatter kernel on ONE B200.

For a K-split problem (M x N output, K = world * K_r) it times, with CUDA
events on the launching stream after warm-up:
  * unfused, per rank: contract(slab, out_dtype=f32) (the tcgen05 GEMM with
    its own split-K + reduce) — what ksplit_contract does before the NCCL
    reduce_scatter;
  * fused, per rank and for both reduction placements: the rank kernel of
    the first and of the last emulated rank (in-kernel mode: the last one
    also reduces every tile of every owner), and in deferred mode one
    owner's bgx_rs_reduce;
  * fused world=1: FusedKSplit on local buffers (GEMM + local split reduce +
    owner reduce + cast in one kernel) vs contract() with bf16 output.
Prints one JSON line per measurement.
"""

import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2503_04771_b200 import _lib, shard
if os.environ.get("BGX_PROBE_LIB"):          # A/B of two builds (probe only)
    _lib.LIB_PATH = os.environ["BGX_PROBE_LIB"]
from paper_2503_04771_b200.api import contract

MM = "(i,k),(k,j)->(i,j)"


def timed(fn, iters=20, warm=5):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(iters):
        s.record()
        fn()
        e.record()
        e.synchronize()
        ts.append(s.elapsed_time(e))
    ts.sort()
    return ts[len(ts) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--M", type=int, default=1024)
    ap.add_argument("--N", type=int, default=1024)
    ap.add_argument("--K", type=int, default=1 << 21)
    ap.add_argument("--world", type=int, default=8)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    M, N, K, W = args.M, args.N, args.K, args.world
    Kr = K // W
    a = torch.randn(M, Kr, device=dev).bfloat16()
    b = torch.randn(Kr, N, device=dev).bfloat16()
    flops_rank = 2 * M * N * Kr

    ms = timed(lambda: contract(MM, a, b, out_dtype=torch.float32))
    print(json.dumps({"what": "unfused rank GEMM -> f32 partial", "M": M, "N": N, "K_r": Kr,
                      "ms": ms, "tflops": flops_rank / ms / 1e9}))

    # emulated fused ranks, both reduction placements (bgx.h bgx_rs_plan.mode)
    d, _ = shard._rs_desc(MM, a, b, torch.bfloat16)
    lib = _lib.load()
    st = torch.cuda.current_stream().cuda_stream
    for mode in (_lib.RS_IN_KERNEL, _lib.RS_DEFERRED):
        pl = shard.rs_plan(MM, a, b, W)
        shard._finish_plan(pl, M, N, pl.local_splits, mode)
        rpo = pl.rows_per_owner
        slots = torch.empty(W, pl.slot_bytes // 4, device=dev)
        counters = torch.zeros(W, max(4, pl.counter_bytes // 4), dtype=torch.int32, device=dev)
        out = torch.empty(W * rpo, N, dtype=torch.bfloat16, device=dev)
        rs = _lib.BgxReduceScatter()
        for r in range(W):
            rs.slots[r], rs.counters[r], rs.out[r] = (slots[r].data_ptr(),
                                                      counters[r].data_ptr(),
                                                      out[r * rpo].data_ptr())
        ws = wsc = None
        if pl.ws_bytes > 0:
            ws = torch.empty(pl.ws_bytes, dtype=torch.uint8, device=dev)
            wsc = torch.zeros(max(16, pl.counter_bytes), dtype=torch.uint8, device=dev)
            rs.ws, rs.ws_counters = ws.data_ptr(), wsc.data_ptr()

        def launch(r):
            pl.rank = r
            rs.plan = pl
            _lib.check(lib.bgx_contract_reduce_scatter(d, rs, st), "rs")

        def reduce(r):
            pl.rank = r
            rs.plan = pl
            _lib.check(lib.bgx_rs_reduce(d, rs, st), "rs_reduce")

        def round_():
            for r in range(W):
                launch(r)
            if mode == _lib.RS_DEFERRED:
                for r in range(W):
                    reduce(r)

        t_round = timed(round_, iters=10, warm=3)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ts0, tsl, tsr = [], [], []
        for _ in range(10):
            torch.cuda.synchronize()
            s.record(); launch(0); e.record(); e.synchronize(); ts0.append(s.elapsed_time(e))
            for r in range(1, W - 1):
                launch(r)
            s.record(); launch(W - 1); e.record(); e.synchronize(); tsl.append(s.elapsed_time(e))
            if mode == _lib.RS_DEFERRED:
                for r in range(1, W):
                    reduce(r)
                # owner 0's reduce, 20 back to back (a lone launch would time
                # the host's launch latency, not the kernel)
                s.record()
                for _ in range(20):
                    reduce(0)
                e.record(); e.synchronize()
                tsr.append(s.elapsed_time(e) / 20)
        ts0.sort(); tsl.sort(); tsr.sort()
        print(json.dumps({"what": f"fused emulated world={W}",
                          "mode": "deferred" if mode == _lib.RS_DEFERRED else "in_kernel",
                          "plan": {"cta_group": pl.cta_group, "tile_n": pl.tile_n,
                                   "rows_per_owner": rpo, "local_splits": pl.local_splits},
                          "ms_round_all_ranks": t_round, "ms_rank_kernel_first": ts0[5],
                          "ms_rank_kernel_last": tsl[5],
                          "ms_owner_reduce": tsr[5] if tsr else None,
                          "tflops_rank_kernel": flops_rank / ts0[5] / 1e9}), flush=True)

    # world = 1: fused GEMM + reduce + cast vs contract() bf16 out
    a1 = torch.randn(M, Kr, device=dev).bfloat16()
    b1 = torch.randn(Kr, N, device=dev).bfloat16()
    f = shard.FusedKSplit(MM, a1, b1)
    t_f = timed(lambda: f(a1, b1))
    t_c = timed(lambda: contract(MM, a1, b1))
    print(json.dumps({"what": "world=1 fused vs contract", "ms_fused": t_f, "ms_contract": t_c,
                      "tflops_fused": flops_rank / t_f / 1e9,
                      "tflops_contract": flops_rank / t_c / 1e9}))


if __name__ == "__main__":
    main()
