"""Outer products (no reduction): GEMM tiles with K = 1 vs the generic path
(now bcast_ew_kernel), plan.OUTER_TO_LOOP_NEST off / on, us per call."""
import statistics
import sys

import torch

sys.path.insert(0, ".")
from paper_2503_04771_b200 import api, contract, executor, plan  # noqa: E402

dev = torch.device("cuda", 0)
CASES = [("(a),(b)->(a,b)", dict(a=4096, b=8192)), ("(a),(b)->(a,b)", dict(a=1024, b=1024)),
         ("(a),(b)->(a,b)", dict(a=256, b=65536)), ("(b),(a,c)->(a,c,b)", dict(a=256, c=256, b=256)),
         ("(a,c),(b)->(a,b,c)", dict(a=64, b=512, c=1024)), ("(i),(j)->(j,i)", dict(i=4096, j=4096))]
for dt in (torch.float32, torch.bfloat16, torch.float64):
    for text, ext in CASES:
        ins, out = text.split("->")
        tups = [t.strip("()").split(",") for t in ins.split("),(")]
        otup = out.strip("()").split(",")
        xs = [torch.randn([ext[a] for a in t], device=dev).to(dt) for t in tups]
        o = torch.empty([ext[a] for a in otup], device=dev, dtype=dt)
        res = {}
        outs = {}
        for flag in (False, True):
            plan.OUTER_TO_LOOP_NEST = flag
            plan._plan_cached.cache_clear()
            api._fast_cache().clear()
            executor._exec_cache().clear()
            executor.reset_launch_log()
            for _ in range(3):
                contract(text, *xs, out=o)
            torch.cuda.synchronize()
            kinds = executor.launch_log()[-1:]
            ts = []
            for _ in range(5):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(); contract(text, *xs, out=o); e1.record(); torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1) * 1e3)
            res[flag] = (statistics.median(ts), kinds)
            outs[flag] = o.clone()
        same = torch.equal(outs[False], outs[True])
        print(f"{text:22s} {str(ext):34s} {str(dt)[6:]:9s} gemm {res[False][0]:8.1f} us {res[False][1]}"
              f"  generic {res[True][0]:8.1f} us {res[True][1]}  equal={same}", flush=True)
