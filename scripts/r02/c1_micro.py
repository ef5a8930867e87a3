"""Host cost of the pieces of a replayed run_function call (BASELINE C1),
each timed alone over many iterations (us per call)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2503_04771_b200 import _lib, executor  # noqa: E402
from paper_2503_04771_b200 import einsum as E  # noqa: E402
from paper_2503_04771_b200 import interp as I  # noqa: E402

dev = torch.device("cuda", 0)
rng = np.random.default_rng(1)
ts = [torch.from_numpy(rng.standard_normal((256, 256), dtype=np.float32)).to(dev) for _ in range(2)]
ts.append(torch.zeros(256, 256, device=dev))
mod = E.build_einsum_function(None, E.parse_einsum("(i,j),(j,k)->(i,k)"))
vals = [I.TensorValue(E.F32, (256, 256), t) for t in ts]
for _ in range(50):
    I.run_function(mod, "einsum", vals, step_limit=None)
torch.cuda.synchronize()
spec = mod.lookup_symbol("einsum").ops[0].spec
o = torch.empty(256, 256, device=dev)
a, b, c = ts
lib = _lib.load()
N = 500


def t(name, fn):
    """host cost per call: the GPU is held by a long spin kernel, so
    launches only queue and the loop measures the issuing thread alone"""
    for _ in range(200):
        fn()
    torch.cuda.synchronize()
    best = None
    for _ in range(5):
        torch.cuda._sleep(int(2e8))          # ~100 ms of GPU spin
        t0 = time.perf_counter()
        for _ in range(N):
            fn()
        dt = (time.perf_counter() - t0) / N * 1e6
        torch.cuda.synchronize()
        best = dt if best is None else min(best, dt)
    print(f"{name:40s} {best:7.2f} us", flush=True)


t("run_function (replay)", lambda: I.run_function(mod, "einsum", vals, step_limit=None))
t("executor.execute (fast cache)", lambda: executor.execute(spec, [a, b], c, o))
t("_replay_key", lambda: I._replay_key(mod, "einsum", vals, "auto", None, None))
t("_exec_key", lambda: executor._exec_key(spec, [a, b], c, o, "auto", "auto"))
t("torch.empty 256x256", lambda: torch.empty((256, 256), dtype=torch.float32, device=dev))
t("TensorValue(...)", lambda: I.TensorValue(E.F32, (256, 256), o))
t("_on_device(dev) enter/exit", lambda: executor._on_device(dev).__enter__())
t("_stream_ptr", lambda: executor._stream_ptr(o))
t("t.stride()", lambda: a.stride())
t("t.data_ptr()", lambda: a.data_ptr())
t("t.device", lambda: a.device)
t("t.is_cuda", lambda: a.is_cuda)
t("t.shape", lambda: a.shape)
d = _lib.BgxContractDesc()
d.batch, d.M, d.N, d.K = 1, 256, 256, 256
d.a, d.b, d.out = a.data_ptr(), b.data_ptr(), o.data_ptr()
d.a_stride[:] = [0, 256, 1]
d.b_stride[:] = [0, 256, 1]
d.o_stride[:] = [0, 256, 1]
d.in_dtype = d.out_dtype = _lib.F32
d.mode = _lib.MODE_EXACT
st = executor._stream_ptr(o)
t("raw lib.bgx_contract (ctypes)", lambda: lib.bgx_contract(d, st))


def setp():
    d.a, d.b, d.out = a.data_ptr(), b.data_ptr(), o.data_ptr()


t("desc pointer patch (3 fields)", setp)
