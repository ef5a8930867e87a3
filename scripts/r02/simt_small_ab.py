"""Small exact f32 GEMMs: raw bgx_contract back-to-back time per call, and
bit-equality against the oracle (run twice: BGX_SIMT_SMALL=0 / 1)."""
import os
import statistics
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle  # noqa: E402
from paper_2503_04771_b200 import _lib  # noqa: E402

dev = torch.device("cuda", 0)
lib = _lib.load()
st = torch.cuda.current_stream().cuda_stream
for (M, N, K) in [(256, 256, 256), (128, 128, 128), (512, 512, 512), (256, 256, 4096),
                  (64, 1024, 256), (333, 257, 129), (332, 260, 132), (100, 36, 1000), (1024, 1024, 1024), (2048, 2048, 512)]:
    rng = np.random.default_rng(M + N + K)
    ah = rng.standard_normal((M, K), dtype=np.float32)
    bh = rng.standard_normal((K, N), dtype=np.float32)
    a, b = torch.from_numpy(ah).to(dev), torch.from_numpy(bh).to(dev)
    out = torch.empty(M, N, device=dev)
    d = _lib.BgxContractDesc()
    d.batch, d.M, d.N, d.K = 1, M, N, K
    d.a, d.b, d.out = a.data_ptr(), b.data_ptr(), out.data_ptr()
    d.a_stride[:] = [0, K, 1]
    d.b_stride[:] = [0, N, 1]
    d.o_stride[:] = [0, N, 1]
    d.in_dtype = d.out_dtype = _lib.F32
    d.mode = _lib.MODE_EXACT
    fn = lambda: lib.bgx_contract(d, st)  # noqa: E731
    for _ in range(50):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(2000):
        fn()
    torch.cuda.synchronize()
    us = (time.perf_counter() - t0) / 2000 * 1e6
    # device time of 200 back-to-back launches (host issue rate hidden:
    # queue them behind a 5 ms spin first)
    torch.cuda._sleep(int(5e6))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(200):
        fn()
    e1.record()
    torch.cuda.synchronize()
    dev_us = e0.elapsed_time(e1) / 200 * 1e3
    exact = np.array_equal(out.cpu().numpy(), oracle.gemm_kseq(ah, bh))
    print(f"variant {os.environ.get('BGX_SIMT_SMALL', '1')} {M}x{N}x{K}: {us:7.2f} us/call "
          f"device {dev_us:7.2f} us/launch bit-exact={exact}", flush=True)
