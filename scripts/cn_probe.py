"""Bit-equality and timing of the A-multicast cluster (cluster_n=2) vs the
plain CTA-pair kernel on a few shapes (run under `timeout`)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_04771_b200.api import contract  # noqa: E402

dev = torch.device("cuda", 0)
MM = "(i,k),(k,j)->(i,j)"
for (M, N, K, bn) in [(512, 512, 256, 256), (1024, 1536, 1024, 256), (4096, 4096, 4096, 256),
                      (4096, 4096, 8192, 512), (768, 1280, 640, 256), (8192, 8192, 8192, 512),
                      (8192, 8192, 8192, 256)]:
    a = torch.randn(M, K, device=dev).bfloat16()
    b = torch.randn(K, N, device=dev).bfloat16()
    base = contract(MM, a, b, schedule={"tile_n": bn, "cta_group": 2})
    torch.cuda.synchronize()
    y = contract(MM, a, b, schedule={"tile_n": bn, "cta_group": 2, "cluster_n": 2})
    torch.cuda.synchronize()
    eq = torch.equal(y.view(torch.int16), base.view(torch.int16))
    ts = {}
    for cn in (1, 2, 1, 2):
        sc = {"tile_n": bn, "cta_group": 2, "cluster_n": cn}
        for _ in range(3):
            contract(MM, a, b, schedule=sc)
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record()
        for _ in range(10):
            contract(MM, a, b, schedule=sc)
        s1.record()
        torch.cuda.synchronize()
        ts.setdefault(cn, []).append(s0.elapsed_time(s1) / 10)
    f = 2 * M * N * K
    print(f"{M}x{N}x{K} bn={bn} bitequal={eq} cn1={[round(f/t/1e9) for t in ts[1]]} "
          f"cn2={[round(f/t/1e9) for t in ts[2]]} TFLOP/s", flush=True)
