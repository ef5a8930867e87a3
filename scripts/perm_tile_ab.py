"""A/B of the vectorised transpose tile shape (BGX_PERM_TILE is read once per
process, so each variant runs in its own process): C2a / C2b GB/s."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_04771_b200 import contract  # noqa: E402

dev = torch.device("cuda", 0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for name, spec, shape in (("c2a", "(i,j)->(j,i)", (8192, 8192)),
                          ("c2b", "(i,j,k)->(k,j,i)", (256, 512, 512))):
    x = torch.randn(shape, device=dev)
    out = contract(spec, x)
    ref = x.permute(*reversed(range(x.dim()))).contiguous()
    assert torch.equal(out, ref)
    ts = []
    for _ in range(30):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); contract(spec, x, out=out); e.record(); e.synchronize()
        ts.append(s.elapsed_time(e))
    ms = statistics.median(ts)
    print(f"tile={os.environ.get('BGX_PERM_TILE', '0')} {name}: {ms * 1e3:.1f} us "
          f"{2 * x.numel() * 4 / ms / 1e6:.0f} GB/s", flush=True)
