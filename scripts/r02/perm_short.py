import statistics
import sys
import torch
sys.path.insert(0, ".")
from paper_2503_04771_b200 import contract  # noqa: E402
dev = torch.device("cuda", 0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
def t(fn):
    fn(); ts = []
    for _ in range(10):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); ts.append((a, b))
    torch.cuda.synchronize()
    return statistics.median(x.elapsed_time(y) for x, y in ts) * 1e3
for spec, shape, perm in [("(c,a,b)->(a,c,b)", (256, 256, 64), (1, 0, 2)), ("(c,a,b)->(a,c,b)", (1024, 1024, 16), (1, 0, 2)),
                          ("(a,b,c,d)->(b,a,c,d)", (64, 64, 64, 64), (1, 0, 2, 3)), ("(a,b,c)->(b,a,c)", (2048, 2048, 8), (1, 0, 2))]:
    for dt in (torch.float32, torch.bfloat16):
        x = torch.randn(shape, device=dev).to(dt)
        y = contract(spec, x)
        ok = torch.equal(y, x.permute(*perm).contiguous())
        us = t(lambda: contract(spec, x))
        print(f"{spec:22s} {str(shape):20s} {str(dt):15s} {us:8.1f} us {2*x.numel()*x.element_size()/us/1e3:7.0f} GB/s exact={ok}", flush=True)
