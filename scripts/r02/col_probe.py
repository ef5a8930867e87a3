import statistics
import sys
import torch
sys.path.insert(0, ".")
from paper_2503_04771_b200 import contract  # noqa: E402
dev = torch.device("cuda", 0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
def t(fn):
    fn(); ts = []
    for _ in range(5):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); ts.append((a, b))
    torch.cuda.synchronize()
    return statistics.median(x.elapsed_time(y) for x, y in ts) * 1e3
for K, J in [(8192, 8192), (8192, 16384), (16384, 8192), (4096, 16384)]:
    A = torch.randn(K, J, device=dev).bfloat16(); x = torch.randn(K, device=dev).bfloat16()
    r1 = t(lambda: contract("(k,j)->(j)", A))
    r2 = t(lambda: contract("(k),(k,j)->(j)", x, A))
    r3 = t(lambda: contract("(k,j),(k)->(j)", A, x))
    print(f"K={K} J={J}: (k,j)->(j) {r1:7.1f} us   (k),(k,j)->(j) {r2:7.1f} us   (k,j),(k)->(j) {r3:7.1f} us", flush=True)
