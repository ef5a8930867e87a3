"""PCIe picture for the e2e chain step: H2D alone, D2H alone, both at once
(duplex?), and contract_host at several chunk sizes.  CUDA events on the
copy streams; 1 s idle between measurements."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_04771_b200.api import contract_host  # noqa: E402

dev = torch.device("cuda", 0)
GB = 1e9
hin = torch.empty(768 << 20, dtype=torch.uint8, pin_memory=True)
hout = torch.empty(512 << 20, dtype=torch.uint8, pin_memory=True)
din = torch.empty(768 << 20, dtype=torch.uint8, device=dev)
dout = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(2):
    din.copy_(hin, non_blocking=True)
    hout.copy_(dout, non_blocking=True)
torch.cuda.synchronize()


def timed(fn):
    torch.cuda.synchronize()
    time.sleep(0.5)
    t0 = time.perf_counter()
    fn()
    torch.cuda.synchronize()
    return time.perf_counter() - t0


t = timed(lambda: din.copy_(hin, non_blocking=True))
print(f"H2D alone 768 MiB: {t*1e3:.2f} ms = {din.numel()/t/GB:.1f} GB/s")
t = timed(lambda: hout.copy_(dout, non_blocking=True))
print(f"D2H alone 512 MiB: {t*1e3:.2f} ms = {dout.numel()/t/GB:.1f} GB/s")


def both():
    with torch.cuda.stream(s1):
        din.copy_(hin, non_blocking=True)
    with torch.cuda.stream(s2):
        hout.copy_(dout, non_blocking=True)


t = timed(both)
print(f"H2D 768 MiB + D2H 512 MiB concurrently: {t*1e3:.2f} ms "
      f"(sum of alone would be the serial time)")
I, K = 32768, 8192
hA = torch.randn(I, K).bfloat16().pin_memory()
hB = torch.randn(K, K).bfloat16().pin_memory()
hC = torch.randn(K, K).bfloat16().pin_memory()
hO = torch.empty(I, K, dtype=torch.bfloat16).pin_memory()
for cr in (1024, 2048, 4096, 2048):
    f = lambda: contract_host("(i,k),(k,j),(j,l)->(i,l)", hA, hB, hC, out=hO, device=dev,  # noqa
                              chunk_rows=cr)
    f()
    f()
    ts = [timed(f) * 1e3 for _ in range(3)]
    print(f"contract_host chunk_rows={cr}: " + " ".join(f"{x:.2f}" for x in ts) + " ms")
