import sys, statistics, torch
sys.path.insert(0, ".")
from paper_2503_04771_b200 import contract, executor
dev = torch.device("cuda", 0)
for spec, shapes in [("(i,k),(k)->(i)", [(8192, 8192), (8192,)]), ("(k,i),(k)->(i)", [(8192, 8192), (8192,)]),
                     ("(b,i,k),(b,k)->(b,i)", [(64, 1024, 1024), (64, 1024)]), ("(i,k)->(i)", [(8192, 8192)]),
                     ("(i,k)->(k)", [(8192, 8192)]), ("(i,k)->()", [(8192, 8192)])]:
    for dt in (torch.bfloat16, torch.float32):
        xs = [torch.randn(s, device=dev).to(dt) for s in shapes]
        f = lambda: contract(spec, *xs)
        for _ in range(3): f()
        torch.cuda.synchronize(); executor.reset_launch_log(); f(); kinds = executor.launch_log()
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); f(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
        ms = statistics.median(ts); byts = sum(x.numel() for x in xs) * xs[0].element_size()
        print(f"{spec:22s} {str(dt)[6:]:9s} {ms*1e3:8.1f} us  {byts/ms/1e6:7.0f} GB/s  {kinds}", flush=True)
