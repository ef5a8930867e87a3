"""Host-buffer API (the e2e path of bench.py): pipelined row-chunked
H2D / compute / D2H must give the same result as the device API."""

import numpy as np
import pytest
import torch

import oracle
from paper_2503_04771_b200 import contract
from paper_2503_04771_b200.api import contract_host

pytestmark = pytest.mark.gpu


def pinned(t):
    return torch.empty(t.shape, dtype=t.dtype, pin_memory=True).copy_(t)


@pytest.mark.parametrize("spec,shapes", [
    ("(i,k),(k,j),(j,l)->(i,l)", [(1000, 256), (256, 192), (192, 320)]),
    ("(i,k),(k,j)->(i,j)", [(1500, 320), (320, 256)]),
])
def test_chunked_host_pipeline_matches_device(dev, spec, shapes):
    g = torch.Generator().manual_seed(0)
    hs = [pinned(torch.randn(s, generator=g).bfloat16()) for s in shapes]
    want = contract(spec, *[h.to(dev) for h in hs]).cpu()
    got = contract_host(spec, *hs, device=dev, chunk_rows=256)
    assert got.is_pinned() and got.shape == want.shape
    assert torch.allclose(got.float(), want.float(), rtol=1e-2, atol=1e-2)
    same = torch.equal(got, want)
    got1 = contract_host(spec, *[h.clone() for h in hs], device=dev)  # unpinned: no pipeline
    assert torch.allclose(got1.float(), want.float(), rtol=1e-2, atol=1e-2)
    if len(shapes) == 2:
        ref = oracle.gemm_kseq(hs[0].float().numpy(), hs[1].float().numpy())
        assert oracle.rel_frobenius(got.float().numpy(), ref) <= 1e-2
    print("bit-identical to unchunked:", same)


def test_chunked_host_fp32_exact_with_c0(dev):
    g = torch.Generator().manual_seed(1)
    a, b, c0 = (pinned(torch.randn(s, generator=g)) for s in ((700, 64), (64, 48), (700, 48)))
    got = contract_host("(i,k),(k,j)->(i,j)", a, b, c0=c0, device=dev, chunk_rows=128)
    want = oracle.gemm_kseq(a.numpy(), b.numpy(), c0.numpy())
    assert np.array_equal(got.numpy(), want)


def test_contract_devices_matches_single_device(dev):
    """One-process M-shard over a device list (here the same GPU twice and
    three times): bit-identical rows to the unsharded call."""
    a = torch.randn(3000, 1024, device=dev).bfloat16()
    b = torch.randn(1024, 768, device=dev).bfloat16()
    c = torch.randn(768, 512, device=dev).bfloat16()
    spec = "(i,k),(k,j),(j,l)->(i,l)"
    whole = contract(spec, a, b, c, schedule={"splits": 1})
    for devs in ([0, 0], [0, 0, 0]):
        sh = contract(spec, a, b, c, devices=devs, schedule={"splits": 1})
        assert torch.equal(sh, whole)
    # leading output index not the first axis of operand 0 (strided slab)
    at = a.t().contiguous()
    whole = contract("(k,i),(k,j)->(i,j)", at, b, schedule={"splits": 1})
    assert torch.equal(contract("(k,i),(k,j)->(i,j)", at, b, devices=[0, 0],
                                schedule={"splits": 1}), whole)
    # leading output index carried by operand 1
    whole = contract("(k,j),(i,k)->(i,j)", b, a, schedule={"splits": 1})
    assert torch.equal(contract("(k,j),(i,k)->(i,j)", b, a, devices=[0, 0, 0],
                                schedule={"splits": 1}), whole)
    with pytest.raises(ValueError, match="rank-0"):
        contract("(i),(i)->()", a[:, 0], a[:, 1], devices=[0, 0])


@pytest.mark.parametrize("spec,shape", [("(i,j)->(j,i)", (1000, 777)),
                                        ("(i,j,k)->(k,j,i)", (33, 64, 130)),
                                        ("(i,j,k)->(j,k,i)", (17, 300, 9))])
def test_contract_devices_permutation(dev, spec, shape):
    """§8e permutation shard: each device writes a slab of output rows from a
    strided slab of the input — bit-exact against the unsharded kernel and
    torch's own permute."""
    from paper_2503_04771_b200.einsum import parse_einsum
    x = torch.randn(shape, device=dev)
    sp = parse_einsum(spec)
    perm = [sp.inputs[0].index(ax) for ax in sp.output]
    want = x.permute(perm).contiguous()
    assert torch.equal(contract(spec, x), want)
    for devs in ([0, 0], [0, 0, 0, 0]):
        assert torch.equal(contract(spec, x, devices=devs), want)


def test_contract_host_fuzz(dev):
    """contract_host over random row counts around the chunk size, with and
    without c0 / pinned buffers: identical to contract() on the device."""
    import random
    r = random.Random(12)
    for it in range(12):
        rows = r.choice([1, 100, 2047, 2048, 2049, 5000])
        K, N = 8 * r.randint(1, 64), 8 * r.randint(1, 64)
        pinned = r.random() < 0.8
        a = torch.randn(rows, K).bfloat16()
        b = torch.randn(K, N).bfloat16()
        c0 = torch.randn(rows, N).bfloat16() if r.random() < 0.4 else None
        if pinned:
            a, b = a.pin_memory(), b.pin_memory()
            c0 = c0.pin_memory() if c0 is not None else None
        got = contract_host("(i,k),(k,j)->(i,j)", a, b, c0=c0, device=dev,
                            chunk_rows=r.choice([None, 512, 2048]))
        want = contract("(i,k),(k,j)->(i,j)", a.to(dev), b.to(dev),
                        c0=c0.to(dev) if c0 is not None else None)
        assert torch.equal(got, want.cpu()), (it, rows, K, N, pinned)


def test_concurrent_threads_and_streams(dev):
    """Several host threads, each on its own CUDA stream, issuing contractions
    concurrently (per-thread launch caches and logs, thread-safe plan cache):
    every result equals the single-threaded one."""
    import threading
    specs = [("(i,k),(k,j)->(i,j)", [(512, 256), (256, 384)], torch.bfloat16),
             ("(i,j)->(j,i)", [(300, 700)], torch.float32),
             ("(i,j)->(i)", [(200, 4000)], torch.float32),
             ("(b,i,k),(b,k,j)->(b,i,j)", [(3, 128, 64), (3, 64, 96)], torch.float32)]
    inputs = [[torch.randn(s, device=dev).to(dt) for s in shapes] for _, shapes, dt in specs]
    want = [contract(sp, *xs) for (sp, _, _), xs in zip(specs, inputs)]
    errors = []

    def worker(tid):
        try:
            st = torch.cuda.Stream(dev)
            with torch.cuda.stream(st):
                for it in range(20):
                    k = (tid + it) % len(specs)
                    got = contract(specs[k][0], *inputs[k])
                    st.synchronize()
                    if not torch.equal(got, want[k]):
                        errors.append((tid, it, specs[k][0]))
        except Exception as e:  # noqa: BLE001
            errors.append((tid, repr(e)))

    threads = [threading.Thread(target=worker, args=(t,)) for t in range(4)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors[:3]


def test_execute_launch_cache_matches_uncached(dev):
    """The per-signature GEMM launch cache (executor._fast_gemm): repeated
    calls, views at other offsets (different 16-byte alignment), c0 on/off,
    f32 exact and bf16 tensor-core plans — identical results and launch-log
    names to the uncached path."""
    from paper_2503_04771_b200 import executor
    g = torch.Generator(device=dev).manual_seed(3)
    base = torch.randn(300 * 130 + 64, device=dev, generator=g)
    b = torch.randn(128, 96, device=dev, generator=g)
    c0 = torch.randn(300, 96, device=dev, generator=g)
    spec = "(i,k),(k,j)->(i,j)"
    for dt in (torch.float32, torch.bfloat16):
        for off in (0, 1, 4, 0, 1):           # revisit signatures: cache hits
            a = base[off:off + 300 * 128].view(300, 128).to(dt)
            if off % 4:                        # misaligned view of the same shape
                a = base.to(dt)[off:off + 300 * 128].view(300, 128)
            for c in (None, c0.to(dt)):
                executor._exec_cache().clear()
                executor.reset_launch_log()
                want = contract(spec, a, b.to(dt), c0=c)
                first = executor.launch_log()
                executor.reset_launch_log()
                got1 = contract(spec, a, b.to(dt), c0=c)     # builds the cache entry
                got2 = contract(spec, a, b.to(dt), c0=c)     # cached launch
                assert torch.equal(got1, want) and torch.equal(got2, want)
                assert executor.launch_log() == first * 2


@pytest.mark.parametrize("spec,shape", [("(i,j)->(j,i)", (300, 257)), ("(i,j,k)->(k,j,i)", (7, 9, 33)),
                                        ("(i,j)->(i,j)", (64, 64))])
def test_execute_launch_cache_permutations(dev, spec, shape):
    """Cached permutation launches: bit-exact, including strided views."""
    from paper_2503_04771_b200 import executor
    from paper_2503_04771_b200.einsum import parse_einsum
    sp = parse_einsum(spec)
    perm = [sp.inputs[0].index(ax) for ax in sp.output]
    base = torch.randn((shape[0] * 2,) + tuple(shape[1:]), device=dev)
    for x in (base[: shape[0]], base[::2], base[: shape[0]]):
        executor.reset_launch_log()
        for _ in range(3):
            y = contract(spec, x)
            assert torch.equal(y, x.permute(perm).contiguous())
        assert executor.launch_log() == ["permute"] * 3
