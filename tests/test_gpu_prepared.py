"""prepare(): plan once / launch many, and CUDA-graph replay — identical
results to contract() for every plan class."""

import pytest
import torch

import paper_2503_04771_b200 as bgx
from paper_2503_04771_b200 import executor

pytestmark = pytest.mark.gpu

CASES = [
    ("(i,k),(k,j)->(i,j)", [(256, 192), (192, 320)], torch.bfloat16),
    ("(i,k),(k,j)->(i,j)", [(100, 70), (70, 50)], torch.float32),
    ("(b,i,j),(b,j,k)->(b,i,k)", [(4, 128, 64), (4, 64, 96)], torch.float16),
    ("(i,j,k)->(k,j,i)", [(16, 33, 40)], torch.float32),
    ("(i,j)->(i)", [(50, 77)], torch.float32),
    ("(i,j),(j,k),(k,l)->(i,l)", [(9, 10), (10, 11), (11, 12)], torch.float32),
    ("(i,k),(k,j),(j,l)->(i,l)", [(512, 256), (256, 128), (128, 64)], torch.bfloat16),
]


@pytest.mark.parametrize("spec,shapes,dt", CASES, ids=[c[0] for c in CASES])
@pytest.mark.parametrize("graph", [False, True])
def test_prepared_matches_contract(dev, spec, shapes, dt, graph):
    g = torch.Generator(device=dev).manual_seed(0)
    xs = [torch.randn(s, generator=g, device=dev).to(dt) for s in shapes]
    want = bgx.contract(spec, *xs)
    p = bgx.prepare(spec, *xs, graph=graph)
    got = p()
    assert torch.equal(got, want)
    # new data through the same plan
    for x in p.inputs:
        x.copy_(torch.randn(x.shape, generator=g, device=dev).to(dt))
    want2 = bgx.contract(spec, *p.inputs)
    got2 = p() if graph else p(*p.inputs)
    assert torch.equal(got2, want2)


def test_prepared_fast_path_and_errors(dev):
    a = torch.randn(128, 64, device=dev).bfloat16()
    b = torch.randn(64, 256, device=dev).bfloat16()
    p = bgx.prepare("(i,k),(k,j)->(i,j)", a, b)
    assert p._fast is not None
    executor.reset_launch_log()
    p(a, b)
    assert executor.launch_log() == []      # no executor round trip
    with pytest.raises(ValueError, match="different shapes"):
        p(torch.randn(64, 64, device=dev).bfloat16(), b)


def test_prepared_fuzz_matches_contract(dev):
    """prepare() (pre-built descriptors, pointer patching) and its CUDA-graph
    form give exactly what contract() gives, over random specs, dtypes and
    strided views."""
    import random
    from paper_2503_04771_b200 import contract, prepare
    r = random.Random(5)
    specs = ["(i,k),(k,j)->(i,j)", "(b,i,k),(b,k,j)->(b,i,j)", "(i,j)->(j,i)", "(i,j)->(i)",
             "(i,j),(i,j)->(i,j)", "(i,k),(j,k)->(i,j)", "(i,j,k)->(k,i,j)"]
    for it in range(30):
        text = r.choice(specs)
        dt = r.choice([torch.float32, torch.bfloat16])
        spec_ins = [t.split(",") for t in text.split("->")[0][1:-1].split("),(")]
        ext = {a: 8 * r.randint(1, 40) for t in spec_ins for a in t}
        xs = [torch.randn([ext[a] for a in t], device=dev).to(dt) for t in spec_ins]
        if r.random() < 0.3 and xs[0].dim() >= 2:
            xs[0] = xs[0].transpose(0, 1).contiguous().transpose(0, 1)
        want = contract(text, *xs)
        p = prepare(text, *xs)
        assert torch.equal(p(*xs), want), text
        g = prepare(text, *xs, graph=True)
        assert torch.equal(g(), want), text
