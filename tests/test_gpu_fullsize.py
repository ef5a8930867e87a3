"""BASELINE configs 1 and 2 at FULL size on the B200 against the reference's
own outputs (tests/golden/fullsize_*: bridgegen run_function on the whole
problem): C1 256^3 f32 bit-identical through the reference-shaped API, C2a /
C2b permutations byte-identical (SHA-256 of the output); C3 / C4 / C5 at
full size through bit-exact size-independent properties (scaling by 2, row
permutation) plus f64 row samples."""

import numpy as np
import pytest
import torch

import _golden as G
from paper_2503_04771_b200 import einsum as E
from paper_2503_04771_b200 import executor
from paper_2503_04771_b200 import interp as I
from paper_2503_04771_b200.api import contract

pytestmark = pytest.mark.gpu


def test_c1_fullsize_bit_exact_reference_api(dev):
    a, b = G.fullsize_inputs("c1")
    mod = E.build_einsum_function(None, E.parse_einsum(G.FULLSIZE_SPECS["c1"]))
    vals = [I.TensorValue(E.F32, x.shape, x) for x in (a, b, np.zeros((256, 256), np.float32))]
    executor.reset_launch_log()
    [got] = I.run_function(mod, "einsum", vals, step_limit=None)
    assert executor.launch_log() == ["simt-exact"]
    assert np.array_equal(np.asarray(got.data).view(np.uint32), G.fullsize_c1().view(np.uint32))


def test_c1_fullsize_bit_exact_device_api(dev):
    a, b = (torch.from_numpy(x).to(dev) for x in G.fullsize_inputs("c1"))
    y = contract(G.FULLSIZE_SPECS["c1"], a, b, mode="exact")
    assert G.sha256(y.cpu().numpy()) == G.fullsize_meta()["configs"]["c1"]["out_sha256"]


@pytest.mark.parametrize("config", ["c2a", "c2b"])
def test_c2_fullsize_permutation_digest(dev, config):
    [x] = G.fullsize_inputs(config)
    executor.reset_launch_log()
    y = contract(G.FULLSIZE_SPECS[config], torch.from_numpy(x).to(dev))
    assert executor.launch_log() == ["permute"]
    meta = G.fullsize_meta()["configs"][config]
    assert list(y.shape) == meta["out_shape"]
    assert G.sha256(y.cpu().numpy()) == meta["out_sha256"]


# ---- C3 / C4 / C5 at full size: size-independent properties -------------------
# The oracle cannot run these sizes whole, so besides row samples against the
# f64 oracle (test_gpu_gemm / bench) the device results are checked for
# properties every correct evaluation has, bit for bit: scaling an input by 2
# scales every output by 2 exactly (powers of two commute with f32 sums and
# bf16 rounding when nothing overflows), and permuting the free rows of the
# first operand permutes the output rows (each output element
# is computed from its own row in the same k order wherever its tile lands).

def _bf16(shape, seed, dev):
    g = torch.Generator(device=dev).manual_seed(seed)
    return torch.randn(shape, device=dev, generator=g).bfloat16()


@pytest.mark.parametrize("cfg", ["c3", "c4", "c5"])
def test_fullsize_scaling_and_row_permutation(dev, cfg):
    import oracle
    if cfg == "c3":
        spec, ops = "(b,i,j),(b,j,k)->(b,i,k)", [_bf16((64, 1024, 1024), 1, dev),
                                                 _bf16((64, 1024, 1024), 2, dev)]
    elif cfg == "c4":
        spec, ops = "(i,k),(k,j)->(i,j)", [_bf16((4096, 4096), 1, dev), _bf16((4096, 4096), 2, dev)]
    else:
        spec, ops = "(i,k),(k,j),(j,l)->(i,l)", [_bf16((32768, 8192), 1, dev),
                                                 _bf16((8192, 8192), 2, dev),
                                                 _bf16((8192, 8192), 3, dev)]
    out = contract(spec, *ops)
    assert torch.isfinite(out.float()).all()
    twice = contract(spec, ops[0] * 2, *ops[1:])
    assert torch.equal(twice, out * 2)
    g = torch.Generator(device=dev).manual_seed(5)
    ax = 1 if cfg == "c3" else 0          # the free row index i of operand 0
    perm = torch.randperm(ops[0].shape[ax], device=dev, generator=g)
    permuted = contract(spec, ops[0].index_select(ax, perm).contiguous(), *ops[1:])
    assert torch.equal(permuted, out.index_select(ax, perm))
    if cfg == "c5":   # row samples against the f64 oracle (ladder L3)
        rows = np.random.default_rng(3).choice(32768, 4, replace=False)
        want = oracle.chain_f64(ops[0][torch.as_tensor(rows, device=dev)].float().cpu().numpy(),
                                ops[1].float().cpu().numpy(), ops[2].float().cpu().numpy(),
                                slice(None))
        got = out[torch.as_tensor(rows, device=dev)].float().cpu().numpy()
        assert oracle.rel_frobenius(got, want) <= 1e-2
