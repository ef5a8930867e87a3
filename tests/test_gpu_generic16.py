"""bf16/f16 bodies the GEMM planner does not map (reductions, Hadamard and
outer products, rank-0 outputs, passthrough, 3-operand bodies) through the
reference-shaped API and ``contract``: the generic kernel widens to f32, runs
the reference's loop order with per-op f32 rounding and rounds once — so it
is bit-equal to the C oracle on the f32-widened inputs followed by one
round-to-nearest-even to the storage type."""

import numpy as np
import pytest
import torch

import oracle
from paper_2503_04771_b200 import einsum as E
from paper_2503_04771_b200 import executor
from paper_2503_04771_b200 import interp as I
from paper_2503_04771_b200.api import contract

pytestmark = pytest.mark.gpu

SPECS = ["(i,j)->(i)", "(i,j)->(j)", "(i,j)->()", "(i,j),(i,j)->(i,j)", "(i),(j)->(i,j)",
         "(i,j,k)->(k,i)", "(i,k),(k,j),(j)->(i)", "(i)->(i)", "(b,i,j),(b,j)->(b,i)"]


def _shapes(spec, ext):
    return [tuple(ext[x] for x in t) for t in spec.inputs], tuple(ext[x] for x in spec.output)


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16])
@pytest.mark.parametrize("text", SPECS)
def test_generic16_matches_widened_oracle(dev, text, dtype):
    spec = E.parse_einsum(text)
    rng = np.random.default_rng(len(text))
    ext = {a: int(rng.integers(3, 40)) for a in spec.axes}
    in_shapes, out_shape = _shapes(spec, ext)
    ins = [torch.from_numpy(rng.standard_normal(s).astype(np.float32)).to(dtype) for s in in_shapes]
    c0 = torch.from_numpy(rng.standard_normal(out_shape).astype(np.float32)).to(dtype)
    executor.reset_launch_log()
    got = contract(spec, *[t.to(dev) for t in ins], c0=c0.to(dev))
    if text == "(i)->(i)":
        assert torch.equal(got.cpu(), ins[0])
        return
    want32 = oracle.generic(list(spec.inputs), spec.output, [t.float().numpy() for t in ins],
                            c0.float().numpy())
    want = torch.from_numpy(np.asarray(want32, np.float32)).to(dtype)
    if executor.launch_log() != ["generic"]:
        # GEMM-shaped 16-bit bodies (incl. GEMV and multi-operand chains) run
        # on the GEMM kernels (f32 accumulate with FMA / tensor cores, 16-bit
        # intermediates between chain steps): tolerance, not bits
        w = want32.astype(np.float64)
        relf = float(np.linalg.norm(got.cpu().double().numpy() - w) / np.linalg.norm(w))
        assert relf <= 1e-2, (text, relf)
        return
    assert torch.equal(got.cpu().view(torch.int16), want.view(torch.int16)), text


def test_generic16_through_run_function(dev):
    spec = E.parse_einsum("(i,j)->(i)")
    mod = E.build_einsum_function(None, spec, elem=E.BF16)
    x = torch.randn(17, 300, device=dev).bfloat16()
    z = torch.zeros(17, device=dev, dtype=torch.bfloat16)
    executor.reset_launch_log()
    [got] = I.run_function(mod, "einsum", [I.TensorValue(E.BF16, x.shape, x),
                                          I.TensorValue(E.BF16, z.shape, z)], step_limit=None)
    assert executor.launch_log() == ["generic"]
    want = torch.from_numpy(np.asarray(oracle.generic([("i", "j")], ("i",), [x.float().cpu().numpy()],
                                                      np.zeros(17, np.float32)), np.float32))
    assert torch.equal(got.data.cpu().float(), want.bfloat16().float())


@pytest.mark.parametrize("text,ext", [
    ("(b,d,a),(d,c),(b,d,a)->()", dict(b=3, d=256, a=64, c=16)),   # was 1.1e-1 through a bf16 chain
    ("(b,c),(b),(b)->()", dict(b=64, c=256)),                      # was 2.4e-2
])
def test_small_multi_operand_16bit_bodies_round_once(dev, text, ext):
    """16-bit bodies with 3+ operands small enough to walk directly keep f32
    arithmetic over the whole product space and round once (a pairwise chain
    rounded each intermediate to bf16; with cancellation that broke 1e-2)."""
    s = E.parse_einsum(text)
    rng = np.random.default_rng(99)
    xs = [torch.from_numpy(rng.standard_normal([ext[a] for a in t])).to(dev).bfloat16()
          for t in s.inputs]
    got = contract(text, *xs).double()
    tt = ",".join("".join(t) for t in s.inputs) + "->" + "".join(s.output)
    want = torch.einsum(tt, *[x.double() for x in xs])
    assert ((got - want).norm() / want.norm()).item() <= 1e-2


@pytest.mark.parametrize("text,ext", [
    ("(a,c,d),(b)->()", dict(a=512, c=8, d=256, b=64)),           # both operands fully private
    ("(a,c,d),(b,c,a)->()", dict(a=64, c=256, d=64, b=64)),       # 32x blow-up: pre-reduced
    ("(a,d),(c,a,b)->(c,d)", dict(c=32, d=32, a=64, b=512)),
])
def test_16bit_prereduced_private_axes_accuracy(dev, text, ext):
    """16-bit tolerance bodies whose product space is >= 16x the operands sum
    each operand over its private reduction axes first (one extra 16-bit
    rounding of the partial sums, as torch.einsum's pairwise contraction
    stores them): within 2e-2 of the f64 sum on positive data."""
    s = E.parse_einsum(text)
    g = torch.Generator(device=dev).manual_seed(5)
    xs = [torch.rand([ext[a] for a in t], generator=g, device=dev).to(torch.bfloat16) for t in s.inputs]
    executor.reset_launch_log()
    got = contract(text, *xs).double()
    kinds = executor.launch_log()
    assert len(kinds) >= 2, kinds                                    # the pre-reductions ran
    letters = {a: chr(97 + n) for n, a in enumerate(s.axes)}
    eq = ",".join("".join(letters[a] for a in t) for t in s.inputs) + "->" + \
        "".join(letters[a] for a in s.output)
    want = torch.einsum(eq, *[x.double() for x in xs])
    err = ((got - want).abs().max() / want.abs().max()).item()
    assert err <= 2e-2, err


@pytest.mark.parametrize("text,ext", [
    ("(i,k)->(i)", dict(i=300, k=517)),                  # ragged tiles, thin rows
    ("(i,k),(k)->(i)", dict(i=5000, k=200)),             # broadcast vector, 4-warp blocks
    ("(i,k),(i,k)->(i)", dict(i=64, k=1000)),
    ("(c,a,b)->(a,c)", dict(a=16, c=40, b=64)),          # transposed output rows
    ("(i,k),(i)->(i)", dict(i=700, k=96)),               # per-row factor (invariant operand)
])
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16])
def test_16bit_rows_on_staged_kernel_bit_exact(dev, text, ext, dtype):
    """16-bit row reductions now run on the staged row kernel (16-byte
    rows, f32 fold): still the reference's sequential order on the widened
    values with one final rounding — bit-equal to the oracle on f32-widened
    inputs, c0 included."""
    s = E.parse_einsum(text)
    g = torch.Generator().manual_seed(47)
    xs = [torch.randn([ext[a] for a in t], generator=g).to(dtype) for t in s.inputs]
    c0 = torch.randn([ext[a] for a in s.output], generator=g).to(dtype)
    want = np.asarray(oracle.generic(s.inputs, s.output, [x.float().numpy() for x in xs],
                                     c0.float().numpy()))
    want16 = torch.from_numpy(want.astype(np.float32)).to(dtype)
    got = contract(text, *[x.to(dev) for x in xs], c0=c0.to(dev)).cpu()
    assert torch.equal(got.view(torch.int16), want16.view(torch.int16)), text


@pytest.mark.parametrize("text,ext", [
    ("(k,i)->(i)", dict(k=300, i=8192)),            # 32 columns per warp, ragged tile
    ("(k,i),(k,i)->(i)", dict(k=100, i=1024)),      # 8 columns per warp
    ("(a,b,d)->(b,d)", dict(a=64, b=32, d=64)),
    ("(k,i),(k)->(i)", dict(k=300, i=2048)),        # shared vector, 16-byte staged
    ("(k),(k,i)->(i)", dict(k=77, i=1024)),         # shared operand first, ragged tail
    ("(b,k,i),(b,k)->(b,i)", dict(b=3, k=200, i=512)),  # shared within a warp only
])
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16])
def test_16bit_columns_on_staged_kernel_bit_exact(dev, text, ext, dtype):
    """16-bit column reductions with per-column operands run on the staged
    column-chain kernel (16-byte copies, f32 fold, one rounding): bit-equal
    to the oracle on f32-widened inputs, c0 included."""
    s = E.parse_einsum(text)
    g = torch.Generator().manual_seed(53)
    xs = [torch.randn([ext[a] for a in t], generator=g).to(dtype) for t in s.inputs]
    c0 = torch.randn([ext[a] for a in s.output], generator=g).to(dtype)
    want = np.asarray(oracle.generic(s.inputs, s.output, [x.float().numpy() for x in xs],
                                     c0.float().numpy()))
    want16 = torch.from_numpy(want.astype(np.float32)).to(dtype)
    got = contract(text, *[x.to(dev) for x in xs], c0=c0.to(dev)).cpu()
    assert torch.equal(got.view(torch.int16), want16.view(torch.int16)), text
