"""Edge cases the reference handles: empty and extent-1 axes,
empty reductions (K = 0 -> out = c0), rank-0 outputs, maximum operand count
/ axis count of the generic kernel, non-contiguous views, and errors."""

import numpy as np
import pytest
import torch

import oracle
from paper_2503_04771_b200 import contract
from paper_2503_04771_b200 import einsum as E
from paper_2503_04771_b200 import interp as I

pytestmark = pytest.mark.gpu


def run_ref_api(text, ins, init):
    mod = E.build_einsum_function(None, E.parse_einsum(text))
    vals = [I.TensorValue(E.F32, x.shape, x) for x in (*ins, init)]
    [got] = I.run_function(mod, "einsum", vals, step_limit=None)
    return got.data


def oracle_of(text, ins, init):
    s = E.parse_einsum(text)
    return oracle.generic(s.inputs, s.output, ins, init)


@pytest.mark.parametrize("text,shapes", [
    ("(i,k),(k,j)->(i,j)", [(4, 0), (0, 5), (4, 5)]),      # empty reduction: out = c0
    ("(i,k),(k,j)->(i,j)", [(0, 3), (3, 5), (0, 5)]),      # empty output
    ("(i,j)->(i)", [(6, 0), (6,)]),
    ("(i,j)->()", [(0, 4), ()]),
    ("(i,k),(k,j)->(i,j)", [(1, 1), (1, 1), (1, 1)]),
    ("(a,b,c,d,e),(e,f)->(a,b,c,d,f)", [(2, 1, 3, 1, 4), (4, 5), (2, 1, 3, 1, 5)]),
    ("(a,b),(b,c),(c,d),(d,e),(e,f),(f,g)->(a,g)",
     [(2, 3), (3, 2), (2, 3), (3, 2), (2, 2), (2, 3), (2, 3)]),  # 6 inputs (ABI max)
    ("(i)->()", [(1000,), ()]),
])
def test_edge_shapes_bit_exact(dev, text, shapes):
    rng = np.random.default_rng(0)
    arrs = [rng.standard_normal(s).astype(np.float32) for s in shapes]
    ins, init = arrs[:-1], arrs[-1]
    got = run_ref_api(text, ins, init)
    want = oracle_of(text, ins, init)
    assert got.shape == want.shape
    assert np.array_equal(got.reshape(-1).view(np.uint32), want.reshape(-1).view(np.uint32))


def test_bf16_empty_reduction_and_views(dev):
    a = torch.randn(64, 0, device=dev).bfloat16()
    b = torch.randn(0, 32, device=dev).bfloat16()
    c0 = torch.randn(64, 32, device=dev).bfloat16()
    out = contract("(i,k),(k,j)->(i,j)", a, b, c0=c0)
    assert torch.equal(out, c0)
    big = torch.randn(300, 500, device=dev).bfloat16()
    view = big[10:266:2, 100:420]          # strided rows (not TMA-legal -> copy / SIMT)
    w = torch.randn(320, 96, device=dev).bfloat16()
    got = contract("(i,k),(k,j)->(i,j)", view, w, out_dtype=torch.float32)
    want = oracle.gemm_kseq(view.float().cpu().numpy(), w.float().cpu().numpy())
    assert oracle.rel_frobenius(got.cpu().numpy(), want) <= 1e-2


def test_errors_raise_without_fallback(dev):
    with pytest.raises(ValueError, match="inconsistent extent"):
        contract("(i,k),(k,j)->(i,j)", torch.zeros(4, 3, device=dev), torch.zeros(2, 5, device=dev))
    with pytest.raises(ValueError, match="CUDA tensors only"):
        contract("(i,k),(k,j)->(i,j)", torch.zeros(4, 3), torch.zeros(3, 5))
    with pytest.raises(E.EinsumError):
        contract("ij,jk->ik", torch.zeros(4, 3, device=dev), torch.zeros(3, 5, device=dev))


def test_clock_sample_one_cta_per_sm(dev):
    """bgx_clock_sample: one record per SM (distinct smids), clocks advance and
    the derived frequency is physical."""
    from paper_2503_04771_b200 import _lib
    lib = _lib.load()
    n = lib.bgx_sm_count()
    buf = torch.zeros(2, n * 3, dtype=torch.int64, device=dev)
    st = torch.cuda.current_stream().cuda_stream
    _lib.check(lib.bgx_clock_sample(buf[0].data_ptr(), st), "clock")
    torch.cuda._sleep(50_000_000)
    _lib.check(lib.bgx_clock_sample(buf[1].data_ptr(), st), "clock")
    torch.cuda.synchronize()
    h = buf.cpu().numpy().reshape(2, n, 3)
    assert len(set(h[0, :, 0].tolist())) == n and len(set(h[1, :, 0].tolist())) == n
    import bench
    c = bench.inband_clock(buf.cpu().numpy())
    assert c["inband_sms"] == n and 200 < c["sm_mhz_inband"] < 2500


@pytest.mark.parametrize("text,shapes,dtype", [
    ("(i,j)->(i)", [(1000, 3001)], np.float32),
    ("(i,j)->(i)", [(37, 64)], np.float64),
    ("(i,j),(i,j)->(i)", [(517, 1025), (517, 1025)], np.float32),
    ("(i,j),(j)->(i)", [(300, 4097)], np.float32),
    ("(b,i,j),(b,j)->(b,i)", [(3, 100, 777), (3, 777)], np.float64),
    ("(b,i,j)->(b,i)", [(5, 64, 300)], np.float32),
    ("(i,j)->(j)", [(3001, 1000)], np.float32),
    ("(i,j)->(j)", [(64, 37)], np.float64),
    ("(i,j),(i)->(j)", [(2049, 515), (2049,)], np.float32),
    ("(b,i,j)->(b,j)", [(3, 700, 96)], np.float64),
    ("(i,j),(i,j)->(j)", [(130, 100), (130, 100)], np.float32),
    ("(i,j)->()", [(300, 301)], np.float32),
    ("(i,j),(i,j)->()", [(129, 257), (129, 257)], np.float64),
])
def test_row_reduction_kernel_bit_exact(dev, text, shapes, dtype):
    """Row reductions / matrix-vector bodies (one reduction axis, contiguous):
    staged through shared memory by the row-reduction kernel, bit-identical to
    the reference loop nest (oracle), with c0, ragged tiles and a broadcast
    vector operand."""
    spec = E.parse_einsum(text)
    rng = np.random.default_rng(sum(sum(s) for s in shapes))
    if text == "(i,j),(j)->(i)":
        shapes = [shapes[0], (shapes[0][1],)]
    if text == "(i,j),(i)->(j)":
        shapes = [shapes[0], (shapes[0][0],)]
    arrs = [rng.standard_normal(s).astype(dtype) for s in shapes]
    ext = {}
    for a, tup in zip(arrs, spec.inputs):
        ext.update(dict(zip(tup, a.shape)))
    c0 = rng.standard_normal(tuple(ext[x] for x in spec.output)).astype(dtype)
    got = contract(text, *[torch.from_numpy(a).to(dev) for a in arrs], c0=torch.from_numpy(c0).to(dev))
    want = oracle.generic(list(spec.inputs), spec.output, arrs, c0)
    uint = np.uint32 if dtype == np.float32 else np.uint64
    assert np.array_equal(got.cpu().numpy().view(uint), np.asarray(want).view(uint)), text
    # strided rows (a column slice): still one contiguous reduction axis per row
    if text == "(i,j)->(i)" and dtype == np.float32:
        big = torch.from_numpy(rng.standard_normal((1000, 4000)).astype(np.float32)).to(dev)
        sl = big[:, 500:3501]
        got2 = contract(text, sl)
        want2 = oracle.generic([("i", "j")], ("i",), [sl.cpu().numpy()], np.zeros(1000, np.float32))
        assert np.array_equal(got2.cpu().numpy().view(np.uint32), np.asarray(want2).view(np.uint32))


def test_random_specs_larger_extents_bit_exact(dev):
    """Property check over many random einsum specs with extents large
    enough to reach every f32 kernel class (row/column reductions, the loop
    nest, SIMT GEMM, permutations): every result bit-identical to the
    oracle's reference loop nest."""
    import random
    r = random.Random(20261018)
    nr = np.random.default_rng(20261018)
    letters = ["i", "j", "k", "l"]
    seen = 0
    while seen < 40:
        ins = [tuple(r.sample(letters, r.randint(1, 3))) for _ in range(r.randint(1, 2))]
        used = sorted({x for t in ins for x in t})
        out = tuple(r.sample(used, r.randint(0, min(2, len(used)))))
        text = ",".join("(" + ",".join(t) + ")" for t in ins) + "->(" + ",".join(out) + ")"
        try:
            spec = E.parse_einsum(text)
        except E.EinsumError:
            continue
        ext = {a: r.choice([1, 7, 33, 64, 97, 130]) for a in spec.axes}
        if np.prod([ext[a] for a in spec.axes]) > 4_000_000:
            continue
        arrs = [nr.standard_normal(tuple(ext[x] for x in t)).astype(np.float32) for t in spec.inputs]
        c0 = nr.standard_normal(tuple(ext[x] for x in spec.output)).astype(np.float32)
        got = contract(spec, *[torch.from_numpy(a).to(dev) for a in arrs],
                       c0=torch.from_numpy(c0).to(dev)).cpu().numpy()
        if spec.inputs == (spec.output,) or (len(spec.inputs) == 1 and set(spec.inputs[0]) == set(spec.output)):
            want = np.ascontiguousarray(arrs[0].transpose([spec.inputs[0].index(a) for a in spec.output]))
        else:
            want = np.asarray(oracle.generic(list(spec.inputs), spec.output, arrs, c0))
        assert np.array_equal(np.asarray(got).view(np.uint32), want.view(np.uint32)), (text, ext)
        seen += 1


def test_generic_fuzz_strided_views(dev):
    """Random 1-2 input bodies on strided views (transposes, slices, step
    slicing) through every f32 kernel class: bit-identical to the oracle
    evaluated on the same (materialised) values."""
    import random
    r = random.Random(777)
    nr = np.random.default_rng(777)
    letters = ["i", "j", "k"]
    done = 0
    while done < 60:
        ins = [tuple(r.sample(letters, r.randint(1, 3))) for _ in range(r.randint(1, 2))]
        used = sorted({x for t in ins for x in t})
        out = tuple(r.sample(used, r.randint(0, min(2, len(used)))))
        text = ",".join("(" + ",".join(t) + ")" for t in ins) + "->(" + ",".join(out) + ")"
        try:
            spec = E.parse_einsum(text)
        except E.EinsumError:
            continue
        ext = {a: r.choice([1, 5, 40, 70, 133]) for a in spec.axes}
        tensors, host = [], []
        for t in spec.inputs:
            shape = tuple(ext[x] for x in t)
            mode = r.choice(["plain", "transpose", "slice", "step"])
            if mode == "transpose" and len(shape) >= 2:
                base = torch.from_numpy(nr.standard_normal(shape[::-1]).astype(np.float32)).to(dev)
                x = base.permute(*reversed(range(len(shape))))
            elif mode == "slice":
                base = torch.from_numpy(nr.standard_normal(tuple(s + 3 for s in shape)).astype(np.float32)).to(dev)
                x = base[tuple(slice(1, 1 + s) for s in shape)]
            elif mode == "step":
                base = torch.from_numpy(nr.standard_normal(tuple(2 * s for s in shape)).astype(np.float32)).to(dev)
                x = base[tuple(slice(0, 2 * s, 2) for s in shape)]
            else:
                x = torch.from_numpy(nr.standard_normal(shape).astype(np.float32)).to(dev)
            tensors.append(x)
            host.append(np.ascontiguousarray(x.cpu().numpy()))
        c0 = nr.standard_normal(tuple(ext[x] for x in spec.output)).astype(np.float32)
        got = contract(spec, *tensors, c0=torch.from_numpy(c0).to(dev)).cpu().numpy()
        if len(spec.inputs) == 1 and set(spec.inputs[0]) == set(spec.output):
            want = np.ascontiguousarray(host[0].transpose([spec.inputs[0].index(a) for a in spec.output]))
        else:
            want = np.asarray(oracle.generic(list(spec.inputs), spec.output, host, c0))
        assert np.array_equal(np.asarray(got).view(np.uint32), want.view(np.uint32)), (text, ext)
        done += 1


@pytest.mark.parametrize("text,ext,dtype", [
    ("(a),(b,c,d)->()", dict(a=4, b=8, c=64, d=64), np.float32),          # broadcast operand
    ("(d,a),(d,b,c)->(a)", dict(a=8, d=64, b=32, c=32), np.float32),     # few outputs, 2 inputs
    ("(b,c,d),(b,c),(d)->()", dict(b=64, c=64, d=8), np.float32),        # 3 inputs, rank 0
    ("(c,a,b),(b,c)->(a)", dict(a=3, b=512, c=40), np.float64),          # f64, transposed walk
    ("(i,j)->(j)", dict(i=20000, j=5), np.float32),                      # strided columns
])
def test_few_outputs_long_reductions_bit_exact(dev, text, ext, dtype):
    """Block-per-output chains (chain_general_kernel): the products are formed
    by other warps in any order, the adds stay one chain in the reference's
    point order — bit-identical to the oracle, with and without c0."""
    s = E.parse_einsum(text)
    rng = np.random.default_rng(3)
    ins = [rng.standard_normal([ext[a] for a in t]).astype(dtype) for t in s.inputs]
    for with_c0 in (False, True):
        init = (rng.standard_normal([ext[a] for a in s.output]).astype(dtype) if with_c0
                else np.zeros([ext[a] for a in s.output], dtype))
        want = oracle.generic(s.inputs, s.output, ins, init)
        got = contract(text, *[torch.from_numpy(x).to(dev) for x in ins],
                       c0=torch.from_numpy(init).to(dev) if with_c0 else None).cpu().numpy()
        assert np.array_equal(got.reshape(-1).view(np.uint8), want.reshape(-1).view(np.uint8)), \
            (text, with_c0)


@pytest.mark.parametrize("text,ext", [
    ("(d,a,c),(c,d,b)->(b,c,d)", dict(b=33, c=40, d=17, a=9)),     # walk c innermost
    ("(d,b,a),(c,d,b)->(a,b,d)", dict(a=21, b=40, d=13, c=7)),     # walk b innermost
    ("(i,k),(j,k)->(j,i)", dict(i=37, j=45, k=5)),
])
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_generic_walk_order_bit_exact(dev, text, ext, dtype):
    """The per-thread loop nest walks the parallel axes with the streamed
    operands' contiguous axis innermost (not the output's): outputs land at
    their own offsets, each still one chain in the reference's order."""
    s = E.parse_einsum(text)
    rng = np.random.default_rng(5)
    ins = [rng.standard_normal([ext[a] for a in t]).astype(dtype) for t in s.inputs]
    init = rng.standard_normal([ext[a] for a in s.output]).astype(dtype)
    want = oracle.generic(s.inputs, s.output, ins, init)
    got = contract(text, *[torch.from_numpy(x).to(dev) for x in ins],
                   c0=torch.from_numpy(init).to(dev), mode="exact").cpu().numpy()
    assert np.array_equal(got.reshape(-1).view(np.uint8), want.reshape(-1).view(np.uint8))


@pytest.mark.parametrize("text,ext", [
    ("(a,b,c),(b)->(c,b,a)", dict(a=128, b=64, c=130)),      # transposed input materialised first
    ("(a,b),(b,a)->(b,a)", dict(a=1030, b=1024)),
])
def test_elementwise_transposed_operand_bit_exact(dev, text, ext):
    """No-reduction bodies over >= 2^20 outputs copy a row-walked input into
    the output's axis order first (bytes moved): still the reference's
    fl(fl(x*y) + c0) per element, signed zeros included."""
    s = E.parse_einsum(text)
    rng = np.random.default_rng(9)
    ins = [rng.standard_normal([ext[a] for a in t]).astype(np.float32) for t in s.inputs]
    ins[0].reshape(-1)[::7] = -0.0
    for init in (np.zeros([ext[a] for a in s.output], np.float32),
                 rng.standard_normal([ext[a] for a in s.output]).astype(np.float32)):
        want = oracle.generic(s.inputs, s.output, ins, init)
        got = contract(text, *[torch.from_numpy(x).to(dev) for x in ins],
                       c0=torch.from_numpy(init).to(dev)).cpu().numpy()
        assert np.array_equal(got.reshape(-1).view(np.uint32), want.reshape(-1).view(np.uint32))


def test_random_specs_round2_kernel_classes_bit_exact(dev):
    """Random bodies sized for the round-2 exact paths — block-per-output
    chains (few outputs, >= 7168 points each), the walk-ordered loop nest
    (several parallel axes with a reduction), no-reduction bodies over
    >= 2^20 outputs with row-walked inputs, matrix-vector bodies of any
    layout — every result bit-identical to the oracle."""
    import random
    r = random.Random(20261019)
    nr = np.random.default_rng(20261019)
    letters = ["a", "b", "c", "d"]
    seen = 0
    while seen < 30:
        ins = [tuple(r.sample(letters, r.randint(1, 3))) for _ in range(r.randint(1, 3))]
        used = sorted({x for t in ins for x in t})
        out = tuple(r.sample(used, r.randint(0, min(3, len(used)))))
        text = ",".join("(" + ",".join(t) + ")" for t in ins) + "->(" + ",".join(out) + ")"
        try:
            spec = E.parse_einsum(text)
        except E.EinsumError:
            continue
        if len(spec.inputs) == 1 and set(spec.inputs[0]) == set(spec.output):
            continue   # permutations are covered elsewhere
        ext = {a: r.choice([3, 16, 64, 130, 512, 1024]) for a in spec.axes}
        n_out = int(np.prod([ext[a] for a in spec.output])) if spec.output else 1
        pts = int(np.prod([ext[a] for a in spec.axes]))
        if pts > 12_000_000 or pts < 20_000:
            continue
        arrs = [nr.standard_normal(tuple(ext[x] for x in t)).astype(np.float32) for t in spec.inputs]
        c0 = nr.standard_normal(tuple(ext[x] for x in spec.output)).astype(np.float32)
        got = contract(spec, *[torch.from_numpy(a).to(dev) for a in arrs],
                       c0=torch.from_numpy(c0).to(dev), mode="exact").cpu().numpy()
        want = np.asarray(oracle.generic(list(spec.inputs), spec.output, arrs, c0))
        assert np.array_equal(np.asarray(got).view(np.uint32), want.view(np.uint32)), \
            (text, ext, n_out)
        seen += 1


@pytest.mark.parametrize("text,ext", [
    ("(i,k),(i)->(i)", dict(i=300, k=1000)),                     # per-row factor, thin rows
    ("(d,a,b),(c)->(d,c,a)", dict(d=3, c=50, a=40, b=700)),      # factor indexed by another output axis
    ("(i,k),(i)->(i)", dict(i=20000, k=130)),                    # many rows, 4-warp blocks
])
def test_row_reduction_with_invariant_factor_bit_exact(dev, text, ext):
    """Row reductions where one operand is constant along the reduction (a
    per-output factor, loaded once per lane in the staged kernel): still the
    reference's fold and order, bit for bit."""
    s = E.parse_einsum(text)
    rng = np.random.default_rng(17)
    ins = [rng.standard_normal([ext[a] for a in t]).astype(np.float32) for t in s.inputs]
    init = rng.standard_normal([ext[a] for a in s.output]).astype(np.float32)
    want = oracle.generic(s.inputs, s.output, ins, init)
    got = contract(text, *[torch.from_numpy(x).to(dev) for x in ins],
                   c0=torch.from_numpy(init).to(dev)).cpu().numpy()
    assert np.array_equal(got.reshape(-1).view(np.uint32), want.reshape(-1).view(np.uint32))


@pytest.mark.parametrize("text,ext,dtype", [
    ("(k,i)->(i)", dict(k=777, i=8192), np.float32),               # 32 columns per warp, tail tile
    ("(k,i),(k)->(i)", dict(k=1000, i=1024), np.float32),          # 8 columns per warp, shared vector
    ("(k),(k,i)->(i)", dict(k=300, i=2048), np.float32),           # shared operand first
    ("(k,i),(k,i)->(i)", dict(k=130, i=5120), np.float32),         # both operands per column
    ("(b,k,i),(b,k)->(b,i)", dict(b=3, k=500, i=512), np.float64),  # operand shared within a warp only
    ("(a,b,c)->(a,c)", dict(a=4, b=333, c=256), np.float64),
    ("(k,i)->(i)", dict(k=64, i=520), np.float32),                 # shortest staged reduction
])
def test_column_chains_bit_exact(dev, text, ext, dtype):
    """Column sums and vector-matrix products on the staged column-chain
    kernel (16-byte copies, 8 or 32 adjacent columns per warp): every output's
    chain runs the reference's order, bit for bit, with c0."""
    s = E.parse_einsum(text)
    rng = np.random.default_rng(23)
    ins = [rng.standard_normal([ext[a] for a in t]).astype(dtype) for t in s.inputs]
    init = rng.standard_normal([ext[a] for a in s.output]).astype(dtype)
    want = np.asarray(oracle.generic(s.inputs, s.output, ins, init))
    got = contract(text, *[torch.from_numpy(x).to(dev) for x in ins],
                   c0=torch.from_numpy(init).to(dev)).cpu().numpy()
    uint = np.uint32 if dtype == np.float32 else np.uint64
    assert np.array_equal(got.reshape(-1).view(uint), want.reshape(-1).view(uint)), text


def test_column_chains_unaligned_view_bit_exact(dev):
    """A column slice starting off a 16-byte boundary cannot be staged with
    16-byte copies: the planner's other exact path takes it, same bits."""
    rng = np.random.default_rng(29)
    big = torch.from_numpy(rng.standard_normal((700, 4100)).astype(np.float32)).to(dev)
    for lo in (1, 4):
        sl = big[:, lo:lo + 4096]
        got = contract("(k,i)->(i)", sl).cpu().numpy()
        want = np.asarray(oracle.generic([("k", "i")], ("i",), [sl.cpu().numpy()], np.zeros(4096, np.float32)))
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), lo


@pytest.mark.parametrize("text,ext,dtype", [
    ("(d,b,a)->(a)", dict(d=300, b=8, a=1024), np.float32),        # (d,b) merge: one column chain axis
    ("(d,b,a)->(a)", dict(d=100, b=8, a=1024), np.float64),
    ("(d,b,a)->(d)", dict(d=256, b=64, a=64), np.float32),          # (b,a) merge: row chains
    ("(a,b,c),(c)->(a,b)", dict(a=16, b=64, c=300), np.float32),   # (a,b) parallel merge
    ("(j,l,k)->(l,j)", dict(j=7, l=7, k=1), np.float32),           # every reduction axis unit
    ("(a,k,b),(k)->(a,b)", dict(a=1, k=1, b=40), np.float64),      # unit axes of both kinds
    ("(a,c,b),(b,a),(b)->(b)", dict(a=64, c=256, b=256), np.float32),  # block-per-output gathers
])
def test_coalesced_axes_bit_exact(dev, text, ext, dtype):
    """Neighbouring axes every input walks as one are merged (and unit axes
    dropped) before kernel selection; the merged walk visits the reduction
    points in the reference's order, so results stay bit-identical, c0
    included."""
    s = E.parse_einsum(text)
    rng = np.random.default_rng(31)
    ins = [rng.standard_normal([ext[a] for a in t]).astype(dtype) for t in s.inputs]
    init = rng.standard_normal([ext[a] for a in s.output]).astype(dtype)
    want = np.asarray(oracle.generic(s.inputs, s.output, ins, init))
    got = contract(text, *[torch.from_numpy(x).to(dev) for x in ins],
                   c0=torch.from_numpy(init).to(dev)).cpu().numpy()
    uint = np.uint32 if dtype == np.float32 else np.uint64
    assert np.array_equal(got.reshape(-1).view(uint), want.reshape(-1).view(uint)), text


@pytest.mark.parametrize("text,ext", [
    ("(c),(a,c),(b)->(c,a,b)", dict(c=8, a=64, b=512)),   # two broadcasts and a row vector
    ("(a),(b)->(a,b)", dict(a=300, b=1024)),              # outer product
    ("(a,b),(b)->(a,b)", dict(a=33, b=4096)),             # row scaling
    ("(b,a),(b)->(a,b)", dict(a=128, b=256)),             # transposed (strided) operand
])
@pytest.mark.parametrize("dtype", [torch.float32, torch.float64, torch.bfloat16])
def test_broadcast_elementwise_bit_exact(dev, text, ext, dtype):
    """Elementwise bodies with broadcast / strided operands run V outputs per
    thread with 16-byte stores (bcast_ew_kernel): the same per-element
    arithmetic as the loop nest (product, then + c0), checked bit for bit
    against the oracle (f32/f64) and against the loop nest itself (bf16)."""
    s = E.parse_einsum(text)
    g = torch.Generator().manual_seed(37)
    ins = [torch.randn([ext[a] for a in t], generator=g, dtype=torch.float64).to(dtype) for t in s.inputs]
    init = torch.randn([ext[a] for a in s.output], generator=g, dtype=torch.float64).to(dtype)
    got = contract(text, *[x.to(dev) for x in ins], c0=init.to(dev)).cpu()
    if dtype == torch.bfloat16:
        # reference arithmetic for 16-bit elementwise bodies: f32 products and add, one rounding
        ref = _ew_f32(s, ext, [x.float() for x in ins]) + init.float()
        assert torch.equal(got, ref.to(torch.bfloat16)), text
    else:
        want = np.asarray(oracle.generic(s.inputs, s.output, [x.numpy() for x in ins], init.numpy()))
        uint = np.uint32 if dtype == torch.float32 else np.uint64
        assert np.array_equal(got.numpy().reshape(-1).view(uint), want.reshape(-1).view(uint)), text


def _ew_f32(s, ext, xs):
    """Left-fold product of the operands broadcast to the output axes, in f32."""
    out = None
    for t, x in zip(s.inputs, xs):
        perm = [t.index(a) for a in s.output if a in t]
        y = x.permute(*perm) if perm else x
        shape = [ext[a] if a in t else 1 for a in s.output]
        y = y.reshape(shape)
        out = y if out is None else out * y
    return out.expand([ext[a] for a in s.output])


@pytest.mark.parametrize("text,ext,dtype", [
    ("(b,a,c),(c,a)->(b)", dict(b=300, a=32, c=64), np.float32),           # operand transposed vs the walk
    ("(d,a,c),(c,a),(c)->(d)", dict(d=200, a=8, c=160), np.float64),       # three operands, 1280-point chains
    ("(b,a,c),(c,a)->(b)", dict(b=64, a=33, c=37), np.float32),            # ragged last tile
])
def test_block_chains_for_uncoalesced_walks_bit_exact(dev, text, ext, dtype):
    """Reductions the row / column kernels cannot take and the per-thread
    loop nest cannot coalesce run as block-per-output chains (producer warps
    read each output's points contiguously, one thread folds them in order):
    bit-identical to the reference order, c0 included."""
    s = E.parse_einsum(text)
    rng = np.random.default_rng(41)
    ins = [rng.standard_normal([ext[a] for a in t]).astype(dtype) for t in s.inputs]
    init = rng.standard_normal([ext[a] for a in s.output]).astype(dtype)
    want = np.asarray(oracle.generic(s.inputs, s.output, ins, init))
    got = contract(text, *[torch.from_numpy(x).to(dev) for x in ins],
                   c0=torch.from_numpy(init).to(dev)).cpu().numpy()
    uint = np.uint32 if dtype == np.float32 else np.uint64
    assert np.array_equal(got.reshape(-1).view(uint), want.reshape(-1).view(uint)), text


def test_cached_transposed_elementwise_repeat_calls_bit_exact(dev):
    """A repeated elementwise signature whose input is materialised in the
    output's axis order runs from the cached launcher (copy + one launch);
    every call sees its own data, bit for bit."""
    g = torch.Generator(device=dev).manual_seed(43)
    outs = torch.empty(2048, 1024, device=dev)
    for _ in range(3):
        x = torch.randn(1024, 2048, device=dev, generator=g)
        v = torch.randn(1024, device=dev, generator=g)
        got = contract("(b,c),(b)->(c,b)", x, v, out=outs)
        want = (x * v[:, None]).t() + 0.0
        assert torch.equal(got, want)
