"""Planner (host logic, CPU): kernel-variant choice and group flattening."""

import pytest

import _golden as G
from paper_2503_04771_b200 import plan as P
from paper_2503_04771_b200.einsum import parse_einsum


def cstrides(shape):
    st, acc = [], 1
    for e in reversed(shape):
        st.append(acc)
        acc *= e
    return tuple(reversed(st))


def plan_of(text, ext, dtype="bf16", mode="auto", strides=None, **kw):
    spec = parse_einsum(text)
    shapes = [tuple(ext[a] for a in t) for t in (*spec.inputs, spec.output)]
    strides = strides or [cstrides(s) for s in shapes]
    return P.plan_generic(spec, shapes, strides, dtype=dtype, mode=mode, **kw)


def test_permutation():
    p = plan_of("(i,j,k)->(k,j,i)", dict(i=2, j=3, k=4), dtype="f32")
    assert isinstance(p, P.PermutePlan) and p.perm == (2, 1, 0)


def test_baseline_gemm_groups():
    p = plan_of("(i,k),(k,j)->(i,j)", dict(i=4096, j=4096, k=4096))
    assert isinstance(p, P.GemmPlan)
    assert (p.batch, p.M, p.N, p.K) == (1, 4096, 4096, 4096)
    assert p.a_view.strides == (0, 4096, 1) and p.b_view.strides == (0, 4096, 1)
    assert p.flops == 2 * 4096 ** 3
    p = plan_of("(b,i,j),(b,j,k)->(b,i,k)", dict(b=64, i=1024, j=1024, k=1024))
    assert (p.batch, p.M, p.N, p.K) == (64, 1024, 1024, 1024)
    assert p.a_view.strides == (1024 * 1024, 1024, 1)


def test_role_swap_for_transposed_output():
    p = plan_of("(i,k),(k,j)->(j,i)", dict(i=8, j=16, k=4))
    assert (p.a, p.b) == (1, 0) and p.m_axes == ("j",) and p.n_axes == ("i",)
    assert p.o_view.strides == (0, 8, 1)


def test_multi_axis_groups_flatten_or_copy():
    p = plan_of("(i,k,l),(k,l,j)->(i,j)", dict(i=4, j=6, k=3, l=5))
    assert p.K == 15 and p.k_axes == ("k", "l") and not p.a_view.needs_copy
    # reduction order (k, l) = the reference's lexicographic order (einsum.py:81)
    # axes (i, j, l, k): the reference reduces l outer, k inner
    p = plan_of("(i,l,k),(k,l,j)->(i,j)", dict(i=4, j=6, k=3, l=5))
    assert p.k_axes == ("l", "k") and not p.a_view.needs_copy and p.b_view.needs_copy


def test_generic_fallbacks():
    assert isinstance(plan_of("(i,j)->(i)", dict(i=3, j=4), dtype="f32"), P.GenericPlan)
    assert isinstance(plan_of("(i,j),(i,j)->(i,j)", dict(i=3, j=4), dtype="f32"), P.GenericPlan)
    assert isinstance(plan_of("(i,k),(k)->()", dict(i=3, k=4), dtype="f32"), P.GenericPlan)
    assert isinstance(plan_of("(i,j),(j,k),(k,l)->(i,l)", dict(i=2, j=3, k=2, l=4), dtype="f32"),
                      P.GenericPlan)


def test_chain_orders_c5():
    ext = dict(i=32768, k=8192, j=8192, l=8192)
    left = plan_of("(i,k),(k,j),(j,l)->(i,l)", ext)
    assert isinstance(left, P.ChainPlan) and left.flops == 8_796_093_022_208
    opt = plan_of("(i,k),(k,j),(j,l)->(i,l)", ext, chain_order="optimal")
    assert opt.flops == 5_497_558_138_880
    assert left.steps[0].out_axes == ("i", "j") and left.steps[1].out_axes == ("i", "l")


def test_every_golden_spec_plans():
    for name, text, ins, init, want in G.generic_cases():
        spec = parse_einsum(text)
        shapes = [x.shape for x in ins] + [init.shape]
        strides = [cstrides(s) for s in shapes]
        p = P.plan_generic(spec, shapes, strides, dtype="f32")
        assert p.kind in ("permute", "generic", "gemm"), name


def test_inconsistent_extent():
    spec = parse_einsum("(i,k),(k,j)->(i,j)")
    with pytest.raises(ValueError, match="inconsistent"):
        P.plan_generic(spec, [(4, 3), (2, 5), (4, 5)], [(3, 1), (5, 1), (5, 1)], dtype="f32")


def test_reference_dtypes_stay_exact_at_any_size():
    """'auto' on f32/f64 must keep the reference's unfactored loop
    nest (bit-exact) however many points; pairwise chains only on request."""
    ext = dict(i=1024, k=1024, j=1024, l=1024)   # 2^40 points > GENERIC_POINT_LIMIT
    for dt in ("f32", "f64"):
        for mode in ("auto", "exact"):
            p = plan_of("(i,k),(k,j),(j,l)->(i,l)", ext, dtype=dt, mode=mode)
            assert isinstance(p, P.GenericPlan) and "exact loop nest" in p.reason
        for mode in ("tf32", "ffma"):
            assert isinstance(plan_of("(i,k),(k,j),(j,l)->(i,l)", ext, dtype=dt, mode=mode),
                              P.ChainPlan)
    assert isinstance(plan_of("(i,k),(k,j),(j,l)->(i,l)", ext, dtype="bf16"), P.ChainPlan)


@pytest.mark.parametrize("dtype", ["bf16", "f16", "f32", "f64"])
@pytest.mark.parametrize("text", ["(i,j),(i,j)->(i,j)", "(i,j),(i,j),(i,j)->(i,j)",
                                  "(b,i),(b,i)->(b,i)", "(i,j),(j)->(i,j)"])
def test_hadamard_bodies_are_elementwise_not_gemm(text, dtype):
    """Round 2: 16-bit Hadamard bodies planned as a batch x 1 x 1 x 1 GEMM
    (8192^2 bf16 took 2 s); every dtype now takes the elementwise kernels."""
    p = plan_of(text, dict(i=8192, j=8192, b=8, k=1), dtype=dtype)
    assert isinstance(p, P.GenericPlan), p
