"""Pin the CPU oracle to the reference (no GPU needed).

The fixtures in tests/golden/ were produced by bridgegen itself
(tests/golden/make_golden.py); the oracle must reproduce them bit-for-bit.
When /root/reference is present (build container) the oracle is also
cross-checked live against bridgegen on fresh random specs.
"""

import os
import random
import sys

import numpy as np
import pytest

import _golden as G
import oracle

CASES = G.generic_cases()


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_oracle_matches_reference_fixtures(case):
    name, text, ins, init, want = case
    i, o = G.split_spec(text)
    assert G.bits_equal(oracle.generic(i, o, ins, init), want), name


def test_kseq_restatement_equals_generic():
    rng = np.random.default_rng(0)
    a = rng.standard_normal((3, 17, 33), dtype=np.float32)
    b = rng.standard_normal((3, 33, 9), dtype=np.float32)
    c = rng.standard_normal((3, 17, 9), dtype=np.float32)
    g1 = oracle.gemm_kseq(a, b, c)
    g2 = oracle.generic([("b", "i", "k"), ("b", "k", "j")], ("b", "i", "j"), [a, b], c)
    assert np.array_equal(g1, g2)
    # np.matmul is NOT the reference's arithmetic (different summation order)
    assert not np.array_equal(g1, np.matmul(a, b) + c)


def test_kseq_row_range_and_strided_operands():
    rng = np.random.default_rng(1)
    a = rng.standard_normal((40, 64), dtype=np.float32)
    bt = rng.standard_normal((24, 64), dtype=np.float32)  # B given transposed (strided view)
    full = oracle.gemm_kseq(a, bt.T)
    part = oracle.gemm_kseq(a, bt.T, rows=(10, 20))
    assert np.array_equal(part[10:20], full[10:20])
    assert not part[:10].any() and not part[20:].any()
    assert np.array_equal(full, oracle.generic([("i", "k"), ("k", "j")], ("i", "j"),
                                               [a, bt.T], np.zeros((40, 24), np.float32)))


def test_case_study_gemm_kernel_known_answer():
    """the naive FIR GEMM kernel run by bridgegen's
    simulated grid equals the einsum oracle bit-for-bit."""
    k = G.kernel_cases()
    n = 8
    assert np.array_equal(k["fir_gemm_c"].reshape(n, n), k["fir_gemm_einsum"])
    got = oracle.gemm_kseq(k["fir_gemm_a"].reshape(n, n), k["fir_gemm_b"].reshape(n, n))
    assert np.array_equal(got, k["fir_gemm_einsum"])
    assert np.array_equal(k["vadd_c"], np.array([11, 22, 33, 44, 55, 66, 77, 88], np.float32))


def test_output_range_sampling():
    rng = np.random.default_rng(2)
    ins = [rng.standard_normal(s, dtype=np.float32) for s in ((6, 5), (5, 4), (4, 3))]
    spec = ([("i", "k"), ("k", "j"), ("j", "l")], ("i", "l"))
    full = oracle.generic(*spec, ins, np.zeros((6, 3), np.float32))
    part = oracle.generic(*spec, ins, np.zeros((6, 3), np.float32), out_range=(4, 11))
    assert np.array_equal(part.reshape(-1)[4:11], full.reshape(-1)[4:11])


def test_chain_f64_close_to_exact():
    rng = np.random.default_rng(3)
    a, b, c = (rng.standard_normal(s, dtype=np.float32) for s in ((12, 10), (10, 9), (9, 7)))
    exact = oracle.generic([("i", "k"), ("k", "j"), ("j", "l")], ("i", "l"), [a, b, c],
                           np.zeros((12, 7), np.float32))
    f64 = oracle.chain_f64(a, b, c, slice(0, 12))
    assert oracle.rel_frobenius(exact, f64) < 1e-5


REF = "/root/reference/pkg/src"


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference not mounted (GPU box)")
def test_oracle_live_against_reference():
    sys.path.insert(0, REF)
    try:
        from bridgegen import einsum, interp, intrinsics, ir
        from bridgegen.gpu import register_gpu_intrinsics
    finally:
        sys.path.remove(REF)
    reg = intrinsics.default_registry()
    register_gpu_intrinsics(reg)
    r = random.Random(777)
    nr = np.random.default_rng(777)
    letters = ["i", "j", "k", "l", "m"]
    done = 0
    while done < 25:
        ins = [tuple(r.sample(letters, r.randint(1, 3))) for _ in range(r.randint(1, 3))]
        used = sorted({x for t in ins for x in t})
        out = tuple(r.sample(used, r.randint(0, min(3, len(used)))))
        text = ",".join("(" + ",".join(t) + ")" for t in ins) + "->(" + ",".join(out) + ")"
        spec = einsum.parse_einsum(text)
        ext = {a: r.randint(1, 5) for a in spec.axes}
        arrs = [nr.standard_normal(tuple(ext[x] for x in t)).astype(np.float32) for t in spec.inputs]
        init = nr.standard_normal(tuple(ext[x] for x in spec.output)).astype(np.float32)
        mod = einsum.build_einsum_function(reg, spec)
        vals = [interp.TensorValue(ir.F32, x.shape, x) for x in arrs + [init]]
        [ref] = interp.run_function(mod, "einsum", vals)
        got = oracle.generic(spec.inputs, spec.output, arrs, init)
        assert G.bits_equal(got, ref.data), text
        done += 1
