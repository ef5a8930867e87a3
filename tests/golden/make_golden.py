"""Generate tests/golden/*.npz + parse_golden.json by RUNNING THE REFERENCE.

Run in the build container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports ``bridgegen`` from /root/reference/pkg/src (or baseline/_ref) and
records inputs and the reference evaluator's outputs
(``interp.run_function`` → ``_Machine._generic``, interp.py:372-424) for the
cases the reference's own tests use, replaying their seeds and RNG call order:

  * test_interp.py:218-232   matmul 4x3·3x5, default_rng(11)
  * test_interp.py:244-253   accumulate-from-initial (ones, C0 = 10 -> 12)
  * test_einsum.py:104-119   (i,j),(j,k),(k,l)->(i,l), default_rng(2)
  * test_einsum.py:169-202   chained generics (a@b)@b, default_rng(4)
  * test_interp.py:301-339   12 random specs, Random(5)/default_rng(5)
  * test_acceptance.py:281-330  criterion 8: matmul + 20 specs, seed 88
  * test_interp.py:256-298 / test_acceptance.py:333-353  vadd known answers
  * SURVEY Appendix A.3      naive FIR GEMM kernel via run_kernel, n = 8
plus extra cases this repo needs (permutations with IEEE specials, f64, batch,
beta != 0, reductions, Hadamard/outer products, the BASELINE configs'
index patterns at small extents).  The GPU tests load these fixtures; nothing
at test time reads /root/reference.
"""

from __future__ import annotations

import json
import os
import random
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
for cand in ("/root/reference/pkg/src",
             os.path.join(HERE, "..", "..", "baseline", "_ref")):
    if os.path.isdir(os.path.join(cand, "bridgegen")):
        sys.path.insert(0, cand)
        break

from bridgegen import codegen, einsum, fir, interp, intrinsics, ir  # noqa: E402
from bridgegen.gpu import register_gpu_intrinsics  # noqa: E402


def registry():
    reg = intrinsics.default_registry()
    register_gpu_intrinsics(reg)
    return reg


REG = registry()


def run_ref(text, inputs, out, elem=fir.F32, step_limit=10 ** 9):
    spec = einsum.parse_einsum(text)
    module = einsum.build_einsum_function(REG, spec, elem=elem)
    e = ir.F32 if elem == fir.F32 else ir.F64
    vals = [interp.TensorValue(e, x.shape, x) for x in inputs]
    vals.append(interp.TensorValue(e, out.shape, out))
    [got] = interp.run_function(module, "einsum", vals, step_limit=step_limit)
    return got.data


CASES = []  # (name, spec, inputs, out_init, result)


def add(name, text, inputs, out, elem=fir.F32):
    res = run_ref(text, inputs, out, elem)
    CASES.append((name, text, inputs, out, np.array(res, copy=True)))


def random_spec(rng, variant):
    """Replays the random-spec generators of test_interp.py:323-339
    (variant 'interp') and test_acceptance.py:316-330 ('acceptance')."""
    letters = ["i", "j", "k", "l"]
    while True:
        inputs = []
        if variant == "interp":
            n_inputs = rng.randint(1, 3)
            for _ in range(n_inputs):
                rank = rng.randint(1, 3)
                inputs.append(tuple(rng.sample(letters, rank)))
            used = [n for tup in inputs for n in tup]
            out_rank = rng.randint(0, min(3, len(set(used))))
            output = tuple(rng.sample(sorted(set(used)), out_rank))
        else:
            for _ in range(rng.randint(1, 3)):
                inputs.append(tuple(rng.sample(letters, rng.randint(1, 3))))
            used = sorted({n for tup in inputs for n in tup})
            output = tuple(rng.sample(used, rng.randint(0, min(3, len(used)))))
        text = ",".join("(" + ",".join(t) + ")" for t in inputs)
        text += "->(" + ",".join(output) + ")"
        try:
            return einsum.parse_einsum(text), text
        except einsum.EinsumError:
            continue


def reference_suites():
    # test_interp.py:218-232
    rng = np.random.default_rng(11)
    a = rng.random((4, 3)).astype(np.float32)
    b = rng.random((3, 5)).astype(np.float32)
    add("interp_matmul_seed11", "(i,k),(k,j)->(i,j)", [a, b], np.zeros((4, 5), np.float32))
    # test_interp.py:244-253
    add("interp_accumulate", "(i,k),(k,j)->(i,j)",
        [np.ones((2, 2), np.float32), np.ones((2, 2), np.float32)],
        np.full((2, 2), 10.0, np.float32))
    # test_einsum.py:104-119
    rng = np.random.default_rng(2)
    a = rng.random((2, 3)).astype(np.float32)
    b = rng.random((3, 2)).astype(np.float32)
    c = rng.random((2, 4)).astype(np.float32)
    add("einsum_triple_seed2", "(i,j),(j,k),(k,l)->(i,l)", [a, b, c],
        np.zeros((2, 4), np.float32))
    # test_einsum.py:169-202 — two chained generics = two reference calls
    rng = np.random.default_rng(4)
    a = rng.random((3, 3)).astype(np.float32)
    b = rng.random((3, 3)).astype(np.float32)
    zero = np.zeros((3, 3), np.float32)
    t = run_ref("(i,k),(k,j)->(i,j)", [a, b], zero)
    add("einsum_chained_seed4_step2", "(i,k),(k,j)->(i,j)", [np.array(t), b], zero)
    CASES.append(("einsum_chained_seed4_step1", "(i,k),(k,j)->(i,j)", [a, b], zero, np.array(t)))
    # test_interp.py:301-339
    r = random.Random(5)
    nr = np.random.default_rng(5)
    for n in range(12):
        spec, text = random_spec(r, "interp")
        extents = {name: r.randint(1, 4) for name in spec.axes}
        ins = [nr.random(tuple(extents[x] for x in tup)).astype(np.float32) for tup in spec.inputs]
        out = np.zeros(tuple(extents[x] for x in spec.output), np.float32)
        add(f"interp_random_seed5_{n:02d}", text, ins, out)
    # test_acceptance.py:281-330
    r = random.Random(88)
    nr = np.random.default_rng(88)
    a = nr.random((4, 3)).astype(np.float32)
    b = nr.random((3, 5)).astype(np.float32)
    add("crit8_matmul_seed88", "(i,k),(k,j)->(i,j)", [a, b], np.zeros((4, 5), np.float32))
    for n in range(20):
        spec, text = random_spec(r, "acceptance")
        extents = {name: r.randint(1, 5) for name in spec.axes}
        ins = [nr.random(tuple(extents[x] for x in tup)).astype(np.float32) for tup in spec.inputs]
        out = np.zeros(tuple(extents[x] for x in spec.output), np.float32)
        add(f"crit8_random_seed88_{n:02d}", text, ins, out)


def extra_cases():
    rng = np.random.default_rng(1234)
    f = lambda *s: rng.standard_normal(s).astype(np.float32)  # noqa: E731
    # permutations incl. IEEE specials (quiet NaN, +-inf, -0, subnormals)
    x = f(64, 64)
    x.flat[[0, 5, 77, 130, 999]] = [np.inf, -np.inf, -0.0, np.float32(1e-40), np.nan]
    add("perm_ij_ji_64", "(i,j)->(j,i)", [x], np.zeros((64, 64), np.float32))
    add("perm_ijk_kji_16", "(i,j,k)->(k,j,i)", [f(16, 16, 16)], np.zeros((16, 16, 16), np.float32))
    add("perm_ijk_kij_odd", "(i,j,k)->(k,i,j)", [f(5, 33, 7)], np.zeros((7, 5, 33), np.float32))
    add("perm_copy_rank1", "(i)->(i)", [f(37)], np.full((37,), 3.0, np.float32))
    add("perm_rank4", "(a,b,c,d)->(d,b,a,c)", [f(3, 4, 5, 6)], np.zeros((6, 4, 3, 5), np.float32))
    # C1 index pattern at small extents, with beta != 0
    add("c1_matmul_32_48_40_beta", "(i,j),(j,k)->(i,k)", [f(32, 48), f(48, 40)], f(32, 40))
    # C3 pattern
    add("c3_batched_3x8x16x12", "(b,i,j),(b,j,k)->(b,i,k)", [f(3, 8, 16), f(3, 16, 12)],
        np.zeros((3, 8, 12), np.float32))
    # C5 pattern (unfactored 3-operand loop nest)
    add("c5_chain_6x5x4x3", "(i,k),(k,j),(j,l)->(i,l)", [f(6, 5), f(5, 4), f(4, 3)],
        np.zeros((6, 3), np.float32))
    # transposed operands / output
    add("matmul_tn", "(k,i),(k,j)->(i,j)", [f(9, 7), f(9, 5)], np.zeros((7, 5), np.float32))
    add("matmul_nt_out_t", "(i,k),(j,k)->(j,i)", [f(7, 9), f(5, 9)], np.zeros((5, 7), np.float32))
    # reductions, Hadamard, outer, rank-0
    add("reduce_rows", "(i,j)->(i)", [f(7, 11)], np.zeros((7,), np.float32))
    add("reduce_all", "(i,j)->()", [f(7, 11)], np.array(0.5, np.float32))
    add("hadamard", "(i,j),(i,j)->(i,j)", [f(6, 5), f(6, 5)], f(6, 5))
    add("outer", "(i),(j)->(i,j)", [f(6), f(5)], np.zeros((6, 5), np.float32))
    add("dot", "(k),(k)->()", [f(50), f(50)], np.array(0.0, np.float32))
    add("multi_reduce", "(i,k,l),(k,l,j)->(i,j)", [f(4, 3, 5), f(3, 5, 6)], np.zeros((4, 6), np.float32))
    # float64
    g = lambda *s: rng.standard_normal(s)  # noqa: E731
    add("f64_matmul", "(i,k),(k,j)->(i,j)", [g(9, 13), g(13, 6)], g(9, 6), elem=fir.F64)
    add("f64_perm", "(i,j)->(j,i)", [g(8, 3)], np.zeros((3, 8)), elem=fir.F64)
    add("f64_triple", "(i,j),(j,k),(k,l)->(i,l)", [g(3, 4), g(4, 2), g(2, 5)], np.zeros((3, 5)), elem=fir.F64)


GEMM_FIR = """\
fn gemm(_1: memref{f32,1}, _2: memref{f32,1}, _3: memref{f32,1})
1:
  %1 = invoke block_idx_x() :: index
  %2 = invoke thread_idx_x() :: index
  %3 = invoke block_dim_x() :: index
  goto #2
2:
  %4 = phi (#1 => 0, #3 => %10) :: index
  %5 = phi (#1 => 0.0, #3 => %9) :: f32
  %6 = invoke <(%4, %3) :: i1
  goto #4 ifnot %6
3:
  %11 = invoke *(%1, %3) :: index
  %12 = invoke +(%11, %4) :: index
  %13 = invoke load(_1, %12) :: f32
  %14 = invoke *(%4, %3) :: index
  %15 = invoke +(%14, %2) :: index
  %16 = invoke load(_2, %15) :: f32
  %17 = invoke *(%13, %16) :: f32
  %9 = invoke +(%17, %5) :: f32
  %10 = invoke +(%4, 1) :: index
  goto #2
4:
  %18 = invoke *(%1, %3) :: index
  %19 = invoke +(%18, %2) :: index
  %20 = invoke store(%5, _3, %19) :: Nothing
  return
"""

VADD_FIR = """\
fn vadd(_1: memref{f32,1}, _2: memref{f32,1}, _3: memref{f32,1})
1:
  %1 = invoke block_idx_x() :: index
  %2 = invoke block_dim_x() :: index
  %3 = invoke *(%1, %2) :: index
  %4 = invoke thread_idx_x() :: index
  %5 = invoke +(%3, %4) :: index
  %6 = invoke load(_1, %5) :: f32
  %7 = invoke load(_2, %5) :: f32
  %8 = invoke +(%6, %7) :: f32
  %9 = invoke store(%8, _3, %5) :: Nothing
  return
"""


def pipeline(text, entry):
    program = fir.parse_program(text)
    fn = program.functions[entry]
    inl = fir.inline_calls(program, entry,
                           lambda name, types: REG.has_name(name) or name == fir.BOOL_CONVERSION)
    conv = fir.insert_bool_conversions(inl)
    return codegen.generate(REG, conv, [fir.memref_of(fir.F32, 1)] * 3)


def kernel_cases():
    """GPU case study: vadd and the naive GEMM kernel."""
    out = {}
    vadd = pipeline(VADD_FIR, "vadd")
    bufs = [interp.MemRefValue(ir.F32, (8,), x) for x in
            (np.arange(1, 9, dtype=np.float32), np.arange(10, 90, 10, dtype=np.float32),
             np.zeros(8, np.float32))]
    interp.run_kernel(vadd, "vadd", interp.LaunchConfig((2, 1, 1), (4, 1, 1)), bufs)
    out["vadd_a"], out["vadd_b"], out["vadd_c"] = (np.array(b.data) for b in bufs)
    n = 8
    rng = np.random.default_rng(7)
    A = rng.standard_normal(n * n).astype(np.float32)
    B = rng.standard_normal(n * n).astype(np.float32)
    gemm = pipeline(GEMM_FIR, "gemm")
    bufs = [interp.MemRefValue(ir.F32, (n * n,), x.copy()) for x in (A, B, np.zeros(n * n, np.float32))]
    interp.run_kernel(gemm, "gemm", interp.LaunchConfig((n, 1, 1), (n, 1, 1)), bufs)
    out["fir_gemm_a"], out["fir_gemm_b"], out["fir_gemm_c"] = A, B, np.array(bufs[2].data)
    ein = run_ref("(i,k),(k,j)->(i,j)", [A.reshape(n, n), B.reshape(n, n)], np.zeros((n, n), np.float32))
    out["fir_gemm_einsum"] = np.array(ein)
    assert np.array_equal(out["fir_gemm_c"].reshape(n, n), out["fir_gemm_einsum"])
    return out


def parse_cases():
    """Spec strings -> parse result or error message, and derived maps."""
    texts = [
        "(i,k),(k,j)->(i,j)", "(i)->(i)", "(i,j)->(k)", "(i,i)->(i)",
        "( i , k ), ( k , j ) -> ( i , j )", "(i,j)->()", "i,k->i",
        "(i,k)(k,j)->(i,j)", "(i,k)->", "->(i)", "ij,jk->ik", "(i,j),(j,k)->(i,k)",
        "(b,i,j),(b,j,k)->(b,i,k)", "(i,j,k)->(k,j,i)", "(i,k),(k,j),(j,l)->(i,l)",
        "(a,b),(b,c),(c,d)->(a,d)", "(i,j)->(j)", "(i,,j)->(i)", "(1i)->(i)",
        "(i)->(i)->(i)", "(ij,jk)->(ij)", "(i) , (j) -> (i , j)", "(_x,y2)->(y2)",
        "((i))->(i)", "(i)->(i),(j)", "", "(i,j)->(j,i) ", " (i)->(i)", "(i-j)->(i)",
    ]
    rng = random.Random(2024)
    alphabet = ["i", "j", "k", ",", "(", ")", "->", " ", "x1", "_", "(", ")"]
    for _ in range(400):
        texts.append("".join(rng.choice(alphabet) for _ in range(rng.randint(1, 14))))
    r5 = random.Random(99)
    for _ in range(200):
        texts.append(random_spec(r5, "interp")[1])
    rows = []
    for t in texts:
        try:
            spec = einsum.parse_einsum(t)
            maps, its = einsum.derive_maps(spec)
            rows.append({"text": t, "ok": True, "inputs": [list(x) for x in spec.inputs],
                         "output": list(spec.output), "axes": list(spec.axes),
                         "maps": [[m.n_axes, list(m.targets)] for m in maps],
                         "iterators": its})
        except einsum.EinsumError as e:
            rows.append({"text": t, "ok": False, "error": str(e)})
    return rows


def printed_cases():
    out = {}
    for t in ["(i,k),(k,j)->(i,j)", "(i)->(i)", "(i,j)->()", "(i,j),(j,k),(k,l)->(i,l)",
              "(i,j)->(j,i)"]:
        spec = einsum.parse_einsum(t)
        out[t + "|f32"] = ir.print_module(einsum.build_einsum_function(REG, spec))
        out[t + "|f64"] = ir.print_module(einsum.build_einsum_function(REG, spec, elem=fir.F64))
    return out


def main():
    reference_suites()
    extra_cases()
    arrays = {}
    index = []
    for name, text, ins, out, res in CASES:
        for k, x in enumerate(ins):
            arrays[f"{name}__in{k}"] = x
        arrays[f"{name}__init"] = out
        arrays[f"{name}__out"] = res
        index.append({"name": name, "spec": text, "n_in": len(ins),
                      "dtype": str(np.asarray(res).dtype)})
    np.savez_compressed(os.path.join(HERE, "generic_cases.npz"), **arrays)
    np.savez_compressed(os.path.join(HERE, "kernel_cases.npz"), **kernel_cases())
    with open(os.path.join(HERE, "generic_cases.json"), "w") as fh:
        json.dump(index, fh, indent=1)
    with open(os.path.join(HERE, "parse_golden.json"), "w") as fh:
        json.dump(parse_cases(), fh, indent=0)
    with open(os.path.join(HERE, "printed_golden.json"), "w") as fh:
        json.dump(printed_cases(), fh, indent=1)
    print(f"{len(CASES)} generic cases written")


if __name__ == "__main__":
    main()
