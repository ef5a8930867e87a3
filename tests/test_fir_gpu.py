"""GPU case study on real hardware: bridgegen FIR kernels
(vadd, the naive GEMM of SURVEY A.3, a runaway loop) translated to CUDA C,
compiled by NVRTC and launched.  CPU part: the generated source compiles for
sm_100a with nvcc; GPU part: the reference's kernel known-answer tests
(test_interp.py:256-298, test_acceptance.py:333-353) through the drop-in."""

import os
import subprocess
import sys

import numpy as np
import pytest

import _golden as G

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
bridgegen = G.import_bridgegen()   # hard failure, never a skip
from bridgegen import codegen, fir, interp, intrinsics, ir  # noqa: E402
from bridgegen.gpu import register_gpu_intrinsics  # noqa: E402

from paper_2503_04771_b200 import fir_gpu  # noqa: E402

sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
from make_golden import GEMM_FIR, VADD_FIR  # noqa: E402

LOOP_FIR = "fn f(_1: memref{f32,1})\n1:\n  goto #2\n2:\n  goto #2\n"


def pipeline(text, entry, types):
    reg = intrinsics.default_registry()
    register_gpu_intrinsics(reg)
    program = fir.parse_program(text)
    inl = fir.inline_calls(program, entry,
                           lambda name, tys: reg.has_name(name) or name == fir.BOOL_CONVERSION)
    return codegen.generate(reg, fir.insert_bool_conversions(inl), types)


MEM3 = [fir.memref_of(fir.F32, 1)] * 3


@pytest.mark.parametrize("text,entry,types", [(VADD_FIR, "vadd", MEM3), (GEMM_FIR, "gemm", MEM3),
                                              (LOOP_FIR, "f", [fir.memref_of(fir.F32, 1)])])
def test_generated_source_compiles_for_sm100a(tmp_path, text, entry, types):
    mod = pipeline(text, entry, types)
    src, kinds = fir_gpu.translate(mod.lookup_symbol(entry))
    f = tmp_path / "k.cu"
    f.write_text(src)
    r = subprocess.run(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a",
                        "--fmad=false", "-c", str(f), "-o", str(tmp_path / "k.o")],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr + src
    assert all(k[0] == "memref" for k in kinds)


def vadd_buffers():
    a = np.arange(1, 9, dtype=np.float32)
    b = np.arange(10, 90, 10, dtype=np.float32)
    c = np.zeros(8, dtype=np.float32)
    return [interp.MemRefValue(ir.F32, (8,), x) for x in (a, b, c)]


@pytest.mark.gpu
def test_vadd_known_answers(dev):
    mod = pipeline(VADD_FIR, "vadd", MEM3)
    launch = interp.LaunchConfig((2, 1, 1), (4, 1, 1))
    fwd = vadd_buffers()
    out = fir_gpu.run_kernel(mod, "vadd", launch, fwd)
    assert out[2] is fwd[2]                                   # mutated in place
    assert np.array_equal(fwd[2].data, np.array([11, 22, 33, 44, 55, 66, 77, 88], np.float32))
    rev = vadd_buffers()
    fir_gpu.run_kernel(mod, "vadd", launch, rev, reverse=True)
    assert np.array_equal(rev[2].data, fwd[2].data)
    k = G.kernel_cases()
    assert np.array_equal(fwd[2].data, k["vadd_c"])


@pytest.mark.gpu
def test_out_of_bounds_message_matches_reference(dev):
    mod = pipeline(VADD_FIR, "vadd", MEM3)
    with pytest.raises(interp.OutOfBounds, match="index 8 out of bounds") as ei:
        fir_gpu.run_kernel(mod, "vadd", interp.LaunchConfig((3, 1, 1), (4, 1, 1)), vadd_buffers())
    ref_bufs = vadd_buffers()
    with pytest.raises(interp.OutOfBounds) as er:
        interp.run_kernel(mod, "vadd", interp.LaunchConfig((3, 1, 1), (4, 1, 1)), ref_bufs)
    assert str(ei.value) == str(er.value)
    # reversed visiting order: the first offending coordinate is the last thread
    with pytest.raises(interp.OutOfBounds) as ei2:
        fir_gpu.run_kernel(mod, "vadd", interp.LaunchConfig((3, 1, 1), (4, 1, 1)),
                           vadd_buffers(), reverse=True)
    with pytest.raises(interp.OutOfBounds) as er2:
        interp.run_kernel(mod, "vadd", interp.LaunchConfig((3, 1, 1), (4, 1, 1)),
                          vadd_buffers(), reverse=True)
    assert str(ei2.value) == str(er2.value)


@pytest.mark.gpu
def test_case_study_gemm_kernel_bit_exact(dev):
    """the naive one-thread-per-output FIR GEMM, n = 8 (golden
    from the reference's simulated grid) and n = 64 (vs the oracle)."""
    import oracle
    mod = pipeline(GEMM_FIR, "gemm", MEM3)
    k = G.kernel_cases()
    n = 8
    bufs = [interp.MemRefValue(ir.F32, (n * n,), x.copy())
            for x in (k["fir_gemm_a"], k["fir_gemm_b"], np.zeros(n * n, np.float32))]
    fir_gpu.run_kernel(mod, "gemm", interp.LaunchConfig((n, 1, 1), (n, 1, 1)), bufs)
    assert np.array_equal(bufs[2].data, k["fir_gemm_c"])
    n = 64
    rng = np.random.default_rng(3)
    A = rng.standard_normal(n * n).astype(np.float32)
    B = rng.standard_normal(n * n).astype(np.float32)
    bufs = [interp.MemRefValue(ir.F32, (n * n,), x) for x in (A.copy(), B.copy(), np.zeros(n * n, np.float32))]
    fir_gpu.run_kernel(mod, "gemm", interp.LaunchConfig((n, 1, 1), (n, 1, 1)), bufs)
    assert np.array_equal(bufs[2].data.reshape(n, n), oracle.gemm_kseq(A.reshape(n, n), B.reshape(n, n)))


@pytest.mark.gpu
def test_runaway_kernel_hits_step_budget(dev):
    mod = pipeline(LOOP_FIR, "f", [fir.memref_of(fir.F32, 1)])
    buf = [interp.MemRefValue(ir.F32, (4,), np.zeros(4, np.float32))]
    with pytest.raises(interp.StepLimitExceeded, match="step budget of 1000"):
        fir_gpu.run_kernel(mod, "f", interp.LaunchConfig((64, 1, 1), (128, 1, 1)), buf,
                           step_limit=1000)


@pytest.mark.gpu
def test_compat_installs_run_kernel(dev):
    from paper_2503_04771_b200 import compat
    mod = pipeline(VADD_FIR, "vadd", MEM3)
    with compat.backend():
        assert interp.run_kernel is fir_gpu.run_kernel
        bufs = vadd_buffers()
        interp.run_kernel(mod, "vadd", interp.LaunchConfig((2, 1, 1), (4, 1, 1)), bufs)
        assert np.array_equal(bufs[2].data, np.array([11, 22, 33, 44, 55, 66, 77, 88], np.float32))
    assert interp.run_kernel is not fir_gpu.run_kernel


def _outcome(fn):
    try:
        fn()
    except interp.InterpError as e:
        return type(e).__name__, str(e)
    return None, None


@pytest.mark.gpu
@pytest.mark.parametrize("reverse", [False, True])
def test_many_failing_threads_report_reference_first(dev, reverse):
    """more failing coordinates than error-record slots (4792 here
    vs 1024) must still report the reference's first offending coordinate
    in its visiting order, with its thread context."""
    mod = pipeline(VADD_FIR, "vadd", MEM3)
    launch = interp.LaunchConfig((600, 1, 1), (8, 1, 1))
    got = _outcome(lambda: fir_gpu.run_kernel(mod, "vadd", launch, vadd_buffers(), reverse=reverse))
    want = _outcome(lambda: interp.run_kernel(mod, "vadd", launch, vadd_buffers(), reverse=reverse))
    assert want[0] == "OutOfBounds" and got == want


@pytest.mark.gpu
@pytest.mark.parametrize("reverse", [False, True])
def test_step_budget_vs_out_of_bounds_order(dev, reverse):
    """Tick-then-execute per op (interp.py:231-233): for every budget, the
    error kind and message equal the reference's (an OOB access and an
    overrun inside the same block)."""
    mod = pipeline(VADD_FIR, "vadd", MEM3)
    launch = interp.LaunchConfig((3, 1, 1), (4, 1, 1))
    seen = set()
    for limit in range(1, 40):
        got = _outcome(lambda: fir_gpu.run_kernel(mod, "vadd", launch, vadd_buffers(),
                                                  step_limit=limit, reverse=reverse))
        want = _outcome(lambda: interp.run_kernel(mod, "vadd", launch, vadd_buffers(),
                                                  step_limit=limit, reverse=reverse))
        assert got == want, limit
        seen.add(want[0])
    assert seen == {"StepLimitExceeded", "OutOfBounds"}
