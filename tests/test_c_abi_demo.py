"""The C ABI from plain C (examples/c_abi_demo.c, gcc + include/bgx.h +
libbgx.so, no Python or torch in the process): compiled here on CPU, run on
the B200 (bit-identical GEMM, byte-exact permute, reference-order row sums)."""

import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CUDA = "/usr/local/cuda"


def _build(tmp_path):
    exe = str(tmp_path / "c_abi_demo")
    cmd = ["gcc", "-O2", "-std=c11", "-Wall", "-I", os.path.join(ROOT, "include"),
           "-I", os.path.join(CUDA, "include"), os.path.join(ROOT, "examples", "c_abi_demo.c"),
           "-L", os.path.join(ROOT, "paper_2503_04771_b200"), "-lbgx",
           "-L", os.path.join(CUDA, "lib64"), "-lcudart",
           "-Wl,-rpath," + os.path.join(ROOT, "paper_2503_04771_b200"),
           "-Wl,-rpath," + os.path.join(CUDA, "lib64"), "-o", exe]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_c_demo_compiles_against_the_header(tmp_path):
    _build(tmp_path)


@pytest.mark.gpu
def test_c_demo_runs(dev, tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "c_abi_demo ok" in r.stdout
