"""``python -m paper_2503_04771_b200.cli einsum`` against bridgegen's einsum
subcommand (cli.py:286-322): same printed module, same shape-check and spec
error messages and exit codes; ``--run`` executes on the GPU (gpu marker)."""

import subprocess
import sys

import pytest

import _golden as G
from paper_2503_04771_b200 import cli


def run_cli(*argv, capsys):
    rc = cli.main(list(argv))
    out, err = capsys.readouterr()
    return rc, out, err


def test_prints_reference_module(capsys):
    rc, out, err = run_cli("einsum", "(i,k),(k,j)->(i,j)", capsys=capsys)
    assert rc == 0 and err == ""
    assert out == G.printed_cases()["(i,k),(k,j)->(i,j)|f32"]


@pytest.mark.parametrize("shapes,msg", [
    ("4x3,3x5", "3 operand shape(s) expected, got 2"),
    ("4x3,3,4x5", "shape (3,) does not match index tuple ('k', 'j')"),
    ("4x3,4x5,4x5", "index 'k' has inconsistent extents 3 and 4"),
    ("4xa,3x5,4x5", "bad shape '4xa'"),
])
def test_shape_errors_match_reference(capsys, shapes, msg):
    rc, out, err = run_cli("einsum", "(i,k),(k,j)->(i,j)", "--shapes", shapes, capsys=capsys)
    assert rc == 1 and out == ""
    assert err == f"error: {msg}\n"


def test_spec_error_and_usage(capsys):
    rc, _, err = run_cli("einsum", "ij,jk->ik", capsys=capsys)
    assert rc == 1 and err.startswith("error: ")
    rc, _, _ = run_cli("einsum", capsys=capsys)
    assert rc == 2


def test_out_file_and_schedule(tmp_path, capsys):
    path = tmp_path / "m.mlir"
    rc, out, _ = run_cli("einsum", "(i,k),(k,j)->(i,j)", "--elem", "bf16", "--schedule",
                         "tile_n=256,cta_group=2", "--out", str(path), capsys=capsys)
    assert rc == 0 and out == ""
    text = path.read_text()
    assert 'bgx.schedule = "tile_n=256,cta_group=2"' in text and "bf16" in text


def test_module_entry_point():
    r = subprocess.run([sys.executable, "-m", "paper_2503_04771_b200.cli", "einsum", "(i)->(i)"],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "linalg.generic" in r.stdout


@pytest.mark.gpu
def test_run_on_gpu(dev, capsys):
    import json
    rc, out, err = run_cli("einsum", "(i,k),(k,j)->(i,j)", "--shapes", "256x512,512x384,256x384",
                           "--elem", "bf16", "--run", capsys=capsys)
    assert rc == 0, err
    summary = json.loads(out.strip().splitlines()[-1])
    assert summary["out_shape"] == [256, 384] and summary["kernels"][0].startswith("tcgen05")
    rc, out, _ = run_cli("einsum", "(i,j)->(j,i)", "--shapes", "64x32,32x64", "--run",
                         capsys=capsys)
    assert json.loads(out.strip().splitlines()[-1])["kernels"] == ["permute"]
