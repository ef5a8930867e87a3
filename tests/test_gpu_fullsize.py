"""BASELINE configs 1 and 2 at FULL size on the B200 against the reference's
own outputs (tests/golden/fullsize_*: bridgegen run_function on the whole
problem): C1 256^3 f32 bit-identical through the reference-shaped API, C2a /
C2b permutations byte-identical (SHA-256 of the output)."""

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
