"""Oracle pinned at the FULL BASELINE sizes of configs 1 and 2 against
outputs of the reference itself (tests/golden/make_fullsize_golden.py ran
bridgegen's run_function on the whole 256^3 matmul and both 2^26-element
permutations): the C restatement reproduces C1 bit-for-bit and the
transposition oracle reproduces the reference's permutation digests."""

import numpy as np
import pytest

import _golden as G
import oracle


def test_oracle_c1_bit_exact_at_full_size():
    a, b = G.fullsize_inputs("c1")
    want = G.fullsize_c1()
    got = oracle.generic([("i", "j"), ("j", "k")], ("i", "k"), [a, b],
                         np.zeros((256, 256), np.float32))
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    assert G.sha256(want) == G.fullsize_meta()["configs"]["c1"]["out_sha256"]


@pytest.mark.parametrize("config,perm", [("c2a", (1, 0)), ("c2b", (2, 1, 0))])
def test_transpose_oracle_matches_reference_digest(config, perm):
    [x] = G.fullsize_inputs(config)
    meta = G.fullsize_meta()["configs"][config]
    out = np.ascontiguousarray(x.transpose(perm))
    assert list(out.shape) == meta["out_shape"]
    assert G.sha256(out) == meta["out_sha256"]
