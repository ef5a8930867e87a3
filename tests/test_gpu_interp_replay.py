"""run_function's replay of a device-resident signature that already ran
(interp._replay): same results as the first (full) evaluation, fresh output
tensors every call, new data honoured, and the step budget still enforced
exactly as the reference does (interp.py:205-209)."""

import numpy as np
import pytest
import torch

import oracle
from paper_2503_04771_b200 import einsum as E
from paper_2503_04771_b200 import executor
from paper_2503_04771_b200 import interp as I

pytestmark = pytest.mark.gpu


def _vals(dev, seed, shapes=((64, 48), (48, 40), (64, 40))):
    g = torch.Generator(device=dev).manual_seed(seed)
    return [I.TensorValue(E.F32, s, torch.randn(s, device=dev, generator=g)) for s in shapes]


def test_replay_matches_full_run_and_allocates_fresh_outputs(dev):
    mod = E.build_einsum_function(None, E.parse_einsum("(i,j),(j,k)->(i,k)"))
    vals = _vals(dev, 1)
    I._replay.d = {}
    [first] = I.run_function(mod, "einsum", vals, step_limit=None)
    assert len(I._replay.d) == 1
    executor.reset_launch_log()
    [again] = I.run_function(mod, "einsum", vals, step_limit=None)        # replay
    assert executor.launch_log() == ["simt-exact"]
    assert torch.equal(first.data, again.data) and first.data.data_ptr() != again.data.data_ptr()
    a, b, c = (v.data.cpu().numpy() for v in vals)
    assert np.array_equal(again.data.cpu().numpy(), oracle.gemm_kseq(a, b, c))
    new = _vals(dev, 2)                                                    # same signature, new data
    [res] = I.run_function(mod, "einsum", new, step_limit=None)
    a, b, c = (v.data.cpu().numpy() for v in new)
    assert np.array_equal(res.data.cpu().numpy(), oracle.gemm_kseq(a, b, c))
    assert res.dims == (64, 40) and res.elem == E.F32


def test_replay_respects_step_limit(dev):
    mod = E.build_einsum_function(None, E.parse_einsum("(i,j),(j,k)->(i,k)"))
    vals = _vals(dev, 3)
    I._replay.d = {}
    I.run_function(mod, "einsum", vals, step_limit=None)                   # cache entry
    need = 2 + 3 * 64 * 48 * 40          # 3 steps per point + 2 per call
    with pytest.raises(I.StepLimitExceeded):
        I.run_function(mod, "einsum", vals, step_limit=need - 1)
    [ok] = I.run_function(mod, "einsum", vals, step_limit=need)
    assert ok.dims == (64, 40)


def test_replay_keyed_by_module_and_signature(dev):
    m1 = E.build_einsum_function(None, E.parse_einsum("(i,j),(j,k)->(i,k)"))
    m2 = E.build_einsum_function(None, E.parse_einsum("(i,j),(j,k)->(k,i)"))
    vals = _vals(dev, 4)
    vals2 = vals[:2] + [I.TensorValue(E.F32, (40, 64), torch.zeros(40, 64, device=dev))]
    I._replay.d = {}
    [y1] = I.run_function(m1, "einsum", vals, step_limit=None)
    [y2] = I.run_function(m2, "einsum", vals2, step_limit=None)
    [y1b] = I.run_function(m1, "einsum", vals, step_limit=None)
    [y2b] = I.run_function(m2, "einsum", vals2, step_limit=None)
    assert torch.equal(y1.data, y1b.data) and torch.equal(y2.data, y2b.data)
    a, b = (v.data.cpu().numpy() for v in vals[:2])
    assert np.array_equal(y2.data.cpu().numpy(), oracle.gemm_kseq(a, b).T)   # m2 from zeros
    with pytest.raises(I.InterpError):                          # wrong rank still rejected
        I.run_function(m1, "einsum", vals[:2] + [I.TensorValue(E.F32, (64,), torch.zeros(64, device=dev))],
                       step_limit=None)
