"""Drop-in backend for an installed ``bridgegen``: route its evaluator's
``linalg.generic`` execution to the B200.

The reference has no backend plugin API — ``_Machine.execute`` dispatches the
op name ``"linalg.generic"`` straight to ``self._generic(op, env)``
(/root/reference/pkg/src/bridgegen/interp.py:351-352).  ``install()`` replaces
that one method; everything else (parsing, IR building, verification, the
function-call machinery, error types) stays the reference's own.  A bridgegen
user switches backends with two lines::

    import paper_2503_04771_b200.compat as bgx_compat
    bgx_compat.install()          # bridgegen.interp now runs generics on the GPU

The replacement keeps ``_generic``'s contract (interp.py:372-424):
  * the same operand checks and InterpError messages ("one indexing map per
    operand required", "operands must be tensor values", "map/operand rank
    mismatch", "inconsistent extent for axis dN: a vs b", "no operand
    constrains axis dN");
  * a FRESH result TensorValue, the output operand never mutated (interp.py:399);
  * the step budget charged as the reference's loop would tick it (one per
    body op per iteration point), raising the reference's StepLimitExceeded;
  * results bit-identical to the reference for its f32/f64 types (the
    reference's exact-rounding kernels: bgx_generic / SIMT exact GEMM /
    bgx_permute).
Bodies other than the einsum bodies of einsum.py:100-118 (passthrough, or
mulf-chain + addf into the output) raise InterpError — there is no CPU
fallback.
"""

from __future__ import annotations

import contextlib

import numpy as np
import torch

from . import executor
from .einsum import EinsumSpec
from .schedule import as_schedule_dict

_saved = {}


def _interp_module():
    from bridgegen import interp  # noqa: WPS433 (the reference, installed by the user)
    return interp


def classify_body(block, n_in: int) -> str:
    """'permute' | 'contract' for the einsum bodies of einsum.py:100-118,
    checking the SSA wiring, not just the op names."""
    ops = list(block.operations)
    args = list(block.arguments)
    names = [o.name for o in ops]
    if names == ["linalg.yield"] and n_in == 1 and ops[0].operands == [args[0]]:
        return "permute"
    if len(ops) != n_in + 1 or names[-1] != "linalg.yield":
        return ""
    if names[:-1] != ["arith.mulf"] * (n_in - 1) + ["arith.addf"]:
        return ""
    acc = args[0]
    for k in range(1, n_in):
        mul = ops[k - 1]
        if mul.operands != [acc, args[k]]:
            return ""
        acc = mul.results[0]
    add = ops[n_in - 1]
    if add.operands != [acc, args[n_in]]:
        return ""
    if ops[-1].operands != [add.results[0]]:
        return ""
    return "contract"


def _generic_b200(self, op, env):
    interp = _interp_module()
    maps = list(op.attributes["indexing_maps"].elements)
    operands = [env[v] for v in op.operands]
    if len(maps) != len(operands):
        raise interp.InterpError("linalg.generic: one indexing map per operand required")
    n_axes = maps[0].n_axes if maps else 0
    extents = {}
    for which, (m, v) in enumerate(zip(maps, operands)):
        if not isinstance(v, interp.TensorValue):
            raise interp.InterpError("linalg.generic operands must be tensor values")
        if m.n_axes != n_axes or len(m.targets) != v.data.ndim:
            raise interp.InterpError(
                f"linalg.generic: map/operand rank mismatch on operand {which}")
        for d, axis in enumerate(m.targets):
            e = v.data.shape[d]
            if axis in extents and extents[axis] != e:
                raise interp.InterpError(
                    f"linalg.generic: inconsistent extent for axis d{axis}: "
                    f"{extents[axis]} vs {e}")
            extents[axis] = e
    missing = [a for a in range(n_axes) if a not in extents]
    if missing:
        raise interp.InterpError(f"linalg.generic: no operand constrains axis d{missing[0]}")
    n_in = len(operands) - 1
    block = op.regions[0].blocks[0]
    kind = classify_body(block, n_in)
    out_targets = tuple(maps[-1].targets)
    if kind == "permute" and set(out_targets) != set(range(n_axes)):
        kind = ""  # passthrough with a reduction axis: not an einsum body
    if not kind or len(set(out_targets)) != len(out_targets) or any(
            len(set(m.targets)) != len(m.targets) for m in maps):
        raise interp.InterpError(
            "linalg.generic: body/maps not supported by the B200 backend "
            "(einsum bodies of einsum.py:100-118 only)")
    # step budget, charged as the reference loop would tick (interp.py:232)
    points = 1
    for a in range(n_axes):
        points *= extents[a]
    self.steps += points * len(block.operations)
    if self.steps > self.step_limit:
        raise interp.StepLimitExceeded(f"step budget of {self.step_limit} operations exceeded")
    name = [f"d{a}" for a in range(n_axes)]
    spec_out = tuple(name[a] for a in out_targets)
    spec_in = tuple(tuple(name[a] for a in m.targets) for m in maps[:-1])
    red = tuple(name[a] for a in range(n_axes) if a not in out_targets)
    spec = EinsumSpec(spec_in, spec_out, spec_out + red)
    out = operands[-1]
    dev = torch.device("cuda", torch.cuda.current_device())
    tens = [torch.from_numpy(np.ascontiguousarray(v.data)).to(dev) for v in operands]
    res = torch.empty(tuple(out.data.shape), dtype=tens[-1].dtype, device=dev)
    sched_attr = op.attributes.get("bgx.schedule")
    sched = as_schedule_dict(getattr(sched_attr, "text", sched_attr)) if sched_attr else None
    executor.execute(spec, tens[:-1], tens[-1], res, mode=_saved.get("mode", "auto"),
                     schedule=sched)
    result = res.cpu().numpy()
    env[op.results[0]] = interp.TensorValue(out.elem, result.shape, result)
    return None


def install(mode: str = "auto", kernels: bool = True) -> None:
    """Route ``bridgegen.interp._Machine._generic`` to libbgx.so.  ``mode``:
    'auto' (bit-exact for f32/f64), 'exact', 'ffma', 'tc', 'simt'.  With
    ``kernels`` also replace ``interp.run_kernel`` (the simulated thread grid,
    interp.py:434-461) by real NVRTC-compiled launches (fir_gpu.run_kernel)."""
    from . import fir_gpu
    interp = _interp_module()
    if "orig" not in _saved:
        _saved["orig"] = interp._Machine._generic
        _saved["orig_run_kernel"] = interp.run_kernel
    _saved["mode"] = mode
    interp._Machine._generic = _generic_b200
    if kernels:
        interp.run_kernel = fir_gpu.run_kernel


def uninstall() -> None:
    if "orig" in _saved:
        interp = _interp_module()
        interp._Machine._generic = _saved.pop("orig")
        interp.run_kernel = _saved.pop("orig_run_kernel")


def installed() -> bool:
    try:
        return _interp_module()._Machine._generic is _generic_b200
    except ImportError:
        return False


@contextlib.contextmanager
def backend(mode: str = "auto"):
    """``with compat.backend(): ...`` — install for the duration of a block."""
    was = installed()
    install(mode)
    try:
        yield
    finally:
        if not was:
            uninstall()
