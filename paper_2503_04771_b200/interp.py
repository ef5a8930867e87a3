"""``run_function`` for einsum modules — drop-in mirror of bridgegen's
evaluator entry point (/root/reference/pkg/src/bridgegen/interp.py:427-431)
with every ``linalg.generic`` executed on the B200 through libbgx.so.

Kept from the reference (same names, argument meaning, error types/messages):
  * ``InterpError``, ``StepLimitExceeded`` (interp.py:39-44),
    ``DEFAULT_STEP_LIMIT`` (interp.py:36);
  * ``TensorValue(elem, dims, data)`` (interp.py:97-104);
  * ``run_function(module, symbol, inputs, step_limit, thread_ctx)``: symbol
    lookup, arity and per-argument type checks (interp.py:211-221, 156-169),
    extent inference with "inconsistent extent" (interp.py:379-396), a FRESH
    result with the output operand untouched (interp.py:399);
  * the step budget: charged exactly as the reference's loop nest would tick
    (one per function-level op, plus one per body op per iteration point,
    interp.py:232), so ``StepLimitExceeded`` fires for the same inputs.  Pass
    ``step_limit=None`` to disable the budget (the GPU has no runaway loop).

Device residency: numpy inputs are copied to the device once per call and the
result copied back; torch CUDA tensors stay on the device, and intermediate
SSA values of multi-generic functions never leave it.
"""

from __future__ import annotations

from dataclasses import dataclass
import threading

import numpy as np
import torch

from . import executor
from .einsum import BF16, F16, F32, F64, ElemType, Module, TensorType, elem_type
from .schedule import as_schedule_dict

__all__ = ["InterpError", "StepLimitExceeded", "DEFAULT_STEP_LIMIT", "TensorValue",
           "run_function"]

DEFAULT_STEP_LIMIT = 10 ** 7


class InterpError(Exception):
    pass


class StepLimitExceeded(InterpError):
    pass


_NP = {F32: np.float32, F64: np.float64, F16: np.float16}
_TORCH = {F32: torch.float32, F64: torch.float64, BF16: torch.bfloat16, F16: torch.float16}


def _np_bf16():
    try:
        import ml_dtypes  # noqa: F401  (optional: host-side bf16 arrays)
        return np.dtype("bfloat16")
    except Exception:  # pragma: no cover
        return None


@dataclass
class TensorValue:
    """Runtime tensor (interp.py:97-104).  ``data`` is a row-major numpy array
    (host) or a torch CUDA tensor (device-resident)."""
    elem: ElemType
    dims: tuple
    data: object

    def __post_init__(self):
        self.elem = elem_type(self.elem)
        if isinstance(self.data, torch.Tensor):
            want = _TORCH[self.elem]
            if self.data.dtype != want:
                raise InterpError(f"tensor dtype {self.data.dtype} does not match {self.elem}")
            if tuple(self.data.shape) != tuple(self.dims):
                self.data = self.data.reshape(tuple(self.dims))
        else:
            npd = _NP.get(self.elem) or _np_bf16()
            if npd is None:
                raise InterpError(f"no host dtype for {self.elem}; pass a torch tensor")
            self.data = np.asarray(self.data, dtype=npd).reshape(tuple(self.dims))
        self.dims = tuple(self.data.shape)


def _check_arg(t: TensorType, v, where: str):
    ok = isinstance(v, TensorValue) and v.elem == t.elem and len(v.dims) == t.rank
    if not ok:
        raise InterpError(f"{where}: value {v!r} does not match type {t}")


def _to_device(v: TensorValue, device) -> torch.Tensor:
    if isinstance(v.data, torch.Tensor):
        if not v.data.is_cuda:
            return v.data.to(device)
        return v.data
    arr = v.data
    if arr.dtype == _np_bf16():
        return torch.from_numpy(arr.view(np.uint16).copy()).view(torch.bfloat16).to(device)
    return torch.from_numpy(np.ascontiguousarray(arr)).to(device)


def _to_host(t: torch.Tensor, elem: ElemType) -> np.ndarray:
    if elem == BF16:
        bf = _np_bf16()
        return t.view(torch.int16).cpu().numpy().view(bf)
    return t.cpu().numpy()


_replay = threading.local()


def _replay_key(module, symbol, inputs, mode, device, schedule):
    """Signature of a device-resident call (None when the call does not
    qualify): everything the interpreter's checks and plans depend on."""
    sig = []
    for v in inputs:
        if type(v) is not TensorValue or not isinstance(v.data, torch.Tensor) or not v.data.is_cuda:
            return None
        sig.append((v.elem, v.dims, v.data.device))
    sk = schedule if schedule is None or isinstance(schedule, str) else repr(schedule)
    return (id(module), symbol, mode, device, sk, tuple(sig))


def run_function(module: Module, symbol: str, inputs, step_limit=DEFAULT_STEP_LIMIT,
                 thread_ctx=None, *, mode: str = "auto", device=None, schedule=None):
    """Execute ``@symbol`` on ``inputs`` (list of TensorValue); returns the
    list of result TensorValues.  ``mode`` selects the kernel class for
    contractions ('auto', 'exact', 'ffma', 'tc', 'simt' — see bgx.h);
    'auto' is bit-exact with the reference for f32/f64 inputs.

    A device-resident call whose signature (module, symbol, element types,
    shapes, devices, mode, schedule) already ran to completion replays the
    recorded op sequence without re-deriving extents and step counts — the
    checks would pass again and the step count is a function of the shapes,
    so the replay is taken only when that count fits ``step_limit``."""
    inputs = list(inputs)
    key = _replay_key(module, symbol, inputs, mode, device, schedule)
    cache = getattr(_replay, "d", None)
    if cache is None:
        cache = _replay.d = {}
    if key is not None:
        hit = cache.get(key)
        if hit is not None and hit[0] is module and (step_limit is None or hit[1] <= step_limit):
            return hit[2](inputs)
    results, steps, replay = _run_function(module, symbol, inputs, step_limit, mode, device,
                                           schedule)
    if key is not None and replay is not None:
        if len(cache) > 64:
            cache.clear()
        cache[key] = (module, steps, replay)
    return results


def _run_function(module, symbol, inputs, step_limit, mode, device, schedule):
    fn = module.lookup_symbol(symbol)
    if fn is None:
        raise InterpError(f"no function @{symbol} in the module")
    inputs = list(inputs)
    if len(inputs) != len(fn.arguments):
        raise InterpError(
            f"@{symbol} takes {len(fn.arguments)} argument(s), got {len(inputs)}")
    for i, (arg, v) in enumerate(zip(fn.arguments, inputs)):
        _check_arg(arg.type, v, f"@{symbol} argument {i}")
    if device is None:
        device = next((v.data.device for v in inputs
                       if isinstance(v.data, torch.Tensor) and v.data.is_cuda),
                      torch.device("cuda", torch.cuda.current_device()))
    host_io = any(not isinstance(v.data, torch.Tensor) for v in inputs)
    env = {id(a): v for a, v in zip(fn.arguments, inputs)}
    dev = {}
    steps = 0
    plan = []

    def tick(n=1):
        nonlocal steps
        steps += n
        if step_limit is not None and steps > step_limit:
            raise StepLimitExceeded(f"step budget of {step_limit} operations exceeded")

    def device_of(val):
        key = id(val)
        if key not in dev:
            dev[key] = _to_device(env[key], device)
        return dev[key]

    for op in fn.ops:
        tick()
        vals = [env[id(v)] for v in op.operands]
        extents = {}
        for which, (m, v) in enumerate(zip(op.maps, vals)):
            if len(m.targets) != len(v.dims):
                raise InterpError(
                    f"linalg.generic: map/operand rank mismatch on operand {which}")
            for d, axis in enumerate(m.targets):
                e = v.dims[d]
                if axis in extents and extents[axis] != e:
                    raise InterpError(
                        f"linalg.generic: inconsistent extent for axis d{axis}: "
                        f"{extents[axis]} vs {e}")
                extents[axis] = e
        points = 1
        for a in range(op.maps[0].n_axes if op.maps else 0):
            points *= extents[a]
        tick(points * len(op.body))
        tensors = [device_of(v) for v in op.operands]
        out_t = torch.empty(tuple(vals[-1].dims), dtype=_TORCH[op.elem], device=device)
        with executor._on_device(device):
            sched = as_schedule_dict(op.schedule if op.schedule is not None else schedule)
            executor.execute(op.spec, tensors[:-1], tensors[-1], out_t, mode=mode,
                             schedule=sched)
        res = op.results[0]
        env[id(res)] = TensorValue(op.elem, tuple(out_t.shape), out_t)
        dev[id(res)] = out_t
        plan.append((op, tuple(vals[-1].dims), _TORCH[op.elem], sched))
    tick()  # func.return
    results = []
    for v in fn.returns:
        tv = env[id(v)]
        if host_io and isinstance(tv.data, torch.Tensor):
            tv = TensorValue(tv.elem, tv.dims, _to_host(tv.data, tv.elem))
        results.append(tv)
    replay = None
    if not host_io:
        args, rets = fn.arguments, fn.returns

        def replay(new_inputs):
            env2 = {id(a): v.data for a, v in zip(args, new_inputs)}
            with executor._on_device(device):
                for op, dims, dtype, sch in plan:
                    ts = [env2[id(x)] for x in op.operands]
                    o = torch.empty(dims, dtype=dtype, device=device)
                    executor.execute(op.spec, ts[:-1], ts[-1], o, mode=mode, schedule=sch)
                    env2[id(op.results[0])] = o
            return [TensorValue(elem_of[id(v)], tuple(env2[id(v)].shape), env2[id(v)])
                    for v in rets]
        elem_of = {id(v): env[id(v)].elem for v in rets}
        if not all(isinstance(env[id(v)].data, torch.Tensor) for v in rets):
            replay = None
        else:
            replay = _direct_replay(fn, plan, env, dev, mode, device, replay) or replay
    return results, steps, replay


def _fresh_value(elem, dims, data) -> TensorValue:
    """TensorValue for a tensor this module just allocated with the right
    dtype and shape (skips the constructor's conversions)."""
    v = object.__new__(TensorValue)
    v.elem, v.dims, v.data = elem, dims, data
    return v


def _direct_replay(fn, plan, env, dev, mode, device, general):
    """Replay of a one-op function whose op ran through a cached launcher
    (``executor.fast_launcher``: a pre-built descriptor, pointers patched per
    call): per call only the operand layout is re-checked (strides and
    16-byte alignment — the replay key already fixed shapes, dtypes and
    devices), the fresh result allocated and the launcher called.  Anything
    else (several ops, a different layout) takes the general replay."""
    if len(plan) != 1 or len(fn.returns) != 1:
        return None
    op, dims, dtype, sch = plan[0]
    if sch or fn.returns[0] is not op.results[0]:
        return None
    pos = {id(a): i for i, a in enumerate(fn.arguments)}
    if not all(id(x) in pos for x in op.operands):
        return None
    idx = [pos[id(x)] for x in op.operands]
    ts = [dev[id(x)] for x in op.operands]
    out_t = dev[id(op.results[0])]
    fast = executor.fast_launcher(op.spec, ts[:-1], ts[-1], out_t, mode)
    if fast is None:
        return None
    sig = [(t.stride(), t.data_ptr() % 16) for t in ts]
    elem = env[id(op.results[0])].elem
    n_in = len(idx) - 1

    def replay(new_inputs):
        xs = [new_inputs[i].data for i in idx]
        for t, (st, al) in zip(xs, sig):
            if t.stride() != st or t.data_ptr() % 16 != al:
                return general(new_inputs)
        o = torch.empty(dims, dtype=dtype, device=device)
        fast(xs[:n_in], o, xs[n_in])
        return [_fresh_value(elem, dims, o)]
    return replay
