"""Torch-facing entry point: ``contract(spec, *tensors)`` on CUDA tensors.

This is the device-resident form of the reference's einsum path
(bridgegen einsum.build_einsum_function + interp.run_function,
einsum.py:164-191 / interp.py:427-431): same spec language, same semantics
(``out = c0 + sum prod``, passthrough for a lone all-parallel input), but
operands are torch CUDA tensors that stay in HBM, 16-bit inputs run on the
tcgen05 tensor cores with f32 accumulation, and the output dtype may be
widened to f32.
"""

from __future__ import annotations

import torch

from . import executor
from .einsum import EinsumSpec, parse_einsum
from .plan import extents_of


def output_shape(spec: EinsumSpec, operands) -> tuple:
    ext = {}
    for t, tup in zip(operands, spec.inputs):
        if t.dim() != len(tup):
            raise ValueError(f"operand rank {t.dim()} does not match index tuple {tup}")
        for e, n in zip(t.shape, tup):
            if n in ext and ext[n] != e:
                raise ValueError(f"inconsistent extent for index {n}: {ext[n]} vs {e}")
            ext[n] = int(e)
    return tuple(ext[n] for n in spec.output)


def contract(spec, *operands: torch.Tensor, out: torch.Tensor | None = None,
             c0: torch.Tensor | None = None, out_dtype: torch.dtype | None = None,
             mode: str = "auto", schedule: dict | None = None,
             chain_order: str = "left") -> torch.Tensor:
    """Evaluate an einsum spec such as ``"(i,k),(k,j)->(i,j)"`` on CUDA tensors.

    ``c0``: initial output (the reference's output operand; None = zeros).
    ``out``: optional preallocated result (may alias nothing else).
    ``mode``: 'auto' | 'exact' | 'ffma' | 'tc' | 'simt' (include/bgx.h).
    ``chain_order``: 'left' or 'optimal' pairwise order for 3+ inputs."""
    if not isinstance(spec, EinsumSpec):
        spec = parse_einsum(spec)
    if len(operands) != len(spec.inputs):
        raise ValueError(f"expected {len(spec.inputs)} input(s), got {len(operands)}")
    shape = output_shape(spec, operands)
    dt = out_dtype or operands[0].dtype
    if out is None:
        out = torch.empty(shape, dtype=dt, device=operands[0].device)
    elif tuple(out.shape) != shape:
        raise ValueError(f"out shape {tuple(out.shape)} != {shape}")
    if out.dtype != operands[0].dtype:
        # widened output (16-bit in, f32 out): only the GEMM path supports it
        return _contract_widened(spec, operands, c0, out, mode, schedule)
    extents_of(spec, [t.shape for t in operands] + [out.shape])
    return executor.execute(spec, list(operands), c0, out, mode=mode, schedule=schedule,
                            chain_order=chain_order)


def _contract_widened(spec, operands, c0, out, mode, schedule):
    from .plan import GemmPlan
    plan = executor.plan_for(spec, list(operands), out, mode=mode)
    if not isinstance(plan, GemmPlan):
        raise NotImplementedError("a widened output dtype needs a 2-input contraction")
    return executor.run_gemm(plan, spec, list(operands), c0, out, mode=mode, schedule=schedule)


def contract_host(spec, *host_operands: torch.Tensor, out: torch.Tensor | None = None,
                  device=None, **kw) -> torch.Tensor:
    """Host-buffer form of ``contract`` (what a numpy/CPU caller of the
    reference API pays for): copies the operands host→device on the current
    stream (async when they are pinned), runs the contraction on the device,
    and copies the result back into ``out`` (a host tensor; pinned for an
    async copy) or a fresh host tensor.  Synchronises before returning."""
    device = torch.device(device) if device is not None else torch.device(
        "cuda", torch.cuda.current_device())
    dev_ops = [t.to(device, non_blocking=True) for t in host_operands]
    c0 = kw.pop("c0", None)
    if c0 is not None:
        c0 = c0.to(device, non_blocking=True)
    res = contract(spec, *dev_ops, c0=c0, **kw)
    if out is None:
        out = torch.empty(res.shape, dtype=res.dtype, pin_memory=True)
    out.copy_(res, non_blocking=True)
    torch.cuda.current_stream(device).synchronize()
    return out
