"""Multi-GPU execution: one process per GPU, torch.distributed
for the plumbing.

* M-sharding (``row_range`` + ``contract`` on the local slab): contractions
  with a free M or batch index split their output rows into contiguous slabs,
  one per rank; the other operands are replicated.  No collective on the data
  path — each rank's output slab is final.  Used for the 3-operand chain
  (``(A_r @ B) @ C`` per rank) and the batched / plain GEMMs.
* K-split (``ksplit_contract``): for large-K / small-MN contractions each rank
  takes a K slab, produces f32 partial sums with the tcgen05 kernel, and the
  partials are reduced with one NCCL collective over NVLink
  (``reduce_scatter_tensor`` when the output rows divide by the world size,
  else ``all_reduce``); the reduced f32 tile is cast (and c0 added) by
  ``bgx_cast_f32``.  That collective is the only data exchange anywhere in
  the framework.
"""

from __future__ import annotations

import torch
import torch.distributed as dist

from . import _lib, executor
from .api import contract
from .einsum import EinsumSpec, parse_einsum


def row_range(total: int, world: int, rank: int, align: int = 128):
    """Contiguous, ``align``-multiple slab of ``total`` rows for ``rank``
    (the last rank takes the remainder)."""
    if world <= 1:
        return 0, total
    units = (total + align - 1) // align
    per, extra = divmod(units, world)
    start = rank * per + min(rank, extra)
    stop = start + per + (1 if rank < extra else 0)
    return min(total, start * align), min(total, stop * align)


def k_range(total: int, world: int, rank: int, align: int = 64):
    return row_range(total, world, rank, align)


def sharded_contract(spec, *local_operands, **kw) -> torch.Tensor:
    """M-sharded contraction: every rank passes its own slab of the first
    operand (rows ``row_range``) and the full remaining operands; returns the
    rank's output slab.  No communication."""
    return contract(spec, *local_operands, **kw)


def _cast(src: torch.Tensor, out: torch.Tensor, c0: torch.Tensor | None):
    lib = _lib.load()
    rc = lib.bgx_cast_f32(src.data_ptr(), c0.data_ptr() if c0 is not None else None,
                          out.data_ptr(), executor.TORCH_TO_BGX[out.dtype], src.numel(),
                          torch.cuda.current_stream(src.device).cuda_stream)
    _lib.check(rc, "bgx_cast_f32")
    executor._log("cast")
    return out


def ksplit_reduce(partial: torch.Tensor, *, c0: torch.Tensor | None = None, out_dtype=None,
                  group=None, scatter: bool = False, cast=None) -> torch.Tensor:
    """Reduce this rank's f32 partial sums of a K-split contraction over the
    process group — ``reduce_scatter_tensor`` (each rank keeps its row slab)
    when ``scatter`` and the rows divide evenly, else ``all_reduce`` — then
    add ``c0`` and cast to ``out_dtype`` with ``bgx_cast_f32``.  ``cast`` is
    injectable only so the collective logic can be tested on CPU with gloo."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    dt = out_dtype or partial.dtype
    if world > 1 and scatter and partial.shape[0] % world == 0:
        rows = partial.shape[0] // world
        red = torch.empty((rows, *partial.shape[1:]), dtype=torch.float32, device=partial.device)
        dist.reduce_scatter_tensor(red, partial.contiguous(), op=dist.ReduceOp.SUM, group=group)
        r = dist.get_rank(group)
        c0_local = c0[r * rows:(r + 1) * rows] if c0 is not None else None
    else:
        if world > 1:
            dist.all_reduce(partial, op=dist.ReduceOp.SUM, group=group)
        red, c0_local = partial, c0
    if dt == torch.float32 and c0_local is None:
        return red
    out = torch.empty(red.shape, dtype=dt, device=red.device)
    fn = cast or _cast
    return fn(red.contiguous(), out, c0_local.contiguous() if c0_local is not None else None)


def ksplit_contract(spec, a_slab: torch.Tensor, b_slab: torch.Tensor, *,
                    c0: torch.Tensor | None = None, out_dtype=None, group=None,
                    scatter: bool = False) -> torch.Tensor:
    """K-split 2-operand contraction.  ``a_slab``/``b_slab`` hold this rank's
    K range (``k_range``) of the reduction index of ``spec``.  The local
    partial is a tcgen05 (or SIMT) contraction with f32 output; the partials
    are then combined by ``ksplit_reduce`` (one NCCL collective).  Returns the
    full output on every rank, or this rank's row slab with ``scatter``."""
    if not isinstance(spec, EinsumSpec):
        spec = parse_einsum(spec)
    partial = contract(spec, a_slab, b_slab, out_dtype=torch.float32)
    return ksplit_reduce(partial, c0=c0, out_dtype=out_dtype or a_slab.dtype, group=group,
                         scatter=scatter)
