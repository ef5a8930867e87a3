"""Multi-GPU execution: one process per GPU, torch.distributed
for the plumbing.

* M-sharding (``row_range`` + ``contract`` on the local slab): contractions
  with a free M or batch index split their output rows into contiguous slabs,
  one per rank; the other operands are replicated.  No collective on the data
  path — each rank's output slab is final.  Used for the 3-operand chain
  (``(A_r @ B) @ C`` per rank), the batched / plain GEMMs and permutations
  (output rows of a transpose = a strided input slab); ``shard_operands`` /
  ``lead_slabs`` cut the views.
* K-split (``ksplit_contract``): for large-K / small-MN contractions each rank
  takes a K slab, produces f32 partial sums with the tcgen05 kernel, and the
  partials are reduced with one NCCL collective over NVLink
  (``reduce_scatter_tensor`` when the output rows divide by the world size,
  else ``all_reduce``); the reduced f32 tile is cast (and c0 added) by
  ``bgx_cast_f32``.  That collective is the only data exchange anywhere in
  the framework.
"""

from __future__ import annotations

import ctypes

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


def sharded_contract(spec, *operands, group=None, align: int = 128, **kw):
    """M-sharded contraction, one process per GPU: every rank passes the FULL
    (replicated) operands; this rank contracts only its output row slab —
    rows ``row_range`` of the output's leading index, from the operand views
    ``shard_operands`` cuts (narrowed along that index, the rest whole) — and
    returns ``(lo, hi, slab)``.  No communication: the slabs are independent
    and each is computed exactly as on one device (§8e).  ``group`` (default:
    the world group when torch.distributed is initialised, else a single
    rank) gives world size and rank."""
    if not isinstance(spec, EinsumSpec):
        spec = parse_einsum(spec)
    if not spec.output:
        raise ValueError(f"{spec}: a rank-0 output has no rows to shard")
    if dist.is_available() and dist.is_initialized():
        world, rank = dist.get_world_size(group), dist.get_rank(group)
    else:
        world, rank = 1, 0
    lo, hi, views = shard_operands(spec, operands, world, rank, align)
    if hi <= lo:   # more ranks than row slabs: this rank owns nothing
        from .api import output_shape
        shape = output_shape(spec, operands)
        dt = kw.get("out_dtype") or operands[0].dtype
        return lo, hi, torch.empty((0, *shape[1:]), dtype=dt, device=operands[0].device)
    c0 = kw.pop("c0", None)
    if c0 is not None:
        c0 = c0[lo:hi]
    return lo, hi, contract(spec, *views, c0=c0, **kw)


def _cast(src: torch.Tensor, out: torch.Tensor, c0: torch.Tensor | None):
    lib = _lib.load()
    rc = lib.bgx_cast_f32(src.data_ptr(), c0.data_ptr() if c0 is not None else None,
                          out.data_ptr(), executor.TORCH_TO_BGX[out.dtype], src.numel(),
                          torch.cuda.current_stream(src.device).cuda_stream)
    _lib.check(rc, "bgx_cast_f32")
    executor._log("cast")
    return out


class NcclComm:
    """The library's own NCCL communicator (C ABI ``bgx_nccl_*``), for the
    native K-split exchange ``bgx_ksplit_reduce``.  Created collectively: rank
    0 draws the unique id and the process group (``group``, default world)
    broadcasts it; every rank initialises on its current device.  Without a
    process group it is a single-rank communicator."""

    def __init__(self, group=None):
        lib = _lib.load()
        if dist.is_available() and dist.is_initialized():
            self.world, self.rank = dist.get_world_size(group), dist.get_rank(group)
        else:
            self.world, self.rank = 1, 0
        uid = ctypes.create_string_buffer(128)
        if self.rank == 0:
            _lib.check(lib.bgx_nccl_unique_id(uid), "bgx_nccl_unique_id")
        if self.world > 1:
            box = [bytes(uid.raw)]
            dist.broadcast_object_list(box, src=dist.get_global_rank(group, 0)
                                       if group is not None else 0, group=group)
            uid = ctypes.create_string_buffer(box[0], 128)
        handle = _lib._vp()
        _lib.check(lib.bgx_nccl_comm_init(ctypes.byref(handle), self.world, self.rank, uid),
                   "bgx_nccl_comm_init")
        self.handle = handle

    def close(self):
        if self.handle is not None and self.handle.value:
            _lib.check(_lib.load().bgx_nccl_comm_destroy(self.handle), "bgx_nccl_comm_destroy")
        self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 - interpreter teardown
            pass


def _ksplit_reduce_native(partial, comm: NcclComm, c0, dt, scatter):
    """bgx_ksplit_reduce: ncclReduceScatter / ncclAllReduce of the f32
    partials inside libbgx, then c0 + cast (bgx_cast_f32)."""
    rows = partial.shape[0]
    cols = partial.numel() // max(1, rows)
    scatter = bool(scatter and rows % comm.world == 0)
    got = rows // comm.world if scatter else rows
    out = torch.empty((got, *partial.shape[1:]), dtype=dt, device=partial.device)
    c0_local = (c0[comm.rank * got:(comm.rank + 1) * got] if scatter else c0) \
        if c0 is not None else None
    ws = None
    if not (dt == torch.float32 and c0_local is None):
        ws = torch.empty(out.shape, dtype=torch.float32, device=partial.device)
    _lib.check(_lib.load().bgx_ksplit_reduce(
        partial.contiguous().data_ptr(), out.data_ptr(),
        c0_local.contiguous().data_ptr() if c0_local is not None else None,
        executor.TORCH_TO_BGX[dt], rows, cols, 1 if scatter else 0,
        ws.data_ptr() if ws is not None else None, comm.handle,
        torch.cuda.current_stream(partial.device).cuda_stream), "bgx_ksplit_reduce")
    executor._log("ksplit-reduce")
    return out


def ksplit_reduce(partial: torch.Tensor, *, c0: torch.Tensor | None = None, out_dtype=None,
                  group=None, scatter: bool = False, cast=None,
                  comm: NcclComm | None = None) -> torch.Tensor:
    """Reduce this rank's f32 partial sums of a K-split contraction over the
    process group — ``reduce_scatter_tensor`` (each rank keeps its row slab)
    when ``scatter`` and the rows divide evenly, else ``all_reduce`` — then
    add ``c0`` and cast to ``out_dtype`` with ``bgx_cast_f32``.  With
    ``comm`` (an ``NcclComm``) the whole exchange runs inside libbgx
    (``bgx_ksplit_reduce``: the library's own NCCL communicator) instead of
    through torch.distributed.  ``cast`` is injectable only so the collective
    logic can be tested on CPU with gloo."""
    if comm is not None:
        return _ksplit_reduce_native(partial, comm, c0, out_dtype or partial.dtype, scatter)
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


_FUSED_CACHE: dict = {}
FUSED_CACHE_LIMIT = 4   # live FusedKSplit plans (each holds a symmetric-memory buffer)


def _fused_plan(key, build):
    """LRU of FusedKSplit plans keyed by shape/dtype/group.  Ranks call with
    the same shapes in the same order, so every rank evicts the same plan;
    an evicted plan releases its symmetric-memory buffer."""
    f = _FUSED_CACHE.pop(key, None)
    if f is None:
        while len(_FUSED_CACHE) >= FUSED_CACHE_LIMIT:
            _FUSED_CACHE.pop(next(iter(_FUSED_CACHE))).close()
        f = build()
    _FUSED_CACHE[key] = f          # most recently used last
    return f


def ksplit_contract(spec, a_slab: torch.Tensor, b_slab: torch.Tensor, *,
                    c0: torch.Tensor | None = None, out_dtype=None, group=None,
                    scatter: bool = False, fused: bool = False,
                    out: torch.Tensor | None = None,
                    comm: NcclComm | None = None) -> torch.Tensor:
    """K-split 2-operand contraction.  ``a_slab``/``b_slab`` hold this rank's
    K range (``k_range``) of the reduction index of ``spec``.  The local
    partial is a tcgen05 (or SIMT) contraction with f32 output; the partials
    are then combined by ``ksplit_reduce`` (one NCCL collective).  Returns the
    full output on every rank, or this rank's row slab with ``scatter``.
    ``fused=True`` (with ``scatter``) runs the GEMM and the reduce-scatter as
    one kernel (``FusedKSplit``, cached per shape/dtype/group, at most
    ``FUSED_CACHE_LIMIT`` live plans); the returned slab is then
    ``owned_rows`` of the output (rows per owner rounded to 128), copied out
    of the plan's symmetric buffer into ``out`` (or a fresh tensor), so it
    stays valid across later calls.  ``comm``: exchange through libbgx's own
    NCCL communicator (``bgx_ksplit_reduce``) instead of torch.distributed."""
    if not isinstance(spec, EinsumSpec):
        spec = parse_einsum(spec)
    if fused:
        if not scatter:
            raise ValueError("fused K-split returns this rank's row slab: pass scatter=True")
        key = (spec, tuple(a_slab.shape), tuple(a_slab.stride()), tuple(b_slab.shape),
               tuple(b_slab.stride()), a_slab.dtype, out_dtype, id(group), c0 is not None,
               a_slab.device)
        f = _fused_plan(key, lambda: FusedKSplit(spec, a_slab, b_slab, out_dtype=out_dtype,
                                                 group=group, with_c0=c0 is not None))
        c0_local = None
        if c0 is not None:
            lo, hi = owned_rows(f.M, f.plan.rows_per_owner, f.rank)
            c0_local = c0[lo:hi]
        slab = f(a_slab, b_slab, c0=c0_local)
        if out is None:
            return slab.clone()
        return out.copy_(slab)
    partial = contract(spec, a_slab, b_slab, out_dtype=torch.float32)
    return ksplit_reduce(partial, c0=c0, out_dtype=out_dtype or a_slab.dtype, group=group,
                         scatter=scatter, comm=comm)


# ---------------------------------------------------------------------------
# K-split fused with the reduce-scatter (bgx_contract_reduce_scatter)

def _align(n: int, a: int = 256) -> int:
    return (n + a - 1) // a * a


def _rs_desc(spec, a_slab: torch.Tensor, b_slab: torch.Tensor, out_dtype):
    """bgx_contract_desc for this rank's K slab of a plain (batch-free) GEMM
    spec; the output fields are unused by the fused kernel except the row
    stride (dense slabs: N)."""
    from .plan import GemmPlan, extents_of, plan_generic
    if not isinstance(spec, EinsumSpec):
        spec = parse_einsum(spec)
    ins = [a_slab, b_slab]
    ext = extents_of(spec, [t.shape for t in ins])
    oshape = tuple(ext[x] for x in spec.output)
    ostride = tuple(int(s) for s in torch.empty(oshape, device="meta").stride())
    p = plan_generic(spec, [tuple(t.shape) for t in ins] + [oshape],
                     [tuple(t.stride()) for t in ins] + [ostride],
                     dtype=executor.DTYPE_NAME[a_slab.dtype])
    if not isinstance(p, GemmPlan) or p.batch != 1 or p.a_view.needs_copy or p.b_view.needs_copy:
        raise ValueError(f"fused K-split needs a batch-free GEMM spec with strided operands: {spec}")
    sa = executor._group_strides(ins[p.a], spec.inputs[p.a], p.a_view.axes, ext)
    sb = executor._group_strides(ins[p.b], spec.inputs[p.b], p.b_view.axes, ext)
    d = _lib.BgxContractDesc()
    d.batch, d.M, d.N, d.K = 1, p.M, p.N, p.K
    for i in range(3):
        d.a_stride[i], d.b_stride[i] = sa[i], sb[i]
    d.o_stride[0], d.o_stride[1], d.o_stride[2] = p.M * p.N, p.N, 1
    d.c_stride[0], d.c_stride[1], d.c_stride[2] = p.M * p.N, p.N, 1
    d.a, d.b = ins[p.a].data_ptr(), ins[p.b].data_ptr()
    d.in_dtype = executor.TORCH_TO_BGX[a_slab.dtype]
    d.out_dtype = executor.TORCH_TO_BGX[out_dtype]
    d.mode = _lib.MODE_TC
    return d, p


def rs_plan(spec, a_slab, b_slab, world: int, out_dtype=None) -> _lib.BgxRsPlan:
    """The fused kernel's plan (tile, rows per owner, local split, buffer
    bytes) — identical on every rank for identical slab shapes."""
    lib = _lib.load()
    d, _ = _rs_desc(spec, a_slab, b_slab, out_dtype or a_slab.dtype)
    pl = _lib.BgxRsPlan()
    _lib.check(lib.bgx_contract_rs_plan(d, world, pl), "bgx_contract_rs_plan")
    return pl


_BK = 64   # bf16/f16 elements per tcgen05 k-block (gemm_tc.cu Elem<2>::BK)


def _finish_plan(pl, M: int, N: int, splits: int, mode: int | None):
    """Set the agreed local split (and mode) on a plan and recompute the
    buffer sizes that depend on them (bgx.h bgx_rs_plan)."""
    if mode is not None:
        pl.mode = mode
    pl.local_splits = max(1, int(splits))
    S, rpo = pl.local_splits, pl.rows_per_owner
    if pl.mode == _lib.RS_DEFERRED:
        pl.slot_bytes, pl.ws_bytes = pl.world * S * rpo * N * 4, 0
    else:
        pl.slot_bytes = pl.world * rpo * N * 4
        pl.ws_bytes = S * M * N * 4 if S > 1 else 0
    return pl


def owned_rows(M: int, rows_per_owner: int, rank: int):
    """Output rows [lo, hi) the fused reduce-scatter leaves on ``rank``."""
    lo = min(M, rank * rows_per_owner)
    return lo, min(M, lo + rows_per_owner)


class FusedKSplit:
    """K-split contraction whose reduce-scatter is fused into the tcgen05
    GEMM epilogue (one kernel per rank; bgx.h ``bgx_contract_reduce_scatter``).

    Each rank passes its K slab; partial tiles travel over NVLink into the
    owner's symmetric-memory slot as they finish and the last contributor of
    each tile reduces it (rank order, deterministic) into the owner's output
    rows.  Peer buffers come from ``torch.distributed._symmetric_memory``
    (world > 1); one device-side barrier before (slot reuse) and after (all of
    this rank's rows delivered) each call.  ``__call__`` returns this rank's
    ``owned_rows`` slab as a VIEW of the symmetric buffer: the next call (on
    this rank, or a peer delivering into it) overwrites it — clone it, or use
    ``ksplit_contract(fused=True)``, which copies it out.  This replaces ``ksplit_contract(..., scatter=True)`` (GEMM ->
    ``reduce_scatter_tensor`` -> cast) with no NCCL on the data path."""

    def __init__(self, spec, a_slab: torch.Tensor, b_slab: torch.Tensor, *, out_dtype=None,
                 group=None, with_c0: bool = False, local_splits: int | None = None,
                 mode: int | None = None, barrier_timeout_ms: int = 60000):
        self.spec = spec if isinstance(spec, EinsumSpec) else parse_einsum(spec)
        self.group = group
        # device barriers give up (a CUDA error, not a hang) if a peer never
        # arrives — e.g. a rank that failed between two calls
        self.barrier_timeout_ms = int(barrier_timeout_ms)
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.out_dtype = out_dtype or a_slab.dtype
        self.dev = a_slab.device
        self._lib = _lib.load()
        d, p = _rs_desc(self.spec, a_slab, b_slab, self.out_dtype)
        self.M, self.N = p.M, p.N
        pl = _lib.BgxRsPlan()
        _lib.check(self._lib.bgx_contract_rs_plan(d, self.world, pl), "bgx_contract_rs_plan")
        pl.rank = self.rank
        if local_splits is not None and local_splits < 1:
            raise ValueError(f"local_splits must be >= 1, got {local_splits}")
        # every rank must use the same local split (deferred mode: it fixes
        # the slot layout) and it may not exceed any rank's k-blocks
        S = local_splits if local_splits is not None else pl.local_splits
        kb = -(-p.K // _BK)
        if self.world > 1:
            dev = self.dev if dist.get_backend(group) == "nccl" else torch.device("cpu")
            t = torch.tensor([S, kb], dtype=torch.int64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
            S, kb = int(t[0]), int(t[1])
        _finish_plan(pl, self.M, self.N, min(S, kb), mode)
        self.plan = pl
        rpo, N = pl.rows_per_owner, self.N
        esz = torch.tensor([], dtype=self.out_dtype).element_size()
        regions = [("slots", pl.slot_bytes), ("counters", pl.counter_bytes),
                   ("out", rpo * N * esz), ("c0", rpo * N * esz if with_c0 else 0)]
        offs, total = {}, 0
        for name, nbytes in regions:
            offs[name] = total
            total += _align(nbytes)
        if dist.is_initialized() and self.dev.type == "cuda":
            from torch.distributed import _symmetric_memory as symm_mem
            self.buf = symm_mem.empty(total, dtype=torch.uint8, device=self.dev)
            self.buf[offs["counters"]:offs["counters"] + pl.counter_bytes].zero_()
            self.hdl = symm_mem.rendezvous(self.buf, self.group or dist.group.WORLD)
            bases = list(self.hdl.buffer_ptrs)
            self.hdl.barrier(0, self.barrier_timeout_ms)
        else:
            self.buf = torch.zeros(total, dtype=torch.uint8, device=self.dev)
            self.hdl = None
            bases = [self.buf.data_ptr()]
        rs = _lib.BgxReduceScatter()
        rs.plan = pl
        for r, base in enumerate(bases):
            rs.slots[r] = base + offs["slots"]
            rs.counters[r] = base + offs["counters"]
            rs.out[r] = base + offs["out"]
            rs.c0[r] = base + offs["c0"] if with_c0 else None
        self.ws = None
        if pl.ws_bytes > 0:             # in-kernel mode with a local split
            self.ws = torch.empty(pl.ws_bytes, dtype=torch.uint8, device=self.dev)
            self.ws_counters = torch.zeros(max(16, pl.counter_bytes), dtype=torch.uint8,
                                           device=self.dev)
            rs.ws, rs.ws_counters = self.ws.data_ptr(), self.ws_counters.data_ptr()
        self.rs = rs
        self.desc = d
        self._a_idx = p.a
        lo, hi = owned_rows(self.M, rpo, self.rank)
        o = offs["out"]
        self.out = self.buf[o:o + rpo * N * esz].view(self.out_dtype).view(rpo, N)[:hi - lo]
        self.c0_buf = (self.buf[offs["c0"]:offs["c0"] + rpo * N * esz].view(self.out_dtype)
                       .view(rpo, N)[:hi - lo]) if with_c0 else None

    def close(self):
        """Release the symmetric-memory buffer (and local workspaces)."""
        self.hdl = None
        self.buf = self.out = self.c0_buf = self.ws = None

    def __call__(self, a_slab: torch.Tensor, b_slab: torch.Tensor, c0=None) -> torch.Tensor:
        if self.buf is None:
            raise RuntimeError("FusedKSplit used after close()")
        if (c0 is not None) != (self.c0_buf is not None):
            raise ValueError("c0 must be given iff the FusedKSplit was built with_c0=True")
        if c0 is not None:
            self.c0_buf.copy_(c0)
        ins = (a_slab, b_slab)
        self.desc.a = ins[self._a_idx].data_ptr()
        self.desc.b = ins[1 - self._a_idx].data_ptr()
        if self.hdl is not None:
            self.hdl.barrier(0, self.barrier_timeout_ms)
        stream = torch.cuda.current_stream(self.dev).cuda_stream
        _lib.check(self._lib.bgx_contract_reduce_scatter(self.desc, self.rs, stream),
                   "bgx_contract_reduce_scatter")
        executor._log("tcgen05-rs")
        if self.hdl is not None:
            self.hdl.barrier(0, self.barrier_timeout_ms)
        if self.plan.mode == _lib.RS_DEFERRED:   # every partial of my rows is in my slots
            _lib.check(self._lib.bgx_rs_reduce(self.desc, self.rs, stream), "bgx_rs_reduce")
            executor._log("rs-reduce")
        return self.out


def emulate_fused_ksplit(spec, a_slabs, b_slabs, *, c0=None, out_dtype=None,
                         mode: int | None = None, local_splits: int | None = None) -> torch.Tensor:
    """Run the fused K-split reduce-scatter of ``len(a_slabs)`` ranks on ONE
    GPU: the same kernel, launched once per emulated rank in rank order, with
    the owners' slots / counters / outputs as local buffers.  No launch waits
    for another (the last contributor of each tile does the reduction), so
    this is exactly the multi-GPU computation, serialised.  In deferred mode
    (the planner's default) the launches only deliver, and each owner's
    bgx_rs_reduce then runs once, as it would after the barrier.  Returns the
    full M x N output (the owners' slabs stacked)."""
    if not isinstance(spec, EinsumSpec):
        spec = parse_einsum(spec)
    world = len(a_slabs)
    lib = _lib.load()
    out_dtype = out_dtype or a_slabs[0].dtype
    d, p = _rs_desc(spec, a_slabs[0], b_slabs[0], out_dtype)
    pl = _lib.BgxRsPlan()
    _lib.check(lib.bgx_contract_rs_plan(d, world, pl), "bgx_contract_rs_plan")
    M, N, rpo = p.M, p.N, pl.rows_per_owner
    kb = min(-(-_rs_desc(spec, a, b, out_dtype)[1].K // _BK) for a, b in zip(a_slabs, b_slabs))
    _finish_plan(pl, M, N, min(local_splits or pl.local_splits, kb), mode)
    dev = a_slabs[0].device
    slots = torch.empty(world, pl.slot_bytes // 4, dtype=torch.float32, device=dev)
    counters = torch.zeros(world, max(4, pl.counter_bytes // 4), dtype=torch.int32, device=dev)
    out = torch.empty(world * rpo, N, dtype=out_dtype, device=dev)
    c0_pad = None
    if c0 is not None:
        c0_pad = torch.zeros(world * rpo, N, dtype=out_dtype, device=dev)
        c0_pad[:M].copy_(c0)
    rs = _lib.BgxReduceScatter()
    for r in range(world):
        rs.slots[r] = slots[r].data_ptr()
        rs.counters[r] = counters[r].data_ptr()
        rs.out[r] = out[r * rpo].data_ptr()
        rs.c0[r] = c0_pad[r * rpo].data_ptr() if c0_pad is not None else None
    if pl.ws_bytes > 0:
        ws = torch.empty(pl.ws_bytes, dtype=torch.uint8, device=dev)
        wsc = torch.zeros(max(16, pl.counter_bytes), dtype=torch.uint8, device=dev)
        rs.ws, rs.ws_counters = ws.data_ptr(), wsc.data_ptr()
    stream = torch.cuda.current_stream(dev).cuda_stream
    for r in range(world):
        dr, pr = _rs_desc(spec, a_slabs[r], b_slabs[r], out_dtype)
        if (pr.M, pr.N) != (M, N):
            raise ValueError("all ranks' slabs must produce the same M x N output")
        pl.rank = r
        rs.plan = pl
        _lib.check(lib.bgx_contract_reduce_scatter(dr, rs, stream), "bgx_contract_reduce_scatter")
        executor._log("tcgen05-rs")
    if pl.mode == _lib.RS_DEFERRED:
        for r in range(world):
            pl.rank = r
            rs.plan = pl
            _lib.check(lib.bgx_rs_reduce(d, rs, stream), "bgx_rs_reduce")
            executor._log("rs-reduce")
    return out[:M]


# ---------------------------------------------------------------------------
# one process, several devices (``einsum(..., devices=...)``)

def lead_slabs(spec, operands, lo: int, hi: int):
    """Views of ``operands`` restricted to rows ``[lo, hi)`` of the output's
    leading index (§8e): every operand that carries that index is narrowed
    along it (a strided view when it is not the operand's first axis — e.g.
    the input columns of a transpose ``(i,j)->(j,i)``), the rest are returned
    whole.  The output's leading index is parallel (it is an output index), so
    output rows ``[lo, hi)`` depend on nothing else and every element is
    evaluated exactly as in the unsharded call."""
    if not isinstance(spec, EinsumSpec):
        spec = parse_einsum(spec)
    if not spec.output:
        raise ValueError(f"{spec}: a rank-0 output has no rows to shard")
    lead = spec.output[0]
    return [t.narrow(tup.index(lead), lo, hi - lo) if lead in tup else t
            for t, tup in zip(operands, spec.inputs)]


def shard_operands(spec, operands, world: int, rank: int, align: int = 128):
    """One-process-per-GPU form of the M-shard: rank ``rank``'s output row
    range ``(lo, hi)`` (``row_range`` of the output's leading extent) and the
    operand views that produce it (``lead_slabs``)."""
    from .api import output_shape
    if not isinstance(spec, EinsumSpec):
        spec = parse_einsum(spec)
    rows = output_shape(spec, operands)[0] if spec.output else 0
    lo, hi = row_range(rows, world, rank, align)
    return lo, hi, lead_slabs(spec, operands, lo, hi)


def contract_devices(spec, *operands: torch.Tensor, devices, out=None, **kw) -> torch.Tensor:
    """M-sharded contraction driven from ONE process over ``devices``: rows of
    the output's leading index are split into contiguous slabs
    (``row_range``); the operand views that produce slab r (``lead_slabs``:
    narrowed along that index, the other operands whole) are copied to
    ``devices[r]`` (peer copies over NVLink), each device contracts its slab
    on its own current stream — launches are asynchronous, so the devices run
    concurrently — and the slabs are copied back into ``out`` on the
    operands' device.  When every slab is a plain GEMM the slabs are launched
    by ONE C-ABI call, ``bgx_contract_sharded`` (a descriptor per slab, each
    on its own device and stream).  Covers contractions (leading index from operand 0, 1,
    or several operands) and permutations (a transpose's output rows are a
    strided column slab of its input, §8e).  No collective: the slabs are
    independent, so every row is computed as on one device — bit for bit
    unless the planner splits K differently for a slab (long K), which only
    reorders the f32 summation."""
    from .api import output_shape
    if not isinstance(spec, EinsumSpec):
        spec = parse_einsum(spec)
    devices = [torch.device("cuda", d) if isinstance(d, int) else torch.device(d) for d in devices]
    if not spec.output:
        raise ValueError(f"{spec}: a rank-0 output has no rows to shard")
    home = operands[0].device
    shape = output_shape(spec, operands)
    dt = kw.get("out_dtype") or operands[0].dtype
    if out is None:
        out = torch.empty(shape, dtype=dt, device=home)
    c0 = kw.pop("c0", None)
    rows = shape[0]
    n = len(devices)
    # stage every slab on its device (peer copies), then launch
    slabs = []
    for r, dev in enumerate(devices):
        lo, hi = row_range(rows, n, r)
        if hi <= lo:
            continue
        with torch.cuda.device(dev):
            local = [t.to(dev, non_blocking=True) for t in lead_slabs(spec, operands, lo, hi)]
            cc = c0[lo:hi].to(dev, non_blocking=True) if c0 is not None else None
            y = torch.empty((hi - lo, *shape[1:]), dtype=dt, device=dev)
        slabs.append((lo, hi, dev, local, cc, y))
    descs = _sharded_descriptors(spec, slabs, kw) if slabs else None
    if descs is not None:
        # every slab is a plain GEMM: ONE C-ABI call launches them all, each
        # on its own device and current stream (bgx_contract_sharded)
        lib = _lib.load()
        arr = (_lib.BgxContractDesc * len(descs))(*descs)
        devs = (_lib._i32 * len(descs))(*[dev.index for _, _, dev, *_ in slabs])
        streams = (_lib._vp * len(descs))(*[torch.cuda.current_stream(dev).cuda_stream
                                              for _, _, dev, *_ in slabs])
        _lib.check(lib.bgx_contract_sharded(arr, devs, streams, len(descs)),
                   "bgx_contract_sharded")
        executor._log("sharded")
    else:
        for lo, hi, dev, local, cc, y in slabs:
            with torch.cuda.device(dev):
                contract(spec, *local, c0=cc, out=y, **kw)
    pending = []
    for lo, hi, dev, local, cc, y in slabs:
        done = torch.cuda.Event()
        with torch.cuda.device(dev):
            done.record(torch.cuda.current_stream(dev))
        pending.append((lo, hi, y, done))
    home_stream = torch.cuda.current_stream(home)
    for lo, hi, y, done in pending:
        home_stream.wait_event(done)
        out[lo:hi].copy_(y, non_blocking=True)
    return out


def _sharded_descriptors(spec, slabs, kw):
    """One bgx_contract_desc per slab when every slab is a plain GEMM the
    planner would launch as one bgx_contract (executor.gemm_descriptor), else
    None (permutations, chains, operand copies, split-K: per-device path)."""
    if kw.get("schedule") or kw.get("chain_order", "auto") not in ("left", "auto") or len(spec.inputs) != 2:
        return None
    mode = kw.get("mode", "auto")
    from .plan import GemmPlan
    descs = []
    for lo, hi, dev, local, cc, y in slabs:
        if any(t.dtype != local[0].dtype for t in local):
            return None
        plan = executor.plan_for(spec, local, y, mode=mode)
        if not isinstance(plan, GemmPlan):
            return None
        got = executor.gemm_descriptor(plan, spec, local, cc, y, mode)
        if got is None:
            return None
        descs.append(got[0])
    return descs
