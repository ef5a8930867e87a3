"""Device-resident execution of planned generic ops through libbgx.so.

Torch is plumbing here (device memory, the current CUDA stream); every byte
of compute is one of the sm_100a kernels behind include/bgx.h.  There is no
CPU path: CPU tensors are rejected, and a missing libbgx.so raises
``BackendUnavailable``.

Semantics follow bridgegen ``_generic`` (interp.py:372-424): the result is a
FRESH tensor holding ``c0 + sum(prod(inputs))`` (``c0`` = the output operand,
never mutated, interp.py:399) — or the permuted input for a passthrough body.
"""

from __future__ import annotations

import contextlib
import threading

import torch

from . import _lib
from .einsum import EinsumSpec
from .plan import (ChainPlan, GemmPlan, GenericPlan, PermutePlan, extents_of,
                   plan_generic)

TORCH_TO_BGX = {torch.float32: _lib.F32, torch.float64: _lib.F64,
                torch.bfloat16: _lib.BF16, torch.float16: _lib.F16}
DTYPE_NAME = {torch.float32: "f32", torch.float64: "f64", torch.bfloat16: "bf16",
              torch.float16: "f16"}
MODES = {"auto": _lib.MODE_AUTO, "exact": _lib.MODE_EXACT, "ffma": _lib.MODE_FFMA,
         "tc": _lib.MODE_TC, "simt": _lib.MODE_SIMT, "tf32": _lib.MODE_TF32}

_trace = threading.local()


def launch_log() -> list:
    """Kernels launched by this thread since the last ``reset_launch_log``."""
    if not hasattr(_trace, "log"):
        _trace.log = []
    return _trace.log


def reset_launch_log():
    _trace.log = []
    _trace.tiles = []


def tile_log() -> list:
    """(cta_group, tile_n, splits) of each tcgen05 launch made under an
    explicit schedule since the last ``reset_launch_log`` — how a
    ``Schedule`` attached to a generic op is observed to take effect."""
    if not hasattr(_trace, "tiles"):
        _trace.tiles = []
    return _trace.tiles


def _log(name: str):
    launch_log().append(name)


@contextlib.contextmanager
def timed_launches():
    """Record a CUDA event pair around every library launch this thread makes
    (on the stream the kernel is launched on) while the context is open;
    yields the list of ``(kernel_name, start_event, end_event)``.  Used by
    bench.py to time the dominant kernel inside a public-API step."""
    prev = getattr(_trace, "events", None)
    _trace.events = []
    try:
        yield _trace.events
    finally:
        _trace.events = prev


def _ev_begin(out):
    evs = getattr(_trace, "events", None)
    if evs is None:
        return None
    e0 = torch.cuda.Event(enable_timing=True)
    e0.record(torch.cuda.current_stream(out.device))
    return e0


def _ev_end(e0, name, out):
    if e0 is not None:
        e1 = torch.cuda.Event(enable_timing=True)
        e1.record(torch.cuda.current_stream(out.device))
        _trace.events.append((name, e0, e1))


CACHE_LIMIT = 256


def _cache_put(cache: dict, key, value, limit: int = CACHE_LIMIT):
    """Insert into a per-thread launch cache, evicting the oldest entry once
    ``limit`` entries are held (dicts keep insertion order)."""
    if key not in cache and len(cache) >= limit:
        cache.pop(next(iter(cache)))
    cache[key] = value


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def _stream_ptr(t: torch.Tensor):
    """cudaStream_t of torch's current stream on ``t``'s device (as int);
    the raw getter skips building a torch.cuda.Stream object per launch."""
    if _raw_stream is not None and t.device.index is not None:
        return _raw_stream(t.device.index)
    return torch.cuda.current_stream(t.device).cuda_stream


def _on_device(dev):
    """Context switching torch's current device to ``dev`` only when needed
    (entering ``torch.cuda.device`` costs microseconds on every call)."""
    if dev.index is None or dev.index == torch.cuda.current_device():
        return contextlib.nullcontext()
    return torch.cuda.device(dev)


def _check_device(tensors):
    dev = None
    for t in tensors:
        if t is None:
            continue
        if not t.is_cuda:
            raise ValueError("bgx executes on CUDA tensors only (no CPU fallback)")
        if dev is None:
            dev = t.device
        elif t.device != dev:
            raise ValueError(f"operands on different devices: {dev} vs {t.device}")
    return dev


# ---------------------------------------------------------------------------
# raw kernel calls

def permute(x: torch.Tensor, out: torch.Tensor, perm) -> torch.Tensor:
    lib = _lib.load()
    ti, to = _lib.BgxTensor(), _lib.BgxTensor()
    for t, desc in ((x, ti), (out, to)):
        desc.data = t.data_ptr()
        desc.dtype = TORCH_TO_BGX[t.dtype]
        desc.rank = t.dim()
        for d in range(t.dim()):
            desc.shape[d] = t.shape[d]
            desc.stride[d] = t.stride(d)
    p = (_lib._i32 * max(1, len(perm)))(*perm)
    with _on_device(x.device):
        _lib.check(lib.bgx_permute(ti, to, p, _stream_ptr(x)), "bgx_permute")
    _log("permute")
    return out


def _generic_desc(spec: EinsumSpec, inputs, c0, out):
    """bgx_generic_desc of one generic op (c0: contiguous or None)."""
    if out.dtype not in TORCH_TO_BGX:
        raise NotImplementedError(f"bgx_generic: unsupported dtype {out.dtype}")
    if len(inputs) > _lib.MAX_OPERANDS or len(spec.axes) > _lib.MAX_AXES:
        raise NotImplementedError("bgx_generic: too many operands/axes")
    d = _lib.BgxGenericDesc()
    d.n_in = len(inputs)
    d.n_axes = len(spec.axes)
    d.n_par = len(spec.output)
    d.dtype = TORCH_TO_BGX[out.dtype]
    ext = extents_of(spec, [t.shape for t in inputs] + [out.shape])
    for a, name in enumerate(spec.axes):
        d.extents[a] = ext[name]
    for k, (t, tup) in enumerate(zip(inputs, spec.inputs)):
        d.ins[k] = t.data_ptr()
        for dim, name in enumerate(tup):
            d.strides[k][spec.axes.index(name)] = t.stride(dim)
    d.c0 = c0.data_ptr() if c0 is not None else None   # NULL: zero initial output
    d.out = out.data_ptr()
    return d


def _launch_generic(lib, d, tree: bool, out):
    """bgx_generic, or bgx_generic_tree with a workspace from the allocator."""
    with _on_device(out.device):
        if tree:
            ws_bytes = _lib._i64(0)
            _lib.check(lib.bgx_generic_tree_plan(d, ws_bytes), "bgx_generic_tree_plan")
            ws = torch.empty(max(1, ws_bytes.value), dtype=torch.uint8, device=out.device)
            _lib.check(lib.bgx_generic_tree(d, ws.data_ptr(), ws_bytes.value, _stream_ptr(out)),
                       "bgx_generic_tree")
            _log("generic-tree")
        else:
            _lib.check(lib.bgx_generic(d, _stream_ptr(out)), "bgx_generic")
            _log("generic")
    return out


def generic(spec: EinsumSpec, inputs, c0: torch.Tensor | None, out: torch.Tensor, *,
            tree: bool = False) -> torch.Tensor:
    """The reference loop nest on the device (bit-exact for f32/f64; bf16/f16
    widened to f32, per-op f32 rounding, one final rounding to the storage
    type — the tensor-core path's semantics).  ``tree=True`` (tolerance
    mode, bodies with a reduction): block-wide tree reductions instead of one
    sequential chain per output (``bgx_generic_tree``, not bit-exact)."""
    lib = _lib.load()
    assert out.is_contiguous()
    if c0 is not None and not c0.is_contiguous():
        c0 = permute(c0, torch.empty(c0.shape, dtype=c0.dtype, device=c0.device),
                     list(range(c0.dim())))
    spec, inputs = _materialize_transposed(spec, inputs, out)
    d = _generic_desc(spec, inputs, c0, out)
    return _launch_generic(lib, d, tree and len(spec.axes) > len(spec.output), out)


TRANSPOSE_MIN_ELEMS = 1 << 20


def _transposed_inputs(spec: EinsumSpec, inputs, out) -> bool:
    """True when ``generic`` would materialise a transposed input (then the
    launch is not cached as a plain pointer patch)."""
    if len(spec.axes) != len(spec.output) or not spec.output or out.numel() < TRANSPOSE_MIN_ELEMS:
        return False
    last = spec.output[-1]
    return any(_is_transposed(t, tup, last, out) for t, tup in zip(inputs, spec.inputs))


def _is_transposed(t, tup, last, out) -> bool:
    """A large input (>= 1/4 of the output's elements; small ones stay in
    cache) that carries the output's contiguous axis at a non-unit stride."""
    return (last in tup and t.stride(tup.index(last)) != 1 and t.shape[tup.index(last)] > 1
            and 4 * t.numel() >= out.numel())


def _materialize_transposed(spec: EinsumSpec, inputs, out):
    """Bodies with no reduction (elementwise over the output, read once):
    an input walked across its rows — it carries the output's contiguous
    axis at a non-unit stride — is first copied into the output's axis order
    by the tiled transpose (bytes moved, bit-exact), so the loop nest reads
    every operand coalesced; one extra pass over that operand instead of a
    warp-divergent load per element (profiles/r02_exact_chains.txt)."""
    if len(spec.axes) != len(spec.output) or not spec.output or out.numel() < TRANSPOSE_MIN_ELEMS:
        return spec, inputs
    last = spec.output[-1]
    new_tups, new_ins, changed = [], [], False
    for t, tup in zip(inputs, spec.inputs):
        if _is_transposed(t, tup, last, out):
            order = tuple(a for a in spec.output if a in tup)
            perm = [tup.index(a) for a in order]
            y = torch.empty([t.shape[i] for i in perm], dtype=t.dtype, device=t.device)
            permute(t, y, perm)
            new_tups.append(order)
            new_ins.append(y)
            changed = True
        else:
            new_tups.append(tup)
            new_ins.append(t)
    if not changed:
        return spec, inputs
    return _spec_of(new_tups, spec.output), new_ins


def _tree_output_order(spec, inputs):
    """(spec with the output axes reordered, permutation back to the
    requested order) when the largest input's unit-stride axis is an output
    axis other than the innermost one — e.g. (d,a,b),(b)->(b,d) — and the
    reduction is long enough for the extra move of the result not to matter;
    else None."""
    if len(spec.axes) == len(spec.output) or len(spec.output) < 2:
        return None
    k = max(range(len(inputs)), key=lambda i: inputs[i].numel())
    x = inputs[k]
    tup = spec.inputs[k]
    unit = [a for d, a in enumerate(tup) if x.shape[d] > 1 and x.stride(d) == 1]
    if not unit or unit[0] not in spec.output or unit[0] == spec.output[-1]:
        return None
    inner = spec.output[-1]
    if inner in tup and x.stride(tup.index(inner)) == 1:
        return None
    n_out = 1
    for a in spec.output:
        for t, y in zip(spec.inputs, inputs):
            if a in t:
                n_out *= y.shape[t.index(a)]
                break
    if x.numel() < 16 * n_out:
        return None
    new_out = tuple(a for a in spec.output if a != unit[0]) + (unit[0],)
    text = ",".join("(" + ",".join(t) + ")" for t in spec.inputs) + "->(" + ",".join(new_out) + ")"
    from .einsum import parse_einsum
    return parse_einsum(text), [new_out.index(a) for a in spec.output]


def _fast_generic_materialized(spec, inputs, c0, out, tree: bool):
    """_fast_generic for bodies whose transposed inputs are first copied
    into the output's axis order (_materialize_transposed): the copies'
    permutations and the generic descriptor over the copies are fixed per
    signature, so a repeat call is the copies plus one launch (the planner
    and descriptor build — ~60 us of host time — are skipped)."""
    if not out.is_contiguous() or (c0 is not None and not c0.is_contiguous()):
        return None
    last = spec.output[-1]
    moves, new_tups, probe = [], [], list(inputs)
    for k, (t, tup) in enumerate(zip(inputs, spec.inputs)):
        if _is_transposed(t, tup, last, out):
            order = tuple(a for a in spec.output if a in tup)
            perm = [tup.index(a) for a in order]
            shape = [t.shape[i] for i in perm]
            moves.append((k, perm, shape))
            new_tups.append(order)
            probe[k] = torch.empty(shape, dtype=t.dtype, device=t.device)
        else:
            new_tups.append(tup)
    if not moves:
        return None
    spec2 = _spec_of(new_tups, spec.output)
    lib = _lib.load()
    d = _generic_desc(spec2, probe, c0, out)
    tree = tree and len(spec2.axes) > len(spec2.output)
    n = len(inputs)

    def run(xs, o, c):
        for k in range(n):
            d.ins[k] = xs[k].data_ptr()
        tmps = []
        for k, perm, shape in moves:
            y = torch.empty(shape, dtype=xs[k].dtype, device=xs[k].device)
            permute(xs[k], y, perm)
            d.ins[k] = y.data_ptr()
            tmps.append(y)   # stream-ordered frees: safe once the launch is queued
        d.c0 = c.data_ptr() if c is not None else None
        d.out = o.data_ptr()
        _launch_generic(lib, d, tree, o)
    return run


def _fast_generic(spec, inputs, c0, out, tree: bool):
    """Pre-built descriptor for a repeated generic signature: later calls
    patch the pointers and launch (the planning, extents and Python
    descriptor build — tens of microseconds — are skipped)."""
    if not out.is_contiguous() or (c0 is not None and not c0.is_contiguous()):
        return None
    lib = _lib.load()
    d = _generic_desc(spec, inputs, c0, out)
    tree = tree and len(spec.axes) > len(spec.output)
    n = len(inputs)

    def run(xs, o, c):
        for k in range(n):
            d.ins[k] = xs[k].data_ptr()
        d.c0 = c.data_ptr() if c is not None else None
        d.out = o.data_ptr()
        _launch_generic(lib, d, tree, o)
    return run


def contract_raw(a, a_strides, b, b_strides, out, o_strides, *, batch, M, N, K, c0=None,
                 c_strides=(0, 0, 0), mode="auto", schedule=None, in_dtype=None) -> int:
    """One ``bgx_contract`` call on raw (tensor, 3 strides) views; returns the
    kernel id that ran (_lib.KERNEL_*)."""
    lib = _lib.load()
    if mode == "tf32" and schedule and schedule.get("tf32_kmajor"):
        # optional: materialise MN-major operands K-major first (comparison path)
        if a_strides[2] != 1 and K > 1:
            a3 = torch.as_strided(a, (batch, M, K), a_strides)
            a = permute(a3, torch.empty((batch, M, K), dtype=a.dtype, device=a.device), (0, 1, 2))
            a_strides = (M * K, K, 1)
        if b_strides[1] != 1 and K > 1:
            b3 = torch.as_strided(b, (batch, K, N), b_strides)
            b = permute(b3, torch.empty((batch, N, K), dtype=b.dtype, device=b.device), (0, 2, 1))
            b_strides = (N * K, 1, K)
    # memoised launch decision: everything the kernel choice depends on (shape,
    # strides, dtypes, mode, schedule, pointer alignment); a hit skips the
    # descriptor build and the planning calls — only the pointers change
    key = None
    if a is not None and b is not None and not (mode == "tf32" and schedule
                                                and schedule.get("tf32_kmajor")):
        sk = tuple(sorted((k, tuple(v) if isinstance(v, (list, tuple)) else v)
                          for k, v in schedule.items())) if schedule else ()
        key = (batch, M, N, K, tuple(a_strides), tuple(b_strides), tuple(c_strides),
               tuple(o_strides), in_dtype or a.dtype, out.dtype, mode, sk, c0 is None,
               a.data_ptr() % 16, b.data_ptr() % 16, out.data_ptr() % 16,
               (c0.data_ptr() % 16) if c0 is not None else 0, out.device.index)
        hit = _launch_cache().get(key)
        if hit is not None:
            d, kind, splits_v, ws_v, tile = hit
            d.a, d.b, d.out = a.data_ptr(), b.data_ptr(), out.data_ptr()
            d.c0 = c0.data_ptr() if c0 is not None else None
            if tile is not None:
                tile_log().append(tile)
            return _launch(lib, d, kind, splits_v, ws_v, out)
    d = _lib.BgxContractDesc()
    d.batch, d.M, d.N, d.K = batch, M, N, K
    d.a = a.data_ptr() if a is not None else None
    d.b = b.data_ptr() if b is not None else None
    d.c0 = c0.data_ptr() if c0 is not None else None
    d.out = out.data_ptr()
    for i in range(3):
        d.a_stride[i], d.b_stride[i] = a_strides[i], b_strides[i]
        d.c_stride[i], d.o_stride[i] = c_strides[i], o_strides[i]
    d.in_dtype = TORCH_TO_BGX[in_dtype or a.dtype]
    d.out_dtype = TORCH_TO_BGX[out.dtype]
    d.mode = MODES[mode]
    if schedule:
        for k, v in schedule.items():
            if k in ("splits", "no_splitk", "tf32_kmajor"):
                continue
            if k == "reserved":
                for i, x in enumerate(v):
                    d.sched.reserved[i] = int(x)
            elif k == "cluster_n":
                d.sched.reserved[1] = int(v)
            else:
                setattr(d.sched, k, int(v))
    kind = lib.bgx_contract_kernel(d)
    pad_ok = a is not None and b is not None and not getattr(_trace, "in_pad", False)
    if pad_ok and ((kind == _lib.KERNEL_SIMT16 and mode == "auto"
                    and 2 * batch * M * N * K >= PAD_MIN_FLOP)
                   or (kind == _lib.ERR_UNSUPPORTED and mode in ("tc", "tf32")
                       and in_dtype is None and a.dtype in (torch.bfloat16, torch.float16,
                                                            torch.float32))):
        # operands whose strides/extents are not TMA-legal (odd K or N,
        # unaligned views): stage zero-padded, aligned copies and run on the
        # tensor cores instead of the CUDA-core fallback (~40x slower at scale)
        # or, in the tensor-core-only modes, instead of failing
        return _contract_padded(a, a_strides, b, b_strides, out, o_strides, batch=batch, M=M,
                                N=N, K=K, c0=c0, c_strides=c_strides, schedule=schedule,
                                mode=mode)
    _lib.check(kind if kind < 0 else 0, "bgx_contract_kernel")
    splits = _lib._i32(1)
    ws_bytes = _lib._i64(0)
    if kind == _lib.KERNEL_TC and not (schedule and schedule.get("no_splitk")):
        _lib.check(lib.bgx_contract_splitk_plan(d, splits, ws_bytes), "bgx_contract_splitk_plan")
        if schedule and schedule.get("splits"):
            splits.value = int(schedule["splits"])
            if splits.value < -1:   # forced tail split: upper-bound workspace
                ws_bytes.value = lib.bgx_sm_count() * (-splits.value * 256 * 512 * 4 + 8) + 256
            else:
                ws_bytes.value = splits.value * batch * M * N * 4
    tile = None
    if schedule and kind == _lib.KERNEL_TC:
        cg, bn = _lib._i32(0), _lib._i32(0)
        _lib.check(lib.bgx_contract_tile(d, cg, bn), "bgx_contract_tile")
        tile = (cg.value, bn.value, splits.value)
        tile_log().append(tile)
    if key is not None:
        _cache_put(_launch_cache(), key, (d, kind, splits.value, ws_bytes.value, tile), 512)
    return _launch(lib, d, kind, splits.value, ws_bytes.value, out)


def _launch_cache() -> dict:
    if not hasattr(_trace, "launch_cache"):
        _trace.launch_cache = {}
    return _trace.launch_cache


def _launch(lib, d, kind, splits, ws_bytes, out) -> int:
    with _on_device(out.device):
        if splits > 1 or splits < -1:
            ws = torch.empty(ws_bytes, dtype=torch.uint8, device=out.device)
            name = "tcgen05-splitk" if splits > 1 else "tcgen05-tailsplit"
            e0 = _ev_begin(out)
            _lib.check(lib.bgx_contract_splitk(d, splits, ws.data_ptr(), ws_bytes,
                                               _stream_ptr(out)), "bgx_contract_splitk")
            _ev_end(e0, name, out)
            _log(name)
            return kind
        name = _lib.KERNEL_NAMES.get(kind, "contract")
        e0 = _ev_begin(out)
        _lib.check(lib.bgx_contract(d, _stream_ptr(out)), "bgx_contract")
        _ev_end(e0, name, out)
    _log(name)
    return kind


PAD_MIN_FLOP = 1 << 28
TREE_16BIT_POINTS = 1024
PREREDUCE_16BIT_BLOWUP = 16   # product space vs operands; 64 left the perf fuzz's 2^30-2^31-point bf16 bodies (32-64x) on an 8-20 ms direct walk


def _contract_padded(a, a_strides, b, b_strides, out, o_strides, *, batch, M, N, K, c0,
                     c_strides, schedule, mode="auto") -> int:
    """K and N rounded up to 16-byte multiples with zero padding (zero
    products leave every sum unchanged), operands copied by bgx_permute into
    aligned dense buffers, one tcgen05 contraction, valid columns copied back."""
    dev = out.device
    q = 16 // a.element_size()
    kp, np_ = (K + q - 1) // q * q, (N + q - 1) // q * q
    av = torch.as_strided(a, (batch, M, K), a_strides, a.storage_offset())
    bv = torch.as_strided(b, (batch, K, N), b_strides, b.storage_offset())
    ap = torch.zeros((batch, M, kp), dtype=a.dtype, device=dev)
    bp = torch.zeros((batch, kp, np_), dtype=b.dtype, device=dev)
    permute(av, ap[:, :, :K], (0, 1, 2))
    permute(bv, bp[:, :K, :N], (0, 1, 2))
    cp = None
    cs = (0, 0, 0)
    if c0 is not None:
        cv = torch.as_strided(c0, (batch, M, N), c_strides, c0.storage_offset())
        cp = torch.zeros((batch, M, np_), dtype=c0.dtype, device=dev)
        permute(cv, cp[:, :, :N], (0, 1, 2))
        cs = (M * np_, np_, 1)
    op = torch.empty((batch, M, np_), dtype=out.dtype, device=dev)
    _trace.in_pad = True     # thread-local: the padded call must not pad again
    try:
        kind = contract_raw(ap, (M * kp, kp, 1), bp, (kp * np_, np_, 1), op, (M * np_, np_, 1),
                            batch=batch, M=M, N=np_, K=kp, c0=cp, c_strides=cs,
                            mode="tc" if mode == "auto" else mode, schedule=schedule)
    finally:
        _trace.in_pad = False
    ov = torch.as_strided(out, (batch, M, N), o_strides, out.storage_offset())
    permute(op[:, :, :N], ov, (0, 1, 2))
    return kind


# ---------------------------------------------------------------------------
# plan execution

def _materialise(t: torch.Tensor, tup, group_axes) -> torch.Tensor:
    """Copy ``t`` (indexed by ``tup``) into a contiguous tensor whose dims are
    the concatenation of ``group_axes`` (a permute pre-pass on the device)."""
    order = [a for g in group_axes for a in g]
    perm = [tup.index(a) for a in order]
    dst = torch.empty([t.shape[p] for p in perm], dtype=t.dtype, device=t.device)
    return permute(t, dst, perm), tuple(order)


def _group_strides(t, tup, view_axes, ext):
    from .plan import flatten_group
    by = dict(zip(tup, t.stride()))
    return tuple(flatten_group(g, ext, by) if g else 0 for g in view_axes)


def run_gemm(p: GemmPlan, spec: EinsumSpec, inputs, c0, out, *, mode, schedule):
    ext = extents_of(spec, [t.shape for t in inputs] + [out.shape])
    a, b = inputs[p.a], inputs[p.b]
    a_tup, b_tup = spec.inputs[p.a], spec.inputs[p.b]
    if p.a_view.needs_copy:
        a, a_tup = _materialise(a, a_tup, p.a_view.axes)
    if p.b_view.needs_copy:
        b, b_tup = _materialise(b, b_tup, p.b_view.axes)
    sa = _group_strides(a, a_tup, p.a_view.axes, ext)
    sb = _group_strides(b, b_tup, p.b_view.axes, ext)
    o_tup = spec.output
    tmp_out = out
    so = _group_strides(out, o_tup, p.o_view.axes, ext)
    if any(s is None for s in so):
        order = [x for g in p.o_view.axes for x in g]
        tmp_out = torch.empty([ext[x] for x in order], dtype=out.dtype, device=out.device)
        o_tup = tuple(order)
        so = _group_strides(tmp_out, o_tup, p.o_view.axes, ext)
    sc = (0, 0, 0)
    if c0 is not None:
        c_tup = spec.output
        sc = _group_strides(c0, c_tup, p.o_view.axes, ext)
        if any(s is None for s in sc):
            c0, c_tup = _materialise(c0, c_tup, p.o_view.axes)
            sc = _group_strides(c0, c_tup, p.o_view.axes, ext)
    contract_raw(a, sa, b, sb, tmp_out, so, batch=p.batch, M=p.M, N=p.N, K=p.K, c0=c0,
                 c_strides=sc, mode=mode, schedule=schedule)
    if tmp_out is not out:
        perm = [o_tup.index(x) for x in spec.output]
        permute(tmp_out, out, perm)
    return out


def _step_spec(lhs_axes, rhs_axes, out_axes) -> EinsumSpec:
    seen = list(dict.fromkeys((*lhs_axes, *rhs_axes)))
    axes = tuple(out_axes) + tuple(a for a in seen if a not in out_axes)
    return EinsumSpec((tuple(lhs_axes), tuple(rhs_axes)), tuple(out_axes), axes)


def run_chain(p: ChainPlan, spec: EinsumSpec, inputs, c0, out, *, mode, schedule):
    ext = extents_of(spec, [t.shape for t in inputs] + [out.shape])
    temps = []
    for i, st in enumerate(p.steps):
        last = i == len(p.steps) - 1
        lhs = inputs[st.lhs] if isinstance(st.lhs, int) else temps[st.lhs[1]]
        rhs = inputs[st.rhs] if isinstance(st.rhs, int) else temps[st.rhs[1]]
        sspec = _step_spec(st.lhs_axes, st.rhs_axes, st.out_axes)
        dst = out if last else torch.empty([ext[a] for a in st.out_axes], dtype=out.dtype,
                                           device=out.device)
        execute(sspec, [lhs, rhs], c0 if last else None, dst, mode=mode, schedule=schedule)
        temps.append(dst)
    return out


def _exec_key(spec, inputs, c0, out, mode, chain_order):
    """Everything a plain GEMM launch decision depends on (shapes, strides,
    dtypes, devices, 16-byte alignment of every pointer, mode)."""
    parts = [spec, mode, chain_order, out.dtype, out.device,
             (out.shape, out.stride(), out.data_ptr() % 16)]
    for t in inputs:
        parts.append((t.shape, t.stride(), t.dtype, t.device, t.data_ptr() % 16))
    parts.append(None if c0 is None else
                 (c0.shape, c0.stride(), c0.dtype, c0.device, c0.data_ptr() % 16))
    return tuple(parts)


def _exec_cache() -> dict:
    if not hasattr(_trace, "exec_cache"):
        _trace.exec_cache = {}
    return _trace.exec_cache


def fast_launcher(spec, inputs, c0, out, mode: str = "auto", chain_order: str = "auto"):
    """The cached launcher ``execute`` uses for this exact call signature
    (shapes, strides, dtypes, devices, pointer alignment, mode), or None when
    the signature has none (not yet run, or a path without one).  Called as
    ``launcher(inputs, out, c0)``."""
    return _exec_cache().get(_exec_key(spec, inputs, c0, out, mode, chain_order))


def gemm_descriptor(plan, spec, inputs, c0, out, mode):
    """A complete ``bgx_contract_desc`` for a plain GEMM plan — no operand
    copy, no output permute, no split-K workspace, no padding — or None when
    the plan needs any of those (the planner's full path handles it).
    Returns ``(desc, kind)``."""
    if plan.a_view.needs_copy or plan.b_view.needs_copy or mode == "tf32":
        return None
    ext = extents_of(spec, [t.shape for t in inputs] + [out.shape])
    so = _group_strides(out, spec.output, plan.o_view.axes, ext)
    sc = (0, 0, 0) if c0 is None else _group_strides(c0, spec.output, plan.o_view.axes, ext)
    if any(x is None for x in (*so, *sc)):
        return None
    ia, ib = plan.a, plan.b
    sa = _group_strides(inputs[ia], spec.inputs[ia], plan.a_view.axes, ext)
    sb = _group_strides(inputs[ib], spec.inputs[ib], plan.b_view.axes, ext)
    lib = _lib.load()
    d = _lib.BgxContractDesc()
    d.batch, d.M, d.N, d.K = plan.batch, plan.M, plan.N, plan.K
    for i in range(3):
        d.a_stride[i], d.b_stride[i], d.c_stride[i], d.o_stride[i] = sa[i], sb[i], sc[i], so[i]
    d.in_dtype = TORCH_TO_BGX[inputs[0].dtype]
    d.out_dtype = TORCH_TO_BGX[out.dtype]
    d.mode = MODES[mode]
    d.a, d.b, d.out = inputs[ia].data_ptr(), inputs[ib].data_ptr(), out.data_ptr()
    d.c0 = c0.data_ptr() if c0 is not None else None
    with _on_device(out.device):
        kind = lib.bgx_contract_kernel(d)
        if kind < 0 or (kind == _lib.KERNEL_SIMT16 and mode == "auto"
                        and 2 * plan.batch * plan.M * plan.N * plan.K >= PAD_MIN_FLOP):
            return None
        if kind == _lib.KERNEL_TC:
            sp, ws = _lib._i32(1), _lib._i64(0)
            _lib.check(lib.bgx_contract_splitk_plan(d, sp, ws), "bgx_contract_splitk_plan")
            if sp.value != 1:
                return None
    return d, kind


def _fast_gemm(plan, spec, inputs, c0, out, mode, log: bool = True):
    """Pre-built descriptor for a plain GEMM (``gemm_descriptor``): later
    calls with the same signature patch the pointers and call bgx_contract
    directly — what ``prepare()`` does (it builds its GEMM launcher here too),
    applied automatically to repeated ``execute`` calls (the reference-shaped
    ``run_function`` path of BASELINE config 1)."""
    got = gemm_descriptor(plan, spec, inputs, c0, out, mode)
    if got is None:
        return None
    d, kind = got
    ia, ib = plan.a, plan.b
    lib = _lib.load()
    launch = lib.bgx_contract
    name = _lib.KERNEL_NAMES.get(kind, "contract")
    dev_index = out.device.index

    def run(xs, o, c):
        d.a, d.b, d.out = xs[ia].data_ptr(), xs[ib].data_ptr(), o.data_ptr()
        d.c0 = c.data_ptr() if c is not None else None
        if (_raw_stream is not None and getattr(_trace, "events", None) is None
                and torch.cuda.current_device() == dev_index):
            # common case (no event tracing, right device): straight to the C ABI
            rc = launch(d, _raw_stream(dev_index))
            if rc:
                _lib.check(rc, "bgx_contract")
        else:
            with _on_device(o.device):
                e0 = _ev_begin(o)
                _lib.check(launch(d, _stream_ptr(o)), "bgx_contract")
                _ev_end(e0, name, o)
        if log:
            _log(name)
    return run


def _fast_permute(x, out, perm):
    """Pre-built bgx_tensor pair for a repeated permutation signature."""
    lib = _lib.load()
    ti, to = _lib.BgxTensor(), _lib.BgxTensor()
    for t, desc in ((x, ti), (out, to)):
        desc.dtype, desc.rank = TORCH_TO_BGX[t.dtype], t.dim()
        for d in range(t.dim()):
            desc.shape[d], desc.stride[d] = t.shape[d], t.stride(d)
    p = (_lib._i32 * max(1, len(perm)))(*perm)

    def run(xs, o, c):
        ti.data, to.data = xs[0].data_ptr(), o.data_ptr()
        with _on_device(o.device):
            _lib.check(lib.bgx_permute(ti, to, p, _stream_ptr(o)), "bgx_permute")
        _log("permute")
    return run


def _spec_of(inputs, output) -> EinsumSpec:
    """EinsumSpec for index tuples (axis order of einsum.py:81: output
    indices, then input-only ones in first-appearance order)."""
    seen = list(dict.fromkeys(a for t in inputs for a in t))
    axes = tuple(output) + tuple(a for a in seen if a not in output)
    return EinsumSpec(tuple(tuple(t) for t in inputs), tuple(output), axes)


def _private_axes(spec: EinsumSpec) -> dict:
    """Input k -> its reduction axes that no other operand carries."""
    res = {}
    for k, tup in enumerate(spec.inputs):
        others = set(spec.output)
        for j, t2 in enumerate(spec.inputs):
            if j != k:
                others.update(t2)
        priv = [a for a in tup if a not in others]
        if priv:
            res[k] = priv
    return res


def _tolerance(mode: str, dt) -> bool:
    """Paths free to reorder sums: FFMA mode, and 16-bit storage in auto mode
    (no reference arithmetic exists for it)."""
    return mode == "ffma" or (mode == "auto" and dt in (torch.bfloat16, torch.float16))


def _prereduce(spec, inputs, mode):
    """Tolerance paths: sum each input over the reduction axes only it
    carries before it meets the others — sum_{d,b,c} x[d,a] y[d,b,c] =
    sum_d x[d,a] (sum_{b,c} y[d,b,c]) — so no kernel walks the product space
    of unrelated axes.  Returns the reduced (spec, inputs) or None."""
    priv = _private_axes(spec)
    if len(spec.inputs) < 2 or not priv:
        return None
    if inputs[0].dtype in (torch.bfloat16, torch.float16):
        # 16-bit: the reduced operand is stored at 16 bits (one more rounding
        # of an intermediate), so only where the product space dwarfs the
        # operands (>= PREREDUCE_16BIT_BLOWUP x) — there the direct walk is
        # the pathological part
        ext = extents_of(spec, [t.shape for t in inputs])
        pts = 1
        for e in ext.values():
            pts *= e
        if pts < PREREDUCE_16BIT_BLOWUP * sum(t.numel() for t in inputs):
            return None
    new_tups, new_ins = [], []
    for k, (tup, x) in enumerate(zip(spec.inputs, inputs)):
        if k not in priv:
            new_tups.append(tup)
            new_ins.append(x)
            continue
        keep = tuple(a for a in tup if a not in priv[k])
        sub = _spec_of([tup], keep)
        y = torch.empty([x.shape[tup.index(a)] for a in keep], dtype=x.dtype, device=x.device)
        execute(sub, [x], None, y, mode=mode)
        new_tups.append(keep)
        new_ins.append(y)
    return _spec_of(new_tups, spec.output), new_ins


def execute(spec: EinsumSpec, inputs, c0: torch.Tensor | None, out: torch.Tensor, *,
            mode: str = "auto", schedule=None, chain_order: str = "auto"):
    """Run one generic op into ``out`` (fresh, contiguous-or-strided device
    tensor).  ``c0`` is the initial output (None = zeros); ignored by a
    passthrough body, exactly as in the reference (einsum.py:105-108)."""
    key = None
    if schedule is None and all(isinstance(t, torch.Tensor) and t.is_cuda for t in inputs) \
            and out.is_cuda and (c0 is None or c0.is_cuda):
        key = _exec_key(spec, inputs, c0, out, mode, chain_order)
        fast = _exec_cache().get(key)
        if fast is not None:
            fast(inputs, out, c0)
            return out
    _check_device(list(inputs) + [c0, out])
    dt = out.dtype
    for t in inputs:
        if t.dtype != dt:
            raise TypeError("operands must share one element type")
    if _tolerance(mode, dt) and len(inputs) >= 2:
        red = _prereduce(spec, inputs, mode)
        if red is not None:
            return execute(red[0], red[1], c0, out, mode=mode, schedule=schedule,
                           chain_order=chain_order)
    shapes = [tuple(t.shape) for t in inputs] + [tuple(out.shape)]
    strides = [tuple(t.stride()) for t in inputs] + [tuple(out.stride())]
    plan = plan_generic(spec, shapes, strides, dtype=DTYPE_NAME[dt], mode=mode,
                        chain_order=chain_order)
    if isinstance(plan, PermutePlan):
        permute(inputs[0], out, plan.perm)
        if key is not None:
            _cache_put(_exec_cache(), key, _fast_permute(inputs[0], out, plan.perm))
        return out
    if isinstance(plan, GenericPlan):
        # tolerance mode: tree reductions; 16-bit storage (no reference
        # arithmetic to reproduce) also takes them once each output sums
        # TREE_16BIT_POINTS or more points — shorter reductions keep the
        # sequential f32 chain (bit-equal to the oracle on widened inputs)
        tree = mode == "ffma"
        if not tree and mode == "auto" and dt in (torch.bfloat16, torch.float16):
            red_pts = 1
            for a, e in extents_of(spec, [t.shape for t in inputs] + [out.shape]).items():
                if a not in spec.output:
                    red_pts *= e
            tree = red_pts >= TREE_16BIT_POINTS
        if tree:
            ro = _tree_output_order(spec, inputs)
            if ro is not None:
                # the tree kernels' column layout needs the streamed input's
                # contiguous axis innermost in the OUTPUT: reduce into that
                # order, then move the (small) result
                spec2, to_out = ro
                ext = extents_of(spec, [t.shape for t in inputs])
                tmp = torch.empty([ext[a] for a in spec2.output], dtype=dt, device=out.device)
                c0p = None if c0 is None else \
                    c0.permute([spec.output.index(a) for a in spec2.output]).contiguous()
                generic(spec2, inputs, c0p, tmp, tree=True)
                return permute(tmp, out, to_out)
        if out.is_contiguous():
            generic(spec, inputs, c0, out, tree=tree)
            if key is not None:
                fast = _fast_generic_materialized(spec, inputs, c0, out, tree) \
                    if _transposed_inputs(spec, inputs, out) else _fast_generic(spec, inputs, c0, out, tree)
                if fast is not None:
                    _cache_put(_exec_cache(), key, fast)
            return out
        tmp = torch.empty(out.shape, dtype=dt, device=out.device)
        generic(spec, inputs, c0, tmp, tree=tree)
        return permute(tmp, out, list(range(out.dim())))
    if isinstance(plan, GemmPlan):
        run_gemm(plan, spec, inputs, c0, out, mode=mode, schedule=schedule)
        if key is not None and dt == inputs[0].dtype:
            fast = _fast_gemm(plan, spec, inputs, c0, out, mode)
            if fast is not None:
                _cache_put(_exec_cache(), key, fast)
        return out
    if isinstance(plan, ChainPlan):
        return run_chain(plan, spec, inputs, c0, out, mode=mode, schedule=schedule)
    raise AssertionError(plan)


def gemm_plan_for(spec: EinsumSpec, inputs, out):
    """The GEMM plan of a 2-input contraction regardless of the planner's
    preference for other kernels (widened outputs exist only on the GEMM
    path), or None when the body has no batch/M/N/K structure."""
    from .plan import classify_two, plan_gemm
    if len(inputs) != 2:
        return None
    shapes = [tuple(t.shape) for t in inputs] + [tuple(out.shape)]
    strides = [tuple(t.stride()) for t in inputs] + [tuple(out.stride())]
    ext = extents_of(spec, shapes)
    groups = classify_two(spec, ext)
    if isinstance(groups, str):
        return None
    return plan_gemm(spec, ext, strides, groups)


def plan_for(spec: EinsumSpec, inputs, out, *, mode="auto", chain_order="auto"):
    shapes = [tuple(t.shape) for t in inputs] + [tuple(out.shape)]
    strides = [tuple(t.stride()) for t in inputs] + [tuple(out.stride())]
    return plan_generic(spec, shapes, strides, dtype=DTYPE_NAME[out.dtype], mode=mode,
                        chain_order=chain_order)
