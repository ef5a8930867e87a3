"""Real GPU execution of the GPU case study's kernels.

bridgegen runs a FIR GPU kernel by simulating the thread grid: one fresh
interpreter per (block, thread) coordinate, sequentially, in lexicographic or
reversed order (/root/reference/pkg/src/bridgegen/interp.py:434-461).  Here the
kernel's IR (``func.func`` with ``gpu.*``, ``memref.*``, ``arith.*``,
``math.exp`` and ``cf.*`` ops — what bridgegen's codegen produces from FIR,
gpu.py:64-96) is translated to CUDA C, compiled by NVRTC for sm_100a
(``bgx_rtc_compile``) and launched for real (``bgx_rtc_launch``): one device
thread per logical (block, thread) coordinate.

Kept from the reference ``run_kernel``:
  * signature ``run_kernel(module, symbol, launch, inputs, step_limit, reverse)``
    and the returned ``inputs`` list with memref data updated in place;
  * arity / type checks and messages of ``_Machine.call`` (interp.py:211-221);
  * ``OutOfBounds`` with the reference message, reported for the FIRST
    offending coordinate in the reference's visiting order (``reverse``
    honoured), including the thread-context dict (interp.py:359-370);
  * the per-thread step budget (a fresh budget per coordinate, ticking one per
    op) → ``StepLimitExceeded`` — so a runaway kernel cannot hang the GPU;
  * IEEE binary32/64 arithmetic per op (NVRTC ``--fmad=false -ftz=false``):
    results equal the reference's for race-free kernels (vadd, the naive GEMM
    of SURVEY A.3 — pinned by tests/test_gpu_fir.py).
Differences: all coordinates run concurrently, so kernels with write races
behave like real GPUs (the reference is order-dependent there); after an
error the memref buffers are left unchanged (the reference leaves the partial
state of the coordinates it visited before the failing one); ``math.exp`` uses
CUDA's ``expf``/``exp`` (within 2 ulp of numpy's).
"""

from __future__ import annotations

import ctypes
import hashlib
import struct
import threading

import numpy as np
import torch

from . import _lib

_ERR_SLOTS = 1024
_cache = {}
_cache_lock = threading.Lock()


class TranslationError(Exception):
    pass


def _tname(t) -> str:
    return type(t).__name__


def _ctype(t) -> str:
    n = _tname(t)
    if n == "Float32Type":
        return "float"
    if n == "Float64Type":
        return "double"
    if n in ("IntType", "IndexType"):
        return "i64"
    raise TranslationError(f"no device scalar type for {t}")


def _wrap(expr: str, t) -> str:
    """Two's-complement wrap of an i64 expression to IntType(width)
    (interp.py:76-80); index values are unbounded in the reference and i64
    here."""
    if _tname(t) != "IntType":
        return expr
    w = t.width
    if w == 1:
        return f"((i64)(({expr}) & 1))"
    if w >= 64:
        return f"((i64)({expr}))"
    return f"((i64)((unsigned long long)({expr}) << {64 - w}) >> {64 - w})"


def _fconst(value: float, t) -> str:
    if _tname(t) == "Float32Type":
        bits = struct.unpack("<I", struct.pack("<f", float(np.float32(value))))[0]
        return f"__int_as_float(0x{bits:08x})"
    bits = struct.unpack("<Q", struct.pack("<d", float(value)))[0]
    return f"__longlong_as_double(0x{bits:016x}LL)"


_CMP = {"eq": "==", "ne": "!=", "slt": "<", "sle": "<=", "sgt": ">", "sge": ">="}


def translate(func, kernel_name: str = "bgx_fir_kernel"):
    """CUDA C source for one IR ``func.func`` kernel; returns (source,
    param_kinds) where param_kinds[i] is ('memref', rank, ctype) or
    ('scalar', ctype)."""
    region = func.regions[0]
    fty = func.attributes["function_type"].type
    params, kinds = [], []
    for i, t in enumerate(fty.inputs):
        if _tname(t) == "MemRefType":
            ct = _ctype(t.elem)
            params.append(f"{ct}* __restrict__ p{i}")
            params += [f"i64 p{i}_d{d}" for d in range(t.rank)]
            kinds.append(("memref", t.rank, ct))
        else:
            params.append(f"{_ctype(t)} p{i}")
            kinds.append(("scalar", _ctype(t)))
    names = {}
    decls = []

    def var(v):
        if id(v) not in names:
            names[id(v)] = f"v{len(names)}"
            decls.append(f"  {_ctype(v.type)} {names[id(v)]} = 0;")
        return names[id(v)]

    entry = region.blocks[0]
    for i, a in enumerate(entry.arguments):
        names[id(a)] = f"p{i}"
    memref_rank = {id(a): t.rank for a, t in zip(entry.arguments, fty.inputs)
                   if _tname(t) == "MemRefType"}
    body = []
    site = 0
    labels = {id(b): f"B{k}" for k, b in enumerate(region.blocks)}

    def jump(succ, indent):
        out = []
        tmps = []
        for k, (formal, actual) in enumerate(zip(succ.block.arguments, succ.args)):
            tmp = f"t_{labels[id(succ.block)]}_{k}"
            out.append(f"{indent}{_ctype(formal.type)} {tmp} = {var(actual)};")
            tmps.append((formal, tmp))
        for formal, tmp in tmps:
            out.append(f"{indent}{var(formal)} = {tmp};")
        out.append(f"{indent}goto {labels[id(succ.block)]};")
        return out

    for blk in region.blocks:
        body.append(f"{labels[id(blk)]}: {{")
        for op in blk.operations:
            # tick, then execute (interp.py:231-233): a step-limit overrun
            # and an out-of-bounds access in one block raise what the
            # reference raises
            body.append("  if (++steps > step_limit) "
                        "{ bgx_report(hdr, tab, key, 2, 0, 0, 0, 0); return; }")
            name = op.name
            res = op.results[0] if op.results else None
            o = [var(x) for x in op.operands]
            if name == "arith.constant":
                attr = op.attributes["value"]
                if _tname(attr) == "FloatAttr":
                    body.append(f"  {var(res)} = {_fconst(attr.value, res.type)};")
                else:
                    body.append(f"  {var(res)} = {_wrap(f'(i64){int(attr.value)}LL', res.type)};")
            elif name in ("arith.addf", "arith.subf", "arith.mulf", "arith.divf"):
                sym = {"arith.addf": "+", "arith.subf": "-", "arith.mulf": "*", "arith.divf": "/"}[name]
                body.append(f"  {var(res)} = {o[0]} {sym} {o[1]};")
            elif name == "arith.negf":
                body.append(f"  {var(res)} = -{o[0]};")
            elif name == "math.exp":
                fn = "expf" if _tname(res.type) == "Float32Type" else "exp"
                body.append(f"  {var(res)} = {fn}({o[0]});")
            elif name in ("arith.addi", "arith.subi", "arith.muli"):
                sym = {"arith.addi": "+", "arith.subi": "-", "arith.muli": "*"}[name]
                expr = f"(i64)((unsigned long long){o[0]} {sym} (unsigned long long){o[1]})"
                body.append(f"  {var(res)} = {_wrap(expr, res.type)};")
            elif name == "arith.cmpi":
                pred = op.attributes["predicate"].text
                if pred not in _CMP:
                    raise TranslationError(f"unknown cmpi predicate '{pred}'")
                body.append(f"  {var(res)} = ({o[0]} {_CMP[pred]} {o[1]}) ? 1 : 0;")
            elif name == "arith.index_cast":
                body.append(f"  {var(res)} = {_wrap(o[0], res.type)};")
            elif name in ("gpu.thread_id", "gpu.block_id", "gpu.block_dim"):
                dim = op.attributes["dimension"].text
                src = {"gpu.thread_id": "t", "gpu.block_id": "bk", "gpu.block_dim": "bd"}[name]
                body.append(f"  {var(res)} = {src}{dim};")
            elif name in ("memref.load", "memref.store"):
                buf_i = 0 if name == "memref.load" else 1
                buf = op.operands[buf_i]
                idx = o[buf_i + 1:]
                if id(buf) not in memref_rank:
                    raise TranslationError("memref operand is not a kernel argument")
                rank = memref_rank[id(buf)]
                if len(idx) != rank:
                    raise TranslationError(f"rank mismatch: {len(idx)} indices for rank {rank}")
                p = names[id(buf)]
                lin = "0"
                for d, ix in enumerate(idx):
                    body.append(f"  if ({ix} < 0 || {ix} >= {p}_d{d}) "
                                f"{{ bgx_report(hdr, tab, key, 1, {site}, {d}, {ix}, {p}_d{d}); return; }}")
                    lin = f"({lin}) * {p}_d{d} + {ix}"
                if name == "memref.load":
                    body.append(f"  {var(res)} = {p}[{lin}];")
                else:
                    body.append(f"  {p}[{lin}] = {o[0]};")
                site += 1
            elif name == "cf.br":
                body += jump(op.successors[0], "  ")
            elif name == "cf.cond_br":
                body.append(f"  if ({o[0]}) {{")
                body += jump(op.successors[0], "    ")
                body.append("  } else {")
                body += jump(op.successors[1], "    ")
                body.append("  }")
            elif name == "func.return":
                body.append("  return;")
            else:
                raise TranslationError(f"unsupported operation '{name}'")
        body.append("}")
    src = [
        "typedef long long i64;",
        "struct ErrRec { unsigned long long key; i64 kind, site, dim, index, extent; };",
        "__device__ __forceinline__ void bgx_report(unsigned long long* hdr, ErrRec* tab,",
        "    unsigned long long key, i64 kind, i64 site, i64 dim, i64 index, i64 extent) {",
        "  unsigned long long slot = atomicAdd(&hdr[0], 1ULL);",
        "  atomicMin(&hdr[1], key);",
        f"  if (slot < {_ERR_SLOTS}ULL) {{ ErrRec r = {{key, kind, site, dim, index, extent}};"
        " tab[slot] = r; }",
        "}",
        f'extern "C" __global__ void {kernel_name}(' + ", ".join(
            params + ["unsigned long long* hdr", "ErrRec* tab", "i64 step_limit",
                      "unsigned long long total", "int reverse",
                      "i64 gx", "i64 gy", "i64 gz", "i64 bx", "i64 by", "i64 bz",
                      "unsigned long long only"]) + ") {",
        "  unsigned long long L = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;",
        "  if (L >= total) return;",
        # re-run of the single first-failing coordinate (see run_kernel)
        "  if (only != ~0ULL && (reverse ? total - 1 - L : L) != only) return;",
        # visiting order of interp.py:445-451: block x,y,z then thread x,y,z
        "  unsigned long long r = L;",
        "  i64 tz = r % bz; r /= bz; i64 ty = r % by; r /= by; i64 tx = r % bx; r /= bx;",
        "  i64 bkz = r % gz; r /= gz; i64 bky = r % gy; r /= gy; i64 bkx = (i64)r;",
        "  i64 bdx = bx, bdy = by, bdz = bz;",
        "  unsigned long long key = reverse ? total - 1 - L : L;",
        "  i64 steps = 0;",
        *decls,
        "  goto B0;",
        *body,
        "}",
    ]
    return "\n".join(src) + "\n", kinds


def _compile(src: str, name: str):
    h = hashlib.sha256(src.encode()).hexdigest()
    dev = torch.cuda.current_device()
    with _cache_lock:
        hit = _cache.get((h, dev))
        if hit is not None:
            return hit
    lib = _lib.load()
    handle = ctypes.c_void_p()
    log = ctypes.create_string_buffer(4096)
    _lib.check(lib.bgx_rtc_compile(src.encode(), name.encode(), ctypes.byref(handle), log, 4096),
               "bgx_rtc_compile")
    with _cache_lock:
        _cache[(h, dev)] = handle
    return handle


_TORCH = {"float": torch.float32, "double": torch.float64, "i64": torch.int64}


def run_kernel(module, symbol, launch, inputs, step_limit=None, reverse=False):
    """Drop-in for bridgegen ``interp.run_kernel`` executing on the B200."""
    from bridgegen import interp  # the reference's error types and values
    if step_limit is None:
        step_limit = interp.DEFAULT_STEP_LIMIT
    func = module.lookup_symbol(symbol)
    if func is None or func.name != "func.func":
        raise interp.InterpError(f"no function @{symbol} in the module")
    fty = func.attributes["function_type"].type
    inputs = list(inputs)
    if len(inputs) != len(fty.inputs):
        raise interp.InterpError(
            f"@{symbol} takes {len(fty.inputs)} argument(s), got {len(inputs)}")
    for i, (t, v) in enumerate(zip(fty.inputs, inputs)):
        interp._check_compatible(t, v, f"@{symbol} argument {i}")
    gx, gy, gz = launch.grid
    bx, by, bz = launch.block
    total = gx * gy * gz * bx * by * bz
    try:
        src, kinds = translate(func)
    except TranslationError as e:
        raise interp.InterpError(str(e)) from e
    handle = _compile(src, "bgx_fir_kernel")
    dev = torch.device("cuda", torch.cuda.current_device())
    lib = _lib.load()
    stream = torch.cuda.current_stream(dev).cuda_stream

    def launch(only):
        """One launch over all coordinates (``only`` = -1) or over the single
        coordinate whose visiting-order key is ``only``; fresh device copies
        of the memrefs every time (returns them and the error header/table)."""
        keep, args = [], []
        for v, kind in zip(inputs, kinds):
            if kind[0] == "memref":
                t = torch.from_numpy(np.ascontiguousarray(v.data)).to(dev)
                keep.append(t)
                args.append(ctypes.c_void_p(t.data_ptr()))
                args += [ctypes.c_int64(int(e)) for e in v.data.shape]
            else:
                val = v.value
                args.append(ctypes.c_float(val) if kind[1] == "float" else
                            ctypes.c_double(val) if kind[1] == "double" else ctypes.c_int64(int(val)))
        hdr = torch.tensor([0, (1 << 63) - 1], dtype=torch.int64, device=dev)
        tab = torch.zeros((_ERR_SLOTS, 6), dtype=torch.int64, device=dev)
        args += [ctypes.c_void_p(hdr.data_ptr()), ctypes.c_void_p(tab.data_ptr()),
                 ctypes.c_int64(int(step_limit)), ctypes.c_uint64(total),
                 ctypes.c_int32(1 if reverse else 0)]
        args += [ctypes.c_int64(e) for e in (gx, gy, gz, bx, by, bz)]
        args.append(ctypes.c_uint64(only & 0xFFFFFFFFFFFFFFFF))
        argv = (ctypes.c_void_p * len(args))(
            *[ctypes.cast(ctypes.pointer(a), ctypes.c_void_p) for a in args])
        block = 256
        grid = (total + block - 1) // block
        _lib.check(lib.bgx_rtc_launch(handle, grid, block, argv, stream), "bgx_rtc_launch")
        torch.cuda.synchronize(dev)
        return keep, hdr, tab

    keep, hdr, tab = launch(-1)
    count = int(hdr[0].item())
    if count:
        first = int(hdr[1].item())
        rows = tab[:min(count, _ERR_SLOTS)].cpu().numpy()
        hits = [r for r in rows if int(r[0]) == first]
        if not hits:
            # more failing coordinates than record slots and the first one's
            # record was dropped: re-run that coordinate alone (its own
            # fresh budget and inputs, as the reference would visit it)
            _, _, tab1 = launch(first)
            hits = [tab1[0].cpu().numpy()]
        key, kind, _site, dim, index, extent = (int(x) for x in hits[0])
        lin = (total - 1 - key) if reverse else key
        tz, r = lin % bz, lin // bz
        ty, r = r % by, r // by
        tx, r = r % bx, r // bx
        bkz, r = r % gz, r // gz
        bky, bkx = r % gy, r // gy
        ctx = {"x": (tx, bkx, bx), "y": (ty, bky, by), "z": (tz, bkz, bz)}
        if kind == 2:
            raise interp.StepLimitExceeded(f"step budget of {step_limit} operations exceeded")
        raise interp.OutOfBounds(
            f"index {index} out of bounds for dimension {dim} of extent {extent} "
            f"(thread context {ctx})")
    for v, kind, t in zip([v for v, k in zip(inputs, kinds) if k[0] == "memref"],
                          [k for k in kinds if k[0] == "memref"], keep):
        np.copyto(v.data, t.cpu().numpy().reshape(v.data.shape))
    return inputs
