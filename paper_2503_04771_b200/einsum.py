"""Einsum DSL → ``linalg.generic`` — drop-in mirror of bridgegen's einsum API.

Same names, signatures, semantics and error messages as
/root/reference/pkg/src/bridgegen/einsum.py:
  * ``EinsumError``, ``EinsumSpec``            (einsum.py:27-38)
  * ``parse_einsum(text)``                     (einsum.py:57-82)
  * ``derive_maps(spec)``                      (einsum.py:85-94)
  * ``build_generic(ctx, registry, spec, operands)``   (einsum.py:121-161)
  * ``build_einsum_function(registry, spec, elem, symbol)`` (einsum.py:164-191)
plus ``print_module`` producing the reference printer's text for these modules
(bridgegen ir.py:814-900; pinned by tests/golden/printed_golden.json).

What is built is not the reference's general IR but the part of it the hot
path reads: per generic op the indexing maps, iterator types,
the body's op sequence (``arith.mulf``… ``arith.addf`` ``linalg.yield``, or a
passthrough ``linalg.yield``) and the element type.  ``interp.run_function``
executes these on the GPU.  The IR verifier / FIR front end / codegen are out
of scope (build-time, not on the data-parallel path).

Element types: the reference's f32/f64 plus bf16/f16 — the
tensor-core input types.
"""

from __future__ import annotations

import functools
import itertools
from dataclasses import dataclass, field

__all__ = [
    "EinsumError", "EinsumSpec", "parse_einsum", "derive_maps", "build_generic",
    "build_einsum_function", "IndexMap", "ElemType", "F32", "F64", "BF16", "F16",
    "TensorType", "Value", "GenericOp", "Function", "Module", "FunctionBuilder",
    "print_module", "elem_type",
]


class EinsumError(Exception):
    pass


# ---------------------------------------------------------------------------
# element / tensor types (bridgegen ir.py:71-106 — f32/f64; bf16/f16 added)

@dataclass(frozen=True)
class ElemType:
    name: str
    itemsize: int

    def __str__(self) -> str:
        return self.name


F32 = ElemType("f32", 4)
F64 = ElemType("f64", 8)
BF16 = ElemType("bf16", 2)
F16 = ElemType("f16", 2)
_ELEMS = {e.name: e for e in (F32, F64, BF16, F16)}


def elem_type(x) -> ElemType:
    """Accept our ElemType, a name ('f32'…), or a bridgegen fir/ir type whose
    ``str`` is one of those names (fir.F32 prints as Float32 — mapped too)."""
    if isinstance(x, ElemType):
        return x
    s = str(x)
    aliases = {"Float32": "f32", "Float64": "f64", "BFloat16": "bf16", "Float16": "f16",
               "float32": "f32", "float64": "f64", "bfloat16": "bf16", "float16": "f16"}
    s = aliases.get(s, s)
    if s in _ELEMS:
        return _ELEMS[s]
    raise EinsumError(f"element type {x} is not a float type")


@dataclass(frozen=True)
class TensorType:
    elem: ElemType
    rank: int

    def __str__(self) -> str:
        dims = "?x" * self.rank
        return f"tensor<{dims}{self.elem}>"


@dataclass(frozen=True)
class IndexMap:
    """``IndexMapAttr`` (bridgegen ir.py:182-195): operand dim d reads axis
    ``targets[d]`` of an ``n_axes``-dimensional iteration space."""
    n_axes: int
    targets: tuple

    def __str__(self) -> str:
        axes = ", ".join(f"d{i}" for i in range(self.n_axes))
        tg = ", ".join(f"d{t}" for t in self.targets)
        return f"affine_map<({axes}) -> ({tg})>"


# ---------------------------------------------------------------------------
# spec parsing (einsum.py:31-94)

@dataclass(frozen=True)
class EinsumSpec:
    inputs: tuple   # tuple of index-name tuples
    output: tuple   # index-name tuple
    axes: tuple     # iteration-space axis order (distinct index names)

    def axis_of(self, index: str) -> int:
        return self.axes.index(index)


def _groups(side: str):
    """Contents of ``ws (…) ws [, ws (…) ws]*`` or None when ``side`` has any
    other shape (no nested or stray parentheses)."""
    out = []
    i, n = 0, len(side)
    want_group = True
    while True:
        while i < n and side[i].isspace():
            i += 1
        if want_group:
            if i >= n or side[i] != "(":
                return None
            close = side.find(")", i + 1)
            if close < 0 or "(" in side[i + 1:close]:
                return None
            out.append(side[i + 1:close])
            i = close + 1
            want_group = False
        elif i == n:
            return out
        elif side[i] == ",":
            i += 1
            want_group = True
        else:
            return None


def _is_index_name(s: str) -> bool:
    if not s or not (s[0] == "_" or ("a" <= s[0] <= "z") or ("A" <= s[0] <= "Z")):
        return False
    return all(c == "_" or c.isalnum() for c in s[1:])


def _index_tuple(body: str, what: str) -> tuple:
    names = [part.strip() for part in body.split(",")]
    names = [n for n in names if n]
    for n in names:
        if not _is_index_name(n):
            raise EinsumError(f"bad index name '{n}' in {what}")
    if len(names) != len(set(names)):
        raise EinsumError(
            f"repeated index within one {what} tuple (diagonals unsupported)")
    return tuple(names)


def parse_einsum(text: str) -> EinsumSpec:
    """Parse ``(i,k),(k,j)->(i,j)``; axis order = output indices, then the
    input-only indices in first-appearance order (einsum.py:57-82).
    Results are memoised per text (EinsumSpec is immutable; errors are not
    cached, so every bad spec raises again)."""
    if isinstance(text, str):
        return _parse_cached(text)
    return _parse(text)


def _parse(text: str) -> EinsumSpec:
    if "->" not in text:
        raise EinsumError("einsum spec needs '->'")
    lhs, rhs = text.split("->", 1)
    lhs_groups, rhs_groups = _groups(lhs), _groups(rhs)
    if lhs_groups is None or rhs_groups is None or len(rhs_groups) != 1:
        raise EinsumError(f"cannot parse einsum spec '{text}'")
    inputs = tuple(_index_tuple(g, "input") for g in lhs_groups)
    output = _index_tuple(rhs_groups[0], "output")
    first_seen = list(dict.fromkeys(itertools.chain.from_iterable(inputs)))
    for n in output:
        if n not in first_seen:
            raise EinsumError(f"output index '{n}' does not appear in any input")
    axes = output + tuple(n for n in first_seen if n not in output)
    return EinsumSpec(inputs, output, axes)


_parse_cached = functools.lru_cache(maxsize=4096)(_parse)


def derive_maps(spec: EinsumSpec):
    """(indexing maps for inputs then output, per-axis iterator kinds);
    an axis is parallel iff it appears in the output (einsum.py:85-94)."""
    pos = {a: i for i, a in enumerate(spec.axes)}
    maps = [IndexMap(len(spec.axes), tuple(pos[n] for n in tup))
            for tup in (*spec.inputs, spec.output)]
    iterators = ["parallel" if a in spec.output else "reduction" for a in spec.axes]
    return maps, iterators


def body_ops(spec: EinsumSpec) -> tuple:
    """Op names of the synthesised per-point body (einsum.py:100-118)."""
    n = len(spec.inputs)
    if n == 1 and all(a in spec.output for a in spec.axes):
        return ("linalg.yield",)
    return ("arith.mulf",) * (n - 1) + ("arith.addf", "linalg.yield")


# ---------------------------------------------------------------------------
# module data model (the subset of bridgegen's IrModule the hot path reads)

@dataclass(eq=False)
class Value:
    type: TensorType
    name: str = ""          # "%argN" for function arguments

    def __repr__(self) -> str:
        return f"<value {self.name or '?'} : {self.type}>"


@dataclass(eq=False)
class GenericOp:
    spec: EinsumSpec
    maps: list
    iterators: list
    body: tuple
    elem: ElemType
    operands: list
    results: list = field(default_factory=list)
    name: str = "linalg.generic"
    schedule: object = None   # schedule.Schedule (transform-style tiling parameters)

    @property
    def attributes(self):
        attrs = {"indexing_maps": self.maps, "iterator_types": self.iterators}
        if self.schedule is not None:
            attrs["bgx.schedule"] = str(self.schedule)
        return attrs


@dataclass(eq=False)
class Function:
    symbol: str
    arguments: list
    ops: list = field(default_factory=list)
    returns: list = field(default_factory=list)
    result_types: list = field(default_factory=list)


@dataclass(eq=False)
class Module:
    functions: dict = field(default_factory=dict)

    def lookup_symbol(self, symbol: str):
        return self.functions.get(symbol)


class FunctionBuilder:
    """The ``ctx`` of ``build_generic`` (stands in for codegen.BuilderContext):
    owns one function; ``arguments`` are its SSA parameters."""

    def __init__(self, module: Module, symbol: str, arg_types):
        self.module = module
        args = [Value(t, f"%arg{i}") for i, t in enumerate(arg_types)]
        self.function = Function(symbol, args)
        module.functions[symbol] = self.function

    @property
    def arguments(self):
        return self.function.arguments

    def append(self, op: GenericOp):
        self.function.ops.append(op)

    def ret(self, values):
        self.function.returns = list(values)
        self.function.result_types = [v.type for v in values]


def build_generic(ctx: FunctionBuilder, registry, spec: EinsumSpec, operands,
                  schedule=None) -> GenericOp:
    """One ``linalg.generic``; ``operands`` = input tensors then the output
    (einsum.py:121-161, same checks and messages).  ``registry`` is accepted
    for signature compatibility and unused.  ``schedule`` (optional
    ``schedule.Schedule`` or its string form) pins the kernel variant."""
    if len(operands) != len(spec.inputs) + 1:
        raise EinsumError(
            f"expected {len(spec.inputs)} input(s) plus one output operand, "
            f"got {len(operands)}")
    elem = None
    for v, tup in zip(operands, (*spec.inputs, spec.output)):
        t = getattr(v, "type", None)
        if not isinstance(t, TensorType):
            raise EinsumError(f"operand {v!r} is not a tensor")
        if t.rank != len(tup):
            raise EinsumError(f"operand rank {t.rank} does not match index tuple {tup}")
        if not isinstance(t.elem, ElemType):
            raise EinsumError(f"element type {t.elem} is not a float type")
        if elem is None:
            elem = t.elem
        elif t.elem != elem:
            raise EinsumError("operands must share one element type")
    maps, iterators = derive_maps(spec)
    op = GenericOp(spec, maps, iterators, body_ops(spec), elem, list(operands))
    if schedule is not None:
        from .schedule import Schedule
        op.schedule = schedule if isinstance(schedule, Schedule) else Schedule.parse(str(schedule))
    op.results = [Value(operands[-1].type)]
    ctx.append(op)
    return op


def build_einsum_function(registry, spec: EinsumSpec, elem=F32,
                          symbol: str = "einsum", schedule=None) -> Module:
    """``func.func @symbol(inputs…, out) -> out_type`` holding one generic
    (einsum.py:164-191)."""
    e = elem_type(elem)
    module = Module()
    types = [TensorType(e, len(t)) for t in (*spec.inputs, spec.output)]
    ctx = FunctionBuilder(module, symbol, types)
    op = build_generic(ctx, registry, spec, list(ctx.arguments), schedule=schedule)
    ctx.ret([op.results[0]])
    return module


# ---------------------------------------------------------------------------
# printer (text identical to bridgegen ir.print_module for these modules)

def print_module(module: Module) -> str:
    lines = ["module {"]
    counter = itertools.count()
    for fn in module.functions.values():
        names = {id(a): a.name for a in fn.arguments}
        args = ", ".join(f"{a.name}: {a.type}" for a in fn.arguments)
        res = ", ".join(str(t) for t in fn.result_types)
        lines.append(f"  func.func @{fn.symbol}({args}) -> {res} {{")
        for op in fn.ops:
            rname = f"%{next(counter)}"
            names[id(op.results[0])] = rname
            ins, out = op.operands[:-1], op.operands[-1]
            maps = ", ".join(str(m) for m in op.maps)
            its = ", ".join(f'"{s}"' for s in op.iterators)
            sched = f', bgx.schedule = "{op.schedule}"' if op.schedule is not None else ""
            lines.append(
                f"    {rname} = linalg.generic {{indexing_maps = [{maps}], "
                f"iterator_types = [{its}]{sched}}} ins({', '.join(names[id(v)] for v in ins)} : "
                f"{', '.join(str(v.type) for v in ins)}) outs({names[id(out)]} : {out.type}) {{")
            bargs = [f"%{next(counter)}" for _ in op.operands]
            e = op.elem
            lines.append("      ^bb0(" + ", ".join(f"{b}: {e}" for b in bargs) + "):")
            if op.body == ("linalg.yield",):
                lines.append(f"        linalg.yield {bargs[0]} : {e}")
            else:
                acc = bargs[0]
                for k in range(1, len(ins)):
                    nxt = f"%{next(counter)}"
                    lines.append(f"        {nxt} = arith.mulf {acc}, {bargs[k]} : {e}")
                    acc = nxt
                nxt = f"%{next(counter)}"
                lines.append(f"        {nxt} = arith.addf {acc}, {bargs[-1]} : {e}")
                lines.append(f"        linalg.yield {nxt} : {e}")
            lines.append(f"    }} -> {op.results[0].type}")
        rets = ", ".join(names[id(v)] for v in fn.returns)
        lines.append(f"    return {rets} : {', '.join(str(t) for t in fn.result_types)}")
        lines.append("  }")
    lines.append("}")
    return "\n".join(lines) + "\n"

