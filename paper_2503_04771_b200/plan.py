"""Classify a ``linalg.generic`` (einsum spec + operand layouts) into a kernel
plan — the "index-to-loop lowering chooses the kernel variant" step.

Input is what bridgegen's ``_generic`` reads (interp.py:372-424): the spec's
index tuples (→ indexing maps, einsum.py:85-94), the body kind
(einsum.py:100-118) and the operands' extents; plus what a B200 backend needs
on top: element strides and dtype.  Output is one of

  PermutePlan  passthrough body → ``bgx_permute`` (bit-exact copy);
  GemmPlan     2 inputs whose axes split into batch / M / N / K groups
                → ``bgx_contract``; each group is flattened
               to one extent+stride per operand when the strides compose,
               otherwise the operand is first materialised in group order by
               a permute pre-pass (``needs_copy``);
  GenericPlan  anything else (single-input reductions, Hadamard / outer
               products, A-only reduction axes, rank-0 outputs, 3+ f32/f64 inputs in
               'auto'/'exact' mode) → ``bgx_generic`` (the reference's loop nest on the
               device, bit-exact);
  ChainPlan    3+ 16-bit inputs (or any dtype in a non-exact mode) evaluated
               as pairwise contractions (left-to-right or
               min-flop order) → a sequence of GemmPlans over intermediates.

Everything here is host logic over integers — unit-tested on the CPU
(tests/test_plan.py) — no kernels are launched.
"""

from __future__ import annotations

import functools

from dataclasses import dataclass, field

from .einsum import EinsumSpec

# group names
BATCH, MGRP, NGRP, KGRP = "batch", "m", "n", "k"

# f32/f64 multi-operand specs in 'auto' / 'exact' mode always run the
# reference's unfactored loop nest (bit-exact, interp.py:407-420): pairwise
# evaluation ((a*b) summed, then *c) changes the arithmetic, so it is only
# planned for 16-bit operands or when the caller asks for a non-exact mode
# ('tc', 'tf32', 'ffma', 'simt').  Above this many iteration points the
# exact plan is still chosen but logged as slow (plan.kind says so).
GENERIC_POINT_LIMIT = 1 << 28


@dataclass
class PermutePlan:
    perm: tuple          # output dim d reads input dim perm[d]
    kind: str = "permute"


@dataclass
class GenericPlan:
    reason: str
    kind: str = "generic"


@dataclass
class OperandView:
    """An operand seen as 3 flattened groups (elements strides)."""
    groups: tuple                 # e.g. (BATCH, MGRP, KGRP)
    axes: tuple                   # per group: tuple of index names (group order)
    strides: tuple                # per group flattened stride (None if not flattenable)

    @property
    def needs_copy(self) -> bool:
        return any(s is None for s in self.strides)


@dataclass
class GemmPlan:
    a: int                        # which input is the GEMM "A" (M x K)
    b: int                        # which input is the GEMM "B" (K x N)
    batch_axes: tuple
    m_axes: tuple
    n_axes: tuple
    k_axes: tuple
    batch: int
    M: int
    N: int
    K: int
    a_view: OperandView
    b_view: OperandView
    o_view: OperandView
    kind: str = "gemm"

    @property
    def flops(self) -> int:
        return 2 * self.batch * self.M * self.N * self.K


@dataclass
class ChainStep:
    lhs: object                   # int (input index) or ("t", step index)
    rhs: object
    lhs_axes: tuple
    rhs_axes: tuple
    out_axes: tuple               # intermediate (or final) index tuple
    flops: int


@dataclass
class ChainPlan:
    steps: list = field(default_factory=list)
    order: str = "left"
    kind: str = "chain"

    @property
    def flops(self) -> int:
        return sum(s.flops for s in self.steps)


def _prod(xs) -> int:
    p = 1
    for x in xs:
        p *= int(x)
    return p


def extents_of(spec: EinsumSpec, shapes) -> dict:
    """Axis extents from operand shapes (inputs then output), with the
    reference's consistency rule (interp.py:379-396)."""
    ext = {}
    for shape, tup in zip(shapes, (*spec.inputs, spec.output)):
        for e, n in zip(shape, tup):
            if n in ext and ext[n] != e:
                raise ValueError(f"inconsistent extent for {n}: {ext[n]} vs {e}")
            ext[n] = int(e)
    return ext


def flatten_group(axes, ext, strides_by_axis):
    """One stride for the row-major flattening of ``axes`` (extent-1 axes
    ignored), or None if the operand's strides do not compose."""
    live = [a for a in axes if ext[a] != 1]
    if not live:
        return 0
    s = strides_by_axis[live[-1]]
    for hi, lo in zip(live[-2::-1], live[:0:-1]):
        if strides_by_axis[hi] != strides_by_axis[lo] * ext[lo]:
            return None
    return s


def classify_two(spec: EinsumSpec, ext: dict):
    """Axis groups for a 2-input spec, or a reason string when it is not a
    batch/M/N/K contraction."""
    A, B = set(spec.inputs[0]), set(spec.inputs[1])
    O = set(spec.output)
    batch = [a for a in spec.output if a in A and a in B]
    m = [a for a in spec.output if a in A and a not in B]
    n = [a for a in spec.output if a in B and a not in A]
    k = [a for a in spec.axes if a in A and a in B and a not in O]
    only = [a for a in spec.axes if a not in O and ((a in A) != (a in B))]
    if only:
        return f"reduction axis {only[0]!r} indexes only one input"
    return batch, m, n, k


SMALL_16BIT_DIRECT_POINTS = 1 << 24
SMALL_BATCHED_GEMM = True      # A/B switch
SMALL_BATCHED_MN = 1024        # output elements per batch entry (<= 32 x 32), f32/f64
SMALL_BATCHED_MN_16BIT = 256   # 16-bit: the tensor-core tiles win from 32 x 32 up
SMALL_BATCHED_K = 256
OUTER_TO_LOOP_NEST = True      # A/B switches (outer products: the broadcast elementwise kernel, 1-4x faster than K = 1 GEMM tiles, scripts/r02/outer_ab.py)
SKINNY_TO_LOOP_NEST = True
SKINNY_MN = 8


def plan_generic(spec: EinsumSpec, shapes, strides, *, dtype: str, mode: str = "auto",
                 out_strides=None, chain_order: str = "auto"):
    """Plan one generic op.  ``shapes``/``strides``: per operand (inputs then
    output), element strides.  ``dtype``: 'f32'|'f64'|'bf16'|'f16'.
    ``mode``: 'auto' | 'exact' | 'ffma' | 'tc' | 'simt'.  Plans are pure
    functions of these arguments and are memoised (callers treat them as
    read-only); invalid shapes raise every time."""
    key = (spec, tuple(tuple(s) for s in shapes), tuple(tuple(s) for s in strides), dtype, mode,
           None if out_strides is None else tuple(out_strides), chain_order)
    try:
        return _plan_cached(*key)
    except TypeError:          # unhashable argument: plan without the cache
        return _plan_generic(spec, shapes, strides, dtype=dtype, mode=mode,
                             out_strides=out_strides, chain_order=chain_order)


@functools.lru_cache(maxsize=4096)
def _plan_cached(spec, shapes, strides, dtype, mode, out_strides, chain_order):
    return _plan_generic(spec, shapes, strides, dtype=dtype, mode=mode, out_strides=out_strides,
                         chain_order=chain_order)


def _plan_generic(spec: EinsumSpec, shapes, strides, *, dtype: str, mode: str = "auto",
                  out_strides=None, chain_order: str = "auto"):
    n_in = len(spec.inputs)
    ext = extents_of(spec, shapes)
    all_par = all(a in spec.output for a in spec.axes)
    if n_in == 1 and all_par:
        perm = tuple(spec.inputs[0].index(a) for a in spec.output)
        return PermutePlan(perm)
    ref_types = dtype in ("f32", "f64")
    if n_in == 1:
        return GenericPlan("single-input reduction")
    if n_in >= 3 and all_par:
        return GenericPlan("elementwise product (no reduction)")
    if n_in >= 3:
        points = _prod(ext[a] for a in spec.axes)
        if ref_types and mode in ("auto", "exact"):
            why = "multi-operand body, exact loop nest"
            if points > GENERIC_POINT_LIMIT:
                why += f" ({points} points: pass mode='tf32'/'ffma' for pairwise GEMMs)"
            return GenericPlan(why)
        if mode == "auto" and points <= SMALL_16BIT_DIRECT_POINTS:
            # 16-bit bodies small enough to walk directly: f32 arithmetic over
            # the whole product space and one final rounding — a pairwise
            # chain would round each intermediate to 16 bits, which a body
            # with cancellation turns into > 1e-2 errors
            # (scripts/r02/prereduce_acc.py)
            return GenericPlan("multi-operand 16-bit body, direct loop nest (f32, one rounding)")
        return plan_chain(spec, ext, order=chain_order)
    groups = classify_two(spec, ext)
    if isinstance(groups, str):
        return GenericPlan(groups)
    batch, m, n, k = groups
    if batch and k and SMALL_BATCHED_GEMM and \
            _prod(ext[a] for a in m) * _prod(ext[a] for a in n) <= \
            (SMALL_BATCHED_MN if ref_types else SMALL_BATCHED_MN_16BIT) and \
            _prod(ext[a] for a in k) <= SMALL_BATCHED_K:
        # many tiny matrices: a GEMM tile (>= 128 x 64) would be almost all
        # padding; the loop nest (one chain per output, coalescing walk
        # order, operands reused from cache) moves the bytes instead
        return GenericPlan("small batched GEMM")
    if not k and OUTER_TO_LOOP_NEST:
        # no reduction at all (outer products included): every output is one
        # product, written once — the broadcast elementwise kernel
        # (bcast_ew_kernel) moves the bytes; GEMM tiles with K = 1 were equal
        # to 4x slower (scripts/r02/outer_ab.py, profiles/r02_exact_chains.txt)
        return GenericPlan("outer / elementwise product (no reduction)")
    if ref_types and k and SKINNY_TO_LOOP_NEST and (
            _prod(ext[a] for a in m) <= SKINNY_MN or _prod(ext[a] for a in n) <= SKINNY_MN):
        # exact f32/f64 with at most 8 rows or columns: the SIMT tiles
        # (>= 16 x 32) would be mostly padding
        return GenericPlan("skinny exact GEMM")
    if not k and (not m or not n):
        # Hadamard-type bodies (no reduction, no M x N structure): a GEMM plan
        # would be batch x 1 x 1 x 1 (round 2: a 16-bit 8192^2 Hadamard took
        # 2 s on the SIMT GEMM); the dense/strided elementwise kernels move
        # the bytes at HBM speed.  16-bit: f32 arithmetic, one final rounding
        # (the GEMM path's semantics).  Outer products (M x N, K = 1) stay
        # GEMMs: their tiles write the output at full width.
        return GenericPlan("elementwise product (no reduction)")
    if not ref_types and (_prod(ext[a] for a in m) == 1 or _prod(ext[a] for a in n) == 1):
        # 16-bit matrix-vector / batched dot products: a GEMM with one live
        # row or column per tile (or batch x 1 x 1 x K) wastes the tensor
        # cores; reductions on the generic path (tree sums when long)
        return GenericPlan("matrix-vector / dot products (16-bit)")
    if mode == "ffma" and k and (_prod(ext[a] for a in m) == 1 or _prod(ext[a] for a in n) == 1):
        # tolerance mode: dot products and matrix-vector bodies are block-wide
        # tree reductions (bgx_generic_tree), not GEMM tiles with one live
        # row or column
        return GenericPlan("matrix-vector / dot product (tree reduction)")
    if ref_types and mode in ("auto", "exact") and not batch and k and \
            _prod(ext[a] for a in m) == 1 and _prod(ext[a] for a in n) == 1:
        # a full dot product: one sequential chain (the chain kernel's case)
        return GenericPlan("dot product (one chain)")
    if ref_types and mode in ("auto", "exact") and k and (
            _prod(ext[a] for a in m) == 1 or _prod(ext[a] for a in n) == 1):
        # matrix-vector / batched row dots: one sequential chain per output —
        # the row-reduction kernel's case along contiguous rows or columns,
        # else the loop nest with its coalescing walk order (a GEMM tile
        # would leave all but one row or column of every tile idle: a
        # 4096-batch (1024 x 8) . (8) body took 1.04 ms on SIMT tiles)
        return GenericPlan("matrix-vector (row / column reductions)")
    return plan_gemm(spec, ext, strides, (batch, m, n, k), out_strides)


def _view(groups, axes_per_group, ext, tup, st):
    by_axis = dict(zip(tup, st))
    flat = []
    for axes in axes_per_group:
        flat.append(flatten_group(axes, ext, by_axis) if axes else 0)
    return OperandView(groups, tuple(tuple(a) for a in axes_per_group), tuple(flat))


def plan_gemm(spec, ext, strides, groups, out_strides=None):
    batch, m, n, k = groups
    o_st = strides[-1] if out_strides is None else out_strides
    o_by = dict(zip(spec.output, o_st))
    # The output's unit-stride group becomes N (the epilogue writes rows of N);
    # if that group belongs to input 0, swap the roles of the two inputs.
    a_i, b_i, m_ax, n_ax = 0, 1, m, n
    live = [a for a in spec.output if ext[a] != 1]
    if live and m and n:
        inner = min(live, key=lambda a: o_by[a])
        if inner in m:
            a_i, b_i, m_ax, n_ax = 1, 0, n, m
    a_tup, b_tup = spec.inputs[a_i], spec.inputs[b_i]
    a_view = _view((BATCH, MGRP, KGRP), (batch, m_ax, k), ext, a_tup, strides[a_i])
    b_view = _view((BATCH, KGRP, NGRP), (batch, k, n_ax), ext, b_tup, strides[b_i])
    o_view = _view((BATCH, MGRP, NGRP), (batch, m_ax, n_ax), ext, spec.output, o_st)
    return GemmPlan(a_i, b_i, tuple(batch), tuple(m_ax), tuple(n_ax), tuple(k),
                    _prod(ext[x] for x in batch), _prod(ext[x] for x in m_ax),
                    _prod(ext[x] for x in n_ax), _prod(ext[x] for x in k),
                    a_view, b_view, o_view)


def _pair_out(lhs_axes, rhs_axes, keep):
    """Index tuple of a pairwise intermediate: axes of lhs/rhs still needed
    later (``keep``), in first-appearance order."""
    seen = list(dict.fromkeys((*lhs_axes, *rhs_axes)))
    return tuple(a for a in seen if a in keep)


CHAIN_AUTO_FACTOR = 4


def plan_chain(spec: EinsumSpec, ext: dict, order: str = "left") -> ChainPlan:
    """Pairwise evaluation of a 3+-input contraction.  ``order='left'`` folds
    inputs left to right (the order that shards on the output's leading free
    index with no collective); ``'optimal'`` picks the cheapest binary order
    by exhaustive search (fine for the <= 6 operands the ABI allows);
    ``'auto'`` keeps left to right unless it costs more than
    CHAIN_AUTO_FACTOR x the optimal order (a left fold can build an outer
    product of unrelated operands; BASELINE C5's left order is 1.6x)."""
    if order == "auto":
        left = plan_chain(spec, ext, "left")
        best = plan_chain(spec, ext, "optimal")
        return left if left.flops <= CHAIN_AUTO_FACTOR * best.flops else best
    ins = list(spec.inputs)

    def needed_after(pending):
        keep = set(spec.output)
        for tup in pending:
            keep.update(tup)
        return keep

    if order == "left":
        steps = []
        cur, cur_axes = 0, ins[0]
        for j in range(1, len(ins)):
            keep = needed_after(ins[j + 1:])
            out_axes = _pair_out(cur_axes, ins[j], keep) if j < len(ins) - 1 else spec.output
            all_axes = set(cur_axes) | set(ins[j])
            flops = 2 * _prod(ext[a] for a in all_axes)
            steps.append(ChainStep(cur, j, tuple(cur_axes), tuple(ins[j]), tuple(out_axes), flops))
            cur, cur_axes = ("t", len(steps) - 1), out_axes
        return ChainPlan(steps, "left")

    # 'optimal': dynamic programming over subsets (matrix-chain-style, any shape)
    n = len(ins)
    best = {}
    for i in range(n):
        best[1 << i] = (0, None, tuple(ins[i]))
    full = (1 << n) - 1

    for size in range(2, n + 1):
        for mask in range(1, full + 1):
            if bin(mask).count("1") != size:
                continue
            rest = [ins[i] for i in range(n) if not mask >> i & 1]
            keep = set(spec.output)
            for t in rest:
                keep.update(t)
            sub = (mask - 1) & mask
            while sub:
                other = mask ^ sub
                if sub < other and sub in best and other in best:
                    c1, _, ax1 = best[sub]
                    c2, _, ax2 = best[other]
                    cost = c1 + c2 + 2 * _prod(ext[a] for a in set(ax1) | set(ax2))
                    out_axes = spec.output if mask == full else _pair_out(ax1, ax2, keep)
                    if mask not in best or cost < best[mask][0]:
                        best[mask] = (cost, (sub, other), tuple(out_axes))
                sub = (sub - 1) & mask
    steps = []

    def emit(mask):
        cost, split, axes = best[mask]
        if split is None:
            return next(i for i in range(n) if mask >> i & 1), axes
        l, r = split
        lref, lax = emit(l)
        rref, rax = emit(r)
        flops = 2 * _prod(ext[a] for a in set(lax) | set(rax))
        steps.append(ChainStep(lref, rref, tuple(lax), tuple(rax), tuple(axes), flops))
        return ("t", len(steps) - 1), axes

    emit(full)
    return ChainPlan(steps, "optimal")
