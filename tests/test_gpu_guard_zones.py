"""Guard-zone checks for every kernel class (the in-repo stand-in for
compute-sanitizer memcheck, which the GPU pool refuses —
profiles/r02_sanitizer.txt).

Every operand is a view into a larger buffer whose head and tail are NaN, so
an out-of-bounds READ that feeds an accumulation turns the result NaN (NaN*0
is NaN; hardware TMA zero-fill never touches memory).  Every output is a view
into a buffer whose head and tail hold a sentinel pattern, so an
out-of-bounds WRITE shows as a changed sentinel.  Shapes are ragged (not
multiples of any tile) and each result is compared with torch.einsum in f64.
"""

import math

import pytest
import torch

from paper_2503_04771_b200 import contract

pytestmark = pytest.mark.gpu

GUARD = 4096          # elements each side; multiple of 64 keeps 128-B alignment
SENTINEL = 12345.0


def _guarded(shape, dt, fill, gen, dev):
    n = math.prod(shape)
    base = torch.full((n + 2 * GUARD,), fill, dtype=dt, device=dev)
    view = base[GUARD:GUARD + n].view(shape)
    if gen is not None:
        view.copy_(torch.randn(shape, generator=gen, device=dev))
    return base, view


def _torch_spec(spec):
    ins, out = spec.split("->")
    conv = lambda s: s.replace("(", "").replace(")", "").replace(",", "")
    return ",".join(conv(t) for t in ins.split("),(")) + "->" + conv(out)


def _extents(spec, shapes):
    ins, out = spec.split("->")
    ext = {}
    for tup, shp in zip(ins.split("),("), shapes):
        for n, e in zip(conv_tuple(tup), shp):
            ext[n] = e
    return ext, tuple(ext[n] for n in conv_tuple(out))


def conv_tuple(t):
    t = t.strip("()")
    return [x for x in t.split(",") if x]


F32, BF16, F16, F64 = torch.float32, torch.bfloat16, torch.float16, torch.float64

# (spec, shapes, dtype, kwargs) — one row per kernel class
CASES = [
    ("(i,j)->(j,i)", [(200, 136)], F32, {}),                                    # vec transpose
    ("(i,j,k)->(k,i,j)", [(5, 33, 7)], F32, {}),                                 # generic transpose
    ("(c,a,b)->(a,c,b)", [(70, 90, 64)], F32, {}),                               # short-row copy
    ("(i)->(i)", [((1 << 20) + 3,)], F32, {}),                                      # chunked row copy
    ("(i,j)->(i)", [(50, 77)], F32, {}),                                         # exact row reduction
    ("(i,j)->(i)", [(700, 4096)], F32, {}),                                      # rowreduce thin
    ("(i,j)->(i)", [(20000, 96)], F32, {}),                                      # rowreduce 4-warp
    ("(i,j),(i,j)->(i,j)", [(301, 137), (301, 137)], F32, {}),                   # dense Hadamard
    ("(i,j),(i,j)->(i,j)", [(300, 136), (300, 136)], BF16, {}),                  # dense Hadamard 16-bit
    ("(i,j),(j,k),(k,l)->(i,l)", [(9, 10), (10, 11), (11, 12)], F32, {}),        # exact chain
    ("(i,j),(j,k),(k,l)->(i,l)", [(90, 100), (100, 110), (110, 120)], BF16, {}),  # 16-bit chain
    ("(i,j)->()", [(3000, 700)], F32, {"mode": "ffma"}),                         # tree contig
    ("(i,j)->(i)", [(3000, 700)], F32, {"mode": "ffma"}),                        # tree warp
    ("(i,j)->(j)", [(3000, 700)], F32, {"mode": "ffma"}),                        # tree column
    ("(i,j)->(j)", [(3000, 702)], BF16, {}),                                     # tree column2
    ("(k),(k,j)->(j)", [(3000,), (3000, 702)], BF16, {}),                        # 16-bit matvec
    ("(i,j,k)->(j)", [(40, 37, 300)], F32, {"mode": "ffma"}),                    # tree general
    ("(i,k),(k,j)->(i,j)", [(300, 200), (200, 260)], F32, {}),                   # SIMT exact
    ("(i,k),(k,j)->(i,j)", [(1300, 200), (200, 1260)], F32, {"mode": "ffma"}),   # SIMT big
    ("(i,k),(k,j)->(i,j)", [(77, 64), (64, 50)], F64, {}),                       # f64
    ("(i,k),(j,k)->(i,j)", [(200, 96), (136, 96)], F32, {"mode": "tf32"}),       # tf32 TC
    ("(i,k),(k,j)->(i,j)", [(128, 16384), (16384, 128)], BF16, {}),              # split-K
    ("(b,i,j),(b,j,k)->(b,i,k)", [(3, 130, 72), (3, 72, 200)], F16, {}),         # batched TC
] + [
    ("(i,k),(k,j)->(i,j)", [(300, 640), (640, 1088)], BF16,
     {"schedule": {"cta_group": cg, "tile_n": bn}})
    for cg, bn in ((1, 64), (1, 256), (2, 256), (2, 512))
]


def _tol(dt, red, kw):
    if dt in (BF16, F16):
        return 2e-2                      # 16-bit output rounding (+ chain intermediates)
    if kw.get("mode") == "tf32":
        return 5e-3
    if dt == F64:
        return 1e-10 * max(red, 1)
    return 2e-5 * math.sqrt(max(red, 1)) + 1e-5


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[0]}-{c[2]}-{c[3]}")
def test_guard_zones(case):
    spec, shapes, dt, kw = case
    dev = torch.device("cuda", 0)
    gen = torch.Generator(device=dev).manual_seed(7)
    bases, ops = zip(*[_guarded(s, dt, float("nan"), gen, dev) for s in shapes])
    ext, oshape = _extents(spec, shapes)
    obase, out = _guarded(oshape, dt, SENTINEL, None, dev)
    snap_in = [b.clone() for b in bases]
    res = contract(spec, *ops, out=out, **kw)
    torch.cuda.synchronize()
    assert res.data_ptr() == out.data_ptr()
    # no write outside the output view
    head, tail = obase[:GUARD], obase[GUARD + out.numel():]
    assert bool((head == SENTINEL).all()), "write before the output"
    assert bool((tail == SENTINEL).all()), "write past the output"
    # inputs untouched (guards included)
    for b, s in zip(bases, snap_in):
        assert torch.equal(b.isnan(), s.isnan()) and torch.equal(
            torch.nan_to_num(b), torch.nan_to_num(s)), "an input buffer was written"
    # no NaN leaked in from a guard, and the value is right
    assert not bool(out.isnan().any()), "NaN from an out-of-bounds read"
    want = torch.einsum(_torch_spec(spec), *[o.double() for o in ops])
    red = max(1, math.prod(ext.values()) // max(1, out.numel()))   # points per output
    scale = want.abs().max().item() + 1.0
    err = (out.double() - want).abs().max().item() / scale
    assert err <= _tol(dt, red, kw), f"max rel err {err}"
