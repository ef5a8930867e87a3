"""TEST INFRASTRUCTURE ONLY — CPU oracle for the einsum / linalg.generic path.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this package, and
only as the checker / reported CPU baseline.  The product package
``paper_2503_04771_b200`` never imports it and has no CPU fallback.

Parity ladder:
  * ``generic``    — C restatement of bridgegen ``interp._Machine._generic``
                     (interp.py:372-424) with the einsum body of einsum.py:100-118;
                     bit-exact with the reference (pinned by tests/test_oracle.py
                     against tests/golden/*.npz made by the reference itself).
  * ``gemm_kseq``  — the same arithmetic for 2-operand, single-reduction-group
                     contractions, loop-reordered so it vectorises; bit-exact.
  * ``chain_f64``  — float64 factored reference ``(A@B)@C`` for row samples of
                     the 3-operand chain (the reference's unfactored 2^54-point
                     loop nest is infeasible; SURVEY §8c ladder L3).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

_i64 = ctypes.c_int64
_P = ctypes.c_void_p


def build() -> str:
    """Compile liboracle.so with the committed Makefile (gcc, no GPU)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        src = os.path.join(_HERE, "generic_oracle.c")
        if (not os.path.exists(_LIB_PATH)
                or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src)):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        for name in ("oracle_generic_f32", "oracle_generic_f64"):
            f = getattr(L, name)
            f.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, _P, _P, _P,
                          _P, _P, _i64, _i64, ctypes.c_int]
            f.restype = ctypes.c_int
        f = L.oracle_chain3_f32
        f.argtypes = [_i64, _i64, _i64, _i64, _P, _P, _P, _P, _i64, _i64, _i64, _i64,
                      ctypes.c_int]
        f.restype = ctypes.c_int
        f = L.oracle_gemm_kseq_f32
        f.argtypes = [_i64, _i64, _i64, _i64, _P, _i64, _i64, _i64,
                      _P, _i64, _i64, _i64, _P, _P, _i64, _i64, ctypes.c_int]
        f.restype = ctypes.c_int
        _lib = L
    return _lib


def _axes_of(inputs, output):
    """Axis order of einsum.py:81: output indices, then input-only indices in
    first-appearance order."""
    seen = []
    for tup in inputs:
        for n in tup:
            if n not in seen:
                seen.append(n)
    return list(output) + [n for n in seen if n not in output]


def generic(in_tuples, output, arrays, out_init, *, out_range=None,
            threads: int = 0) -> np.ndarray:
    """Evaluate ``out = out_init + sum prod(arrays)`` with the reference's exact
    rounding.  ``in_tuples``/``output`` are index-name tuples, e.g.
    ``[("i","k"),("k","j")], ("i","j")``.  ``out_range=(lo, hi)`` computes only
    output linear indices [lo, hi) (the rest of the result is ``out_init``)."""
    arrays = [np.asarray(a) for a in arrays]
    dtype = np.dtype(out_init.dtype)
    if dtype not in (np.float32, np.float64):
        raise TypeError("oracle.generic: f32/f64 only (the reference's types)")
    arrays = [np.asarray(a, dtype=dtype) for a in arrays]  # any strides
    axes = _axes_of(in_tuples, output)
    extents = {}
    for a, tup in zip(arrays + [out_init], list(in_tuples) + [tuple(output)]):
        assert a.ndim == len(tup), (a.shape, tup)
        for e, n in zip(a.shape, tup):
            assert extents.setdefault(n, e) == e, f"inconsistent extent {n}"
    ext = np.array([extents[n] for n in axes], dtype=np.int64)
    strides = np.zeros((len(arrays), len(axes)), dtype=np.int64)
    for k, (a, tup) in enumerate(zip(arrays, in_tuples)):
        for d, n in enumerate(tup):
            strides[k, axes.index(n)] = a.strides[d] // a.itemsize
    c0 = np.array(out_init, dtype=dtype, order="C", copy=True)
    out = c0.copy()
    ptrs = (ctypes.c_void_p * len(arrays))(*[a.ctypes.data for a in arrays])
    n_out = int(np.prod([extents[n] for n in output], dtype=np.int64)) if output else 1
    lo, hi = out_range if out_range is not None else (0, n_out)
    fn = lib().oracle_generic_f32 if dtype == np.float32 else lib().oracle_generic_f64
    rc = fn(len(arrays), len(axes), len(output), ext.ctypes.data, ptrs,
            strides.ctypes.data, c0.ctypes.data, out.ctypes.data, lo, hi, threads)
    if rc != 0:
        raise ValueError("oracle.generic: bad arguments")
    return out


def gemm_kseq(a: np.ndarray, b: np.ndarray, c0: np.ndarray | None = None, *,
              rows=None, threads: int = 0) -> np.ndarray:
    """Bit-exact reference arithmetic for ``(b,i,k),(b,k,j)->(b,i,j)`` (or the
    unbatched 2-D form) in float32.  ``rows=(lo, hi)`` restricts to rows
    [lo, hi) of every batch (others are left equal to ``c0``)."""
    squeeze = a.ndim == 2
    a3 = a[None] if squeeze else a
    b3 = b[None] if squeeze else b
    a3 = np.asarray(a3, dtype=np.float32)
    b3 = np.asarray(b3, dtype=np.float32)
    Bt, M, K = a3.shape
    _, K2, N = b3.shape
    assert K == K2 and b3.shape[0] == Bt
    if c0 is None:
        c = np.zeros((Bt, M, N), dtype=np.float32)
    else:
        c = np.ascontiguousarray((c0[None] if squeeze else c0), dtype=np.float32).copy()
    lo, hi = rows if rows is not None else (0, M)
    isz = 4
    lib().oracle_gemm_kseq_f32(
        Bt, M, N, K,
        a3.ctypes.data, a3.strides[0] // isz, a3.strides[1] // isz, a3.strides[2] // isz,
        b3.ctypes.data, b3.strides[0] // isz, b3.strides[1] // isz, b3.strides[2] // isz,
        c.ctypes.data, c.ctypes.data, lo, hi, threads)
    return c[0] if squeeze else c


def chain3(a, b, c, out_init, *, rows=None, cols=None, threads: int = 0):
    """Reference (unfactored) semantics of (i,k),(k,j),(j,l)->(i,l) in f32,
    vectorised over l; bit-equal to ``generic`` on the same spec.  Computes
    rows [r0, r1) x cols [c0, c1) of the result (the rest = out_init)."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    b = np.ascontiguousarray(b, dtype=np.float32)
    c = np.ascontiguousarray(c, dtype=np.float32)
    out = np.array(out_init, dtype=np.float32, order="C", copy=True)
    I, K = a.shape
    J, L = c.shape
    r0, r1 = rows if rows is not None else (0, I)
    c0_, c1_ = cols if cols is not None else (0, L)
    lib().oracle_chain3_f32(I, K, J, L, a.ctypes.data, b.ctypes.data, c.ctypes.data,
                            out.ctypes.data, r0, r1, c0_, c1_, threads)
    return out


def chain_f64(a: np.ndarray, b: np.ndarray, c: np.ndarray, rows) -> np.ndarray:
    """Float64 ``(A[rows] @ B) @ C`` — ladder L3 for the 3-operand chain."""
    a64 = np.asarray(a[rows], dtype=np.float64)
    return (a64 @ np.asarray(b, dtype=np.float64)) @ np.asarray(c, dtype=np.float64)


def rel_frobenius(got, want) -> float:
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    den = np.linalg.norm(want)
    num = np.linalg.norm(got - want)
    return float(num / den) if den > 0 else float(num)
