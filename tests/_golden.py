"""Loader for the reference-generated fixtures in tests/golden/ (see
tests/golden/make_golden.py, which ran bridgegen itself to make them)."""

from __future__ import annotations

import json
import os
import re

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def split_spec(text: str):
    """Index tuples of a parenthesised spec (fixtures only hold valid specs)."""
    lhs, rhs = text.split("->")
    tup = lambda s: tuple(x.strip() for x in s.split(",") if x.strip())  # noqa: E731
    ins = [tup(t) for t in re.findall(r"\(([^()]*)\)", lhs)]
    out = tup(re.findall(r"\(([^()]*)\)", rhs)[0])
    return ins, out


def generic_cases():
    with open(os.path.join(GOLDEN, "generic_cases.json")) as fh:
        index = json.load(fh)
    z = np.load(os.path.join(GOLDEN, "generic_cases.npz"))
    cases = []
    for c in index:
        n = c["name"]
        ins = [z[f"{n}__in{k}"] for k in range(c["n_in"])]
        cases.append((n, c["spec"], ins, z[f"{n}__init"], z[f"{n}__out"]))
    return cases


def kernel_cases():
    return dict(np.load(os.path.join(GOLDEN, "kernel_cases.npz")))


def parse_cases():
    with open(os.path.join(GOLDEN, "parse_golden.json")) as fh:
        return json.load(fh)


def printed_cases():
    with open(os.path.join(GOLDEN, "printed_golden.json")) as fh:
        return json.load(fh)


def bits_equal(a, b) -> bool:
    a = np.asarray(a)
    b = np.asarray(b)
    return a.shape == b.shape and a.dtype == b.dtype and np.array_equal(
        a.reshape(-1).view(np.uint8), b.reshape(-1).view(np.uint8))


# ---- full-size BASELINE configs 1 and 2 (tests/golden/make_fullsize_golden.py)

FULLSIZE_SPECS = {"c1": "(i,j),(j,k)->(i,k)", "c2a": "(i,j)->(j,i)", "c2b": "(i,j,k)->(k,j,i)"}


def fullsize_inputs(config: str):
    """The BASELINE inputs (standard_normal f32, seeds A = 1, B = 2)."""
    if config == "c1":
        a = np.random.default_rng(1).standard_normal((256, 256), dtype=np.float32)
        b = np.random.default_rng(2).standard_normal((256, 256), dtype=np.float32)
        return [a, b]
    if config == "c2a":
        return [np.random.default_rng(1).standard_normal((8192, 8192), dtype=np.float32)]
    if config == "c2b":
        return [np.random.default_rng(1).standard_normal((256, 512, 512), dtype=np.float32)]
    raise KeyError(config)


def fullsize_meta():
    with open(os.path.join(GOLDEN, "fullsize_golden.json")) as fh:
        return json.load(fh)


def fullsize_c1():
    return np.load(os.path.join(GOLDEN, "fullsize_c1.npz"))["out"]


def sha256(a) -> str:
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def import_bridgegen():
    """Import the REAL reference package for the drop-in tests.

    On the GPU box the reference tree is absent; ``__graft_entry__.build()``
    pip-installs it (pure Python, ``--no-deps``) into the git-ignored
    ``baseline/_ref``, which travels with the snapshot.  Here (build
    container) ``/root/reference/pkg/src`` is used when the install is
    missing.  A missing package is a hard error, never a skip: a green GPU
    run must not hide zero coverage of the plug-in path."""
    import importlib
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for cand in (os.path.join(root, "baseline", "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(cand, "bridgegen")):
            if cand not in sys.path:
                sys.path.append(cand)
            break
    try:
        return importlib.import_module("bridgegen")
    except ImportError as e:  # pragma: no cover - exercised only on a broken box
        raise ImportError(
            "bridgegen (the reference package) is not importable: run "
            "`python -c 'import __graft_entry__ as g; g.build()'` in the build "
            "container so baseline/_ref ships with the snapshot") from e
