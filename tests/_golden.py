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
