"""Full-size reference outputs for BASELINE configs 1 and 2, made by RUNNING
THE REFERENCE (oracle ladder L0) in this container:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_fullsize_golden.py

  * C1  (i,j),(j,k)->(i,k) f32 256 x 256 x 256, C0 = 0
  * C2a (i,j)->(j,i)       f32 8192 x 8192
  * C2b (i,j,k)->(k,j,i)   f32 256 x 512 x 512
Inputs: np.random.default_rng(seed).standard_normal(shape, dtype=np.float32),
seeds A = 1, B = 2.  Each config is row-sharded over worker
processes: every worker runs bridgegen's own ``build_einsum_function`` +
``interp.run_function`` (``_Machine._generic``, interp.py:372-424) on a slab
of the first input's leading index, which leaves every output element's
evaluation order unchanged (bit-identical to one big run).  C1's output is
stored (256 KiB); for the 256 MiB permutation outputs only SHA-256 digests of
the output bytes are stored.  Nothing at test time reads /root/reference.
"""

from __future__ import annotations

import hashlib
import json
import multiprocessing as mp
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)


sys.path.insert(0, os.path.dirname(HERE))
from _golden import FULLSIZE_SPECS as SPECS  # noqa: E402
from _golden import fullsize_inputs as inputs  # noqa: E402


def _run_slab(args):
    config, lo, hi = args
    sys.path.insert(0, REF)
    from bridgegen import einsum, fir, interp, intrinsics, ir
    ins = inputs(config)
    ins[0] = np.ascontiguousarray(ins[0][lo:hi])
    spec = einsum.parse_einsum(SPECS[config])
    ext = {}
    for arr, tup in zip(ins, spec.inputs):
        for n, e in zip(tup, arr.shape):
            ext[n] = e
    out0 = np.zeros(tuple(ext[x] for x in spec.output), np.float32)
    mod = einsum.build_einsum_function(intrinsics.default_registry(), spec, elem=fir.F32)
    vals = [interp.TensorValue(ir.F32, x.shape, x) for x in ins + [out0]]
    [res] = interp.run_function(mod, "einsum", vals, step_limit=10 ** 12)
    return lo, hi, np.array(np.asarray(res.data), dtype=np.float32, copy=True)


def run(config: str, workers: int):
    n0 = inputs(config)[0].shape[0]
    step = (n0 + 4 * workers - 1) // (4 * workers)
    jobs = [(config, lo, min(n0, lo + step)) for lo in range(0, n0, step)]
    with mp.get_context("spawn").Pool(workers) as pool:
        parts = pool.map(_run_slab, jobs)
    parts.sort()
    if config == "c1":
        return np.concatenate([p for _, _, p in parts], axis=0)
    if config == "c2a":      # out (j, i): slabs of i are column blocks
        return np.concatenate([p for _, _, p in parts], axis=1)
    return np.concatenate([p for _, _, p in parts], axis=2)   # c2b out (k, j, i)


def sha256(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    workers = int(os.environ.get("WORKERS", os.cpu_count() or 1))
    meta = {"seeds": {"A": 1, "B": 2}, "generator": "np.random.default_rng(seed)."
            "standard_normal(shape, dtype=np.float32)", "numpy": np.__version__,
            "workers": workers, "configs": {}}
    for config in ("c1", "c2a", "c2b"):
        t0 = time.time()
        out = run(config, workers)
        dt = time.time() - t0
        meta["configs"][config] = {"spec": SPECS[config], "out_shape": list(out.shape),
                                   "out_sha256": sha256(out), "reference_seconds": dt}
        if config == "c1":
            np.savez_compressed(os.path.join(HERE, "fullsize_c1.npz"), out=out)
        print(config, out.shape, f"{dt:.1f}s", meta["configs"][config]["out_sha256"], flush=True)
    with open(os.path.join(HERE, "fullsize_golden.json"), "w") as fh:
        json.dump(meta, fh, indent=1)


if __name__ == "__main__":
    main()
