"""`bench.py --gpus 2` on ONE GPU with the gloo process group: the
self-launched two-rank job runs the real strong-scaling step (each rank half
of the 32768 rows, no data-path collective — the ranks' kernels never wait on
one another) and rank 0 prints one JSON line with n_gpus = 2."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_bench_two_ranks_one_gpu():
    env = dict(os.environ, BGX_DIST_BACKEND="gloo")
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                        "--steps", "3", "--warmup", "3", "--no-aux", "--no-cpu", "--no-e2e"],
                       capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong"
    assert d["config"]["I"] == 32768 and d["config"]["I_per_rank"] == 16384
    assert d["value"] > 0 and d["gpu_launches"] > 0
    assert d["parity"]["relF_row_samples_max_over_ranks"] <= 1e-2
    assert d["weak"]["I"] == 65536 and d["weak"]["value"] > 0
