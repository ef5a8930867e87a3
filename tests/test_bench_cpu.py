"""bench.py contract checks that need no GPU: the reference arm (oracle port
of the reference loop nest on the host cores) prints one JSON line with the
keys the driver reads."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--steps", "1", "--warmup", "0"], capture_output=True, text=True,
                       timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "TFLOP/s"
    assert d["warmup"] >= 3                       # the contract's minimum
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["config"]["workload"].startswith("chain")


def test_peaks_file_or_fallback():
    sys.path.insert(0, ROOT)
    import bench
    p = bench.peaks()
    assert p["bf16"] > 1000 and p["hbm"] > 5000 and "source" in p


def _run_bench(*args, env_extra=None, timeout=600):
    env = dict(os.environ, **(env_extra or {}))
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args],
                       capture_output=True, text=True, timeout=timeout, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_gpus_n_self_launches_ranks():
    """`bench.py --gpus 2` outside torchrun starts 2 ranks itself (verdict r1:
    --gpus was ignored without torchrun); rank 0 alone prints one line whose
    n_gpus is the real world size, and the strong split covers the job."""
    d = _run_bench("--gpus", "2", "--dry-run", "--steps", "1", "--warmup", "0",
                   env_extra={"BGX_DIST_BACKEND": "gloo"})
    assert d["n_gpus"] == 2 and d["scaling"] == "strong"
    assert d["config"]["I"] == 32768 and d["config"]["rows_covered"] == 32768
    assert d["config"]["I_per_rank"] == 16384


def test_gpus_n_weak_split():
    d = _run_bench("--gpus", "3", "--dry-run", "--scaling", "weak",
                   env_extra={"BGX_DIST_BACKEND": "gloo"})
    assert d["n_gpus"] == 3 and d["config"]["rows_covered"] == 3 * 32768


def test_reference_arm_step_is_the_sample():
    """The reference arm's ms_per_step is the measured sample step (so the
    driver's clock around the run agrees), the extrapolated job time has its
    own key."""
    d = _run_bench("--impl", "reference", "--steps", "1", "--warmup", "0")
    assert d["ms_per_step"] < 600e3
    assert d["job_seconds_extrapolated"] > d["ms_per_step"] / 1e3
