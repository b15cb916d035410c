"""bench.py command-line contract on CPU: the reference arm (the float64 oracle on the
host cores) prints exactly ONE JSON line on stdout -- also when self-launched as two
torchrun ranks (rank 0 prints, the other exits without work) -- with the keys the
driver reads.  (The apex arm needs a GPU; its line is checked in profiles/.)"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"}


def _run(extra):
    env = dict(os.environ, OMP_NUM_THREADS="2")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "c1",
                        "--steps", "1", "--warmup", "0", "--ref-seconds", "1", *extra], capture_output=True, text=True, timeout=600,
                       cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [x for x in r.stdout.splitlines() if x.strip()]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert KEYS <= set(d), KEYS - set(d)
    assert d["impl"] == "reference" and d["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] == 0
    return d


def test_reference_arm_one_json_line():
    d = _run([])
    assert d["n_gpus"] == 1 and d["cpu_baseline"]["kind"] == "oracle"


def test_reference_arm_two_ranks_one_json_line():
    d = _run(["--gpus", "2"])
    assert d["n_gpus"] == 2
