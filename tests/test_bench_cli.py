"""bench.py's launch contract on the CPU (no GPU needed): the reference arm's
JSON line carries the contract keys with a real per-step time, --gpus must
match WORLD_SIZE under torchrun, and --impl reference under several ranks
prints from rank 0 only."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env=None, timeout=300):
    e = dict(os.environ)
    e.pop("WORLD_SIZE", None)
    e.update(env or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], env=e,
                          capture_output=True, text=True, timeout=timeout, cwd=ROOT)


def test_reference_arm_line_contract():
    r = _run(["--impl", "reference", "--config", "tiny", "--steps", "2", "--warmup", "3"])
    assert r.returncode == 0, r.stderr
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["dtype"] == "f64"
    assert line["steps"] == 2 and line["warmup"] == 3
    assert line["value"] > 0 and line["ms_per_step"] > 0
    # value is the whole E-exit step's rate at the measured per-exit step time
    E = line["config"]["exits"]
    n = 32
    assert abs(line["value"] - n / (E * line["ms_per_step"] / 1e3)) <= 1e-6 * line["value"]
    assert line["e2e"]["h2d_bytes_per_step"] == 0
    assert line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["cores"] >= 1


def test_gpus_must_match_world_size():
    r = _run(["--impl", "reference", "--config", "tiny", "--gpus", "2"],
             env={"WORLD_SIZE": "1", "RANK": "0", "LOCAL_RANK": "0"})
    assert r.returncode != 0
    assert "WORLD_SIZE" in (r.stderr + r.stdout)


def test_reference_arm_rank_nonzero_prints_nothing():
    r = _run(["--impl", "reference", "--config", "tiny", "--gpus", "2", "--steps", "1"],
             env={"WORLD_SIZE": "2", "RANK": "1", "LOCAL_RANK": "1"})
    assert r.returncode == 0, r.stderr
    assert r.stdout.strip() == ""
