"""bench.py's JSON-line contract, checked on CPU through the reference arm
(the oracle port; `--impl ours` needs a B200 and is exercised by the driver)."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_bench(*args, env=None):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT,
                         capture_output=True, text=True, timeout=300,
                         env={**os.environ, **(env or {})})
    assert out.returncode == 0, out.stderr[-2000:]
    return out.stdout.strip().splitlines()


def test_reference_arm_line():
    lines = run_bench("--impl", "reference", "--scale", "10", "--steps", "2", "--warmup", "1")
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference"
    assert d["metric"] == "PageRank GTEPS per iteration" and d["unit"] == "GTEPS"
    assert d["steps"] == 2 and d["warmup"] == 1 and d["value"] > 0
    assert d["config"]["graph"] == "rmat:10:16:1" and d["config"]["num_edges"] == 16 * 1024
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": "GTEPS", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}


def test_reference_arm_silent_on_other_ranks():
    # under torchrun only rank 0 runs and prints; the others exit 0 without work
    assert run_bench("--impl", "reference", "--scale", "10", "--steps", "1", "--warmup", "1",
                     env={"RANK": "1", "WORLD_SIZE": "2"}) == []
