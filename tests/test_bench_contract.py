"""bench.py's JSON-line contract, checked on CPU through the reference arm
(the oracle port; `--impl ours` needs a B200 and is exercised by the driver)."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_bench(*args, env=None):
    full = {**os.environ, **(env or {})}
    full = {k: v for k, v in full.items() if v is not None}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT,
                         capture_output=True, text=True, timeout=300, env=full)
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


def test_reference_arm_times_whole_calls():
    # one step = one pr_blocked call of --iters iterations (cli.py:256-262),
    # the same work the GPU arm times; per-call setup is reported apart
    d = json.loads(run_bench("--impl", "reference", "--scale", "12", "--steps", "2", "--warmup",
                             "1", "--iters", "10")[0])
    cb = d["cpu_baseline"]
    assert "x 10 iterations" in cb["sample"]
    assert d["config"]["iterations_per_step"] == 10
    assert cb["ms_per_iteration"] > 0 and cb["ms_setup_per_call"] >= 0
    # value = |E| x iterations / step time (printed rounded: ms to 4, value to 3 decimals)
    want = 16 * 4096 * 10 / (d["ms_per_step"] / 1e3) / 1e9
    assert abs(d["value"] - want) <= (1e-3 + 1e-4 / d["ms_per_step"]) * d["value"] + 5e-4


def test_gpus_flag_must_match_world():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                          "--steps", "1", "--warmup", "1", "--scale", "10"], cwd=ROOT,
                         capture_output=True, text=True, timeout=300,
                         env={**os.environ, "WORLD_SIZE": "1", "RANK": "0"})
    assert out.returncode != 0 and "WORLD_SIZE" in out.stderr


def test_gpus_flag_launches_ranks():
    # --gpus 2 outside torchrun starts two ranks itself; the reference arm
    # prints one line from rank 0 and reports the job's world size
    lines = run_bench("--impl", "reference", "--gpus", "2", "--scale", "10", "--steps", "1",
                      "--warmup", "1", env={"WORLD_SIZE": None, "RANK": None})
    lines = [x for x in lines if x.startswith("{")]
    assert len(lines) == 1
    assert json.loads(lines[0])["n_gpus"] == 2
