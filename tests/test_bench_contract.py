"""bench.py's reference arm on CPU (-m "not gpu"): the reference's own CPU
march (oracle/_ref, or the port) on this host's cores prints one JSON line in
the driver's contract."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_prints_contract_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--steps", "2", "--warmup", "1", "--ref-seconds", "1"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "higher_is_better",
              "scaling", "dtype", "config", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["value"] > 0 and line["e2e"]["h2d_bytes_per_step"] == 0
    assert line["cpu_baseline"]["kind"] in ("reference", "port")
    assert line["cpu_baseline"]["cores"] >= 1


@pytest.mark.gpu
def test_bench_gpus_2_spawns_two_ranks():
    """`bench.py --gpus 2` without a launcher spawns two ranks itself (on a
    one-GPU box they share the device over gloo) and reports n_gpus = 2 with
    both ranks' updates in the whole-job value."""
    env = dict(os.environ)
    env["VLBM_BENCH_BACKEND"] = "gloo"
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                        "--steps", "3", "--warmup", "3", "--samples", "4", "--grid", "200x40",
                        "--t-start", "0", "--no-cpu-baseline", "--no-postproc", "--no-late",
                        "--no-first-order"],
                       capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2
    assert line["config"]["parallelism"] == "samples/2"
    # 2 ranks x 4 samples x 3 steps x 8000 cells in the timed region
    assert abs(line["value"] * line["ms_per_step"] * line["steps"] * 1e-3 - 2 * 4 * 3 * 8000) < 1
