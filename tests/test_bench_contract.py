"""bench.py's reference arm on CPU: the JSON line carries the contract keys,
and ranks other than 0 exit 0 without work (the driver launches the arm
under torchrun for N > 1).  The GPU arm is exercised by `-m gpu` runs."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env=None):
    e = dict(os.environ)
    e.update(env or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT, env=e,
                          capture_output=True, text=True, timeout=600)


def test_reference_arm_line_c2():
    r = _run(["--impl", "reference", "--config", "c2", "--steps", "1", "--warmup", "0"])
    assert r.returncode == 0, r.stderr
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert d["impl"] == "reference" and d["metric"] == "path_samples_per_s" and d["value"] > 0
    assert d["unit"] == "path_samples/s" and d["higher_is_better"] is True and d["steps"] == 1
    assert d["config"]["workload"] == "c2" and d["config"]["W"] == 128 and d["config"]["spp"] == 4
    cb = d["cpu_baseline"]
    assert cb["kind"] == "port" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


def test_reference_arm_other_ranks_exit_quietly():
    r = _run(["--impl", "reference", "--config", "c4", "--gpus", "2", "--steps", "1", "--warmup", "0"],
             env={"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"})
    assert r.returncode == 0, r.stderr
    assert r.stdout.strip() == ""
