"""bench.py --impl reference runs on the host alone (the C port of the
reference's path): its JSON line on CPU, and the silent exit of non-zero ranks
under torchrun (only rank 0 prints)."""
import json
import os
import subprocess
import sys

from conftest import ROOT

SMALL = ["--impl", "reference", "--transpose-rows", "512", "--transpose-cols", "1024",
         "--reduce-n", str(1 << 20), "--steps", "3", "--warmup", "3"]


def _run(env_extra, extra=()):
    env = dict(os.environ, **env_extra)
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *SMALL, *extra], cwd=ROOT, env=env,
                          capture_output=True, text=True, timeout=600)


def test_reference_arm_json_on_cpu():
    r = _run({"RANK": "0"}, ["--no-cpu"])
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["value"] > 0 and d["steps"] == 3 and d["warmup"] == 3
    assert d["unit"] == "GB/s" and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"] == {"value": d["value"], "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


def test_reference_arm_other_ranks_silent():
    r = _run({"RANK": "1", "WORLD_SIZE": "2"})
    assert r.returncode == 0 and not [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
