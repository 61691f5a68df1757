"""bench.py keeps the driver's JSON contract (both arms), on small sizes."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu
SMALL = ["--transpose-rows", "4096", "--transpose-cols", "4096", "--reduce-n", str(1 << 24),
         "--steps", "3", "--warmup", "3"]


def _run(extra):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *SMALL, *extra], cwd=ROOT,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_gpu_arm_contract():
    d = _run(["--no-cpu"])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["higher_is_better"] is True
    assert d["value"] > 0 and d["gpu_launches"] > 0 and "workload" in d["config"]
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] < 1.5
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])


def test_reference_arm_contract():
    d = _run(["--impl", "reference", "--no-cpu"])
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] in ("port", "reference") and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    g = _run(["--no-cpu", "--no-e2e"])
    assert d["metric"] == g["metric"] and d["config"] == g["config"]


def _torchrun(extra, port):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(ROOT, "bench.py"), "--gpus", "2", *SMALL, *extra]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


@pytest.mark.parametrize("scaling", ["strong", "weak"])
@pytest.mark.parametrize("combine", ["fused", "nccl"])
def test_gpu_arm_two_ranks(combine, scaling):
    """The N > 1 path as the driver launches it (torchrun, one JSON line from rank 0,
    max-over-ranks timing, cross-rank combine checked inside bench.py) with both
    ranks on this box's one GPU: gloo for the host collectives, so `--combine nccl`
    exercises the collective fallback and `fused` the in-kernel mailbox combine.
    Strong scaling (the default, BASELINE configs[2]/[3]) splits the global problem
    into row blocks / shards; the reference arm reports the identical config."""
    port = 29500 + 2 * (combine == "nccl") + (scaling == "weak")
    extra = ["--no-e2e", "--dist-backend", "gloo", "--combine", combine]
    if scaling == "weak":
        extra += ["--scaling", "weak"]
    d = _torchrun(extra + (["--no-cpu"] if scaling == "weak" else []), port)
    assert d["n_gpus"] == 2 and d["scaling"] == scaling and d["value"] > 0
    assert d["combine_note"] is None
    assert ("fused" in d["combine"]) == (combine == "fused")
    if scaling == "strong":
        assert d["shard"]["rank0_rows"] == 2048 and d["shard"]["rank0_n"] == 1 << 23
        assert d["cpu_baseline"]["cores"] >= 1  # rank 0 carries the CPU yardstick at N > 1 too
        ref = _torchrun(["--impl", "reference", "--no-cpu"], port + 10)
        assert ref["config"] == d["config"] and ref["n_gpus"] == 2
