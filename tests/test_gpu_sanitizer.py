"""compute-sanitizer over every libb200k kernel.

The reference proves race freedom and barrier placement statically (checker.py
E-DESYNC :447-452, E-THREADS-CTX :782-789, GMem single-thread access :417-422);
the B200 kernels keep the same barrier structure and are checked dynamically:
racecheck (shared-memory hazards), synccheck (illegal / divergent barriers),
memcheck (out-of-bounds / misaligned accesses, incl. TMA and the IPC mailbox)
and initcheck (reads of uninitialised device memory). The driver
(tools/sanitize_driver.py) also asserts parity of every result.
"""
import os
import re
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SAN = "/usr/local/cuda/bin/compute-sanitizer"

CASES = [
    ("memcheck", "transpose"), ("memcheck", "transpose_big"), ("memcheck", "reduce"),
    ("memcheck", "fused"), ("memcheck", "multi"), ("memcheck", "codegen"),
    ("racecheck", "transpose"), ("racecheck", "reduce"), ("racecheck", "fused"), ("racecheck", "multi"),
    ("racecheck", "codegen"),
    ("synccheck", "transpose"), ("synccheck", "reduce"), ("synccheck", "codegen"),
    ("initcheck", "transpose"), ("initcheck", "reduce"),
]


@pytest.mark.parametrize("tool,group", CASES)
def test_sanitizer_clean(tool, group):
    if not os.path.exists(SAN):
        pytest.skip("compute-sanitizer not installed")
    cmd = [SAN, "--tool", tool, "--error-exitcode", "99", "--print-limit", "20"]
    if tool == "memcheck":
        cmd += ["--leak-check", "no"]
    cmd += [sys.executable, os.path.join(ROOT, "tools", "sanitize_driver.py"), group]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    log = r.stdout + r.stderr
    assert r.returncode == 0, log[-4000:]
    assert f"sanitize-driver {group} ok" in log, log[-4000:]
    if tool == "racecheck":  # racecheck prints its own summary line
        m = re.search(r"RACECHECK SUMMARY: (\d+) hazards displayed \((\d+) errors, (\d+) warnings\)", log)
        assert m and m.groups() == ("0", "0", "0"), log[-4000:]
    else:
        m = re.search(r"ERROR SUMMARY: (\d+) error", log)
        assert m and m.group(1) == "0", log[-4000:]
