"""Pin the BASELINE configurations C1 and C2 at FULL size to the reference itself.

C1: fp32 1024x1024 transpose through minigpu.interp.run_program (Appendix A.1,
    ~8 s here) -> sha256 of the reference's output bytes.
C2: fp32 sum over 2^24 elements (Appendix A.2, naive sequential binary32, ~85 s
    per input here) -> the reference's result bits, for U[0,1) and U[-1,1).
Inputs are regenerated from the recorded seeds (numpy default_rng), so only
hashes / scalars are committed (tests/golden/fullsize_ref.json). Runs only in
the build container, where /root/reference exists:

    python tests/golden/gen_fullsize.py
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

REF = os.environ.get("MINIGPU_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)
from minigpu.interp import Array, run_program  # noqa: E402  (reference)
from minigpu.parser import parse_program  # noqa: E402  (reference)

HERE = os.path.dirname(os.path.abspath(__file__))


def load(name):
    with open(os.path.join(HERE, "programs", name)) as f:
        return parse_program(f.read(), name)


def c1_input(seed):
    return np.random.default_rng(seed).uniform(-1, 1, (1024, 1024)).astype(np.float32)


def c2_input(seed, lo):
    return np.random.default_rng(seed).uniform(lo, 1, 1 << 24).astype(np.float32)


def main():
    out = {"generator": "tests/golden/gen_fullsize.py", "reference": "minigpu.interp.run_program (interp.py:380)"}
    a = c1_input(101)
    t0 = time.perf_counter()
    _, outs = run_program(load("transpose_naive.optc"), "transpose", {
        "in": Array([1024, 1024], a.reshape(-1).tolist(), "float"), "out": Array.alloc([1024, 1024], "float"),
        "W": 1024, "H": 1024})
    got = np.array(outs["out"], dtype=np.float32)
    out["C1"] = {"seed": 101, "dist": "uniform(-1,1) float32 1024x1024", "program": "transpose_naive.optc",
                 "sha256_out_f32": hashlib.sha256(got.tobytes()).hexdigest(),
                 "ref_seconds": time.perf_counter() - t0}
    print("C1", out["C1"], flush=True)
    out["C2"] = []
    for seed, lo in [(202, 0.0), (203, -1.0)]:
        x = c2_input(seed, lo)
        t0 = time.perf_counter()
        r, _ = run_program(load("reduce_naive_f32.optc"), "reduce", {"arr": x.tolist(), "N": x.size})
        rec = {"seed": seed, "lo": lo, "n": int(x.size), "program": "reduce_naive_f32.optc",
               "result": r, "result_f32_bits": int(np.float32(r).view(np.uint32)),
               "ref_seconds": time.perf_counter() - t0}
        out["C2"].append(rec)
        print("C2", rec, flush=True)
    with open(os.path.join(HERE, "fullsize_ref.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
