"""Reference run_program outcomes (minigpu.interp, interp.py:380) on the hot-path
programs with bad / edge inputs -> tests/golden/ref_interp_errors.json: which
error (type + message) the reference raises first, or that it succeeds. Build
container only:   python tests/golden/gen_interp_errors.py
"""
import json
import os
import sys

sys.path.insert(0, os.environ.get("MINIGPU_REF", "/root/reference/pkg/src"))
from minigpu.interp import Array, run_program  # noqa: E402  (reference)
from minigpu.parser import parse_program  # noqa: E402  (reference)

HERE = os.path.dirname(os.path.abspath(__file__))


def arr(dims, fill=0.0, ctype="float", none_at=(), freed=False):
    n = 1
    for d in dims:
        n *= d
    data = [fill] * n
    for k in none_at:
        data[k] = None
    return {"dims": dims, "data": data, "ctype": ctype, "freed": freed}


def materialise(A, spec):
    return {k: (A(list(v["dims"]), list(v["data"]), v["ctype"], v["freed"]) if isinstance(v, dict) else v)
            for k, v in spec.items()}


TN, TY, TG = "transpose_naive.optc", "transpose_naive_yx.optc", "transpose_gpu.optc"
RF, RI, RT = "reduce_naive_f32.optc", "reduce_naive_int.optc", "reduce_tree_f32.optc"
CASES = [
    (TN, "transpose", {"in": arr([2, 3]), "out": arr([3, 2]), "W": 3}),
    (TN, "transpose", {"in": arr([2, 3]), "out": arr([3, 2]), "W": 4, "H": 2}),
    (TN, "transpose", {"in": arr([2, 3]), "out": arr([3, 2]), "W": 3, "H": 3}),
    (TN, "transpose", {"in": arr([2, 3]), "out": arr([2, 2]), "W": 3, "H": 2}),
    (TN, "transpose", {"in": arr([2, 3]), "out": arr([3, 1]), "W": 3, "H": 2}),
    (TN, "transpose", {"in": arr([2, 2]), "out": arr([3, 1]), "W": 3, "H": 2}),
    (TN, "transpose", {"in": arr([2, 3], none_at=(4,)), "out": arr([3, 2]), "W": 3, "H": 2}),
    (TN, "transpose", {"in": arr([2, 3], none_at=(5, 2)), "out": arr([3, 2]), "W": 3, "H": 2}),
    (TN, "transpose", {"in": arr([2, 3], none_at=(5,)), "out": arr([3, 2]), "W": 4, "H": 2}),
    (TN, "transpose", {"in": arr([2, 3], freed=True), "out": arr([3, 2]), "W": 3, "H": 2}),
    (TN, "transpose", {"in": arr([2, 3]), "out": arr([3, 2], freed=True), "W": 3, "H": 2}),
    (TN, "transpose", {"in": arr([2, 3, 1]), "out": arr([3, 2]), "W": 3, "H": 2}),
    (TN, "transpose", {"in": arr([2, 3]), "out": arr([3, 2, 1]), "W": 3, "H": 2}),
    (TN, "transpose", {"in": arr([2, 3]), "out": arr([3, 2]), "W": 0, "H": 2}),
    (TN, "transpose", {"in": arr([2, 3]), "out": arr([3, 2]), "W": -1, "H": 2}),
    (TY, "transpose", {"src": arr([2, 3]), "dst": arr([3, 2]), "W": 4, "H": 3}),
    (TY, "transpose", {"src": arr([2, 3], none_at=(3,)), "dst": arr([3, 2]), "W": 3, "H": 2}),
    (TY, "transpose", {"src": arr([2, 3], none_at=(2,)), "dst": arr([1, 2]), "W": 3, "H": 2}),
    ("transpose_naive_int.optc", "transpose",
     {"in": arr([2, 3], 1, "int", none_at=(0,)), "out": arr([3, 2], 0, "int"), "W": 3, "H": 2}),
    (TG, "transpose", {"in": [0.0] * (33 * 32), "out": [0.0] * (33 * 32), "W": 32, "H": 33}),
    (TG, "transpose", {"in": [0.0] * (32 * 32), "out": [0.0] * (32 * 32), "W": 64, "H": 32}),
    (TG, "transpose", {"in": [0.0] * (64 * 32), "out": [0.0] * (32 * 32), "W": 64, "H": 32}),
    (TG, "transpose", {"in": arr([32 * 32], none_at=(5,)), "out": [0.0] * (32 * 32), "W": 32, "H": 32}),
    (TG, "transpose", {"in": [0.0] * (32 * 32), "out": [0.0] * (32 * 32), "W": 32}),
    (TG, "transpose", {"in": arr([32 * 32], none_at=(900,)), "out": [0.0] * 16, "W": 32, "H": 40}),
    (RF, "reduce", {"arr": [1.0] * 4, "N": 5}),
    (RF, "reduce", {"arr": [1.0] * 4}),
    (RF, "reduce", {"arr": arr([4], freed=True), "N": 4}),
    (RF, "reduce", {"arr": arr([4], none_at=(2,)), "N": 4}),
    (RF, "reduce", {"arr": arr([4], none_at=(2,)), "N": 9}),
    (RF, "reduce", {"arr": arr([2, 2]), "N": 4}),
    (RI, "reduce", {"arr": [1, 2, 3], "N": 4}),
    (RI, "reduce", {"arr": arr([3], 1, "int", none_at=(1,)), "N": 3}),
    (RT, "reduce", {"arr": [1.0] * 513, "N": 513}),
    (RT, "reduce", {"arr": [1.0] * 512, "N": 1024}),
    (RT, "reduce", {"arr": arr([512], none_at=(511,)), "N": 512}),
    (RT, "reduce", {"arr": arr([600], none_at=(599,)), "N": 1024}),
    (RT, "reduce", {"arr": [1.0] * 512}),
    # the GPU forms only touch host arrays through memcpy: freed arrays pass (no error)
    (TG, "transpose", {"in": arr([32 * 32], 1.0, freed=True), "out": arr([32 * 32], 0.0, freed=True),
                       "W": 32, "H": 32}),
    (RT, "reduce", {"arr": arr([512], 1.0, freed=True), "N": 512}),
]


def main():
    out = []
    for prog, entry, spec in CASES:
        with open(os.path.join(HERE, "programs", prog)) as f:
            p = parse_program(f.read(), prog)
        rec = {"program": prog, "entry": entry, "inputs": spec}
        try:
            ret, outs = run_program(p, entry, materialise(Array, spec))
            rec["error"] = None
            rec["ret"] = ret
        except Exception as e:  # noqa: BLE001
            rec["type"], rec["error"] = type(e).__name__, str(e)
        out.append(rec)
    with open(os.path.join(HERE, "ref_interp_errors.json"), "w") as f:
        json.dump(out, f)
    print(len(out), "cases;", sum(r["error"] is not None for r in out), "raise")


if __name__ == "__main__":
    main()
