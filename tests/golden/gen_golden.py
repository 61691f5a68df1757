"""Generate the golden parity fixtures from the REFERENCE interpreter.

This script is the only place that executes the reference implementation
(`minigpu.interp.run_program`, /root/reference/pkg/src/minigpu/interp.py:380).
It runs in the build container, where /root/reference exists; the GPU box never
reads the reference, it only sees the committed outputs:

    tests/golden/golden.npz      arrays (inputs + reference outputs) per case
    tests/golden/manifest.json   case list: program, entry, shapes, result

Run:  PYTHONPATH=/root/reference/pkg/src python tests/golden/gen_golden.py

Inputs are handed to the interpreter as Python values (`.tolist()`), never as
numpy scalars (SURVEY 8c "harness hazard": numpy int32 scalars would wrap).
"""
from __future__ import annotations

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
PROG = os.path.join(HERE, "programs")


def load(name):
    with open(os.path.join(PROG, name)) as f:
        return parse_program(f.read(), name)


def main():
    cases = []
    arrays = {}

    def add(case, **arrs):
        cid = f"c{len(cases):03d}"
        case["id"] = cid
        for k, v in arrs.items():
            arrays[f"{cid}_{k}"] = v
        cases.append(case)
        print(cid, case["kind"], case.get("shape", case.get("n")), case.get("note", ""),
              f"{case['ref_seconds']:.3f}s", flush=True)

    # ---------------- transposes ----------------
    def transpose_case(prog_name, H, W, a, cell, note, bits=None):
        prog = load(prog_name)
        params = [p for p, _ in prog.fn("transpose").params]
        pin, pout = params[0], params[1]
        t0 = time.perf_counter()
        _, outs = run_program(prog, "transpose", {
            pin: Array([H, W], a.reshape(-1).tolist(), cell),
            pout: Array.alloc([W, H], cell), "W": W, "H": H})
        dt = time.perf_counter() - t0
        out = np.array(outs[pout], dtype=a.dtype).reshape(W, H)
        add({"kind": "transpose", "program": prog_name, "shape": [H, W], "cell": cell,
             "dtype": str(a.dtype), "bits": bits, "note": note, "ref_seconds": dt},
            inp=a, out=out)

    rng = np.random.default_rng(20260517)
    idx8 = np.arange(64, dtype=np.float32).reshape(8, 8)
    transpose_case("transpose_naive.optc", 8, 8, idx8, "float", "SPEC.md:502 8x8 index matrix")
    for (H, W) in [(1, 1), (1, 17), (17, 1), (33, 65), (64, 96), (7, 128), (129, 31)]:
        a = rng.uniform(-1, 1, (H, W)).astype(np.float32)
        transpose_case("transpose_naive.optc", H, W, a, "float", "fp32 U[-1,1)")
    a = rng.standard_normal((40, 24)).astype(np.float32) * np.float32(1e30)
    transpose_case("transpose_naive_yx.optc", 40, 24, a, "float", "loops swapped, wide exponents")
    # bit-pattern transposes through int cells: fp64, bf16, int32
    f64 = rng.standard_normal((5, 7))
    transpose_case("transpose_naive_int.optc", 5, 7, f64.view(np.uint64).copy(), "int",
                   "fp64 bit patterns", bits="f64")
    bf16 = (rng.standard_normal((33, 65)).astype(np.float32).view(np.uint32) >> 16).astype(np.uint16)
    transpose_case("transpose_naive_int.optc", 33, 65, bf16, "int", "bf16 bit patterns", bits="bf16")
    i32 = rng.integers(-2**31, 2**31, (48, 80), dtype=np.int64).astype(np.int32)
    transpose_case("transpose_naive_int.optc", 48, 80, i32, "int", "int32 full range")
    for (H, W) in [(32, 32), (64, 96), (96, 64)]:
        a = rng.uniform(-1, 1, (H, W)).astype(np.float32)
        transpose_case("transpose_gpu.optc", H, W, a, "float", "GPU form (A.4)")

    # ---------------- reductions ----------------
    def reduce_case(prog_name, x, note):
        prog = load(prog_name)
        t0 = time.perf_counter()
        ret, _ = run_program(prog, "reduce", {"arr": x.tolist(), "N": int(x.size)})
        dt = time.perf_counter() - t0
        if isinstance(ret, float):
            res = {"result_f32_bits": int(np.float32(ret).view(np.uint32)), "result": ret}
            assert float(np.float32(ret)) == ret
        else:
            res = {"result_int": str(ret), "result": float(ret)}
        add({"kind": "reduce", "program": prog_name, "n": int(x.size), "dtype": str(x.dtype),
             "note": note, "ref_seconds": dt, **res}, inp=x)

    reduce_case("reduce_naive_f32.optc", np.arange(1, 13, dtype=np.float32), "SPEC.md:501 [1..12] -> 78")
    reduce_case("reduce_naive_int.optc", np.arange(1, 13, dtype=np.int32), "SPEC.md:501 [1..12] -> 78")
    reduce_case("reduce_naive_int.optc", np.full(4, 2**31 - 1, dtype=np.int32), "4 x INT32_MAX, no wrap")
    reduce_case("reduce_naive_int.optc", np.full(5, -2**31, dtype=np.int32), "5 x INT32_MIN, no wrap")
    for n in [1, 7, 1000, 4096, 1 << 14]:
        for dist in ["u01", "um11", "wide"]:
            if dist == "u01":
                x = rng.uniform(0, 1, n).astype(np.float32)
            elif dist == "um11":
                x = rng.uniform(-1, 1, n).astype(np.float32)
            else:
                x = (rng.standard_normal(n) * np.exp2(rng.integers(-20, 20, n))).astype(np.float32)
            reduce_case("reduce_naive_f32.optc", x, f"fp32 sequential {dist}")
    for n in [1, 1000, 1 << 14]:
        x = rng.integers(-2**31, 2**31, n, dtype=np.int64).astype(np.int32)
        reduce_case("reduce_naive_int.optc", x, "int32 full range")
    for n in [512, 4096, 1 << 14]:
        for dist in ["u01", "um11"]:
            lo = 0.0 if dist == "u01" else -1.0
            x = rng.uniform(lo, 1, n).astype(np.float32)
            reduce_case("reduce_tree_f32.optc", x, f"A.5 tree order {dist}")

    # ---------------- parser parity: reference ASTs of every fixture program ----------------
    from tests_ast_dump import dump_program  # noqa: E402  (tests/golden/tests_ast_dump.py)
    asts = {}
    for name in sorted(os.listdir(PROG)):
        asts[name] = dump_program(load(name))
    with open(os.path.join(HERE, "ref_asts.json"), "w") as f:
        json.dump(asts, f, indent=None, sort_keys=True)

    # ---------------- error behaviour of the reference on bad inputs ----------------
    from minigpu.interp import InterpError  # noqa: E402
    errs = []

    def err_case(prog_name, entry, inputs, note):
        try:
            run_program(load(prog_name), entry, inputs)
            errs.append({"program": prog_name, "note": note, "error": None})
        except Exception as e:  # noqa: BLE001
            errs.append({"program": prog_name, "note": note, "type": type(e).__name__,
                         "interp_error": isinstance(e, InterpError), "error": str(e)})

    err_case("transpose_naive.optc", "transpose", {"in": Array([2, 3], [0.0] * 6, "float"),
             "out": Array.alloc([3, 2], "float"), "W": 3}, "missing input H")
    err_case("transpose_naive.optc", "transpose", {"in": Array([2, 3], [0.0] * 6, "float"),
             "out": Array.alloc([3, 2], "float"), "W": 4, "H": 2}, "W larger than in columns")
    err_case("transpose_naive.optc", "transpose", {"in": Array([2, 3], [0.0] * 5 + [None], "float"),
             "out": Array.alloc([3, 2], "float"), "W": 3, "H": 2}, "uninitialised input cell")
    err_case("transpose_gpu.optc", "transpose", {"in": [0.0] * (33 * 32),
             "out": [0.0] * (33 * 32), "W": 32, "H": 33}, "A.4 with 32 not dividing H")
    err_case("reduce_tree_f32.optc", "reduce", {"arr": [1.0] * 513, "N": 513}, "A.5 with 512 not dividing N")
    err_case("reduce_naive_f32.optc", "reduce", {"arr": [1.0] * 4, "N": 5}, "N beyond the array")
    err_case("reduce_naive_f32.optc", "reduce", {"arr": [1.0] * 4, "N": 0}, "N = 0")
    err_case("reduce_naive_int.optc", "reduce", {"arr": [1, 2, 3], "N": -3}, "negative N")
    freed = Array([4], [1.0] * 4, "float", freed=True)
    err_case("reduce_naive_f32.optc", "reduce", {"arr": freed, "N": 4}, "use after free")
    with open(os.path.join(HERE, "ref_errors.json"), "w") as f:
        json.dump(errs, f, indent=1)

    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    with open(os.path.join(HERE, "manifest.json"), "w") as f:
        json.dump({"generator": "tests/golden/gen_golden.py",
                   "reference": "minigpu.interp.run_program (interp.py:380)",
                   "cases": cases}, f, indent=1)
    print(len(cases), "cases written")


def codegen_cases():
    """Reference outputs for GPU-form programs beyond the canonical templates,
    used to pin the code generator (paper_2605_13864_b200/codegen.py)."""
    rng = np.random.default_rng(77)
    cases, arrays = [], {}

    def add(case, **arrs):
        cid = f"g{len(cases):03d}"
        case["id"] = cid
        for k, v in arrs.items():
            arrays[f"{cid}_{k}"] = v
        cases.append(case)
        print(cid, case["program"], case.get("note", ""), flush=True)

    def run_t(prog_name, H, W, note):
        a = rng.uniform(-1, 1, (H, W)).astype(np.float32)
        _, outs = run_program(load(prog_name), "transpose", {"in": a.reshape(-1).tolist(),
                                                              "out": [0.0] * (H * W), "W": W, "H": H})
        add({"kind": "transpose", "program": prog_name, "shape": [H, W], "note": note},
            inp=a, out=np.array(outs["out"], dtype=np.float32).reshape(W, H))

    run_t("transpose_gpu.optc", 64, 96, "A.4 via codegen")
    run_t("transpose_gpu_t64.optc", 128, 192, "64x64-tile variant")
    for prog_name, x, note in [
        ("reduce_tree_f32.optc", rng.uniform(-1, 1, 4096).astype(np.float32), "A.5 via codegen"),
        ("reduce_tree_int256.optc", rng.integers(-2**31, 2**31, 4096, dtype=np.int64).astype(np.int32),
         "int tree, 256 blocks"),
        ("scale_then_reduce.optc", rng.uniform(-1, 1, 2048).astype(np.float32), "two kernels, binary64 eval"),
    ]:
        ret, _ = run_program(load(prog_name), "reduce", {"arr": x.tolist(), "N": int(x.size)})
        res = {"result_int": str(ret)} if isinstance(ret, int) else \
            {"result_f32_bits": int(np.float32(ret).view(np.uint32)), "result": ret}
        add({"kind": "reduce", "program": prog_name, "n": int(x.size), "note": note, **res}, inp=x)
    errs = []
    for prog_name, entry, inputs, note in [
        ("oob_kernel.optc", "shift", {"arr": [0.5] * 128, "N": 128}, "out-of-bounds kernel write"),
        ("transpose_gpu_t64.optc", "transpose", {"in": [0.0] * (96 * 64), "out": [0.0] * (96 * 64),
                                                 "W": 96, "H": 64}, "64 not dividing W"),
        ("reduce_tree_int256.optc", "reduce", {"arr": [1] * 300, "N": 300}, "256 not dividing N"),
    ]:
        try:
            run_program(load(prog_name), entry, inputs)
            errs.append({"program": prog_name, "entry": entry, "note": note, "error": None})
        except Exception as e:  # noqa: BLE001
            errs.append({"program": prog_name, "entry": entry, "note": note, "type": type(e).__name__,
                         "error": str(e)})
    np.savez_compressed(os.path.join(HERE, "golden_codegen.npz"), **arrays)
    with open(os.path.join(HERE, "manifest_codegen.json"), "w") as f:
        json.dump({"generator": "tests/golden/gen_golden.py (codegen_cases)", "cases": cases,
                   "errors": errs}, f, indent=1)


def family_cases():
    """Reference outputs for members of the parametrised program families
    (tests/program_families.py); pins the numpy restatement of each family."""
    sys.path.insert(0, os.path.dirname(HERE))
    from program_families import np_reduce_family, reduce_family, transpose_family
    from minigpu.parser import parse_program as ref_parse
    rng = np.random.default_rng(99)
    out = []
    for T, R in [(8, 2), (16, 16), (32, 8), (64, 4)]:
        H, W = 2 * T, 3 * T
        a = rng.uniform(-1, 1, (H, W)).astype(np.float32)
        _, o = run_program(ref_parse(transpose_family(T, R)), "transpose",
                           {"in": a.reshape(-1).tolist(), "out": [0.0] * (H * W), "W": W, "H": H})
        ok = np.array_equal(np.array(o["out"], np.float32).reshape(W, H), a.T)
        out.append({"family": "transpose", "T": T, "R": R, "shape": [H, W], "ref_equals_transpose": bool(ok)})
        print(out[-1], flush=True)
    for B, cell in [(64, "float"), (128, "int"), (256, "float"), (1024, "float"), (2048, "int")]:
        n = 4 * B
        x = rng.uniform(-1, 1, n).astype(np.float32) if cell == "float" else \
            rng.integers(-2**31, 2**31, n, dtype=np.int64).astype(np.int32)
        ret, _ = run_program(ref_parse(reduce_family(B, cell)), "reduce", {"arr": x.tolist(), "N": n})
        mine = np_reduce_family(x, B)
        ok = (np.float32(ret).view(np.uint32) == np.float32(mine).view(np.uint32)) if cell == "float" else ret == mine
        out.append({"family": "reduce", "B": B, "cell": cell, "n": n, "ref_equals_restatement": bool(ok)})
        print(out[-1], flush=True)
    with open(os.path.join(HERE, "families_pinned.json"), "w") as f:
        json.dump({"generator": "tests/golden/gen_golden.py (family_cases)", "members": out}, f, indent=1)


if __name__ == "__main__":
    if not os.environ.get("GOLDEN_CODEGEN_ONLY"):
        main()
    codegen_cases()
    family_cases()
