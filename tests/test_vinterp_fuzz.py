"""Random programs through the vectorised interpreter restatement vs the
reference interpreter itself (build container only; the GPU box lacks the
reference). The generator draws loop nests (seq / thread for, literal or
parameter bounds, triangular bounds), affine array reads and writes (in-place
updates, shifted reads that create loop-carried dependences), scalar cells,
reductions, if/else on index predicates and exact_div / pow2 / % index math —
the constructs whose lock-step execution vinterp must prove or demote."""
import random

import pytest

from conftest import reference_available
from oracle import vinterp
from paper_2605_13864_b200 import parse_program

N_PROGRAMS = 150


def _gen(rng: random.Random):
    arrays = ["a", "b"]
    depth = rng.randint(1, 3)
    idx_names = ["i", "j", "k"][:depth]
    lines = []
    n_par = "N"
    bounds = []
    for d in range(depth):
        if d > 0 and rng.random() < 0.25:
            bounds.append(idx_names[d - 1])          # triangular
        else:
            bounds.append(rng.choice(["N", "4", "3", "exact_div(N, 2)"]))
    cell_red = rng.random() < 0.5
    ctype = rng.choice(["int", "float"])
    lit = "2" if ctype == "int" else "2.0"
    if cell_red:
        lines.append(f"    {ctype} s = {'0' if ctype == 'int' else '0.'};")
    ind = "    "
    for d in range(depth):
        mode = rng.choice(["for", "for", "thread for"])
        lines.append(f"{ind}{mode} (int {idx_names[d]} = 0; {idx_names[d]} < {bounds[d]}; {idx_names[d]}++) {{")
        ind += "    "
    inner = idx_names[-1]

    def aff():
        v = rng.choice(idx_names)
        c = rng.choice(["", " + 1", " * 2", " % 3", " + pow2(1)"])
        e = f"({v}{c})"
        return f"({e} % N)"
    stmts = []
    for _ in range(rng.randint(1, 3)):
        kind = rng.random()
        tgt = rng.choice(arrays)
        if kind < 0.35:
            stmts.append(f"{tgt}[{aff()}] = {rng.choice(arrays)}[{aff()}] + {lit};")
        elif kind < 0.55:
            stmts.append(f"{tgt}[{aff()}] += {rng.choice(arrays)}[{aff()}];")
        elif kind < 0.75 and cell_red:
            stmts.append(f"s += {rng.choice(arrays)}[{aff()}];")
        elif kind < 0.9:
            stmts.append(f"if ({inner} % 2 == 0) {{ {tgt}[{aff()}] = {lit}; }} else {{ {tgt}[{aff()}] = {rng.choice(arrays)}[{aff()}]; }}")
        else:
            stmts.append(f"{ctype} t = {rng.choice(arrays)}[{aff()}]; {tgt}[{aff()}] = t * {lit};")
    for st in stmts:
        lines.append(ind + st)
    for _ in range(depth):
        ind = ind[:-4]
        lines.append(f"{ind}}}")
    ret = "s" if cell_red else "0"
    rtype = ctype if cell_red else "int"
    src = f"{rtype} f({ctype}* a, {ctype}* b, int N) {{\n" + "\n".join(lines) + f"\n    return {ret};\n}}\n"
    n = rng.choice([4, 6, 8])
    if ctype == "int":
        av = [rng.randint(-50, 50) for _ in range(n)]
        bv = [rng.randint(-50, 50) for _ in range(n)]
    else:
        av = [rng.uniform(-2, 2) for _ in range(n)]
        bv = [rng.uniform(-2, 2) for _ in range(n)]
    return src, av, bv, n


@pytest.mark.skipif(not reference_available(), reason="reference only in the build container")
def test_random_programs_match_reference():
    from minigpu.interp import run_program as rrun
    from minigpu.parser import parse_program as rparse
    rng = random.Random(2605)
    checked = restarted = declined = 0
    for _ in range(N_PROGRAMS):
        src, av, bv, n = _gen(rng)
        inp = lambda: {"a": list(av), "b": list(bv), "N": n}  # noqa: E731
        try:
            want = rrun(rparse(src), "f", inp())
        except Exception as e:  # noqa: BLE001
            want = ("ERR", type(e).__name__, str(e))
        it = vinterp.VInterp(parse_program(src), lane_budget=5)
        try:
            ret, arrays = it.run("f", inp())
            got_ret = ret[1] if isinstance(ret, tuple) else ret
            got = (got_ret, {k: [None if not ok else v for v, ok in zip(arr.data.tolist(), arr.init.tolist())]
                             for k, (arr, _) in arrays.items()})
        except Exception as e:  # noqa: BLE001
            got = ("ERR", type(e).__name__, str(e))
        if got[0] == "ERR" and got[1] == "VUnsupported" and want[0] != "ERR":
            declined += 1  # e.g. ints past int64: refused explicitly, never a wrong answer
            continue
        if want[0] == "ERR" or got[0] == "ERR":
            assert got == want, src
        else:
            assert got[0] == want[0], src
            assert got[1] == want[1], src
        checked += 1
        restarted += it.restarts > 0
    assert checked + declined == N_PROGRAMS and declined < N_PROGRAMS // 10
    assert restarted > 5  # the fuzzer does exercise demotion
