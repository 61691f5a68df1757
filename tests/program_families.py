"""Parametrised families of GPU-form programs (points of OptiGPU's transformation
space around A.4 / A.5), used to fuzz the code generator against
(a) the reference interpreter on small members (tests/golden, generated here in
the build container) and (b) numpy restatements on every member (GPU tests).
"""
import numpy as np


from paper_2605_13864_b200.programs import reduce_tree_family as reduce_family  # noqa: E402,F401
from paper_2605_13864_b200.programs import transpose_gpu_family as transpose_family  # noqa: E402,F401


def np_reduce_family(x: np.ndarray, B: int):
    """numpy restatement of reduce_family(B): the exact evaluation order."""
    if x.dtype == np.float32:
        b = x.reshape(-1, B)
        s = b[:, 0::2] + b[:, 1::2]
        h = B // 4
        while h >= 1:
            s = s.copy()
            s[:, :h] = s[:, :h] + s[:, h:2 * h]
            h //= 2
        acc = np.float32(0)
        for p in s[:, 0]:
            acc = np.float32(acc + p)
        return float(acc)
    return int(x.astype(np.int64).sum())


def thread_index_nests(count: int, seed: int = 0):
    """SPEC acceptance 9: random `thread for` nests (<= 4 loops, concrete bounds,
    grid <= 4096). Each nest is (bounds, tpb) with prod(bounds) = bpg * tpb."""
    rng = np.random.default_rng(seed)
    nests = []
    while len(nests) < count:
        k = int(rng.integers(1, 5))
        bounds = [int(rng.choice([1, 2, 3, 4, 5, 6, 7, 8, 12, 16, 31, 32, 64])) for _ in range(k)]
        total = int(np.prod(bounds))
        if total > 4096:
            continue
        # threads per block: a suffix product of the bounds that fits a block
        tpb = 1
        for b in reversed(bounds):
            if tpb * b > 1024:
                break
            tpb *= b
        nests.append((bounds, tpb))
    return nests


def thread_index_program(nests) -> str:
    """One kernel scope per nest; nest q writes d[off_q + rowmajor(i)] = f(i)."""
    names = ["i0", "i1", "i2", "i3"]
    total = sum(int(np.prod(b)) for b, _ in nests)
    out = [f"void idx(int* res, int N) {{",
           "    int* const d = gmem_malloc1<int>(N);"]
    off = 0
    for bounds, tpb in nests:
        P = int(np.prod(bounds))
        bpg = P // tpb
        out.append("    {")
        out.append(f"        kernel_launch({bpg}, {tpb}, 0);")
        out.append("        kernel_setup_end();")
        ind = "        "
        for j, b in enumerate(bounds):
            out.append(f"{ind}thread for (int {names[j]} = 0; {names[j]} < {b}; {names[j]}++) {{")
            ind += "    "
        lin = names[0]
        for j in range(1, len(bounds)):
            lin = f"({lin}) * {bounds[j]} + {names[j]}"
        val = " + ".join(f"{names[j]} * {[1000003, 1009, 31, 1][j]}" for j in range(len(bounds)))
        out.append(f"{ind}d[{off} + {lin}] = {val} + {off};")
        for _ in bounds:
            ind = ind[:-4]
            out.append(f"{ind}}}")
        out.append("        kernel_teardown_begin();")
        out.append("        kernel_kill();")
        out.append("    }")
        off += P
    out.append("    memcpy_device_to_host1(res, d, N);")
    out.append("    gmem_free(d);")
    out.append("}")
    assert off == total
    return "\n".join(out) + "\n"


def np_thread_index(nests) -> np.ndarray:
    vals = []
    off = 0
    for bounds, _ in nests:
        grids = np.meshgrid(*[np.arange(b) for b in bounds], indexing="ij")
        v = sum(g * [1000003, 1009, 31, 1][j] for j, g in enumerate(grids)) + off
        vals.append(np.asarray(v).reshape(-1))
        off += int(np.prod(bounds))
    return np.concatenate(vals).astype(np.int64)
