"""Parametrised families of GPU-form programs (points of OptiGPU's transformation
space around A.4 / A.5), used to fuzz the code generator against
(a) the reference interpreter on small members (tests/golden, generated here in
the build container) and (b) numpy restatements on every member (GPU tests).
"""
import numpy as np


def transpose_family(T: int, R: int) -> str:
    """T x T shared tiles, R x T threads per block, T / R rows per thread."""
    assert T % R == 0 and R * T <= 1024
    J = T // R
    return f"""
void transpose(float* in, float* out, int W, int H) {{
    float* const d_in = gmem_malloc2<float>(H, W);
    memcpy_host_to_device2(d_in, in, H, W);
    float* const d_out = gmem_malloc2<float>(W, H);
    {{
        kernel_launch((W/{T})*(H/{T}), {R} * {T}, 4 * {T} * {T});
        float* const tile = __smem_malloc2<float>({T}, {T});
        kernel_setup_end();
        thread for (int by = 0; by < H/{T}; by++) {{
            thread for (int bx = 0; bx < W/{T}; bx++) {{
                for (int j = 0; j < {J}; j++) {{
                    thread for (int y = 0; y < {R}; y++) {{
                        thread for (int x = 0; x < {T}; x++) {{
                            tile[DMINDEX2(H/{T}, W/{T}, by, bx)][j*{R} + y][x] = d_in[by*{T} + j*{R} + y][bx*{T} + x];
                        }}
                    }}
                }}
                blocksync();
                for (int j = 0; j < {J}; j++) {{
                    thread for (int y = 0; y < {R}; y++) {{
                        thread for (int x = 0; x < {T}; x++) {{
                            d_out[bx*{T} + j*{R} + y][by*{T} + x] = tile[DMINDEX2(H/{T}, W/{T}, by, bx)][x][j*{R} + y];
                        }}
                    }}
                }}
            }}
        }}
        kernel_teardown_begin();
        __smem_free2(tile, {T}, {T});
        kernel_kill();
    }}
    memcpy_device_to_host2(out, d_out, W, H);
    gmem_free(d_out);
    gmem_free(d_in);
}}
"""


def reduce_family(B: int, cell: str = "float") -> str:
    """B-element blocks, B/2 threads: adjacent-pair load, log2(B/2)-level smem tree,
    host sum of the partials (A.5 is B = 512, float)."""
    t = B // 2
    levels = t.bit_length() - 1
    assert 1 << levels == t and t <= 1024
    zero = "0." if cell == "float" else "0"
    return f"""
{cell} reduce({cell}* arr, int N) {{
    {cell}* const d_a = gmem_malloc1<{cell}>(N);
    memcpy_host_to_device1(d_a, arr, N);
    {cell}* const d_p = gmem_malloc1<{cell}>(N / {B});
    {{
        kernel_launch(N / {B}, {t}, 4 * {t});
        {cell}* const s = __smem_malloc1<{cell}>({t});
        kernel_setup_end();
        thread for (int b = 0; b < N / {B}; b++) {{
            thread for (int t = 0; t < {t}; t++) {{
                s[DMINDEX1(N / {B}, b)][t] = d_a[b * {B} + 2 * t] + d_a[b * {B} + 2 * t + 1];
            }}
            blocksync();
            for (int k = 0; k < {levels}; k++) {{
                thread for (int t = 0; t < {t}; t++) {{
                    if (t < pow2({levels - 1} - k)) {{
                        s[DMINDEX1(N / {B}, b)][t] = s[DMINDEX1(N / {B}, b)][t] + s[DMINDEX1(N / {B}, b)][t + pow2({levels - 1} - k)];
                    }}
                }}
                blocksync();
            }}
            thread for (int t = 0; t < {t}; t++) {{
                if (t == 0) {{
                    d_p[b] = s[DMINDEX1(N / {B}, b)][0];
                }}
            }}
        }}
        kernel_teardown_begin();
        __smem_free1(s, {t});
        kernel_kill();
    }}
    {cell}* const p = MALLOC1<{cell}>(N / {B});
    memcpy_device_to_host1(p, d_p, N / {B});
    {cell} sum = {zero};
    for (int i = 0; i < N / {B}; i++) {{
        sum += p[i];
    }}
    free(p);
    gmem_free(d_p);
    gmem_free(d_a);
    return sum;
}}
"""


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
