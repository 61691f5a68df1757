"""SASS evidence for the default kernels of libb200k.so (runs here, no GPU):
registers / shared memory / spills (cuobjdump --dump-resource-usage) and the
static counts of the instructions that carry the design — 128-bit loads
(LDG.E.128 / .NA.128), 256-bit stores (STG.E.256), swizzled shared-memory
traffic (STS.128 / LDS.128), barriers (BAR.SYNC), shuffles (SHFL), TMA
(UTMALDG / UTMASTG) and the grid-combine atomics (ATOMG / RED).

usage: python tools/sass_evidence.py > profiles/sass_evidence.md
"""
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2605_13864_b200", "libb200k.so")

DEFAULTS = [  # (demangled-name prefix, role)
    ("transpose_cpa_kernel<4, 256, 16, 256, 2, 1>", "C4 fp32 transpose (bench): cp.async-loaded 256x64 tiles, 2 stages"),
    ("transpose_cpa_kernel<8, 256, 16, 256, 2, 1>", "fp64 aligned transpose > 256 MB, cp.async-loaded"),
    ("transpose_cpa_kernel<2, 128, 16, 512, 4, 0>", "bf16 aligned transpose > 256 MB, cp.async-loaded"),
    ("transpose_vec_kernel<4, 64, 32, 512>", "fp32 aligned <= 256 MB, 256x128 LDG tile (round-1 C4 default)"),
    ("transpose_vec_kernel<8, 128, 32, 512>", "fp64 aligned <= 256 MB, 256x64 LDG tile"),
    ("transpose_vec_kernel<2, 16, 16, 256>", "bf16 aligned <= 256 MB, 128x128 LDG tile"),
    ("transpose_vec_kernel<4, 16, 16, 256>", "fp32 small / mid transpose, 64x64 tile"),
    ("transpose_staged_kernel<unsigned short, 64, 128, 256, 4, 0>", "2-byte odd pitches >= 2^22 cells, cp.async-staged ring"),
    ("transpose_staged_kernel<unsigned int, 128, 64, 256, 2, 0>", "odd pitches > 256 MB (any width), 128-row staged tiles"),
    ("transpose_scalar_kernel<unsigned short, 128>", "2-byte odd pitches (small), padded 64x128 tile"),
    ("transpose_scalar_kernel<unsigned int, 64>", "4-byte odd pitches, padded 64x64 tile"),
    ("reduce_kernel<int, 512, 4, 1>", "C3 int32 sum (bench)"),
    ("reduce_kernel<float, 512, 4, 1>", "fp32 sum"),
    ("tree_kernel<512, 256>", "A.5 tree order, bit-exact"),
    ("transpose_tmar_kernel<256, 2, 2>", "TMA-staged variant (knob, not default)"),
]
OPS = [("LDG.128", r"LDG\.E[.A-Z0-9_]*\.128"), ("LDG.256", r"LDG\.E[.A-Z0-9_]*\.256"), ("STG.128", r"STG\.E[.A-Z0-9_]*\.128"),
       ("STG.256", r"STG\.E[.A-Z0-9_]*\.256"), ("STS.128", r"STS\.128"), ("LDS.128", r"LDS\.128"),
       ("LDG.16/32", r"LDG\.E(\.U16|\.U8)?(\.CONSTANT)? "), ("BAR.SYNC", r"BAR\.SYNC"), ("SHFL", r"SHFL\."),
       ("PRMT", r"PRMT "), ("UTMALDG", r"UTMALDG"), ("ATOMG/RED", r"ATOMG|REDG|RED\."), ("SYNCS", r"SYNCS\."),
       ("LDGSTS", r"LDGSTS"), ("F2F.F64", r"F2F\.F64\.F32"), ("DADD", r"DADD")]


def demangle(names):
    r = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True)
    return r.stdout.splitlines()


def main():
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    res = subprocess.run(["cuobjdump", "--dump-resource-usage", LIB], capture_output=True, text=True).stdout
    funcs, cur = {}, None
    for ln in sass.splitlines():
        m = re.search(r"Function : (\S+)", ln)
        if m:
            cur = m.group(1)
            funcs[cur] = []
        elif cur and re.search(r"/\*[0-9a-f]{4}\*/", ln):
            funcs[cur].append(ln)
    usage = {}
    lines = res.splitlines()
    for i, ln in enumerate(lines):
        m = re.search(r"Function (\S+):", ln)
        if m and i + 1 < len(lines):
            usage[m.group(1)] = lines[i + 1].strip()
    mangled = list(funcs)
    dem = dict(zip(mangled, demangle(mangled)))
    out = ["# SASS evidence (sm_100a, `tools/sass_evidence.py`)", "",
           "Static instruction counts per kernel (not executed counts) and resource usage from",
           "`cuobjdump` of the in-tree `libb200k.so`.", "",
           "| kernel | role | regs | smem (static) | local | " + " | ".join(o for o, _ in OPS) + " |",
           "|---|---|---|---|---|" + "---|" * len(OPS)]
    for pref, role in DEFAULTS:
        hits = [k for k, d in dem.items() if pref in d]
        if not hits:
            out.append(f"| `{pref}` | {role} | (not found) |")
            continue
        k = hits[0]
        body = funcs[k]
        u = usage.get(k, "")
        reg = re.search(r"REG:(\d+)", u)
        sh = re.search(r"SHARED:(\d+)", u)
        lo = re.search(r"LOCAL:(\d+)", u)
        counts = [sum(1 for ln in body if re.search(rx, ln)) for _, rx in OPS]
        out.append(f"| `{pref}` | {role} | {reg.group(1) if reg else '?'} | {sh.group(1) if sh else '?'} | "
                   f"{lo.group(1) if lo else '?'} | " + " | ".join(str(c) for c in counts) + " |")
    out += ["", "Dynamic shared memory (the 128-KB tiles) is not in the static column; local = 0 means no",
            "register spills."]
    print("\n".join(out))


if __name__ == "__main__":
    sys.exit(main())
