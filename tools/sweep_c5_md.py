"""Markdown table from a sweep_c5.json: python tools/sweep_c5_md.py <json> <tag> > <md>."""
import json
import sys

d = json.load(open(sys.argv[1]))
tag = sys.argv[2] if len(sys.argv) > 2 else ""
f = lambda v, p=0: "-" if v is None else f"{v:.{p}f}"  # noqa: E731
L = [f"# {tag} — BASELINE config C5 sweep (one B200)", "",
     "`tools/sweep_c5.py`: every result parity-checked against the C oracle. `median` / `best` over",
     "100 single launches between CUDA events, L2 cold (252 MB read pass before each launch) when the",
     "working set is < 4x L2 (these include the ~6 us CUDA-event floor). `pipelined`: one CUDA graph",
     "of back-to-back launches over R >= 2 rotating copies (cold = R x bytes >= 3x L2; tiny cases stay",
     "L2-resident, R <= 64): the steady state of a stream of launches, including the write-back of",
     "the previous launch's dirty lines.", "",
     "| transpose | shape | median GB/s | best GB/s | median us | pipelined GB/s | pipelined us | R | cold |",
     "|---|---|---|---|---|---|---|---|---|"]
for r in d:
    if r["what"] == "transpose":
        L.append(f"| {r['dtype']} | {r['shape'][0]}x{r['shape'][1]} | {f(r['GBps'])} | {f(r.get('GBps_best'))} | "
                 f"{f(r['us'], 1)} | {f(r.get('GBps_pipelined'))} | {f(r.get('us_pipelined'), 2)} | "
                 f"{r.get('rotating', '')} | {r.get('pipelined_cold', '')} |")
L += ["", "| reduce | n | median GB/s | best GB/s | median us | pipelined GB/s | pipelined us | R | cold |",
      "|---|---|---|---|---|---|---|---|---|"]
for r in d:
    if r["what"] == "reduce":
        L.append(f"| {r['dtype']} | 2^{r['log2n']} | {f(r['GBps'])} | {f(r.get('GBps_best'))} | {f(r['us'], 1)} | "
                 f"{f(r.get('GBps_pipelined'))} | {f(r.get('us_pipelined'), 2)} | {r.get('rotating', '')} | "
                 f"{r.get('pipelined_cold', '')} |")
inter = [r for r in d if r["what"] == "interference"]
if inter:
    L += ["", "| C4 + C3 interference | ms |", "|---|---|"] + [f"| {r['mode']} | {r['ms']:.3f} |" for r in inter]
L += ["", f"{sum(r['what'] != 'interference' for r in d)} results, parity failures: "
      f"{sum(not r.get('parity', True) for r in d)}."]
print("\n".join(L))
