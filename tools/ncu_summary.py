"""Summarise ncu captures (gpurun_out/*.ncu-rep + launches.csv) into profiles/.

usage: python tools/ncu_summary.py <tag>     (reads gpurun_out/, writes profiles/<tag>_*.{json,md}
       and refreshes profiles/ncu_summary.json, which bench.py reads for `traffic`)
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_static",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_sectors_srcunit_tex_op_write.sum",
    "sm__cycles_elapsed.avg.per_second", "dram__cycles_elapsed.avg.per_second",
    "smsp__inst_executed.sum",
]


def raw(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    out = []
    for vals in rows[2:]:
        d = {"kernel": vals[hdr.index("Kernel Name")]}
        for m in METRICS:
            if m in hdr:
                i = hdr.index(m)
                d[m] = {"value": vals[i], "unit": units[i]}
        out.append(d)
    return out


def to_bytes(v):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    return float(v["value"].replace(",", "")) * scale[v["unit"]]


def to_ns(v):
    scale = {"ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6, "nsecond": 1}
    return float(v["value"].replace(",", "")) * scale[v["unit"]]


def launches(path):
    per = {}
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    rows = list(csv.reader(lines))
    hdr = rows[0]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    idi = hdr.index("ID")
    recs = {}
    for r in rows[1:]:
        recs.setdefault((r[idi], r[ki]), {})[r[mi]] = float(r[vi].replace(",", ""))
    for (lid, k), m in recs.items():
        per.setdefault(k, []).append(m)
    return per


def main(tag):
    os.makedirs(PROF, exist_ok=True)
    summary = {"tag": tag}
    for name, rep in [("transpose", "prof_transpose.ncu-rep"), ("reduce", "prof_reduce.ncu-rep")]:
        p = os.path.join(OUT, rep)
        if not os.path.exists(p):
            continue
        r = raw(p)[0]
        rb, wb = to_bytes(r["dram__bytes_read.sum"]), to_bytes(r["dram__bytes_write.sum"])
        ns = to_ns(r["gpu__time_duration.sum"])
        summary[name] = {"kernel": r["kernel"], "source": f"ncu --set full ({rep})",
                         "dram_bytes_per_launch": rb + wb, "dram_read": rb, "dram_write": wb,
                         # tools/prof_run.py default sizes: fp32 32768^2 / int32 2^30
                         "algorithmic_bytes": 2 * 32768 * 32768 * 4 if name == "transpose" else (1 << 30) * 4 + 8,
                         "duration_ns_ncu": ns, "dram_GBps_ncu": (rb + wb) / ns,
                         "metrics": {k: v for k, v in r.items() if k != "kernel"}}
    lp = os.path.join(OUT, "launches.csv")
    if os.path.exists(lp):
        per = launches(lp)
        tot = sum(m.get("gpu__time_duration.sum", 0) for ms in per.values() for m in ms)
        tot_b2 = sum(m.get("gpu__time_duration.sum", 0) for k, ms in per.items() if "b2::" in k
                     for m in ms)
        summary["launch_list"] = {
            k: {"launches": len(ms),
                "mean_ns": sum(m.get("gpu__time_duration.sum", 0) for m in ms) / len(ms),
                "share": sum(m.get("gpu__time_duration.sum", 0) for m in ms) / tot if tot else None,
                "share_of_b2_step": (sum(m.get("gpu__time_duration.sum", 0) for m in ms) / tot_b2
                                     if tot_b2 and "b2::" in k else None),
                "mean_dram_bytes": sum(m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
                                       for m in ms) / len(ms)}
            for k, ms in per.items() if "b2::" in k or "--all" in sys.argv}
        # the bench STEP = the C4 transpose + the C3 reduction (the >= 1 GB launches);
        # their share of it is what the in-step CUDA events must agree with (the
        # paper_configs' small latency-bound launches also appear in the list)
        step = {k: v for k, v in summary["launch_list"].items() if v["mean_dram_bytes"] >= 1e9}
        tot_step = sum(v["mean_ns"] for v in step.values())
        for k, v in step.items():
            v["share_of_bench_step"] = v["mean_ns"] / tot_step
    with open(os.path.join(PROF, f"{tag}_ncu.json"), "w") as f:
        json.dump(summary, f, indent=1)
    with open(os.path.join(PROF, "ncu_summary.json"), "w") as f:
        json.dump(summary, f, indent=1)
    print(json.dumps({k: (v if not isinstance(v, dict) or "metrics" not in v else
                          {kk: vv for kk, vv in v.items() if kk != "metrics"})
                      for k, v in summary.items()}, indent=1))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r01")
