#!/usr/bin/env python
"""Benchmark: effective GB/s of the OptiGPU transpose + tree reduction on B200.

One step = one pass of the hot path over one batch of synthetic input:
  * transpose  fp32 32768 x 32768 (BASELINE config C4: 4 GiB in + 4 GiB out)
  * reduction  int32 sum over 2^30 elements (config C3: 4 GiB in, int64 result)
    plus, at N > 1 GPUs, the cross-GPU combine of the per-GPU int64 partials
    (fused into the reduction kernel over NVLink, or one NCCL reduce).
Strong scaling (default, BASELINE configs[2] / [3]: the global problem is fixed
and "sharded at 1/2/4/8"): rank g transposes a 64-row-tile-aligned row block of
the 32768 x 32768 matrix and sums a contiguous 1/N of the 2^30 cells.
`--scaling weak` gives every rank a full-size C3 + C4 instead.

metric value = algorithmic bytes of all ranks / max-over-ranks device time,
bytes = 2*H*W*4 (transpose) + N*4 + 8 (reduction).
Inputs (4 GiB each) are larger than the 126 MB L2, so no flush is needed.

`--impl reference` times the reference's CPU path instead (the oracle port of
minigpu.interp; the reference itself is Python and cannot run at these sizes).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

TILE_ROWS, TILE_COLS = 32768, 32768
RED_N = 1 << 30
L2_BYTES = 126 * 1024 * 1024
FALLBACK_HBM = 6650.0
NOMINAL_HBM = 8000.0  # B200 HBM3e datasheet figure (north star: 'the ~8 TB/s HBM3e peak')


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--scaling", choices=["weak", "strong"], default="strong")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-ref-c2", action="store_true",
                   help="reference arm: skip the ~100 s full-size C2 run of the reference interpreter")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--no-graph", action="store_true", help="eager launches instead of a CUDA graph")
    p.add_argument("--combine", default="fused", choices=["fused", "nccl"],
                   help="N > 1: cross-GPU combine of the reduction partials")
    p.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                   help="gloo only to exercise the multi-rank path with several ranks on one GPU")
    p.add_argument("--paper-configs", action="store_true", default=True)
    # (long names: torchrun's own parser would swallow abbreviations like --n)
    p.add_argument("--transpose-rows", dest="rows", type=int, default=TILE_ROWS)
    p.add_argument("--transpose-cols", dest="cols", type=int, default=TILE_COLS)
    p.add_argument("--reduce-n", dest="n", type=int, default=RED_N)
    return p.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return FALLBACK_HBM, "fallback (B200_PROFILING.md 6.65 TB/s)"


def shard_sizes(args, world, rank):
    """Per-rank transpose rows and reduction elements: strong scaling splits the
    global C4 matrix into 64-row-tile-aligned row blocks and the C3 array into
    contiguous 16-B-aligned shards (shard.row_blocks)."""
    if args.scaling == "weak":
        return args.rows, args.cols, args.n
    r0, r1 = row_blocks(args.rows, world, 64)[rank]
    e0, e1 = row_blocks(args.n, world, 4)[rank]
    return r1 - r0, args.cols, e1 - e0


def row_blocks(H, world, align):
    """[(r0, r1)] per rank: align-multiple near-equal blocks covering [0, H)
    (the same split as paper_2605_13864_b200.shard.row_blocks, restated here so the
    reference arm needs nothing from the product package)."""
    units = -(-H // align) if H > 0 else 0
    base, extra = divmod(units, world)
    out, r = [], 0
    for g in range(world):
        r1 = min(H, r + (base + (1 if g < extra else 0)) * align)
        out.append((r, r1))
        r = r1
    return out


def workload_name(args, world):
    lg = int(np.log2(args.n)) if args.n > 0 and (args.n & (args.n - 1)) == 0 else None
    red = f"2^{lg}" if lg is not None else f"n={args.n}"
    if args.scaling == "weak":
        return (f"C4 fp32 {args.rows}x{args.cols} transpose + C3 int32 {red} sum per GPU "
                f"(weak scaling: global {world * args.rows}x{args.cols} + {world} x {red})")
    return (f"C4 fp32 {args.rows}x{args.cols} transpose + C3 int32 {red} sum "
            f"(global, strong scaling: row blocks / shards over {world} GPU{'s' if world > 1 else ''})")


def transpose_kernel_label(rows, cols):
    """The kernel the library dispatches for an aligned fp32 rows x cols transpose
    (transpose.cu dispatch / transpose_cpa.cu transpose_cpa_wanted, at the knob values
    this process runs with)."""
    from paper_2605_13864_b200 import _lib
    cpa, sms = _lib.tuning("transpose.cpa"), 148
    if cpa == 2 or (cpa == 1 and rows * cols * 4 >= 256 << 20 and (rows // 256) * (cols // 64) >= 2 * sms):
        if cpa == 2:
            return f"transpose_cpa_kernel variant {_lib.tuning('transpose.cpa_variant')} (forced)"
        return ("transpose_cpa_kernel<4,256,16,256,2,1> (cp.async-loaded 256x64 fp32 tiles, "
                "2 x 64-KB stages, L2 evict-first loads, 1 CTA/SM)")
    if (rows // 256) * (cols // 128) >= 8 * sms:
        return "transpose_vec_kernel<4,64,32,512> (256x128 fp32 tile, 1 CTA/SM)"
    return "transpose_vec_kernel<4,16,16,256> (64x64 fp32 tile)"


def config_for(args, world):
    """The workload config, identical in both arms (the driver compares them)."""
    return {"workload": workload_name(args, world), "rows": args.rows, "cols": args.cols, "n": args.n,
            "scaling": args.scaling, "l2": l2_note(args, world)}


def l2_note(args, world):
    rows, cols, n = shard_sizes(args, world, world - 1)  # the smallest shard
    small = min(rows * cols * 4, n * 4)
    return (f"per-GPU inputs >= {small / 2**20:.0f} MiB, larger than 2x L2 (126 MB): no flush needed"
            if small > 2 * L2_BYTES else "WARNING: per-GPU inputs not larger than 2x L2")


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """Polls NVML (SM clock + throttle reasons) in a thread while the GPU works."""

    REASONS = {
        "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4,
        "hw_slowdown": 0x8, "sync_boost": 0x10, "sw_thermal_slowdown": 0x20,
        "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80,
        "display_clock_setting": 0x100,
    }

    def __init__(self, dev):
        self.samples = []
        self.window = None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(dev)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # pragma: no cover
            self.nv = None
            self.err = str(e)
            self.max_mhz = None

    def start(self):
        if self.nv is None:
            return
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.samples.append((time.perf_counter(), sm, rs))
            except Exception:
                pass
            time.sleep(0.002)

    def stop(self):
        self._stop.set()
        if self.nv is not None:
            self.t.join()

    def summary(self):
        if self.nv is None:
            return {"error": getattr(self, "err", "nvml unavailable")}
        t0, t1 = self.window if self.window else (0, float("inf"))
        win = [s for s in self.samples if t0 <= s[0] <= t1]
        use = win if len(win) >= 3 else self.samples
        mhz = [s[1] for s in use]
        reasons = set()
        for _, _, rs in use:
            for k, bit in self.REASONS.items():
                if rs & bit and k != "gpu_idle":
                    reasons.add(k)
        return {"sm_mhz": statistics.median(mhz) if mhz else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(reasons), "samples": len(use),
                "window": "timed region" if use is win else "warmup+timed region"}


# ----------------------------------------------------------------------------- CPU legs
def cpu_leg(rows, cols, n, budget_s=10.0, max_reps=40):
    """Oracle (C restatement of minigpu.interp) on host cores: GB/s on a bounded
    sample, repeated for ~budget_s of CPU work (the first rep also faults in the
    output pages and is not timed); median over the timed reps."""
    from oracle import oracle
    threads = oracle.max_threads()
    a = np.empty((rows, cols), dtype=np.float32)
    oracle.fill_u32(a.view(np.uint32).reshape(-1), 1)
    out = np.empty((cols, rows), dtype=np.float32)
    x = np.empty(n, dtype=np.int32)
    oracle.fill_u32(x.view(np.uint32), 2)
    oracle.transpose_into(a, out)  # warm-up: thread pool, page faults of `out`
    s = oracle.reduce_i32(x)
    times = []
    t_all = time.perf_counter()
    while len(times) < max_reps and (len(times) < 3 or time.perf_counter() - t_all < budget_s):
        t0 = time.perf_counter()
        oracle.transpose_into(a, out)
        t1 = time.perf_counter()
        s = oracle.reduce_i32(x)
        t2 = time.perf_counter()
        times.append((t1 - t0) + (t2 - t1))
    bytes_ = 2 * rows * cols * 4 + n * 4 + 8
    assert np.array_equal(out[:5, :7].view(np.uint32), a[:7, :5].T.view(np.uint32))
    return {"value": bytes_ / statistics.median(times) / 1e9, "unit": "GB/s", "cores": threads,
            "reps": len(times), "seconds": time.perf_counter() - t_all, "checksum": s}


def interp_leg(rows, cols, n):
    """The reference's interpreter semantics on host cores: the A.1 transpose and
    A.3 int reduce PROGRAMS executed by oracle/vinterp.py (vectorised restatement
    of minigpu.interp, one core, numpy) on a bounded sample — what running the
    reference's own program path costs once it is not a per-element Python walk."""
    import paper_2605_13864_b200 as b2
    from oracle import oracle, vinterp
    a = np.empty((rows, cols), dtype=np.float32)
    oracle.fill_u32(a.view(np.uint32).reshape(-1), 3)
    a[~np.isfinite(a)] = 0.0  # finite cells, like the GPU leg's inputs
    out = np.zeros(rows * cols, np.float32)
    x = np.empty(n, dtype=np.int32)
    oracle.fill_u32(x.view(np.uint32), 4)
    tp = b2.parse_program(b2.programs.TRANSPOSE_NAIVE)
    rp = b2.parse_program(b2.programs.REDUCE_NAIVE_INT)
    t0 = time.perf_counter()
    vinterp.run_program(tp, "transpose", {"in": b2.Array([rows, cols], a.reshape(-1), "float"),
                                          "out": b2.Array([cols, rows], out, "float"), "W": cols, "H": rows},
                        as_numpy=True)
    t1 = time.perf_counter()
    s, _ = vinterp.run_program(rp, "reduce", {"arr": b2.Array([n], x, "int"), "N": n}, as_numpy=True)
    t2 = time.perf_counter()
    assert s == oracle.reduce_i32(x)
    assert np.array_equal(out.reshape(cols, rows)[:5, :7], a[:7, :5].T)
    bytes_ = 2 * rows * cols * 4 + n * 4 + 8
    return {"value": bytes_ / (t2 - t0) / 1e9, "unit": "GB/s", "cores": 1, "kind": "port",
            "transpose_s": t1 - t0, "reduce_s": t2 - t1,
            "sample": (f"programs A.1 (fp32 {rows}x{cols}) + A.3 (int32 n={n}) run by oracle/vinterp.py, "
                       "the vectorised restatement of minigpu.interp (single core)")}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from oracle import oracle
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    # strong scaling: the global C3 + C4 problem (one host does all of it); weak: the
    # per-GPU problem (the line is a rate, GB/s, so either is the same measurement)
    rows, cols, n = args.rows, args.cols, args.n
    threads = oracle.max_threads()
    a = np.empty((rows, cols), dtype=np.float32)
    oracle.fill_u32(a.view(np.uint32).reshape(-1), 1)
    out = np.empty((cols, rows), dtype=np.float32)
    x = np.empty(n, dtype=np.int32)
    oracle.fill_u32(x.view(np.uint32), 2)
    bytes_ = 2 * rows * cols * 4 + n * 4 + 8
    for _ in range(args.warmup):
        oracle.transpose_into(a, out)
        oracle.reduce_i32(x)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle.transpose_into(a, out)
        oracle.reduce_i32(x)
    dt = time.perf_counter() - t0
    v = bytes_ * args.steps / dt / 1e9
    sample = (f"full per-GPU workload each step: fp32 {rows}x{cols} transpose + int32 n={n} sum, "
              f"oracle C port of minigpu.interp (OpenMP, {threads} threads)")
    line = {
        "metric": "effective_GBps_transpose_plus_reduce", "value": v, "unit": "GB/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None, "dtype": "f32+i32", "data": "synthetic (splitmix64 bits)",
        "config": config_for(args, world),
        "impl": "reference",
        "cpu_baseline": {"value": v, "unit": "GB/s", "cores": threads, "kind": "port",
                         "sample": sample},
        "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": ("reference = minigpu.interp (pure Python, ~1 MB/s single core; cannot run 12 GiB "
                 "workloads), timed through its C restatement oracle/oracle.c; interp_semantics = "
                 "the same programs through the vectorised interpreter restatement"),
    }
    if not args.no_cpu:
        line["interp_semantics"] = interp_leg(min(rows, 2048), cols, min(n, 1 << 26))
        line["reference_interp"] = reference_interp_leg()
        if not args.no_ref_c2:
            line["reference_interp_c2"] = reference_c2_leg()
    print(json.dumps(line), flush=True)
    return 0


REF_INTERP_SCRIPT = r"""
import json, sys, time
sys.path.insert(0, sys.argv[1])
from minigpu.parser import parse_program
from minigpu.interp import Array, run_program
import numpy as np
tp, rp = parse_program(sys.argv[2]), parse_program(sys.argv[3])
rng = np.random.default_rng(1)
a = rng.uniform(-1, 1, (1024, 1024)).astype(np.float32)
inp = {"in": Array([1024, 1024], a.reshape(-1).tolist(), "float"),
       "out": Array.alloc([1024, 1024], "float"), "W": 1024, "H": 1024}
t0 = time.perf_counter()
_, outs = run_program(tp, "transpose", inp)
t1 = time.perf_counter()
ok_t = np.array_equal(np.array(outs["out"], np.float32), a.T.reshape(-1))
n = 1 << 20
x = rng.integers(-2**31, 2**31, n, dtype=np.int64).astype(np.int32).tolist()
t2 = time.perf_counter()
s, _ = run_program(rp, "reduce", {"arr": x, "N": n})
t3 = time.perf_counter()
print(json.dumps({"transpose_s": t1 - t0, "reduce_s": t3 - t2, "ok": bool(ok_t and s == sum(x))}))
"""


REF_C2_SCRIPT = r"""
import json, sys, time
sys.path.insert(0, sys.argv[1])
from minigpu.parser import parse_program
from minigpu.interp import run_program
import numpy as np
p = parse_program(sys.argv[2])
pin = json.loads(sys.argv[3])
x = np.random.default_rng(pin["seed"]).uniform(pin["lo"], 1, pin["n"]).astype(np.float32).tolist()
t0 = time.perf_counter()
s, _ = run_program(p, "reduce", {"arr": x, "N": len(x)})
t1 = time.perf_counter()
bits = int(np.float32(s).view(np.uint32))
print(json.dumps({"seconds": t1 - t0, "result_f32_bits": bits, "ok": bits == pin["result_f32_bits"]}))
"""


def reference_c2_leg(timeout_s=400):
    """The reference ITSELF on the paper's case study 2 / BASELINE C2 at full size:
    program A.2 (naive fp32 sum) over 2^24 cells, the input of the first pinned C2 case
    (tests/golden/fullsize_ref.json, generated by the reference here); its binary32
    result must equal the pinned bits. ~100 s of one core in the build container."""
    import subprocess
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "minigpu")):
        return {"unavailable": "baseline/_ref/minigpu not installed (run __graft_entry__.build())"}
    sys.path.insert(0, ROOT)
    from paper_2605_13864_b200 import programs
    try:
        with open(os.path.join(ROOT, "tests", "golden", "fullsize_ref.json")) as f:
            pin = json.load(f)["C2"][0]
        r = subprocess.run([sys.executable, "-c", REF_C2_SCRIPT, ref, programs.source(programs.REDUCE_NAIVE, "float"),
                            json.dumps(pin)], capture_output=True, text=True, timeout=timeout_s)
        d = json.loads(r.stdout.strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001 - reported, not fatal
        return {"unavailable": f"reference C2 run failed: {str(e)[:200]}"}
    nb = pin["n"] * 4 + 4
    return {"kind": "reference", "cores": 1, "value": nb / d["seconds"] / 1e9, "unit": "GB/s",
            "seconds": d["seconds"], "bit_exact_vs_pin": d["ok"],
            "sample": ("minigpu.interp.run_program (baseline/_ref, unmodified) on program A.2 over fp32 "
                       f"2^24 cells (BASELINE C2 / paper case study 2, seed {pin['seed']}), single core")}


def reference_interp_leg(timeout_s=240):
    """The reference ITSELF (minigpu.interp.run_program, pure Python, one core) on
    BASELINE C1 (fp32 1024^2, program A.1) and an int32 2^20 sum (program A.3),
    from the copy `__graft_entry__.build()` pip-installs into baseline/_ref (it
    travels to the GPU box; /root/reference does not). A separate process with a
    timeout; its GB/s anchors what the C port stands in for at C3/C4 sizes."""
    import subprocess
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "minigpu")):
        return {"unavailable": "baseline/_ref/minigpu not installed (run __graft_entry__.build())"}
    sys.path.insert(0, ROOT)
    from paper_2605_13864_b200 import programs
    try:
        r = subprocess.run([sys.executable, "-c", REF_INTERP_SCRIPT, ref, programs.TRANSPOSE_NAIVE,
                            programs.REDUCE_NAIVE_INT], capture_output=True, text=True, timeout=timeout_s)
        d = json.loads(r.stdout.strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001 - reported, not fatal
        return {"unavailable": f"reference interpreter run failed: {str(e)[:200]}"}
    bt, br = 2 * 1024 * 1024 * 4, (1 << 20) * 4 + 8
    return {"kind": "reference", "cores": 1, "value": (bt + br) / (d["transpose_s"] + d["reduce_s"]) / 1e9,
            "unit": "GB/s", "transpose_GBps": bt / d["transpose_s"] / 1e9,
            "reduce_GBps": br / d["reduce_s"] / 1e9, "seconds": d["transpose_s"] + d["reduce_s"],
            "bit_exact": d["ok"],
            "sample": ("minigpu.interp.run_program (baseline/_ref, unmodified) on program A.1 over fp32 "
                       "1024x1024 (BASELINE C1) + program A.3 over int32 2^20, single core")}


# ----------------------------------------------------------------------------- GPU arm
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    # one process per GPU; the modulo only matters for --dist-backend gloo test runs
    # that put several ranks on one device to exercise the N > 1 code path
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(args.dist_backend)

    import paper_2605_13864_b200 as b2
    from paper_2605_13864_b200 import ops

    ops.set_host_device(local)
    dev = torch.device("cuda", local)
    rows, cols, n = shard_sizes(args, world, rank)
    g = torch.Generator(device=dev).manual_seed(1234 + rank)
    a = torch.rand((rows, cols), device=dev, generator=g) * 2 - 1
    out = torch.empty((cols, rows), device=dev)
    x = torch.randint(-2**31, 2**31, (n,), device=dev, dtype=torch.int64, generator=g).to(torch.int32)
    partial = torch.zeros(1, dtype=torch.int64, device=dev)
    torch.cuda.synchronize()

    st = torch.cuda.current_stream(dev)

    # N > 1 combine of the per-GPU partials: fused into the reduction kernel (the
    # partial goes straight into rank 0's mailbox over NVLink) or one NCCL reduce
    combine = args.combine if world > 1 else "none"
    fused = None
    combine_note = None
    if combine == "fused":
        try:
            from paper_2605_13864_b200 import shard
            fused = shard.FusedReduce()
        except Exception as e:  # e.g. no CUDA IPC / peer access between these GPUs
            combine, combine_note = "nccl", f"fused combine unavailable ({e}); NCCL reduce used"

    def step(ev=None):
        if ev is not None:
            ev[0].record(st)
        b2.transpose(a, out)
        if ev is not None:
            ev[1].record(st)
        if fused is not None:
            fused(x, out=partial)
        else:
            b2.reduce_sum(x, out=partial)
        if ev is not None:
            ev[2].record(st)
        if world > 1 and fused is None:
            if args.dist_backend == "nccl":
                dist.reduce(partial, dst=0)  # one NCCL reduce of the 8-byte partial
            else:
                dist.all_reduce(partial)  # gloo has no CUDA reduce

    # correctness spot checks (cheap, outside the timed region)
    want = x.to(torch.int64).sum().reshape(1)
    if world > 1:
        dist.all_reduce(want)
    step()
    torch.cuda.synchronize()
    assert torch.equal(out[:64, :64], a[:64, :64].t()) and torch.equal(out[-64:, -64:], a[-64:, -64:].t())
    if fused is not None:
        bad = torch.tensor([0 if (rank != 0 or (int(partial.item()) == int(want.item())
                                                and fused.status() == 0)) else 1], device=dev)
        dist.all_reduce(bad)
        if int(bad.item()):
            fused, combine = None, "nccl"
            combine_note = "fused combine failed its check; NCCL reduce used"
            step()
            torch.cuda.synchronize()
    if rank == 0:
        assert int(partial.item()) == int(want.item()), "reduction combine mismatch"

    clk = ClockSampler(local)
    clk.start()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    # N = 1: the K timed steps are captured once into a CUDA graph (with external
    # event-record nodes around every kernel) and replayed once: no per-launch host
    # overhead between kernels. N > 1 keeps eager launches (the NCCL combine).
    use_graph = world == 1 and not args.no_graph
    mk = (lambda: torch.cuda.Event(enable_timing=True, external=True)) if use_graph else \
        (lambda: torch.cuda.Event(enable_timing=True))
    evs = [[mk() for _ in range(3)] for _ in range(args.steps)]
    t_start, t_end = mk(), mk()
    graph = None
    launches_per_run = None
    if use_graph:
        cs = torch.cuda.Stream(dev)
        cs.wait_stream(st)
        graph = torch.cuda.CUDAGraph()
        l0 = b2.launch_count()
        with torch.cuda.stream(cs):
            with torch.cuda.graph(graph, stream=cs):
                st = torch.cuda.current_stream(dev)
                t_start.record(st)
                for i in range(args.steps):
                    step(evs[i])
                t_end.record(st)
        launches_per_run = b2.launch_count() - l0
        st = torch.cuda.current_stream(dev)
        graph.replay()  # untimed warm replay
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = b2.launch_count()
    w0 = time.perf_counter()
    torch.cuda.nvtx.range_push("bench.timed_region")
    if use_graph:
        graph.replay()
    else:
        t_start.record(st)
        for i in range(args.steps):
            step(evs[i])
        t_end.record(st)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()
    w1 = time.perf_counter()
    if world > 1:
        dist.barrier()
    clk.window = (w0, w1)
    clk.stop()
    launches = launches_per_run if use_graph else b2.launch_count() - launches0
    ms = t_start.elapsed_time(t_end)
    ms_t = statistics.mean(e[0].elapsed_time(e[1]) for e in evs)
    ms_r = statistics.mean(e[1].elapsed_time(e[2]) for e in evs)
    ms_max = ms
    ms_k = (ms_t + ms_r) * args.steps  # transpose + reduce kernels (a separate NCCL combine excluded)
    if world > 1:
        tt = torch.tensor([ms, ms_k], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms_max, ms_k = float(tt[0].item()), float(tt[1].item())

    bytes_t = 2 * rows * cols * 4
    bytes_r = n * 4 + 8
    tot_rows = rows * world if args.scaling == "weak" else args.rows
    tot_n = n * world if args.scaling == "weak" else args.n
    total_bytes = 2 * tot_rows * cols * 4 + tot_n * 4 + 8 * world  # every rank reads its cells once
    # and writes one 8-byte partial
    value = total_bytes * args.steps / (ms_max / 1e3) / 1e9
    # aggregate GB/s also without the combine step (with the fused combine
    # it runs inside the reduction kernel and cannot be separated)
    value_k = total_bytes * args.steps / (ms_k / 1e3) / 1e9
    peak, peak_src = peaks()
    ach_t = bytes_t / (ms_t / 1e3) / 1e9
    ach_r = bytes_r / (ms_r / 1e3) / 1e9
    # ncu DRAM bytes of the profiled launch (profiles/ncu_summary.json, tools/prof_run.py
    # at the default sizes); only meaningful when this run's launch has the same size
    traffic = traffic_r = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            prof = json.load(f)
        pt, pr = prof.get("transpose", {}), prof.get("reduce", {})
        if pt.get("algorithmic_bytes", 2 * TILE_ROWS * TILE_COLS * 4) == bytes_t:
            traffic = pt.get("dram_bytes_per_launch")
        if pr.get("algorithmic_bytes", RED_N * 4 + 8) == bytes_r:
            traffic_r = pr.get("dram_bytes_per_launch")
    except Exception:
        pass

    res = {
        "metric": "effective_GBps_transpose_plus_reduce", "value": value, "unit": "GB/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_max / args.steps, "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None, "dtype": "f32+i32", "data": "synthetic (torch.rand / randint on device)",
        "config": config_for(args, world),
        "shard": {"rank0_rows": rows, "cols": cols, "rank0_n": n,
                  "split": ("64-row-tile-aligned row blocks + contiguous 16-B-aligned reduction shards"
                            if args.scaling == "strong" else "every rank a full-size C3 + C4")},
        "combine": ("fused into the reduction kernel (partial -> rank 0 mailbox over "
                    "NVLink, release/acquire epochs)" if combine == "fused" else
                    f"{args.dist_backend} {'reduce' if args.dist_backend == 'nccl' else 'all_reduce'}"
                    " of the int64 partial" if world > 1 else "none (1 GPU)"),
        "combine_note": combine_note,
        "roofline": {"bound": "hbm",
                     "kernel": transpose_kernel_label(rows, cols),
                     "achieved": ach_t, "peak": peak, "unit": "GB/s", "frac": ach_t / peak,
                     "traffic": traffic, "algorithmic_bytes": bytes_t, "peak_source": peak_src,
                     "frac_nominal_8TBs": ach_t / NOMINAL_HBM},
        "kernels": {
            "transpose": {"ms": ms_t, "GBps": ach_t, "frac": ach_t / peak, "bytes": bytes_t,
                          "traffic": traffic},
            "reduce": {"ms": ms_r, "GBps": ach_r, "frac": ach_r / peak, "bytes": bytes_r,
                       "traffic": traffic_r},
        },
        "gpu_launches": launches,
        "value_kernels_only": value_k,
        # north star: whole-job GB/s as a fraction of the aggregate HBM roofline (N x peak)
        "aggregate_roofline": {"peak": peak * world, "unit": "GB/s", "frac": value / (peak * world),
                               "frac_kernels_only": value_k / (peak * world),
                               "frac_nominal_8TBs": value / (NOMINAL_HBM * world)},
        "launch_mode": ("CUDA graph: K steps captured once, replayed once in the timed region"
                        if use_graph else "eager stream launches"),
        "clocks": clk.summary(),
    }

    if not args.no_e2e:
        # pinned host buffers: 12 GiB per rank at the default sizes; if the host cannot
        # pin that much, measure the same path on half-height / half-length shards
        try:
            res["e2e"] = e2e_leg(b2, a, x, rows, cols, n, args, world, dev)
        except (RuntimeError, MemoryError) as e:
            import gc
            gc.collect()
            torch.cuda.empty_cache()
            res["e2e"] = e2e_leg(b2, a[: rows // 2], x[: n // 2], rows // 2, cols, n // 2, args, world, dev)
            res["e2e"]["note"] = f"half-size shards: full-size pinned buffers failed ({str(e)[:120]})"
    if args.paper_configs and world == 1:
        res["paper_configs"] = paper_configs(b2, dev)
    if rank == 0 and not args.no_cpu:
        # on rank 0 at every N (the other ranks wait at the barrier below): the SCALE
        # series then carries the same CPU yardstick on every line
        c = cpu_leg(min(rows, 8192), cols, min(n, 1 << 28))
        res["cpu_baseline"] = {
            "value": c["value"], "unit": "GB/s", "cores": c["cores"], "kind": "port",
            "sample": (f"oracle C port on fp32 {min(rows, 8192)}x{cols} transpose + int32 "
                       f"n={min(n, 1 << 28)} sum: median of {c['reps']} reps over {c['seconds']:.1f} s "
                       "after one untimed rep; same byte formula"),
        }
    if world > 1:
        dist.barrier()
    if rank == 0:
        print(json.dumps(res), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def e2e_leg(b2, a, x, rows, cols, n, args, world, dev):
    """Same step through the host-buffer public API: pinned host inputs, H2D +
    kernels + D2H inside the timed region (wall clock around the synchronous calls)."""
    import torch
    import torch.distributed as dist
    hin = torch.empty((rows, cols), dtype=torch.float32, pin_memory=True)
    hout = torch.empty((cols, rows), dtype=torch.float32, pin_memory=True)
    hx = torch.empty(n, dtype=torch.int32, pin_memory=True)
    hin.copy_(a)
    hx.copy_(x)
    hin_n, hout_n, hx_n = hin.numpy(), hout.numpy(), hx.numpy()
    steps = max(1, min(args.steps, 5))
    # the reference-facing API: run_program on the paper's programs, host Arrays
    tp = b2.parse_program(b2.programs.TRANSPOSE_NAIVE)
    rp = b2.parse_program(b2.programs.REDUCE_NAIVE_INT)
    t_in = {"in": b2.Array.from_numpy(hin_n), "out": b2.Array.from_numpy(hout_n),
            "W": cols, "H": rows}
    r_in = {"arr": b2.Array.from_numpy(hx_n, "int"), "N": n}

    def e2e_step():
        b2.run_program(tp, "transpose", t_in)
        return b2.run_program(rp, "reduce", r_in)[0]

    s = e2e_step()  # warm the staging buffers
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        s = e2e_step()
    dt = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([dt], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dt = float(t.item())
    assert np.array_equal(hout_n[:8, :8], hin_n[:8, :8].T)
    tot = (2 * rows * cols * 4 + n * 4 + 8) * world
    return {"value": tot * steps / dt / 1e9, "unit": "GB/s", "steps": steps,
            "h2d_bytes_per_step": rows * cols * 4 + n * 4,
            "d2h_bytes_per_step": rows * cols * 4 + 8,
            "api": "run_program(transpose A.1) + run_program(reduce A.3) on pinned numpy-backed "
                   "Arrays -> b2_transpose_host / b2_reduce_sum_host (H2D, kernel, D2H overlapped)",
            "checksum": int(s)}


def paper_configs(b2, dev):
    """PAPER.md Table 7.4 workloads (4096^2 fp32 transpose, 2^24 fp32 sum) and
    BASELINE C1 (1024^2 fp32 transpose), timed two ways against cold L2:
    - single launch between CUDA events after a read pass over 2x L2 (includes the
      event-pair floor, ~6 us here: profiles/r01i_small_sizes.json);
    - pipelined: one CUDA graph of back-to-back launches over R rotating inputs
      whose total is >= 3x L2, so no launch finds its input in L2."""
    import torch
    # cold L2 without dirty lines: a READ pass over 2x L2 before every launch (a
    # write flush would leave ~L2 of dirty lines whose write-back lands inside the
    # timed kernel)
    flush = torch.ones(2 * L2_BYTES // 4, dtype=torch.float32, device=dev)
    out = {}

    def transpose_case(n):
        R = max(2, -(-3 * L2_BYTES // (2 * n * n * 4)))
        a = [torch.rand((n, n), device=dev) for _ in range(R)]
        o = [torch.empty_like(a[0]) for _ in range(R)]
        return R, (lambda i: b2.transpose(a[i], o[i])), (a, o)

    def reduce_case(n):
        R = max(2, -(-3 * L2_BYTES // (n * 4)))
        x = [torch.rand(n, device=dev) for _ in range(R)]
        r = [torch.empty(1, device=dev) for _ in range(R)]
        return R, (lambda i: b2.reduce_sum(x[i], out=r[i])), (x, r)

    for name, make, n, bytes_, paper in [
        ("transpose_1024sq_f32", transpose_case, 1024, 2 * 1024 * 1024 * 4, None),
        ("transpose_4096sq_f32", transpose_case, 4096, 2 * 4096 * 4096 * 4, 340.6),
        ("reduce_2^24_f32", reduce_case, 1 << 24, (1 << 24) * 4 + 4, 376.8),
    ]:
        R, fn, keep = make(n)
        ts = []
        for i in range(23):
            flush.sum()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn(0)
            e1.record()
            torch.cuda.synchronize()
            if i >= 3:
                ts.append(e0.elapsed_time(e1))
        med = statistics.median(ts)
        K = max(2 * R, 64)
        s = torch.cuda.Stream(device=dev)
        with torch.cuda.stream(s):
            for i in range(R):
                fn(i)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for i in range(K):
                fn(i % R)
        tp = []
        for i in range(8):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            if i >= 2:
                tp.append(e0.elapsed_time(e1) / K)
        pip = statistics.median(tp)
        out[name] = {"ms_median": med, "GBps": bytes_ / (med / 1e3) / 1e9,
                     "ms_pipelined": pip, "GBps_pipelined": bytes_ / (pip / 1e3) / 1e9,
                     "paper_best_rtx5060_GBps": paper,
                     "l2": "cold: 252 MB read pass (clean lines) before every single launch; "
                           f"pipelined: graph of {K} launches over {R} rotating inputs (>= 3x L2)"}
        del g, keep
        torch.cuda.empty_cache()
    return out


if __name__ == "__main__":
    sys.exit(main())
