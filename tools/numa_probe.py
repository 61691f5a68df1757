"""Host topology vs PCIe bandwidth: H2D/D2H of 4 GiB pinned buffers allocated
(first touch) from CPUs of each NUMA node, and the NVML-reported CPU affinity of GPU 0."""
import json
import os
import subprocess
import sys
import time

import torch

out = {}
out["lscpu"] = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
out["topo"] = subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True).stdout
nodes = sorted(int(d[4:]) for d in os.listdir("/sys/devices/system/node") if d.startswith("node") and d[4:].isdigit())
cpus = {}
for nd in nodes:
    s = open(f"/sys/devices/system/node/node{nd}/cpulist").read().strip()
    lst = []
    for part in s.split(","):
        if "-" in part:
            a, b = part.split("-")
            lst += list(range(int(a), int(b) + 1))
        elif part:
            lst.append(int(part))
    cpus[nd] = lst
out["nodes"] = {k: len(v) for k, v in cpus.items()}
try:
    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    aff = pynvml.nvmlDeviceGetCpuAffinity(h, 4)
    bits = []
    for w, word in enumerate(aff):
        for b in range(64):
            if word >> b & 1:
                bits.append(w * 64 + b)
    out["nvml_affinity"] = bits
except Exception as e:  # noqa: BLE001
    out["nvml_affinity"] = str(e)
print(json.dumps({k: v for k, v in out.items() if k not in ("lscpu",)}, indent=1))
print(out["lscpu"])
n = 1 << 30
d = torch.empty(n, dtype=torch.float32, device="cuda")
res = []
for nd, cl in cpus.items():
    if not cl:
        continue
    os.sched_setaffinity(0, cl)
    h = torch.empty(n, dtype=torch.float32, pin_memory=True)
    h.numpy()[:] = 1.0  # first touch on this node
    for name, fn in [("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))]:
        fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / 3
        res.append({"node": nd, "what": name, "GBps": 4 * n / dt / 1e9})
        print(json.dumps(res[-1]), flush=True)
    del h
os.makedirs("gpurun_out", exist_ok=True)
json.dump({"res": res, "nodes": out["nodes"], "nvml_affinity": out["nvml_affinity"], "topo": out["topo"]},
          open("gpurun_out/numa_probe.json", "w"), indent=1)
