"""Probe the GPU box: host, PCIe H2D/D2H pinned bandwidth, HBM copy."""
import os, subprocess, json, time
import torch
out = {}
out["nproc"] = os.cpu_count()
try:
    out["lscpu"] = subprocess.run(["bash", "-c", "lscpu | grep -E 'Model name|Socket|Core|Thread|NUMA node'"], capture_output=True, text=True).stdout
    out["mem"] = subprocess.run(["free", "-g"], capture_output=True, text=True).stdout
    out["smi"] = subprocess.run(["nvidia-smi"], capture_output=True, text=True).stdout
    out["topo"] = subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True).stdout
except Exception as e:
    out["err"] = str(e)
dev = torch.device("cuda:0")
res = {}
for mb in (1, 3.24, 5.4, 16, 64, 256):
    n = int(mb * 1e6)
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    s = torch.cuda.Stream()
    for _ in range(3):
        with torch.cuda.stream(s):
            d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    reps = 20
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        e0.record(s)
        for _ in range(reps):
            d.copy_(h, non_blocking=True)
        e1.record(s)
    torch.cuda.synchronize()
    h2d = n * reps / (e0.elapsed_time(e1) * 1e-3) / 1e9
    with torch.cuda.stream(s):
        e0.record(s)
        for _ in range(reps):
            h.copy_(d, non_blocking=True)
        e1.record(s)
    torch.cuda.synchronize()
    d2h = n * reps / (e0.elapsed_time(e1) * 1e-3) / 1e9
    res[str(mb)] = {"h2d_gbs": round(h2d, 2), "d2h_gbs": round(d2h, 2)}
out["pcie"] = res
print(json.dumps(out, indent=1))
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/probe_box.json", "w"), indent=1)
