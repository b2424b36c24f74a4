"""One-off GPU-box probe: host cores, RAM, H2D/D2H pinned bandwidth, HBM copy."""
import os, subprocess, time, json
import torch
out = {}
out["nproc"] = os.cpu_count()
try:
    out["cpu"] = [l for l in open("/proc/cpuinfo") if l.startswith("model name")][0].split(":")[1].strip()
except Exception as e:
    out["cpu"] = str(e)
out["mem"] = open("/proc/meminfo").readline().strip()
out["ngpu"] = torch.cuda.device_count()
out["name"] = torch.cuda.get_device_name(0)
n = 1 << 30
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for _ in range(2):
    d.copy_(h, non_blocking=True); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); d.copy_(h, non_blocking=True); e1.record(); torch.cuda.synchronize()
out["h2d_GBs"] = n / e0.elapsed_time(e1) / 1e6
e0.record(); h.copy_(d, non_blocking=True); e1.record(); torch.cuda.synchronize()
out["d2h_GBs"] = n / e0.elapsed_time(e1) / 1e6
print(json.dumps(out))
