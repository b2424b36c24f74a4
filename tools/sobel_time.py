"""C4 Sobel kernel time at 16384^2 / 64 bands (one process; the variant comes
from the environment: UCG_SOBEL_VARIANT, UCG_SOBEL_ROWS_MINB). Prints one
JSON line with the mean of 20 launches (CUDA events; the 276 MB input is
2x L2) and an FNV of the output for cross-variant equality."""
import hashlib
import json
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_1505_01120_b200 import ops  # noqa: E402

H = W = 16384
R = 256
nb = H // R
inp = torch.empty(nb * (R + 2) * W, dtype=torch.uint8, device="cuda")
ops.fill_bytes_(inp, 7)
out = torch.empty(H * W, dtype=torch.uint8, device="cuda")
args = (inp, [b * (R + 2) * W for b in range(nb)], out, [b * R * W for b in range(nb)], [R] * nb, W)
for _ in range(3):
    ops.sobel_bands(*args)
iters = int(os.environ.get("SOBEL_ITERS", "20"))
clk = []
if iters > 20:  # long runs: sample the SM clock and power while the loop runs (pynvml)
    import threading

    import pynvml

    pynvml.nvmlInit()
    hdl = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
    stop = threading.Event()

    def sample():
        while not stop.is_set():
            clk.append((pynvml.nvmlDeviceGetClockInfo(hdl, pynvml.NVML_CLOCK_SM),
                        pynvml.nvmlDeviceGetPowerUsage(hdl) / 1000.0))
            stop.wait(0.005)

    th = threading.Thread(target=sample)
    th.start()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record()
for _ in range(iters):
    ops.sobel_bands(*args)
e1.record()
torch.cuda.synchronize()
if iters > 20:
    stop.set()
    th.join()
us = e0.elapsed_time(e1) / iters * 1e3
algo = inp.numel() + out.numel()
print(json.dumps({"variant": os.environ.get("UCG_SOBEL_VARIANT", "0"), "minb": os.environ.get("UCG_SOBEL_ROWS_MINB", "5"),
                  "us": us, "gbs": algo / us / 1e3, "iters": iters,
                  "sm_mhz_median": sorted(c for c, _ in clk)[len(clk) // 2] if clk else None,
                  "watts_median": sorted(w for _, w in clk)[len(clk) // 2] if clk else None, "md5": hashlib.md5(out.cpu().numpy().tobytes()).hexdigest()}))
