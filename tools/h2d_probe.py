"""Pinned host->device copy bandwidth with 1, 2 and 4 concurrent copy streams
(4 GiB total). Dev tool for the e2e roofline."""
import torch

n = 1 << 30
h = torch.empty(n, dtype=torch.float32).pin_memory()
d = torch.empty(n, dtype=torch.float32, device="cuda")
for ns in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    per = n // ns
    for rep in range(3):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i, s in enumerate(streams):
            s.wait_event(e0)
            with torch.cuda.stream(s):
                d[i * per:(i + 1) * per].copy_(h[i * per:(i + 1) * per], non_blocking=True)
        for s in streams:
            torch.cuda.current_stream().wait_stream(s)
        e1.record()
        e1.synchronize()
        if rep == 2:
            print(ns, "streams:", round(4 * n / (e0.elapsed_time(e1) * 1e-3) / 1e9, 1), "GB/s")
