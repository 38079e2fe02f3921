"""Host<->device copy rates (pinned, 731 MB, one direction and both at once)."""
import json
import time

import torch

n = 24 * 119056 * 128
x = torch.empty(n, dtype=torch.bfloat16).pin_memory()
y = torch.empty(n, dtype=torch.bfloat16, device="cuda")
x2 = torch.empty(n, dtype=torch.bfloat16).pin_memory()
y2 = torch.empty(n, dtype=torch.bfloat16, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
res = {}
s3 = torch.cuda.Stream()
half = n // 2
for name in ("h2d", "d2h", "both", "h2d_2streams", "h2d_8chunks"):
    ts = []
    for _ in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if name in ("h2d", "both"):
            with torch.cuda.stream(s1):
                y.copy_(x, non_blocking=True)
        if name in ("d2h", "both"):
            with torch.cuda.stream(s2):
                x2.copy_(y2, non_blocking=True)
        if name == "h2d_2streams":  # two halves on two streams at once (two copy engines?)
            with torch.cuda.stream(s1):
                y[:half].copy_(x[:half], non_blocking=True)
            with torch.cuda.stream(s3):
                y[half:].copy_(x[half:], non_blocking=True)
        if name == "h2d_8chunks":  # the host pipeline's granularity: 8 copies in a row
            with torch.cuda.stream(s1):
                for c in range(8):
                    sl = slice(c * n // 8, (c + 1) * n // 8)
                    y[sl].copy_(x[sl], non_blocking=True)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    res[name + "_GBps"] = round(n * 2 / min(ts) / 1e9, 1)
t0 = time.perf_counter()
z = torch.empty(n, dtype=torch.bfloat16, pin_memory=True)
res["pin_alloc_731MB_ms"] = round((time.perf_counter() - t0) * 1e3, 1)
print(json.dumps(res))
