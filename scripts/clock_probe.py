"""Kernel time together with SM clock / power under sustained load: our
dense (all-FULL) and sparse layer launches vs cuDNN SDPA on the same inputs.
Under the B200's 1000 W cap the clock a kernel sustains depends on its
energy per step, so time alone does not separate issue efficiency from
power.  SVD_LIB selects a kernel variant library."""
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import torch
import torch.nn.functional as F
from torch.nn.attention import SDPBackend, sdpa_kernel

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2506_03065_b200 as S  # noqa: E402


class Sampler:
    def __init__(self):
        self.rows = []

    def __enter__(self):
        self.p = subprocess.Popen(["nvidia-smi", "--id=0", "--query-gpu=clocks.sm,power.draw",
                                   "--format=csv,noheader,nounits", "-lms", "50"],
                                  stdout=subprocess.PIPE, text=True)
        self.t = threading.Thread(target=lambda: [self.rows.append(l) for l in self.p.stdout], daemon=True)
        self.t.start()
        return self

    def __exit__(self, *a):
        self.p.terminate()
        self.p.wait()

    def summary(self):
        mhz, w = [], []
        for r in self.rows:
            try:
                a, b = (float(x) for x in r.split(","))
            except ValueError:
                continue
            mhz.append(a)
            w.append(b)
        n = len(mhz)
        mhz, w = mhz[n // 4:], w[n // 4:]  # drop the ramp
        return {"mhz": statistics.median(mhz) if mhz else None, "watts": statistics.median(w) if w else None}


def timed(fn, seconds=4.0):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Sampler() as s:
        t0 = time.time()
        n = 0
        a.record()
        while time.time() - t0 < seconds:
            fn()
            n += 1
            if n % 4 == 0:
                torch.cuda.synchronize()
        b.record()
        torch.cuda.synchronize()
    return {"ms": round(a.elapsed_time(b) / n, 3), **s.summary(), "reps": n}


cfgs = sys.argv[1:] or ["hunyuan"]
out = {"lib": os.environ.get("SVD_LIB", "default")}
for c in cfgs:
    cfg = bench.CONFIGS[c]
    layout = S.TokenLayout(*cfg["layout"])
    n, H, d = layout.total_tokens, cfg["heads"], cfg["d"]
    q, k, v = (torch.randn(1, H, n, d, device="cuda").to(torch.bfloat16) for _ in range(3))
    o = torch.empty_like(q)
    sp = S.plan_for_assignment(bench.assignment_for(cfg, S), layout)
    dp = S.plan_for_assignment([S.full_spec()] * H, layout)
    r = {"sparse": timed(lambda: sp.forward(q, k, v, o, head_dim=d)),
         "dense": timed(lambda: dp.forward(q, k, v, o, head_dim=d))}
    if os.environ.get("PROBE_CUDNN", "1") == "1":
        with sdpa_kernel([SDPBackend.CUDNN_ATTENTION]):
            r["cudnn_dense"] = timed(lambda: F.scaled_dot_product_attention(q, k, v))
    r["sparse"]["active_tflops"] = round(sp.active_flops(d) / r["sparse"]["ms"] / 1e9, 1)
    r["dense"]["tflops"] = round(dp.dense_flops(d) / r["dense"]["ms"] / 1e9, 1)
    if "cudnn_dense" in r:
        r["cudnn_dense"]["tflops"] = round(dp.dense_flops(d) / r["cudnn_dense"]["ms"] / 1e9, 1)
    out[c] = r
    del q, k, v, o
print(json.dumps(out), flush=True)
