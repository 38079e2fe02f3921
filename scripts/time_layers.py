"""Kernel-only timing of the fused layer for several configs (CUDA events,
inputs > L2).  Used to compare kernel variants (SVD_LIB=<.so>)."""
import json
import os
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2506_03065_b200 as S  # noqa: E402

configs = sys.argv[1:] or ["hunyuan", "cogvideo", "wan"]
res = {"lib": os.environ.get("SVD_LIB", "default")}
for c in configs:
    dense = c.endswith("-dense")
    cfg = bench.CONFIGS[c.replace("-dense", "")]
    layout = S.TokenLayout(*cfg["layout"])
    n, H, d = layout.total_tokens, cfg["heads"], cfg["d"]
    specs = [S.full_spec()] * H if dense else bench.assignment_for(cfg, S)
    plan = S.plan_for_assignment(specs, layout)
    q, k, v = (torch.randn(1, H, n, d, device="cuda").to(torch.bfloat16) for _ in range(3))
    out = torch.empty_like(q)
    for _ in range(3):
        plan.forward(q, k, v, out, head_dim=d)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = int(os.environ.get("REPS", 3 if dense else 8))
    a.record()
    for _ in range(reps):
        plan.forward(q, k, v, out, head_dim=d)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    res[c] = {"ms": round(ms, 3), "active_tflops": round(plan.active_flops(d) / ms / 1e9, 1),
              "finite": bool(torch.isfinite(out).all())}
print(json.dumps(res))
