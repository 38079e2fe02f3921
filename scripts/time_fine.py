"""Kernel time of a layer whose block size is off the 64-token segment grain
(FINE masks: per-element block lookups) vs. the same mix at block 64.

    python scripts/time_fine.py"""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2506_03065_b200 as S  # noqa: E402

cfg = bench.CONFIGS["hunyuan"]
H, d = cfg["heads"], cfg["d"]
res = {}
for block in (64, 32, 96):
    text, frames, tpf, _ = cfg["layout"]
    layout = S.TokenLayout(text, frames, tpf, block)
    asg = bench.assignment_for({**cfg, "layout": (text, frames, tpf, block)}, S)
    plan = S.plan_for_assignment(asg, layout)
    n = layout.total_tokens
    q, k, v = (torch.randn(1, H, n, d, device="cuda").bfloat16() for _ in range(3))
    out = torch.empty_like(q)
    for kind, heads in (("all", tuple(range(H))), ("full", tuple(h for h in range(H) if int(asg[h].mode) == 0))):
        sub = plan.heads_subplan(heads)
        qs, ks, vs = (t[:, list(heads)].contiguous() for t in (q, k, v))
        os_ = torch.empty_like(qs)
        sub.forward(qs, ks, vs, os_)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(3):
            sub.forward(qs, ks, vs, os_)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 3
        res[f"b{block}_{kind}"] = {"ms": round(ms, 2), "active_tflops": round(sub.active_flops(d) / ms / 1e9, 1),
                                   "fine": bool(sub.info.fine_mask)}
print(json.dumps(res))
