"""Strong-scaling proxy on one GPU: time every rank's shard kernel of a bench
layer for world = 1, 2, 4, 8 (packed-row output, CUDA events), with the
planner's split-KV on and off.  max over ranks of the shard time is the
per-GPU compute time of an N-GPU run (NVLink stores excluded); efficiency =
T_1 / (N * max_r T_r)."""
import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2506_03065_b200 as S  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "hunyuan"
cfg = bench.CONFIGS[cfgname]
layout = S.TokenLayout(*cfg["layout"])
n, H, d = layout.total_tokens, cfg["heads"], cfg["d"]
plan = S.plan_for_assignment(bench.assignment_for(cfg, S), layout)
q, k, v = (torch.randn(1, H, n, d, device="cuda").to(torch.bfloat16) for _ in range(3))


def timed(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


out = torch.empty_like(q)
t1 = timed(lambda: plan.forward(q, k, v, out, head_dim=d))
res = {"config": cfgname, "t1_ms": round(t1, 3)}
policies = sys.argv[2].split(",") if len(sys.argv) > 2 else ["auto", "none"]
for pol in policies:
    for world in (2, 4, 8):
        times = []
        for r in range(world):
            part = "items"
            if pol == "auto":
                cap = 0
            elif pol == "heads":  # contiguous head ranges, split cap chosen by the planner
                cap, part = 0, "heads"
            elif pol == "none":
                cap = -1
            else:  # "divN": cap = mean per-SM load / N
                per_sm = plan.shard(world, r, max_item_tiles=-1).info.computed_tiles / 2 / 148
                cap = max(32, int(per_sm / float(pol[3:])))
            sh = plan.shard(world, r, max_item_tiles=cap, partition=part)
            rows = max(1, len(sh.shard_rows()[0]))
            packed = torch.empty(rows, d, dtype=torch.bfloat16, device="cuda")
            times.append(timed(lambda: sh.forward(q, k, v, packed, head_dim=d), reps=3))
        res[f"w{world}_{pol}"] = {"max_ms": round(max(times), 3), "min_ms": round(min(times), 3),
                                  "efficiency": round(t1 / (world * max(times)), 3)}
print(json.dumps(res))
