"""Run one fused layer launch of a bench config (for ncu captures)."""
import argparse
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2506_03065_b200 as S  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="hunyuan")
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--dense", action="store_true")
a = ap.parse_args()
cfg = bench.CONFIGS[a.config]
layout = S.TokenLayout(*cfg["layout"])
n, H, d = layout.total_tokens, cfg["heads"], cfg["d"]
specs = [S.full_spec()] * H if a.dense else bench.assignment_for(cfg, S)
plan = S.plan_for_assignment(specs, layout)
q, k, v = (torch.randn(1, H, n, d, device="cuda").to(torch.bfloat16) for _ in range(3))
out = torch.empty_like(q)
for _ in range(a.reps):
    plan.forward(q, k, v, out, head_dim=d)
torch.cuda.synchronize()
print("ok", plan.info.n_work_items, plan.info.computed_tiles)
