"""Per-kind kernel efficiency at a production layout: the layer's FULL heads
alone, its sparse heads alone, and the whole layer (active TF/s each).

    python scripts/time_head_kinds.py [hunyuan|cogvideo|wan]"""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2506_03065_b200 as S  # noqa: E402


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


name = sys.argv[1] if len(sys.argv) > 1 else "hunyuan"
cfg = bench.CONFIGS[name]
layout = S.TokenLayout(*cfg["layout"])
asg = bench.assignment_for(cfg, S)
H, d, n = cfg["heads"], cfg["d"], layout.total_tokens
q, k, v = (torch.randn(1, H, n, d, device="cuda").bfloat16() for _ in range(3))
out = torch.empty_like(q)
plan = S.plan_for_assignment(asg, layout)
res = {"config": name}
for kind, heads in (("all", tuple(range(H))),
                    ("full", tuple(h for h in range(H) if int(asg[h].mode) == 0)),
                    ("sparse", tuple(h for h in range(H) if int(asg[h].mode) not in (0, 1)))):
    sub = plan.heads_subplan(heads)
    qs, ks, vs = (t[:, list(heads)].contiguous() for t in (q, k, v))
    os_ = torch.empty_like(qs)
    ms = timed(lambda: sub.forward(qs, ks, vs, os_))
    items, _ = sub.schedule()
    flops = sub.active_flops(d)
    res[kind] = {"heads": len(heads), "ms": round(ms, 3), "active_tflops": round(flops / ms / 1e9, 1),
                 "items": int(len(items)), "issued_tile_steps": int(items[:, 3].clip(0).sum())}
print(json.dumps(res))
