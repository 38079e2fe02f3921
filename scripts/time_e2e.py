"""Time the host-buffer public API path (pinned bf16 Q/K/V in, O out) per
step, with a fresh pinned result per call and with a caller-owned pinned out=
buffer, for head-chunk counts given on the command line."""
import json
import sys
import time
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2506_03065_b200 as S  # noqa: E402
from paper_2506_03065_b200 import attention as A  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "hunyuan"]
layout = S.TokenLayout(*cfg["layout"])
n, H, d = layout.total_tokens, cfg["heads"], cfg["d"]
groups = S.group_heads(bench.assignment_for(cfg, S), S.block_grid(layout))
q, k, v = (torch.randn(1, H, n, d).to(torch.bfloat16).pin_memory() for _ in range(3))
hout = torch.empty(q.shape, dtype=torch.bfloat16).pin_memory()
res = {}
for chunks in [int(c) for c in (sys.argv[2:] or ["0", "6"])]:  # 0 = flow-shop schedule
    A.HOST_CHUNKS = chunks
    for mode in ("alloc", "out"):
        kw = {"out": hout} if mode == "out" else {}
        for _ in range(2):
            S.fused_layer_attention(q, k, v, groups, **kw)
        ts = []
        for _ in range(6):
            t0 = time.perf_counter()
            S.fused_layer_attention(q, k, v, groups, **kw)
            ts.append(round((time.perf_counter() - t0) * 1e3, 1))
        res[f"{chunks}_{mode}"] = ts
print(json.dumps({"e2e_wall_ms": res}))
