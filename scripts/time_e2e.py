"""Time the host-buffer public API path (pinned bf16 Q/K/V in, O out) for
head-chunk counts given on the command line."""
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
res = {}
for chunks in [int(c) for c in (sys.argv[2:] or ["1", "2", "4", "8"])]:
    A.HOST_CHUNKS = chunks
    for _ in range(2):
        S.fused_layer_attention(q, k, v, groups)
    ts = []
    for _ in range(4):
        t0 = time.perf_counter()
        S.fused_layer_attention(q, k, v, groups)
        ts.append((time.perf_counter() - t0) * 1e3)
    res[chunks] = round(sorted(ts)[len(ts) // 2], 2)
# raw transfer rates for reference
x = torch.empty(3 * H * n * d, dtype=torch.bfloat16).pin_memory()
y = torch.empty_like(x, device="cuda")
torch.cuda.synchronize()
t0 = time.perf_counter(); y.copy_(x, non_blocking=True); torch.cuda.synchronize()
h2d = x.numel() * 2 / (time.perf_counter() - t0) / 1e9
t0 = time.perf_counter(); x.copy_(y, non_blocking=True); torch.cuda.synchronize()
d2h = x.numel() * 2 / (time.perf_counter() - t0) / 1e9
print(json.dumps({"e2e_ms_by_chunks": res, "h2d_GBps": round(h2d, 1), "d2h_GBps": round(d2h, 1)}))
