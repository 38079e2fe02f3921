"""Timeline of the host-buffer pipeline (copy-in / kernel / copy-out per
chunk) from CUDA events: where the end-to-end time goes."""
import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2506_03065_b200 as S  # noqa: E402
from paper_2506_03065_b200 import attention as A  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "hunyuan"]
A.HOST_CHUNKS = int(sys.argv[2]) if len(sys.argv) > 2 else 0
layout = S.TokenLayout(*cfg["layout"])
n, H, d = layout.total_tokens, cfg["heads"], cfg["d"]
specs = bench.assignment_for(cfg, S)
plan = S.plan_for_assignment(specs, layout)
q, k, v = (torch.randn(1, H, n, d).to(torch.bfloat16).pin_memory() for _ in range(3))
hout = torch.empty(q.shape, dtype=torch.bfloat16).pin_memory()
groups = S.group_heads(specs, S.block_grid(layout))
for _ in range(2):
    S.fused_layer_attention(q, k, v, groups, out=hout)
order, bounds = A._host_schedule(plan, 1, n, d)
st = A._host_staging(plan, torch.device("cuda", 0), 1, n, d, d)
dev = torch.device("cuda", 0)
compute = torch.cuda.current_stream(dev)
E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
t0 = E()
t0.record(compute)
ev = {"in": [], "k": [], "out": []}
st.s_in.wait_stream(compute)
loaded = []
with torch.cuda.stream(st.s_in):
    for c in range(len(bounds) - 1):
        a = E(); a.record(st.s_in)
        for slot in range(bounds[c], bounds[c + 1]):
            for x, buf in zip((q, k, v), st.qkv):
                buf[:, slot].copy_(x[:, order[slot]], non_blocking=True)
        b = E(); b.record(st.s_in)
        ev["in"].append((a, b)); loaded.append(b)
comp = []
for c in range(len(bounds) - 1):
    s0, s1 = bounds[c], bounds[c + 1]
    compute.wait_event(loaded[c])
    a = E(); a.record(compute)
    plan.heads_subplan(tuple(order[s0:s1])).forward(*(buf[:, s0:s1] for buf in st.qkv), st.o[:, s0:s1],
                                                     head_dim=d, stream=compute)
    b = E(); b.record(compute)
    ev["k"].append((a, b)); comp.append(b)
with torch.cuda.stream(st.s_out):
    for c in range(len(bounds) - 1):
        st.s_out.wait_event(comp[c])
        a = E(); a.record(st.s_out)
        for slot in range(bounds[c], bounds[c + 1]):
            hout[:, order[slot]].copy_(st.o[:, slot], non_blocking=True)
        b = E(); b.record(st.s_out)
        ev["out"].append((a, b))
torch.cuda.synchronize()
res = {"bounds": bounds, "order": order}
for key, lst in ev.items():
    res[key] = [(round(t0.elapsed_time(a), 2), round(t0.elapsed_time(b), 2)) for a, b in lst]
print(json.dumps(res))
