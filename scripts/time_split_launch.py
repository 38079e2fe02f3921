"""Whole layer as one launch vs the FULL-head and sparse-head sub-plans as
two launches (one stream, either order; or two streams).

    python scripts/time_split_launch.py [hunyuan|cogvideo|wan]"""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2506_03065_b200 as S  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "hunyuan"
cfg = bench.CONFIGS[name]
layout = S.TokenLayout(*cfg["layout"])
asg = bench.assignment_for(cfg, S)
H, d, n = cfg["heads"], cfg["d"], layout.total_tokens
q, k, v = (torch.randn(1, H, n, d, device="cuda").bfloat16() for _ in range(3))
out = torch.empty_like(q)
plan = S.plan_for_assignment(asg, layout)
full = tuple(h for h in range(H) if int(asg[h].mode) == 0)
rest = tuple(h for h in range(H) if int(asg[h].mode) != 0)
pf, pr = plan.heads_subplan(full), plan.heads_subplan(rest)
mf, mr = (torch.tensor(hs, dtype=torch.int32, device="cuda") for hs in (full, rest))
qf, kf, vf = (t[:, list(full)].contiguous() for t in (q, k, v))
qr, kr, vr = (t[:, list(rest)].contiguous() for t in (q, k, v))
s2 = torch.cuda.Stream()
main = torch.cuda.current_stream()


def one():
    plan.forward(q, k, v, out)


def seq_fr():
    pf.forward(qf, kf, vf, out, o_head_map=mf)
    pr.forward(qr, kr, vr, out, o_head_map=mr)


def seq_rf():
    pr.forward(qr, kr, vr, out, o_head_map=mr)
    pf.forward(qf, kf, vf, out, o_head_map=mf)


def two():
    s2.wait_stream(main)
    pf.forward(qf, kf, vf, out, o_head_map=mf)
    with torch.cuda.stream(s2):
        pr.forward(qr, kr, vr, out, o_head_map=mr, stream=s2)
    main.wait_stream(s2)


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return round(a.elapsed_time(b) / reps, 3)


res = {"config": name}
for rnd in range(2):
    for label, fn in (("one_launch", one), ("full_then_rest", seq_fr), ("rest_then_full", seq_rf),
                      ("two_streams", two)):
        res.setdefault(label, []).append(timed(fn))
print(json.dumps(res))
