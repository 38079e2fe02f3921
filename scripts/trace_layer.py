"""Run one fused layer with the SVD_TRACE build and summarise the pipeline
timeline of the first traced CTAs (clock cycles)."""
import ctypes
import json
import os
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
os.environ.setdefault("SVD_LIB", str(ROOT / "paper_2506_03065_b200/variants/trace.so"))
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2506_03065_b200 as S  # noqa: E402
from paper_2506_03065_b200 import _native as nat  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "hunyuan"
cfg = bench.CONFIGS[cfgname]
layout = S.TokenLayout(*cfg["layout"])
n, H, d = layout.total_tokens, cfg["heads"], cfg["d"]
plan = S.plan_for_assignment(bench.assignment_for(cfg, S), layout)
q, k, v = (torch.randn(1, H, n, d, device="cuda").to(torch.bfloat16) for _ in range(3))
out = torch.empty_like(q)
lib = nat.lib()
lib.svd_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32]
plan.forward(q, k, v, out, head_dim=d)
buf = np.zeros((8, 4, 2048, 2), dtype=np.uint32)
nat.check(lib.svd_debug_trace(None, 0, 1))
plan.forward(q, k, v, out, head_dim=d)
nat.check(lib.svd_debug_trace(buf.ctypes.data, buf.nbytes, 0))
res = {}
for cta in range(8):
    ev = {}
    for st in range(4):
        for clk, w in buf[cta, st]:
            if w == 0 and clk == 0:
                continue
            ev.setdefault(st, []).append((int(clk), int(w) >> 8, int(w) & 255))
    def times(st, code):
        return {j: c for c, j, cd in ev.get(st, []) if cd == code}
    r = {}
    for x in (0, 1):
        before, ready, done = times(x, 0), times(x, 1), times(x, 2)
        js = [j for j in range(20, 400) if j in ready and j in done and j + 1 in ready and j in before]
        if not js:
            continue
        act = np.median([(done[j] - ready[j]) & 0xFFFFFFFF for j in js])
        wait = np.median([(ready[j] - before[j]) & 0xFFFFFFFF for j in js])
        per = np.median([(ready[j + 1] - ready[j]) & 0xFFFFFFFF for j in js])
        r[f"tile{x}"] = {"softmax_active": float(act), "wait_S": float(wait), "period": float(per)}
        ph = {c: times(x, c) for c in (3, 4, 5, 6)}
        if not ph[5]:  # no ping-pong turn event: the exp phase starts at event 4
            ph[5] = ph[4]
        def med(a, b):
            v = [(b[j] - a[j]) & 0xFFFFFFFF for j in js if j in a and j in b]
            return float(np.median(v)) if v else None
        r[f"tile{x}"].update({"ready_to_loaded": med(ready, ph[3]), "loaded_to_max": med(ph[3], ph[4]),
                              "turn_wait": med(ph[4], ph[5]), "exp_half0": med(ph[5], ph[6]),
                              "exp_half1": med(ph[6], done)})
    m = ev.get(2, [])
    by = {}
    for c, j, cd in m:
        by.setdefault((j, cd), c)
    gaps = {"waitP0_A": [], "P0toP1_A": [], "waitP0_B": [], "P0toP1_B": [], "pvA_to_sA": [],
            "sA_to_pvB": [], "pvA_to_KF": [], "issue_sA": [], "commit_sA": [], "Kload_to_KF": []}
    pe = {}
    for c, j, cd in ev.get(3, []):
        pe.setdefault((j, cd), c)
    for j in range(20, 300):
        try:
            gaps["waitP0_A"].append((by[(j, 40)] - by[(j, 30)]) & 0xFFFFFFFF)
            gaps["P0toP1_A"].append((by[(j, 50)] - by[(j, 40)]) & 0xFFFFFFFF)
            gaps["waitP0_B"].append((by[(j, 41)] - by[(j, 31)]) & 0xFFFFFFFF)
            gaps["P0toP1_B"].append((by[(j, 51)] - by[(j, 41)]) & 0xFFFFFFFF)
            gaps["pvA_to_sA"].append((by[(j + 1, 20)] - by[(j, 10)]) & 0xFFFFFFFF)
            gaps["sA_to_pvB"].append((by[(j, 11)] - by[(j + 1, 20)]) & 0xFFFFFFFF)
            gaps["pvA_to_KF"].append((by[(j + 1, 60)] - by[(j, 10)]) & 0xFFFFFFFF)
            gaps["issue_sA"].append((by[(j + 1, 61)] - by[(j + 1, 60)]) & 0xFFFFFFFF)
            gaps["commit_sA"].append((by[(j + 1, 20)] - by[(j + 1, 61)]) & 0xFFFFFFFF)
            gaps["Kload_to_KF"].append((by[(j + 1, 60)] - pe[(j + 1, 70)]) & 0xFFFFFFFF)
        except KeyError:
            pass
    r["mma"] = {k2: float(np.median(v2)) for k2, v2 in gaps.items() if v2}
    res[cta] = r
print(json.dumps(res, indent=1))
