"""Absolute per-event timeline (cycles) of one traced CTA over a few KV
steps: softmax tile A / B events and the MMA issuer's events."""
import ctypes
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

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "hunyuan"]
j0 = int(sys.argv[2]) if len(sys.argv) > 2 else 100
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
names = {0: "top", 1: "S-ready", 3: "S-loaded", 4: "max-done", 6: "P0", 2: "P1",
         30: "wait-P", 40: "got-P", 50: "got-P1", 10: "PV-issued", 60: "K-ready", 61: "S-issued",
         20: "S-commit", 21: "S-commit", 70: "K-slot-free"}
ev = []
cta = 0
for st in range(4):
    for clk, w in buf[cta, st]:
        if clk == 0 and w == 0:
            continue
        j, code = int(w) >> 8, int(w) & 255
        if j0 <= j < j0 + 3:
            who = {0: "A", 1: "B", 2: "MMA", 3: "TMA"}[st]
            if st == 2 and code in (30, 40, 50, 10):
                who += "ab"[code % 10] if code % 10 < 2 else ""
            ev.append((int(clk), who, j, names.get(code - (code % 10) if st == 2 and code >= 10 and code not in (60, 61, 70) else code, str(code))))
ev.sort()
t0 = ev[0][0]
for clk, who, j, name in ev:
    print(f"{clk - t0:7d}  {who:5s} j={j:3d} {name}")
