"""SVD_HP_TRACE build of the half-row pair kernel: per-step phase durations
(cycles) of one warp per key half and of the MMA issuer, all-FULL layer."""
import ctypes
import os
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
os.environ.setdefault("SVD_LIB", str(ROOT / "paper_2506_03065_b200/variants/hptrace.so"))
os.environ["SVD_HP"] = "1"
sys.path.insert(0, str(ROOT))
import paper_2506_03065_b200 as S  # noqa: E402
from paper_2506_03065_b200 import _native as nat  # noqa: E402

H, n, d = 8, 32768, 128
lay = S.TokenLayout(0, 1, n, 64)
plan = S.plan_for_assignment([S.full_spec()] * H, lay)
q, k, v = (torch.randn(1, H, n, d, device="cuda").to(torch.bfloat16) for _ in range(3))
o = torch.empty_like(q)
lib = nat.lib()
lib.svd_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32]
plan.forward(q, k, v, o, head_dim=d)
buf = np.zeros((4, 3, 4096, 2), dtype=np.uint32)
nat.check(lib.svd_debug_trace(None, 0, 1))
plan.forward(q, k, v, o, head_dim=d)
nat.check(lib.svd_debug_trace(buf.ctypes.data, buf.nbytes, 0))
for cta in range(2):
    ev = {}
    for st in range(3):
        for clk, w in buf[cta, st]:
            if clk == 0 and w == 0:
                continue
            ev.setdefault(st, {})[(int(w) >> 8, int(w) & 255)] = int(clk)
    def med(st, a, b, js=range(20, 200)):
        x = [(ev[st][(j, b)] - ev[st][(j, a)]) & 0xFFFFFFFF for j in js if (j, a) in ev.get(st, {}) and (j, b) in ev.get(st, {})]
        return float(np.median(x)) if x else None
    def period(st, code):
        x = [(ev[st][(j + 1, code)] - ev[st][(j, code)]) & 0xFFFFFFFF for j in range(20, 200)
             if (j, code) in ev.get(st, {}) and (j + 1, code) in ev.get(st, {})]
        return float(np.median(x)) if x else None
    out = {"cta": cta}
    for h in (0, 1):
        out[f"half{h}"] = {"period": period(h, 0), "wait_S": med(h, 0, 1), "load": med(h, 1, 2),
                           "max_vote": med(h, 2, 3), "exps_store": med(h, 3, 4), "handoff": med(h, 4, 5)}
    if 2 in ev:
        out["issuer"] = {"period": period(2, 10), "wait_V": med(2, 10, 11), "V_to_P0": med(2, 11, 12),
                         "P0_to_P1": med(2, 12, 13), "P1_to_S": med(2, 13, 14), "issue_S": med(2, 14, 15)}
    print(out)
