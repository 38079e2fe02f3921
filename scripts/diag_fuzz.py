"""Diagnose one randomised fuzz case: per-head error of the kernel vs the
fp64 oracle and vs a NumPy emulation of the kernel's numerics (fp32 scores,
exp2, bf16 P, fp32 sums)."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
for p in (ROOT, ROOT / "oracle", ROOT / "tests"):
    sys.path.insert(0, str(p))
import paper_2506_03065_b200 as S  # noqa: E402
import svdit_oracle as O  # noqa: E402
from test_gpu_fuzz import _random_case  # noqa: E402

seed_off, case_id = int(sys.argv[1]), int(sys.argv[2])
rng = np.random.default_rng(1234 + seed_off)
for c in range(case_id + 1):
    lay, specs, d, B, qs = _random_case(rng)
print(lay, d, B, qs, [int(s.mode) for s in specs])
og = O.block_grid(*lay)
groups = O.group_heads(specs, og)
q, k, v = O.random_qkv(50 + case_id, B, len(specs), og.n, d)
q, k, v = O.bf16_round(q * np.float32(qs)), O.bf16_round(k), O.bf16_round(v)
want = O.fused_layer_attention(q, k, v, groups, og)
layout = S.TokenLayout(*lay)
tq, tk, tv = (torch.from_numpy(x).cuda().to(torch.bfloat16) for x in (q, k, v))
if case_id % 2:
    tq, tk, tv = (t.transpose(1, 2).contiguous().transpose(1, 2) for t in (tq, tk, tv))
got = S.fused_layer_attention(tq, tk, tv, S.group_heads(specs, S.block_grid(layout))).float().cpu().numpy()


def emu(qh, kh, vh, tm):
    s = (qh.astype(np.float32) @ kh.astype(np.float32).T).astype(np.float32)
    s = np.where(tm, s * np.float32(np.log2(np.e) / np.sqrt(d)), -np.inf)
    p = np.exp2(s - s.max(1, keepdims=True)).astype(np.float32)
    pb = O.bf16_round(p)
    return O.bf16_round(((pb.astype(np.float64) @ vh) / p.astype(np.float64).sum(1, keepdims=True)).astype(np.float32))


for spec, heads, mask in groups:
    tm = None if int(spec.mode) == 1 else (np.ones((og.n, og.n), bool) if mask is None else O.token_mask(mask, og))
    for h in heads:
        for b in range(B):
            e = np.abs(got[b, h] - want[b, h])
            r, c = np.unravel_index(e.argmax(), e.shape)
            line = f"b{b} h{h} mode{int(spec.mode)} kernel-oracle max {e.max():.4f} @({r},{c}) mean {e.mean():.2e}"
            if tm is not None:
                em = emu(q[b, h], k[b, h], v[b, h], tm)
                ee = np.abs(em - want[b, h])
                line += f" | emu-oracle max {ee.max():.4f} mean {ee.mean():.2e} | kernel-emu max {np.abs(got[b,h]-em).max():.4f}"
                line += f" | row {r}: n_active {int(tm[r].sum())} got {got[b,h,r,c]:.4f} want {want[b,h,r,c]:.4f} emu {em[r,c]:.4f}"
            print(line)
