"""BASELINE config 5: per-pattern latency sweep of the fused sm_100a kernel
over sparsity and 16k-128k tokens, and the fitted B200 latency model.

python scripts/costmodel_sweep.py [--out profiles/r1/costmodel_sweep.json]

Layouts keep HunyuanVideo's text/frame structure (256 text tokens, 3600
tokens per frame) and vary the frame count.  Each point: 8 heads of one
mode, kernel time by CUDA events (median of 5 after 2 warm-ups).  The fit
t(ms) = launch + tiles * ms_per_tile(d) uses the plan's issued 128x128 tile
count, which the kernel time is linear in; it is written to
paper_2506_03065_b200/data/b200_latency.json for B200LatencyModel.
"""

import argparse
import json
import statistics
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_2506_03065_b200 as S  # noqa: E402


def time_plan(plan, q, k, v, out, d, reps=5):
    for _ in range(2):
        plan.forward(q, k, v, out, head_dim=d)
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        plan.forward(q, k, v, out, head_dim=d)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=str(ROOT / "profiles" / "r1" / "costmodel_sweep.json"))
    ap.add_argument("--heads", type=int, default=8)
    args = ap.parse_args()
    H = args.heads
    frames_list = [4, 9, 18, 27, 35]  # 14.7k .. 126k tokens
    rng = np.random.default_rng(5)
    points = []
    for d in (128, 64):
        for frames in (frames_list if d == 128 else [9, 27]):
            layout = S.TokenLayout(256, frames, 3600, 64)
            n = layout.total_tokens
            nb = layout.n_blocks
            modes = {
                "full": [S.full_spec()] * H,
                "diag_hw0": [S.diagonal_spec(0)] * H,
                "diag_hw1": [S.diagonal_spec(1)] * H,
                "diag_hw2": [S.diagonal_spec(2)] * H,
                "mdiag_hw0": [S.multi_diagonal_spec()] * H,
                "mdiag_hw1": [S.multi_diagonal_spec(md_halfwidth=1)] * H,
                "stripe_1": [S.vertical_stripe_spec(1, tuple(rng.choice(nb, 1, replace=False)))
                             for _ in range(H)],
                "stripe_2": [S.vertical_stripe_spec(2, tuple(rng.choice(nb, 2, replace=False)))
                             for _ in range(H)],
                "stripe_8": [S.vertical_stripe_spec(8, tuple(rng.choice(nb, 8, replace=False)))
                             for _ in range(H)],
            }
            q, k, v = (torch.randn(1, H, n, d, device="cuda").to(torch.bfloat16) for _ in range(3))
            out = torch.empty_like(q)
            for name, asg in modes.items():
                plan = S.plan_for_assignment(asg, layout)
                info = plan.info
                ms = time_plan(plan, q, k, v, out, d)
                points.append({"mode": name, "d": d, "n_tokens": n, "heads": H, "ms": ms,
                               "computed_tiles": info.computed_tiles,
                               "density": plan.active_flops(d) / plan.dense_flops(d),
                               "active_tflops": plan.active_flops(d) / ms / 1e9})
                print(json.dumps(points[-1]), flush=True)
            del q, k, v, out
            torch.cuda.empty_cache()
    fit = {}
    for d in (128, 64):
        pts = [p for p in points if p["d"] == d]
        x = np.array([p["computed_tiles"] for p in pts], dtype=np.float64)
        y = np.array([p["ms"] for p in pts])
        A = np.stack([np.ones_like(x), x], 1)
        (a, b), *_ = np.linalg.lstsq(A, y, rcond=None)
        pred = A @ np.array([a, b])
        fit[d] = {"launch_ms": float(a), "ms_per_tile": float(b),
                  "max_rel_err": float(np.max(np.abs(pred - y) / y)), "points": len(pts)}
    model = S.B200LatencyModel(launch_ms=float(np.mean([fit[d]["launch_ms"] for d in fit])),
                               ms_per_tile={d: fit[d]["ms_per_tile"] for d in fit},
                               source="costmodel_sweep.py (BASELINE config 5), B200")
    data_dir = ROOT / "paper_2506_03065_b200" / "data"
    data_dir.mkdir(exist_ok=True)
    model.save(data_dir / "b200_latency.json")
    Path(args.out).parent.mkdir(parents=True, exist_ok=True)
    Path(args.out).write_text(json.dumps({"points": points, "fit": fit}, indent=1) + "\n")
    print(json.dumps({"fit": fit}))


if __name__ == "__main__":
    main()
