"""Time the search's per-layer candidate evaluation (calibrate.CandidateEvaluator,
search.py:334-372) at a production layout, device-resident q/k/v:
stripe calibration (block_key_mass) + FULL / diagonal / multi-diagonal /
stripe candidates + per-head MSE + mode selection.

    python scripts/time_evaluator.py [hunyuan|cogvideo|wan]"""
import json
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2506_03065_b200 as S  # noqa: E402
from paper_2506_03065_b200.calibrate import CandidateEvaluator, block_key_mass  # noqa: E402

CFG = {"hunyuan": ((256, 33, 3600, 64), 24, 128), "cogvideo": ((226, 21, 4080, 64), 48, 64),
       "wan": ((0, 21, 3600, 64), 40, 128)}


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "hunyuan"
    lay, H, d = CFG[name]
    grid = S.block_grid(S.TokenLayout(*lay))
    N = grid.layout.total_tokens
    g = torch.Generator(device="cuda").manual_seed(0)
    q, k, v = ((torch.randn(1, H, N, d, device="cuda", generator=g) * s).bfloat16() for s in (2, 1, 1))
    ev = CandidateEvaluator(grid, S.SearchParams())
    ev.evaluate(q, k, v)  # warm-up (plans, workspaces)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = ev.evaluate(q, k, v)
    torch.cuda.synchronize()
    total = (time.perf_counter() - t0) * 1e3
    t0 = time.perf_counter()
    block_key_mass(q, k, grid)
    torch.cuda.synchronize()
    km = (time.perf_counter() - t0) * 1e3
    counts = {}
    for c in res.choices:
        counts[c.name] = counts.get(c.name, 0) + 1
    print(json.dumps({"config": name, "N": N, "H": H, "d": d, "evaluate_ms": round(total, 1),
                      "block_key_mass_ms": round(km, 1), "candidates_and_mse_ms": round(total - km, 1),
                      "choices": counts}))


if __name__ == "__main__":
    main()
