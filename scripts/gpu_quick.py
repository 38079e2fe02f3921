"""Quick GPU sanity run: tiny cases through the kernel with max-error prints
(used while bringing up the kernel; the real gates are tests/ -m gpu)."""

import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))

import paper_2506_03065_b200 as S  # noqa: E402
import svdit_oracle as O  # noqa: E402


def run(lay, specs, d, seed=0, qscale=1.0, B=1):
    og = O.block_grid(*lay)
    H = len(specs)
    q, k, v = O.random_qkv(seed, B, H, og.n, d)
    q, k, v = O.bf16_round(q * qscale), O.bf16_round(k), O.bf16_round(v)
    want = O.fused_layer_attention(q, k, v, O.group_heads(specs, og), og)
    g = S.block_grid(S.TokenLayout(*lay))
    dq, dk, dv = (torch.from_numpy(x).cuda().to(torch.bfloat16) for x in (q, k, v))
    t = time.time()
    out = S.fused_layer_attention(dq, dk, dv, S.group_heads(specs, g))
    torch.cuda.synchronize()
    got = out.float().cpu().numpy()
    err = np.abs(got - want)
    nan = np.isnan(got).sum()
    print(f"{lay} d={d} H={H} B={B}: max {np.nanmax(err):.3e} mean {np.nanmean(err):.3e} nan {nan} "
          f"({time.time() - t:.3f}s) |want| {np.abs(want).mean():.3e}", flush=True)
    if np.nanmax(err) > 2e-2 or nan:
        for h in range(H):
            e = err[:, h]
            print(f"   head {h} {specs[h].mode.name}: max {np.nanmax(e):.3e} rows>tol "
                  f"{np.unique(np.argwhere(e > 2e-2)[:, 1])[:20]}", flush=True)
    return err


if __name__ == "__main__":
    print(torch.cuda.get_device_name(), flush=True)
    run((0, 2, 128, 64), [S.full_spec()], 64)
    run((0, 2, 128, 64), [S.full_spec()], 128)
    run((0, 4, 128, 64), [S.full_spec(), S.diagonal_spec(1)], 64)
    run((0, 4, 128, 64), [S.full_spec(), S.diagonal_spec(1)], 128)
    run((0, 16, 256, 64), [S.full_spec(), S.diagonal_spec(1), S.multi_diagonal_spec(),
                           S.vertical_stripe_spec(stripes=(0, 7)), S.skip_spec()], 64, qscale=4.0)
    run((96, 16, 250, 64), [S.full_spec(), S.diagonal_spec(1), S.multi_diagonal_spec(),
                            S.vertical_stripe_spec(stripes=(0, 7)), S.skip_spec()], 128, qscale=4.0)
    run((3, 4, 96, 32), [S.full_spec(), S.diagonal_spec(1), S.multi_diagonal_spec(period=3)], 64, B=2)
