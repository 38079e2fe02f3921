"""Extended randomised parity fuzz (the generator of tests/test_gpu_fuzz.py,
many seeds): kernel vs the fp64 oracle, plus split-KV shard plans on a
subset.  Prints the worst errors and any failing case."""
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

n_seeds = int(sys.argv[1]) if len(sys.argv) > 1 else 10
worst, fails, done = (0.0, 0.0), [], 0
for seed in range(100, 100 + n_seeds):
    rng = np.random.default_rng(seed)
    for case in range(12):
        lay, specs, d, B, qs = _random_case(rng)
        og = O.block_grid(*lay)
        try:
            groups_o = O.group_heads(specs, og)
        except O.OracleError:
            continue
        q, k, v = O.random_qkv(seed * 100 + case, B, len(specs), og.n, d)
        q, k, v = O.bf16_round(q * np.float32(qs)), O.bf16_round(k), O.bf16_round(v)
        want = O.fused_layer_attention(q, k, v, groups_o, og)
        tq, tk, tv = (torch.from_numpy(x).cuda().to(torch.bfloat16) for x in (q, k, v))
        got = S.fused_layer_attention(tq, tk, tv, S.group_heads(specs, S.block_grid(S.TokenLayout(*lay))))
        got = got.float().cpu().numpy()
        err = np.abs(got.astype(np.float64) - want)
        worst = (max(worst[0], err.max()), max(worst[1], err.mean()))
        done += 1
        if not (err.max() <= 2e-2 and err.mean() <= 2e-3) or np.isnan(got).any():
            fails.append((seed, case, lay, d, B, qs, float(err.max()), float(err.mean())))
        if B == 1 and case % 3 == 0:  # split-KV shard plan, unpacked
            from paper_2506_03065_b200 import _native as nat

            plan = S.LayerPlan.from_specs(specs, S.TokenLayout(*lay))
            sh = plan.shard(1, 0, max_item_tiles=int(rng.integers(1, 6)))
            heads, toks = sh.shard_rows()
            D = 64 if d <= 64 else 128
            pq, pk, pv = (torch.nn.functional.pad(t, (0, D - d)) for t in (tq, tk, tv))
            packed = torch.zeros(max(len(heads), 1), D, dtype=torch.bfloat16, device="cuda")
            sh.forward(pq, pk, pv, packed, head_dim=d)
            out = torch.zeros(1, len(specs), og.n, D, dtype=torch.bfloat16, device="cuda")
            rh, rt = torch.from_numpy(heads).cuda(), torch.from_numpy(toks).cuda()
            nat.check(nat.lib().svd_unpack_rows(
                nat.c_void_p(rh.data_ptr()), nat.c_void_p(rt.data_ptr()), len(heads),
                nat.c_void_p(packed.data_ptr()), int(packed.stride(0)), nat.c_void_p(out.data_ptr()),
                nat.i64x4(out.stride()), D, nat.c_void_p(torch.cuda.current_stream().cuda_stream)))
            e2 = np.abs(out[..., :d].float().cpu().numpy() - want)
            if not (e2.max() <= 2e-2 and e2.mean() <= 2e-3):
                fails.append(("split", seed, case, lay, d, qs, float(e2.max()), float(e2.mean())))
print(f"cases {done}, worst max-abs {worst[0]:.4f}, worst mean-abs {worst[1]:.2e}, failures {len(fails)}")
for f in fails[:20]:
    print("FAIL", f)
