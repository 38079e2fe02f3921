"""Full-size output parity for every BASELINE GPU config (SURVEY §8d configs
2-4) with the bench's own mode mix (bench.assignment_for: FULL, SKIP,
diagonal, multi-diagonal and seeded stripe heads), at q x1 and the peaked
q x4 regime.  Each head's sampled query blocks cover the text / forced rows,
a frame-border (mixed) block, ordinary blocks and the partial tail; the
oracle rows are the fp64 softmax over each block's active keys
(oracle.attention_rows, attention.py:57-98 semantics; pinned to the
streaming oracle in test_oracle_golden).  SKIP heads must be exact zeros over
the whole head.  Tolerance (north_star): max-abs 2e-2, mean-abs 2e-3."""

import numpy as np
import pytest

import bench
import paper_2506_03065_b200 as S
import svdit_oracle as O
from conftest import gpu_available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]

MAX_ABS, MEAN_ABS = 2e-2, 2e-3


def _sample_blocks(og, rng, per_head=5):
    nb = og.n_blocks
    forced = np.flatnonzero(og.forced)
    mixed = np.flatnonzero(og.mixed & ~og.has_text)
    plain = np.flatnonzero(~og.forced[:-1])
    picks = {nb - 1}
    if len(forced):
        picks.add(int(forced[0]))
    if len(mixed):
        picks.add(int(rng.choice(mixed)))
    while len(picks) < per_head:
        picks.add(int(rng.choice(plain)))
    return sorted(int(b) for b in picks)


@pytest.mark.parametrize("qscale", [1.0, 4.0])
@pytest.mark.parametrize("config", ["hunyuan", "cogvideo", "wan"])
def test_baseline_config_full_size(config, qscale):
    import torch

    cfg = bench.CONFIGS[config]
    lay = cfg["layout"]
    og = O.block_grid(*lay)
    n, H, d = og.n, cfg["heads"], cfg["d"]
    specs = bench.assignment_for(cfg, S)
    ospecs = bench.assignment_for(cfg, O)
    gen = torch.Generator(device="cuda").manual_seed(11 + int(qscale))
    q = (torch.randn(1, H, n, d, device="cuda", generator=gen) * qscale).to(torch.bfloat16)
    k = torch.randn(1, H, n, d, device="cuda", generator=gen).to(torch.bfloat16)
    v = torch.randn(1, H, n, d, device="cuda", generator=gen).to(torch.bfloat16)
    out = S.fused_layer_attention(q, k, v, S.group_heads(specs, S.block_grid(S.TokenLayout(*lay))))
    torch.cuda.synchronize()
    rng = np.random.default_rng(hash((config, qscale)) % 2**32)
    worst, total, count = 0.0, 0.0, 0
    kinds = set()
    for h, spec in enumerate(ospecs):
        if int(spec.mode) == O.SKIP:
            assert out[:, h].abs().max().item() == 0.0, f"SKIP head {h} not exactly zero"
            kinds.add(O.SKIP)
            continue
        qbs = _sample_blocks(og, rng)
        sel = np.concatenate([np.arange(og.bounds[b], og.bounds[b + 1]) for b in qbs])
        idx = torch.as_tensor(sel, device="cuda")
        got = out[:, h:h + 1, idx].float().cpu().numpy()
        hq, hk, hv = (x[:, h:h + 1].float().cpu().numpy() for x in (q, k, v))
        want = O.attention_rows(hq, hk, hv, O.build_mask(spec, og), og.bounds, qbs)
        err = np.abs(got.astype(np.float64) - want)
        assert err.max() <= MAX_ABS, f"{config} q x{qscale} head {h} ({spec.mode}): max-abs {err.max():.3e}"
        worst = max(worst, float(err.max()))
        total += float(err.sum())
        count += err.size
        kinds.add(int(spec.mode))
    assert total / count <= MEAN_ABS, f"{config} q x{qscale}: mean-abs {total / count:.3e}"
    assert kinds == {O.FULL, O.SKIP, O.DIAGONAL, O.MULTI_DIAGONAL, O.VERTICAL_STRIPE}
    print(f"{config} q x{qscale}: max-abs {worst:.3e} mean-abs {total / count:.3e} over {count} values")
