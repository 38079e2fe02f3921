"""GPU calibration step vs the oracle: block_key_mass,
stripe selection, per-head MSE and the four-candidate loss / mode choice of
search.py:334-372."""

import numpy as np
import pytest

import paper_2506_03065_b200 as S
import svdit_oracle as O
from conftest import gpu_available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]


def _inputs(seed, h, n, d, qscale=2.0, b=1):
    q, k, v = O.random_qkv(seed, b, h, n, d)
    return O.bf16_round(q * np.float32(qscale)), O.bf16_round(k), O.bf16_round(v)


def test_block_key_mass_golden(golden_attn):
    for bi in range(2):
        lay = [int(x) for x in golden_attn[f"bkm{bi}_layout"]]
        H, d, seed = (int(x) for x in golden_attn[f"bkm{bi}_meta"])
        g = S.block_grid(S.TokenLayout(*lay))
        q, k, _ = O.random_qkv(seed, 1, H, g.layout.total_tokens, d)
        q, k = O.bf16_round(q * np.float32(2.0)), O.bf16_round(k)
        got = S.block_key_mass(q, k, g)
        want = golden_attn[f"bkm{bi}_out"]
        assert got.shape == want.shape
        # fp32 scores of the same bf16 inputs vs the reference's fp64: the
        # masses agree far inside bf16 resolution
        np.testing.assert_allclose(got, want, rtol=0, atol=2e-5)
        # rows normalise by the forward's l (a sum over the bf16-rounded P the
        # PV MMA consumes, 3/8 of the exps on the FMA pipe at d=128): each
        # head's total stays within 5e-5 of 1 (the two-pass kernel's l is fp32)
        np.testing.assert_allclose(got.sum(axis=-1), 1.0, atol=5e-5)


@pytest.mark.parametrize("lay,d", [((96, 16, 250, 64), 128), ((0, 16, 256, 64), 64)])
def test_block_key_mass_vs_oracle_and_topk(lay, d):
    og = O.block_grid(*lay)
    q, k, _ = _inputs(5, 3, og.n, d, 3.0)
    want = O.block_key_mass(q, k, og)
    got = S.block_key_mass(q, k, S.block_grid(S.TokenLayout(*lay)))
    np.testing.assert_allclose(got, want, rtol=0, atol=2e-5)
    from paper_2506_03065_b200.calibrate import top_stripes

    for h in range(3):
        a, b = top_stripes(got[0, h], 2), top_stripes(want[0, h], 2)
        order = np.sort(want[0, h])[::-1]
        if order[1] - order[2] > 1e-4:  # clear margin: selection must agree
            assert a == b


@pytest.mark.parametrize("lay,h,d,b", [
    ((0, 1, 40, 16), 2, 64, 1),       # N = 40 < one 64-row segment
    ((5, 3, 100, 48), 3, 128, 2),     # block 48 (not a multiple of 64), batch 2
    ((70, 4, 300, 100), 2, 32, 1),    # block 100 straddles 128-key tiles; d padded 32 -> 64
    ((0, 2, 128, 128), 2, 128, 1),    # N = 256: exact tiles, block 128
    ((13, 5, 211, 64), 1, 96, 1),     # ragged tail, d 96 -> 128
])
def test_block_key_mass_edges(lay, h, d, b):
    og = O.block_grid(*lay)
    q, k, _ = _inputs(7, h, og.n, d, 3.0, b)
    want = O.block_key_mass(q, k, og)
    got = S.block_key_mass(q, k, S.block_grid(S.TokenLayout(*lay)))
    assert got.shape == want.shape == (b, h, len(og.bounds) - 1)
    np.testing.assert_allclose(got, want, rtol=0, atol=2e-5)
    np.testing.assert_allclose(got.sum(axis=-1), 1.0, atol=1e-5)


def test_block_key_mass_strided_and_deterministic():
    """[B, N, H, d] storage runs without copies; repeated calls are bit-identical."""
    import torch

    lay = (96, 8, 250, 64)
    og = O.block_grid(*lay)
    g = S.block_grid(S.TokenLayout(*lay))
    q, k, _ = _inputs(3, 4, og.n, 128, 3.0)
    qs = torch.from_numpy(np.ascontiguousarray(q.transpose(0, 2, 1, 3))).cuda().bfloat16().permute(0, 2, 1, 3)
    ks = torch.from_numpy(np.ascontiguousarray(k.transpose(0, 2, 1, 3))).cuda().bfloat16().permute(0, 2, 1, 3)
    a = S.block_key_mass(qs, ks, g)
    b = S.block_key_mass(qs, ks, g)
    assert a.dtype == torch.float64 and a.is_cuda
    assert torch.equal(a, b)
    np.testing.assert_allclose(a.cpu().numpy(), O.block_key_mass(q, k, og), rtol=0, atol=2e-5)


def test_head_sqdiff_matches_fp64():
    import torch

    from paper_2506_03065_b200.calibrate import head_sqdiff

    rng = np.random.default_rng(0)
    a = O.bf16_round(rng.standard_normal((2, 3, 500, 64), dtype=np.float32))
    b = O.bf16_round(rng.standard_normal((2, 3, 500, 64), dtype=np.float32))
    ta, tb = (torch.from_numpy(x).cuda().to(torch.bfloat16) for x in (a, b))
    got = head_sqdiff(ta, tb).cpu().numpy()
    want = ((a.astype(np.float64) - b) ** 2).sum(axis=(0, 2, 3))
    np.testing.assert_allclose(got, want, rtol=1e-12)
    np.testing.assert_allclose(head_sqdiff(ta).cpu().numpy(), (a.astype(np.float64) ** 2).sum(axis=(0, 2, 3)),
                               rtol=1e-12)


def test_candidate_evaluator_vs_oracle():
    """Losses (MSE vs FULL + lam * density) within bf16 tolerance of the fp64
    oracle; choices agree wherever the winning margin is clear."""
    from paper_2506_03065_b200.calibrate import CandidateEvaluator

    lay = (96, 16, 250, 64)
    og = O.block_grid(*lay)
    g = S.block_grid(S.TokenLayout(*lay))
    H, d = 6, 64
    q, k, v = _inputs(11, H, og.n, d, 4.0)
    params = S.SearchParams(lam=0.05, epsilon=1.0)
    ev = CandidateEvaluator(g, params)
    res = ev.evaluate(q, k, v)
    # oracle: same stripes (from the GPU's selection) so the candidates coincide
    full = O.full_mask_attention(q, k, v, og)
    pp = params.patterns
    diag = O.sparse_attention(q, k, v, O.build_mask(pp.spec_for(S.Mode.DIAGONAL), og), og.bounds)
    md = O.sparse_attention(q, k, v, O.build_mask(pp.spec_for(S.Mode.MULTI_DIAGONAL), og), og.bounds)
    for h in range(H):
        spec = pp.spec_for(S.Mode.VERTICAL_STRIPE, res.stripes[h])
        st = O.sparse_attention(q[:, h:h + 1], k[:, h:h + 1], v[:, h:h + 1], O.build_mask(spec, og), og.bounds)
        cands = [np.zeros_like(full[:, h:h + 1]), diag[:, h:h + 1], md[:, h:h + 1], st]
        mses = [O.mse(c, full[:, h:h + 1]) for c in cands]
        losses = [S.search.penalized_loss(m, s, params.lam) for m, s in zip(mses, res.sparsities[h])]
        np.testing.assert_allclose(res.mse[h], mses, rtol=5e-2, atol=2e-6)
        np.testing.assert_allclose(res.losses[h], losses, rtol=5e-2, atol=2e-6)
        ranked = sorted(losses)
        if ranked[1] - ranked[0] > 0.1 * ranked[0] and min(losses) <= params.epsilon:
            assert res.choices[h] == S.select_mode(losses, res.sparsities[h], params.epsilon)
    # the selected output carries each head's chosen candidate
    sel = res.selected.float().cpu().numpy()
    for h, ch in enumerate(res.choices):
        if ch is S.Mode.SKIP:
            assert not sel[:, h].any()


def test_resolve_stripes_head_subset():
    """Stripe columns for a head subset equal the full-layer selection's
    (search.py:340-346 computes the mass of every head, then keeps the
    unresolved ones)."""
    from paper_2506_03065_b200.calibrate import CandidateEvaluator, top_stripes

    lay = (96, 16, 250, 64)
    og = O.block_grid(*lay)
    g = S.block_grid(S.TokenLayout(*lay))
    q, k, _ = _inputs(13, 5, og.n, 64, 3.0)
    ev = CandidateEvaluator(g, S.SearchParams())
    full = ev.resolve_stripes(q, k, range(5))
    sub = ev.resolve_stripes(q, k, [3, 1])
    assert sub == {3: full[3], 1: full[1]}
    want = O.block_key_mass(q, k, og)[0]
    for h in range(5):
        order = np.sort(want[h])[::-1]
        if order[1] - order[2] > 1e-4:
            assert full[h] == top_stripes(want[h], 2)
    assert ev.resolve_stripes(q, k, []) == {}


def test_candidate_evaluator_one_launch_path_matches_first_evaluation():
    """With the stripe columns frozen (every evaluation after a layer's first,
    search.py:338-346) the four candidates run as one 4H-head launch; its
    outputs (hence MSEs, losses, choices) equal the first evaluation's
    (FULL + diagonal + multi-diagonal launch, key-sum pass, stripe launch)
    bit for bit."""
    import torch

    from paper_2506_03065_b200.calibrate import CandidateEvaluator

    lay = (96, 16, 250, 64)
    og = O.block_grid(*lay)
    g = S.block_grid(S.TokenLayout(*lay))
    for d in (64, 128):
        q, k, v = _inputs(17, 5, og.n, d, 3.0)
        ev = CandidateEvaluator(g, S.SearchParams(lam=0.05, epsilon=1.0))
        first = ev.evaluate(q, k, v)
        again = ev.evaluate(q, k, v, stripes=first.stripes)
        # identical outputs; the fp64 MSE reduction (atomics) may reorder sums
        np.testing.assert_allclose(first.mse, again.mse, rtol=1e-12, atol=0)
        assert first.choices == again.choices
        assert torch.equal(first.selected, again.selected)


def test_key_mass_from_forward_row_stats():
    """The FULL launch's per-row (-m, 1/l) drive block_key_mass's key-sum pass:
    the masses equal the two-pass kernel's within 1e-6 and the oracle's
    within 2e-5 (attention.py:108-146), for d = 64 / 128 and a ragged tail."""
    import torch

    from paper_2506_03065_b200.calibrate import block_key_mass, block_key_mass_from_stats

    for lay, d in (((96, 16, 250, 64), 128), ((0, 7, 300, 64), 64), ((30, 5, 333, 48), 64)):
        og = O.block_grid(*lay)
        g = S.block_grid(S.TokenLayout(*lay))
        H = 3
        q, k, v = _inputs(19, H, og.n, d, 2.0)
        dq, dk, dv = (torch.from_numpy(x).cuda().to(torch.bfloat16) for x in (q, k, v))
        plan = S.plan_for_assignment([S.full_spec()] * H, g.layout)
        T = (og.n + 127) // 128
        stats = torch.empty(H, T, 2, 128, dtype=torch.float32, device="cuda")
        stats[:, :, 0].fill_(float("-inf"))
        stats[:, :, 1].zero_()
        out = torch.empty_like(dq)
        plan.forward(dq, dk, dv, out, head_dim=d, row_stats=stats, stats_heads=H)
        got = block_key_mass_from_stats(dq, dk, g, stats, head_dim=d).cpu().numpy()
        two_pass = block_key_mass(dq, dk, g).cpu().numpy()
        want = O.block_key_mass(q, k, og)
        np.testing.assert_allclose(got, two_pass, atol=5e-6)
        np.testing.assert_allclose(got, want, atol=2e-5)
        # rows normalise by the forward's l (a sum over the bf16-rounded P the
        # PV MMA consumes, 3/8 of the exps on the FMA pipe at d=128): each
        # head's total stays within 5e-5 of 1 (the two-pass kernel's l is fp32)
        np.testing.assert_allclose(got.sum(axis=-1), 1.0, atol=5e-5)


def test_input_head_map_reads_shared_qkv():
    """A plan whose heads are (copy, head) pairs over one q/k/v (in_head_map)
    gives, per copy, exactly the plain launch's output."""
    import torch

    lay = (96, 16, 250, 64)
    g = S.block_grid(S.TokenLayout(*lay))
    H, d = 3, 128
    gen = torch.Generator(device="cuda").manual_seed(5)
    q, k, v = (torch.randn(1, H, 4096, d, device="cuda", generator=gen).to(torch.bfloat16) for _ in range(3))
    specs = [S.full_spec(), S.diagonal_spec(1), S.vertical_stripe_spec(stripes=(2, 9))]
    ref = torch.empty_like(q)
    S.plan_for_assignment(specs, g.layout).forward(q, k, v, ref, head_dim=d)
    big = S.plan_for_assignment(specs + specs, g.layout)
    out = torch.empty(1, 2 * H, 4096, d, dtype=torch.bfloat16, device="cuda")
    in_map = torch.arange(H, dtype=torch.int32, device="cuda").repeat(2)
    big.forward(q, k, v, out, head_dim=d, in_head_map=in_map)
    assert torch.equal(out[:, :H], ref) and torch.equal(out[:, H:], ref)
