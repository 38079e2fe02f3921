"""Reference-API behaviour that needs no GPU: argument checks raise the
reference's exception classes before any device work (attention.py:27-33,
:66-73, :157-161, :195-199), the strategy-table plugin surface, the cost
model, and the no-CPU-fallback guarantee."""

import json
from pathlib import Path

import numpy as np
import pytest

import paper_2506_03065_b200 as S
from paper_2506_03065_b200 import _native as nat


def qkv(b=1, h=2, n=64, d=8):
    rng = np.random.default_rng(0)
    return [rng.standard_normal((b, h, n, d)).astype(np.float32) for _ in range(3)]


def test_rank_and_shape_checks():
    q, k, v = qkv()
    g = S.block_grid(S.TokenLayout(0, 1, 64, 16))
    with pytest.raises(S.ShapeError):
        S.sparse_attention(q[0], k, v, S.build_mask(S.full_spec(), g))
    with pytest.raises(S.ShapeError):
        S.fused_layer_attention(q, k[:, :1], v, S.group_heads([S.full_spec()] * 2, g))
    with pytest.raises(S.ShapeError):
        S.sparse_attention(q, k, v, S.build_mask(S.full_spec(), S.block_grid(S.TokenLayout(0, 2, 64, 16))))


def test_skip_mask_and_empty_row_rejected():
    q, k, v = qkv()
    g = S.block_grid(S.TokenLayout(0, 1, 64, 16))
    with pytest.raises(S.DegenerateRowError):
        S.sparse_attention(q, k, v, S.build_mask(S.skip_spec(), g))
    active = np.zeros((4, 4), dtype=bool)
    active[0, 0] = True
    with pytest.raises(S.DegenerateRowError):
        S.sparse_attention(q, k, v, S.BlockMask(grid=g, active=active))


def test_groups_must_partition_heads():
    q, k, v = qkv(h=4, n=32)
    g = S.block_grid(S.TokenLayout(0, 2, 16, 16))
    with pytest.raises(S.ConfigError):
        S.fused_layer_attention(q, k, v, S.group_heads([S.full_spec()] * 3, g))
    with pytest.raises(S.ConfigError):
        S.HeadGroup(spec=S.full_spec(), heads=(0, 0), mask=None)
    with pytest.raises(S.ConfigError):
        S.HeadGroup(spec=S.full_spec(), heads=(), mask=None)


def test_no_cpu_fallback():
    """Valid arguments on a host without CUDA: the operator raises, it never
    computes on the CPU."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    q, k, v = qkv(h=1)
    g = S.block_grid(S.TokenLayout(0, 1, 64, 64))
    with pytest.raises(nat.NativeError):
        S.fused_layer_attention(q, k, v, S.group_heads([S.full_spec()], g))
    with pytest.raises(nat.NativeError):
        S.dense_attention(q, k, v)


def test_pattern_config_plugin_surface(tmp_path):
    modes = np.array([[[0, 1, 2, 3, 4]]], dtype=np.uint8)
    cfg = S.PatternConfig(modes=modes, stripes={(0, 4): (1, 3)})
    asg = cfg.assignment(0, 0)
    assert [int(s.mode) for s in asg] == [0, 1, 2, 3, 4]
    assert asg[4].stripes == (1, 3)
    path = tmp_path / "cfg.json"
    cfg.save(path)
    back = S.PatternConfig.load(path)
    assert back.to_json() == cfg.to_json()
    doc = json.loads(path.read_text())
    assert doc["dims"] == [1, 1, 5]
    layout = S.TokenLayout(0, 8, 64, 64)
    groups = S.group_heads(asg, S.block_grid(layout))
    assert len(groups) == 5
    s = S.config_sparsity(cfg, layout)
    assert 0 < s < 1


def test_mode_loss_and_select_mode():
    a = np.zeros((1, 1, 4, 2))
    b = np.ones((1, 1, 4, 2))
    assert S.mode_loss(a, b, 0.75, 0.5) == pytest.approx(1.0 + 0.5 * 0.25)
    assert S.mode_loss(a, b, 0.75, 0.5, "alg1_sparsity") == pytest.approx(1.0 + 0.5 * 0.75)
    assert S.select_mode([2, 2, 2, 2], [1, 0.5, 0.5, 0.5], 1.0) is S.Mode.FULL
    assert S.select_mode([0.1, 0.1, 0.2, 0.3], [1.0, 0.6, 0.5, 0.5], 1.0) is S.Mode.SKIP
    assert S.select_mode([0.3, 0.1, 0.1, 0.3], [1.0, 0.5, 0.6, 0.5], 1.0) is S.Mode.MULTI_DIAGONAL
    with pytest.raises(S.ConfigError):
        S.select_mode([1, 2, 3], [0, 0, 0], 1.0)


def test_cost_model_conventions():
    assert S.attention_flops(1024, 64, 1, 0.0) == 268_435_456
    short = S.attention_latency_share(45_106, 128, 24)
    long = S.attention_latency_share(119_056, 128, 24)
    assert 0 < short < long < 1
    assert round(short, 4) == 0.7099 and round(long, 4) == 0.8659
    m = S.B200LatencyModel(launch_ms=0.01, ms_per_tile={128: 1e-5})
    # per head: the whole-launch constant is left out of the ratio
    assert m.effective_sparsity(500, 1000, 128) == pytest.approx(0.5)
    # head dims the kernel runs zero-padded use the 64 / 128 fits
    m2 = S.B200LatencyModel(ms_per_tile={64: 1e-5, 128: 2e-5})
    assert m2.effective_sparsity(250, 1000, 32) == pytest.approx(0.75)
    assert m2.effective_sparsity(250, 1000, 96) == pytest.approx(0.75)


def test_layer_plan_flops_match_reference_convention():
    layout = S.TokenLayout(0, 16, 256, 64)
    asg = [S.full_spec(), S.diagonal_spec(1), S.skip_spec()]
    plan = S.plan_for_assignment(asg, layout)
    g = S.block_grid(layout)
    want = sum(S.attention_flops(4096, 64, 1, S.sparsity(s, g)) for s in asg if s.mode is not S.Mode.SKIP)
    assert plan.active_flops(64) == pytest.approx(want, rel=1e-12)


def test_host_pipeline_schedule_is_a_partition_and_beats_equal_chunks():
    """The host-buffer pipeline's head order is a permutation, its chunks
    partition it, and the modelled makespan is no worse than 6 equal chunks
    (attention._host_schedule; runs on CPU — plans need no GPU)."""
    from paper_2506_03065_b200 import attention as A

    layout = S.TokenLayout(256, 33, 3600, 64)
    asg = ([S.multi_diagonal_spec(), S.diagonal_spec(1)] * 3 + [S.full_spec()] * 2 + [S.skip_spec()]
           + [S.vertical_stripe_spec(stripes=(5, 900))] + [S.full_spec()] * 2)
    plan = S.plan_for_assignment(asg, layout)
    H, N, d = len(asg), layout.total_tokens, 128
    order, bounds = A._host_schedule(plan, 1, N, d)
    skip = asg.index(S.skip_spec())
    assert plan.skip_heads() == (skip,)
    # SKIP heads never cross PCIe: the order is a permutation of the other heads
    assert sorted(order) == [h for h in range(H) if h != skip]
    assert S.host_transfer_bytes(plan, 1, N, d) == (3 * (H - 1) * N * d * 2, (H - 1) * N * d * 2)
    assert bounds[0] == 0 and bounds[-1] == H - 1 and all(a < b for a, b in zip(bounds, bounds[1:]))
    work, longest = A._launch_model(plan, 1, d)
    sms = A._device_sm_count()
    h2d, d2h = 3 * N * d * 2 / A.PCIE_BYTES_PER_S, N * d * 2 / A.PCIE_BYTES_PER_S

    def makespan(o, bd):
        def kernel(a, b):
            return sum(work[h] for h in o[a:b]) / sms, max(longest[h] for h in o[a:b])
        return A._flow_shop(bd, h2d, kernel, d2h)

    rest = [h for h in range(H) if h != skip]
    equal = [round(i * len(rest) / 6) for i in range(7)]
    assert makespan(order, bounds) <= makespan(rest, equal) + 1e-9
    all_skip = S.plan_for_assignment([S.skip_spec()] * 3, layout)
    assert A._host_schedule(all_skip, 1, N, d) == ([], [0])
    # sub-plans of a head subset keep each head's schedule: same work as the full plan
    assert sum(plan.heads_subplan((h,)).info.computed_tiles for h in range(H)) == plan.info.computed_tiles


REF_SRC = Path("/root/reference/pkg/src")


@pytest.mark.skipif(not REF_SRC.exists(), reason="reference package not mounted (build container only)")
def test_drop_in_accepts_the_reference_objects():
    """A maintainer swapping the imports hands OUR functions the REFERENCE's
    own TokenLayout / BlockGrid / PatternSpec objects (model.py:405-420,
    search.py:142-143): grids, masks, sparsities and grouping come out equal."""
    import sys

    sys.path.insert(0, str(REF_SRC))
    from svdit import attention as RA
    from svdit import layout as RL
    from svdit import patterns as RP

    lay = RL.TokenLayout(96, 8, 250, 64)
    rgrid = RL.block_grid(lay)
    g = S.block_grid(lay)
    np.testing.assert_array_equal(g.bounds, rgrid.bounds)
    np.testing.assert_array_equal(g.forced, rgrid.forced)
    specs = [RP.full_spec(), RP.diagonal_spec(1), RP.skip_spec(), RP.multi_diagonal_spec(),
             RP.vertical_stripe_spec(stripes=(2, 20))]
    for grid in (g, rgrid):
        ours, ref = S.group_heads(specs, grid), RA.group_heads(specs, rgrid)
        assert [x.heads for x in ours] == [x.heads for x in ref]
        for a, b in zip(ours, ref):
            if b.mask is not None:
                np.testing.assert_array_equal(np.asarray(a.mask.active), b.mask.active)
    for sp in specs:
        assert S.sparsity(sp, g) == RP.sparsity(sp, rgrid)


@pytest.mark.skipif(not REF_SRC.exists(), reason="reference package not mounted (build container only)")
def test_reference_head_groups_lower_to_the_same_plan():
    """fused_layer_attention also takes HeadGroups built by the REFERENCE's
    group_heads (attention.py:164-183): they lower to a plan with the same
    grouping, masks and kernel work as our own group_heads gives."""
    import sys

    sys.path.insert(0, str(REF_SRC))
    from svdit import attention as RA
    from svdit import layout as RL
    from svdit import patterns as RP

    from paper_2506_03065_b200 import attention as A

    lay = RL.TokenLayout(20, 6, 300, 64)
    specs = [RP.full_spec(), RP.skip_spec(), RP.diagonal_spec(2), RP.vertical_stripe_spec(stripes=(3, 17)),
             RP.diagonal_spec(2), RP.multi_diagonal_spec()]
    ref_groups = RA.group_heads(specs, RL.block_grid(lay))
    plan = A._plan_for_groups(ref_groups, len(specs), lay.total_tokens)
    ours = S.plan_for_assignment(specs, S.TokenLayout(20, 6, 300, 64))
    assert plan.info.n_groups == ours.info.n_groups == len(ref_groups)
    assert plan.info.computed_tiles == ours.info.computed_tiles
    for g, rg in enumerate(ref_groups):
        assert plan.group_heads(g)[0] == rg.heads
        if rg.mask is not None:
            np.testing.assert_array_equal(plan.group_mask(g), rg.mask.active)


@pytest.mark.skipif(not REF_SRC.exists(), reason="reference package not mounted (build container only)")
def test_plugin_surface_matches_the_reference():
    """The search / cost-model plugin surface gives the reference's numbers on
    the same inputs: attention_flops, layer_linear_flops,
    attention_latency_share (costmodel.py:26-50), mode_loss, select_mode
    (search.py:65-103), sparsity_table, config_sparsity, aggregate_config
    (search.py:233-299) — for a random strategy table with stripe heads."""
    import sys

    sys.path.insert(0, str(REF_SRC))
    from svdit import costmodel as RC
    from svdit import layout as RL
    from svdit import patterns as RP
    from svdit import search as RS

    for n, d, h, sp in [(4096, 64, 8, 0.2), (119056, 128, 24, 0.72), (85906, 64, 48, 0.0)]:
        assert S.attention_flops(n, d, h, sp) == RC.attention_flops(n, d, h, sp)
        assert S.layer_linear_flops(n, d * h) == RC.layer_linear_flops(n, d * h)
        assert S.attention_latency_share(n, d, h) == RC.attention_latency_share(n, d, h)
    rng = np.random.default_rng(5)
    for _ in range(200):
        losses = rng.choice([0.1, 0.2, 0.2, 0.5], size=4)
        spars = rng.choice([0.0, 0.5, 0.9, 0.9], size=4)
        eps = float(rng.choice([0.05, 0.2, 1.0]))
        assert int(S.select_mode(losses, spars, eps)) == int(RS.select_mode(losses, spars, eps))
    a, b = rng.standard_normal((2, 3, 50, 8)).astype(np.float32)
    for pen in ("eq2_density", "alg1_sparsity"):
        assert S.mode_loss(a, b, 0.3, 0.5, pen) == pytest.approx(RS.mode_loss(a, b, 0.3, 0.5, pen), rel=1e-12)
    modes = rng.integers(0, 5, size=(4, 3, 5)).astype(np.uint8)
    stripes = {(l, hh): (1 + l, 7 + hh) for l in range(3) for hh in range(5)}
    lay_ours, lay_ref = S.TokenLayout(32, 6, 200, 64), RL.TokenLayout(32, 6, 200, 64)
    ours = S.PatternConfig(modes=modes, stripes=stripes)
    ref = RS.PatternConfig(modes=modes, stripes=stripes, params=RP.PatternParams())
    np.testing.assert_array_equal(S.sparsity_table(ours, lay_ours), RS.sparsity_table(ref, lay_ref))
    assert S.config_sparsity(ours, lay_ours) == RS.config_sparsity(ref, lay_ref)
    for strat in ("per_step", "majority_over_steps"):
        np.testing.assert_array_equal(S.aggregate_config(ours, lay_ours, strat).modes,
                                      RS.aggregate_config(ref, lay_ref, strat).modes)


def test_heads_subplan_copies_the_parent_schedule():
    """svd_plan_subset: a head subset (any order) carries exactly the work
    items and KV lists a fresh plan of those heads' specs builds; bad head
    lists and shard plans are rejected."""
    import numpy as np

    layout = S.TokenLayout(40, 6, 300, 64)
    asg = [S.full_spec(), S.diagonal_spec(1), S.skip_spec(), S.multi_diagonal_spec(),
           S.vertical_stripe_spec(stripes=(3, 20)), S.diagonal_spec(1)]
    plan = S.plan_for_assignment(asg, layout)
    for heads in [(4, 1), (0,), (5, 2, 3), (1, 5)]:
        sub = plan.heads_subplan(heads)
        fresh = S.LayerPlan.from_specs([asg[h] for h in heads], layout)
        (ia, ka), (ib, kb) = sub.schedule(), fresh.schedule()
        assert np.array_equal(ia, ib) and np.array_equal(ka, kb)
        assert sub.info.n_groups == fresh.info.n_groups
        assert sub.active_flops(64) == fresh.active_flops(64)
        for g in range(sub.info.n_groups):
            assert sub.group_heads(g) == fresh.group_heads(g)
    for bad in [(1, 1), (9,)]:
        with pytest.raises(S.ConfigError):
            plan.heads_subplan(bad)
    with pytest.raises(S.ConfigError):
        plan.shard(2, 0, n_sms=148).heads_subplan((0,))


@pytest.mark.parametrize("block", [64, 128, 32, 48])
def test_plan_schedule_matches_masks(block):
    """Every work item's KV tiles cover exactly the segments its rows need
    (active blocks of the group mask), for block sizes on and off the
    64-token segment grain (the fast block-aligned keyset path and the general one)."""
    import numpy as np

    layout = S.TokenLayout(70, 5, 333, block)
    asg = [S.diagonal_spec(1), S.multi_diagonal_spec(period=3), S.vertical_stripe_spec(stripes=(2, 7)),
           S.full_spec()]
    plan = S.plan_for_assignment(asg, layout)
    grid = S.block_grid(layout)
    n, nseg = layout.total_tokens, -(-layout.total_tokens // 64)
    items, kv = plan.schedule()
    n_all = 0
    for g in range(plan.info.n_groups):
        heads, skip = plan.group_heads(g)
        m = plan.group_mask(g) if int(asg[heads[0]].mode) != 0 else np.ones((grid.n_blocks,) * 2, bool)
        blk = np.minimum(np.arange(nseg * 64) // block, grid.n_blocks - 1)
        need = {}
        for s in range(nseg):
            rows = np.unique(blk[s * 64:min((s + 1) * 64, n)])
            cols = np.flatnonzero(m[rows].any(axis=0))
            segs = set()
            for c in cols:
                c0, c1 = grid.bounds[c], grid.bounds[c + 1]
                segs.update(range(c0 // 64, (c1 - 1) // 64 + 1))
            need[s] = segs
        for it in items[items[:, 0] == heads[0]]:
            got = set()
            for e in kv[it[2]:it[2] + it[3]]:
                got.update(x for x in e[:2] if x >= 0)
                if e[2] & (1 << 8):  # kFlagAll: the kernel applies no mask to this tile
                    n_all += 1
                    assert e[1] >= 0
                    for qs in (x for x in it[4:8] if x >= 0):
                        qb = np.unique(blk[qs * 64:min((qs + 1) * 64, n)])
                        kb = np.unique(blk[e[0] * 64:min(e[0] * 64 + 64, n)].tolist()
                                       + blk[e[1] * 64:min(e[1] * 64 + 64, n)].tolist())
                        assert m[np.ix_(qb, kb)].all()
            want = set().union(*(need[s] for s in it[4:8] if s >= 0))
            assert got == want
    assert n_all > 0  # the FULL head's interior tiles at least


def test_edited_groups_are_lowered_from_their_own_masks():
    """a group rebuilt with dataclasses.replace(g, mask=...) keeps
    g.plan; the fused call must lower the edited mask, not reuse the plan."""
    import dataclasses

    from paper_2506_03065_b200.attention import _mask_plan, _plan_for_groups

    grid = S.block_grid(S.TokenLayout(0, 8, 256, 64))
    groups = S.group_heads([S.diagonal_spec(1), S.full_spec()], grid)
    plan = groups[0].plan
    assert _plan_for_groups(groups, 2, grid.layout.total_tokens) is plan
    # masks handed out by group_heads are shared, so they are read-only
    assert not groups[0].mask.active.flags.writeable
    with pytest.raises(ValueError):
        groups[0].mask.active[0, -1] = True
    edited = dataclasses.replace(groups[0], mask=S.BlockMask(grid=grid, active=np.ones_like(groups[0].mask.active)))
    other = _plan_for_groups([edited, groups[1]], 2, grid.layout.total_tokens)
    assert other is not plan
    assert other.group_mask(0).all()
    # writable masks are keyed by content: an in-place edit gives a new plan
    m = S.build_mask(S.diagonal_spec(1), grid)
    p1 = _mask_plan(m, 1)
    assert _mask_plan(m, 1) is p1
    m.active[0, :] = True
    p2 = _mask_plan(m, 1)
    assert p2 is not p1 and p2.group_mask(0)[0].all()
