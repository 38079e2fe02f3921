"""Native plan builder (C++ behind the C ABI) vs the reference: grids, masks,
CSR tile lists and head grouping bit-exact; error classes identical; kernel
schedule covers exactly the active (query, key) segment pairs.  CPU only."""

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

import paper_2506_03065_b200 as S
import svdit_oracle as O
from conftest import decode_spec, unpack_mask

KINDS = {"config": S.ConfigError, "degenerate_mask": S.DegenerateMaskError,
         "degenerate_row": S.DegenerateRowError, "shape": S.ShapeError}


def test_grids_bit_exact(golden_plan):
    for i, lay in enumerate(golden_plan["layouts"]):
        g = S.block_grid(S.TokenLayout(*[int(x) for x in lay]))
        np.testing.assert_array_equal(g.bounds, golden_plan[f"grid{i}_bounds"])
        np.testing.assert_array_equal(g.has_text, golden_plan[f"grid{i}_has_text"])
        np.testing.assert_array_equal(g.mixed, golden_plan[f"grid{i}_mixed"])
        np.testing.assert_array_equal(g.frame_index, golden_plan[f"grid{i}_frame_index"])
        assert S.frame_period(g) == int(golden_plan[f"grid{i}_frame_period"])


def test_masks_bit_exact(golden_plan):
    for i, lay in enumerate(golden_plan["layouts"]):
        g = S.block_grid(S.TokenLayout(*[int(x) for x in lay]))
        for j, (row, kind) in enumerate(zip(golden_plan[f"masks{i}_specs"], golden_plan[f"masks{i}_kinds"])):
            spec = decode_spec(row)
            if kind != "ok":
                with pytest.raises(KINDS[kind]):
                    S.build_mask(spec, g)
                continue
            m = S.build_mask(spec, g)
            np.testing.assert_array_equal(m.active, unpack_mask(golden_plan[f"mask{i}_{j}"], g.n_blocks))
            assert m.sparsity == float(golden_plan[f"mask{i}_{j}_sparsity"])


def test_mask_error_classes(golden_plan):
    g = S.block_grid(S.TokenLayout(0, 4, 64, 64))
    for row, kind in zip(golden_plan["errors_specs"], golden_plan["errors_kinds"]):
        with pytest.raises(KINDS[kind]):
            S.build_mask(decode_spec(row), g)


def test_grouping_bit_exact(golden_plan):
    ai = 0
    while f"asg{ai}_layout" in golden_plan:
        g = S.block_grid(S.TokenLayout(*[int(x) for x in golden_plan[f"asg{ai}_layout"]]))
        specs = [decode_spec(r) for r in golden_plan[f"asg{ai}_specs"]]
        groups = S.group_heads(specs, g)
        assert len(groups) == int(golden_plan[f"asg{ai}_ngroups"])
        for gi, grp in enumerate(groups):
            assert list(grp.heads) == golden_plan[f"asg{ai}_g{gi}_heads"].tolist()
            key = f"asg{ai}_g{gi}_mask"
            if key in golden_plan:
                np.testing.assert_array_equal(grp.mask.active, unpack_mask(golden_plan[key], g.n_blocks))
            else:
                assert grp.mask is None
        ai += 1


def test_csr_tile_lists_match_active_key_blocks(golden_plan):
    g = S.block_grid(S.TokenLayout(256, 33, 3600, 64))
    specs = [S.diagonal_spec(1), S.multi_diagonal_spec(), S.vertical_stripe_spec(stripes=(3, 700))]
    plan = S.LayerPlan.from_specs(specs, g.layout)
    og = O.block_grid(256, 33, 3600, 64)
    for gi, spec in enumerate(specs):
        row_ptr, col_idx = plan.group_csr(gi)
        active = O.build_mask(spec, og)
        for qb in (0, 1, 2, 17, 55, 56, 57, 900, 1859, 1860):
            np.testing.assert_array_equal(col_idx[row_ptr[qb]:row_ptr[qb + 1]],
                                          O.active_key_blocks(active, qb))
        assert row_ptr[-1] == active.sum()


@pytest.mark.parametrize("tpf,block,want", [(70, 32, 2), (80, 32, 2), (96, 64, 2), (160, 64, 2),
                                            (224, 64, 4), (3600, 64, 56), (4080, 64, 64), (1, 64, 1)])
def test_frame_period_half_even(tpf, block, want):
    g = S.block_grid(S.TokenLayout(0, 2, tpf, block))
    assert S.frame_period(g) == want == O.frame_period(O.block_grid(0, 2, tpf, block))


def test_layout_validation():
    for bad in [(-1, 1, 1, 64), (0, -1, 1, 64), (0, 2, 0, 64), (0, 1, 4, 0), (0, 0, 0, 64)]:
        with pytest.raises(S.ConfigError):
            S.TokenLayout(*bad)


def test_spec_equality_drives_fusion():
    g = S.block_grid(S.TokenLayout(0, 8, 64, 64))
    groups = S.group_heads([S.vertical_stripe_spec(stripes=(1, 2)), S.vertical_stripe_spec(stripes=(2, 1, 2)),
                            S.vertical_stripe_spec(stripes=(1, 3))], g)
    assert [grp.heads for grp in groups] == [(0, 1), (2,)]


@settings(max_examples=60, deadline=None)
@given(text=st.integers(0, 150), frames=st.integers(0, 6), tpf=st.integers(1, 200),
       block=st.sampled_from([4, 8, 16, 24, 32, 48, 64, 128]),
       mode=st.sampled_from([0, 2, 3, 4]), hw=st.integers(0, 3), period=st.integers(0, 5),
       incl=st.booleans())
def test_random_layout_masks_match_oracle(text, frames, tpf, block, mode, hw, period, incl):
    if text + frames * tpf < 1:
        return
    layout = S.TokenLayout(text, frames, tpf, block)
    g = S.block_grid(layout)
    og = O.block_grid(text, frames, tpf, block)
    np.testing.assert_array_equal(g.bounds, og.bounds)
    np.testing.assert_array_equal(g.mixed, og.mixed)
    nb = g.n_blocks
    stripes = tuple(sorted({0, nb // 2, nb - 1})) if mode == 4 else None
    spec = S.PatternSpec(mode=S.Mode(mode), halfwidth=hw, period=period or None, md_halfwidth=min(hw, 1),
                         stripes=stripes, include_diagonal=incl)
    try:
        want = O.build_mask(spec, og)
    except O.OracleError as exc:
        with pytest.raises(KINDS[exc.kind]):
            S.build_mask(spec, g)
        return
    np.testing.assert_array_equal(S.build_mask(spec, g).active, want)


def _check_schedule(plan, layout, groups_masks):
    """Every active (query segment, key segment) pair of every head appears in
    exactly one KV tile of exactly one work item, with its activity bit set;
    and every KV bit that is set is a real active pair."""
    items, kv = plan.schedule()
    n = layout.total_tokens
    nseg = -(-n // 64)
    og = O.block_grid(layout.text_tokens, layout.frames, layout.tokens_per_frame, layout.block_size)
    bs = layout.block_size
    seen = {}
    for it in items:
        head, group, kb0, kc = it[:4]
        qsegs = it[4:8]
        for j in range(kc):
            ks0, ks1, flags, _ = kv[kb0 + j]
            for slot, qs in enumerate(qsegs):
                if qs < 0:
                    continue
                for kslot, ks in enumerate((ks0, ks1)):
                    if ks < 0:
                        continue
                    bit = (flags >> (2 * slot + kslot)) & 1
                    key = (head, qs, ks)
                    assert key not in seen, f"pair {key} scheduled twice"
                    seen[key] = bit
    for h, active in groups_masks.items():
        if active is None:
            continue
        seg_active = np.zeros((nseg, nseg), dtype=bool)
        for qs in range(nseg):
            r0, r1 = qs * 64, min(qs * 64 + 64, n)
            qbs = range(r0 // bs, (r1 - 1) // bs + 1)
            for ks in range(nseg):
                c0, c1 = ks * 64, min(ks * 64 + 64, n)
                kbs = range(c0 // bs, (c1 - 1) // bs + 1)
                seg_active[qs, ks] = active[np.ix_(list(qbs), list(kbs))].any()
        for qs in range(nseg):
            for ks in range(nseg):
                got = seen.get((h, qs, ks), 0)
                assert bool(got) == seg_active[qs, ks], (h, qs, ks)
    # every query segment of every head has exactly one item
    rows = {}
    for it in items:
        for qs in it[4:8]:
            if qs >= 0:
                rows[(it[0], qs)] = rows.get((it[0], qs), 0) + 1
    assert all(c == 1 for c in rows.values())
    assert len(rows) == plan.n_heads * nseg


@pytest.mark.parametrize("lay", [(0, 16, 256, 64), (96, 16, 250, 64), (3, 4, 96, 32), (11, 2, 64, 8),
                                 (5, 7, 45, 128), (40, 3, 150, 64)])
def test_schedule_covers_active_pairs(lay):
    layout = S.TokenLayout(*lay)
    g = S.block_grid(layout)
    nb = g.n_blocks
    specs = [S.full_spec(), S.diagonal_spec(1), S.multi_diagonal_spec(period=2),
             S.vertical_stripe_spec(stripes=(0, nb - 1)), S.skip_spec(), S.diagonal_spec(0)]
    plan = S.LayerPlan.from_specs(specs, layout)
    og = O.block_grid(*lay)
    masks = {h: O.build_mask(s, og) for h, s in enumerate(specs)}
    _check_schedule(plan, layout, masks)


def test_schedule_hunyuan_efficiency():
    """At the HunyuanVideo shape the schedule issues <= 2% more MMA work than
    the active 64x64 tiles (the 4-segment clustering keeps unions tight)."""
    layout = S.TokenLayout(256, 33, 3600, 64)
    asg = ([S.full_spec()] * 6 + [S.skip_spec()] + [S.diagonal_spec(1)] * 6 + [S.multi_diagonal_spec()] * 6
           + [S.vertical_stripe_spec(stripes=(5 + 37 * i, 900 + 101 * i)) for i in range(5)])
    plan = S.plan_for_assignment(asg, layout)
    info = plan.info
    computed_flops = info.computed_tiles * 4.0 * 128 * 128 * 128
    assert computed_flops / plan.active_flops(128) < 1.02
    assert abs(plan.dense_flops(128) / 1e12 - 174.174) < 0.01


@pytest.mark.parametrize("partition", ["items", "heads"])
def test_shards_partition_rows(partition):
    layout = S.TokenLayout(40, 3, 150, 64)
    plan = S.LayerPlan.from_specs([S.full_spec(), S.diagonal_spec(1), S.skip_spec()], layout)
    for world in (1, 2, 3, 8):
        owned = []
        for r in range(world):
            heads, toks = plan.shard(world, r, partition=partition).shard_rows()
            owned += [(int(h), int(t)) for h, t in zip(heads, toks) if h >= 0]
        assert sorted(owned) == [(h, t) for h in range(3) for t in range(layout.total_tokens)]


def test_head_partition_is_balanced_and_head_local():
    """SVD_PARTITION_HEADS (McNaughton over an interleaved head sequence): the
    ranks' head sets cover every head, at most world - 1 heads are shared
    (split by query range), every rank reads about H / world heads, and the
    issued tiles stay within a few percent of an even split (HunyuanVideo mix)."""
    layout = S.TokenLayout(256, 33, 3600, 64)
    asg = ([S.full_spec()] * 6 + [S.skip_spec()] + [S.diagonal_spec(1)] * 6 + [S.multi_diagonal_spec()] * 6
           + [S.vertical_stripe_spec(stripes=(5 + 37 * i, 900 + 101 * i)) for i in range(5)])
    plan = S.plan_for_assignment(asg, layout)
    for world in (2, 4, 8):
        shards = [plan.shard(world, r, n_sms=148, partition="heads") for r in range(world)]
        sets = [set(s.shard_heads()) for s in shards]
        assert set().union(*sets) == set(range(len(asg)))
        assert sum(len(x) for x in sets) - len(asg) <= world - 1  # only boundary heads are shared
        tiles = [s.info.computed_tiles for s in shards]
        assert max(tiles) <= 1.03 * sum(tiles) / world
        assert max(len(x) for x in sets) <= 2 * len(asg) // world + 2
        items_sets = [plan.shard(world, r, n_sms=148).shard_heads() for r in range(world)]
        assert max(len(x) for x in sets) < max(len(x) for x in items_sets)  # vs LPT over items
    with pytest.raises(S.ConfigError):
        plan.shard(2, 0, partition="rows")


@pytest.mark.parametrize("config", ["synthetic4k", "cogvideo", "hunyuan", "wan"])
def test_bench_assignment_same_in_both_arms(config):
    """bench.assignment_for built from the product's spec constructors (GPU
    arm) and from the oracle's (CPU arms) gives the same grouping and
    bit-identical masks, so both arms time the same layer."""
    import bench

    cfg = bench.CONFIGS[config]
    og = O.block_grid(*cfg["layout"])
    ours = S.group_heads(bench.assignment_for(cfg, S), S.block_grid(S.TokenLayout(*cfg["layout"])))
    ref = O.group_heads(bench.assignment_for(cfg, O), og)
    assert [g.heads for g in ours] == [heads for _, heads, _ in ref]
    for g, (spec, heads, mask) in zip(ours, ref):
        assert int(g.spec.mode) == int(spec.mode)
        if mask is None:
            assert g.mask is None
        else:
            np.testing.assert_array_equal(np.asarray(g.mask.active), mask)
