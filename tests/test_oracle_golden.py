"""Pin the CPU oracle against golden vectors produced by the reference itself
(tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

import svdit_oracle as O
from conftest import GOLDEN, decode_spec, unpack_mask


def test_rng_and_random_qkv(golden_attn):
    q, k, v = O.random_qkv(7, 1, 2, 16, 8)
    np.testing.assert_array_equal(q, golden_attn["rng_q"])
    np.testing.assert_array_equal(k, golden_attn["rng_k"])
    np.testing.assert_array_equal(v, golden_attn["rng_v"])


def test_grids(golden_plan):
    for i, lay in enumerate(golden_plan["layouts"]):
        g = O.block_grid(*[int(x) for x in lay])
        np.testing.assert_array_equal(g.bounds, golden_plan[f"grid{i}_bounds"])
        np.testing.assert_array_equal(g.has_text, golden_plan[f"grid{i}_has_text"])
        np.testing.assert_array_equal(g.mixed, golden_plan[f"grid{i}_mixed"])
        np.testing.assert_array_equal(g.frame_index, golden_plan[f"grid{i}_frame_index"])
        assert O.frame_period(g) == int(golden_plan[f"grid{i}_frame_period"])


def test_masks(golden_plan):
    for i, lay in enumerate(golden_plan["layouts"]):
        g = O.block_grid(*[int(x) for x in lay])
        for j, (row, kind) in enumerate(zip(golden_plan[f"masks{i}_specs"], golden_plan[f"masks{i}_kinds"])):
            spec = decode_spec(row)
            if kind != "ok":
                with pytest.raises(O.OracleError) as ei:
                    O.build_mask(spec, g)
                assert ei.value.kind == kind
                continue
            m = O.build_mask(spec, g)
            np.testing.assert_array_equal(m, unpack_mask(golden_plan[f"mask{i}_{j}"], g.n_blocks))


def test_mask_errors(golden_plan):
    g = O.block_grid(0, 4, 64, 64)
    for row, kind in zip(golden_plan["errors_specs"], golden_plan["errors_kinds"]):
        with pytest.raises(O.OracleError) as ei:
            O.build_mask(decode_spec(row), g)
        assert ei.value.kind == kind


def test_grouping(golden_plan):
    ai = 0
    while f"asg{ai}_layout" in golden_plan:
        g = O.block_grid(*[int(x) for x in golden_plan[f"asg{ai}_layout"]])
        specs = [decode_spec(r) for r in golden_plan[f"asg{ai}_specs"]]
        groups = O.group_heads(specs, g)
        assert len(groups) == int(golden_plan[f"asg{ai}_ngroups"])
        for gi, (spec, heads, mask) in enumerate(groups):
            assert list(heads) == golden_plan[f"asg{ai}_g{gi}_heads"].tolist()
            key = f"asg{ai}_g{gi}_mask"
            if key in golden_plan:
                np.testing.assert_array_equal(mask, unpack_mask(golden_plan[key], g.n_blocks))
            else:
                assert mask is None
        ai += 1
    assert ai >= 5


def _c01_case(row):
    text, frames, tpf, block, b, h, d, seed, scale10, kind = (int(x) for x in row[:10])
    spec = decode_spec(row[10:])
    return text, frames, tpf, block, b, h, d, seed, scale10, kind, spec


def test_attention_c01_subset(golden_attn):
    """Acceptance c01 cases (test_acceptance.py:68-122): oracle == reference to 1e-6."""
    desc = golden_attn["c01_desc"]
    assert len(desc) == 100
    for case in range(30):
        text, frames, tpf, block, b, h, d, seed, scale10, kind, spec = _c01_case(desc[case])
        g = O.block_grid(text, frames, tpf, block)
        q, k, v = O.random_qkv(seed, b, h, g.n, d)
        if scale10:
            q = (q * 10.0).astype(np.float32)
        if kind == 0:
            got = O.full_mask_attention(q, k, v, g)
        else:
            got = O.sparse_attention(q, k, v, O.build_mask(spec, g), g.bounds)
        np.testing.assert_allclose(got, golden_attn[f"c01_{case}_out"], rtol=1e-6, atol=1e-7)


def test_attention_fused(golden_attn):
    fi = 0
    while f"fused{fi}_layout" in golden_attn:
        lay = [int(x) for x in golden_attn[f"fused{fi}_layout"]]
        H, d, seed = (int(x) for x in golden_attn[f"fused{fi}_meta"])
        qscale = float(golden_attn[f"fused{fi}_qscale"])
        g = O.block_grid(*lay)
        q, k, v = O.random_qkv(seed, 1, H, g.n, d)
        q = O.bf16_round(q * np.float32(qscale))
        k, v = O.bf16_round(k), O.bf16_round(v)
        specs = [decode_spec(r) for r in golden_attn[f"fused{fi}_specs"]]
        out = O.fused_layer_attention(q, k, v, O.group_heads(specs, g), g)
        # the reference runs FULL groups through dense_attention (fp32-rounded
        # scores/probabilities), the oracle through the streaming kernel: <=1e-6
        np.testing.assert_allclose(out, golden_attn[f"fused{fi}_out"], rtol=0, atol=2e-6)
        fi += 1
    assert fi == 3


def test_masked_dense_matches_streaming():
    g = O.block_grid(5, 3, 40, 16)
    q, k, v = O.random_qkv(3, 1, 2, g.n, 8)
    from types import SimpleNamespace as NS

    m = O.build_mask(NS(mode=O.DIAGONAL, halfwidth=1, period=None, md_halfwidth=0, stripe_count=2,
                        stripes=None, include_diagonal=True), g)
    a = O.sparse_attention(q, k, v, m, g.bounds)
    b = O.masked_dense_attention(q, k, v, O.token_mask(m, g))
    np.testing.assert_allclose(a, b, rtol=1e-5, atol=1e-6)


def test_bf16_round():
    x = np.array([1.0, 1.00390625, 1.005859375, -3.14159, 0.0], dtype=np.float32)
    import torch

    want = torch.from_numpy(x).to(torch.bfloat16).float().numpy()
    np.testing.assert_array_equal(O.bf16_round(x), want)


def test_block_key_mass(golden_attn):
    for bi in range(2):
        lay = [int(x) for x in golden_attn[f"bkm{bi}_layout"]]
        H, d, seed = (int(x) for x in golden_attn[f"bkm{bi}_meta"])
        g = O.block_grid(*lay)
        q, k, _ = O.random_qkv(seed, 1, H, g.n, d)
        q, k = O.bf16_round(q * np.float32(2.0)), O.bf16_round(k)
        got = O.block_key_mass(q, k, g)
        np.testing.assert_allclose(got, golden_attn[f"bkm{bi}_out"], rtol=1e-10, atol=1e-12)
        np.testing.assert_allclose(got.sum(axis=-1), 1.0, atol=1e-9)


# ---------------------------------------------------------------- the block around the operator (f4)
def _golden_layer():
    import hashlib

    g = np.load(GOLDEN / "golden_layer.npz")
    layers, heads, d, seed, li = (int(v) for v in g["meta"])
    w = O.zero_redundant_heads(O.layer_weights(seed, li, heads, d), g["redundant_heads"], d)
    for slot, arr in w.items():
        assert hashlib.sha256(np.ascontiguousarray(arr).tobytes()).digest() == g[f"sha_{slot}"].tobytes(), slot
    pq = {int(h): g[f"planted_q{h}"] for h in g["planted_heads"]}
    pk = {int(h): g[f"planted_k{h}"] for h in g["planted_heads"]}
    return g, w, heads, pq, pk


def test_oracle_layer_weights_match_reference_digests():
    _golden_layer()


def test_oracle_layer_qkv_matches_reference():
    g, w, heads, pq, pk = _golden_layer()
    q, k, v = O.layer_qkv(w, g["x"], heads, pq, pk)
    for name, got in (("q", q), ("k", k), ("v", v)):
        np.testing.assert_allclose(got, g[name], rtol=0, atol=1e-6, err_msg=name)


def test_oracle_layer_finish_matches_reference():
    g, w, *_ = _golden_layer()
    np.testing.assert_allclose(O.layer_finish(w, g["x"], g["attn"]), g["finish"], rtol=0, atol=1e-5)
    # layer_forward = layer_finish(layer_qkv -> fused attention)
    np.testing.assert_array_equal(g["finish"], g["forward"])


def test_attention_rows_equals_streaming_oracle():
    """oracle.attention_rows (one softmax over a block's active keys, used
    for the full-size GPU parity samples) equals the streaming recurrence of
    attention.py:57-98 (oracle.sparse_attention_rows) on text / frame-border /
    tail blocks of a text layout, for every mode, at q x1 and q x8."""
    og = O.block_grid(96, 8, 250, 64)
    specs = [O.full_spec(), O.diagonal_spec(1), O.multi_diagonal_spec(), O.vertical_stripe_spec(stripes=(3, 20))]
    for qscale in (1.0, 8.0):
        q, k, v = O.random_qkv(5, 1, 1, og.n, 32)
        q = q * np.float32(qscale)
        for spec in specs:
            active = O.build_mask(spec, og)
            qbs = [0, 1, 4, 11, og.n_blocks - 1]
            a = O.attention_rows(q, k, v, active, og.bounds, qbs)
            b = O.sparse_attention_rows(q, k, v, active, og.bounds, qbs)
            np.testing.assert_allclose(a, b, rtol=1e-5, atol=1e-6)
