"""Generate golden fixtures by running the REFERENCE (svdit 0.1.0) itself.

Run here (the reference is only mounted in the build container):
    python tests/golden/make_golden.py
Writes tests/golden/golden_plan.npz (grids, masks, grouping, error classes)
and tests/golden/golden_attn.npz (attention outputs on small cases, plus the
100 acceptance-c01 case descriptors drawn with the reference's own RNG).
Nothing at test time reads /root/reference: the tests load these files.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(REF))

from svdit import errors as E  # noqa: E402
from svdit.attention import (  # noqa: E402
    fused_layer_attention,
    full_mask_attention,
    group_heads,
    sparse_attention,
)
from svdit.layout import TokenLayout, block_grid  # noqa: E402
from svdit.numerics import make_rng  # noqa: E402
from svdit.patterns import (  # noqa: E402
    Mode,
    PatternSpec,
    build_mask,
    diagonal_spec,
    frame_period,
    full_spec,
    multi_diagonal_spec,
    skip_spec,
    vertical_stripe_spec,
)

LAYOUTS = [
    (0, 16, 256, 64), (96, 16, 250, 64), (226, 21, 4080, 64), (256, 33, 3600, 64),
    (0, 21, 3600, 64), (226, 11, 4080, 64), (2, 2, 3, 4), (10, 3, 50, 16), (30, 5, 100, 32),
    (0, 4, 70, 32), (8, 0, 0, 32), (3, 4, 96, 32), (0, 8, 3, 4), (64, 6, 64, 64),
    (0, 4, 128, 32), (0, 8, 64, 64), (0, 12, 64, 64), (7, 3, 11, 8), (40, 3, 150, 64),
    (20, 4, 60, 64), (0, 10, 64, 64), (5, 7, 45, 128), (100, 2, 30, 24),
]
BIG = {(226, 21, 4080, 64), (256, 33, 3600, 64), (0, 21, 3600, 64), (226, 11, 4080, 64)}


def random_qkv(seed, b, h, n, d):
    rng = make_rng(seed, 999)
    q = rng.standard_normal((b, h, n, d)).astype(np.float32)
    k = rng.standard_normal((b, h, n, d)).astype(np.float32)
    v = rng.standard_normal((b, h, n, d)).astype(np.float32)
    return q, k, v


def bf16_round(x):
    a = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    return ((a + 0x7FFF + ((a >> 16) & 1)) & 0xFFFF0000).astype(np.uint32).view(np.float32)


def spec_row(spec: PatternSpec):
    """Encode a spec as ints: mode, hw, period(-1), md_hw, count, incl, n_stripes(-1), stripes..."""
    stripes = [] if spec.stripes is None else list(spec.stripes)
    return [int(spec.mode), spec.halfwidth, -1 if spec.period is None else spec.period,
            spec.md_halfwidth, spec.stripe_count, int(spec.include_diagonal),
            -1 if spec.stripes is None else len(stripes)] + stripes


def specs_for(nb):
    out = [full_spec(), diagonal_spec(0), diagonal_spec(1), diagonal_spec(2), multi_diagonal_spec(),
           multi_diagonal_spec(period=4, md_halfwidth=1), multi_diagonal_spec(period=3),
           vertical_stripe_spec(stripes=(0, nb // 2)),
           vertical_stripe_spec(stripes=(nb - 1,), include_diagonal=False)]
    return out


def err_kind(exc):
    if isinstance(exc, E.DegenerateMaskError):
        return "degenerate_mask"
    if isinstance(exc, E.DegenerateRowError):
        return "degenerate_row"
    if isinstance(exc, E.ConfigError):
        return "config"
    if isinstance(exc, E.ShapeError):
        return "shape"
    return type(exc).__name__


def plan_fixtures():
    data = {}
    data["layouts"] = np.array(LAYOUTS, dtype=np.int64)
    for i, lay in enumerate(LAYOUTS):
        grid = block_grid(TokenLayout(*lay))
        data[f"grid{i}_bounds"] = grid.bounds
        data[f"grid{i}_has_text"] = grid.has_text
        data[f"grid{i}_mixed"] = grid.mixed
        data[f"grid{i}_frame_index"] = grid.frame_index
        data[f"grid{i}_frame_period"] = np.array(frame_period(grid))
        specs = specs_for(grid.n_blocks)
        if lay in BIG:
            specs = [diagonal_spec(1), multi_diagonal_spec(), vertical_stripe_spec(stripes=(3, 700))]
        rows, kinds = [], []
        for j, spec in enumerate(specs):
            rows.append(spec_row(spec))
            try:
                m = build_mask(spec, grid)
                kinds.append("ok")
                data[f"mask{i}_{j}"] = np.packbits(m.active.reshape(-1))
                data[f"mask{i}_{j}_sparsity"] = np.array(m.sparsity)
            except E.SvditError as exc:
                kinds.append(err_kind(exc))
        width = max(len(r) for r in rows)
        data[f"masks{i}_specs"] = np.array([r + [0] * (width - len(r)) for r in rows], dtype=np.int64)
        data[f"masks{i}_kinds"] = np.array(kinds)
    # error cases on a pure-video 4-block grid
    grid = block_grid(TokenLayout(0, 4, 64, 64))
    errs = [PatternSpec(mode=Mode.VERTICAL_STRIPE, stripes=(), include_diagonal=False),
            vertical_stripe_spec(stripes=None), vertical_stripe_spec(stripes=(99,)),
            vertical_stripe_spec(stripes=(1, -1))]
    rows, kinds = [], []
    for spec in errs:
        rows.append(spec_row(spec))
        try:
            build_mask(spec, grid)
            kinds.append("ok")
        except E.SvditError as exc:
            kinds.append(err_kind(exc))
    width = max(len(r) for r in rows)
    data["errors_specs"] = np.array([r + [0] * (width - len(r)) for r in rows], dtype=np.int64)
    data["errors_kinds"] = np.array(kinds)
    # grouping
    assignments = []
    g119 = block_grid(TokenLayout(256, 33, 3600, 64))
    hunyuan = ([full_spec()] * 6 + [skip_spec()] + [diagonal_spec(1)] * 6 +
               [multi_diagonal_spec()] * 6 +
               [vertical_stripe_spec(stripes=(5 + 37 * i, 900 + 101 * i)) for i in range(5)])
    order = make_rng(5).permutation(len(hunyuan))
    assignments.append(((256, 33, 3600, 64), [hunyuan[i] for i in order]))
    cfg1 = [full_spec(), diagonal_spec(1), multi_diagonal_spec(), vertical_stripe_spec(stripes=(0, 7)),
            skip_spec(), diagonal_spec(1), multi_diagonal_spec(), vertical_stripe_spec(stripes=(3, 40))]
    assignments.append(((0, 16, 256, 64), cfg1))
    assignments.append(((0, 1, 64, 16), [skip_spec(), diagonal_spec(1), skip_spec(), diagonal_spec(1)]))
    lay = (3, 4, 96, 32)
    grid = block_grid(TokenLayout(*lay))
    rng = make_rng(4242)
    for _ in range(6):
        a = []
        for _h in range(6):
            mode = Mode(int(rng.integers(5)))
            if mode is Mode.VERTICAL_STRIPE:
                a.append(vertical_stripe_spec(stripes=tuple(sorted(int(c) for c in rng.choice(
                    grid.n_blocks, size=2, replace=False)))))
            elif mode is Mode.FULL:
                a.append(full_spec())
            elif mode is Mode.SKIP:
                a.append(skip_spec())
            elif mode is Mode.DIAGONAL:
                a.append(diagonal_spec(int(rng.integers(0, 3))))
            else:
                a.append(multi_diagonal_spec(period=int(rng.integers(2, 4))))
        assignments.append((lay, a))
    # spec-equality corner: FULL with a non-default unused field is a separate group
    assignments.append(((0, 8, 64, 64), [full_spec(), PatternSpec(mode=Mode.FULL, halfwidth=3),
                                          full_spec(), multi_diagonal_spec(period=4),
                                          multi_diagonal_spec(period=None)]))
    for ai, (lay, a) in enumerate(assignments):
        grid = block_grid(TokenLayout(*lay))
        groups = group_heads(a, grid)
        rows = [spec_row(s) for s in a]
        width = max(len(r) for r in rows)
        data[f"asg{ai}_layout"] = np.array(lay, dtype=np.int64)
        data[f"asg{ai}_specs"] = np.array([r + [0] * (width - len(r)) for r in rows], dtype=np.int64)
        data[f"asg{ai}_ngroups"] = np.array(len(groups))
        for gi, g in enumerate(groups):
            data[f"asg{ai}_g{gi}_heads"] = np.array(g.heads, dtype=np.int64)
            if g.mask is not None:
                data[f"asg{ai}_g{gi}_mask"] = np.packbits(g.mask.active.reshape(-1))
    np.savez_compressed(OUT / "golden_plan.npz", **data)


def attn_fixtures():
    data = {}
    # RNG pin
    q, k, v = random_qkv(7, 1, 2, 16, 8)
    data["rng_q"], data["rng_k"], data["rng_v"] = q, k, v
    # acceptance c01 descriptors (test_acceptance.py:68-122), reference RNG draws
    geometries = [(8, 8, 4), (8, 12, 3), (8, 20, 4), (8, 16, 2), (16, 16, 4), (16, 24, 3),
                  (16, 40, 2), (16, 32, 4), (64, 64, 2), (64, 96, 2), (64, 64, 3), (64, 128, 1)]
    rng = make_rng(20260813)
    desc = []
    for case in range(100):
        block, tpf, frames = geometries[rng.integers(len(geometries))]
        text = int(rng.choice([0, 0, 3, 11]))
        layout = TokenLayout(text_tokens=text, frames=frames, tokens_per_frame=tpf, block_size=block)
        grid = block_grid(layout)
        nb = grid.n_blocks
        b = int(rng.integers(1, 3))
        h = int(rng.integers(1, 4))
        d = int(rng.choice([4, 8, 17, 32]))
        seed = int(rng.integers(1 << 30))
        scale10 = bool(rng.random() < 0.25)
        kind = int(rng.integers(4))
        spec = full_spec()
        if kind == 1:
            spec = diagonal_spec(int(rng.integers(0, 3)))
        elif kind == 2:
            period = int(rng.integers(2, 5))
            spec = multi_diagonal_spec(period=period, md_halfwidth=int(rng.integers(0, min(2, period))))
        elif kind == 3:
            count = int(rng.integers(1, min(3, nb) + 1))
            cols = tuple(sorted(int(c) for c in rng.choice(nb, size=count, replace=False)))
            spec = vertical_stripe_spec(stripes=cols, include_diagonal=bool(rng.integers(2)))
        row = [text, frames, tpf, block, b, h, d, seed, int(scale10), kind] + spec_row(spec)
        desc.append(row)
        if case < 30:
            q, k, v = random_qkv(seed, b, h, layout.total_tokens, d)
            if scale10:
                q = (q * 10.0).astype(np.float32)
            if kind == 0:
                got = full_mask_attention(q, k, v, grid)
            else:
                got = sparse_attention(q, k, v, build_mask(spec, grid))
            data[f"c01_{case}_out"] = got
    width = max(len(r) for r in desc)
    data["c01_desc"] = np.array([r + [0] * (width - len(r)) for r in desc], dtype=np.int64)
    # fused layer cases (bf16-rounded inputs, as the GPU sees them)
    fused = [
        ((20, 4, 60, 64), 8, 64, 11, 1.0,
         [full_spec(), diagonal_spec(1), multi_diagonal_spec(), vertical_stripe_spec(stripes=(0, 2)),
          skip_spec(), diagonal_spec(1), multi_diagonal_spec(), vertical_stripe_spec(stripes=(1, 3))]),
        ((40, 3, 150, 64), 4, 128, 12, 4.0,
         [diagonal_spec(1), multi_diagonal_spec(period=2), vertical_stripe_spec(stripes=(0, 3)),
          full_spec()]),
        ((3, 4, 96, 32), 6, 8, 13, 1.0,
         [skip_spec(), diagonal_spec(2), full_spec(), multi_diagonal_spec(period=3),
          vertical_stripe_spec(stripes=(1, 9)), diagonal_spec(2)]),
    ]
    for fi, (lay, H, d, seed, qscale, a) in enumerate(fused):
        layout = TokenLayout(*lay)
        grid = block_grid(layout)
        q, k, v = random_qkv(seed, 1, H, layout.total_tokens, d)
        q = bf16_round(q * np.float32(qscale))
        k, v = bf16_round(k), bf16_round(v)
        out = fused_layer_attention(q, k, v, group_heads(a, grid))
        rows = [spec_row(s) for s in a]
        width = max(len(r) for r in rows)
        data[f"fused{fi}_layout"] = np.array(lay, dtype=np.int64)
        data[f"fused{fi}_meta"] = np.array([H, d, seed], dtype=np.int64)
        data[f"fused{fi}_qscale"] = np.array(qscale)
        data[f"fused{fi}_specs"] = np.array([r + [0] * (width - len(r)) for r in rows], dtype=np.int64)
        data[f"fused{fi}_out"] = out
    # block_key_mass (attention.py:108-146) — the stripe calibration input
    from svdit.attention import block_key_mass

    for bi, (lay, H, d, seed) in enumerate([((3, 4, 96, 32), 2, 16, 21), ((40, 3, 150, 64), 3, 32, 22)]):
        layout = TokenLayout(*lay)
        q, k, _ = random_qkv(seed, 1, H, layout.total_tokens, d)
        q, k = bf16_round(q * np.float32(2.0)), bf16_round(k)
        data[f"bkm{bi}_layout"] = np.array(lay, dtype=np.int64)
        data[f"bkm{bi}_meta"] = np.array([H, d, seed], dtype=np.int64)
        data[f"bkm{bi}_out"] = block_key_mass(q, k, block_grid(layout))
    np.savez_compressed(OUT / "golden_attn.npz", **data)


def layer_fixtures():
    """A planted 2-layer toy model (model.py:307-349): layer 1's layer_qkv,
    the fused attention under a per-head assignment, layer_finish and
    layer_forward (model.py:372-420), all from the reference.  Weights are
    not stored (tests redraw them with the oracle and check these digests)."""
    import hashlib

    from svdit import model as M

    layout = TokenLayout(64, 2, 128, 64)
    plant = {(1, 0): M.PlantDirective("diagonal"), (1, 1): M.PlantDirective("vertical_stripe", 2),
             (1, 2): M.PlantDirective("redundant"), (1, 3): M.PlantDirective("uniform")}
    spec = M.ModelSpec(layers=2, heads=4, head_dim=32, layout=layout, timesteps=2, seed=11, plant=plant)
    model = M.build_model(spec)
    lw = model.layers[1]
    x = make_rng(5, 77).standard_normal((1, layout.total_tokens, spec.hidden_dim)).astype(np.float32)
    q, k, v = M.layer_qkv(model, 1, x)
    stripes = model.planted_stripes[(1, 1)]
    assignment = [diagonal_spec(1), vertical_stripe_spec(stripes=stripes), skip_spec(), full_spec()]
    attn = fused_layer_attention(q, k, v, group_heads(assignment, model.grid))
    data = {
        "layout": np.array([64, 2, 128, 64], dtype=np.int64),
        "meta": np.array([2, 4, 32, 11, 1], dtype=np.int64),  # layers, heads, head_dim, seed, layer
        "stripes": np.array(stripes, dtype=np.int64),
        "x": x, "q": q, "k": k, "v": v, "attn": attn,
        "finish": M.layer_finish(model, 1, x, attn),
        "forward": M.layer_forward(model, 1, x, assignment),
        "planted_heads": np.array(sorted(lw.planted_q), dtype=np.int64),
        "redundant_heads": np.array([2], dtype=np.int64),
    }
    for h in sorted(lw.planted_q):
        data[f"planted_q{h}"] = lw.planted_q[h]
        data[f"planted_k{h}"] = lw.planted_k[h]
    for slot in ("wq", "wk", "wv", "wo", "w1", "w2"):
        digest = hashlib.sha256(np.ascontiguousarray(getattr(lw, slot)).tobytes()).hexdigest()
        data[f"sha_{slot}"] = np.frombuffer(bytes.fromhex(digest), dtype=np.uint8)
    np.savez_compressed(OUT / "golden_layer.npz", **data)


if __name__ == "__main__":
    plan_fixtures()
    attn_fixtures()
    layer_fixtures()
    for f in ("golden_plan.npz", "golden_attn.npz", "golden_layer.npz"):
        print(f, (OUT / f).stat().st_size, "bytes")
