"""sm_100a kernel vs the CPU oracle (which is pinned to the reference by the
golden fixtures).  Tolerance (north_star): bf16 outputs within max-abs 2e-2
and mean-abs 2e-3 of the fp32/fp64 reference on the same (bf16-rounded)
inputs; SKIP heads exactly zero; masks/grouping bit-exact (test_plan_parity).
"""

import numpy as np
import pytest

import paper_2506_03065_b200 as S
import svdit_oracle as O
from conftest import decode_spec, gpu_available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]

MAX_ABS, MEAN_ABS = 2e-2, 2e-3


def _dev(x):
    import torch

    return torch.from_numpy(np.ascontiguousarray(x)).cuda().to(torch.bfloat16)


def _inputs(seed, b, h, n, d, qscale=1.0):
    q, k, v = O.random_qkv(seed, b, h, n, d)
    return O.bf16_round(q * np.float32(qscale)), O.bf16_round(k), O.bf16_round(v)


def _close(got, want, what=""):
    err = np.abs(got.astype(np.float64) - want.astype(np.float64))
    assert err.max() <= MAX_ABS, f"{what}: max-abs {err.max():.3e}"
    assert err.mean() <= MEAN_ABS, f"{what}: mean-abs {err.mean():.3e}"
    return err.max(), err.mean()


def _oracle_fused(lay, specs, q, k, v):
    og = O.block_grid(*lay)
    return O.fused_layer_attention(q, k, v, O.group_heads(specs, og), og)


def _gpu_fused(lay, specs, q, k, v):
    g = S.block_grid(S.TokenLayout(*lay))
    out = S.fused_layer_attention(_dev(q), _dev(k), _dev(v), S.group_heads(specs, g))
    return out.float().cpu().numpy()


def test_fused_golden(golden_attn):
    """Reference outputs (golden) through the numpy-in / numpy-out API."""
    for fi in range(3):
        lay = [int(x) for x in golden_attn[f"fused{fi}_layout"]]
        H, d, seed = (int(x) for x in golden_attn[f"fused{fi}_meta"])
        q, k, v = _inputs(seed, 1, H, sum([lay[0], lay[1] * lay[2]]), d,
                          float(golden_attn[f"fused{fi}_qscale"]))
        specs = [decode_spec(r) for r in golden_attn[f"fused{fi}_specs"]]
        g = S.block_grid(S.TokenLayout(*lay))
        got = S.fused_layer_attention(q, k, v, S.group_heads(specs, g))
        assert isinstance(got, np.ndarray) and got.dtype == np.float32
        want = golden_attn[f"fused{fi}_out"]
        _close(got, want, f"fused{fi}")
        for h, spec in enumerate(specs):
            if spec.mode is S.Mode.SKIP:
                assert not got[:, h].any()


def test_acceptance_c01_100_cases(golden_attn):
    """The reference's 100 randomized kernel cases (test_acceptance.py:68-122):
    block sizes 8/16/64, text 0/3/11, d 4/8/17/32 (zero-padded to 64), 25% q*10."""
    desc = golden_attn["c01_desc"]
    worst = 0.0
    for row in desc:
        text, frames, tpf, block, b, h, d, seed, scale10, kind = (int(x) for x in row[:10])
        spec = decode_spec(row[10:])
        og = O.block_grid(text, frames, tpf, block)
        q, k, v = _inputs(seed, b, h, og.n, d, 10.0 if scale10 else 1.0)
        grid = S.block_grid(S.TokenLayout(text, frames, tpf, block))
        if kind == 0:
            want = O.full_mask_attention(q, k, v, og)
            got = S.full_mask_attention(_dev(q), _dev(k), _dev(v), grid)
        else:
            mask = O.build_mask(spec, og)
            want = O.sparse_attention(q, k, v, mask, og.bounds)
            got = S.sparse_attention(_dev(q), _dev(k), _dev(v), S.build_mask(spec, grid))
        mx, _ = _close(got.float().cpu().numpy(), want, f"c01 {row[:10].tolist()}")
        worst = max(worst, mx)
    print(f"c01 worst max-abs {worst:.3e}")


@pytest.mark.parametrize("qscale", [1.0, 4.0])
def test_config1_synthetic_4k(qscale):
    """BASELINE config 1: TokenLayout(0,16,256,64), 8 heads x d64, table
    [F, D, MD, VS(a), S, D, MD, VS(b)]."""
    lay = (0, 16, 256, 64)
    specs = [S.full_spec(), S.diagonal_spec(1), S.multi_diagonal_spec(), S.vertical_stripe_spec(stripes=(0, 7)),
             S.skip_spec(), S.diagonal_spec(1), S.multi_diagonal_spec(), S.vertical_stripe_spec(stripes=(3, 40))]
    q, k, v = _inputs(0, 1, 8, 4096, 64, qscale)
    got = _gpu_fused(lay, specs, q, k, v)
    want = _oracle_fused(lay, specs, q, k, v)
    _close(got, want, "config1")
    assert not got[:, 4].any()


def test_text_variant_d128():
    """Forced text / mixed blocks and a partial trailing block at d=128."""
    lay = (96, 16, 250, 64)  # 4096 tokens, 17 forced blocks
    specs = [S.diagonal_spec(1), S.multi_diagonal_spec(), S.vertical_stripe_spec(stripes=(5, 33)),
             S.full_spec()]
    q, k, v = _inputs(1, 1, 4, 4096, 128, 4.0)
    got = _gpu_fused(lay, specs, q, k, v)
    want = _oracle_fused(lay, specs, q, k, v)
    _close(got, want, "text-d128")


def test_partial_tail_and_small_blocks():
    for lay, d in [((40, 3, 150, 64), 64), ((7, 9, 45, 32), 128), ((5, 7, 45, 128), 64), ((3, 5, 77, 24), 64)]:
        og = O.block_grid(*lay)
        nb = og.n_blocks
        specs = [S.diagonal_spec(1), S.multi_diagonal_spec(period=3, md_halfwidth=1),
                 S.vertical_stripe_spec(stripes=(0, nb - 1)), S.full_spec(), S.skip_spec()]
        q, k, v = _inputs(2, 1, 5, og.n, d, 4.0)
        _close(_gpu_fused(lay, specs, q, k, v), _oracle_fused(lay, specs, q, k, v), str(lay))


def test_batch_and_strided_views():
    """B=2, and q/k/v given as [B,N,H,d] storage viewed as [B,H,N,d] (no copies)."""
    import torch

    lay = (20, 4, 250, 64)
    og = O.block_grid(*lay)
    specs = [S.diagonal_spec(1), S.full_spec(), S.multi_diagonal_spec(period=2)]
    q, k, v = _inputs(3, 2, 3, og.n, 128)
    want = _oracle_fused(lay, specs, q, k, v)
    g = S.block_grid(S.TokenLayout(*lay))
    qs, ks, vs = (_dev(np.ascontiguousarray(x.transpose(0, 2, 1, 3))).transpose(1, 2) for x in (q, k, v))
    assert qs.stride(-1) == 1 and not qs.is_contiguous()
    got = S.fused_layer_attention(qs, ks, vs, S.group_heads(specs, g)).float().cpu().numpy()
    _close(got, want, "strided-B2")


def test_dense_and_skip_api():
    q, k, v = _inputs(4, 1, 2, 700, 64)
    og = O.block_grid(0, 1, 700, 64)
    got = S.dense_attention(_dev(q), _dev(k), _dev(v)).float().cpu().numpy()
    _close(got, O.full_mask_attention(q, k, v, og), "dense")
    z = S.skip_attention(_dev(q), _dev(k), _dev(v))
    assert z.shape == (1, 2, 700, 64) and not z.any()


def test_ones_probe_and_partition_probe_full_size():
    """Row-stochastic weights at the HunyuanVideo shape: v = ones -> 1; one-hot
    value columns splitting the keys -> per-row masses sum to 1."""
    import torch

    lay = (256, 33, 3600, 64)
    n = 119_056
    specs = [S.diagonal_spec(1), S.multi_diagonal_spec(), S.vertical_stripe_spec(stripes=(3, 700)), S.full_spec()]
    g = S.block_grid(S.TokenLayout(*lay))
    gen = torch.Generator(device="cuda").manual_seed(0)
    q = torch.randn(1, 4, n, 128, device="cuda", generator=gen).to(torch.bfloat16)
    k = torch.randn(1, 4, n, 128, device="cuda", generator=gen).to(torch.bfloat16)
    v = torch.zeros(1, 4, n, 128, device="cuda", dtype=torch.bfloat16)
    v[:, :, : n // 2, 1] = 1.0
    v[:, :, n // 2:, 0] = 1.0
    out = S.fused_layer_attention(q, k, v, S.group_heads(specs, g)).float()
    total = out[..., 0] + out[..., 1]
    assert (total - 1).abs().max().item() < 1e-2
    assert out[..., 2:].abs().max().item() == 0.0


@pytest.mark.parametrize("kernel", ["default", "hp"])
def test_full_size_sampled_rows_vs_oracle(kernel, monkeypatch):
    """HunyuanVideo layout at full N: sampled query blocks (incl. text/forced
    rows and the partial tail) of a diagonal, a multi-diagonal and a FULL head
    (kernel "hp": the opt-in half-row CTA-pair kernel, SVD_HP=1)."""
    import torch

    if kernel == "hp":
        monkeypatch.setenv("SVD_HP", "1")

    lay = (256, 33, 3600, 64)
    og = O.block_grid(*lay)
    n = og.n
    specs = [S.diagonal_spec(1), S.multi_diagonal_spec(), S.full_spec()]
    rng = np.random.default_rng(0)
    q = O.bf16_round(rng.standard_normal((1, 3, n, 128), dtype=np.float32) * 2)
    k = O.bf16_round(rng.standard_normal((1, 3, n, 128), dtype=np.float32))
    v = O.bf16_round(rng.standard_normal((1, 3, n, 128), dtype=np.float32))
    g = S.block_grid(S.TokenLayout(*lay))
    got = S.fused_layer_attention(_dev(q), _dev(k), _dev(v), S.group_heads(specs, g)).float().cpu().numpy()
    qblocks = [0, 3, 4, 57, 58, 900, 1859, 1860]
    rows = np.concatenate([np.arange(og.bounds[b], og.bounds[b + 1]) for b in qblocks])
    for h, spec in enumerate(specs):
        active = O.build_mask(spec, og)
        want = O.sparse_attention_rows(q[:, h:h + 1], k[:, h:h + 1], v[:, h:h + 1], active, og.bounds, qblocks)
        _close(got[:, h:h + 1, rows], want, f"full-size head {h}")


def test_deterministic():
    lay = (0, 16, 256, 64)
    specs = [S.full_spec(), S.diagonal_spec(1)]
    q, k, v = _inputs(5, 1, 2, 4096, 64)
    a = _gpu_fused(lay, specs, q, k, v)
    b = _gpu_fused(lay, specs, q, k, v)
    np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("world,split", [(2, False), (3, False), (2, True), (3, True)])
def test_shard_packed_rows_and_unpack_on_gpu(world, split):
    """The multi-GPU data path on one device: every shard plan writes its
    packed rows, the gathered buffer is unpacked by svd_unpack_rows, and the
    result equals the single-launch layer output — bit for bit without
    split-KV; with the planner's split-KV parts (merged in the kernel, a
    different fp32 summation order) within one bf16 ulp."""
    import torch

    from paper_2506_03065_b200 import _native as nat
    from paper_2506_03065_b200.sharding import gathered_row_maps

    lay = (96, 16, 250, 64)
    specs = [S.full_spec(), S.diagonal_spec(1), S.skip_spec(), S.multi_diagonal_spec(),
             S.vertical_stripe_spec(stripes=(5, 33))]
    q, k, v = (_dev(x) for x in _inputs(9, 1, len(specs), 4096, 128, 2.0))
    plan = S.LayerPlan.from_specs(specs, S.TokenLayout(*lay))
    ref = torch.empty_like(q)
    plan.forward(q, k, v, ref, head_dim=128)
    shards, heads, toks, max_rows = gathered_row_maps(plan, world, max_item_tiles=8 if split else -1)
    assert (sum(sh.info.n_split_groups for sh in shards) > 0) == split
    gathered = torch.zeros(world * max_rows, 128, dtype=torch.bfloat16, device="cuda")
    for r, sh in enumerate(shards):
        sh.forward(q, k, v, gathered[r * max_rows:(r + 1) * max_rows], head_dim=128)
    out = torch.full_like(q, float("nan"))
    rh, rt = torch.from_numpy(heads).cuda(), torch.from_numpy(toks).cuda()
    nat.check(nat.lib().svd_unpack_rows(
        nat.c_void_p(rh.data_ptr()), nat.c_void_p(rt.data_ptr()), int(world * max_rows),
        nat.c_void_p(gathered.data_ptr()), int(gathered.stride(0)), nat.c_void_p(out.data_ptr()),
        nat.i64x4(out.stride()), 128, nat.c_void_p(torch.cuda.current_stream().cuda_stream)))
    torch.cuda.synchronize()
    if split:
        torch.testing.assert_close(out.float(), ref.float(), atol=1.6e-2, rtol=8e-3)
    else:
        assert torch.equal(out, ref)
