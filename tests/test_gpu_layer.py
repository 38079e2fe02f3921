"""The block around the operator on the GPU: layer_qkv /
layer_finish / layer_forward (model.py:372-420) against goldens written by
the reference itself (tests/golden/golden_layer.npz: a planted toy model),
and the streaming kernels (LayerNorm, RoPE, GELU) against the oracle.

Tolerances: the GPU block runs bf16 GEMMs (fp32 accumulation) and bf16
activations where the reference computes in fp64, so errors are stated
relative to the tensor's scale: max-abs <= 2e-2 * max|ref| and mean-abs <=
4e-3 * mean|ref| for Q/K/V and the block outputs."""

from types import SimpleNamespace

import numpy as np
import pytest

import paper_2506_03065_b200 as S
import svdit_oracle as O
from conftest import GOLDEN, gpu_available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]

MAX_REL, MEAN_REL = 2e-2, 4e-3


def _close(got, want, what):
    err = np.abs(np.asarray(got, dtype=np.float64) - want)
    scale_max, scale_mean = np.abs(want).max(), np.abs(want).mean()
    print(f"{what}: max {err.max():.3e} (ref max {scale_max:.3e}) mean {err.mean():.3e} "
          f"(ref mean {scale_mean:.3e})")
    assert err.max() <= MAX_REL * scale_max, what
    assert err.mean() <= MEAN_REL * scale_mean, what


@pytest.fixture(scope="module")
def golden_model():
    g = np.load(GOLDEN / "golden_layer.npz")
    layers, heads, d, seed, li = (int(v) for v in g["meta"])
    w = O.zero_redundant_heads(O.layer_weights(seed, li, heads, d), g["redundant_heads"], d)
    lw = SimpleNamespace(**w, planted_q={int(h): g[f"planted_q{h}"] for h in g["planted_heads"]},
                         planted_k={int(h): g[f"planted_k{h}"] for h in g["planted_heads"]})
    layout = S.TokenLayout(*(int(v) for v in g["layout"]))
    spec = SimpleNamespace(layers=layers, heads=heads, head_dim=d, layout=layout)
    model = SimpleNamespace(spec=spec, layers=[None] * li + [lw])
    return g, model, li


def test_layer_qkv_matches_reference(golden_model):
    g, model, li = golden_model
    q, k, v = S.layer_qkv(model, li, g["x"])
    for name, got in (("q", q), ("k", k), ("v", v)):
        _close(got, g[name], name)


def test_layer_finish_matches_reference(golden_model):
    g, model, li = golden_model
    _close(S.layer_finish(model, li, g["x"], g["attn"]), g["finish"], "layer_finish")


def test_layer_forward_matches_reference(golden_model):
    g, model, li = golden_model
    stripes = tuple(int(s) for s in g["stripes"])
    assignment = [S.diagonal_spec(1), S.vertical_stripe_spec(stripes=stripes), S.skip_spec(), S.full_spec()]
    _close(S.layer_forward(model, li, g["x"], assignment), g["forward"], "layer_forward")


def test_layer_forward_device_tensors(golden_model):
    import torch

    g, model, li = golden_model
    x = torch.from_numpy(g["x"]).cuda()
    f = S.layer_forward(model, li, x)  # every head FULL
    assert f.is_cuda and f.dtype == torch.float32 and f.shape == x.shape
    q, k, v = S.layer_qkv(model, li, x)
    og = O.block_grid(*(int(v) for v in g["layout"]))
    attn = O.fused_layer_attention(*(t.float().cpu().numpy() for t in (q, k, v)),
                                   O.group_heads([S.full_spec()] * model.spec.heads, og), og)
    w = {n: getattr(model.layers[li], n) for n in ("wq", "wk", "wv", "wo", "w1", "w2")}
    want = O.layer_finish(w, g["x"], attn)
    _close(f.cpu().numpy(), want, "layer_forward FULL (device)")


@pytest.mark.parametrize("dim", [64, 3072])
def test_layernorm_and_residual_kernel(dim):
    import torch

    from paper_2506_03065_b200 import _native as nat

    rng = np.random.default_rng(dim)
    x = (rng.standard_normal((300, dim)) * 3 + 1).astype(np.float32)
    r = rng.standard_normal((300, dim)).astype(np.float32)
    xt, rt = torch.from_numpy(x).cuda(), torch.from_numpy(r).cuda()
    a = torch.empty_like(xt)
    y = torch.empty(300, dim, dtype=torch.bfloat16, device="cuda")
    s = nat.c_void_p(torch.cuda.current_stream().cuda_stream)
    nat.check(nat.lib().svd_layernorm(nat.c_void_p(xt.data_ptr()), None, None, nat.c_void_p(y.data_ptr()),
                                      300, dim, 1e-5, s))
    want = O.layernorm(x.astype(np.float64))
    assert np.abs(y.float().cpu().numpy() - want).max() <= 2 ** -7 * np.abs(want).max()
    nat.check(nat.lib().svd_layernorm(nat.c_void_p(xt.data_ptr()), nat.c_void_p(rt.data_ptr()),
                                      nat.c_void_p(a.data_ptr()), nat.c_void_p(y.data_ptr()), 300, dim, 1e-5, s))
    np.testing.assert_array_equal(a.cpu().numpy(), x + r)
    want = O.layernorm((x + r).astype(np.float64))
    assert np.abs(y.float().cpu().numpy() - want).max() <= 2 ** -7 * np.abs(want).max()


def test_rope_and_gelu_kernels():
    import torch

    from paper_2506_03065_b200 import _native as nat

    B, N, H, d = 2, 1000, 3, 64
    rng = np.random.default_rng(3)
    D = H * d
    qkv = O.bf16_round(rng.standard_normal((B * N, 3 * D)).astype(np.float32))
    t = torch.from_numpy(qkv).cuda().to(torch.bfloat16)
    table = torch.empty(N, d // 2, 2, device="cuda")
    s = nat.c_void_p(torch.cuda.current_stream().cuda_stream)
    nat.check(nat.lib().svd_rope_table(nat.c_void_p(table.data_ptr()), N, d, 10000.0, s))
    nat.check(nat.lib().svd_rope_apply(nat.c_void_p(t.data_ptr()), B * N, 3 * D, D, N, H, d,
                                       nat.c_void_p(table.data_ptr()), s))
    got = t.float().cpu().numpy().reshape(B, N, 3, H, d)
    src = qkv.reshape(B, N, 3, H, d)
    for i in (0, 1):  # q and k rotated, v untouched
        want = O.rope(src[:, :, i].transpose(0, 2, 1, 3)).transpose(0, 2, 1, 3)
        assert np.abs(got[:, :, i] - want).max() <= 2 ** -7 * np.abs(want).max()
    np.testing.assert_array_equal(got[:, :, 2], src[:, :, 2])
    u = O.bf16_round(rng.standard_normal(4096).astype(np.float32) * 3)
    ut = torch.from_numpy(u).cuda().to(torch.bfloat16)
    nat.check(nat.lib().svd_gelu(nat.c_void_p(ut.data_ptr()), 4096, s))
    want = O.gelu(u.astype(np.float64))
    assert np.abs(ut.float().cpu().numpy() - want).max() <= 2 ** -8 * np.abs(want).max() + 1e-6
