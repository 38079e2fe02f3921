"""Host-buffer path of the public API: CPU torch tensors are streamed through
the GPU in head chunks (copy-in / kernel / copy-out overlapped) and give the
same bits as the device path."""

import numpy as np
import pytest

import paper_2506_03065_b200 as S
from conftest import gpu_available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]


@pytest.mark.parametrize("d", [64, 128, 40])
def test_host_pipeline_matches_device_path(d):
    import torch

    lay = (96, 16, 250, 64)
    specs = [S.full_spec(), S.diagonal_spec(1), S.skip_spec(), S.multi_diagonal_spec(),
             S.vertical_stripe_spec(stripes=(5, 33)), S.diagonal_spec(1), S.full_spec()]
    g = S.block_grid(S.TokenLayout(*lay))
    gen = torch.Generator().manual_seed(d)
    q, k, v = (torch.randn(1, len(specs), 4096, d, generator=gen).to(torch.bfloat16).pin_memory()
               for _ in range(3))
    groups = S.group_heads(specs, g)
    host = S.fused_layer_attention(q, k, v, groups)
    assert host.device.type == "cpu" and host.dtype == torch.bfloat16 and host.shape == q.shape
    dev = S.fused_layer_attention(q.cuda(), k.cuda(), v.cuda(), groups).cpu()
    assert torch.equal(host, dev)
    assert not host[:, 2].any()


def test_host_pipeline_unpinned_fp32():
    import torch

    g = S.block_grid(S.TokenLayout(0, 8, 128, 64))
    q, k, v = (torch.randn(2, 3, 1024, 64) for _ in range(3))
    specs = [S.diagonal_spec(1), S.full_spec(), S.diagonal_spec(0)]
    host = S.fused_layer_attention(q, k, v, S.group_heads(specs, g))
    dev = S.fused_layer_attention(q.cuda(), k.cuda(), v.cuda(), S.group_heads(specs, g)).cpu()
    assert torch.equal(host, dev)


@pytest.mark.parametrize("d", [64, 40])
def test_out_buffer_host_and_device(d):
    """out= writes the caller's buffer in place (host pinned and device), same
    bits as the allocating call."""
    import torch

    g = S.block_grid(S.TokenLayout(0, 8, 128, 64))
    specs = [S.diagonal_spec(1), S.full_spec(), S.skip_spec()]
    groups = S.group_heads(specs, g)
    q, k, v = (torch.randn(1, 3, 1024, d).to(torch.bfloat16).pin_memory() for _ in range(3))
    want = S.fused_layer_attention(q, k, v, groups)
    hout = torch.full(q.shape, 7.0, dtype=torch.bfloat16).pin_memory()
    got = S.fused_layer_attention(q, k, v, groups, out=hout)
    assert got.data_ptr() == hout.data_ptr() and torch.equal(hout, want)
    dout = torch.full(q.shape, 7.0, dtype=torch.bfloat16, device="cuda")
    got = S.fused_layer_attention(q.cuda(), k.cuda(), v.cuda(), groups, out=dout)
    assert got.data_ptr() == dout.data_ptr() and torch.equal(dout.cpu(), want)
    with pytest.raises(S.ShapeError):
        S.fused_layer_attention(q, k, v, groups, out=torch.empty(1, 3, 1024, d))


def test_host_all_skip_layer():
    """Every head SKIP: nothing crosses PCIe, the host O is zeroed in place."""
    import torch

    g = S.block_grid(S.TokenLayout(0, 8, 128, 64))
    groups = S.group_heads([S.skip_spec()] * 2, g)
    q, k, v = (torch.randn(1, 2, 1024, 64).to(torch.bfloat16).pin_memory() for _ in range(3))
    hout = torch.full(q.shape, 7.0, dtype=torch.bfloat16).pin_memory()
    got = S.fused_layer_attention(q, k, v, groups, out=hout)
    assert got.data_ptr() == hout.data_ptr() and not hout.any()


def test_output_head_map_and_zero_copy(monkeypatch):
    """svd_attn_fwd_ex's output head map (a head-subset plan writing into a
    full-layer O) and the opt-in zero-copy host pipeline give the same bits."""
    import torch

    from paper_2506_03065_b200 import attention as A

    g = S.block_grid(S.TokenLayout(0, 8, 128, 64))
    specs = [S.diagonal_spec(1), S.full_spec(), S.skip_spec(), S.multi_diagonal_spec()]
    plan = S.plan_for_assignment(specs, S.TokenLayout(0, 8, 128, 64))
    q, k, v = (torch.randn(1, 4, 1024, 64, device="cuda").to(torch.bfloat16) for _ in range(3))
    ref = torch.empty_like(q)
    plan.forward(q, k, v, ref)
    heads = (3, 1)
    sub = plan.heads_subplan(heads)
    out = torch.zeros_like(q)
    sub.forward(q[:, list(heads)].contiguous(), k[:, list(heads)].contiguous(), v[:, list(heads)].contiguous(),
                out, o_head_map=torch.tensor(heads, dtype=torch.int32, device="cuda"))
    for h in heads:
        assert torch.equal(out[:, h], ref[:, h])
    assert not out[:, 0].any() and not out[:, 2].any()
    hq, hk, hv = (t.cpu().pin_memory() for t in (q, k, v))
    groups = S.group_heads(specs, g)
    want = S.fused_layer_attention(hq, hk, hv, groups)
    monkeypatch.setattr(A, "HOST_ZERO_COPY", True)
    got = S.fused_layer_attention(hq, hk, hv, groups)
    assert torch.equal(got, want) and torch.equal(got, ref.cpu())


@pytest.mark.parametrize("block", [32, 96])
def test_numpy_path_fine_blocks_match_device_path(block):
    """float32 NumPy in/out (the reference's types) runs the chunked host
    pipeline — head-subset plans (svd_plan_subset) incl. their FINE mask
    tables for block sizes off the 64-token grain — and gives the device
    path's bf16 result exactly."""
    import numpy as np
    import torch

    lay = S.TokenLayout(37, 5, 200, block)
    g = S.block_grid(lay)
    specs = [S.diagonal_spec(1), S.full_spec(), S.skip_spec(), S.multi_diagonal_spec(period=3),
             S.vertical_stripe_spec(stripes=(1, g.n_blocks - 2)), S.diagonal_spec(2)]
    groups = S.group_heads(specs, g)
    rng = np.random.default_rng(block)
    q, k, v = (rng.standard_normal((1, len(specs), lay.total_tokens, 64), dtype=np.float32) for _ in range(3))
    got = S.fused_layer_attention(q, k, v, groups)
    assert got.dtype == np.float32
    dev = S.fused_layer_attention(*(torch.from_numpy(x).cuda() for x in (q, k, v)), groups)
    np.testing.assert_array_equal(got, dev.float().cpu().numpy())
    assert not got[:, 2].any()
