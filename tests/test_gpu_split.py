"""Split-KV (SURVEY §8e load balance): shard plans cut long items along their
KV list and the kernel merges the parts' partial softmax states in the
epilogue of the last part to finish.  Checked on one device against the
unsplit launch and the oracle (2e-2 / 2e-3), repeated launches (the merge
tickets reset themselves), block sizes with per-element masks, d = 64 / 128."""

import numpy as np
import pytest

import paper_2506_03065_b200 as S
import svdit_oracle as O
from conftest import gpu_available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]


def _run_split(lay, specs, d, cap, seed=3, qscale=3.0):
    import torch

    from paper_2506_03065_b200 import _native as nat

    og = O.block_grid(*lay)
    q, k, v = O.random_qkv(seed, 1, len(specs), og.n, d)
    q, k, v = O.bf16_round(q * np.float32(qscale)), O.bf16_round(k), O.bf16_round(v)
    want = O.fused_layer_attention(q, k, v, O.group_heads(specs, og), og)
    tq, tk, tv = (torch.from_numpy(x).cuda().to(torch.bfloat16) for x in (q, k, v))
    plan = S.LayerPlan.from_specs(specs, S.TokenLayout(*lay))
    ref = torch.empty_like(tq)
    plan.forward(tq, tk, tv, ref, head_dim=d)
    sh = plan.shard(1, 0, max_item_tiles=cap)
    info = sh.info
    heads, toks = sh.shard_rows()
    outs = []
    for _ in range(3):  # tickets must reset: every launch merges again
        packed = torch.zeros(max(len(heads), 1), d, dtype=torch.bfloat16, device="cuda")
        sh.forward(tq, tk, tv, packed, head_dim=d)
        out = torch.full_like(tq, float("nan"))
        rh, rt = torch.from_numpy(heads).cuda(), torch.from_numpy(toks).cuda()
        nat.check(nat.lib().svd_unpack_rows(
            nat.c_void_p(rh.data_ptr()), nat.c_void_p(rt.data_ptr()), len(heads),
            nat.c_void_p(packed.data_ptr()), int(packed.stride(0)), nat.c_void_p(out.data_ptr()),
            nat.i64x4(out.stride()), d, nat.c_void_p(torch.cuda.current_stream().cuda_stream)))
        torch.cuda.synchronize()
        outs.append(out)
    return info, ref, outs, want


@pytest.mark.parametrize("d,cap", [(128, 3), (128, 7), (64, 2), (64, 5)])
def test_split_kv_matches_unsplit_and_oracle(d, cap):
    import torch

    lay = (96, 16, 250, 64)
    specs = [S.full_spec(), S.diagonal_spec(1), S.skip_spec(), S.multi_diagonal_spec(),
             S.vertical_stripe_spec(stripes=(5, 33)), S.full_spec()]
    info, ref, outs, want = _run_split(lay, specs, d, cap)
    assert info.n_split_groups > 0 and info.max_split_parts > 1
    for o in outs[1:]:
        assert torch.equal(o, outs[0])
    torch.testing.assert_close(outs[0].float(), ref.float(), atol=1.6e-2, rtol=8e-3)
    got = outs[0].float().cpu().numpy()
    err = np.abs(got - want)
    assert err.max() <= 2e-2 and err.mean() <= 2e-3, (err.max(), err.mean())
    assert not got[:, 2].any()  # SKIP head


def test_split_kv_fine_mask_layout():
    lay = (77, 6, 300, 48)  # block 48: per-element masks, partial tail, text / mixed blocks
    specs = [S.full_spec(), S.diagonal_spec(2), S.vertical_stripe_spec(stripes=(3, 20), include_diagonal=False)]
    info, ref, outs, want = _run_split(lay, specs, 128, 4, seed=8, qscale=8.0)
    assert info.n_split_groups > 0
    err = np.abs(outs[0].float().cpu().numpy() - want)
    assert err.max() <= 2e-2 and err.mean() <= 2e-3, (err.max(), err.mean())
