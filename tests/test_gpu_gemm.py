"""The block's tcgen05 GEMM (csrc/svd_gemm.cu) against a plain PyTorch fp32
reference of the same op (the block's GEMMs, model.py:372-402): bf16
operands, fp32 accumulation; every fused epilogue (RoPE, GELU, fp32 residual),
ragged M / N / K tails and persistent multi-tile schedules."""

import math

import numpy as np
import pytest

from conftest import gpu_available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]


def _ref(a, b):
    return a.float() @ b.float()


@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (300, 200, 72), (1000, 768, 320), (4096, 1536, 1024),
                                   (129, 8, 8)])
def test_gemm_plain(M, N, K):
    import torch

    from paper_2506_03065_b200.layer import EPI_BF16, EPI_F32, _gemm

    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    a = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    b = (torch.randn(K, N, device="cuda", generator=g) / math.sqrt(K)).to(torch.bfloat16)
    want = _ref(a, b)
    o32 = torch.full((M, N), float("nan"), device="cuda")
    _gemm(torch, a, b, o32, EPI_F32)
    torch.testing.assert_close(o32, want, atol=2e-4 * math.sqrt(K) / 8 + 1e-4, rtol=1e-4)
    o16 = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    _gemm(torch, a, b, o16, EPI_BF16)
    torch.testing.assert_close(o16.float(), want, atol=1e-2, rtol=1e-2)


def test_gemm_epilogues():
    import torch

    from paper_2506_03065_b200.layer import EPI_F32_RESID, EPI_GELU, EPI_ROPE, _gemm, _rope_table

    torch.manual_seed(0)
    B, N_tok, H, d = 2, 333, 4, 64
    D = H * d
    M = B * N_tok
    h = torch.randn(M, D, device="cuda").to(torch.bfloat16)
    w = (torch.randn(D, 3 * D, device="cuda") / math.sqrt(D)).to(torch.bfloat16)
    full = _ref(h, w)
    # RoPE on the q / k blocks, pair (2c, 2c+1) of each head by the token's angle
    table = _rope_table(torch, torch.device("cuda", 0), N_tok, d)
    out = torch.empty(M, 3 * D, dtype=torch.bfloat16, device="cuda")
    _gemm(torch, h, w, out, EPI_ROPE, rope=table, rope_cols=2 * D, head_dim=d, n_tokens=N_tok)
    tok = torch.arange(M, device="cuda") % N_tok
    cs = table[tok]  # [M, d/2, 2]
    want = full.clone()
    for blk in range(2):
        x = full[:, blk * D:(blk + 1) * D].view(M, H, d // 2, 2)
        c, s = cs[:, None, :, 0], cs[:, None, :, 1]
        rot = torch.stack([x[..., 0] * c - x[..., 1] * s, x[..., 0] * s + x[..., 1] * c], dim=-1)
        want[:, blk * D:(blk + 1) * D] = rot.reshape(M, D)
    torch.testing.assert_close(out.float(), want, atol=2e-2, rtol=1e-2)
    # GELU (exact erf)
    g = torch.empty(M, 3 * D, dtype=torch.bfloat16, device="cuda")
    _gemm(torch, h, w, g, EPI_GELU)
    torch.testing.assert_close(g.float(), torch.nn.functional.gelu(full), atol=2e-2, rtol=1e-2)
    # fp32 + residual
    r = torch.randn(M, 3 * D, device="cuda")
    f = torch.empty(M, 3 * D, device="cuda")
    _gemm(torch, h, w, f, EPI_F32_RESID, resid=r)
    torch.testing.assert_close(f, full + r, atol=1e-3, rtol=1e-4)
