"""One cuDNN SDPA launch (HunyuanVideo heads, 32k tokens) and one of our dense
launch on the same inputs, for an ncu comparison of the kernels' structure."""
import sys
from pathlib import Path

import torch
import torch.nn.functional as F
from torch.nn.attention import SDPBackend, sdpa_kernel

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_2506_03065_b200 as S  # noqa: E402

H, n, d = 24, 32768, int(sys.argv[1]) if len(sys.argv) > 1 else 128
q, k, v = (torch.randn(1, H, n, d, device="cuda").to(torch.bfloat16) for _ in range(3))
with sdpa_kernel([SDPBackend.CUDNN_ATTENTION]):
    F.scaled_dot_product_attention(q, k, v)
lay = S.TokenLayout(0, 1, n, 64)
plan = S.plan_for_assignment([S.full_spec()] * H, lay)
o = torch.empty_like(q)
plan.forward(q, k, v, o, head_dim=d)
torch.cuda.synchronize()
