"""One QKV-shaped GEMM from our kernel and one from cuBLAS (for an ncu capture)."""
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2506_03065_b200.layer import EPI_BF16, _gemm  # noqa: E402

M, D = 119056, 3072
a = torch.randn(M, D, device="cuda").to(torch.bfloat16)
b = (torch.randn(D, 3 * D, device="cuda") / D ** 0.5).to(torch.bfloat16)
out = torch.empty(M, 3 * D, device="cuda", dtype=torch.bfloat16)
_gemm(torch, a, b, out, EPI_BF16)
torch.mm(a, b)
torch.cuda.synchronize()
