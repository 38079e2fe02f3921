"""One block_key_mass call at a production layout (for ncu):
    python scripts/profile_key_mass.py [hunyuan|cogvideo|wan]"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2506_03065_b200 as S  # noqa: E402
from paper_2506_03065_b200.calibrate import block_key_mass  # noqa: E402

CFG = {"hunyuan": ((256, 33, 3600, 64), 24, 128), "cogvideo": ((226, 21, 4080, 64), 48, 64),
       "wan": ((0, 21, 3600, 64), 40, 128)}
lay, H, d = CFG[sys.argv[1] if len(sys.argv) > 1 else "hunyuan"]
grid = S.block_grid(S.TokenLayout(*lay))
N = grid.layout.total_tokens
q = torch.randn(1, H, N, d, device="cuda").bfloat16()
k = torch.randn(1, H, N, d, device="cuda").bfloat16()
block_key_mass(q, k, grid)
torch.cuda.synchronize()
