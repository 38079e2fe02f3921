"""The block's GEMM shapes (HunyuanVideo: M = 119,056 tokens, D = 3072): our
tcgen05 kernel (svd_gemm, fused epilogues) vs cuBLAS (torch.mm), CUDA events."""
import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2506_03065_b200.layer import EPI_BF16, EPI_F32, EPI_F32_RESID, EPI_GELU, _gemm  # noqa: E402


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


M = int(sys.argv[1]) if len(sys.argv) > 1 else 119056
D = int(sys.argv[2]) if len(sys.argv) > 2 else 3072
res = {"M": M, "D": D}
for name, K, N, epi in (("qkv", D, 3 * D, EPI_BF16), ("wo", D, D, EPI_F32), ("w1", D, 4 * D, EPI_GELU),
                        ("w2", 4 * D, D, EPI_F32_RESID)):
    a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    b = (torch.randn(K, N, device="cuda") / K ** 0.5).to(torch.bfloat16)
    f32 = epi in (EPI_F32, EPI_F32_RESID)
    out = torch.empty(M, N, device="cuda", dtype=torch.float32 if f32 else torch.bfloat16)
    r = torch.randn(M, N, device="cuda") if epi == EPI_F32_RESID else None
    ours = timed(lambda: _gemm(torch, a, b, out, epi, resid=r))
    lib = timed(lambda: torch.mm(a, b, out_dtype=torch.float32) if f32 else torch.mm(a, b))
    err = (out.float() - (a.float() @ b.float() + (r if r is not None else 0)) if epi != EPI_GELU else
           out.float() - torch.nn.functional.gelu(a.float() @ b.float())).abs().max().item() if M <= 8192 else None
    fl = 2.0 * M * N * K
    res[name] = {"ours_ms": round(ours, 3), "cublas_ms": round(lib, 3), "ours_tflops": round(fl / ours / 1e9, 1),
                 "cublas_tflops": round(fl / lib / 1e9, 1), "max_err": err}
    del a, b, out, r
print(json.dumps(res))
