"""Per-GEMM times of the vDiT block in its own flow (ours: svd_gemm with the
fused epilogues; library: torch.mm + this package's row / element passes),
HunyuanVideo shapes, CUDA events around each launch."""
import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_2506_03065_b200 as S  # noqa: E402
from paper_2506_03065_b200 import layer as L  # noqa: E402

nat = S._native
n, H, d = 119056, 24, 128
D = H * d
torch.manual_seed(0)
x = torch.randn(n, D, device="cuda")
o = torch.randn(n, D, device="cuda").to(torch.bfloat16)
wo = (torch.randn(D, D, device="cuda") / D ** 0.5).to(torch.bfloat16)
w1 = (torch.randn(D, 4 * D, device="cuda") / D ** 0.5).to(torch.bfloat16)
w2 = (torch.randn(4 * D, D, device="cuda") / (4 * D) ** 0.5).to(torch.bfloat16)
st = lambda: nat.c_void_p(torch.cuda.current_stream().cuda_stream)  # noqa: E731
a = torch.empty(n, D, device="cuda")
h2 = torch.empty(n, D, dtype=torch.bfloat16, device="cuda")
u = torch.empty(n, 4 * D, dtype=torch.bfloat16, device="cuda")
f = torch.empty(n, D, device="cuda")


def ours():
    yield "wo+resid", lambda: L._gemm(torch, o, wo, a, L.EPI_F32_RESID, resid=x)
    yield "ln", lambda: nat.check(nat.lib().svd_layernorm(nat.c_void_p(a.data_ptr()), None, None,
                                                          nat.c_void_p(h2.data_ptr()), n, D, 1e-5, st()))
    yield "w1+gelu", lambda: L._gemm(torch, h2, w1, u, L.EPI_GELU)
    yield "w2+resid", lambda: L._gemm(torch, u, w2, f, L.EPI_F32_RESID, resid=a)


def lib():
    state = {}
    yield "wo", lambda: state.__setitem__("p", torch.mm(o, wo, out_dtype=torch.float32))
    yield "ln+resid", lambda: nat.check(nat.lib().svd_layernorm(
        nat.c_void_p(x.data_ptr()), nat.c_void_p(state["p"].data_ptr()), nat.c_void_p(a.data_ptr()),
        nat.c_void_p(h2.data_ptr()), n, D, 1e-5, st()))
    yield "w1", lambda: state.__setitem__("u", torch.mm(h2, w1))
    yield "gelu", lambda: nat.check(nat.lib().svd_gelu(nat.c_void_p(state["u"].data_ptr()), state["u"].numel(), st()))
    yield "w2", lambda: state.__setitem__("f", torch.mm(state["u"], w2, out_dtype=torch.float32))
    yield "add", lambda: state["f"].add_(a)


res = {}
for name, flow in (("ours", ours), ("library", lib)):
    steps = list(flow())
    for _ in range(2):
        for _, fn in steps:
            fn()
    torch.cuda.synchronize()
    times = {k: 0.0 for k, _ in steps}
    reps = 5
    for _ in range(reps):
        evs = []
        for k, fn in steps:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            evs.append((k, e0, e1))
        torch.cuda.synchronize()
        for k, e0, e1 in evs:
            times[k] += e0.elapsed_time(e1) / reps
    res[name] = {k: round(v, 3) for k, v in times.items()}
    res[name]["total"] = round(sum(times.values()), 3)
print(json.dumps(res))
