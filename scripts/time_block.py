"""Time the whole vDiT block on the GPU at a bench layer shape: layer_qkv
(LN + fused QKV GEMM + RoPE), the sparse attention, layer_finish (out-proj +
residual LN + GELU MLP) — CUDA events, random weights of the model's shape.
Reports each part's share (the reference's attention_latency_share,
costmodel.py:42-50, measured)."""
import json
import sys
from pathlib import Path
from types import SimpleNamespace

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2506_03065_b200 as S  # noqa: E402
from paper_2506_03065_b200 import layer as L  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "hunyuan"
cfg = bench.CONFIGS[cfgname]
layout = S.TokenLayout(*cfg["layout"])
n, H, d = layout.total_tokens, cfg["heads"], cfg["d"]
D = H * d
rng = np.random.default_rng(0)
w = {k: (rng.standard_normal(s, dtype=np.float32) / np.sqrt(s[0])) for k, s in
     {"wq": (D, D), "wk": (D, D), "wv": (D, D), "wo": (D, D), "w1": (D, 4 * D), "w2": (4 * D, D)}.items()}
model = SimpleNamespace(spec=SimpleNamespace(layers=1, heads=H, head_dim=d, layout=layout),
                        layers=[SimpleNamespace(**w, planted_q={}, planted_k={})])
dm = L.DeviceModel(model)
x = torch.randn(1, n, D, device="cuda")
specs = bench.assignment_for(cfg, S)
groups = S.group_heads(specs, S.block_grid(layout))


def timed(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def _s():
    return S._native.c_void_p(torch.cuda.current_stream().cuda_stream)


def qkv_cublas():
    """The round-1 flow: LN, cuBLAS QKV GEMM, RoPE pass (library GEMM baseline)."""
    nat = S._native
    wl = dm.layer(0)
    rows = n
    h = torch.empty((rows, D), dtype=torch.bfloat16, device="cuda")
    nat.check(nat.lib().svd_layernorm(nat.c_void_p(x.data_ptr()), None, None, nat.c_void_p(h.data_ptr()),
                                      rows, D, L.LN_EPS, _s()))
    qkv = torch.mm(h, wl.wqkv)
    table = L._rope_table(torch, x.device, n, d)
    nat.check(nat.lib().svd_rope_apply(nat.c_void_p(qkv.data_ptr()), rows, 3 * D, D, n, H, d,
                                       nat.c_void_p(table.data_ptr()), _s()))
    return qkv


def finish_cublas(attn):
    """The round-1 flow: cuBLAS out-proj, LN with fused residual, cuBLAS W1, GELU pass, cuBLAS W2, + a."""
    nat = S._native
    wl = dm.layer(0)
    merged = attn.permute(0, 2, 1, 3).reshape(n, D)
    proj = torch.mm(merged, wl.wo, out_dtype=torch.float32)
    a = torch.empty((n, D), dtype=torch.float32, device="cuda")
    h2 = torch.empty((n, D), dtype=torch.bfloat16, device="cuda")
    nat.check(nat.lib().svd_layernorm(nat.c_void_p(x.data_ptr()), nat.c_void_p(proj.data_ptr()),
                                      nat.c_void_p(a.data_ptr()), nat.c_void_p(h2.data_ptr()), n, D, L.LN_EPS, _s()))
    u = torch.mm(h2, wl.w1)
    nat.check(nat.lib().svd_gelu(nat.c_void_p(u.data_ptr()), u.numel(), _s()))
    f = torch.mm(u, wl.w2, out_dtype=torch.float32)
    f += a
    return f


q, k, v = L._qkv(dm, 0, x)
o = torch.empty(1, n, H, d, dtype=torch.bfloat16, device="cuda")
res = {"config": cfgname, "tokens": n, "hidden": D}
res["qkv_ms"] = timed(lambda: L._qkv(dm, 0, x))
res["attention_ms"] = timed(lambda: S.fused_layer_attention(q, k, v, groups, out=o.permute(0, 2, 1, 3)))
res["finish_ms"] = timed(lambda: L._finish(dm, 0, x, o.permute(0, 2, 1, 3)))
res["layer_forward_ms"] = timed(lambda: L.layer_forward(dm, 0, x, specs))
res["qkv_cublas_ms"] = timed(qkv_cublas)
res["finish_cublas_ms"] = timed(lambda: finish_cublas(o.permute(0, 2, 1, 3)))
res["gemm_part_ours_ms"] = res["qkv_ms"] + res["finish_ms"]
res["gemm_part_cublas_ms"] = res["qkv_cublas_ms"] + res["finish_cublas_ms"]
# agreement of the two flows (fp32 accumulation in both; RoPE rounds once in ours, twice in the library flow)
ref = finish_cublas(o.permute(0, 2, 1, 3))
ours = L._finish(dm, 0, x, o.permute(0, 2, 1, 3)).view(n, D)
res["finish_max_abs_diff"] = float((ref - ours).abs().max())
res["qkv_max_abs_diff"] = float((qkv_cublas().float() - torch.cat(
    [t_.permute(0, 2, 1, 3).reshape(n, D).float() for t_ in L._qkv(dm, 0, x)], dim=1)).abs().max())
res["attention_share"] = res["attention_ms"] / (res["qkv_ms"] + res["attention_ms"] + res["finish_ms"])
res["linear_tflops"] = S.layer_linear_flops(n, D) / ((res["qkv_ms"] + res["finish_ms"]) * 1e-3) / 1e12
print(json.dumps({k: (round(v, 4) if isinstance(v, float) else v) for k, v in res.items()}))
