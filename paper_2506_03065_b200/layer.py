"""The vDiT block around the attention operator, on the GPU.

Mirrors the reference's drop-in call site (model.py:405-420):

    layer_forward(model, l, x, assignment)
      = layer_finish(model, l, x, fused_layer_attention(*layer_qkv(model, l, x), groups))

with the same functions and argument meaning: `layer_qkv` (model.py:372-391),
`layer_finish` (model.py:394-402), `layer_forward` (model.py:405-420).
`model` is the reference's Model (or anything shaped like it: .spec.heads,
.spec.head_dim, .spec.layout, .layers[l].{wq,wk,wv,wo,w1,w2,planted_q,planted_k})
or a `DeviceModel` built from one; weights are uploaded once (bf16, Q/K/V
projections fused into one [D, 3D] matrix) and cached per model object.

B200 data flow (no split/merge-heads copies):
  x fp32 --svd_layernorm--> h bf16 --GEMM--> qkv [B*N, 3D] --svd_rope_apply(q, k)-->
  q/k/v = strided [B, H, N, d] views of qkv (the attention kernel reads them
  through TMA strides) --attention--> O stored [B, N, H, d] (= merged heads)
  --GEMM, fp32 out--> svd_layernorm(x + proj) --GEMM--> svd_gelu --GEMM, fp32--> + a
The four GEMMs are this package's tcgen05 kernel (csrc/svd_gemm.cu, bf16
operands, fp32 accumulation in TMEM) with the step after each fused into its
epilogue: RoPE on the q / k column blocks of the QKV projection, the
attention residual (a = x + O Wo, fp32), exact GELU after W1 and the MLP
residual (f = a + u W2, fp32).  LayerNorm stays a row pass
(csrc/svd_layer.cu): its statistics span a whole row of D columns, wider
than an output tile.  The residual stream x stays fp32 like the reference's
float32 latent.
"""

from __future__ import annotations

import weakref

import numpy as np

from . import _native as nat
from .attention import fused_layer_attention, group_heads
from .errors import ConfigError, ShapeError
from .layout import block_grid
from .patterns import full_spec

ROPE_BASE = 10000.0  # model.py:39
LN_EPS = 1e-5        # model.py:355


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise nat.NativeError("a CUDA device is required: the block has no CPU path")
    return torch


def _stream(torch, dev):
    return nat.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


class BlockWeights:
    """One layer's weights on the device: bf16 W_qkv [D, 3D], W_o, W_1, W_2
    and the planted heads' q / k codes (bf16 [N, d])."""

    def __init__(self, layer, heads: int, head_dim: int, device):
        torch = _torch()
        self.heads, self.head_dim, self.device = heads, head_dim, device
        dim = heads * head_dim
        if head_dim % 8 != 0:
            raise nat.NativeError(f"head_dim {head_dim} unsupported (multiple of 8 required)")

        def dev(a):
            return torch.as_tensor(np.asarray(a, dtype=np.float32)).to(device, torch.bfloat16)

        wq, wk, wv = (np.asarray(getattr(layer, n), dtype=np.float32) for n in ("wq", "wk", "wv"))
        if wq.shape != (dim, dim):
            raise ShapeError(f"wq has shape {wq.shape}, expected {(dim, dim)}")
        self.wqkv = dev(np.concatenate([wq, wk, wv], axis=1))
        self.wo, self.w1, self.w2 = dev(layer.wo), dev(layer.w1), dev(layer.w2)
        self.planted_q = {int(h): dev(c) for h, c in getattr(layer, "planted_q", {}).items()}
        self.planted_k = {int(h): dev(c) for h, c in getattr(layer, "planted_k", {}).items()}


class DeviceModel:
    """Device-resident weights of a reference-shaped Model (lazily per layer)."""

    def __init__(self, model, device=None):
        torch = _torch()
        self.model = model
        self.spec = model.spec
        self.device = torch.device(device) if device is not None else torch.device(
            "cuda", torch.cuda.current_device())
        self._layers: dict[int, BlockWeights] = {}

    def layer(self, l: int) -> BlockWeights:
        if not 0 <= l < self.spec.layers:
            raise IndexError(f"layer {l} out of range")
        if l not in self._layers:
            self._layers[l] = BlockWeights(self.model.layers[l], self.spec.heads, self.spec.head_dim,
                                           self.device)
        return self._layers[l]


_DEVICE_MODELS: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()
_ROPE_TABLES: dict = {}


_PINNED_MODELS: dict = {}  # id -> (model, DeviceModel) for objects without weakref support


def _device_model(model) -> DeviceModel:
    if isinstance(model, DeviceModel):
        return model
    try:
        dm = _DEVICE_MODELS.get(model)
        if dm is None:
            dm = _DEVICE_MODELS[model] = DeviceModel(model)
        return dm
    except TypeError:
        hit = _PINNED_MODELS.get(id(model))
        if hit is None or hit[0] is not model:
            while len(_PINNED_MODELS) >= 4:
                _PINNED_MODELS.pop(next(iter(_PINNED_MODELS)))
            hit = _PINNED_MODELS[id(model)] = (model, DeviceModel(model))
        return hit[1]


def _rope_table(torch, dev, n: int, d: int):
    key = (dev.index, n, d)
    t = _ROPE_TABLES.get(key)
    if t is None:
        t = torch.empty((n, d // 2, 2), dtype=torch.float32, device=dev)
        nat.check(nat.lib().svd_rope_table(nat.c_void_p(t.data_ptr()), n, d, ROPE_BASE, _stream(torch, dev)))
        _ROPE_TABLES[key] = t
    return t


def _as_latent(torch, x, dev):
    """x as a contiguous fp32 [B, N, D] device tensor (and whether it was NumPy)."""
    was_numpy = not (type(x).__module__.startswith("torch"))
    if was_numpy:
        t = torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=np.float32))).to(dev)
    else:
        t = x.to(dev, torch.float32).contiguous()
    if t.dim() != 3:
        raise ShapeError(f"x must have rank 3 [B, N, D], got rank {t.dim()}")
    return t, was_numpy


# svd_gemm epilogues (include/svdit_b200.h)
EPI_BF16, EPI_ROPE, EPI_GELU, EPI_F32_RESID, EPI_F32 = range(5)


def _gemm(torch, a, b, out, epilogue: int, resid=None, rope=None, rope_cols: int = 0, head_dim: int = 0,
          n_tokens: int = 0):
    """out = epilogue(a @ b) on the tensor cores (svd_gemm): a [M, K] and b
    [K, N] bf16 row-major, out [M, N] bf16 or fp32 (row-major, unit column
    stride)."""
    M, K = a.shape
    N = b.shape[1]
    for name, t_ in (("a", a), ("b", b), ("out", out)):
        if t_.stride(-1) != 1:
            raise ShapeError(f"gemm: {name} needs a unit column stride")
    nat.check(nat.lib().svd_gemm(
        nat.c_void_p(a.data_ptr()), a.stride(0), nat.c_void_p(b.data_ptr()), b.stride(0),
        nat.c_void_p(out.data_ptr()), out.stride(0), M, N, K, int(epilogue),
        nat.c_void_p(resid.data_ptr()) if resid is not None else None,
        resid.stride(0) if resid is not None else 0,
        nat.c_void_p(rope.data_ptr()) if rope is not None else None, int(rope_cols), int(head_dim),
        int(n_tokens), _stream(torch, a.device)))
    return out


def _qkv(dm: DeviceModel, l: int, x):
    torch = _torch()
    w = dm.layer(l)
    dev = dm.device
    B, N, D = x.shape
    H, d = w.heads, w.head_dim
    if D != H * d:
        raise ShapeError(f"x has hidden size {D}, model has {H}x{d}")
    rows = B * N
    h = torch.empty((rows, D), dtype=torch.bfloat16, device=dev)
    nat.check(nat.lib().svd_layernorm(nat.c_void_p(x.data_ptr()), None, None, nat.c_void_p(h.data_ptr()),
                                      rows, D, LN_EPS, _stream(torch, dev)))
    table = _rope_table(torch, dev, N, d)
    qkv = torch.empty((rows, 3 * D), dtype=torch.bfloat16, device=dev)
    # [B*N, 3D] = h Wqkv with RoPE on the q and k blocks (columns [0, 2D)) in the epilogue
    _gemm(torch, h, w.wqkv, qkv, EPI_ROPE, rope=table, rope_cols=2 * D, head_dim=d, n_tokens=N)
    view = qkv.view(B, N, 3, H, d)
    q, k, v = (view[:, :, i].permute(0, 2, 1, 3) for i in range(3))  # [B, H, N, d] strided views
    for head, code in w.planted_q.items():
        q[:, head].copy_(code.expand(B, N, d))
    for head, code in w.planted_k.items():
        k[:, head].copy_(code.expand(B, N, d))
    return q, k, v


def _finish(dm: DeviceModel, l: int, x, attn):
    torch = _torch()
    w = dm.layer(l)
    dev = dm.device
    B, N, D = x.shape
    H, d = w.heads, w.head_dim
    if tuple(attn.shape) != (B, H, N, d):
        raise ShapeError(f"attention output has shape {tuple(attn.shape)}, expected {(B, H, N, d)}")
    merged = attn.to(dev, torch.bfloat16).permute(0, 2, 1, 3)  # [B, N, H, d]: free when O was stored so
    merged = merged.reshape(B * N, D)
    if merged.data_ptr() % 16 or merged.stride(0) % 8:
        merged = merged.contiguous()
    x2 = x.view(B * N, D)
    a = torch.empty((B * N, D), dtype=torch.float32, device=dev)
    _gemm(torch, merged, w.wo, a, EPI_F32_RESID, resid=x2)  # a = x + O Wo
    h2 = torch.empty((B * N, D), dtype=torch.bfloat16, device=dev)
    nat.check(nat.lib().svd_layernorm(nat.c_void_p(a.data_ptr()), None, None, nat.c_void_p(h2.data_ptr()),
                                      B * N, D, LN_EPS, _stream(torch, dev)))
    u = torch.empty((B * N, w.w1.shape[1]), dtype=torch.bfloat16, device=dev)
    _gemm(torch, h2, w.w1, u, EPI_GELU)  # GELU(h2 W1)
    f = torch.empty((B * N, D), dtype=torch.float32, device=dev)
    _gemm(torch, u, w.w2, f, EPI_F32_RESID, resid=a)  # f = a + u W2
    return f.view(B, N, D)


def layer_qkv(model, layer_idx: int, x):
    """Q, K, V of one layer from latent x [B, N, D] (model.py:372-391).

    Device inputs give bf16 [B, H, N, d] strided views of one fused buffer;
    NumPy inputs give float32 NumPy arrays (the reference's types)."""
    torch = _torch()
    dm = _device_model(model)
    xt, was_numpy = _as_latent(torch, x, dm.device)
    q, k, v = _qkv(dm, layer_idx, xt)
    if was_numpy:
        return tuple(t.float().cpu().numpy() for t in (q, k, v))
    return q, k, v


def layer_finish(model, layer_idx: int, x, attn_out):
    """Output projection + residual, then the GELU MLP residual (model.py:394-402).
    Returns fp32 [B, N, D] (NumPy for NumPy inputs)."""
    torch = _torch()
    dm = _device_model(model)
    xt, was_numpy = _as_latent(torch, x, dm.device)
    at = attn_out
    if not type(attn_out).__module__.startswith("torch"):
        at = torch.from_numpy(np.ascontiguousarray(np.asarray(attn_out, dtype=np.float32))).to(dm.device)
    f = _finish(dm, layer_idx, xt, at)
    return f.cpu().numpy() if was_numpy else f


def layer_forward(model, layer_idx: int, x, assignment=None):
    """One block under a per-head pattern assignment (model.py:405-420); None
    means every head FULL.  The attention output is written straight into
    [B, N, H, d] storage, so merging heads costs nothing."""
    torch = _torch()
    dm = _device_model(model)
    spec = dm.spec
    if assignment is None:
        assignment = [full_spec()] * spec.heads
    if len(assignment) != spec.heads:
        raise ConfigError(f"assignment covers {len(assignment)} heads, model has {spec.heads}")
    xt, was_numpy = _as_latent(torch, x, dm.device)
    q, k, v = _qkv(dm, layer_idx, xt)
    B, H, N, d = q.shape
    o = torch.empty((B, N, H, d), dtype=torch.bfloat16, device=dm.device)
    groups = group_heads(assignment, block_grid(spec.layout))
    fused_layer_attention(q, k, v, groups, out=o.permute(0, 2, 1, 3))
    f = _finish(dm, layer_idx, xt, o.permute(0, 2, 1, 3))
    return f.cpu().numpy() if was_numpy else f


__all__ = ["BlockWeights", "DeviceModel", "layer_qkv", "layer_finish", "layer_forward"]
