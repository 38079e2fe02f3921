"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

A NumPy restatement of the reference's hot path (svdit 0.1.0 under
/root/reference/pkg/src/svdit), used as the checker in tests/, by
__graft_entry__.smoke() and as bench.py's cpu_baseline / --impl reference
arm.  It is never imported by the product package; the product path has no
CPU fallback.

Parity pinning: every integer function here (grid, masks, grouping) and the
streaming attention are checked against golden vectors produced by the
reference itself (tests/golden/make_golden.py imports /root/reference and
writes tests/golden/*.npz; tests/test_oracle_golden.py compares).

Each function cites the reference file:line it restates.
"""

from __future__ import annotations

from typing import NamedTuple

import numpy as np

FULL, SKIP, DIAGONAL, MULTI_DIAGONAL, VERTICAL_STRIPE = range(5)


# ------------------------------------------------------------------ RNG
def _mix64(state: int, word: int) -> int:
    """One splitmix64 fold (numerics.py:24-29)."""
    z = (state + 0x9E3779B97F4A7C15 + word) & 0xFFFFFFFFFFFFFFFF
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & 0xFFFFFFFFFFFFFFFF
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & 0xFFFFFFFFFFFFFFFF
    return z ^ (z >> 31)


def make_rng(seed: int, *stream: int) -> np.random.Generator:
    """Philox keyed by (seed, splitmix-folded stream) (numerics.py:32-43)."""
    sub = 0
    for word in stream:
        sub = _mix64(sub, int(word))
    key = np.array([int(seed) & 0xFFFFFFFFFFFFFFFF, sub], dtype=np.uint64)
    return np.random.Generator(np.random.Philox(key=key))


def random_qkv(seed: int, b: int, h: int, n: int, d: int):
    """Standard-normal q, k, v in that order from make_rng(seed, 999)
    (reference tests/conftest.py:61-66)."""
    rng = make_rng(seed, 999)
    q = rng.standard_normal((b, h, n, d)).astype(np.float32)
    k = rng.standard_normal((b, h, n, d)).astype(np.float32)
    v = rng.standard_normal((b, h, n, d)).astype(np.float32)
    return q, k, v


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round float32 to the nearest bf16 (ties to even), returned as float32."""
    a = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    rounded = (a + 0x7FFF + ((a >> 16) & 1)) & 0xFFFF0000
    return rounded.astype(np.uint32).view(np.float32)


# ------------------------------------------------------------------ layout
class Grid(NamedTuple):
    n: int
    bounds: np.ndarray
    has_text: np.ndarray
    mixed: np.ndarray
    frame_index: np.ndarray
    tokens_per_frame: int
    block_size: int

    @property
    def n_blocks(self) -> int:
        return len(self.bounds) - 1

    @property
    def forced(self) -> np.ndarray:
        return self.has_text | self.mixed  # layout.py:119-122


def block_grid(text: int, frames: int, tpf: int, block: int = 64) -> Grid:
    """layout.py:135-158 (validation layout.py:33-43 is the caller's job)."""
    n = text + frames * tpf
    nb = -(-n // block)
    bounds = np.minimum(np.arange(nb + 1, dtype=np.int64) * block, n)
    has_text = np.zeros(nb, dtype=bool)
    mixed = np.zeros(nb, dtype=bool)
    frame_index = np.full(nb, -1, dtype=np.int64)

    def frame_of(t):  # layout.py:57-63
        return -1 if t < text else (t - text) // tpf

    for b in range(nb):
        t0, t1 = int(bounds[b]), int(bounds[b + 1])
        has_text[b] = t0 < text
        first_video = max(t0, text)
        if first_video < t1:
            frame_index[b] = frame_of(first_video)
            mixed[b] = (t0 < text) or (frame_of(t1 - 1) != frame_index[b])
    return Grid(n, bounds, has_text, mixed, frame_index, tpf, block)


def frame_period(grid: Grid) -> int:
    """patterns.py:176-181: max(1, round(tpf / block)), Python round = half-even."""
    return max(1, round(grid.tokens_per_frame / grid.block_size))


# ------------------------------------------------------------------ specs
class Spec(NamedTuple):
    """PatternSpec's fields and defaults (patterns.py:50-66); enough for
    build_mask / group_heads here.  Stripes are kept sorted and unique like
    PatternSpec.__post_init__ (patterns.py:67-75)."""

    mode: int
    halfwidth: int = 1
    period: int | None = None
    md_halfwidth: int = 0
    stripe_count: int = 2
    stripes: tuple | None = None
    include_diagonal: bool = True


def full_spec() -> Spec:  # patterns.py:106-107
    return Spec(FULL)


def skip_spec() -> Spec:  # patterns.py:110-111
    return Spec(SKIP)


def diagonal_spec(halfwidth: int = 1) -> Spec:  # patterns.py:114-115
    return Spec(DIAGONAL, halfwidth=halfwidth)


def multi_diagonal_spec(period: int | None = None, md_halfwidth: int = 0) -> Spec:  # patterns.py:118-119
    return Spec(MULTI_DIAGONAL, period=period, md_halfwidth=md_halfwidth)


def vertical_stripe_spec(stripe_count: int = 2, stripes=None, include_diagonal: bool = True) -> Spec:
    """patterns.py:122-132."""
    return Spec(VERTICAL_STRIPE, stripe_count=stripe_count,
                stripes=None if stripes is None else tuple(sorted(set(int(s) for s in stripes))),
                include_diagonal=include_diagonal)


# ------------------------------------------------------------------ masks
def spec_key(spec) -> tuple:
    """PatternSpec equality key (all dataclass fields, patterns.py:50-75)."""
    stripes = None if spec.stripes is None else tuple(sorted(set(int(s) for s in spec.stripes)))
    return (int(spec.mode), int(spec.halfwidth), spec.period, int(spec.md_halfwidth),
            int(spec.stripe_count), stripes, bool(spec.include_diagonal))


class OracleError(Exception):
    def __init__(self, kind: str, msg: str):
        super().__init__(msg)
        self.kind = kind  # "config" | "degenerate_mask" | "degenerate_row" | "shape"


def build_mask(spec, grid: Grid):
    """patterns.py:219-259.  Returns None for SKIP, else bool [nb, nb]."""
    nb = grid.n_blocks
    mode = int(spec.mode)
    if mode == SKIP:
        return None
    if mode == FULL:
        return np.ones((nb, nb), dtype=bool)
    idx = np.arange(nb)
    offset = idx[:, None] - idx[None, :]
    if mode == DIAGONAL:
        active = np.abs(offset) <= spec.halfwidth
    elif mode == MULTI_DIAGONAL:
        period = spec.period if spec.period is not None else frame_period(grid)
        folded = np.abs(offset) % period
        active = (folded <= spec.md_halfwidth) | (period - folded <= spec.md_halfwidth)
    else:
        if spec.stripes is None:
            raise OracleError("config", "vertical-stripe spec has no resolved stripe columns")
        active = np.zeros((nb, nb), dtype=bool)
        for col in sorted(set(int(s) for s in spec.stripes)):
            if not 0 <= col < nb:
                raise OracleError("config", f"stripe column {col} outside grid of {nb} blocks")
            active[:, col] = True
        if spec.include_diagonal:
            active |= offset == 0
    forced = grid.forced
    active[forced, :] = True
    active[:, forced] = True
    if not active.any(axis=1).all():
        raise OracleError("degenerate_mask", "query block has no active key blocks")
    return active


def active_key_blocks(active: np.ndarray, qb: int) -> np.ndarray:
    """patterns.py:205-208."""
    return np.flatnonzero(active[qb])


def token_mask(active: np.ndarray, grid: Grid) -> np.ndarray:
    """patterns.py:210-216."""
    sizes = np.diff(grid.bounds)
    return np.repeat(np.repeat(active, sizes, axis=0), sizes, axis=1)


def group_heads(assignment, grid: Grid):
    """attention.py:164-183: [(spec, heads tuple, mask-or-None)] in first-
    occurrence order; masks only for non-FULL/SKIP groups."""
    order, members, first = [], {}, {}
    for h, spec in enumerate(assignment):
        key = spec_key(spec)
        if key not in members:
            members[key] = []
            first[key] = spec
            order.append(key)
        members[key].append(h)
    groups = []
    for key in order:
        spec = first[key]
        mask = None
        if int(spec.mode) not in (FULL, SKIP):
            mask = build_mask(spec, grid)
        groups.append((spec, tuple(members[key]), mask))
    return groups


# ------------------------------------------------------------------ attention
def sparse_attention(q, k, v, active: np.ndarray, bounds: np.ndarray) -> np.ndarray:
    """attention.py:57-98: per query block, online softmax over its active key
    blocks in ascending order, fp64 accumulation, fp32 result."""
    q = np.asarray(q, dtype=np.float32)
    B, H, N, d = q.shape
    if not active.any(axis=1).all():
        raise OracleError("degenerate_row", "mask has a query row with no active key blocks")
    scale = 1.0 / np.sqrt(d)
    q64 = q.astype(np.float64)
    k64 = np.asarray(k, dtype=np.float32).astype(np.float64)
    v64 = np.asarray(v, dtype=np.float32).astype(np.float64)
    out = np.empty_like(q)
    nb = len(bounds) - 1
    for qb in range(nb):
        r0, r1 = int(bounds[qb]), int(bounds[qb + 1])
        rows = r1 - r0
        m = np.full((B, H, rows), -np.inf)
        l = np.zeros((B, H, rows))
        acc = np.zeros((B, H, rows, d))
        for kb in np.flatnonzero(active[qb]):
            c0, c1 = int(bounds[kb]), int(bounds[kb + 1])
            s = np.matmul(q64[:, :, r0:r1], k64[:, :, c0:c1].swapaxes(-1, -2))
            s *= scale
            m_new = np.maximum(m, s.max(axis=-1))
            p = np.exp(s - m_new[..., None])
            alpha = np.exp(m - m_new)
            l = l * alpha + p.sum(axis=-1)
            acc = acc * alpha[..., None] + np.matmul(p, v64[:, :, c0:c1])
            m = m_new
        out[:, :, r0:r1] = (acc / l[..., None]).astype(np.float32)
    if not np.isfinite(out).all():
        raise OracleError("shape", "non-finite values in attention output")
    return out


def sparse_attention_rows(q, k, v, active, bounds, qblocks) -> np.ndarray:
    """The same recurrence restricted to the listed query blocks (for bounded
    CPU-baseline samples at full N).  Returns [B, H, sum rows, d]."""
    B, H, N, d = q.shape
    scale = 1.0 / np.sqrt(d)
    outs = []
    for qb in qblocks:
        r0, r1 = int(bounds[qb]), int(bounds[qb + 1])
        q64 = q[:, :, r0:r1].astype(np.float64)
        m = np.full((B, H, r1 - r0), -np.inf)
        l = np.zeros((B, H, r1 - r0))
        acc = np.zeros((B, H, r1 - r0, d))
        for kb in np.flatnonzero(active[qb]):
            c0, c1 = int(bounds[kb]), int(bounds[kb + 1])
            s = np.matmul(q64, k[:, :, c0:c1].astype(np.float64).swapaxes(-1, -2)) * scale
            m_new = np.maximum(m, s.max(axis=-1))
            p = np.exp(s - m_new[..., None])
            alpha = np.exp(m - m_new)
            l = l * alpha + p.sum(axis=-1)
            acc = acc * alpha[..., None] + np.matmul(p, v[:, :, c0:c1].astype(np.float64))
            m = m_new
        outs.append((acc / l[..., None]).astype(np.float32))
    return np.concatenate(outs, axis=2)


def attention_rows(q, k, v, active, bounds, qblocks) -> np.ndarray:
    """Output rows of the listed query blocks in one shot per block: the
    softmax over the block's active key tokens (ascending, as
    active_key_blocks lists them) in fp64 — the quantity attention.py:57-98's
    streaming recurrence computes (it differs only by fp64 rounding, the
    reference's own dense oracle tests/conftest.py:49-58 makes the same
    comparison).  q, k, v: [B, H, N, d]; returns [B, H, sum rows, d] fp32."""
    B, H, N, d = q.shape
    scale = 1.0 / np.sqrt(d)
    sizes = np.diff(bounds)
    kall = np.asarray(k, dtype=np.float64)
    vall = np.asarray(v, dtype=np.float64)
    outs = []
    for qb in qblocks:
        r0, r1 = int(bounds[qb]), int(bounds[qb + 1])
        kbs = np.flatnonzero(active[qb])
        q64 = np.asarray(q[:, :, r0:r1], dtype=np.float64)
        if len(kbs) == len(sizes):  # every key block active (forced rows, FULL heads)
            k64, v64 = kall, vall
        else:
            cols = np.concatenate([np.arange(bounds[c], bounds[c] + sizes[c]) for c in kbs])
            k64, v64 = kall[:, :, cols], vall[:, :, cols]
        s = np.matmul(q64, k64.swapaxes(-1, -2)) * scale
        s -= s.max(axis=-1, keepdims=True)
        p = np.exp(s)
        outs.append((np.matmul(p, v64) / p.sum(axis=-1, keepdims=True)).astype(np.float32))
    return np.concatenate(outs, axis=2)


def block_key_mass(q, k, grid: Grid) -> np.ndarray:
    """attention.py:108-146: per-head attention mass on each key block,
    streamed with the online-softmax recurrence, / N.  [B, H, nb] float64."""
    q = np.asarray(q, dtype=np.float32)
    B, H, N, d = q.shape
    scale = 1.0 / np.sqrt(d)
    bounds = grid.bounds
    nb = len(bounds) - 1
    q64 = q.astype(np.float64)
    k64 = np.asarray(k, dtype=np.float32).astype(np.float64)
    mass = np.zeros((B, H, nb))
    for qb in range(nb):
        r0, r1 = int(bounds[qb]), int(bounds[qb + 1])
        rows = r1 - r0
        m = np.full((B, H, rows), -np.inf)
        l = np.zeros((B, H, rows))
        partial = np.zeros((B, H, rows, nb))
        for kb in range(nb):
            c0, c1 = int(bounds[kb]), int(bounds[kb + 1])
            s = np.matmul(q64[:, :, r0:r1], k64[:, :, c0:c1].swapaxes(-1, -2)) * scale
            m_new = np.maximum(m, s.max(axis=-1))
            p = np.exp(s - m_new[..., None])
            alpha = np.exp(m - m_new)
            block_total = p.sum(axis=-1)
            l = l * alpha + block_total
            partial *= alpha[..., None]
            partial[:, :, :, kb] = block_total
            m = m_new
        mass += (partial / l[..., None]).sum(axis=2)
    return mass / N


def mse(a, b) -> float:
    """numerics.py:114-121: fp64 mean squared difference."""
    diff = np.asarray(a, dtype=np.float64) - np.asarray(b, dtype=np.float64)
    return float(np.mean(diff * diff)) if diff.size else 0.0


def full_mask_attention(q, k, v, grid: Grid) -> np.ndarray:
    """attention.py:101-105."""
    nb = grid.n_blocks
    return sparse_attention(q, k, v, np.ones((nb, nb), dtype=bool), grid.bounds)


def skip_attention(q, k, v) -> np.ndarray:
    """attention.py:51-54."""
    return np.zeros_like(np.asarray(q, dtype=np.float32))


def masked_dense_attention(q, k, v, tmask: np.ndarray) -> np.ndarray:
    """Dense fp64 oracle with -inf outside the token mask (tests/conftest.py:49-58)."""
    d = q.shape[-1]
    scores = np.matmul(q.astype(np.float64), k.astype(np.float64).swapaxes(-1, -2)) / np.sqrt(d)
    scores = np.where(tmask[None, None], scores, -np.inf)
    m = scores.max(axis=-1, keepdims=True)
    p = np.exp(scores - m)
    p /= p.sum(axis=-1, keepdims=True)
    return np.matmul(p, v.astype(np.float64)).astype(np.float32)


def fused_layer_attention(q, k, v, groups, grid: Grid) -> np.ndarray:
    """attention.py:186-212 with FULL groups on the streaming path
    (full_mask_attention, which the reference's dense path matches to ~3e-8)."""
    out = np.empty_like(np.asarray(q, dtype=np.float32))
    for spec, heads, mask in groups:
        idx = list(heads)
        qs, ks, vs = q[:, idx], k[:, idx], v[:, idx]
        mode = int(spec.mode)
        if mode == FULL:
            res = full_mask_attention(qs, ks, vs, grid)
        elif mode == SKIP:
            res = skip_attention(qs, ks, vs)
        else:
            res = sparse_attention(qs, ks, vs, mask, grid.bounds)
        out[:, idx] = res
    return out


def active_pairs(active: np.ndarray, bounds: np.ndarray) -> float:
    """Sum over active (qb, kb) of |qb|*|kb| (FLOPs = 4*d*this, costmodel.py:26-32)."""
    sizes = np.diff(bounds).astype(np.float64)
    return float(sizes @ active.astype(np.float64) @ sizes)


# ------------------------------------------------------------------ the block around the operator
# (layer_qkv / layer_finish, the steps either side of the
# attention call in model.layer_forward, model.py:405-420)
ROPE_BASE = 10000.0  # model.py:39


def layer_weights(seed: int, layer: int, heads: int, head_dim: int, ffn_mult: int = 4) -> dict:
    """wq, wk, wv, wo, w1, w2 of one layer, drawn like build_model
    (model.py:312-324: make_rng(seed, 1, layer, slot), N(0,1)/sqrt(rows), fp32)."""
    dim = heads * head_dim
    hidden = ffn_mult * dim
    shapes = {"wq": (dim, dim), "wk": (dim, dim), "wv": (dim, dim), "wo": (dim, dim),
              "w1": (dim, hidden), "w2": (hidden, dim)}
    out = {}
    for slot, (name, (rows, cols)) in enumerate(shapes.items()):
        rng = make_rng(seed, 1, layer, slot)
        out[name] = (rng.standard_normal((rows, cols)) / np.sqrt(rows)).astype(np.float32)
    return out


def zero_redundant_heads(w: dict, heads, head_dim: int) -> dict:
    """A "redundant" plant zeroes the head's value and output paths
    (model.py:346-348)."""
    for h in heads:
        w["wv"][:, h * head_dim:(h + 1) * head_dim] = 0.0
        w["wo"][h * head_dim:(h + 1) * head_dim, :] = 0.0
    return w


def layernorm(x64: np.ndarray) -> np.ndarray:
    """model.py:352-355 (no affine, eps 1e-5, biased variance, fp64)."""
    mean = x64.mean(axis=-1, keepdims=True)
    var = x64.var(axis=-1, keepdims=True)
    return (x64 - mean) / np.sqrt(var + 1e-5)


def gelu(x64: np.ndarray) -> np.ndarray:
    """model.py:357-359, exact erf GELU."""
    from math import erf, sqrt

    return 0.5 * x64 * (1.0 + np.vectorize(erf)(x64 / sqrt(2.0)))


def rope(x: np.ndarray) -> np.ndarray:
    """model.py:169-195: pair (2c, 2c+1) rotated by n * base^(-2c/d), fp64, fp32 out."""
    d, n = x.shape[-1], x.shape[-2]
    theta = ROPE_BASE ** (-2.0 * np.arange(d // 2) / d)
    ang = np.arange(n, dtype=np.float64)[:, None] * theta[None, :]
    cos, sin = np.cos(ang), np.sin(ang)
    x64 = x.astype(np.float64)
    even, odd = x64[..., 0::2], x64[..., 1::2]
    out = np.empty_like(x64)
    out[..., 0::2] = even * cos - odd * sin
    out[..., 1::2] = even * sin + odd * cos
    return out.astype(np.float32)


def split_heads(x: np.ndarray, heads: int) -> np.ndarray:
    """model.py:362-364: [B, N, D] -> [B, H, N, d]."""
    b, n, dim = x.shape
    return x.reshape(b, n, heads, dim // heads).transpose(0, 2, 1, 3)


def merge_heads(x: np.ndarray) -> np.ndarray:
    """model.py:367-369: [B, H, N, d] -> [B, N, D]."""
    b, h, n, d = x.shape
    return x.transpose(0, 2, 1, 3).reshape(b, n, h * d)


def layer_qkv(w: dict, x: np.ndarray, heads: int, planted_q=None, planted_k=None):
    """model.py:372-391: LN -> fp64 projections -> fp32 heads -> RoPE(q, k);
    planted heads' q/k replaced by their stored codes after RoPE."""
    h64 = layernorm(np.asarray(x, dtype=np.float64))
    q = split_heads((h64 @ w["wq"].astype(np.float64)).astype(np.float32), heads)
    k = split_heads((h64 @ w["wk"].astype(np.float64)).astype(np.float32), heads)
    v = split_heads((h64 @ w["wv"].astype(np.float64)).astype(np.float32), heads)
    q, k = rope(q), rope(k)
    for head, code in (planted_q or {}).items():
        q[:, head] = code[None]
    for head, code in (planted_k or {}).items():
        k[:, head] = code[None]
    return q, k, v


def layer_finish(w: dict, x: np.ndarray, attn_out: np.ndarray) -> np.ndarray:
    """model.py:394-402: x + merge(attn) Wo, then + GELU(LN(.) W1) W2 (fp64, fp32 out)."""
    x64 = np.asarray(x, dtype=np.float64)
    a = x64 + merge_heads(np.asarray(attn_out, dtype=np.float64)) @ w["wo"].astype(np.float64)
    f = a + gelu(layernorm(a) @ w["w1"].astype(np.float64)) @ w["w2"].astype(np.float64)
    return f.astype(np.float32)
