"""The offline search's per-layer evaluation step on the GPU (SURVEY §8f rows
1 and 2): stripe-column calibration by key-block attention mass, and the
four-candidate loss evaluation that feeds the unchanged Eq. 2 / Eq. 3 plugin
surface (search.py:65-103).

Reference: search.py:334-372 — per (seed, step, layer): FULL output,
SKIP / diagonal / multi-diagonal / per-head-stripe candidates, per-head
mode_loss and select_mode; stripe columns from block_key_mass
(attention.py:108-146) via a stable top-k (search.py:342-346).

Everything runs through the fused sm_100a layer kernel: each candidate is one
launch of the plan for that candidate's per-head specs (the sparse
candidates cost ~3-5% of FULL each), the per-head MSE is an fp64 device
reduction (svd_head_sqdiff), and block_key_mass is its own two-pass
tensor-core kernel (csrc/svd_key_mass.cu).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .attention import _check_qkv, _is_torch, _to_device, plan_for_assignment
from .errors import ShapeError
from .layout import BlockGrid
from .patterns import Mode, full_spec
from .search import SPARSE_MODES, SearchParams, penalized_loss, select_mode


def head_sqdiff(a, b=None):
    """Per-head fp64 sum of squared differences of bf16 [B,H,N,d] CUDA tensors
    (b=None: against zeros).  Returns a CUDA float64 tensor [H]."""
    import torch

    B, H, N, d = a.shape
    out = torch.zeros(H, dtype=torch.float64, device=a.device)
    with torch.cuda.device(a.device):
        nat.check(nat.lib().svd_head_sqdiff(
            nat.c_void_p(a.data_ptr()), nat.c_void_p(b.data_ptr()) if b is not None else None,
            nat.i64x4(a.stride()), nat.i64x4(b.stride() if b is not None else a.stride()), B, H, N, d,
            nat.c_void_p(out.data_ptr()), nat.c_void_p(torch.cuda.current_stream(a.device).cuda_stream)))
    return out


def block_key_mass(q, k, grid: BlockGrid):
    """Per-head attention mass on each key block, [B, H, nb], summing to 1 per
    (batch, head) (attention.py:108-146).  NumPy inputs give a float64 NumPy
    result; CUDA tensors a float64 CUDA tensor.  Computed by
    svd_block_key_mass (csrc/svd_key_mass.cu): a row-statistics pass and a
    per-key-sum pass of QK^T on the tensor cores, then an fp64 block sum."""
    import torch

    for name, t in (("q", q), ("k", k)):
        nd = t.dim() if _is_torch(t) else np.ndim(t)
        if nd != 4:
            raise ShapeError(f"{name} must have rank 4 [B, H, N, d], got rank {nd}")
    if tuple(q.shape) != tuple(k.shape):
        raise ShapeError(f"q and k shapes differ: {tuple(q.shape)} vs {tuple(k.shape)}")
    B, H, N, d = q.shape
    if grid.layout.total_tokens != N:
        raise ShapeError(f"grid covers {grid.layout.total_tokens} tokens, tensors have {N}")
    (qt, kt), was_numpy, dev = _to_device((q, k))
    D = qt.shape[-1]
    nb = grid.n_blocks
    lib = nat.lib()
    ws_bytes = int(lib.svd_key_mass_workspace(B, H, N))
    with torch.cuda.device(dev):
        stream = torch.cuda.current_stream(dev)
        ws = _workspace(dev, stream, ws_bytes)
        mass = torch.empty(B, H, nb, dtype=torch.float64, device=dev)
        nat.check(lib.svd_block_key_mass(
            nat.c_void_p(qt.data_ptr()), nat.c_void_p(kt.data_ptr()), nat.i64x4(qt.stride()),
            nat.i64x4(kt.stride()), B, H, N, d, D, int(grid.layout.block_size), 0,
            nat.c_void_p(ws.data_ptr()), ws_bytes, nat.c_void_p(mass.data_ptr()),
            nat.c_void_p(stream.cuda_stream)))
    if was_numpy:
        return mass.cpu().numpy()
    return mass


def block_key_mass_from_stats(q, k, grid: BlockGrid, row_stats, head_dim: int | None = None):
    """block_key_mass (attention.py:108-146) for bf16 CUDA q, k [B, H, N, D]
    whose row statistics (-m, 1/l) a forward launch already wrote
    (LayerPlan.forward(row_stats=...) on an all-FULL plan): only the key-sum
    pass and the block sum run.  head_dim: the true d when q/k are zero-padded
    to D.  Returns a float64 CUDA tensor [B, H, nb]."""
    import torch

    B, H, N, D = q.shape
    lib = nat.lib()
    ws_bytes = int(lib.svd_key_mass_workspace(B, H, N))
    dev = q.device
    with torch.cuda.device(dev):
        stream = torch.cuda.current_stream(dev)
        ws = _workspace(dev, stream, ws_bytes)
        mass = torch.empty(B, H, grid.n_blocks, dtype=torch.float64, device=dev)
        nat.check(lib.svd_block_key_mass_from_stats(
            nat.c_void_p(q.data_ptr()), nat.c_void_p(k.data_ptr()), nat.i64x4(q.stride()),
            nat.i64x4(k.stride()), B, H, N, int(head_dim or D), D, int(grid.layout.block_size), 0,
            nat.c_void_p(row_stats.data_ptr()), nat.c_void_p(ws.data_ptr()), ws_bytes,
            nat.c_void_p(mass.data_ptr()), nat.c_void_p(stream.cuda_stream)))
    return mass


_WORKSPACES: dict = {}


def _workspace(dev, stream, nbytes: int):
    """A scratch buffer of at least nbytes per (device, stream): calls on one
    stream are ordered, so they can share it (grown, never shrunk)."""
    import torch

    key = (dev.index, stream.cuda_stream)
    buf = _WORKSPACES.get(key)
    if buf is None or buf.numel() < nbytes:
        buf = _WORKSPACES[key] = torch.empty(max(nbytes, 16), dtype=torch.uint8, device=dev)
    return buf


def top_stripes(mass_row: np.ndarray, count: int) -> tuple[int, ...]:
    """The stripe_count heaviest key blocks, stable order, sorted (search.py:344-346)."""
    order = np.argsort(-np.asarray(mass_row, dtype=np.float64), kind="stable")
    return tuple(sorted(int(c) for c in order[:count]))


@dataclass
class LayerEvaluation:
    losses: np.ndarray        # [H, 4] for SKIP, DIAGONAL, MULTI_DIAGONAL, VERTICAL_STRIPE
    sparsities: np.ndarray    # [H, 4]
    mse: np.ndarray           # [H, 4] raw reconstruction errors vs FULL
    choices: list             # [H] Mode
    stripes: dict             # head -> stripe columns used
    selected: object          # [B, H, N, d] bf16 CUDA tensor: the chosen outputs


class CandidateEvaluator:
    """One layer's candidate evaluation (search.py:334-372) on the GPU.

    The four candidates run as ONE launch of the fused layer kernel: its
    plan has 4H heads — (FULL, diagonal, multi-diagonal, stripe) x H, the
    stripe heads with their own columns — all reading the layer's single
    q/k/v through an input head map, heaviest work items first, so the
    sparse candidates' items fill the FULL items' tail instead of paying three
    more launches.  The FULL candidate's launch also writes every row's
    softmax statistics (-m, 1/l), so the stripe calibration
    (block_key_mass, attention.py:108-146) needs only its key-sum pass.

    First evaluation of a layer (stripe columns unknown; the reference
    freezes them there, search.py:338-346): launch 1 = FULL + diagonal +
    multi-diagonal (+ row statistics), key-sum pass -> stripes, launch 2 =
    the stripe candidates.  Every later evaluation (stripes given): one
    launch.  The per-head fp64 MSE is svd_head_sqdiff; mode_loss /
    select_mode are the unchanged reference plugin surface.
    """

    def __init__(self, grid: BlockGrid, params: SearchParams | None = None, latency_model=None):
        """latency_model (a costmodel.B200LatencyModel): when given, the
        penalty uses the B200 "effective sparsity" 1 - t(candidate)/t(full)
        of the fitted per-pattern latency instead of the block sparsity
        (SURVEY §8f row 3); the Eq. 2 / Eq. 3 code path is unchanged."""
        self.grid = grid
        self.params = params or SearchParams()
        self.latency_model = latency_model
        pp = self.params.patterns
        from .patterns import build_mask

        self._diag = pp.spec_for(Mode.DIAGONAL)
        self._md = pp.spec_for(Mode.MULTI_DIAGONAL)
        self._s_diag = build_mask(self._diag, grid).sparsity
        self._s_md = build_mask(self._md, grid).sparsity
        self._s_stripe: dict = {}
        self._maps: dict = {}

    def stripe_sparsity(self, cols) -> float:
        from .patterns import build_mask

        if cols not in self._s_stripe:
            spec = self.params.patterns.spec_for(Mode.VERTICAL_STRIPE, cols)
            self._s_stripe[cols] = build_mask(spec, self.grid).sparsity
        return self._s_stripe[cols]

    def resolve_stripes(self, q, k, heads) -> dict:
        """Stripe columns for the listed heads from block_key_mass (batch 0;
        search.py:340-346).  Heads are independent, so only the listed heads'
        masses are computed."""
        heads = list(heads)
        if not heads:
            return {}
        if len(heads) < q.shape[1]:
            q, k = q[:, heads], k[:, heads]
        mass = block_key_mass(q, k, self.grid)
        m0 = mass[0].double().cpu().numpy() if _is_torch(mass) else mass[0]
        return {h: top_stripes(m0[i], self.params.patterns.stripe_count) for i, h in enumerate(heads)}

    def _stripe_specs(self, stripes, H):
        pp = self.params.patterns
        return [pp.spec_for(Mode.VERTICAL_STRIPE, stripes[h]) for h in range(H)]

    def _in_map(self, dev, H: int, copies: int):
        import torch

        key = (dev.index, H, copies)
        if key not in self._maps:
            self._maps[key] = torch.arange(H, dtype=torch.int32, device=dev).repeat(copies)
        return self._maps[key]

    def _launch(self, asg, qt, kt, vt, d, copies, row_stats=None):
        """One launch of the candidate plan `asg` (copies x H heads over the
        H heads of qt/kt/vt) -> [B, copies * H, N, D] bf16."""
        import torch

        B, H, N, D = qt.shape
        out = torch.empty(B, copies * H, N, D, dtype=torch.bfloat16, device=qt.device)
        plan = plan_for_assignment(asg, self.grid.layout)
        in_map = self._in_map(qt.device, H, copies) if copies > 1 else None
        plan.forward(qt, kt, vt, out, head_dim=d, in_head_map=in_map, row_stats=row_stats,
                     stats_heads=H if row_stats is not None else 0)
        return out

    def evaluate(self, q, k, v, stripes: dict | None = None) -> LayerEvaluation:
        import torch

        B, H, N, d = _check_qkv(q, k, v)
        (qt, kt, vt), _, dev = _to_device((q, k, v))
        D = qt.shape[-1]
        stripes = dict(stripes or {})
        missing = [h for h in range(H) if h not in stripes]
        fulls, diags, mds = [full_spec()] * H, [self._diag] * H, [self._md] * H
        if missing:
            # launch 1: FULL + diagonal + multi-diagonal, FULL rows' statistics
            T = (N + 127) // 128
            stats = torch.empty(B * H, T, 2, 128, dtype=torch.float32, device=dev)
            stats[:, :, 0].fill_(float("-inf"))
            stats[:, :, 1].zero_()
            o3 = self._launch(fulls + diags + mds, qt, kt, vt, d, 3, row_stats=stats)
            mass = block_key_mass_from_stats(qt, kt, self.grid, stats, head_dim=d)
            m0 = mass[0].double().cpu().numpy()
            for h in missing:
                stripes[h] = top_stripes(m0[h], self.params.patterns.stripe_count)
            o_st = self._launch(self._stripe_specs(stripes, H), qt, kt, vt, d, 1)
            outs = {"full": o3[:, :H], "diag": o3[:, H:2 * H], "md": o3[:, 2 * H:], "stripe": o_st}
        else:
            o4 = self._launch(fulls + diags + mds + self._stripe_specs(stripes, H), qt, kt, vt, d, 4)
            outs = {"full": o4[:, :H], "diag": o4[:, H:2 * H], "md": o4[:, 2 * H:3 * H],
                    "stripe": o4[:, 3 * H:]}
        if D != d:
            outs = {c: o[..., :d] for c, o in outs.items()}
        full = outs["full"]
        denom = float(B * N * d)
        sq = torch.stack([head_sqdiff(full), head_sqdiff(outs["diag"], full),
                          head_sqdiff(outs["md"], full), head_sqdiff(outs["stripe"], full)], dim=1)
        mse = (sq / denom).cpu().numpy()
        sparsities = np.array([[1.0, self._s_diag, self._s_md, self.stripe_sparsity(stripes[h])]
                               for h in range(H)])
        if self.latency_model is not None:
            layout = self.grid.layout

            # per-head issued-tile counts of each candidate's schedule
            def head_tiles(asg):
                items, _ = plan_for_assignment(asg, layout).schedule()
                t = np.zeros(H)
                np.add.at(t, items[:, 0], 2 * np.maximum(items[:, 3], 0))
                return t

            t_full = head_tiles(fulls)
            t_c = [head_tiles(c) for c in (diags, mds, self._stripe_specs(stripes, H))]
            lm = self.latency_model
            for h in range(H):
                for ci, tc in enumerate(t_c):
                    sparsities[h, ci + 1] = lm.effective_sparsity(int(tc[h]), int(t_full[h]), d)
        losses = np.array([[penalized_loss(float(mse[h, c]), float(sparsities[h, c]), self.params.lam,
                                           self.params.penalty) for c in range(4)] for h in range(H)])
        choices = [select_mode(losses[h], sparsities[h], self.params.epsilon) for h in range(H)]
        sel = torch.empty_like(full)
        pick = {Mode.FULL: full, Mode.SKIP: None, Mode.DIAGONAL: outs["diag"],
                Mode.MULTI_DIAGONAL: outs["md"], Mode.VERTICAL_STRIPE: outs["stripe"]}
        for h, ch in enumerate(choices):
            src = pick[ch]
            if src is None:
                sel[:, h].zero_()
            else:
                sel[:, h] = src[:, h]
        return LayerEvaluation(losses=losses, sparsities=sparsities, mse=mse, choices=choices,
                               stripes=stripes, selected=sel)


__all__ = ["block_key_mass", "block_key_mass_from_stats", "head_sqdiff", "top_stripes", "CandidateEvaluator", "LayerEvaluation",
           "SPARSE_MODES"]
