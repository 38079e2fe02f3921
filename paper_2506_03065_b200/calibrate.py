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
    """One layer's candidate evaluation (search.py:334-372) on the GPU."""

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

    def evaluate(self, q, k, v, stripes: dict | None = None) -> LayerEvaluation:
        import torch

        B, H, N, d = _check_qkv(q, k, v)
        (qt, kt, vt), _, dev = _to_device((q, k, v))
        stripes = dict(stripes or {})
        missing = [h for h in range(H) if h not in stripes]
        if missing:
            stripes.update(self.resolve_stripes(qt[..., :d], kt[..., :d], missing))
        layout = self.grid.layout
        pp = self.params.patterns
        cands = {
            "full": [full_spec()] * H,
            "diag": [self._diag] * H,
            "md": [self._md] * H,
            "stripe": [pp.spec_for(Mode.VERTICAL_STRIPE, stripes[h]) for h in range(H)],
        }
        outs = {}
        for name, asg in cands.items():
            o = torch.empty_like(qt)
            plan_for_assignment(asg, layout).forward(qt, kt, vt, o, head_dim=d)
            outs[name] = o[..., :d] if o.shape[-1] != d else o
        full = outs["full"]
        denom = float(B * N * d)
        sq = torch.stack([head_sqdiff(full), head_sqdiff(outs["diag"], full),
                          head_sqdiff(outs["md"], full), head_sqdiff(outs["stripe"], full)], dim=1)
        mse = (sq / denom).cpu().numpy()
        sparsities = np.array([[1.0, self._s_diag, self._s_md, self.stripe_sparsity(stripes[h])]
                               for h in range(H)])
        if self.latency_model is not None:
            # per-head issued-tile counts of each candidate's schedule
            def head_tiles(asg):
                items, _ = plan_for_assignment(asg, layout).schedule()
                t = np.zeros(H)
                np.add.at(t, items[:, 0], 2 * np.maximum(items[:, 3], 0))
                return t

            t_full = head_tiles(cands["full"])
            t_c = [head_tiles(cands[c]) for c in ("diag", "md", "stripe")]
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


__all__ = ["block_key_mass", "head_sqdiff", "top_stripes", "CandidateEvaluator", "LayerEvaluation",
           "SPARSE_MODES"]
