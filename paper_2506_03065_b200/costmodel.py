"""FLOP accounting (the reference convention) plus the B200 latency model.

attention_flops / layer_linear_flops / attention_latency_share restate
costmodel.py:26-50 with unchanged signatures and results, so the search's
cost-model plugin surface stays intact.  `B200LatencyModel` is the re-fit
of that model to measured per-pattern latencies of the sm_100a kernel
(BASELINE config 5): it maps (mode, density, N, d, H) -> ms and exposes an
"effective sparsity" 1 - t/t_full that plugs into mode_loss's sparsity slot.
"""

from __future__ import annotations

import json
from dataclasses import dataclass, field
from pathlib import Path

from .errors import ConfigError


def attention_flops(n_tokens: int, head_dim: int, heads: int, sparsity: float) -> float:
    """heads * (1 - sparsity) * 4 * N^2 * d (costmodel.py:26-32)."""
    if n_tokens < 1 or head_dim < 1 or heads < 1:
        raise ConfigError("n_tokens, head_dim, heads must all be >= 1")
    if not 0.0 <= sparsity <= 1.0:
        raise ConfigError(f"sparsity must be in [0, 1], got {sparsity}")
    return heads * (1.0 - sparsity) * 4.0 * float(n_tokens) ** 2 * head_dim


def layer_linear_flops(n_tokens: int, dim: int, ffn_mult: int = 4) -> float:
    """Projections + MLP matmul FLOPs of one block (costmodel.py:35-39)."""
    if n_tokens < 1 or dim < 1 or ffn_mult < 1:
        raise ConfigError("n_tokens, dim, ffn_mult must all be >= 1")
    return 8.0 * n_tokens * float(dim) ** 2 + 4.0 * ffn_mult * n_tokens * float(dim) ** 2


def attention_latency_share(n_tokens: int, head_dim: int, heads: int, ffn_mult: int = 4) -> float:
    """Dense attention's share of per-layer matmul FLOPs (costmodel.py:42-50)."""
    attn = attention_flops(n_tokens, head_dim, heads, 0.0)
    other = layer_linear_flops(n_tokens, heads * head_dim, ffn_mult)
    return attn / (attn + other)


@dataclass
class B200LatencyModel:
    """Measured latency model of the fused sm_100a layer kernel.

    t(ms) = launch_ms + max(tiles * ms_per_tile(d), critical * ms_per_critical_tile(d))
    where `tiles` is the number of 128x128 MMA tiles the plan issues
    (LayerPlan.info.computed_tiles) and `critical` the tiles of its longest
    work item: a launch is either throughput-bound (every SM busy) or bound
    by its longest CTA (forced text/mixed query rows walk every key tile).
    Coefficients come from the BASELINE config-5 sweep
    (scripts/costmodel_sweep.py) and ship in data/b200_latency.json.
    """

    launch_ms: float = 0.01
    ms_per_tile: dict = field(default_factory=lambda: {64: 5.0e-6, 128: 7.4e-6})
    ms_per_critical_tile: dict = field(default_factory=dict)
    source: str = "placeholder (not yet fitted)"

    def predict_ms(self, computed_tiles: int, head_dim: int, critical_tiles: int = 0) -> float:
        per = self.ms_per_tile.get(int(head_dim))
        if per is None:
            raise ConfigError(f"no latency fit for head_dim {head_dim}")
        crit = self.ms_per_critical_tile.get(int(head_dim), 0.0) * critical_tiles
        return self.launch_ms + max(computed_tiles * per, crit)

    def predict_plan_ms(self, plan, head_dim: int) -> float:
        items, _ = plan.schedule()
        crit = int(2 * items[:, 3].max()) if len(items) else 0
        return self.predict_ms(plan.info.computed_tiles, head_dim, crit)

    def effective_sparsity(self, computed_tiles: int, full_tiles: int, head_dim: int) -> float:
        """1 - t(pattern) / t(full) on the throughput term: the latency-weighted
        sparsity that drops into mode_loss's sparsity slot (search.py:65-79).
        Per head: the whole-launch constant launch_ms is left out (it is paid
        once per layer, not per head), and head_dim is the kernel's stored
        width (64 or 128: smaller head dims run zero-padded)."""
        d = 64 if int(head_dim) <= 64 else 128
        per = self.ms_per_tile.get(d)
        if per is None:
            raise ConfigError(f"no latency fit for head_dim {head_dim}")
        if full_tiles <= 0:
            return 0.0
        return min(1.0, max(0.0, 1.0 - (computed_tiles * per) / (full_tiles * per)))

    def save(self, path) -> None:
        Path(path).write_text(json.dumps({
            "launch_ms": self.launch_ms,
            "ms_per_tile": {str(k): v for k, v in self.ms_per_tile.items()},
            "ms_per_critical_tile": {str(k): v for k, v in self.ms_per_critical_tile.items()},
            "source": self.source,
        }, indent=2) + "\n")

    @classmethod
    def default(cls) -> "B200LatencyModel":
        """The fitted model shipped in data/b200_latency.json (config-5 sweep)."""
        path = Path(__file__).resolve().parent / "data" / "b200_latency.json"
        return cls.load(path) if path.exists() else cls()

    @classmethod
    def load(cls, path) -> "B200LatencyModel":
        obj = json.loads(Path(path).read_text())
        return cls(launch_ms=float(obj["launch_ms"]),
                   ms_per_tile={int(k): float(v) for k, v in obj["ms_per_tile"].items()},
                   ms_per_critical_tile={int(k): float(v)
                                         for k, v in obj.get("ms_per_critical_tile", {}).items()},
                   source=obj.get("source", str(path)))
