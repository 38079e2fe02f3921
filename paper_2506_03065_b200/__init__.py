"""B200-native Sparse-vDiT attention hot path (drop-in for svdit's operator layer).

Same public names as the reference package's hot path (svdit 0.1.0:
layout / patterns / attention / PatternConfig / cost model); the block grid,
masks, head grouping and kernel schedule are built by a C++ plan builder and
the attention forward is a hand-written sm_100a (tcgen05 / TMEM / TMA)
kernel, both in the in-tree libsvdit_b200.so behind a C ABI
(include/svdit_b200.h).
"""

__version__ = "0.1.0"

from .errors import (
    ConfigError,
    DegenerateMaskError,
    DegenerateRowError,
    FormatError,
    PlantError,
    ShapeError,
    SvditError,
)
from .layout import BlockGrid, RegionKind, TokenLayout, block_grid, classify_region, total_tokens
from .patterns import (
    MODE_NAMES,
    BlockMask,
    Mode,
    PatternParams,
    PatternSpec,
    build_mask,
    default_sparse_specs,
    diagonal_spec,
    frame_period,
    full_spec,
    multi_diagonal_spec,
    skip_spec,
    sparsity,
    vertical_stripe_spec,
    with_stripes,
)
from .attention import (
    HeadGroup,
    LayerPlan,
    block_key_mass,
    dense_attention,
    full_mask_attention,
    fused_layer_attention,
    group_heads,
    host_transfer_bytes,
    plan_for_assignment,
    skip_attention,
    sparse_attention,
)
from .search import (
    SPARSE_MODES,
    PatternConfig,
    SearchParams,
    aggregate_config,
    config_sparsity,
    mode_loss,
    select_mode,
    sparsity_table,
)
from .layer import DeviceModel, layer_finish, layer_forward, layer_qkv
from .costmodel import B200LatencyModel, attention_flops, attention_latency_share, layer_linear_flops

__all__ = [name for name in dir() if not name.startswith("_")]
