"""Attention operators — the reference API of attention.py, executed by the
native plan (C++) and the sm_100a forward kernel.

Mirrors: _check_qkv (attention.py:27-33), dense_attention (:36-41),
skip_attention (:51-54), sparse_attention (:57-98), full_mask_attention
(:101-105), HeadGroup (:149-161), group_heads (:164-183),
fused_layer_attention (:186-212).

Tensor contract.  Inputs are rank-4 [B, H, N, d].  CUDA torch tensors run
in place (bf16 is used as is; other float dtypes are cast to bf16) and the
result is a bf16 CUDA tensor.  CPU torch tensors (ideally pinned bf16) are
streamed through the GPU in head chunks with copy-in / compute / copy-out
overlapped, and the result is a pinned CPU bf16 tensor.  NumPy inputs (the
reference's own type) are moved to the current CUDA device, computed in bf16
and returned as float32 NumPy arrays.  There is no CPU compute path: without a CUDA device the
attention operators raise.
"""

from __future__ import annotations

import weakref
from collections import OrderedDict
from dataclasses import dataclass, field

import numpy as np

from . import _native as nat
from .errors import ConfigError, DegenerateRowError, ShapeError
from .layout import BlockGrid, TokenLayout
from .patterns import BlockMask, Mode, PatternSpec, full_spec, skip_spec

# ---------------------------------------------------------------- native plan


class LayerPlan:
    """One layer's head->pattern assignment lowered to the kernel schedule.

    Wraps an immutable native svd_plan: reference-exact grouping and masks
    plus the work items / KV tile lists the forward kernel consumes.
    """

    def __init__(self, handle: int, layout: TokenLayout, n_heads: int, sharded: bool = False):
        self._handle = nat.c_void_p(handle)
        self.layout = layout
        self.n_heads = n_heads
        self.sharded = sharded
        self._dev_rows = None
        self._finalizer = weakref.finalize(self, nat.lib().svd_plan_destroy, nat.c_void_p(handle))

    # -- construction
    @classmethod
    def from_specs(cls, assignment, layout: TokenLayout) -> "LayerPlan":
        keep: list = []
        n = len(assignment)
        if n < 1:
            raise ConfigError("assignment must name at least one head")
        specs = (nat.SvdSpec * n)(*[nat.make_spec(s, keep) for s in assignment])
        out = nat.c_void_p()
        nat.check(nat.lib().svd_plan_create(nat.make_layout(layout), specs, n, nat.ctypes.byref(out)))
        return cls(out.value, layout, n)

    @classmethod
    def from_masks(cls, layout: TokenLayout, group_masks, head_group) -> "LayerPlan":
        """group_masks: list of bool [nb, nb] arrays or None (SKIP)."""
        nb = layout.n_blocks
        ng = len(group_masks)
        masks = np.ones((ng, nb, nb), dtype=np.uint8)
        skip = np.zeros(ng, dtype=np.int32)
        for g, m in enumerate(group_masks):
            if m is None:
                skip[g] = 1
            else:
                masks[g] = np.asarray(m, dtype=bool)
        hg = np.ascontiguousarray(np.asarray(head_group, dtype=np.int32))
        out = nat.c_void_p()
        nat.check(nat.lib().svd_plan_create_from_masks(
            nat.make_layout(layout), ng, nat.ptr(skip), nat.ptr(masks), nat.ptr(hg), int(hg.size),
            nat.ctypes.byref(out)))
        return cls(out.value, layout, int(hg.size))

    def head_subplan(self, h0: int, h1: int) -> "LayerPlan":
        """The plan restricted to heads [h0, h1) (cached): lets host-resident
        layers be pipelined head-chunk by head-chunk."""
        return self.heads_subplan(tuple(range(h0, h1)))

    def heads_subplan(self, heads: tuple) -> "LayerPlan":
        """The plan restricted to the listed heads, in that order (cached)."""
        cache = self.__dict__.setdefault("_subplans", {})
        heads = tuple(int(h) for h in heads)
        if heads not in cache:
            if self.sharded:
                raise ConfigError("a shard plan cannot be split by heads")
            arr = np.ascontiguousarray(np.asarray(heads, dtype=np.int32))
            out = nat.c_void_p()
            nat.check(nat.lib().svd_plan_subset(self._handle, nat.ptr(arr), int(arr.size), nat.ctypes.byref(out)))
            cache[heads] = LayerPlan(out.value, self.layout, len(heads))
        return cache[heads]

    # -- queries
    @property
    def handle(self) -> nat.c_void_p:
        return self._handle

    @property
    def info(self) -> nat.SvdPlanInfo:
        info = nat.SvdPlanInfo()
        nat.check(nat.lib().svd_plan_get_info(self._handle, nat.ctypes.byref(info)))
        return info

    def group_heads(self, g: int) -> tuple[tuple[int, ...], bool]:
        n = nat.c_int32(0)
        skip = nat.c_int32(0)
        nat.check(nat.lib().svd_plan_group_heads(self._handle, g, None, nat.ctypes.byref(n),
                                                 nat.ctypes.byref(skip)))
        heads = np.empty(n.value, dtype=np.int32)
        nat.check(nat.lib().svd_plan_group_heads(self._handle, g, nat.ptr(heads),
                                                 nat.ctypes.byref(n), nat.ctypes.byref(skip)))
        return tuple(int(h) for h in heads), bool(skip.value)

    def skip_heads(self) -> tuple[int, ...]:
        """Heads of SKIP groups (exact zeros: no inputs read, no kernel work)."""
        cache = self.__dict__.setdefault("_skip_heads", [])
        if not cache:
            hs = []
            for g in range(self.info.n_groups):
                heads, skip = self.group_heads(g)
                if skip:
                    hs.extend(heads)
            cache.append(tuple(sorted(hs)))
        return cache[0]

    def group_mask(self, g: int) -> np.ndarray:
        nb = self.layout.n_blocks
        active = np.empty((nb, nb), dtype=np.uint8)
        nat.check(nat.lib().svd_plan_group_mask(self._handle, g, nat.ptr(active)))
        return active.view(bool)

    def group_csr(self, g: int) -> tuple[np.ndarray, np.ndarray]:
        nnz = nat.c_int64(0)
        nat.check(nat.lib().svd_plan_group_nnz(self._handle, g, nat.ctypes.byref(nnz)))
        row_ptr = np.empty(self.layout.n_blocks + 1, dtype=np.int64)
        col_idx = np.empty(max(nnz.value, 1), dtype=np.int64)
        nat.check(nat.lib().svd_plan_group_csr(self._handle, g, nat.ptr(row_ptr), nat.ptr(col_idx)))
        return row_ptr, col_idx[: nnz.value]

    def schedule(self) -> tuple[np.ndarray, np.ndarray]:
        """The kernel schedule: items [n, 12] int32 and KV tiles [m, 4] int32."""
        info = self.info
        items = np.zeros((max(info.n_work_items, 1), 12), dtype=np.int32)
        kv = np.zeros((max(info.n_kv_entries, 1), 4), dtype=np.int32)
        nat.check(nat.lib().svd_plan_schedule(self._handle, nat.ptr(items), nat.ptr(kv)))
        return items[: info.n_work_items], kv[: info.n_kv_entries]

    def active_flops(self, head_dim: int) -> float:
        """costmodel.py:26-32 convention: 4 * d * sum of active (qb, kb) token pairs."""
        return 4.0 * head_dim * self.info.active_pairs

    def dense_flops(self, head_dim: int) -> float:
        return 4.0 * head_dim * self.info.dense_pairs

    # -- multi-GPU
    def shard(self, world: int, rank: int, n_sms: int | None = None, max_item_tiles: int = 0,
              partition: str = "items") -> "LayerPlan":
        """This rank's share of the work items, with items longer than
        max_item_tiles KV tiles split along the KV list and merged in the
        kernel (0: chosen by simulating every rank's SM packing on n_sms SMs —
        the current device's count, 148 on B200; < 0: never split).
        partition "items": LPT over all items; "heads": contiguous head ranges
        of equal cost (a rank reads only its own heads' Q/K/V)."""
        if n_sms is None:
            n_sms = _device_sm_count()
        part = {"items": 0, "heads": 1}.get(partition)
        if part is None:
            raise ConfigError(f"unknown partition {partition!r} (items | heads)")
        out = nat.c_void_p()
        nat.check(nat.lib().svd_plan_shard_ex(self._handle, world, rank, int(n_sms), int(max_item_tiles), part,
                                              nat.ctypes.byref(out)))
        return LayerPlan(out.value, self.layout, self.n_heads, sharded=True)

    def shard_subset(self, heads) -> "LayerPlan":
        """The items of this shard plan that belong to `heads` (a shard plan
        with the same packed row layout): one chunk of a pipelined step."""
        arr = np.ascontiguousarray(np.asarray(heads, dtype=np.int32))
        out = nat.c_void_p()
        nat.check(nat.lib().svd_plan_shard_heads(self._handle, nat.ptr(arr), int(arr.size), nat.ctypes.byref(out)))
        return LayerPlan(out.value, self.layout, self.n_heads, sharded=True)

    def shard_heads(self) -> tuple[int, ...]:
        """Heads this shard's items touch (ascending)."""
        items, _ = self.schedule()
        return tuple(sorted({int(h) for h in items[:, 0]}))

    def shard_rows(self) -> tuple[np.ndarray, np.ndarray]:
        n = nat.c_int64(0)
        nat.check(nat.lib().svd_plan_shard_rows(self._handle, nat.ctypes.byref(n), None, None))
        heads = np.empty(max(n.value, 1), dtype=np.int32)
        toks = np.empty(max(n.value, 1), dtype=np.int32)
        nat.check(nat.lib().svd_plan_shard_rows(self._handle, nat.ctypes.byref(n), nat.ptr(heads),
                                                nat.ptr(toks)))
        return heads[: n.value], toks[: n.value]

    # -- execution
    def forward(self, q, k, v, out, head_dim: int | None = None, stream=None, o_head_map=None,
                nonfinite=None, in_head_map=None, row_stats=None, stats_heads: int = 0) -> None:
        """Launch the fused layer kernel on prepared bf16 CUDA tensors.

        q, k, v: [B, H, N, D] views with unit stride on D (D = 64 or 128);
        out: [B, H, N, D] (or the packed [rows, D] buffer of a shard plan).
        No host synchronisation; runs on `stream` (default: current stream).
        o_head_map: optional device int32 [H] tensor — plan head h writes head
        o_head_map[h] of `out` (a head-subset plan into a full-layer O).
        nonfinite: optional device int32 [1] tensor the epilogue ORs 1 into
        when an output row is non-finite (attention.py:98 require_finite).
        in_head_map: optional device int32 [plan heads] — plan head h reads
        q/k/v head in_head_map[h] (q/k/v may then hold fewer heads).
        row_stats / stats_heads: optional float32 device tensor
        [B * stats_heads, ceil(N / 128), 2, 128] receiving (-m, 1/l) of every
        row of plan heads < stats_heads (block_key_mass's row statistics).
        """
        import torch

        d_t = q.shape[-1]
        hd = int(head_dim if head_dim is not None else d_t)
        with torch.cuda.device(q.device):  # plan tables / tensor maps on q's device
            if stream is None:
                stream = torch.cuda.current_stream(q.device)
            a = nat.SvdFwdArgs()
            a.q, a.k, a.v, a.o = q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr()
            a.q_strides[:] = list(q.stride())
            a.k_strides[:] = list(k.stride())
            a.v_strides[:] = list(v.stride())
            if self.sharded:
                a.o_strides[:] = [0, 0, out.stride(0), out.stride(1)]
                a.batch = 1
            else:
                a.o_strides[:] = list(out.stride())
                a.batch = q.shape[0]
            a.head_dim, a.tensor_dim, a.dtype = hd, int(d_t), 0
            a.in_heads = int(q.shape[1]) if in_head_map is not None else 0
            a.in_head_map = in_head_map.data_ptr() if in_head_map is not None else None
            a.o_head_map = o_head_map.data_ptr() if o_head_map is not None else None
            a.nonfinite = nonfinite.data_ptr() if nonfinite is not None else None
            a.row_stats = row_stats.data_ptr() if row_stats is not None else None
            a.stats_heads = int(stats_heads) if row_stats is not None else 0
            nat.check(nat.lib().svd_attn_fwd_args(self._handle, nat.ctypes.byref(a),
                                                  nat.c_void_p(stream.cuda_stream)))


def _device_sm_count() -> int:
    try:
        import torch

        if torch.cuda.is_available():
            return int(torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count)
    except Exception:  # no CUDA runtime: plan for a B200
        pass
    return 148


_PLAN_CACHE: "OrderedDict[tuple, LayerPlan]" = OrderedDict()
_PLAN_CACHE_MAX = 64


def plan_for_assignment(assignment, layout: TokenLayout) -> LayerPlan:
    """Cached native plan for (layout, per-head specs).  The reference rebuilds
    every mask on every call (attention.py:178-182); the plan is immutable, so
    one build per distinct assignment suffices."""
    key = (layout, tuple(assignment))
    plan = _PLAN_CACHE.get(key)
    if plan is None:
        plan = LayerPlan.from_specs(list(assignment), layout)
        _PLAN_CACHE[key] = plan
        while len(_PLAN_CACHE) > _PLAN_CACHE_MAX:
            _PLAN_CACHE.popitem(last=False)
    else:
        _PLAN_CACHE.move_to_end(key)
    return plan


# ---------------------------------------------------------------- tensors


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def _check_qkv(q, k, v):
    """Rank-4 and equal shapes (attention.py:27-33 / numerics.py:46-53)."""
    for name, t in (("q", q), ("k", k), ("v", v)):
        nd = t.dim() if _is_torch(t) else np.ndim(t)
        if nd != 4:
            raise ShapeError(f"{name} must have rank 4 [B, H, N, d], got rank {nd}")
    sq, sk, sv = (tuple(t.shape) for t in (q, k, v))
    if not (sq == sk == sv):
        raise ShapeError(f"q/k/v shapes differ: {sq}, {sk}, {sv}")
    return sq


def _tensor_dim(d: int) -> int:
    if d <= 64:
        return 64
    if d <= 128:
        return 128
    raise nat.NativeError(f"head_dim {d} unsupported by the sm_100a kernel (max 128)")


def _to_device(xs):
    """Stage q, k, v as bf16 CUDA tensors with a 64/128-wide unit-stride last dim.

    Returns (tensors, was_numpy, device)."""
    import torch
    import torch.nn.functional as F

    was_numpy = not _is_torch(xs[0])
    if was_numpy:
        if not torch.cuda.is_available():
            raise nat.NativeError("a CUDA device is required: the sm_100a kernel has no CPU path")
        dev = torch.device("cuda", torch.cuda.current_device())
    else:
        dev = xs[0].device
        if dev.type != "cuda":
            raise nat.NativeError("tensors must live on a CUDA device (no CPU path)")
    out = []
    for x in xs:
        if was_numpy:
            t = torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=np.float32)))
            t = t.pin_memory().to(dev, non_blocking=True).to(torch.bfloat16)
        else:
            t = x if x.dtype == torch.bfloat16 else x.to(torch.bfloat16)
        d = t.shape[-1]
        dt = _tensor_dim(d)
        if dt != d:
            t = F.pad(t, (0, dt - d))
        if t.stride(-1) != 1 or any((s * 2) % 16 for s in t.stride()[:-1]) or t.data_ptr() % 16:
            t = t.contiguous()
        out.append(t)
    return out, was_numpy, dev


# Host-buffer pipeline: head-range chunks flow through copy-in -> kernel ->
# copy-out.  SVD_HOST_CHUNKS=k forces k equal chunks; by default the
# boundaries come from a flow-shop model of the three stages (below).
HOST_CHUNKS = int(__import__("os").environ.get("SVD_HOST_CHUNKS", "0"))
PCIE_BYTES_PER_S = float(__import__("os").environ.get("SVD_PCIE_GBPS", "50")) * 1e9
# opt-in: the kernel writes host-resident results straight into pinned memory
# (no copy-out stage) — measured 1.8x SLOWER end to end on B200 / PCIe: the
# epilogue's scattered 16-byte stores over PCIe stall the CTAs
HOST_ZERO_COPY = __import__("os").environ.get("SVD_HOST_ZERO_COPY", "0") == "1"
# consecutive chunk kernels on two alternating streams (SVD_HOST_OVERLAP=0: one)
HOST_OVERLAP = __import__("os").environ.get("SVD_HOST_OVERLAP", "1") == "1"
# attention.py:98 require_finite on every call (a device flag set by the
# kernel epilogue, read back after the launch); SVD_REQUIRE_FINITE=0 skips it
REQUIRE_FINITE = __import__("os").environ.get("SVD_REQUIRE_FINITE", "1") != "0"
# Per-SM kernel time per KV step of a work item (two 128-row tiles x 128
# keys), measured on B200 at power-capped clocks: HunyuanVideo 40.5 ms x 148
# SMs / 2.89 M steps (d=128), CogVideoX 35.7 ms x 148 / 3.48 M (d=64); plus a
# fixed per-CTA cost (TMEM / barrier setup, Q load, epilogue).
STEP_SECONDS = {64: 1.52e-6, 128: 2.07e-6}
ITEM_SECONDS = 5e-6
LAUNCH_SECONDS = 15e-6


def _flow_shop(bounds, h2d, kernel, d2h) -> float:
    """Makespan of chunks [bounds[i], bounds[i+1]) of a head order through
    three in-order stages (H2D stream, compute, D2H stream; PCIe is full
    duplex).  kernel(a, b) -> (SM-throughput time, longest item) of the launch
    of order[a:b].  Consecutive launches overlap (two compute streams,
    HOST_OVERLAP): a launch holds the SMs for its throughput time, and its
    output is complete once its longest item is too; with one stream a
    launch occupies the GPU for max(throughput, longest)."""
    t1 = t2 = t3 = 0.0
    for c in range(len(bounds) - 1):
        a, b = bounds[c], bounds[c + 1]
        t1 += h2d * (b - a)
        thr, longest = kernel(a, b)
        start = max(t2, t1)
        if HOST_OVERLAP:
            t2 = start + thr
            done = max(t2, start + longest) + LAUNCH_SECONDS
        else:
            t2 = done = start + max(thr, longest) + LAUNCH_SECONDS
        t3 = max(t3, done) + d2h * (b - a)
    return t3


def _launch_model(plan: "LayerPlan", B: int, d: int):
    """Per head: (SM-seconds of work, longest item in seconds).  A launch of
    a head set takes max(total work / SMs, longest item) + launch latency:
    every head of a text/frame layout has full-length forced rows, so a
    launch of a few sparse heads is bound by its longest item, not its work."""
    step = STEP_SECONDS[_tensor_dim(d)]
    work, longest = [], []
    for h in range(plan.n_heads):
        items, _ = plan.heads_subplan((h,)).schedule()
        kv = items[:, 3].astype(np.float64) if len(items) else np.zeros(1)
        work.append(B * float(np.sum(kv * step + ITEM_SECONDS)))
        longest.append(float(kv.max()) * step + ITEM_SECONDS)
    return work, longest


def _host_schedule(plan: LayerPlan, B: int, N: int, d: int):
    """(head order, chunk boundaries) for the host pipeline.

    Stage times per head: H2D 3*B*N*d*2 bytes, the kernel by the head's
    issued tiles (a FULL head costs ~30x a sparse one), D2H B*N*d*2 bytes.
    Heads are ordered by Johnson's rule for the copy-in -> kernel flow shop
    (kernel-heavy heads first, so the kernel starts early and the copies of
    the light heads hide under it; then the rest by falling kernel time), and
    the chunk boundaries by local search from equal chunks (a small first
    chunk starts the kernel early, a small last one shortens the drain)."""
    skip = set(plan.skip_heads())
    active = [h for h in range(plan.n_heads) if h not in skip]  # SKIP heads never cross PCIe
    H = len(active)
    cache = plan.__dict__.setdefault("_host_sched", {})
    key = (B, N, d, HOST_CHUNKS, HOST_ZERO_COPY)
    if key in cache:
        return cache[key]
    if H == 0:
        cache[key] = ([], [0])
        return cache[key]
    h2d = 3 * B * N * d * 2 / PCIE_BYTES_PER_S
    # zero-copy results leave with the kernel's own stores: no copy-out stage
    d2h = 0.0 if (HOST_ZERO_COPY and _tensor_dim(d) == d) else B * N * d * 2 / PCIE_BYTES_PER_S
    if HOST_CHUNKS > 0:
        order = list(active)
        k = max(1, min(HOST_CHUNKS, H))
        bounds = [round(i * H / k) for i in range(k + 1)]
    else:
        work, longest = _launch_model(plan, B, d)
        sms = _device_sm_count()
        solo = [max(w / sms, t) for w, t in zip(work, longest)]
        heavy = sorted((h for h in active if solo[h] >= h2d), key=lambda h: (-solo[h], h))
        light = sorted((h for h in active if solo[h] < h2d), key=lambda h: (-solo[h], h))
        hpre = {}

        def cost(o, bd):
            wp = [0.0]
            for h in o:
                wp.append(wp[-1] + work[h])

            def kernel(a, b):
                return (wp[b] - wp[a]) / sms, max(longest[h] for h in o[a:b])

            return _flow_shop(bd, h2d, kernel, d2h)

        def improve_bounds(o, bd, c0):
            improved = True
            while improved:  # boundary moves, merges and splits
                improved = False
                cands = []
                for i in range(1, len(bd) - 1):
                    for delta in (-2, -1, 1, 2):
                        nb = list(bd)
                        nb[i] += delta
                        if nb[i - 1] < nb[i] < nb[i + 1]:
                            cands.append(nb)
                    cands.append(bd[:i] + bd[i + 1:])
                for i in range(len(bd) - 1):
                    if bd[i + 1] - bd[i] > 1:
                        cands.append(bd[:i + 1] + [(bd[i] + bd[i + 1]) // 2] + bd[i + 1:])
                for nb in cands:
                    c = cost(o, nb)
                    if c < c0 * 0.999:
                        bd, c0, improved = nb, c, True
            return bd, c0

        best_all = None
        for cand_order in (heavy + light, list(active)):  # Johnson's order, the given order
            bd, c0 = None, float("inf")
            for k in range(1, min(H, 12) + 1):
                nb = [round(i * H / k) for i in range(k + 1)]
                c = cost(cand_order, nb)
                if c < c0:
                    bd, c0 = nb, c
            bd, c0 = improve_bounds(cand_order, bd, c0)
            if best_all is None or c0 < best_all[0]:
                best_all = (c0, list(cand_order), bd)
        # then alternate: head moves between chunks (first improvement), bounds
        c0, o, bd = best_all
        for _ in range(8):
            moved = False
            for i in range(H):
                for j in range(H):
                    if i == j:
                        continue
                    no = list(o)
                    no.insert(j, no.pop(i))
                    c = cost(no, bd)
                    if c < c0 * 0.999:
                        o, c0, moved = no, c, True
            bd, c0 = improve_bounds(o, bd, c0)
            if not moved:
                break
        best_all = (c0, o, bd)
        _, order, bounds = best_all
    cache[key] = (order, bounds)
    return order, bounds


class _Staging:
    """Device staging for the host-buffer path, owned by a plan and reused
    across calls: Q/K/V/O at the kernel's head width (zero padding written
    once), the copy-in / copy-out streams, and a lock (one host call at a
    time per plan and device)."""

    def __init__(self, dev, B: int, H: int, N: int, D: int):
        import threading

        import torch

        self.qkv = [torch.zeros((B, H, N, D), dtype=torch.bfloat16, device=dev) for _ in range(3)]
        self.o = torch.empty((B, H, N, D), dtype=torch.bfloat16, device=dev)
        self.s_in, self.s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        # chunk kernels alternate between the caller's stream and this one, so
        # the next chunk's CTAs fill the SMs the previous chunk's tail frees
        self.s_comp = torch.cuda.Stream(dev)
        self.lock = threading.Lock()
        self._maps = {}
        self._dev = dev
        self._host = {}

    def host_buffers(self, kind: str, count: int, B: int, N: int, d: int):
        """Resident pinned bf16 host staging [B, H, N, d] (slot-indexed like
        the device staging) for inputs / results that are not pinned bf16."""
        import torch

        bufs = self._host.get(kind)
        if bufs is None:
            H = self.qkv[0].shape[1]
            bufs = self._host[kind] = [torch.empty((B, H, N, d), dtype=torch.bfloat16, pin_memory=True)
                                       for _ in range(count)]
        return bufs

    def head_map(self, order, s0: int, s1: int):
        """Device int32 tensor of the output heads of staging slots [s0, s1)."""
        import torch

        key = (tuple(order), s0, s1)
        t = self._maps.get(key)
        if t is None:
            t = self._maps[key] = torch.tensor(order[s0:s1], dtype=torch.int32, device=self._dev)
        return t


def _host_staging(plan: "LayerPlan", dev, B: int, N: int, d: int, D: int) -> _Staging:
    cache = plan.__dict__.setdefault("_staging", {})
    key = (dev.index, B, N, d, D)  # d too: columns [d, D) must stay the zeros written once
    st = cache.get(key)
    if st is None:
        cache.clear()  # one resident staging set per plan
        st = cache[key] = _Staging(dev, B, plan.n_heads, N, D)
    return st


def _check_out(out, shape, device_type: str):
    import torch

    if not _is_torch(out) or out.dtype != torch.bfloat16 or tuple(out.shape) != tuple(shape):
        raise ShapeError(f"out must be a bf16 torch tensor of shape {tuple(shape)}")
    if out.device.type != device_type:
        raise ShapeError(f"out must live on the {device_type} like q/k/v")
    if out.stride(-1) != 1:
        raise ShapeError("out must have a unit-stride last dimension")


def _run_host(plan: LayerPlan, q, k, v, out=None, numpy_out: bool = False):
    """Host (CPU torch) tensors: pipeline head chunks through copy-in,
    compute and copy-out streams so the PCIe/C2C transfers overlap the kernel
    (the end-to-end path of the operator with host buffers).  Returns a CPU
    bf16 tensor (pinned), or writes `out` (a caller-owned, ideally pinned, CPU
    bf16 tensor: no per-call host allocation); numpy_out: a float32 NumPy
    result checked for finiteness (the reference's own types).

    Inputs that are not pinned bf16 (e.g. the reference's float32 NumPy
    arrays) are converted chunk by chunk on the host's cores into resident
    pinned bf16 staging, so the conversion of chunk c+1 overlaps the copies
    and the kernel of chunk c, and only bf16 crosses PCIe."""
    import torch

    B, H, N, d = q.shape
    dev = torch.device("cuda", torch.cuda.current_device())
    D = _tensor_dim(d)
    order, bounds = _host_schedule(plan, B, N, d)
    chunks = len(bounds) - 1
    if numpy_out:
        res = np.empty((B, H, N, d), dtype=np.float32)
        out_host = torch.from_numpy(res)
    elif out is None:
        out_host = torch.empty((B, H, N, d), dtype=torch.bfloat16, pin_memory=True)
    else:
        _check_out(out, (B, H, N, d), "cpu")
        out_host = out
    skip = plan.skip_heads()
    if chunks == 0:  # every head SKIP
        out_host.zero_()
        return res if numpy_out else out_host
    # staging slot s holds head order[s]; chunks are contiguous slot ranges
    st = _host_staging(plan, dev, B, N, d, D)
    direct_in = all(x.dtype == torch.bfloat16 and x.is_pinned() for x in (q, k, v))
    direct_out = not numpy_out and out_host.is_pinned()
    with st.lock:
        host_in = None if direct_in else st.host_buffers("in", 3, B, N, d)
        host_out = None if direct_out else st.host_buffers("out", 1, B, N, d)[0]
        compute = torch.cuda.current_stream(dev)
        s_in, s_out = st.s_in, st.s_out
        # zero-copy result: the kernel stores rows straight into the pinned
        # host O through a per-chunk head map (no copy-out stage to drain)
        zero_copy = (HOST_ZERO_COPY and D == d and direct_out and out_host.is_contiguous())
        streams = (compute, st.s_comp) if HOST_OVERLAP else (compute,)
        # attention.py:98 require_finite, fused into the kernel epilogue
        flag = torch.zeros(1, dtype=torch.int32, device=dev) if REQUIRE_FINITE else None
        st.s_comp.wait_stream(compute)  # the caller's prior work on its stream (and the flag's zero-fill)
        copied = []   # per chunk: D2H done event
        drained = 0   # chunks whose results are in out_host

        def drain(upto: int, block: bool) -> int:
            # host-side finish of chunks [drained, upto): widen to out_host
            n_done = drained
            while n_done < upto:
                if not block and not copied[n_done].query():
                    break
                copied[n_done].synchronize()
                for slot in range(bounds[n_done], bounds[n_done + 1]):
                    out_host[:, order[slot]].copy_(host_out[:, slot])
                n_done += 1
            return n_done

        for c in range(chunks):
            s0, s1 = bounds[c], bounds[c + 1]
            with torch.cuda.stream(s_in):
                for slot in range(s0, s1):
                    h = order[slot]
                    for i, (x, buf) in enumerate(zip((q, k, v), st.qkv)):
                        xc = x[:, h]
                        if not direct_in:  # widen / narrow on the host cores into pinned bf16
                            host_in[i][:, slot].copy_(xc)
                            xc = host_in[i][:, slot]
                        buf[:, slot, :, :d].copy_(xc, non_blocking=True)
                loaded = torch.cuda.Event()
                loaded.record(s_in)
            cs = streams[c % len(streams)]
            cs.wait_event(loaded)
            qc, kc, vc = (buf[:, s0:s1] for buf in st.qkv)
            sub = plan.heads_subplan(tuple(order[s0:s1]))
            if zero_copy:
                sub.forward(qc, kc, vc, out_host, head_dim=d, stream=cs,
                            o_head_map=st.head_map(order, s0, s1), nonfinite=flag)
                continue
            sub.forward(qc, kc, vc, st.o[:, s0:s1], head_dim=d, stream=cs, nonfinite=flag)
            computed = torch.cuda.Event()
            computed.record(cs)
            with torch.cuda.stream(s_out):
                s_out.wait_event(computed)
                for slot in range(s0, s1):
                    dst = out_host[:, order[slot]] if direct_out else host_out[:, slot]
                    dst.copy_(st.o[:, slot, :, :d], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(s_out)
                copied.append(ev)
            if not direct_out:
                drained = drain(c, block=False)
        if len(streams) > 1:
            compute.wait_stream(st.s_comp)  # the caller's stream sees every chunk
        for h in skip:  # SKIP heads (attention.py:51-54): zeros written on the host, under the GPU work
            out_host[:, h].zero_()
        if zero_copy:
            compute.synchronize()
        elif direct_out:
            s_out.synchronize()  # a host result must be readable on return
        else:
            drain(chunks, block=True)
        if flag is not None and int(flag.item()) != 0:
            raise ShapeError("non-finite values in attention output")
    return res if numpy_out else out_host


def host_transfer_bytes(plan: LayerPlan, B: int, N: int, d: int) -> tuple[int, int]:
    """(H2D, D2H) bytes one host-buffer call moves: bf16 Q/K/V in and O out
    for every head except SKIP heads (their zeros are written on the host)."""
    h = plan.n_heads - len(plan.skip_heads())
    return 3 * B * h * N * d * 2, B * h * N * d * 2


def _run(plan: LayerPlan, q, k, v, out=None):
    import torch

    shape = _check_qkv(q, k, v)
    B, H, N, d = shape
    if _is_torch(q) and q.device.type == "cpu":
        if plan.layout.total_tokens != N:
            raise ShapeError(f"mask grid covers {plan.layout.total_tokens} tokens, tensors have {N}")
        if plan.n_heads != H:
            raise ConfigError(f"plan covers {plan.n_heads} heads, tensors have {H}")
        if not torch.cuda.is_available():
            raise nat.NativeError("a CUDA device is required: the sm_100a kernel has no CPU path")
        return _run_host(plan, q, k, v, out)
    if plan.layout.total_tokens != N:
        raise ShapeError(f"mask grid covers {plan.layout.total_tokens} tokens, tensors have {N}")
    if plan.n_heads != H:
        raise ConfigError(f"plan covers {plan.n_heads} heads, tensors have {H}")
    if out is not None and not _is_torch(q):
        raise ShapeError("out= is supported for torch tensors only")
    if not _is_torch(q):
        # the reference's own types (float32 NumPy in and out): the pipelined
        # host path, converting on the host cores chunk by chunk
        if not torch.cuda.is_available():
            raise nat.NativeError("a CUDA device is required: the sm_100a kernel has no CPU path")
        ts = [torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=np.float32))) for x in (q, k, v)]
        return _run_host(plan, *ts, numpy_out=True)
    (qt, kt, vt), was_numpy, dev = _to_device((q, k, v))
    dt = qt.shape[-1]
    # attention.py:98 require_finite: the epilogue flags non-finite rows; reading
    # the flag back synchronises (SVD_REQUIRE_FINITE=0 keeps the call async)
    flag = torch.zeros(1, dtype=torch.int32, device=dev) if REQUIRE_FINITE else None
    if out is not None:
        _check_out(out, (B, H, N, d), "cuda")
        if dt == d and all((st * 2) % 16 == 0 for st in out.stride()[:-1]) and out.data_ptr() % 16 == 0:
            plan.forward(qt, kt, vt, out, head_dim=d, nonfinite=flag)
        else:
            tmp = torch.empty((B, H, N, dt), dtype=torch.bfloat16, device=dev)
            plan.forward(qt, kt, vt, tmp, head_dim=d, nonfinite=flag)
            out.copy_(tmp[..., :d])
        _require_finite(flag)
        return out
    out = torch.empty((B, H, N, dt), dtype=torch.bfloat16, device=dev)
    plan.forward(qt, kt, vt, out, head_dim=d, nonfinite=flag)
    if dt != d:
        out = out[..., :d]
    _require_finite(flag)
    if was_numpy:
        return out.float().cpu().numpy()
    return out


def _require_finite(flag) -> None:
    if flag is not None and int(flag.item()) != 0:
        raise ShapeError("non-finite values in attention output")


# ---------------------------------------------------------------- reference API


@dataclass(frozen=True, eq=False)
class HeadGroup:
    """Heads of one layer sharing a pattern (attention.py:149-161)."""

    spec: PatternSpec
    heads: tuple[int, ...]
    mask: BlockMask | None
    plan: LayerPlan | None = field(default=None, repr=False, compare=False)

    def __post_init__(self):
        if not self.heads:
            raise ConfigError("head group must contain at least one head")
        if len(set(self.heads)) != len(self.heads):
            raise ConfigError(f"duplicate heads in group: {self.heads}")


_GROUP_CACHE: "OrderedDict[tuple, list]" = OrderedDict()


def group_heads(assignment, grid: BlockGrid) -> list[HeadGroup]:
    """Fuse same-pattern heads; groups in first-occurrence order (attention.py:164-183).

    Grouping, masks and the kernel schedule come from the native plan builder;
    the returned groups share that plan, so fused_layer_attention launches it
    without rebuilding anything."""
    assignment = list(assignment)
    key = (grid.layout, tuple(assignment))
    cached = _GROUP_CACHE.get(key)
    if cached is not None:
        _GROUP_CACHE.move_to_end(key)
        return list(cached)
    plan = plan_for_assignment(assignment, grid.layout)
    groups = []
    for g in range(plan.info.n_groups):
        heads, skip = plan.group_heads(g)
        spec = assignment[heads[0]]
        mask = None
        if int(spec.mode) not in (Mode.FULL, Mode.SKIP):
            active = plan.group_mask(g)
            active.setflags(write=False)  # shared by every caller: immutable like the plan
            mask = BlockMask(grid=grid, active=active)
        groups.append(HeadGroup(spec=spec, heads=heads, mask=mask, plan=plan))
    plan.__dict__["_groups"] = tuple(groups)
    _GROUP_CACHE[key] = groups
    while len(_GROUP_CACHE) > _PLAN_CACHE_MAX:
        _GROUP_CACHE.popitem(last=False)
    return list(groups)


def _plan_for_groups(groups, H: int, N: int) -> LayerPlan:
    # groups may also be the reference's own HeadGroups (no plan attached)
    plans = {id(getattr(g, "plan", None)) for g in groups}
    first = getattr(groups[0], "plan", None)
    if len(plans) == 1 and first is not None and first.n_heads == H:
        # the groups came from one group_heads() call: reuse its plan only if
        # every group is still what that call produced (same heads, spec and
        # the very mask object — dataclasses.replace(g, mask=...) keeps
        # g.plan, so an edited group must be lowered from its own mask)
        made = first.__dict__.get("_groups", ())
        if len(made) == len(groups) and all(
                g.heads == m.heads and g.spec == m.spec and g.mask is m.mask
                for g, m in zip(groups, made)):
            return first
    # hand-built groups: lower their masks explicitly
    layout = None
    masks, head_group = [], np.zeros(H, dtype=np.int32)
    for gi, g in enumerate(groups):
        if g.mask is not None:
            layout = g.mask.grid.layout
        if int(g.spec.mode) == Mode.SKIP:
            masks.append(None)
        elif int(g.spec.mode) == Mode.FULL or g.mask is None:
            masks.append("full")
        else:
            masks.append(g.mask.active)
        for h in g.heads:
            head_group[h] = gi
    if layout is None:
        layout = _dense_layout(N)
    nb = layout.n_blocks
    masks = [np.ones((nb, nb), dtype=bool) if isinstance(m, str) else m for m in masks]
    return LayerPlan.from_masks(layout, masks, head_group)


def fused_layer_attention(q, k, v, groups, out=None):
    """One layer's attention, every head in one kernel launch (attention.py:186-212).

    `out` (extension; torch tensors only): a caller-owned bf16 result buffer
    on the device of q/k/v (a CPU one for host tensors, ideally pinned), written
    in place and returned — a serving loop then allocates nothing per call."""
    B, H, N, d = _check_qkv(q, k, v)
    seen: list[int] = []
    for g in groups:
        seen.extend(g.heads)
    if sorted(seen) != list(range(H)):
        raise ConfigError(f"groups cover heads {sorted(seen)}, tensors have {H} heads")
    for g in groups:
        if g.mask is not None and g.mask.grid.layout.total_tokens != N:
            raise ShapeError(
                f"mask grid covers {g.mask.grid.layout.total_tokens} tokens, tensors have {N}")
    return _run(_plan_for_groups(groups, H, N), q, k, v, out)


_MASK_PLANS: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()
_MASK_CONTENT_PLANS: "OrderedDict[tuple, LayerPlan]" = OrderedDict()


def _mask_plan(mask: BlockMask, H: int) -> LayerPlan:
    """Plan for one mask over H heads.  Read-only masks (the ones group_heads /
    build_mask hand out) are cached by identity; a writable mask may be edited
    in place between calls, so it is keyed by its content."""
    active = np.asarray(mask.active)
    if not active.flags.writeable:
        per_mask = _MASK_PLANS.setdefault(mask, {})
        plan = per_mask.get(H)
        if plan is None:
            plan = per_mask[H] = LayerPlan.from_masks(mask.grid.layout, [active], np.zeros(H, dtype=np.int32))
        return plan
    import hashlib

    key = (mask.grid.layout, H, active.shape,
           hashlib.blake2b(np.packbits(active.astype(bool, copy=False)).tobytes(), digest_size=16).digest())
    plan = _MASK_CONTENT_PLANS.get(key)
    if plan is None:
        plan = LayerPlan.from_masks(mask.grid.layout, [active], np.zeros(H, dtype=np.int32))
        _MASK_CONTENT_PLANS[key] = plan
        while len(_MASK_CONTENT_PLANS) > _PLAN_CACHE_MAX:
            _MASK_CONTENT_PLANS.popitem(last=False)
    else:
        _MASK_CONTENT_PLANS.move_to_end(key)
    return plan


def sparse_attention(q, k, v, mask: BlockMask):
    """Block-sparse attention restricted to `mask` (attention.py:57-98)."""
    B, H, N, d = _check_qkv(q, k, v)
    if mask.grid.layout.total_tokens != N:
        raise ShapeError(f"mask grid covers {mask.grid.layout.total_tokens} tokens, tensors have {N}")
    if mask.is_skip:
        raise DegenerateRowError("skip mask defines no softmax; use skip_attention")
    if not np.asarray(mask.active).any(axis=1).all():
        raise DegenerateRowError("mask has a query row with no active key blocks")
    return _run(_mask_plan(mask, H), q, k, v)


def full_mask_attention(q, k, v, grid: BlockGrid):
    """The streaming kernel with every block active (attention.py:101-105)."""
    H = _check_qkv(q, k, v)[1]
    return _run(plan_for_assignment([full_spec()] * H, grid.layout), q, k, v)


def _dense_layout(n: int) -> TokenLayout:
    return TokenLayout(text_tokens=0, frames=1, tokens_per_frame=n, block_size=64)


def dense_attention(q, k, v):
    """softmax(q k^T / sqrt(d)) v (attention.py:36-41) — the all-active kernel;
    no [N, N] score matrix is materialised."""
    B, H, N, d = _check_qkv(q, k, v)
    return _run(plan_for_assignment([full_spec()] * H, _dense_layout(N)), q, k, v)


def skip_attention(q, k, v):
    """SKIP mode: exact zeros, zero FLOPs (attention.py:51-54)."""
    B, H, N, d = _check_qkv(q, k, v)
    return _run(plan_for_assignment([skip_spec()] * H, _dense_layout(N)), q, k, v)


def block_key_mass(q, k, grid: BlockGrid):
    """Per-head attention mass per key block [B, H, nb] (attention.py:108-146);
    computed on the GPU by calibrate.block_key_mass."""
    from .calibrate import block_key_mass as _bkm

    return _bkm(q, k, grid)


__all__ = [
    "LayerPlan", "HeadGroup", "group_heads", "host_transfer_bytes", "fused_layer_attention", "sparse_attention", "block_key_mass",
    "full_mask_attention", "dense_attention", "skip_attention", "plan_for_assignment",
]
