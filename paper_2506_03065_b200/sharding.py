"""Head / query-range sharding of one layer over the GPUs of a box.

Heads are independent (attention.py:211 writes only out[:, idx]) and so are
query blocks within a head (attention.py:81-97).  The plan's work items —
(head, four query segments) with their KV tile lists — are dealt to ranks
balancing tile cost (svd_plan_shard_ex): by default head-locally (each rank
holds ~H/N heads, at most its two boundary heads split by query range), or
by LPT over all items.  PeerShardedLayer (default) fuses the reassembly into
the kernel: each rank's shard stores its rows into every rank's O over peer
memory.  HeadShardedLayer writes packed rows that one NCCL all-gather plus
the unpack kernel scatter back into O[B=1, H, N, d].  Device-resident Q/K/V
are taken as given on every rank (as layer_qkv produces them,
model.py:372-391); from host buffers a rank copies in only its own heads.
"""

from __future__ import annotations

import numpy as np

from . import _native as nat
from .attention import LayerPlan

# head chunks of a rank's pipelined end-to-end step (PeerShardedLayer.e2e)
E2E_CHUNKS = int(__import__("os").environ.get("SVD_E2E_CHUNKS", "3"))


def gathered_row_maps(plan: LayerPlan, world: int, max_item_tiles: int = 0):
    """(shards, row_head, row_token, max_rows) for the all-gathered buffer:
    rank r's packed rows occupy [r*max_rows, (r+1)*max_rows); padding rows and
    rows past the sequence end carry head -1 (skipped by the unpack)."""
    shards = [plan.shard(world, r, max_item_tiles=max_item_tiles) for r in range(world)]
    rows = [s.shard_rows() for s in shards]
    max_rows = max(1, max(len(h) for h, _ in rows))
    heads = np.full(world * max_rows, -1, dtype=np.int32)
    toks = np.full(world * max_rows, -1, dtype=np.int32)
    for r, (h, t) in enumerate(rows):
        heads[r * max_rows: r * max_rows + len(h)] = h
        toks[r * max_rows: r * max_rows + len(t)] = t
    return shards, heads, toks, max_rows


class PeerShardedLayer:
    """One layer over `world` ranks with the reassembly fused into the kernel.

    Every rank owns one device buffer holding two O buffers [B, H, N, D]
    (double-buffered across steps) and an int32 flag array; the buffers are
    exchanged once as CUDA IPC handles over the process group and mapped into
    every rank (NVLink peer memory between GPUs).  A step launches this rank's
    shard with svd_attn_fwd_peers — the kernel epilogue stores each finished
    row into the step's O buffer of all `world` ranks, so the transfer
    overlaps the attention math tile by tile and no all-gather / unpack runs
    — then svd_peer_barrier, a stream-ordered barrier over the flag arrays:
    no host synchronisation and no process-group call on the data path.

    Buffer lifetime: the O returned by step t is complete once the caller's
    stream passes that step's barrier, and stays valid until the step after
    next (t + 2) starts writing the same buffer.  Work the caller enqueues on
    this stream between the calls (e.g. consuming step t's O before calling
    step t + 1) is ordered before every peer's t + 2 stores by the t + 1
    barrier.
    """

    def __init__(self, plan: LayerPlan, world: int, rank: int, head_dim: int, device, shape,
                 max_item_tiles: int | None = None, partition: str = "heads", timeout_s: float = 30.0):
        import torch
        import torch.distributed as dist

        self.plan = plan
        self.world = world
        self.rank = rank
        self.head_dim = head_dim
        self.device = device
        self.timeout_s = float(timeout_s)
        # a shard view (split-KV balanced) for N > 1, the plain plan for one rank
        # unless a split cap is forced (tests).  "heads": contiguous head
        # ranges of equal cost, so a rank's inputs are its own heads only
        if world > 1 or max_item_tiles is not None:
            self.shard = plan.shard(world, rank, max_item_tiles=max_item_tiles or 0, partition=partition)
        else:
            self.shard = plan
        # heads whose Q/K/V this rank reads (about H / world of them for "heads")
        self.heads = self.shard.shard_heads() if self.shard is not plan else tuple(range(plan.n_heads))
        self._inputs = None
        # one allocation per rank: [O buffer 0 | O buffer 1 | flags int32[8]]
        o_elems = 1
        for s in shape:
            o_elems *= int(s)
        o_bytes = (o_elems * 2 + 255) // 256 * 256
        self._buf = torch.zeros(2 * o_bytes + 256, dtype=torch.uint8, device=device)
        self.outs = [self._buf[i * o_bytes: i * o_bytes + o_elems * 2].view(torch.bfloat16).view(*shape)
                     for i in range(2)]
        self.flags = self._buf[2 * o_bytes: 2 * o_bytes + 32].view(torch.int32)
        self.timed_out = torch.zeros(1, dtype=torch.int32, device=device)
        self._o_bytes = o_bytes
        off = nat.c_int64(0)
        hbuf = (nat.c_uint8 * 64)()
        nat.check(nat.lib().svd_ipc_export(nat.c_void_p(self._buf.data_ptr()), hbuf, nat.ctypes.byref(off)))
        gathered = [None] * world
        if world > 1:
            dist.all_gather_object(gathered, (rank, bytes(hbuf), int(off.value)))
        else:
            gathered = [(rank, bytes(hbuf), int(off.value))]
        self._opened = []
        bases = []
        for r, h, o in sorted(gathered):
            if r == rank:
                bases.append(self._buf.data_ptr())
                continue
            p = nat.c_void_p()
            hb = (nat.c_uint8 * 64).from_buffer_copy(h)
            nat.check(nat.lib().svd_ipc_import(hb, o, nat.ctypes.byref(p)))
            self._opened.append((p.value, o))
            bases.append(p.value)
        self.peer_ptrs = [(nat.c_void_p * world)(*[b + i * o_bytes for b in bases]) for i in range(2)]
        self.flag_ptrs = (nat.c_void_p * world)(*[b + 2 * o_bytes for b in bases])
        self.step = 0
        torch.cuda.synchronize(device)
        if world > 1:
            dist.barrier()  # every rank's flags are zero before any step runs

    @property
    def out(self):
        """The O buffer of the latest step (buffer 0 before the first step)."""
        return self.outs[(self.step - 1) % 2] if self.step else self.outs[0]

    def __call__(self, q, k, v, out=None, kernel_events=None):
        """Run this rank's shard and the step barrier; returns this rank's
        complete O (all rows) — stream-ordered, no host synchronisation."""
        import torch

        b = self.step % 2
        stream = torch.cuda.current_stream(self.device)
        with torch.cuda.device(self.device):
            if kernel_events is not None:
                kernel_events[0].record(stream)
            st = [nat.i64x4(t.stride()) for t in (q, k, v)]
            nat.check(nat.lib().svd_attn_fwd_peers(
                self.shard.handle, nat.c_void_p(q.data_ptr()), nat.c_void_p(k.data_ptr()),
                nat.c_void_p(v.data_ptr()), self.peer_ptrs[b], self.world, st[0], st[1], st[2],
                nat.i64x4(self.outs[b].stride()), 1, int(self.head_dim), int(q.shape[-1]), 0,
                nat.c_void_p(stream.cuda_stream)))
            if kernel_events is not None:
                kernel_events[1].record(stream)
            if self.world > 1:
                nat.check(nat.lib().svd_peer_barrier(
                    self.flag_ptrs, self.world, self.rank, nat.c_int32((self.step + 1) & 0xFFFFFFFF).value,
                    nat.c_void_p(self.timed_out.data_ptr()), self.timeout_s, nat.c_void_p(stream.cuda_stream)))
        self.step += 1
        res = self.outs[b]
        if out is not None and out.data_ptr() != res.data_ptr():
            out.copy_(res)
            return out
        return res

    def check(self) -> None:
        """Raise if a step barrier timed out (a peer never arrived).  Reads a
        device flag: synchronises the stream."""
        if int(self.timed_out.item()) != 0:
            raise nat.NativeError("peer barrier timed out: a rank did not finish its step")

    def _e2e_plan(self, n_tokens: int):
        """(chunks, owned) for the pipelined end-to-end step: this rank's heads
        in up to E2E_CHUNKS chunks of about equal copy-in bytes, the
        kernel-heaviest first (the first kernel starts early, the light heads'
        copies hide under the heavy heads' kernels), each with its sub-plan;
        and the heads whose rows this rank computes all of (their D2H can
        leave right after their chunk's kernel — a boundary head shared with
        a neighbour waits for the step barrier)."""
        cached = self.__dict__.get("_e2e_cache")
        if cached is not None and cached[0] == n_tokens:
            return cached[1], cached[2]
        items, _ = self.shard.schedule()
        cost = {h: 0.0 for h in self.heads}
        for it in items:
            cost[int(it[0])] = cost.get(int(it[0]), 0.0) + float(it[3]) + 4.0
        order = sorted(self.heads, key=lambda h: (-cost[h], h))
        k = max(1, min(E2E_CHUNKS, len(order)))
        bounds = [round(i * len(order) / k) for i in range(k + 1)]
        chunks = []
        for c in range(k):
            hs = tuple(order[bounds[c]:bounds[c + 1]])
            sub = self.shard.shard_subset(hs) if self.shard.sharded else self.shard.heads_subplan(hs)
            chunks.append((hs, sub))
        if self.world == 1 or not self.shard.sharded:
            owned = set(self.heads)
        else:
            rh, rt = self.shard.shard_rows()
            valid = rt >= 0
            counts = np.bincount(rh[valid], minlength=self.plan.n_heads)
            owned = {h for h in self.heads if counts[h] == n_tokens}
        self._e2e_cache = (n_tokens, chunks, owned)
        return chunks, owned

    def e2e(self, hq, hk, hv, hout, groups=None):
        """End-to-end step from pinned host buffers, pipelined per head chunk:
        H2D of chunk c (copy stream) overlaps the shard kernel of chunk c-1
        (the caller's stream; rows land in every rank's O), the D2H of the
        heads this rank fully computes follows each chunk's kernel on a third
        stream, the boundary heads' D2H follows the stream-ordered step
        barrier.  Returns once hout holds this rank's heads."""
        import torch

        B, H, N, D = hq.shape
        if B != 1:
            raise nat.NativeError("the multi-GPU layer runs batch 1")
        if self._inputs is None or self._inputs[0].shape != hq.shape:
            self._inputs = [torch.empty(hq.shape, dtype=hq.dtype, device=self.device) for _ in range(3)]
        if self.__dict__.get("_streams") is None:
            self._streams = (torch.cuda.Stream(self.device), torch.cuda.Stream(self.device))
        s_in, s_out = self._streams
        chunks, owned = self._e2e_plan(N)
        comp = torch.cuda.current_stream(self.device)
        b = self.step % 2
        o = self.outs[b]
        st = [nat.i64x4(t.stride()) for t in self._inputs]
        with torch.cuda.device(self.device):
            s_in.wait_stream(comp)  # the previous step's kernels are done reading the inputs
            for hs, sub in chunks:
                with torch.cuda.stream(s_in):
                    for src, dst in zip((hq, hk, hv), self._inputs):
                        for h in hs:
                            dst[:, h].copy_(src[:, h], non_blocking=True)
                    loaded = torch.cuda.Event()
                    loaded.record(s_in)
                comp.wait_event(loaded)
                nat.check(nat.lib().svd_attn_fwd_peers(
                    sub.handle, nat.c_void_p(self._inputs[0].data_ptr()), nat.c_void_p(self._inputs[1].data_ptr()),
                    nat.c_void_p(self._inputs[2].data_ptr()), self.peer_ptrs[b], self.world, st[0], st[1], st[2],
                    nat.i64x4(o.stride()), 1, int(self.head_dim), int(D), 0, nat.c_void_p(comp.cuda_stream)))
                mine = [h for h in hs if h in owned]
                if mine:
                    done = torch.cuda.Event()
                    done.record(comp)
                    with torch.cuda.stream(s_out):
                        s_out.wait_event(done)
                        for h in mine:
                            hout[:, h].copy_(o[:, h], non_blocking=True)
            if self.world > 1:
                nat.check(nat.lib().svd_peer_barrier(
                    self.flag_ptrs, self.world, self.rank, nat.c_int32((self.step + 1) & 0xFFFFFFFF).value,
                    nat.c_void_p(self.timed_out.data_ptr()), self.timeout_s, nat.c_void_p(comp.cuda_stream)))
            rest = [h for h in self.heads if h not in owned]
            if rest:
                s_out.wait_stream(comp)
                with torch.cuda.stream(s_out):
                    for h in rest:
                        hout[:, h].copy_(o[:, h], non_blocking=True)
        self.step += 1
        s_out.synchronize()
        comp.synchronize()
        return hout

    def e2e_bytes(self, shape) -> tuple[int, int]:
        """(H2D, D2H) bytes of this rank's e2e step for bf16 [B, H, N, d] tensors."""
        B, _, N, d = shape
        h = len(self.heads)
        return 3 * B * h * N * d * 2, B * h * N * d * 2

    def nvlink_bytes(self, tensor_dim: int) -> int:
        """Bytes this rank's epilogue stores into its peers' O per step: every
        row it computes, once per other rank (bf16 [tensor_dim])."""
        if self.world == 1:
            return 0
        heads, _ = self.shard.shard_rows()
        return int(len(heads)) * tensor_dim * 2 * (self.world - 1)

    def close(self):
        for p, o in self._opened:
            nat.lib().svd_ipc_close(nat.c_void_p(p), o)
        self._opened = []


class HeadShardedLayer:
    """Callable running one layer's attention on `world` ranks (1 = plain launch)."""

    def __init__(self, plan: LayerPlan, world: int, rank: int, head_dim: int, device):
        import torch

        self.plan = plan
        self.world = world
        self.rank = rank
        self.head_dim = head_dim
        self.device = device
        self.tensor_dim = 64 if head_dim <= 64 else 128
        if world == 1:
            self.shard = None
            return
        shards, heads, toks, self.max_rows = gathered_row_maps(plan, world)
        self.shard = shards[rank]
        self.row_head = torch.from_numpy(heads).to(device)
        self.row_token = torch.from_numpy(toks).to(device)
        self.packed = torch.empty(self.max_rows, self.tensor_dim, dtype=torch.bfloat16, device=device)
        self.gathered = torch.empty(world * self.max_rows, self.tensor_dim, dtype=torch.bfloat16,
                                    device=device)

    def __call__(self, q, k, v, out, kernel_events=None):
        import torch

        stream = torch.cuda.current_stream(self.device)
        if kernel_events is not None:
            kernel_events[0].record(stream)
        if self.shard is None:
            self.plan.forward(q, k, v, out, head_dim=self.head_dim, stream=stream)
            if kernel_events is not None:
                kernel_events[1].record(stream)
            return out
        self.shard.forward(q, k, v, self.packed, head_dim=self.head_dim, stream=stream)
        if kernel_events is not None:
            kernel_events[1].record(stream)
        import torch.distributed as dist

        if dist.get_backend() == "nccl":
            dist.all_gather_into_tensor(self.gathered, self.packed)
        else:  # gloo (CPU test harness): list form
            dist.all_gather(list(self.gathered.view(self.world, self.max_rows, -1).unbind(0)),
                            self.packed)
        ost = nat.i64x4(out.stride())
        nat.check(nat.lib().svd_unpack_rows(
            nat.c_void_p(self.row_head.data_ptr()), nat.c_void_p(self.row_token.data_ptr()),
            int(self.world * self.max_rows), nat.c_void_p(self.gathered.data_ptr()),
            int(self.gathered.stride(0)), nat.c_void_p(out.data_ptr()), ost, int(self.tensor_dim),
            nat.c_void_p(stream.cuda_stream)))
        return out

    def e2e(self, hq, hk, hv, hout, groups):
        """End-to-end step from pinned host buffers: H2D, attention, D2H."""
        import torch

        from .attention import fused_layer_attention

        if self.shard is None:
            # the public API with host buffers: head-chunk pipelined H2D / kernel / D2H
            return fused_layer_attention(hq, hk, hv, groups, out=hout)
        q = hq.to(self.device, non_blocking=True)
        k = hk.to(self.device, non_blocking=True)
        v = hv.to(self.device, non_blocking=True)
        out = torch.empty(hout.shape, dtype=torch.bfloat16, device=self.device)
        self(q, k, v, out)
        hout.copy_(out, non_blocking=True)
        return hout
