"""Benchmark: one vDiT sparse-attention layer (the Sparse-vDiT hot path) on B200.

python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                [--config hunyuan|cogvideo|wan|synthetic4k] [--sweep]

A step = the whole layer's attention for one batch: every head of the layer,
FULL / SKIP / diagonal / multi-diagonal / vertical-stripe heads in ONE fused
kernel launch (plus, for N>1, the NCCL all-gather that reassembles the head
dimension and the unpack kernel).  Inputs are synthetic bf16 Q/K/V of the
named layer shape, resident in HBM; the 2+ GB of inputs exceed the 126 MB L2,
so no L2 flush is needed between steps.

value = effective (dense-equivalent) TFLOP/s = 4*N^2*d*H / t for the whole
job; ms_per_step = ms per layer.  roofline = active-tile FLOPs (the
reference's FLOP convention, costmodel.py:26-32) / kernel time vs the measured
bf16 tensor peak.  e2e = the same layer through the public API with host
(pinned) Q/K/V copied in and O copied out every step.  cpu_baseline = the
reference algorithm (oracle port, fp64 NumPy) timed on this host on a bounded
sample of query blocks, extrapolated by active FLOPs.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "vDiT sparse-attn ms/layer & effective TFLOPS at 86k/120k tokens, 1/2/4/8 B200"

# BASELINE.json configs / SURVEY §8(d): layout, heads x head_dim, mode mix F/S/D/MD/VS
CONFIGS = {
    "hunyuan": dict(name="HunyuanVideo layer (119,056 tokens, 24x128)", layout=(256, 33, 3600, 64),
                    heads=24, d=128, mix=(6, 1, 6, 6, 5)),
    "cogvideo": dict(name="CogVideoX1.5 layer (85,906 tokens, 48x64)", layout=(226, 21, 4080, 64),
                     heads=48, d=64, mix=(14, 2, 11, 11, 10)),
    "wan": dict(name="Wan2.1 layer (75,600 tokens, 40x128)", layout=(0, 21, 3600, 64),
                heads=40, d=128, mix=(17, 2, 7, 7, 7)),
    "synthetic4k": dict(name="synthetic 4k layer (4,096 tokens, 8x64)", layout=(0, 16, 256, 64),
                        heads=8, d=64, mix=None),
}


UNIT = "TFLOP/s (effective, dense-equivalent 4*N^2*d*H)"
MODE_LABELS = {0: "full", 1: "skip", 2: "diagonal", 3: "multi_diagonal", 4: "vertical_stripe"}


def assignment_for(cfg, S):
    """Per-head specs for a config: the paper-derived mode mix with distinct
    stripe columns per stripe head (seeded), in a fixed shuffled head order.
    S supplies the spec constructors: the product package (GPU arm) or the
    oracle (CPU arms) — both give the same table."""
    text, frames, tpf, bs = cfg["layout"]
    nb = -(-(text + frames * tpf) // bs)
    if cfg["mix"] is None:  # config 1 table
        return [S.full_spec(), S.diagonal_spec(1), S.multi_diagonal_spec(),
                S.vertical_stripe_spec(stripes=(0, 7)), S.skip_spec(), S.diagonal_spec(1),
                S.multi_diagonal_spec(), S.vertical_stripe_spec(stripes=(3, 40))]
    f, s, d, md, vs = cfg["mix"]
    rng = np.random.default_rng(2506_03065)
    stripes = [tuple(int(c) for c in rng.choice(nb, size=2, replace=False)) for _ in range(vs)]
    specs = ([S.full_spec()] * f + [S.skip_spec()] * s + [S.diagonal_spec(1)] * d +
             [S.multi_diagonal_spec()] * md + [S.vertical_stripe_spec(stripes=c) for c in stripes])
    order = rng.permutation(len(specs))
    return [specs[i] for i in order]


def config_dict(cfg, density: float, parallelism: str) -> dict:
    """The workload description both arms print (same keys, same values)."""
    H, d = cfg["heads"], cfg["d"]
    n = cfg["layout"][0] + cfg["layout"][1] * cfg["layout"][2]
    return {
        "workload": cfg["name"],
        "layout": {"text_tokens": cfg["layout"][0], "frames": cfg["layout"][1],
                   "tokens_per_frame": cfg["layout"][2], "block_size": cfg["layout"][3]},
        "tokens": n, "heads": H, "head_dim": d, "batch": 1,
        "mode_mix_F_S_D_MD_VS": cfg["mix"],
        "density": round(density, 4),
        "parallelism": parallelism,
        "l2": (("inputs 3 x %.0f MB bf16 > 126 MB L2: no flush" if H * n * d * 2 * 3 > 126e6 else
                "inputs 3 x %.1f MB bf16 fit in L2 (a parity-size case, not the metric's config)")
               % (H * n * d * 2 / 1e6)),
    }


def _oracle():
    """The CPU oracle — imported only by the CPU legs (cpu_baseline, the
    reference arm and the parity checker), never by the measured GPU path."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import svdit_oracle as O

    return O


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """SM clocks / throttle reasons sampled during the timed region: NVML
    polled every 20 ms from a thread (a 10-step region of ~40 ms steps gets
    ~20 samples), nvidia-smi -lms 100 if NVML is unavailable."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    # NVML clocks-event-reason bits (nvml.h)
    REASON_BITS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20,
                   "hw_thermal_slowdown": 0x40}

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []
        self.samples: list[tuple[float, int]] = []  # NVML: (sm MHz, reason bits)
        self.max_mhz = None
        self._stop = threading.Event()
        self._nvml = None

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            h = self._nvml_handle(pynvml)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
            self._nvml = (pynvml, h)
            self.thread = threading.Thread(target=self._poll, daemon=True)
            self.thread.start()
            return self
        except Exception:
            self._nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _nvml_handle(self, nv):
        """The NVML handle of torch's device `index` (by UUID: NVML indices
        ignore CUDA_VISIBLE_DEVICES); the NVML index as a fallback."""
        try:
            import torch

            uuid = str(torch.cuda.get_device_properties(self.index).uuid)
            return nv.nvmlDeviceGetHandleByUUID(("GPU-" + uuid) if not uuid.startswith("GPU-") else uuid)
        except Exception:
            return nv.nvmlDeviceGetHandleByIndex(self.index)

    def _poll(self):
        nv, h = self._nvml
        while not self._stop.is_set():
            try:
                mhz = float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
                try:
                    bits = int(nv.nvmlDeviceGetCurrentClocksEventReasons(h))
                except AttributeError:
                    bits = int(nv.nvmlDeviceGetCurrentClocksThrottleReasons(h))
                self.samples.append((mhz, bits))
            except Exception:
                pass
            self._stop.wait(0.02)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        self._stop.set()
        if self._nvml is not None:
            self.thread.join(timeout=1)
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        sm, mx, reasons = [], self.max_mhz, set()
        for mhz, bits in self.samples:
            sm.append(mhz)
            for name, bit in self.REASON_BITS.items():
                if bits & bit:
                    reasons.add(name)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for name, val in zip(names, parts[5:9]):
                if val.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm),
                "source": "nvml 20 ms" if self.samples else "nvidia-smi 100 ms"}


def measured_peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        obj = json.loads(p.read_text())
        return {"bf16": obj.get("bf16_tflops"), "bf16_sustained": obj.get("bf16_tflops_sustained"),
                "hbm": obj.get("hbm_gbs"), "source": "measured"}
    return {"bf16": 1590.0, "bf16_sustained": 1400.0, "hbm": 6650.0, "source": "fallback"}


def ncu_traffic(cfg_key: str):
    """dram bytes per launch of the fused kernel from the committed ncu capture."""
    p = ROOT / "profiles" / "ncu_summary.json"
    if not p.exists():
        return None
    try:
        obj = json.loads(p.read_text())
        return obj.get(cfg_key, {}).get("dram_bytes_per_launch")
    except (ValueError, OSError):
        return None


# ----------------------------------------------------------------- CPU baseline (oracle port)
_CPU = {}  # per-worker state of the CPU baseline (built once by _cpu_init)


def _cpu_init(layout, d, mode_specs):
    """Spawned-worker initializer: the oracle, the grid, seeded Q/K/V (one
    head at full N) and the per-mode masks — rebuilt in every worker, so the
    pool never inherits the parent's CUDA / BLAS thread state."""
    O = _oracle()
    og = O.block_grid(*layout)
    rng = np.random.default_rng(0)
    _CPU.update(O=O, grid=og,
                q=rng.standard_normal((1, 1, og.n, d), dtype=np.float32),
                k=rng.standard_normal((1, 1, og.n, d), dtype=np.float32),
                v=rng.standard_normal((1, 1, og.n, d), dtype=np.float32),
                active={m: O.build_mask(O.Spec(*sp), og) for m, sp in mode_specs.items()})


def _cpu_worker(args):
    """One process of the CPU baseline: the oracle's streaming attention on
    its share of the query blocks, one BLAS thread, until the time slice ends."""
    m, qbs, slice_s = args
    O = _CPU["O"]
    try:
        from threadpoolctl import threadpool_limits

        limiter = threadpool_limits(1)
    except ImportError:  # single-threaded BLAS anyway once forked per core
        limiter = None
    og, q, k, v = _CPU["grid"], _CPU["q"], _CPU["k"], _CPU["v"]
    active = _CPU["active"][m]
    d = q.shape[-1]
    t0 = time.perf_counter()
    done = 0.0
    nq = 0
    for qb in qbs:
        O.sparse_attention_rows(q, k, v, active, og.bounds, [int(qb)])
        rows = og.bounds[qb + 1] - og.bounds[qb]
        done += 4.0 * d * rows * float(np.diff(og.bounds)[active[qb]].sum())
        nq += 1
        if time.perf_counter() - t0 > slice_s:
            break
    if limiter is not None:
        limiter.restore_original_limits()
    return done, time.perf_counter() - t0, nq


class CpuBaseline:
    """The reference algorithm (fp64 streaming online softmax, the oracle port
    of attention.py:57-98) on this host's cores: bounded samples of query
    blocks of one head per distinct mode at full N, extrapolated to the whole
    layer by active FLOPs per mode.  Query blocks are independent
    (attention.py:81-97), so one spawned worker per core runs the unchanged
    per-block algorithm with one BLAS thread each.  The worker pool is built
    once and reused by every sample."""

    def __init__(self, cfg):
        import multiprocessing as mp

        O = _oracle()
        self.cfg = cfg
        self.og = og = O.block_grid(*cfg["layout"])
        self.d = cfg["d"]
        self.specs = assignment_for(cfg, O)
        per_mode = {}
        for spec in self.specs:
            per_mode.setdefault(int(spec.mode), spec)
        self.modes = [m for m in per_mode if m != O.SKIP]
        self.heads = {m: sum(1 for s in self.specs if int(s.mode) == m) for m in self.modes}
        pairs = {m: 0.0 for m in self.modes}
        dense_pairs = float(og.n) * float(og.n)
        for s in self.specs:  # masks are bit-exact with the plan builder's
            if int(s.mode) != O.SKIP:
                pairs[int(s.mode)] += O.active_pairs(O.build_mask(s, og), og.bounds)
        self.flops = {m: 4.0 * self.d * pairs[m] for m in self.modes}
        self.density = sum(pairs.values()) / (dense_pairs * len(self.specs))
        self.workers = max(1, os.cpu_count() or 1)
        self.rng = np.random.default_rng(1)
        ctx = mp.get_context("spawn")
        env_blas = {k: os.environ.get(k) for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS")}
        for k in env_blas:  # spawned workers start with single-threaded BLAS
            os.environ[k] = "1"
        try:
            self.pool = ctx.Pool(self.workers, initializer=_cpu_init,
                                 initargs=(cfg["layout"], self.d,
                                           {m: tuple(per_mode[m]) for m in self.modes}))
        finally:
            for k, val in env_blas.items():
                if val is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = val

    def sample(self, budget_s: float) -> dict:
        """One bounded sample (~budget_s of wall time on all workers)."""
        og, n, d = self.og, self.og.n, self.d
        slice_s = budget_s / max(1, len(self.modes))
        total_flops, total_time, sampled = 0.0, 0.0, []
        w0 = time.perf_counter()
        for m in self.modes:
            order = self.rng.permutation(og.n_blocks)
            shares = [order[w::self.workers] for w in range(self.workers)]
            res = self.pool.map(_cpu_worker, [(m, sh, slice_s) for sh in shares])
            done = sum(r[0] for r in res)
            wall = max(r[1] for r in res)
            nq = sum(r[2] for r in res)
            rate = done / wall
            total_flops += self.flops[m]
            total_time += self.flops[m] / rate
            sampled.append(f"{MODE_LABELS[m]}:{nq}qb/{self.heads[m]}h {rate / 1e9:.1f}GF/s")
        wall_ms = (time.perf_counter() - w0) * 1e3
        dense = 4.0 * n * n * d * self.cfg["heads"]
        return {
            "value": dense / total_time / 1e12,
            "unit": UNIT,
            "ms_per_layer": total_time * 1e3,
            "extrapolated": True,
            "sample_wall_ms": round(wall_ms, 1),
            "active_gflops_per_s": total_flops / total_time / 1e9,
            "cores": self.workers,
            "kind": "port",
            "sample": (f"fp64 NumPy oracle (attention.py:57-98 restated), 1 head per mode at full N={n}, "
                       f"random query blocks for ~{slice_s:.1f}s each on {self.workers} worker processes x "
                       f"1 BLAS thread [{'; '.join(sampled)}], layer time extrapolated by active FLOPs"),
        }

    def close(self):
        self.pool.close()
        self.pool.join()


def cpu_baseline(cfg, budget_s: float = 15.0) -> dict:
    cb = CpuBaseline(cfg)
    try:
        return cb.sample(budget_s)
    finally:
        cb.close()


def oracle_parity(cfg, q, k, v, out, specs, per_head: int = 4) -> dict:
    """Checker (outside the timed region): sampled output rows of the bench
    layer against the oracle — every head, query blocks chosen to cover the
    text / forced rows, a frame-border (mixed) block, an ordinary block and
    the partial tail — max-abs / mean-abs over the sampled elements, the
    north_star bar being 2e-2 / 2e-3 (bf16 output vs the fp32 reference)."""
    import torch

    O = _oracle()
    og = O.block_grid(*cfg["layout"])
    nb = og.n_blocks
    rng = np.random.default_rng(7)
    forced = np.flatnonzero(og.forced)
    mixed = np.flatnonzero(og.mixed & ~og.has_text)
    plain = np.flatnonzero(~og.forced[:-1])
    t0 = time.perf_counter()
    errs, n_el, rows = [], 0, 0
    worst = 0.0
    for h, spec in enumerate(specs):
        picks = {int(nb - 1)}
        if len(forced):
            picks.add(int(forced[0]))
        if len(mixed):
            picks.add(int(rng.choice(mixed)))
        while len(picks) < per_head:
            picks.add(int(rng.choice(plain)))
        qbs = sorted(picks)
        sel = np.concatenate([np.arange(og.bounds[b], og.bounds[b + 1]) for b in qbs])
        got = out[:, h:h + 1, torch.as_tensor(sel, device=out.device)].float().cpu().numpy()
        if int(spec.mode) == O.SKIP:
            want = np.zeros_like(got)
        else:
            hq, hk, hv = (x[:, h:h + 1].float().cpu().numpy() for x in (q, k, v))
            want = O.attention_rows(hq, hk, hv, O.build_mask(spec, og), og.bounds, qbs)
        e = np.abs(got - want)
        errs.append(float(e.sum()))
        n_el += e.size
        rows += len(sel)
        worst = max(worst, float(e.max()))
    return {"max_abs": worst, "mean_abs": sum(errs) / max(1, n_el), "tol_max_abs": 2e-2,
            "tol_mean_abs": 2e-3, "ok": bool(worst <= 2e-2 and sum(errs) / max(1, n_el) <= 2e-3),
            "rows_checked": rows, "heads_checked": len(specs), "seconds": round(time.perf_counter() - t0, 1),
            "how": ("fp64 oracle rows (oracle.attention_rows, attention.py:57-98 semantics) for "
                    f"{per_head} query blocks per head (text/forced, frame-border, ordinary, partial tail) "
                    "of the bench's own inputs and mode mix, against the timed kernel's bf16 output")}


# ----------------------------------------------------------------- GPU arm
def library_dense(q, k, v, dev, reps: int = 3):
    """Dense attention through torch SDPA on the same GPU and inputs — a
    library baseline beside our own dense sm_100a launch (first backend that
    runs: cuDNN, then flash, then memory-efficient)."""
    import torch
    import torch.nn.functional as F
    from torch.nn.attention import SDPBackend, sdpa_kernel

    for be in (SDPBackend.CUDNN_ATTENTION, SDPBackend.FLASH_ATTENTION, SDPBackend.EFFICIENT_ATTENTION):
        try:
            with sdpa_kernel([be]):
                o = F.scaled_dot_product_attention(q, k, v)
                torch.cuda.synchronize(dev)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                for _ in range(reps):
                    o = F.scaled_dot_product_attention(q, k, v)
                b.record()
                torch.cuda.synchronize(dev)
            del o
            return {"backend": f"torch SDPA {be.name}", "ms": round(a.elapsed_time(b) / reps, 3)}
        except Exception as exc:  # backend unavailable for this shape / build
            last = f"{be.name}: {type(exc).__name__}"
            torch.cuda.synchronize(dev)
    return {"backend": None, "ms": None, "error": last}


def _numpy_e2e(S, hq, hk, hv, groups, e2e_bytes):
    """The reference's own call with its own types: float32 NumPy in, float32
    NumPy out (attention.py:186-212), wall clock per call (1 GPU)."""
    try:
        nq, nk, nv = (t.float().numpy() for t in (hq, hk, hv))
        S.fused_layer_attention(nq, nk, nv, groups)
        walls = []
        for _ in range(3):
            w0 = time.perf_counter()
            S.fused_layer_attention(nq, nk, nv, groups)
            walls.append(round((time.perf_counter() - w0) * 1e3, 2))
        numpy_e2e = {"ms_per_layer": min(walls), "wall_ms_steps": walls,
                     "h2d_bytes_per_step": e2e_bytes[0], "d2h_bytes_per_step": e2e_bytes[1],
                     "path": ("fused_layer_attention(float32 NumPy q/k/v) -> float32 NumPy: converted to "
                              "bf16 on the host cores chunk by chunk into pinned staging, same pipeline")}
        del nq, nk, nv
        return numpy_e2e
    except Exception as exc:  # informational extra: never sink the bench line
        return {"error": f"{type(exc).__name__}: {exc}"}


def _search_step(S, layout, q, k, v, stream, dev):
    """The offline search's per-layer step on the bench layer (SURVEY §8f rows
    1-2, search.py:334-372): the first evaluation of a layer (stripe
    calibration: FULL + diagonal + multi-diagonal launch that also writes the
    row statistics, the key-sum pass, the stripe launch) and every later one
    (stripes frozen, search.py:338-346: ONE launch of all four candidates),
    beside the FULL candidate alone and the stand-alone two-pass key mass."""
    import torch

    from paper_2506_03065_b200.calibrate import CandidateEvaluator, block_key_mass

    grid = S.block_grid(layout)
    ev = CandidateEvaluator(grid, S.SearchParams())
    first = ev.evaluate(q, k, v)  # builds the candidate plans
    ev.evaluate(q, k, v, stripes=first.stripes)
    H, d = q.shape[1], q.shape[-1]
    full_plan = S.plan_for_assignment([S.full_spec()] * H, layout)
    o = torch.empty_like(q)
    full_plan.forward(q, k, v, o, head_dim=d)  # device tables uploaded outside the timed region
    ev_ = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    ev_[0].record(stream)
    block_key_mass(q, k, grid)
    ev_[1].record(stream)
    ev.evaluate(q, k, v)
    ev_[2].record(stream)
    ev.evaluate(q, k, v, stripes=first.stripes)
    ev_[3].record(stream)
    full_plan.forward(q, k, v, o, head_dim=d)
    ev_[4].record(stream)
    torch.cuda.synchronize(dev)
    full_ms = ev_[3].elapsed_time(ev_[4])
    steady = ev_[2].elapsed_time(ev_[3])
    return {"block_key_mass_ms": round(ev_[0].elapsed_time(ev_[1]), 2),
            "first_evaluation_ms": round(ev_[1].elapsed_time(ev_[2]), 2),
            "candidate_evaluation_ms": round(steady, 2),
            "full_candidate_alone_ms": round(full_ms, 2),
            "candidate_evaluation_over_full": round(steady / full_ms, 3),
            "what": "calibrate.CandidateEvaluator.evaluate: FULL / diagonal / multi-diagonal / stripe "
                    "candidates as (candidate, head) pairs of one fused launch + per-head fp64 MSE + "
                    "mode_loss / select_mode (search.py:334-372); first evaluation adds the stripe "
                    "calibration from the FULL launch's row statistics (key-sum pass only)"}


def init_dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl" if os.environ.get("SVD_BACKEND", "nccl") == "nccl" else "gloo")
    return world, rank, local


def run_ours(args):
    import torch

    import paper_2506_03065_b200 as S
    from paper_2506_03065_b200.sharding import HeadShardedLayer

    world, rank, local = init_dist()
    # SVD_FORCE_DEVICE: test harness only — put every rank on one GPU (with
    # SVD_BACKEND=gloo) to exercise the multi-rank path where one GPU exists
    local = int(os.environ.get("SVD_FORCE_DEVICE", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    cfg = CONFIGS[args.config]
    layout = S.TokenLayout(*cfg["layout"])
    n, H, d = layout.total_tokens, cfg["heads"], cfg["d"]
    specs = assignment_for(cfg, S)
    plan = S.plan_for_assignment(specs, layout)
    info = plan.info
    f_active = plan.active_flops(d)
    f_dense = plan.dense_flops(d)

    gen = torch.Generator(device=dev).manual_seed(1234)
    q = torch.randn(1, H, n, d, device=dev, generator=gen, dtype=torch.float32).to(torch.bfloat16)
    k = torch.randn(1, H, n, d, device=dev, generator=gen, dtype=torch.float32).to(torch.bfloat16)
    v = torch.randn(1, H, n, d, device=dev, generator=gen, dtype=torch.float32).to(torch.bfloat16)
    # N>1: the fused path (shard kernel stores rows into every rank's O over
    # peer memory) unless SVD_MULTI_GPU=nccl selects packed rows + NCCL
    # all-gather + unpack
    mgpu = os.environ.get("SVD_MULTI_GPU", "p2p") if world > 1 else "single"
    if mgpu == "p2p":
        import torch.distributed as dist

        from paper_2506_03065_b200.sharding import PeerShardedLayer

        try:
            layer = PeerShardedLayer(plan, world, rank, d, dev, (1, H, n, d))
            ok = 1
        except Exception as exc:  # no peer access between these GPUs: NCCL path
            print(f"rank {rank}: peer-memory path unavailable ({exc}); using NCCL all-gather",
                  file=sys.stderr)
            layer, ok = None, 0
        flag = torch.tensor([ok], device=dev)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        if int(flag[0]) == 1:
            out = layer.out
        else:
            if layer is not None:
                layer.close()
            mgpu = "nccl"
    if mgpu != "p2p":  # one GPU, or packed rows + NCCL all-gather + unpack
        layer = HeadShardedLayer(plan, world, rank, head_dim=d, device=dev)
        out = torch.empty(1, H, n, d, device=dev, dtype=torch.bfloat16)
    stream = torch.cuda.current_stream(dev)

    def barrier():
        if world > 1:
            import torch.distributed as dist

            dist.barrier()
        torch.cuda.synchronize(dev)

    # the peer layer double-buffers O: call it without out= and keep the result
    step = (lambda ev=None: layer(q, k, v, kernel_events=ev)) if mgpu == "p2p" else \
        (lambda ev=None: layer(q, k, v, out, kernel_events=ev))
    for _ in range(args.warmup):
        out = step()
    barrier()
    # kernel-only events around each fused launch (same stream) for the roofline
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(torch.cuda.current_device()) as clocks:
        barrier()
        t0.record(stream)
        for i in range(args.steps):
            out = step(kev[i])
        t1.record(stream)
        barrier()
    ms = t0.elapsed_time(t1) / args.steps
    kms = statistics.mean(a.elapsed_time(b) for a, b in kev)
    if world > 1:
        import torch.distributed as dist

        tt = torch.tensor([ms, kms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms, kms = float(tt[0]), float(tt[1])
    clock = clocks.summary()
    if not bool(torch.isfinite(out).all()):
        raise RuntimeError("non-finite values in the layer output")

    # end to end through the public API: pinned host Q/K/V in, O out, every step
    hq, hk, hv = (t.cpu().pin_memory() for t in (q, k, v))
    hout = torch.empty(out.shape, dtype=out.dtype).pin_memory()
    e2e_steps = max(1, min(args.steps, 5))
    groups = S.group_heads(specs, S.block_grid(layout))
    for _ in range(2):
        layer.e2e(hq, hk, hv, hout, groups)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2e_walls = []
    e0.record(stream)
    for _ in range(e2e_steps):
        w0 = time.perf_counter()
        layer.e2e(hq, hk, hv, hout, groups)
        e2e_walls.append(round((time.perf_counter() - w0) * 1e3, 2))
    e1.record(stream)
    barrier()
    e2e_ms = e0.elapsed_time(e1) / e2e_steps
    # bytes copied per step (whole job): one GPU pipelines every non-SKIP head's
    # Q/K/V in and O out; a peer-memory shard rank copies its own head range in
    # and out, an NCCL shard rank the full Q/K/V in and the full O out
    if world == 1:
        e2e_bytes = S.host_transfer_bytes(plan, 1, n, d)
    elif mgpu == "p2p":
        e2e_bytes = layer.e2e_bytes((1, H, n, d))
    else:
        e2e_bytes = (3 * H * n * d * 2, H * n * d * 2)
    # peer-memory bytes a rank's epilogue stores into the other ranks' O per
    # step (p2p), or receives through the NCCL all-gather (nccl)
    if world == 1:
        link_bytes = 0
    elif mgpu == "p2p":
        link_bytes = layer.nvlink_bytes(d)
    else:
        link_bytes = (world - 1) * layer.max_rows * layer.tensor_dim * 2
    if world > 1:
        import torch.distributed as dist

        lt = torch.tensor([float(link_bytes)], device=dev, dtype=torch.float64)
        dist.all_reduce(lt, op=dist.ReduceOp.MAX)
        link_bytes = int(lt[0])
        tt = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_ms = float(tt[0])
        bt = torch.tensor(list(e2e_bytes), device=dev, dtype=torch.float64)
        dist.all_reduce(bt, op=dist.ReduceOp.SUM)
        e2e_bytes = (int(bt[0]), int(bt[1]))

    # the reference's own call with its own types: float32 NumPy in, float32
    # NumPy out (attention.py:186-212), wall clock per call (1 GPU)
    numpy_e2e = None
    if world == 1:
        numpy_e2e = _numpy_e2e(S, hq, hk, hv, groups, e2e_bytes)

    # the offline search's per-layer step on this layer:
    # stripe calibration (block_key_mass) and the four-candidate evaluation
    search_step = None
    if world == 1 and not args.no_dense:
        try:
            search_step = _search_step(S, layout, q, k, v, stream, dev)
        except Exception as exc:  # informational extra: never sink the bench line
            search_step = {"error": f"{type(exc).__name__}: {exc}"}

    # dense sm_100a baseline on the same GPU: every head FULL through the same kernel
    dense_ms = None
    if not args.no_dense and world == 1:
        dplan = S.plan_for_assignment([S.full_spec()] * H, layout)
        dense_out = torch.empty_like(out)
        for _ in range(2):
            dplan.forward(q, k, v, dense_out, head_dim=d)
        torch.cuda.synchronize(dev)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        reps = 3
        for _ in range(reps):
            dplan.forward(q, k, v, dense_out, head_dim=d)
        b.record(stream)
        torch.cuda.synchronize(dev)
        dense_ms = a.elapsed_time(b) / reps
        del dense_out
    dense_lib = library_dense(q, k, v, dev) if (not args.no_dense and world == 1) else None

    # the checker: sampled rows of the timed output vs the oracle (not timed)
    parity = None
    if rank == 0 and not args.no_parity:
        try:
            parity = oracle_parity(cfg, q, k, v, out, specs)
        except Exception as exc:  # never sink the bench line; the gpu tests gate parity
            parity = {"error": f"{type(exc).__name__}: {exc}"}
    if rank != 0:
        return
    peaks = measured_peaks()
    # the fused kernel launch per rank handles 1/world of the active FLOPs
    achieved = f_active / world / (kms * 1e-3) / 1e12
    traffic = ncu_traffic(args.config)
    line = {
        "metric": METRIC,
        "value": round(f_dense / (ms * 1e-3) / 1e12, 2),
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms, 4),
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic (torch.randn Q/K/V, seed 1234)",
        "config": config_dict(cfg, f_active / f_dense, parallelism_label(mgpu, world)),
        "ms_per_layer": round(ms, 4),
        "active_tflops": round(f_active / (ms * 1e-3) / 1e12, 2),
        "kernel_ms": round(kms, 4),
        "dense_ms": round(dense_ms, 3) if dense_ms else None,
        "speedup_vs_dense": round(dense_ms / ms, 3) if dense_ms else None,
        "dense_library": dense_lib,
        "speedup_vs_dense_library": (round(dense_lib["ms"] / ms, 3)
                                     if dense_lib and dense_lib.get("ms") else None),
        "roofline": {
            "bound": "tensor",
            "achieved": round(achieved, 2),
            "peak": peaks["bf16"],
            "unit": "TFLOP/s",
            "frac": round(achieved / peaks["bf16"], 4),
            "traffic": traffic,
            "traffic_source": ("dram__bytes_read.sum + dram__bytes_write.sum per launch from the committed "
                               "ncu --set full capture of this kernel on this config (profiles/ncu_summary.json), "
                               "not measured in this run"),
            "peak_kind": f"{peaks['source']} burst cuBLAS bf16 (each ~40 ms launch is timed on its own)",
            "frac_of_sustained_peak": round(achieved / peaks["bf16_sustained"], 4),
            "sustained_peak": peaks["bf16_sustained"],
            "algorithmic_flops_per_launch": f_active / world,
            "issued_tile_flops_per_launch": info.computed_tiles * 4.0 * 128 * 128 * d / world,
        },
        "e2e": {
            "value": round(f_dense / (e2e_ms * 1e-3) / 1e12, 2),
            "unit": UNIT,
            "ms_per_layer": round(e2e_ms, 3),
            "wall_ms_steps": e2e_walls,
            "h2d_bytes_per_step": e2e_bytes[0],
            "d2h_bytes_per_step": e2e_bytes[1],
            "path": ("fused_layer_attention(pinned host bf16 Q/K/V, out=pinned O): heads reordered and "
                     "chunked by a flow-shop model, H2D / kernel / D2H streams overlapped; SKIP heads "
                     "never cross PCIe (zeros written on the host)") if world == 1 else
                    ("per rank: H2D of its own heads (equal-cost head partition, ~H/N heads per rank), "
                     "shard kernel storing rows into every rank's O over peer memory, D2H of its heads"
                     if mgpu == "p2p" else "per rank: full H2D, shard kernel, NCCL all-gather, full D2H"),
        },
        "e2e_reference_types": numpy_e2e,
        "search_step": search_step,
        "nvlink_bytes_per_rank_per_step": link_bytes,
        "gpu_launches": args.steps * (2 if mgpu in ("nccl", "p2p") and world > 1 else 1),
        "clocks": clock,
    }
    line["parity"] = parity
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(cfg, budget_s=args.cpu_budget)
    print(json.dumps(line), flush=True)


def parallelism_label(mgpu: str, world: int) -> str:
    return {"p2p": f"head/q-range sharded x{world}, rows stored to every rank's O "
                   "from the kernel epilogue over peer memory",
            "nccl": f"head/q-range sharded x{world} + NCCL all-gather + unpack",
            "single": "1 GPU"}[mgpu]


def run_reference(args):
    """--impl reference: the reference algorithm on the host cores (the oracle
    port — /root/reference is not available on the GPU box).
    Nothing from the product package is imported.  Each step is one bounded
    sample of the layer (every non-SKIP mode at full N, ~budget seconds on all
    cores); the layer time is extrapolated by active FLOPs and the line says
    so.  Under torchrun only rank 0 runs."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    world = int(os.environ.get("WORLD_SIZE", "1"))
    cfg = CONFIGS[args.config]
    budget = max(1.0, min(10.0, 120.0 / max(1, args.steps + args.warmup)))
    cb = CpuBaseline(cfg)
    try:
        for _ in range(args.warmup):
            cb.sample(budget)
        vals = [cb.sample(budget) for _ in range(args.steps)]
    finally:
        cb.close()
    value = statistics.median(v["value"] for v in vals)
    layer_ms = statistics.median(v["ms_per_layer"] for v in vals)
    step_ms = statistics.mean(v["sample_wall_ms"] for v in vals)
    base = dict(vals[0])
    base["value"] = value
    base["ms_per_layer"] = layer_ms
    mgpu = "single" if world == 1 else os.environ.get("SVD_MULTI_GPU", "p2p")
    line = {
        "metric": METRIC, "value": value, "unit": UNIT,
        "impl": "reference", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(step_ms, 1),
        "step": (f"one bounded sample of the layer: every non-SKIP mode's query blocks at full N for "
                 f"up to ~{budget:.1f} s on {base['cores']} cores; ms_per_step is that sample's wall time"),
        "ms_per_layer": round(layer_ms, 1), "extrapolated": True,
        "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded N(0,1) Q/K/V, one head per mode)",
        "config": config_dict(cfg, cb.density, parallelism_label(mgpu, world)),
        "cpu_baseline": base,
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="hunyuan")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-dense", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--no-parity", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)
    if int(os.environ.get("WORLD_SIZE", "1")) > 1:
        import torch.distributed as dist

        if dist.is_initialized():
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
