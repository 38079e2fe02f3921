"""The B200 latency model fitted on the config-5 sweep (single-mode layers,
profiles/r1/costmodel_sweep.json) predicts the mixed production layers it
never saw, and plugs into the search's sparsity slot.  CPU only."""

import json
from pathlib import Path

import pytest

import bench
import paper_2506_03065_b200 as S

ROOT = Path(__file__).resolve().parent.parent

# kernel-only B200 measurements of the current build (profiles/r1/costmodel_sweep.log run,
# scripts/time_layers.py, same session as the sweep's kernel version)
MEASURED_MS = {"hunyuan": 39.04, "cogvideo": 35.95, "wan": 42.42}


def test_shipped_fit_exists_and_is_sane():
    m = S.B200LatencyModel.default()
    assert "config 5" in m.source
    assert set(m.ms_per_tile) == {64, 128}
    fit = json.loads((ROOT / "profiles" / "r1" / "costmodel_sweep.json").read_text())["fit"]
    # RMS fit over 45 / 18 single-mode points; sub-2 ms points are noisy
    assert fit["128"]["rms_rel_err"] < 0.2 and fit["64"]["rms_rel_err"] < 0.2
    assert fit["128"]["max_rel_err"] < 0.4 and fit["64"]["max_rel_err"] < 0.4


@pytest.mark.parametrize("cfg", sorted(MEASURED_MS))
def test_predicts_mixed_layers(cfg):
    m = S.B200LatencyModel.default()
    c = bench.CONFIGS[cfg]
    plan = S.plan_for_assignment(bench.assignment_for(c, S), S.TokenLayout(*c["layout"]))
    pred = m.predict_plan_ms(plan, c["d"])
    assert abs(pred - MEASURED_MS[cfg]) / MEASURED_MS[cfg] < 0.10


def test_effective_sparsity_orders_modes():
    """Latency-weighted sparsity: FULL 0 < multi-diag < diag, all in [0, 1]."""
    m = S.B200LatencyModel.default()
    layout = S.TokenLayout(256, 33, 3600, 64)
    full = S.plan_for_assignment([S.full_spec()], layout).info.computed_tiles
    diag = S.plan_for_assignment([S.diagonal_spec(1)], layout).info.computed_tiles
    md = S.plan_for_assignment([S.multi_diagonal_spec()], layout).info.computed_tiles
    s_full = m.effective_sparsity(full, full, 128)
    s_diag = m.effective_sparsity(diag, full, 128)
    s_md = m.effective_sparsity(md, full, 128)
    assert s_full == 0.0 and 0 < s_md < s_diag < 1
