"""Shared test helpers.  `-m gpu` tests need a B200; everything else runs on CPU."""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))

GOLDEN = Path(__file__).resolve().parent / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (sm_100a) device")


@pytest.fixture(scope="session")
def golden_plan():
    return np.load(GOLDEN / "golden_plan.npz")


@pytest.fixture(scope="session")
def golden_attn():
    return np.load(GOLDEN / "golden_attn.npz")


def decode_spec(row):
    """Golden spec row -> product PatternSpec (see make_golden.spec_row)."""
    import paper_2506_03065_b200 as S

    mode, hw, period, mdhw, count, incl, ns = (int(x) for x in row[:7])
    stripes = None if ns < 0 else tuple(int(x) for x in row[7:7 + ns])
    return S.PatternSpec(mode=S.Mode(mode), halfwidth=hw, period=None if period < 0 else period,
                         md_halfwidth=mdhw, stripe_count=count, stripes=stripes,
                         include_diagonal=bool(incl))


def unpack_mask(packed, nb):
    return np.unpackbits(packed)[: nb * nb].reshape(nb, nb).astype(bool)


def gpu_available() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False
