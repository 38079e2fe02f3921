"""The C-ABI library loads without a GPU and exports every symbol that
include/svdit_b200.h declares; status codes map onto the reference's
exception classes.  No compute calls (CPU only)."""

import ctypes
import re
from pathlib import Path

import pytest

import paper_2506_03065_b200 as S
from paper_2506_03065_b200 import _native as nat

HEADER = Path(__file__).resolve().parent.parent / "include" / "svdit_b200.h"


def declared_symbols():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"\b(svd_[a-z_0-9]+)\s*\(", text)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for want in ("svd_grid_arrays", "svd_mask_build", "svd_plan_create", "svd_plan_create_from_masks",
                 "svd_attn_fwd", "svd_plan_shard", "svd_unpack_rows", "svd_last_error"):
        assert want in syms


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(str(nat.LIB_PATH))
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_binding_covers_every_declared_symbol():
    assert set(declared_symbols()) == set(nat.SIGNATURES)


def test_version_string():
    assert b"sm_100a" in nat.lib().svd_version()


@pytest.mark.parametrize("status,exc", [(1, S.ShapeError), (2, S.DegenerateRowError),
                                        (3, S.DegenerateMaskError), (4, S.ConfigError),
                                        (5, nat.NativeError), (6, nat.NativeError)])
def test_status_mapping(status, exc):
    with pytest.raises(exc):
        nat.check(status)


def test_plan_create_from_masks_rejects_empty_row():
    layout = S.TokenLayout(0, 4, 64, 64)
    import numpy as np

    m = np.eye(4, dtype=bool)
    m[2, 2] = False
    with pytest.raises(S.DegenerateRowError):
        S.LayerPlan.from_masks(layout, [m], [0])


def test_block_key_mass_argument_checks_without_a_gpu():
    """svd_block_key_mass validates its arguments before touching the device;
    svd_key_mass_workspace sizes (-m, 1/l) rows + fp64 key sums per 128-token tile."""
    lib = nat.lib()
    assert lib.svd_key_mass_workspace(1, 24, 119056) == 24 * 931 * (256 * 4 + 128 * 8)
    assert lib.svd_key_mass_workspace(0, 1, 1) == 0
    st = nat.i64x4((128, 128, 128, 1))
    dummy = ctypes.c_void_p(16)

    def call(q=dummy, k=dummy, batch=1, heads=1, n=128, head_dim=64, tensor_dim=64, block=64, dtype=0,
             ws=dummy, ws_bytes=1 << 20, mass=dummy):
        return lib.svd_block_key_mass(q, k, st, st, batch, heads, n, head_dim, tensor_dim, block, dtype,
                                      ws, ws_bytes, mass, None)

    assert call(q=None) == 4                      # NULL tensor -> ConfigError
    assert call(dtype=1) == 6                     # fp16 unsupported
    assert call(batch=0) == 1                     # bad shape
    assert call(block=0) == 4
    assert call(head_dim=96, tensor_dim=64) == 1  # head_dim > tensor_dim
    assert call(ws_bytes=100) == 4                # workspace too small
    assert b"workspace" in lib.svd_last_error()
    assert call(tensor_dim=96, head_dim=96) == 6  # tensor width 64 or 128 only
