"""im2col: oracle pinned to the reference's outputs, routine validation
(CPU; no GPU needed).  GPU parity lives in tests/test_im2col_gpu.py."""

import json

import numpy as np
import pytest

import paper_1705_05249_b200 as tb
from paper_1705_05249_b200 import Precision
from paper_1705_05249_b200.kernels.engine import launch_grid
from paper_1705_05249_b200.kernels.params import curated_configurations, default_config
from conftest import GOLDEN_DIR, HAS_GPU
from oracle import gemm_oracle as orc

META = json.loads((GOLDEN_DIR / "im2col_golden.json").read_text())
CASES = META["cases"]
ARR = np.load(GOLDEN_DIR / "im2col_golden.npz")


@pytest.mark.parametrize("i", range(len(CASES)))
def test_oracle_matches_reference_bitwise(i):
    cs = CASES[i]
    col = ARR[f"i{i}_col_in"].copy()
    orc.port_im2col(ARR[f"i{i}_im"], cs["im_off"], cs["c"], cs["h"], cs["w"], cs["kh"], cs["kw"],
                    cs["ph"], cs["pw"], cs["sh"], cs["sw"], cs["dh"], cs["dw"], col, cs["col_off"])
    assert np.array_equal(col.view(np.uint8), ARR[f"i{i}_col_out"].view(np.uint8))


def test_golden_covers_reference_test_geometries():
    geos = {(c["c"], c["h"], c["w"], c["kh"], c["kw"], c["ph"], c["pw"], c["sh"], c["sw"], c["dh"], c["dw"])
            for c in CASES}
    assert (1, 3, 3, 3, 3, 1, 1, 1, 1, 1, 1) in geos          # padding (test_extras.py:103)
    assert (3, 7, 8, 3, 2, 1, 0, 2, 1, 2, 1) in geos          # stride + dilation (:121)
    assert any(c["ph"] < 0 for c in CASES)                   # cropping
    assert any(c["im_off"] and c["col_off"] for c in CASES)  # offsets
    assert {c["prec"] for c in CASES} == {"S", "H"}


def test_validation_errors_match_reference(ctx):
    im = tb.buffer_alloc(ctx, Precision.S, 64)
    col = tb.buffer_alloc(ctx, Precision.S, 64)
    with pytest.raises(tb.UsageError, match="image and kernel dimensions must be >= 1"):
        tb.im2col(ctx, 0, 2, 2, 1, 1, 0, 0, 1, 1, 1, 1, im, col)
    with pytest.raises(tb.UsageError, match="strides and dilations must be >= 1"):
        tb.im2col(ctx, 1, 2, 2, 1, 1, 0, 0, 0, 1, 1, 1, im, col)
    # reference test_im2col_invalid_geometry (test_extras.py:141-145)
    with pytest.raises(tb.UsageError, match="convolution output dimensions are not positive"):
        tb.im2col(ctx, 1, 2, 2, 3, 3, 0, 0, 1, 1, 1, 1, im, col)
    with pytest.raises(tb.RangeError):
        tb.im2col(ctx, 1, 8, 9, 1, 1, 0, 0, 1, 1, 1, 1, im, col)          # image span 72 > 64
    with pytest.raises(tb.RangeError):
        tb.im2col(ctx, 1, 4, 4, 3, 3, 1, 1, 1, 1, 1, 1, im, col)          # col 9 x 16 > 64
    with pytest.raises(tb.RangeError):
        tb.im2col(ctx, 1, 4, 4, 1, 1, 0, 0, 1, 1, 1, 1, im, col, col_offset=60)
    half = tb.buffer_alloc(ctx, Precision.H, 64)
    with pytest.raises(tb.UsageError):
        tb.im2col(ctx, 1, 2, 2, 1, 1, 0, 0, 1, 1, 1, 1, im, half)


@pytest.mark.skipif(HAS_GPU, reason="checks the no-GPU failure mode")
def test_im2col_without_gpu_fails_loudly(ctx):
    im = tb.buffer_alloc(ctx, Precision.S, 16)
    col = tb.buffer_alloc(ctx, Precision.S, 16)
    with pytest.raises(tb.NativeLibraryError):
        tb.im2col(ctx, 1, 4, 4, 1, 1, 0, 0, 1, 1, 1, 1, im, col)


def test_transform_family_matches_reference_contract():
    dev = tb.host_device()
    cfg = default_config("transform", dev, Precision.S)      # TransformParams() (params.py:150-157)
    assert cfg.as_dict() == {"TDX": 16, "TDY": 16}
    g = launch_grid("transform", (27, 100), cfg)             # engine.py:79-84
    assert g.work_groups == (2, 7) and g.work_group_size == 256
    assert len(curated_configurations("transform")) == 9     # params.py:280-284
