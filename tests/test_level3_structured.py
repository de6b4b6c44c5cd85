"""Structured level-3 routines: argument checks and error text mirror the
reference (routines/level3.py:152-537); runs on CPU (no compute)."""

import pytest

import paper_1705_05249_b200 as tb
from paper_1705_05249_b200 import Diagonal, Layout, Precision, Side, Transpose, Triangle
from conftest import HAS_GPU

COL, ROW = Layout.COL_MAJOR, Layout.ROW_MAJOR


def bufs(ctx, *sizes, prec=Precision.S):
    return [tb.buffer_alloc(ctx, prec, s) for s in sizes]


def test_complex_only_routines_reject_real(ctx):
    a, b, c = bufs(ctx, 16, 16, 16)
    with pytest.raises(tb.UsageError, match="hemm is complex-only; use symm"):
        tb.hemm(ctx, COL, Side.LEFT, Triangle.UPPER, 4, 4, 1.0, a, b, 0.0, c)
    with pytest.raises(tb.UsageError, match="herk is complex-only; use syrk"):
        tb.herk(ctx, COL, Triangle.UPPER, Transpose.NO, 4, 4, 1.0, a, 0.0, c)
    with pytest.raises(tb.UsageError, match="her2k is complex-only; use syr2k"):
        tb.her2k(ctx, COL, Triangle.UPPER, Transpose.NO, 4, 4, 1.0, a, b, 0.0, c)


def test_negative_dimensions_and_noops(ctx):
    a, b, c = bufs(ctx, 16, 16, 16)
    with pytest.raises(tb.UsageError, match="dimensions must be >= 0"):
        tb.symm(ctx, COL, Side.LEFT, Triangle.UPPER, -1, 4, 1.0, a, b, 0.0, c)
    with pytest.raises(tb.UsageError, match="dimensions must be >= 0"):
        tb.syrk(ctx, COL, Triangle.UPPER, Transpose.NO, 4, -1, 1.0, a, 0.0, c)
    with pytest.raises(tb.UsageError, match="dimensions must be >= 0"):
        tb.trsm(ctx, COL, Side.LEFT, Triangle.UPPER, Transpose.NO, Diagonal.NON_UNIT, 4, -2, 1.0, a, b)
    # zero sizes return before any range check or GPU work (level3.py:163-164)
    tb.symm(ctx, COL, Side.LEFT, Triangle.UPPER, 0, 4, 1.0, a, b, 0.0, c)
    tb.syrk(ctx, COL, Triangle.UPPER, Transpose.NO, 0, 4, 1.0, a, 0.0, c)
    tb.trmm(ctx, ROW, Side.RIGHT, Triangle.LOWER, Transpose.YES, Diagonal.UNIT, 3, 0, 1.0, a, b)


def test_range_and_precision_errors(ctx):
    a, b, c = bufs(ctx, 8, 16, 16)
    with pytest.raises(tb.RangeError):      # A is 4 x 4 = 16 > 8
        tb.symm(ctx, COL, Side.LEFT, Triangle.UPPER, 4, 4, 1.0, a, b, 0.0, c)
    with pytest.raises(tb.RangeError):      # C 5 x 5 > 16
        tb.syrk(ctx, ROW, Triangle.LOWER, Transpose.YES, 5, 1, 1.0, b, 0.0, c)
    h = tb.buffer_alloc(ctx, Precision.H, 16)
    with pytest.raises(tb.UsageError):
        tb.trmm(ctx, COL, Side.LEFT, Triangle.UPPER, Transpose.NO, Diagonal.NON_UNIT, 4, 4, 1.0, b, h)
    with pytest.raises(tb.UsageError, match="leading dimension"):
        tb.trsm(ctx, COL, Side.LEFT, Triangle.UPPER, Transpose.NO, Diagonal.NON_UNIT, 4, 4, 1.0, b, c, lda=2)


@pytest.mark.skipif(HAS_GPU, reason="checks the no-GPU failure mode")
def test_structured_without_gpu_fails_loudly(ctx):
    a, b, c = bufs(ctx, 16, 16, 16)
    with pytest.raises(tb.NativeLibraryError):
        tb.symm(ctx, COL, Side.LEFT, Triangle.UPPER, 4, 4, 1.0, a, b, 0.0, c)
    with pytest.raises(tb.NativeLibraryError):
        tb.trsm(ctx, COL, Side.LEFT, Triangle.UPPER, Transpose.NO, Diagonal.NON_UNIT, 4, 4, 1.0, a, b)
