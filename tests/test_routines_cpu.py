"""Host-side argument validation of the GEMM routines — same checks, order
and error text as the reference (level3.py:106-133, extras.py:116-348) —
and the loud failure when no GPU is present (no CPU fallback)."""

import numpy as np
import pytest

import paper_1705_05249_b200 as tb
from paper_1705_05249_b200 import Layout, Precision, Transpose
from conftest import HAS_GPU

COL, NO = Layout.COL_MAJOR, Transpose.NO


def bufs(ctx, n=1000, prec=Precision.S):
    return [tb.buffer_alloc(ctx, prec, n) for _ in range(3)]


def test_gemm_validation_errors(ctx):
    a, b, c = bufs(ctx)
    with pytest.raises(tb.UsageError, match="dimensions must be >= 0"):
        tb.gemm(ctx, COL, NO, NO, -1, 2, 2, 1.0, a, b, 0.0, c)
    with pytest.raises(tb.UsageError, match="kernel must be"):
        tb.gemm(ctx, COL, NO, NO, 2, 2, 2, 1.0, a, b, 0.0, c, kernel="fast")
    with pytest.raises(tb.UsageError, match="leading dimension 3 < row count 4"):
        tb.gemm(ctx, COL, NO, NO, 4, 4, 4, 1.0, a, b, 0.0, c, lda=3)
    with pytest.raises(tb.RangeError, match="outside buffer of length 1000"):
        tb.gemm(ctx, COL, NO, NO, 40, 40, 40, 1.0, a, b, 0.0, c)
    with pytest.raises(tb.UsageError, match="complex scalar"):
        tb.gemm(ctx, COL, NO, NO, 4, 4, 4, 1j, a, b, 0.0, c)
    h = tb.buffer_alloc(ctx, Precision.H, 100)
    with pytest.raises(tb.UsageError, match="operand 1 has precision H"):
        tb.gemm(ctx, COL, NO, NO, 4, 4, 4, 1.0, a, h, 0.0, c)
    d = [tb.buffer_alloc(ctx, Precision.D, 100) for _ in range(3)]
    with pytest.raises(tb.UsageError, match="not supported by the B200 GEMM path"):
        tb.gemm(ctx, COL, NO, NO, 4, 4, 4, 1.0, *d[:2], 0.0, d[2])
    other = tb.context_create(tb.host_device())
    with pytest.raises(tb.UsageError, match="different context"):
        tb.gemm(other, COL, NO, NO, 4, 4, 4, 1.0, a, b, 0.0, c)


def test_zero_sizes_are_noops_without_range_checks(ctx):
    a = tb.buffer_alloc(ctx, Precision.S, 1)
    c = tb.buffer_alloc(ctx, Precision.S, 1)
    tb.buffer_write(c, 0, [7.0])
    tb.gemm(ctx, COL, NO, NO, 0, 0, 0, 1.0, a, a, 0.0, c)
    tb.gemm(ctx, COL, NO, NO, 5, 0, 5, 1.0, a, a, 0.0, c)
    assert c.data.tolist() == [7.0]


def test_row_major_views_checked_in_storage_orientation(ctx):
    a, b, c = bufs(ctx, 100)
    # row-major A (m=4, k=20): stored as col-major (20, 4) with ld >= 20
    with pytest.raises(tb.UsageError, match="leading dimension 10 < row count 20"):
        tb.gemm(ctx, Layout.ROW_MAJOR, NO, NO, 4, 4, 20, 1.0, a, b, 0.0, c, lda=10)


def test_batched_instance_named(ctx):
    a, b, c = bufs(ctx, 200)
    with pytest.raises(tb.UsageError, match="batched gemm instance 2: access"):
        tb.gemm_batched(ctx, COL, NO, NO, 4, 4, 4, [1.0] * 3, a, [0, 16, 190], b, [0, 16, 32],
                        [0.0] * 3, c, [0, 16, 32], 3)
    with pytest.raises(tb.UsageError, match="must all have length batch_count"):
        tb.gemm_batched(ctx, COL, NO, NO, 4, 4, 4, [1.0] * 2, a, [0, 16, 32], b, [0, 16, 32],
                        [0.0] * 3, c, [0, 16, 32], 3)
    with pytest.raises(tb.UsageError, match="batch_count must be >= 1"):
        tb.gemm_batched(ctx, COL, NO, NO, 4, 4, 4, [], a, [], b, [], [], c, [], 0)


def test_batched_overlap_rejected(ctx):
    a, b, c = bufs(ctx, 1000)
    with pytest.raises(tb.UsageError, match="overlap between instances 0 and 1"):
        tb.gemm_batched(ctx, COL, NO, NO, 8, 8, 8, [1.0, 1.0], a, [0, 64], b, [0, 64],
                        [0.0, 0.0], c, [0, 32], 2)
    # A and B may alias; C spans exactly adjacent are fine (validation only)
    if not HAS_GPU:
        with pytest.raises(tb.NativeLibraryError):
            tb.gemm_batched(ctx, COL, NO, NO, 8, 8, 8, [1.0, 1.0], a, [0, 0], b, [0, 0],
                            [0.0, 0.0], c, [0, 64], 2)


def test_strided_stride_too_small(ctx):
    a, b, c = bufs(ctx, 10000)
    with pytest.raises(tb.UsageError, match="stride_a = 63 smaller than one instance extent 64"):
        tb.gemm_strided_batched(ctx, COL, NO, NO, 8, 8, 8, 1.0, a, 63, b, 64, 0.0, c, 64, 4)
    with pytest.raises(tb.UsageError, match="stride_c"):
        tb.gemm_strided_batched(ctx, Layout.ROW_MAJOR, NO, NO, 8, 9, 8, 1.0, a, 64, b, 72, 0.0, c,
                                70, 4)


@pytest.mark.skipif(HAS_GPU, reason="checks the no-GPU behaviour")
def test_compute_without_gpu_fails_loudly(ctx):
    a, b, c = bufs(ctx, 64)
    with pytest.raises(tb.NativeLibraryError, match="no CPU fallback"):
        tb.gemm(ctx, COL, NO, NO, 4, 4, 4, 1.0, a, b, 0.0, c)
    with pytest.raises(tb.NativeLibraryError):
        tb.gemm_strided_batched(ctx, COL, NO, NO, 2, 2, 2, 1.0, a, 4, b, 4, 0.0, c, 4, 2)
    with pytest.raises(tb.NativeLibraryError):
        tb.netlib_call("sgemm", COL, NO, NO, 2, 2, 2, 1.0, np.zeros(4, np.float32),
                       np.zeros(4, np.float32), 0.0, np.zeros(4, np.float32), ctx=ctx)


def test_netlib_rejects_unknown_ids():
    with pytest.raises(tb.UsageError):
        tb.netlib_call("xgemm")
    with pytest.raises(tb.UsageError, match="not part of the B200 GEMM path"):
        tb.netlib_call("daxpy")


def test_netlib_split_predicates_mirror_the_native_rules():
    """The host-side mirrors netlib uses to decide whether a call may be cut
    (sub-blocks must take the same split-K decision as the whole call):
    hgemm.cu hgemm_split_ks and the S route's split eligibility on 148 SMs."""
    from paper_1705_05249_b200.routines import netlib

    # H: canonical column-major (m, n); C3 (4096, 128, 9216) row-major is (128, 4096)
    assert netlib._hgemm_split_ks(128, 4096, 9216, 148) == 4
    assert netlib._hgemm_split_ks(8192, 8192, 8192, 148) == 1
    assert netlib._hgemm_split_ks(512, 512, 16384, 148) == 4      # KS 8 only within a quarter of the SMs
    assert netlib._hgemm_split_ks(256, 256, 32768, 148) == 8
    assert netlib._hgemm_split_ks(1024, 1024, 1024, 148) == 1     # fewer than 32 K blocks per rank
    # S: may split only with at most half the SMs' worth of 128 x 64 tiles
    assert netlib._sgemm_may_split(128, 4096, 148)                # C3: 64 tiles
    assert netlib._sgemm_may_split(3136, 64, 148)                 # C3b: 25 tiles
    assert not netlib._sgemm_may_split(1024, 1024, 148)           # C1: 128 tiles
    assert not netlib._sgemm_may_split(8192, 8192, 148)
