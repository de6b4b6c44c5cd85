"""Netlib host-array layer == device routine, bitwise (reference
tests/test_netlib.py:19-36), including the pipelined path: sub-blocks cut
along C's contiguous axis, pinned and pageable host arrays, leading
dimensions with gaps (elements outside C come back unchanged), beta != 0,
untransposable cuts, and the strided batched routine."""

import numpy as np
import pytest

import paper_1705_05249_b200 as tb
from paper_1705_05249_b200 import Layout, Precision, Transpose
from paper_1705_05249_b200.routines import netlib
from conftest import make_buffer

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("rid,prec", [("sgemm", Precision.S), ("hgemm", Precision.H)])
@pytest.mark.parametrize("layout", [Layout.COL_MAJOR, Layout.ROW_MAJOR])
def test_netlib_gemm_matches_device_call_bitwise(ctx, rid, prec, layout):
    rng = np.random.default_rng(100)
    m, n, k = 17, 13, 9
    av = rng.standard_normal((m, k)).astype(prec.dtype)
    bv = rng.standard_normal((k, n)).astype(prec.dtype)
    cv = rng.standard_normal((m, n)).astype(prec.dtype)
    c_host = cv.copy()
    tb.netlib_call(rid, layout, Transpose.NO, Transpose.NO, m, n, k, 1.5, av, bv, 0.5, c_host,
                   ctx=ctx)
    a, b, c = (make_buffer(ctx, x, prec, layout) for x in (av, bv, cv))
    tb.gemm(ctx, layout, Transpose.NO, Transpose.NO, m, n, k, 1.5, a, b, 0.5, c)
    flat = tb.buffer_read(c, 0, m * n)
    dev = flat.reshape((n, m)).T if layout is Layout.COL_MAJOR else flat.reshape((m, n))
    assert c_host.tobytes() == np.ascontiguousarray(dev).tobytes()


def test_netlib_default_context_and_zero_size():
    x = np.zeros(0, dtype=np.float32)
    tb.netlib_call("sgemm", Layout.COL_MAJOR, Transpose.NO, Transpose.NO, 0, 0, 0, 1.0, x, x, 0.0, x)
    assert tb.default_context() is tb.default_context()


def _flat(rng, n, prec, pinned):
    arr = netlib.pinned_empty(n, prec) if pinned else np.empty(n, prec.dtype)
    arr[:] = rng.uniform(-1, 1, n).astype(prec.dtype)
    return arr


@pytest.mark.parametrize("prec", [Precision.S, Precision.H])
@pytest.mark.parametrize("layout", [Layout.ROW_MAJOR, Layout.COL_MAJOR])
@pytest.mark.parametrize("ta,tbn", [("n", "n"), ("t", "t"), ("n", "t"), ("t", "n")])
@pytest.mark.parametrize("pinned", [True, False])
def test_pipelined_gemm_bitwise(ctx, monkeypatch, prec, layout, ta, tbn, pinned):
    """Large enough to be cut into sub-blocks (CHUNK_BYTES lowered), with
    offsets, gapped leading dimensions and beta != 0 on half the cases."""
    monkeypatch.setattr(netlib, "CHUNK_BYTES", 1 << 20)
    T = {"n": Transpose.NO, "t": Transpose.YES}
    m, n, k = 1100, 900, 700
    rng = np.random.default_rng(hash((prec.value, layout.name, ta, tbn, pinned)) % 2 ** 31)
    a_rows, a_cols = (m, k) if ta == "n" else (k, m)
    b_rows, b_cols = (k, n) if tbn == "n" else (n, k)
    row = layout is Layout.ROW_MAJOR
    lda = (a_cols if row else a_rows) + 3
    ldb = (b_cols if row else b_rows) + 5
    ldc = (n if row else m) + (2 if pinned else 0)
    a_off, b_off, c_off = 7, 3, 11
    a_len = a_off + lda * ((a_rows if row else a_cols) - 1) + (a_cols if row else a_rows) + 4
    b_len = b_off + ldb * ((b_rows if row else b_cols) - 1) + (b_cols if row else b_rows) + 4
    c_len = c_off + ldc * ((m if row else n) - 1) + (n if row else m) + 4
    av, bv, cv = _flat(rng, a_len, prec, pinned), _flat(rng, b_len, prec, pinned), _flat(rng, c_len, prec, pinned)
    beta = 0.5 if pinned else 0.0
    c_host = cv.copy()
    kw = dict(a_offset=a_off, lda=lda, b_offset=b_off, ldb=ldb, c_offset=c_off, ldc=ldc)
    rid = "sgemm" if prec is Precision.S else "hgemm"
    tb.netlib_call(rid, layout, T[ta], T[tbn], m, n, k, 1.25, av, bv, beta, c_host, ctx=ctx, **kw)
    a, b, c = (make_buffer(ctx, x, prec) for x in (av, bv, cv))
    tb.gemm(ctx, layout, T[ta], T[tbn], m, n, k, 1.25, a, b, beta, c, **kw)
    want = tb.buffer_read(c, 0, c_len)
    assert c_host.tobytes() == want.tobytes()


@pytest.mark.parametrize("prec", [Precision.S, Precision.H])
@pytest.mark.parametrize("pinned", [True, False])
def test_pipelined_strided_batched_bitwise(ctx, monkeypatch, prec, pinned):
    monkeypatch.setattr(netlib, "CHUNK_BYTES", 1 << 18)
    s, batch = 48, 700
    e = s * s
    rng = np.random.default_rng(3)
    av, bv = _flat(rng, batch * e, prec, pinned), _flat(rng, batch * e, prec, pinned)
    stride_c = e + 16                                   # gaps between instances of C
    cv = _flat(rng, batch * stride_c, prec, pinned)
    c_host = cv.copy()
    rid = "sgemm_strided_batched" if prec is Precision.S else "hgemm_strided_batched"
    tb.netlib_call(rid, Layout.ROW_MAJOR, Transpose.NO, Transpose.NO, s, s, s, 1.0, av, e, bv, e, 0.0,
                   c_host, stride_c, batch, ctx=ctx)
    a, b, c = (make_buffer(ctx, x, prec) for x in (av, bv, cv))
    tb.gemm_strided_batched(ctx, Layout.ROW_MAJOR, Transpose.NO, Transpose.NO, s, s, s, 1.0, a, e, b, e,
                            0.0, c, stride_c, batch)
    assert c_host.tobytes() == tb.buffer_read(c, 0, cv.size).tobytes()


def test_pipelined_hgemm_split_shapes_stay_bitwise(ctx, monkeypatch):
    """A shape whose sub-blocks would take the split-K route is not cut."""
    monkeypatch.setattr(netlib, "CHUNK_BYTES", 1 << 16)
    prec = Precision.H
    m, n, k = 1024, 128, 8192
    rng = np.random.default_rng(8)
    av, bv = _flat(rng, m * k, prec, True), _flat(rng, k * n, prec, True)
    c_host = np.zeros(m * n, np.float16)
    tb.netlib_call("hgemm", Layout.ROW_MAJOR, Transpose.NO, Transpose.NO, m, n, k, 1.0, av, bv, 0.0,
                   c_host, ctx=ctx)
    a, b = make_buffer(ctx, av, prec), make_buffer(ctx, bv, prec)
    c = tb.buffer_alloc(ctx, prec, m * n)
    tb.gemm(ctx, Layout.ROW_MAJOR, Transpose.NO, Transpose.NO, m, n, k, 1.0, a, b, 0.0, c)
    assert c_host.tobytes() == tb.buffer_read(c, 0, m * n).tobytes()


@pytest.mark.parametrize("shape", [(4096, 128, 9216), (2048, 2048, 1024), (64, 3136, 576)])
def test_pipelined_sgemm_split_shapes_stay_bitwise(ctx, monkeypatch, shape):
    """SGEMM: a call whose whole problem may take a split-K route (C3
    (4096, 128, 9216) splits in two) is not cut; a cut call's sub-blocks run
    unsplit, as its whole problem does.  Bitwise the device call either way."""
    monkeypatch.setattr(netlib, "CHUNK_BYTES", 1 << 16)
    prec = Precision.S
    m, n, k = shape
    rng = np.random.default_rng(m + n + k)
    av, bv = _flat(rng, m * k, prec, True), _flat(rng, k * n, prec, True)
    c_host = np.zeros(m * n, np.float32)
    tb.netlib_call("sgemm", Layout.ROW_MAJOR, Transpose.NO, Transpose.NO, m, n, k, 1.0, av, bv, 0.0,
                   c_host, ctx=ctx)
    a, b = make_buffer(ctx, av, prec), make_buffer(ctx, bv, prec)
    c = tb.buffer_alloc(ctx, prec, m * n)
    tb.gemm(ctx, Layout.ROW_MAJOR, Transpose.NO, Transpose.NO, m, n, k, 1.0, a, b, 0.0, c)
    assert c_host.tobytes() == tb.buffer_read(c, 0, m * n).tobytes()


def test_netlib_errors_match_device_routine(ctx):
    """Validation happens on the whole call before any copy, with the device
    routine's errors."""
    x = np.zeros(10, np.float32)
    with pytest.raises(tb.RangeError):
        tb.netlib_call("sgemm", Layout.COL_MAJOR, Transpose.NO, Transpose.NO, 4, 4, 4, 1.0, x, x, 0.0,
                       np.zeros(16, np.float32), ctx=ctx)
    with pytest.raises(tb.UsageError, match="leading dimension"):
        tb.netlib_call("sgemm", Layout.COL_MAJOR, Transpose.NO, Transpose.NO, 2, 2, 2, 1.0, x, x, 0.0, x,
                       lda=1, ctx=ctx)
