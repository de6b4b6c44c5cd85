"""Netlib host-array layer == device routine, bitwise (reference tests/test_netlib.py:19-36)."""

import numpy as np
import pytest

import paper_1705_05249_b200 as tb
from paper_1705_05249_b200 import Layout, Precision, Transpose
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
