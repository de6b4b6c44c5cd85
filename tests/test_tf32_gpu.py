"""Opt-in TF32 tensor-core SGEMM (north star: "a TF32 tensor-core variant only
as an explicitly separate flag").  Tolerance: inputs carry 10 mantissa bits,
so 4*2^-10*K*max|a||b| (the FP16 bound) instead of the FP32 one."""

import numpy as np
import pytest

import paper_1705_05249_b200 as tb
from paper_1705_05249_b200 import Layout, Precision, Transpose
from conftest import make_buffer, rand_array, read_mat
from oracle import gemm_oracle as orc

pytestmark = pytest.mark.gpu
T = {"n": Transpose.NO, "t": Transpose.YES}
L = {"col": Layout.COL_MAJOR, "row": Layout.ROW_MAJOR}


def tf32_tol(alpha, beta, a_op, b_op, c):
    tol = abs(alpha) * 4 * 2.0 ** -10 * a_op.shape[1] * (
        np.abs(a_op).max(1, keepdims=True).astype(np.float64) * np.abs(b_op).max(0, keepdims=True))
    return tol + 4 * 2.0 ** -23 * np.abs(beta * c.astype(np.float64)) + 1e-30


# every layout: K-major operands (SWIZZLE_128B) and MN-major ones
# (SWIZZLE_128B_ATOM_32B / descriptor layout SWIZZLE_128B_BASE32B)
@pytest.mark.parametrize("layout", ["col", "row"])
@pytest.mark.parametrize("ta,tbn", [("n", "n"), ("n", "t"), ("t", "n"), ("t", "t")])
@pytest.mark.parametrize("shape", [(512, 640, 256), (300, 200, 132), (1024, 1024, 1024), (4096, 4096, 2048)])
def test_tf32_matches_float64(ctx, layout, ta, tbn, shape):
    """Within the TF32 tolerance of the float64 product in every layout."""
    m, n, k = shape
    rng = np.random.default_rng(m + n)
    av = rand_array(rng, (m, k) if ta == "n" else (k, m), Precision.S)
    bv = rand_array(rng, (k, n) if tbn == "n" else (n, k), Precision.S)
    cv = rand_array(rng, (m, n), Precision.S)
    a, b, c = (make_buffer(ctx, x, Precision.S, L[layout]) for x in (av, bv, cv))
    tb.gemm(ctx, L[layout], T[ta], T[tbn], m, n, k, 1.5, a, b, -0.5, c, tf32=True)
    assert ctx.last_launch.native["kernel"].startswith("sgemm_tf32_tc")
    a_op = av if ta == "n" else av.T
    b_op = bv if tbn == "n" else bv.T
    want = orc.wide_oracle(1.5, a_op, b_op, -0.5, cv)
    assert orc.allclose_tol(read_mat(c, (m, n), L[layout]), want, tf32_tol(1.5, -0.5, a_op, b_op, cv))


def test_tf32_strided_batched_and_default_is_ffma(ctx):
    rng = np.random.default_rng(7)
    s, batch = 128, 40
    e = s * s
    av, bv = rand_array(rng, batch * e, Precision.S), rand_array(rng, batch * e, Precision.S)
    a, b = make_buffer(ctx, av, Precision.S), make_buffer(ctx, bv, Precision.S)
    c = tb.buffer_alloc(ctx, Precision.S, batch * e)
    tb.gemm_strided_batched(ctx, Layout.ROW_MAJOR, Transpose.NO, Transpose.YES, s, s, s, 1.0, a, e,
                            b, e, 0.0, c, e, batch, tf32=True)
    assert ctx.last_launch.native["kernel"].startswith("sgemm_tf32_tc")
    got = tb.buffer_read(c, 0, batch * e)
    for z in (0, 17, batch - 1):
        A = av[z * e:(z + 1) * e].reshape(s, s)
        B = bv[z * e:(z + 1) * e].reshape(s, s).T
        want = orc.wide_oracle(1.0, A, B, 0.0, None)
        assert orc.allclose_tol(got[z * e:(z + 1) * e].reshape(s, s), want, tf32_tol(1.0, 0.0, A, B, want))
    # without the flag the FFMA path runs and differs from TF32
    c2 = tb.buffer_alloc(ctx, Precision.S, batch * e)
    tb.gemm_strided_batched(ctx, Layout.ROW_MAJOR, Transpose.NO, Transpose.YES, s, s, s, 1.0, a, e,
                            b, e, 0.0, c2, e, batch)
    assert not ctx.last_launch.native["kernel"].startswith("sgemm_tf32")
    assert tb.buffer_read(c2, 0, batch * e).tobytes() != got.tobytes()


def test_tf32_rejections(ctx):
    h = tb.buffer_alloc(ctx, Precision.H, 64)
    with pytest.raises(tb.UsageError, match="Precision.S only"):
        tb.gemm(ctx, Layout.COL_MAJOR, Transpose.NO, Transpose.NO, 4, 4, 4, 1.0, h, h, 0.0, h, tf32=True)
    a = tb.buffer_alloc(ctx, Precision.S, 200)
    with pytest.raises(tb.NativeLibraryError, match="16-byte aligned"):
        tb.gemm(ctx, Layout.COL_MAJOR, Transpose.YES, Transpose.NO, 5, 5, 5, 1.0, a, a, 0.0, a,
                a_offset=1, tf32=True)
    b = tb.buffer_alloc(ctx, Precision.S, 256)
    with pytest.raises(tb.NativeLibraryError, match="16-byte aligned"):
        tb.gemm(ctx, Layout.COL_MAJOR, Transpose.NO, Transpose.NO, 8, 8, 8, 1.0, b, b, 0.0, b, lda=9,
                tf32=True)


@pytest.mark.parametrize("layout", ["col", "row"])
def test_tf32_all_layouts_agree(ctx, layout):
    """The MN-major and K-major staging feed the same tensor-core products:
    the four transpose combinations of one mathematical product agree
    within the TF32 tolerance of each other (2x) and of float64."""
    m, n, k = 384, 320, 512
    rng = np.random.default_rng(21)
    A = rand_array(rng, (m, k), Precision.S)
    B = rand_array(rng, (k, n), Precision.S)
    want = orc.wide_oracle(1.0, A, B, 0.0, None)
    tol = tf32_tol(1.0, 0.0, A, B, want)
    outs = []
    for ta in ("n", "t"):
        for tbn in ("n", "t"):
            a = make_buffer(ctx, A if ta == "n" else np.ascontiguousarray(A.T), Precision.S, L[layout])
            b = make_buffer(ctx, B if tbn == "n" else np.ascontiguousarray(B.T), Precision.S, L[layout])
            c = tb.buffer_alloc(ctx, Precision.S, m * n)
            tb.gemm(ctx, L[layout], T[ta], T[tbn], m, n, k, 1.0, a, b, 0.0, c, tf32=True)
            got = read_mat(c, (m, n), L[layout])
            assert orc.allclose_tol(got, want, tol), (ta, tbn)
            outs.append(got)
    for o in outs[1:]:
        assert orc.allclose_tol(o, outs[0], tol, scale=2.0)
