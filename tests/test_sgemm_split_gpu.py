"""The deterministic split-K SGEMM (csrc/sgemm_tma.cuh, KS > 1; routed by
sgemm_tma.cu sgemm_split_ks or a gemm_b200 SPLIT_K configuration): bitwise
equal to the sequential-k chain cut at the rank boundaries and summed in
rank order (oracle.seqk_gemm_split), for every layout; the split is a pure
function of (m, n, k), so batched equals looped bitwise."""

import re

import numpy as np
import pytest

import paper_1705_05249_b200 as tb
from paper_1705_05249_b200 import Layout, Precision, Transpose
from oracle import gemm_oracle as orc

pytestmark = pytest.mark.gpu
S = Precision.S


def _buf(ctx, arr):
    b = tb.buffer_alloc(ctx, S, arr.size)
    tb.buffer_write(b, 0, arr)
    return b


@pytest.mark.parametrize("layout", [Layout.ROW_MAJOR, Layout.COL_MAJOR])
@pytest.mark.parametrize("ta,tbn", [("n", "n"), ("t", "n"), ("n", "t")])
def test_mid_size_long_k_splits_bitwise(ctx, layout, ta, tbn):
    """(512, 512, 4096): 32 tiles of 128 x 64, KS = 4 (three quarters of a
    wave; 88 -> 63.5 us measured)."""
    T = {"n": Transpose.NO, "t": Transpose.YES}
    m, n, k = 512, 512, 4096
    rng = np.random.default_rng(77)
    av = rng.uniform(-1, 1, (m, k) if ta == "n" else (k, m)).astype(np.float32)
    bv = rng.uniform(-1, 1, (k, n) if tbn == "n" else (n, k)).astype(np.float32)
    order = "C" if layout is Layout.ROW_MAJOR else "F"
    a, b = _buf(ctx, av.reshape(-1, order=order)), _buf(ctx, bv.reshape(-1, order=order))
    lda = av.shape[1] if layout is Layout.ROW_MAJOR else av.shape[0]
    ldb = bv.shape[1] if layout is Layout.ROW_MAJOR else bv.shape[0]
    ldc = n if layout is Layout.ROW_MAJOR else m
    c = tb.buffer_alloc(ctx, S, m * n)
    tb.gemm(ctx, layout, T[ta], T[tbn], m, n, k, 1.0, a, b, 0.0, c, lda=lda, ldb=ldb, ldc=ldc)
    kern = ctx.last_launch.native["kernel"]
    got = tb.buffer_read(c, 0, m * n)
    mt = re.search(r"_splitk(\d+)", kern)
    want = np.zeros(m * n, np.float32)
    if mt:
        orc.seqk_gemm_split("S", layout is Layout.ROW_MAJOR, ta == "t", tbn == "t", m, n, k, 1.0,
                            av.reshape(-1, order=order), 0, lda, bv.reshape(-1, order=order), 0, ldb, 0.0,
                            want, 0, ldc, int(mt.group(1)))
    else:   # both operands K-contiguous: the register-staged kernel, unsplit
        orc.seqk_gemm("S", layout is Layout.ROW_MAJOR, ta == "t", tbn == "t", m, n, k, 1.0,
                      av.reshape(-1, order=order), 0, lda, bv.reshape(-1, order=order), 0, ldb, 0.0,
                      want, 0, ldc)
    assert got.tobytes() == want.tobytes(), kern


def test_split_batched_equals_loop_bitwise(ctx):
    m, n, k, batch = 512, 512, 4096, 3
    rng = np.random.default_rng(78)
    av = rng.uniform(-1, 1, batch * m * k).astype(np.float32)
    bv = rng.uniform(-1, 1, batch * k * n).astype(np.float32)
    a, b = _buf(ctx, av), _buf(ctx, bv)
    cb, cl = tb.buffer_alloc(ctx, S, batch * m * n), tb.buffer_alloc(ctx, S, batch * m * n)
    L, T = Layout.ROW_MAJOR, Transpose.NO
    tb.gemm_strided_batched(ctx, L, T, T, m, n, k, 1.0, a, m * k, b, k * n, 0.0, cb, m * n, batch)
    assert "splitk4" in ctx.last_launch.native["kernel"], ctx.last_launch.native
    for z in range(batch):
        tb.gemm(ctx, L, T, T, m, n, k, 1.0, a, b, 0.0, cl, a_offset=z * m * k, b_offset=z * k * n,
                c_offset=z * m * n)
        assert "splitk4" in ctx.last_launch.native["kernel"]
    assert tb.buffer_read(cb, 0, cb.length).tobytes() == tb.buffer_read(cl, 0, cl.length).tobytes()


def test_just_below_three_quarters_of_a_wave_is_not_split(ctx):
    # 128x64 tiles: 3 x 9 = 27 per instance, 27 * 4 < 0.75 * 148
    m, n, k = 300, 520, 4096
    rng = np.random.default_rng(79)
    a = _buf(ctx, rng.uniform(-1, 1, m * k).astype(np.float32))
    b = _buf(ctx, rng.uniform(-1, 1, k * n).astype(np.float32))
    c = tb.buffer_alloc(ctx, S, m * n)
    tb.gemm(ctx, Layout.ROW_MAJOR, Transpose.NO, Transpose.NO, m, n, k, 1.0, a, b, 0.0, c)
    if ctx.device.compute_units >= 148:
        assert "splitk" not in ctx.last_launch.native["kernel"], ctx.last_launch.native
