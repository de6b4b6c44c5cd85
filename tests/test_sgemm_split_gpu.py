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
    """(512, 512, 4096): 32 tiles of 128 x 64, KS = 4 (88 -> 63.5 us
    measured)."""
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


# (m, n, k) -> split factor of the built-in route (sgemm_tma.cu sgemm_split_ks
# on 148 SMs: fewest waves of work per SM, ties to the smaller factor)
ROUTE_KS = [
    ((4096, 128, 9216), 2),   # C3: 64 tiles
    ((768, 768, 2048), 2),    # 72 tiles
    ((512, 512, 4096), 4),    # 32 tiles
    ((300, 520, 4096), 4),    # 25 tiles
    ((1024, 1024, 1024), 1),  # C1: 128 tiles, more than half the SMs
    ((300, 520, 200), 1),     # too few K stages per rank
    ((64, 3136, 576), 1),     # C3b: 18 K stages, the 64x32 tiles instead
]


@pytest.mark.parametrize("shape,ks", ROUTE_KS)
def test_split_factor_rule_and_bits(ctx, shape, ks):
    m, n, k = shape
    rng = np.random.default_rng(m + n + k)
    av = rng.uniform(-1, 1, m * k).astype(np.float32)
    bv = rng.uniform(-1, 1, k * n).astype(np.float32)
    a, b = _buf(ctx, av), _buf(ctx, bv)
    c = tb.buffer_alloc(ctx, S, m * n)
    tb.gemm(ctx, Layout.ROW_MAJOR, Transpose.NO, Transpose.NO, m, n, k, 1.0, a, b, 0.0, c)
    kern = ctx.last_launch.native["kernel"]
    if ctx.device.compute_units == 148:
        assert (f"splitk{ks}" in kern) if ks > 1 else ("splitk" not in kern), kern
    want = np.zeros(m * n, np.float32)
    mt = re.search(r"_splitk(\d+)", kern)
    if mt:
        orc.seqk_gemm_split("S", True, False, False, m, n, k, 1.0, av, 0, k, bv, 0, n, 0.0, want, 0, n,
                            int(mt.group(1)))
    else:
        orc.seqk_gemm("S", True, False, False, m, n, k, 1.0, av, 0, k, bv, 0, n, 0.0, want, 0, n)
    assert tb.buffer_read(c, 0, m * n).tobytes() == want.tobytes(), kern
