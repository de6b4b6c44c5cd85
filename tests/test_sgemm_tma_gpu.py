"""TMA-fed FFMA2 SGEMM (csrc/sgemm_tma.cuh): bitwise parity with the C
sequential-k oracle on every route (big 128x128 / 64x128 tiles, 64x64 tiles,
K tails, ragged M/N, strided batches through 3-D tensor maps), and bitwise
agreement with the cp.async / register-staged kernels it replaces (reference
contract: all S paths reproduce one another, tests/test_extras.py:213-297)."""

import numpy as np
import pytest

import paper_1705_05249_b200 as tb
from paper_1705_05249_b200 import Layout, Precision, Transpose
from oracle import gemm_oracle as orc

pytestmark = pytest.mark.gpu
S = Precision.S
L = {"col": Layout.COL_MAJOR, "row": Layout.ROW_MAJOR}
T = {"n": Transpose.NO, "t": Transpose.YES}


def _run(ctx, layout, ta, tbn, m, n, k, alpha, beta, seed, a_pad=None, b_pad=None, flags=None):
    """a_pad / b_pad None: pad the leading dimensions to multiples of 4 floats
    (16-byte tensor-map strides) so the TMA kernel is eligible."""
    rng = np.random.default_rng(seed)
    row = layout == "row"
    a_rows, a_cols = (k, m) if ta == "t" else (m, k)
    b_rows, b_cols = (n, k) if tbn == "t" else (k, n)
    lda = a_cols if row else a_rows
    ldb = b_cols if row else b_rows
    lda += (-lda) % 4 if a_pad is None else a_pad
    ldb += (-ldb) % 4 if b_pad is None else b_pad
    ldc = n if row else m
    a = rng.uniform(-1, 1, lda * ((a_rows if row else a_cols))).astype(np.float32)
    b = rng.uniform(-1, 1, ldb * ((b_rows if row else b_cols))).astype(np.float32)
    c = rng.uniform(-1, 1, m * n).astype(np.float32)
    bufs = []
    for x in (a, b, c):
        buf = tb.buffer_alloc(ctx, S, x.size)
        tb.buffer_write(buf, 0, x)
        bufs.append(buf)
    kw = {} if flags is None else {"kernel": flags}
    tb.gemm(ctx, L[layout], T[ta], T[tbn], m, n, k, alpha, bufs[0], bufs[1], beta, bufs[2],
            lda=lda, ldb=ldb, ldc=ldc, **kw)
    got = tb.buffer_read(bufs[2], 0, m * n)
    want = c.copy()
    orc.seqk_gemm("S", row, ta == "t", tbn == "t", m, n, k, alpha, a, 0, lda, b, 0, ldb, beta, want, 0,
                  ldc)
    rec = ctx.last_launch
    return got, want, (rec.native or {}).get("kernel", "") if rec is not None else ""


def _canonical_is_both_k(layout, ta, tbn):
    # row-major swaps the operands: canonical A' = op(B)^T, B' = op(A)^T
    if layout == "col":
        return ta == "t" and tbn == "n"
    return tbn == "t" and ta == "n"


@pytest.mark.parametrize("layout", ["col", "row"])
@pytest.mark.parametrize("ta", ["n", "t"])
@pytest.mark.parametrize("tbn", ["n", "t"])
def test_big_tiles_bitwise(ctx, layout, ta, tbn):
    # >= 4 waves of 128x128 tiles, K tail of 13 after two full 32-deep stages
    m, n, k = 3072, 3200, 77   # ld of 77 padded to 80
    got, want, kern = _run(ctx, layout, ta, tbn, m, n, k, 1.25, -0.75, 11)
    assert got.tobytes() == want.tobytes()
    assert kern.startswith("sgemm_tma_"), kern


@pytest.mark.parametrize("layout", ["col", "row"])
@pytest.mark.parametrize("ta", ["n", "t"])
@pytest.mark.parametrize("tbn", ["n", "t"])
@pytest.mark.parametrize("shape", [(200, 300, 333), (130, 67, 32), (1000, 12, 65), (65, 129, 1)])
def test_mid_tiles_ragged_bitwise(ctx, layout, ta, tbn, shape):
    m, n, k = shape
    got, want, kern = _run(ctx, layout, ta, tbn, m, n, k, 0.5, 2.0, sum(shape))
    assert got.tobytes() == want.tobytes(), kern
    assert kern.startswith("sgemm_tma_"), kern
    # both operands K-contiguous: A goes through the shared-memory transpose
    assert ("_kk" in kern) == _canonical_is_both_k(layout, ta, tbn), kern


def test_padded_leading_dims_and_beta_zero(ctx):
    got, want, kern = _run(ctx, "col", "n", "n", 257, 190, 131, 1.0, 0.0, 3, a_pad=11, b_pad=5)  # lda 268, ldb 136
    assert kern.startswith("sgemm_tma_")
    assert got.tobytes() == want.tobytes()


def test_unaligned_ld_repacked_bitwise(ctx):
    # lda not a multiple of 4 floats: no tensor map over the operand as given
    # (16-byte strides); it is copied once into aligned scratch and the TMA
    # kernel runs on the copy ("+pack"), still matching bitwise
    got, want, kern = _run(ctx, "col", "n", "n", 257, 190, 131, 1.0, 0.5, 4, a_pad=1)
    assert kern.startswith("sgemm_tma_") and kern.endswith("+pack"), kern
    assert got.tobytes() == want.tobytes()


def test_tma_equals_general_kernel_bitwise(ctx):
    a_g, _, k1 = _run(ctx, "row", "n", "n", 300, 260, 100, 1.0, 0.0, 9)
    b_g, _, k2 = _run(ctx, "row", "n", "n", 300, 260, 100, 1.0, 0.0, 9, flags="direct")
    assert k1.startswith("sgemm_tma_") and not k2.startswith("sgemm_tma_")
    assert a_g.tobytes() == b_g.tobytes()


@pytest.mark.parametrize("layout", ["col", "row"])
def test_strided_batched_3d_tensor_map_bitwise(ctx, layout):
    rng = np.random.default_rng(5)
    m, n, k, batch = 152, 140, 72, 3
    row = layout == "row"
    lda, ldb, ldc = (k, n, n) if row else (m, k, m)
    sa, sb, sc = m * k + 4, k * n + 8, m * n + 12
    a = rng.uniform(-1, 1, sa * batch).astype(np.float32)
    b = rng.uniform(-1, 1, sb * batch).astype(np.float32)
    c = rng.uniform(-1, 1, sc * batch).astype(np.float32)
    bufs = []
    for x in (a, b, c):
        buf = tb.buffer_alloc(ctx, S, x.size)
        tb.buffer_write(buf, 0, x)
        bufs.append(buf)
    tb.gemm_strided_batched(ctx, L[layout], Transpose.NO, Transpose.NO, m, n, k, 1.0, bufs[0], sa,
                            bufs[1], sb, -1.0, bufs[2], sc, batch, lda=lda, ldb=ldb, ldc=ldc)
    assert ctx.last_launch.native["kernel"].startswith("sgemm_tma_")
    got = tb.buffer_read(bufs[2], 0, c.size)
    want = c.copy()
    orc.seqk_gemm_strided_batched("S", row, False, False, m, n, k, 1.0, a, 0, lda, sa, b, 0, ldb, sb,
                                  -1.0, want, 0, ldc, sc, batch)
    assert got.tobytes() == want.tobytes()


def test_alpha_zero_never_reads_operands(ctx):
    # alpha == 0: C = beta*C without a product (level3.py:125-132); never the TMA kernel
    got, want, kern = _run(ctx, "col", "n", "n", 300, 300, 64, 0.0, 0.5, 6)
    assert not kern.startswith("sgemm_tma_")
    assert got.tobytes() == want.tobytes()
