"""GPU tests of the cluster split-K HGEMM path (csrc/hgemm_tc_splitk.cuh).

Shapes with few 128x128 output tiles and a long K (BASELINE C3
(4096, 128, 9216)) split K over a thread-block cluster and reduce the FP32
partials through distributed shared memory.  The route is a pure function of
(m, n, k), so the TMA and LDG producers, single and batched calls agree
bitwise; against the float64 product the results meet the FP16 tolerance.
"""

import numpy as np
import pytest

import paper_1705_05249_b200 as tb
from paper_1705_05249_b200 import Layout, Precision, Transpose

pytestmark = pytest.mark.gpu

L = {"col": Layout.COL_MAJOR, "row": Layout.ROW_MAJOR}
T = {"n": Transpose.NO, "t": Transpose.YES}


def _operands(ctx, m, n, k, ta, tbn, layout, seed, extra_b=0):
    import torch

    g = torch.Generator(device="cuda").manual_seed(seed)
    at = (torch.rand(m * k, device="cuda", generator=g) * 2 - 1).half()
    bt = (torch.rand(k * n + extra_b, device="cuda", generator=g) * 2 - 1).half()
    a = tb.buffer_from_tensor(ctx, Precision.H, at)
    b = tb.buffer_from_tensor(ctx, Precision.H, bt)
    a_rows, a_cols = (m, k) if ta == "n" else (k, m)
    b_rows, b_cols = (k, n) if tbn == "n" else (n, k)
    lda = a_rows if layout == "col" else a_cols
    ldb = b_rows if layout == "col" else b_cols
    return at, bt, a, b, (a_rows, a_cols, lda), (b_rows, b_cols, ldb)


def _logical(t, rows, cols, ld, layout, off=0):
    flat = t.double()
    if layout == "row":
        return flat[off:off + rows * ld].view(rows, ld)[:, :cols]
    return flat[off:off + cols * ld].view(cols, ld)[:, :rows].t()


def _check(C, A, B, alpha=1.0, beta=0.0, C0=None):
    want = alpha * (A @ B)
    if beta != 0.0:
        want = want + beta * C0
    k = A.shape[1]
    tol = 4 * 2.0 ** -10 * k * abs(alpha) * A.abs().amax(1, keepdim=True) * B.abs().amax(0, keepdim=True) \
        + 2.0 ** -11 * want.abs() + 4 * 2.0 ** -10 * (abs(beta) * C0.abs() if beta != 0.0 else 0.0) + 2.0 ** -24
    err = (C - want).abs()
    assert bool((err <= tol).all()), float((err / tol).max())


@pytest.mark.parametrize("layout,ta,tbn", [("row", "n", "n"), ("col", "n", "n"), ("col", "t", "n"),
                                           ("row", "n", "t"), ("col", "t", "t")])
def test_c3_shape_splits_and_is_accurate(ctx, layout, ta, tbn):
    import torch

    from paper_1705_05249_b200.kernels import native
    from paper_1705_05249_b200.kernels.dispatch import gemm_native

    m, n, k = 4096, 128, 9216
    at, bt, a, b, (ar, ac, lda), (br, bc, ldb) = _operands(ctx, m, n, k, ta, tbn, layout, seed=11)
    ldc = m if layout == "col" else n
    cfg = None  # built-in shape routing (gemm_b200 configurations select kernels)
    outs, kernels = [], []
    for flags in (0, native.FLAG_NO_TMA, native.FLAG_NO_SPLITK):
        c = tb.buffer_alloc(ctx, Precision.H, m * n)
        rec = gemm_native(ctx, Precision.H, L[layout], T[ta], T[tbn], m, n, k, 1.0, a, 0, lda, b, 0, ldb,
                          0.0, c, 0, ldc, cfg, flags)
        outs.append(c.device_tensor().clone())
        kernels.append(rec["kernel"])
    assert "splitk" in kernels[0] and "tma" in kernels[0], kernels
    assert "splitk" in kernels[1] and "ldg" in kernels[1], kernels
    assert "splitk" not in kernels[2], kernels
    # TMA and LDG producers split identically: bitwise equal
    assert torch.equal(outs[0], outs[1]), kernels
    A = _logical(at, ar, ac, lda, layout)
    B = _logical(bt, br, bc, ldb, layout)
    A = A if ta == "n" else A.t()
    B = B if tbn == "n" else B.t()
    for out in (outs[0], outs[2]):
        C = _logical(out, m, n, ldc, layout)
        _check(C, A, B)


def test_splitk_ragged_beta_and_offsets(ctx):
    """Odd m/n tails, K not a multiple of 64, beta != 0, element offsets."""
    import torch

    from paper_1705_05249_b200.kernels.dispatch import gemm_native

    m, n, k = 1000, 200, 5000
    layout, ta, tbn = "col", "n", "n"
    at, bt, a, b, (ar, ac, lda), (br, bc, ldb) = _operands(ctx, m, n, k, ta, tbn, layout, seed=5)
    ldc = m + 8
    g = torch.Generator(device="cuda").manual_seed(9)
    c0 = (torch.rand(ldc * n + 16, device="cuda", generator=g) * 2 - 1).half()
    c = tb.buffer_from_tensor(ctx, Precision.H, c0.clone())
    cfg = None  # built-in shape routing (gemm_b200 configurations select kernels)
    rec = gemm_native(ctx, Precision.H, L[layout], T[ta], T[tbn], m, n, k, 1.5, a, 0, lda, b, 0, ldb,
                      -0.5, c, 8, ldc, cfg, 0)
    assert "splitk" in rec["kernel"], rec
    out = c.device_tensor()
    A = _logical(at, ar, ac, lda, layout)
    B = _logical(bt, br, bc, ldb, layout)
    C = _logical(out, m, n, ldc, layout, off=8)
    C0 = _logical(c0, m, n, ldc, layout, off=8)
    _check(C, A, B, 1.5, -0.5, C0)
    # canaries: padding rows and the region before the offset are untouched
    assert torch.equal(out[:8], c0[:8])
    pad = out[8:8 + ldc * n].view(n, ldc)[:, m:]
    assert torch.equal(pad, c0[8:8 + ldc * n].view(n, ldc)[:, m:])


def test_splitk_batched_equals_loop_bitwise(ctx):
    import torch

    m, n, k, batch = 256, 128, 8192, 3
    prec = Precision.H
    g = torch.Generator(device="cuda").manual_seed(21)
    at = (torch.rand(batch * m * k, device="cuda", generator=g) * 2 - 1).half()
    bt = (torch.rand(batch * k * n, device="cuda", generator=g) * 2 - 1).half()
    a, b = tb.buffer_from_tensor(ctx, prec, at), tb.buffer_from_tensor(ctx, prec, bt)
    cb = tb.buffer_alloc(ctx, prec, batch * m * n)
    tb.gemm_strided_batched(ctx, Layout.ROW_MAJOR, Transpose.NO, Transpose.NO, m, n, k, 1.0, a, m * k,
                            b, k * n, 0.0, cb, m * n, batch)
    assert "splitk" in ctx.last_launch.native["kernel"], ctx.last_launch
    batched = cb.device_tensor().clone()
    for z in range(batch):
        cz = tb.buffer_alloc(ctx, prec, m * n)
        tb.gemm(ctx, Layout.ROW_MAJOR, Transpose.NO, Transpose.NO, m, n, k, 1.0, a, b, 0.0, cz,
                a_offset=z * m * k, b_offset=z * k * n)
        assert "splitk" in ctx.last_launch.native["kernel"]
        assert torch.equal(cz.device_tensor(), batched[z * m * n:(z + 1) * m * n]), z


def test_splitk_deterministic(ctx):
    import torch

    m, n, k = 128, 512, 8192
    prec = Precision.H
    g = torch.Generator(device="cuda").manual_seed(2)
    a = tb.buffer_from_tensor(ctx, prec, (torch.rand(m * k, device="cuda", generator=g) * 2 - 1).half())
    b = tb.buffer_from_tensor(ctx, prec, (torch.rand(k * n, device="cuda", generator=g) * 2 - 1).half())
    outs = []
    for _ in range(3):
        c = tb.buffer_alloc(ctx, prec, m * n)
        tb.gemm(ctx, Layout.COL_MAJOR, Transpose.NO, Transpose.NO, m, n, k, 1.0, a, b, 0.0, c)
        outs.append(c.device_tensor().clone())
    assert "splitk" in ctx.last_launch.native["kernel"]
    assert torch.equal(outs[0], outs[1]) and torch.equal(outs[1], outs[2])


def test_no_split_for_large_or_short_k(ctx):
    """Routing: no split for a square 2048^3 or the short-K C3 shape
    (64, 3136, 576); results on random data within the FP16 tolerance."""
    import torch

    prec = Precision.H
    for (m, n, k) in ((2048, 2048, 2048), (64, 3136, 576)):
        g = torch.Generator(device="cuda").manual_seed(m + n + k)
        at = (torch.rand(m * k, device="cuda", generator=g) * 2 - 1).half()
        bt = (torch.rand(k * n, device="cuda", generator=g) * 2 - 1).half()
        a, b = tb.buffer_from_tensor(ctx, prec, at), tb.buffer_from_tensor(ctx, prec, bt)
        c = tb.buffer_alloc(ctx, prec, m * n)
        tb.gemm(ctx, Layout.ROW_MAJOR, Transpose.NO, Transpose.NO, m, n, k, 1.0, a, b, 0.0, c)
        assert "splitk" not in ctx.last_launch.native["kernel"], (m, n, k, ctx.last_launch.native)
        A, B = at.view(m, k).double(), bt.view(k, n).double()
        want = A @ B
        tol = 4 * 2.0 ** -10 * k * A.abs().amax(1, keepdim=True) * B.abs().amax(0, keepdim=True) \
            + 2.0 ** -11 * want.abs()
        got = c.device_tensor().view(m, n).double()
        assert bool(((got - want).abs() <= tol).all())
