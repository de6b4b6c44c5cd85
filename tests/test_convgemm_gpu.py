"""Implicit GEMM (``convgemm``) on the GPU: the column
matrix is gathered inside the GEMM's producer, never materialised.

Parity (reference tests/test_extras.py:78-145: im2col + gemm == direct
convolution):
* against the REFERENCE's im2col output (tests/golden/im2col_golden.*)
  followed by a GEMM: S bitwise equal to the sequential-k C oracle on the
  golden column matrix; H within the FP16 tolerance of the float64 product;
* against this library's own ``im2col`` + ``gemm`` (bitwise, both precisions:
  the same per-element arithmetic — except few-tile H layers, which split K
  over a cluster and are checked within the FP16 tolerance);
* batched images, offsets, sentinel regions around the result untouched.
"""

import json

import numpy as np
import pytest

import paper_1705_05249_b200 as tb
from paper_1705_05249_b200 import Layout, Precision, Transpose
from conftest import GOLDEN_DIR
from oracle import gemm_oracle as orc

pytestmark = pytest.mark.gpu

META = json.loads((GOLDEN_DIR / "im2col_golden.json").read_text())
CASES = META["cases"]
ARR = np.load(GOLDEN_DIR / "im2col_golden.npz")
P = {"S": Precision.S, "H": Precision.H}


def _buf(ctx, prec, arr):
    b = tb.buffer_alloc(ctx, prec, arr.size)
    tb.buffer_write(b, 0, arr)
    return b


@pytest.mark.parametrize("i", range(len(CASES)))
def test_convgemm_vs_reference_im2col_then_gemm(ctx, i):
    cs = CASES[i]
    prec = P[cs["prec"]]
    rows, cols = cs["rows"], cs["cols"]
    nk = 1 + (i * 7) % 37
    rng = np.random.default_rng(500 + i)
    w = rng.uniform(-1, 1, nk * rows).astype(prec.dtype)        # kernel[f][r], row-major
    sentinel = 3
    res_len = sentinel + nk * cols + sentinel
    im = _buf(ctx, prec, ARR[f"i{i}_im"])
    kern = _buf(ctx, prec, w)
    res = _buf(ctx, prec, np.full(res_len, -5.0, prec.dtype))
    tb.convgemm(ctx, cs["c"], cs["h"], cs["w"], cs["kh"], cs["kw"], cs["ph"], cs["pw"], cs["sh"], cs["sw"],
                cs["dh"], cs["dw"], nk, 1, im, kern, res, im_offset=cs["im_off"], result_offset=sentinel)
    got = tb.buffer_read(res, 0, res_len)
    assert np.all(got[:sentinel] == -5) and np.all(got[sentinel + nk * cols:] == -5)
    got = got[sentinel:sentinel + nk * cols]
    assert ctx.last_launch.family == "convgemm"
    kernel_name = ctx.last_launch.native["kernel"]
    assert "conv" in kernel_name, kernel_name
    # the reference's column matrix (column-major rows x cols, ld = rows)
    col = ARR[f"i{i}_col_out"][cs["col_off"]:cs["col_off"] + rows * cols]
    colm = col.reshape(cols, rows).T                             # (rows, cols)
    W = w.reshape(nk, rows)
    if prec is Precision.S:
        # result[f][q] = sum_r W[f][r] col[r][q]: row-major (nk x cols) = W @ col
        want = np.zeros(nk * cols, np.float32)
        orc.seqk_gemm("S", True, False, False, nk, cols, rows, 1.0, np.ascontiguousarray(W).reshape(-1), 0,
                      rows, np.ascontiguousarray(colm).reshape(-1), 0, cols, 0.0, want, 0, cols)
        assert got.tobytes() == want.tobytes()
    else:
        wide = W.astype(np.float64) @ colm.astype(np.float64)
        tol = orc.gemm_tolerance(W.astype(np.float32), colm.astype(np.float32), "H") \
            + 2.0 ** -11 * np.abs(wide) + 2.0 ** -24
        assert np.all(np.abs(got.reshape(nk, cols).astype(np.float64) - wide) <= tol)


@pytest.mark.parametrize("prec", [Precision.S, Precision.H])
@pytest.mark.parametrize("geom", [
    # c, h, w, kh, kw, ph, pw, sh, sw, dh, dw, filters, batch
    (64, 56, 56, 3, 3, 1, 1, 1, 1, 1, 1, 64, 1),      # BASELINE C3 (64, 3136, 576) layer
    (3, 32, 30, 5, 5, 2, 1, 2, 2, 1, 1, 40, 3),
    (16, 20, 20, 3, 3, 2, 2, 1, 1, 2, 2, 130, 2),
    (256, 14, 14, 1, 1, 0, 0, 1, 1, 1, 1, 300, 4),
])
def test_convgemm_equals_im2col_plus_gemm(ctx, prec, geom):
    """Fused == materialised (this library's im2col then gemm), bitwise, for
    both precisions, with batched images and offsets."""
    import torch

    c, h, w_, kh, kw, ph, pw, sh, sw, dh, dw, nk, batch = geom
    from paper_1705_05249_b200.routines.im2col import im2col_geometry

    out_h, out_w, rows, cols = im2col_geometry(c, h, w_, kh, kw, ph, pw, sh, sw, dh, dw)
    dev = ctx.torch_device
    g = torch.Generator(device=dev).manual_seed(sum(geom))
    im_off, k_off, r_off = 5, 3, 7
    imt = (torch.rand(im_off + batch * c * h * w_, device=dev, generator=g) * 2 - 1).to(prec.torch_dtype)
    kt = (torch.rand(k_off + nk * rows, device=dev, generator=g) * 2 - 1).to(prec.torch_dtype)
    im = tb.buffer_from_tensor(ctx, prec, imt)
    kern = tb.buffer_from_tensor(ctx, prec, kt)
    res = tb.buffer_alloc(ctx, prec, r_off + batch * nk * cols)
    tb.convgemm(ctx, c, h, w_, kh, kw, ph, pw, sh, sw, dh, dw, nk, batch, im, kern, res,
                im_offset=im_off, kernel_offset=k_off, result_offset=r_off)
    conv_kernel = ctx.last_launch.native["kernel"]
    fused = res.device_tensor().clone()
    col = tb.buffer_alloc(ctx, prec, rows * cols)
    ref = tb.buffer_alloc(ctx, prec, r_off + batch * nk * cols)
    for b in range(batch):
        tb.im2col(ctx, c, h, w_, kh, kw, ph, pw, sh, sw, dh, dw, im, col,
                  im_offset=im_off + b * c * h * w_)
        # row-major (nk x cols) = kernel (nk x rows, row-major) @ col (rows x cols; col-major storage)
        tb.gemm(ctx, Layout.ROW_MAJOR, Transpose.NO, Transpose.YES, nk, cols, rows, 1.0, kern, col, 0.0, ref,
                a_offset=k_off, lda=rows, ldb=rows, c_offset=r_off + b * nk * cols, ldc=cols)
    assert torch.equal(fused[:r_off], ref.device_tensor()[:r_off])
    if "splitk" not in conv_kernel:
        assert torch.equal(fused, ref.device_tensor()), conv_kernel
    else:
        # few-tile layers split K (a different summation order): within 2x
        # the FP16 tolerance of the materialised result
        W = kt[k_off:].view(nk, rows).double()
        colm = col.device_tensor().view(cols, rows).t().double()   # last image's column matrix
        want = W @ colm
        tol = 4 * 2.0 ** -10 * rows * W.abs().amax(1, keepdim=True) * colm.abs().amax(0, keepdim=True) \
            + 2.0 ** -11 * want.abs()
        b = batch - 1
        got = fused[r_off + b * nk * cols: r_off + (b + 1) * nk * cols].view(nk, cols).double()
        mat = ref.device_tensor()[r_off + b * nk * cols: r_off + (b + 1) * nk * cols].view(nk, cols).double()
        assert bool(((got - want).abs() <= tol).all()) and bool(((got - mat).abs() <= 2 * tol).all()), conv_kernel


def test_convgemm_validation(ctx):
    prec = Precision.S
    im = tb.buffer_alloc(ctx, prec, 2 * 8 * 8)
    kern = tb.buffer_alloc(ctx, prec, 4 * 18)
    res = tb.buffer_alloc(ctx, prec, 4 * 36)
    with pytest.raises(tb.UsageError, match="output dimensions"):
        tb.convgemm(ctx, 2, 8, 8, 9, 3, 0, 0, 1, 1, 1, 1, 4, 1, im, kern, res)
    with pytest.raises(tb.RangeError):
        tb.convgemm(ctx, 2, 8, 8, 3, 3, 0, 0, 1, 1, 1, 1, 4, 2, im, kern, res)
    tb.convgemm(ctx, 2, 8, 8, 3, 3, 0, 0, 1, 1, 1, 1, 4, 1, im, kern, res)
