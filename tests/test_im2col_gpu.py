"""GPU parity of ``im2col`` (csrc/im2col.cuh through the C-ABI): bitwise
against the reference's own outputs (whole buffer, sentinel regions
included), the reference's launch record, and im2col + gemm == direct
convolution (tests/test_extras.py:88-138 of the reference)."""

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
def test_im2col_matches_reference_bitwise(ctx, i):
    cs = CASES[i]
    prec = P[cs["prec"]]
    im = _buf(ctx, prec, ARR[f"i{i}_im"])
    col = _buf(ctx, prec, ARR[f"i{i}_col_in"])
    tb.im2col(ctx, cs["c"], cs["h"], cs["w"], cs["kh"], cs["kw"], cs["ph"], cs["pw"], cs["sh"], cs["sw"],
              cs["dh"], cs["dw"], im, col, im_offset=cs["im_off"], col_offset=cs["col_off"])
    got = tb.buffer_read(col, 0, col.length)
    assert np.array_equal(got.view(np.uint8), ARR[f"i{i}_col_out"].view(np.uint8))
    rec = ctx.last_launch
    assert rec.family == "transform" and rec.params == {"TDX": 16, "TDY": 16}
    assert rec.work_groups == (-(-cs["rows"] // 16), -(-cs["cols"] // 16))
    assert rec.work_group_size == 256
    assert rec.native["kernel"].startswith(("im2col_b", "im2col_vec_b"))


@pytest.mark.parametrize("prec", ["S", "H"])
def test_im2col_large_vs_oracle_bitwise(ctx, prec):
    rng = np.random.default_rng(7)
    c, h, w, kh, kw = 64, 56, 56, 3, 3
    dt = orc.DTYPE[prec]
    image = rng.uniform(-1, 1, c * h * w).astype(dt)
    rows, cols = c * kh * kw, h * w
    im = _buf(ctx, P[prec], image)
    col = tb.buffer_alloc(ctx, P[prec], rows * cols)
    tb.im2col(ctx, c, h, w, kh, kw, 1, 1, 1, 1, 1, 1, im, col)
    want = orc.port_im2col(image, 0, c, h, w, kh, kw, 1, 1, 1, 1, 1, 1, np.zeros(rows * cols, dt), 0)
    assert np.array_equal(tb.buffer_read(col, 0, rows * cols).view(np.uint8), want.view(np.uint8))


# Geometries for the register-transposed kernel (csrc/im2col.cuh
# im2col_vec_kernel; rows a multiple of the 16-byte vector):
# pixel tiles narrower and wider than a row, strides, dilations, negative
# padding, a ragged last channel block, wide rows (fewer channels per CTA).
STAGED = [
    # c, h, w, kh, kw, ph, pw, sh, sw, dh, dw
    (64, 56, 56, 3, 3, 1, 1, 1, 1, 1, 1),
    (24, 30, 40, 3, 3, 1, 1, 2, 2, 1, 1),
    (16, 9, 8, 3, 3, 2, 2, 1, 1, 2, 2),
    (40, 23, 24, 1, 1, 0, 0, 1, 1, 1, 1),
    (8, 13, 16, 5, 5, -1, 2, 2, 1, 1, 2),
    (20, 12, 232, 3, 3, 1, 1, 1, 1, 1, 1),
    (72, 5, 152, 2, 4, 0, 1, 1, 3, 2, 1),
    (16, 7, 7, 3, 3, 1, 1, 1, 1, 1, 1),
    (5, 9, 10, 3, 3, 1, 1, 1, 1, 1, 1),     # 45 rows: the tile kernel
]


def _vec_eligible(prec, geo):
    """Mirror of tb_im2col's condition for the patch-staged H kernel."""
    c, h, w, kh, kw, ph, pw, sh, sw, dh, dw = geo
    if prec != "H":
        return False
    oh = (h + 2 * ph - (dh * (kh - 1) + 1)) // sh + 1
    ow = (w + 2 * pw - (dw * (kw - 1) + 1)) // sw + 1
    rows, tr = c * kh * kw, 64
    pr = (127 // ow + 1) * sh + (kh - 1) * dh + 1   # IM2COL_VQ = 128 pixels per CTA
    pwid = (ow - 1) * sw + (kw - 1) * dw + 1
    nch = (tr - 1) // (kh * kw) + 2
    return rows % 8 == 0 and nch * pr * pwid * 2 <= 15360


@pytest.mark.parametrize("prec", ["S", "H"])
@pytest.mark.parametrize("geo", STAGED)
def test_im2col_vec_vs_oracle_bitwise(ctx, prec, geo):
    c, h, w, kh, kw, ph, pw, sh, sw, dh, dw = geo
    oh = (h + 2 * ph - (dh * (kh - 1) + 1)) // sh + 1
    ow = (w + 2 * pw - (dw * (kw - 1) + 1)) // sw + 1
    rows, cols = c * kh * kw, oh * ow
    vec = 16 // orc.DTYPE[prec]().itemsize
    rng = np.random.default_rng(c * 1000 + w)
    dt = orc.DTYPE[prec]
    image = rng.uniform(-1, 1, c * h * w).astype(dt)
    im = _buf(ctx, P[prec], image)
    sentinel = np.full(rows * cols + 64, 7, dt)
    col = _buf(ctx, P[prec], sentinel)
    tb.im2col(ctx, c, h, w, kh, kw, ph, pw, sh, sw, dh, dw, im, col)
    assert ctx.last_launch.native["kernel"].startswith("im2col_vec_b" if _vec_eligible(prec, geo) else "im2col_b")
    want = orc.port_im2col(image, 0, c, h, w, kh, kw, ph, pw, sh, sw, dh, dw, sentinel.copy(), 0)
    got = tb.buffer_read(col, 0, col.length)
    assert np.array_equal(got.view(np.uint8), want.view(np.uint8))


def _conv2d(image, weights, pad, stride, dil):
    c, h, w = image.shape
    _, kh, kw = weights.shape
    oh = (h + 2 * pad[0] - (dil[0] * (kh - 1) + 1)) // stride[0] + 1
    ow = (w + 2 * pad[1] - (dil[1] * (kw - 1) + 1)) // stride[1] + 1
    padded = np.zeros((c, h + 2 * pad[0], w + 2 * pad[1]))
    padded[:, pad[0]:pad[0] + h, pad[1]:pad[1] + w] = image
    out = np.zeros((oh, ow))
    for oy in range(oh):
        for ox in range(ow):
            for ky in range(kh):
                for kx in range(kw):
                    y, x = oy * stride[0] + ky * dil[0], ox * stride[1] + kx * dil[1]
                    out[oy, ox] += float(np.dot(weights[:, ky, kx], padded[:, y, x]))
    return out


@pytest.mark.parametrize("prec", ["S", "H"])
def test_im2col_then_gemm_is_convolution(ctx, prec):
    """Weights-as-rows GEMM against the column matrix = cross-correlation,
    with both routines on the GPU (the C3 shapes are exactly these GEMMs)."""
    rng = np.random.default_rng(86)
    c, h, w, kh, kw, nk = 3, 17, 15, 3, 2, 24
    pad, stride, dil = (1, 0), (2, 1), (2, 1)
    dt = orc.DTYPE[prec]
    image = rng.uniform(-1, 1, (c, h, w)).astype(dt)
    weights = rng.uniform(-1, 1, (nk, c, kh, kw)).astype(dt)
    oh = (h + 2 * pad[0] - (dil[0] * (kh - 1) + 1)) // stride[0] + 1
    ow = (w + 2 * pad[1] - (dil[1] * (kw - 1) + 1)) // stride[1] + 1
    rows, cols = c * kh * kw, oh * ow
    im = _buf(ctx, P[prec], image.ravel())
    col = tb.buffer_alloc(ctx, P[prec], rows * cols)
    tb.im2col(ctx, c, h, w, kh, kw, pad[0], pad[1], stride[0], stride[1], dil[0], dil[1], im, col)
    wb = _buf(ctx, P[prec], weights.reshape(nk, rows).ravel())  # row-major nk x rows
    out = tb.buffer_alloc(ctx, P[prec], nk * cols)
    # out (nk x cols, col-major) = W (nk x rows) @ col (rows x cols, col-major)
    tb.gemm(ctx, Layout.COL_MAJOR, Transpose.YES, Transpose.NO, nk, cols, rows, 1.0, wb, col, 0.0, out,
            lda=rows, ldb=rows, ldc=nk)
    got = tb.buffer_read(out, 0, nk * cols).reshape(cols, nk).T.astype(np.float64)
    for f in range(nk):
        want = _conv2d(image.astype(np.float64), weights[f].astype(np.float64), pad, stride, dil).ravel()
        tol = 8 * orc.EPS[prec] * rows * (np.abs(want) + 4)
        assert np.all(np.abs(got[f] - want) <= tol), f
