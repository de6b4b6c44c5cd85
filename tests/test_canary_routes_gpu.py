"""Out-of-bounds guard for every kernel route (compute-sanitizer is closed on
the GPU pool, so this is the memory-safety net): C lives inside a larger
buffer with a sentinel-filled prefix, suffix and leading-dimension gaps;
after the call every element outside the declared C matrix must still hold
the sentinel, and the matrix must match the float64 product within the
tolerance.  One case per kernel family (tcgen05 single / pair / split-K /
small / small-TMA / LDG producer, TMA-fed and register-staged FFMA2, TF32,
implicit GEMM)."""

import numpy as np
import pytest

import paper_1705_05249_b200 as tb
from paper_1705_05249_b200 import Layout, Precision, Transpose
from paper_1705_05249_b200.kernels import native

pytestmark = pytest.mark.gpu

SENT = -3.0
NAMES = ("MWG", "NWG", "KWG", "STAGES", "CTA_GROUP", "SPLIT_K", "GROUP_M")

CASES = [
    # id, prec, m, n, k, batch, gemm_b200 config (or None), flags, expected kernel substring
    ("h_single", "H", 300, 520, 200, 1, None, 0, "hgemm_tc_tma"),
    ("h_pair", "H", 2304, 2560, 512, 1, None, 0, "2sm"),
    ("h_pair512_cfg", "H", 2304, 2600, 256, 1, (256, 512, 64, 0, 2, 1, 0), 0, "256x512"),
    ("h_splitk", "H", 260, 130, 4160, 1, None, 0, "splitk"),
    ("h_splitk_cfg", "H", 300, 200, 1000, 1, (128, 128, 64, 0, 1, 4, 0), 0, "splitk4"),
    ("h_ldg", "H", 300, 520, 200, 1, None, native.FLAG_NO_TMA, "ldg"),
    ("h_small", "H", 40, 56, 72, 37, None, 0, "small"),
    ("h_small_tma", "H", 30, 24, 24, 37, None, 0, "32x32_p4_mk_tma"),
    ("s_tma", "S", 300, 520, 200, 1, None, 0, "sgemm_tma"),
    ("s_simt", "S", 300, 520, 200, 1, (128, 128, 16, 0, 1, 1, 0), 0, "sgemm_simt"),
    ("s_general", "S", 300, 520, 200, 1, None, native.FLAG_SIMT_GENERAL, "gen"),
    ("s_small", "S", 30, 28, 24, 37, None, 0, "sgemm"),
    ("s_tf32", "S", 300, 520, 200, 1, None, native.FLAG_TF32, "tf32"),
    ("s_splitk_auto", "S", 512, 512, 4096, 1, None, 0, "splitk4"),
    ("s_splitk_64x32_cfg", "S", 300, 200, 1000, 1, (64, 32, 32, 0, 1, 2, 0), 0, "64x32x32_4x4_mk_splitk2"),
]


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_no_write_outside_c(ctx, case):
    import torch

    from paper_1705_05249_b200.kernels.dispatch import gemm_native, gemm_strided_batched_native

    _, p, m, n, k, batch, cfgv, flags, want_kernel = case
    prec = Precision.H if p == "H" else Precision.S
    dev = ctx.torch_device
    g = torch.Generator(device=dev).manual_seed(m + n + k)
    lda, ldb = k + 8, n + 8                      # row-major A (m x k), B (k x n) with padded rows
    ldc = n + 8
    sa, sb = m * lda + 16, k * ldb + 16
    sc = m * ldc + 24                            # gaps between instances too
    pre = 40
    at = (torch.rand(sa * batch, device=dev, generator=g) * 2 - 1).to(prec.torch_dtype)
    bt = (torch.rand(sb * batch, device=dev, generator=g) * 2 - 1).to(prec.torch_dtype)
    ct = torch.full((pre + sc * batch + 40,), SENT, device=dev, dtype=prec.torch_dtype)
    a, b, c = (tb.buffer_from_tensor(ctx, prec, x) for x in (at, bt, ct))
    cfg = None if cfgv is None else tb.Configuration.make("gemm_b200", dict(zip(NAMES, cfgv)))
    if batch == 1:
        rec = gemm_native(ctx, prec, Layout.ROW_MAJOR, Transpose.NO, Transpose.NO, m, n, k, 1.0, a, 0, lda,
                          b, 0, ldb, 0.0, c, pre, ldc, cfg, flags)
    else:
        rec = gemm_strided_batched_native(ctx, prec, Layout.ROW_MAJOR, Transpose.NO, Transpose.NO, m, n, k,
                                          1.0, a, 0, lda, sa, b, 0, ldb, sb, 0.0, c, pre, ldc, sc, batch, cfg,
                                          flags)
    torch.cuda.synchronize()
    assert want_kernel in rec["kernel"], rec["kernel"]
    out = ct.double().cpu()
    inside = torch.zeros(out.numel(), dtype=torch.bool)
    for z in range(batch):
        base = pre + z * sc
        idx = base + (torch.arange(m)[:, None] * ldc + torch.arange(n)[None, :]).reshape(-1)
        inside[idx] = True
        A = at[z * sa: z * sa + m * lda].view(m, lda)[:, :k].double()
        B = bt[z * sb: z * sb + k * ldb].view(k, ldb)[:, :n].double()
        want = (A @ B).cpu()
        got = out[idx].view(m, n)
        eps = 2.0 ** -10 if (p == "H" or flags & native.FLAG_TF32) else 2.0 ** -23
        tol = 4 * eps * k * (A.abs().amax(1, keepdim=True) * B.abs().amax(0, keepdim=True)).cpu() \
            + (2.0 ** -11 * want.abs() if p == "H" else 0)
        assert bool(((got - want).abs() <= tol).all()), (case[0], z)
    assert bool((out[~inside] == SENT).all()), f"{case[0]}: writes outside C ({rec['kernel']})"


def test_convgemm_no_write_outside_result(ctx):
    import torch

    for prec in (Precision.H, Precision.S):
        c, h, w, kh, kw, nk, batch = 5, 17, 19, 3, 3, 37, 3
        oh, ow = h - 2, w - 2
        dev = ctx.torch_device
        im = tb.buffer_from_tensor(ctx, prec, torch.rand(3 + batch * c * h * w, device=dev).to(prec.torch_dtype))
        kern = tb.buffer_from_tensor(ctx, prec, torch.rand(nk * c * kh * kw, device=dev).to(prec.torch_dtype))
        pre, post = 11, 13
        rt = torch.full((pre + batch * nk * oh * ow + post,), SENT, device=dev, dtype=prec.torch_dtype)
        res = tb.buffer_from_tensor(ctx, prec, rt)
        tb.convgemm(ctx, c, h, w, kh, kw, 0, 0, 1, 1, 1, 1, nk, batch, im, kern, res, im_offset=3,
                    result_offset=pre)
        torch.cuda.synchronize()
        assert bool((rt[:pre].float() == SENT).all()) and bool((rt[-post:].float() == SENT).all())
        assert bool(torch.isfinite(rt.float()).all())
