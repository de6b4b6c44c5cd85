"""The operator call into libtbgemm.so — replaces the reference's
``run_kernel("gemm" | "gemm_direct", config, args, ctx, precision)``
(pkg/src/tunedblas/kernels/compute.py:116-130).

Arguments are plain device pointers, element offsets and leading dimensions
of the UNPADDED operands; the library does no host-side padding, transposing
or copying (compare level3.py:71-91 and extras.py:230-279).
"""

from __future__ import annotations

import ctypes

import numpy as np

from ..core import Buffer, Context, Layout, Precision, Transpose
from ..errors import UsageError
from . import native
from .params import Configuration

__all__ = ["gemm_native", "gemm_strided_batched_native", "gemm_batched_native",
           "prec_code", "require_gpu"]

_LAYOUT = {Layout.COL_MAJOR: native.COL_MAJOR, Layout.ROW_MAJOR: native.ROW_MAJOR}
_TRANS = {Transpose.NO: native.NO_TRANS, Transpose.YES: native.TRANS,
          Transpose.CONJUGATE: native.CONJ_TRANS}


def prec_code(precision: Precision) -> int:
    if precision is Precision.S:
        return native.PREC_S
    if precision is Precision.H:
        return native.PREC_H
    raise UsageError(
        f"precision {precision.value} is not supported by the B200 GEMM path (H and S only)")


def require_gpu(ctx: Context) -> None:
    if not ctx.on_gpu:
        raise native.NativeLibraryError(
            "the GEMM routines run only on a CUDA device (sm_100a); none is visible "
            "— there is no CPU fallback")


_PARAM_STRUCTS: dict = {}


def native_config(config: Configuration, source: str) -> Configuration | None:
    """The configuration the native dispatcher sees: None for the built-in
    default (the library then picks tiles by shape, from measured crossovers),
    the configuration itself when it came from an override or the tuning DB
    (its MWG / NWG / KWG / VW* then select the kernel)."""
    return None if source == "builtin" else config


def _params(config: Configuration | None):
    if config is None:
        return None
    st = _PARAM_STRUCTS.get(config)
    if st is None:
        st = native.TbGemmParams.from_dict(config.as_dict())
        if len(_PARAM_STRUCTS) < 4096:
            _PARAM_STRUCTS[config] = st
    return ctypes.byref(st)


def _codes(layout: Layout, ta: Transpose, tb: Transpose) -> tuple:
    """C-ABI enum codes (identity tests: cheaper than enum-keyed dicts)."""
    lc = native.ROW_MAJOR if layout is Layout.ROW_MAJOR else native.COL_MAJOR
    tac = native.NO_TRANS if ta is Transpose.NO else (
        native.TRANS if ta is Transpose.YES else native.CONJ_TRANS)
    tbc = native.NO_TRANS if tb is Transpose.NO else (
        native.TRANS if tb is Transpose.YES else native.CONJ_TRANS)
    return lc, tac, tbc


def _stream(ctx: Context) -> int:
    return ctx.stream_handle()


def gemm_native(ctx: Context, precision: Precision, layout: Layout, ta: Transpose, tb: Transpose,
                m: int, n: int, k: int, alpha: float, a: Buffer, a_off: int, lda: int,
                b: Buffer, b_off: int, ldb: int, beta: float, c: Buffer, c_off: int, ldc: int,
                config: Configuration | None, flags: int = 0) -> dict:
    require_gpu(ctx)
    so = native.lib()
    pa, pb = a.data_ptr(), b.data_ptr()
    pc = c.data_ptr()
    lc, tac, tbc = _codes(layout, ta, tb)
    st = so.tb_gemm(prec_code(precision), lc, tac, tbc,
                    m, n, k, float(alpha), pa, a_off, lda, pb, b_off, ldb, float(beta),
                    pc, c_off, ldc, _params(config), flags, _stream(ctx))
    c.mark_device_written()
    native.check(st, "tb_gemm")
    return native.last_launch()


def gemm_strided_batched_native(ctx: Context, precision: Precision, layout: Layout,
                                ta: Transpose, tb: Transpose, m: int, n: int, k: int,
                                alpha: float, a: Buffer, a_off: int, lda: int, stride_a: int,
                                b: Buffer, b_off: int, ldb: int, stride_b: int, beta: float,
                                c: Buffer, c_off: int, ldc: int, stride_c: int, batch: int,
                                config: Configuration | None, flags: int = 0) -> dict:
    require_gpu(ctx)
    so = native.lib()
    pa, pb, pc = a.data_ptr(), b.data_ptr(), c.data_ptr()
    st = so.tb_gemm_strided_batched(
        prec_code(precision), _LAYOUT[layout], _TRANS[ta], _TRANS[tb], m, n, k, float(alpha),
        pa, a_off, lda, stride_a, pb, b_off, ldb, stride_b, float(beta),
        pc, c_off, ldc, stride_c, batch, _params(config), flags, _stream(ctx))
    c.mark_device_written()
    native.check(st, "tb_gemm_strided_batched")
    return native.last_launch()


def gemm_batched_native(ctx: Context, precision: Precision, layout: Layout, ta: Transpose,
                        tb: Transpose, m: int, n: int, k: int, alphas: np.ndarray,
                        a: Buffer, a_offs: np.ndarray, lda: int, b: Buffer, b_offs: np.ndarray,
                        ldb: int, betas: np.ndarray, c: Buffer, c_offs: np.ndarray, ldc: int,
                        config: Configuration | None, flags: int = 0) -> dict:
    import torch

    require_gpu(ctx)
    so = native.lib()
    dev = ctx.torch_device
    batch = int(len(a_offs))
    # Per-instance arrays travel as device arrays (tbgemm.h: tb_gemm_batched).
    packed = torch.from_numpy(np.concatenate([
        np.asarray(a_offs, np.int64), np.asarray(b_offs, np.int64), np.asarray(c_offs, np.int64),
    ])).to(dev, non_blocking=False)
    scal = torch.from_numpy(np.concatenate([
        np.asarray(alphas, np.float32), np.asarray(betas, np.float32)])).to(dev, non_blocking=False)
    vec = 8 if precision is Precision.H else 4
    aligned = int(all(int(np.all(np.asarray(o) % vec == 0)) for o in (a_offs, b_offs)))
    pa, pb, pc = a.data_ptr(), b.data_ptr(), c.data_ptr()
    i64 = packed.element_size()
    st = so.tb_gemm_batched(
        prec_code(precision), _LAYOUT[layout], _TRANS[ta], _TRANS[tb], m, n, k,
        scal.data_ptr(), pa, packed.data_ptr(), lda, pb, packed.data_ptr() + batch * i64, ldb,
        scal.data_ptr() + batch * 4, pc, packed.data_ptr() + 2 * batch * i64, ldc, batch,
        aligned, _params(config), flags, _stream(ctx))
    c.mark_device_written()
    native.check(st, "tb_gemm_batched")
    # `packed`/`scal` were allocated on this stream: the caching allocator only
    # reuses their memory for later work on the same stream, after the kernel.
    return native.last_launch()
