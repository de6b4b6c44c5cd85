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
from .params import Configuration, is_b200_auto

__all__ = ["gemm_native", "gemm_strided_batched_native", "gemm_batched_native",
           "prec_code", "require_gpu", "b200_config"]

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
    if not getattr(ctx, "_native_ready", False):
        # per-device state (wave-barrier counters) allocated once, outside
        # any graph capture, so no later call allocates
        import torch

        with torch.cuda.device(ctx.torch_device):
            native.check(native.lib().tb_prepare_device(), "tb_prepare_device")
        ctx._native_ready = True


_CONFIG_STRUCTS: dict = {}


def b200_config(store, precision: Precision, device, args: tuple) -> Configuration | None:
    """The "gemm_b200" configuration for (m, n, k): an override or an exact
    tuning-DB entry, else None — the library's built-in shape routing.

    The reference's 14 GemmParams (family "gemm") are validated and recorded
    in LaunchRecord.params by the routines, but they describe an OpenCL
    work-group decomposition with no sm_100a meaning and never select a
    kernel here (DESIGN.md §4 "Tuning space")."""
    if not store._overrides and (store.database is None or not store.database.entries):
        return None
    cfg, source = store.resolve("gemm_b200", precision, device, args)
    if source == "builtin" or is_b200_auto(cfg):
        return None
    return cfg


def _params(config: Configuration | None):
    if config is None:
        return None
    st = _CONFIG_STRUCTS.get(config)
    if st is None:
        st = native.TbGemmConfig.from_dict(config.as_dict())
        if len(_CONFIG_STRUCTS) < 4096:
            _CONFIG_STRUCTS[config] = st
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
    # Per-instance arrays travel as device arrays (tbgemm.h: tb_gemm_batched),
    # staged through pinned host memory and copied asynchronously on the
    # call's stream (torch's pinned allocator keeps the staging block alive
    # until the copy has run).  Host arrays are read at call time, so a CUDA
    # graph capturing this routine would replay stale offsets: capture
    # gemm_strided_batched instead.
    offs_h = torch.empty(3 * batch, dtype=torch.int64, pin_memory=True)
    o = offs_h.numpy()
    o[:batch], o[batch:2 * batch], o[2 * batch:] = a_offs, b_offs, c_offs
    scal_h = torch.empty(2 * batch, dtype=torch.float32, pin_memory=True)
    sc = scal_h.numpy()
    sc[:batch], sc[batch:] = alphas, betas
    stream = torch.cuda.current_stream(dev)
    with torch.cuda.stream(stream):
        packed = offs_h.to(dev, non_blocking=True)
        scal = scal_h.to(dev, non_blocking=True)
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
