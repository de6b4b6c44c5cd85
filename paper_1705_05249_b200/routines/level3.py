"""Level-3 GEMM: the public ``gemm`` routine (level3.py:94-149 of the
reference) over the sm_100a kernels.

Validation, defaults, early-outs and error text follow the reference step by
step (SURVEY §9 "Order of checks in gemm").  The reference then materialised
op(A) and op(B)^T, padded them to tile multiples and unpadded the result
(level3.py:134-147, 48-91); here the unpadded operands go straight to
libtbgemm.so, which reads them in place (TMA tensor maps / predicated loads)
and fuses the single rounding into its epilogue.
"""

from __future__ import annotations

from ..core import Buffer, Context, Layout, Precision, Transpose
from ..errors import UsageError
from ..kernels import native
from ..kernels.dispatch import b200_config, gemm_native, prec_code
from ..kernels.engine import pre_launch, record_launch, reference_grid
from .common import check_logical, check_precision, default_ld, get_store, scalar, stored_dims

__all__ = ["gemm", "route_family", "route_flags"]


def route_family(m: int, n: int, k: int, threshold: int, kernel: str | None) -> str:
    """"direct" below the store's threshold (level3.py:57-59), else "indirect"."""
    if kernel is None:
        kernel = "direct" if max(m, n, k) < threshold else "indirect"
    return kernel


def route_flags(kernel_forced: str | None) -> int:
    """An explicit ``kernel="direct"`` selects the bounds-checked producers
    (SIMT general kernel / tcgen05 with LDG producer); they are bitwise
    identical to the tiled ones, so default routing only sets the family."""
    if kernel_forced == "direct":
        return native.FLAG_SIMT_GENERAL | native.FLAG_NO_TMA
    return 0


def gemm(ctx: Context, layout: Layout, trans_a: Transpose, trans_b: Transpose,
         m: int, n: int, k: int, alpha, a: Buffer, b: Buffer, beta, c: Buffer, *,
         a_offset: int = 0, lda: int | None = None,
         b_offset: int = 0, ldb: int | None = None,
         c_offset: int = 0, ldc: int | None = None,
         kernel: str | None = None, tf32: bool = False,
         _config_args: tuple | None = None, _validate_only: bool = False, _flags: int = 0):
    """C = alpha * op(A) op(B) + beta * C on the GPU (asynchronous on the
    context's stream; read results with ``buffer_read`` / ``Buffer.data``).

    ``kernel`` forces the 'direct' or 'indirect' route (reference testing
    knob, level3.py:99,110-111).  ``tf32=True`` (Precision.S only) opts in to
    the TF32 tensor-core kernel: inputs are rounded to TF32, so results meet
    the TF32 tolerance 4*2^-10*K*max|a||b| instead of the FP32 one, and
    operands must be 16-byte aligned.

    ``_config_args`` (internal: the netlib layer's chunked pipeline) resolves
    the configuration and the launch record for that (m, n, k) instead of
    this call's, so every sub-block of one host-array call runs the kernel
    configuration of the whole problem; ``_validate_only`` (internal: the
    netlib layer validates the whole call before its first copy) runs every
    check and returns False for the m == 0 / n == 0 no-op, True otherwise,
    without launching; ``_flags`` (internal: the same layer's sub-blocks) adds
    native launch flags (TB_FLAG_NO_SPLITK).
    """
    precision = a.precision
    check_precision(ctx, precision, a, b, c)
    if m < 0 or n < 0 or k < 0:
        raise UsageError("gemm dimensions must be >= 0")
    if kernel not in (None, "direct", "indirect"):
        raise UsageError("kernel must be None, 'direct' or 'indirect'")
    prec_code(precision)  # H / S only on this path
    if tf32 and precision is not Precision.S:
        raise UsageError("tf32 applies to Precision.S only")
    if m == 0 or n == 0:
        return False if _validate_only else None
    a_rows, a_cols = stored_dims(trans_a, m, k)
    b_rows, b_cols = stored_dims(trans_b, k, n)
    lda = lda if lda is not None else default_ld(layout, a_rows, a_cols)
    ldb = ldb if ldb is not None else default_ld(layout, b_rows, b_cols)
    ldc = ldc if ldc is not None else (m if layout is Layout.COL_MAJOR else n)
    check_logical(a, a_offset, a_rows, a_cols, lda, layout)
    check_logical(b, b_offset, b_rows, b_cols, ldb, layout)
    check_logical(c, c_offset, m, n, ldc, layout)

    alpha = scalar(alpha, precision)
    beta = scalar(beta, precision)
    if _validate_only:
        return True
    store = get_store(ctx)
    if k == 0 or alpha == 0:
        # Only the beta scaling remains; A and B are never read
        # (level3.py:125-132).  No LaunchRecord, as in the reference.
        gemm_native(ctx, precision, layout, trans_a, trans_b, m, n, k, alpha,
                    a, a_offset, lda, b, b_offset, ldb, beta, c, c_offset, ldc, None)
        return

    shape = (m, n, k) if _config_args is None else tuple(_config_args)
    cfg, _ = store.resolve("gemm", precision, ctx.device, shape)
    route = route_family(*shape, store.direct_threshold, kernel)
    family = "gemm_direct" if route == "direct" else "gemm"
    grid = reference_grid(family, shape[0], shape[1], cfg)
    pre_launch(ctx, family, cfg, grid, precision)
    kcfg = b200_config(store, precision, ctx.device, shape)
    launched = gemm_native(ctx, precision, layout, trans_a, trans_b, m, n, k, alpha,
                           a, a_offset, lda, b, b_offset, ldb, beta, c, c_offset, ldc, kcfg,
                           route_flags(kernel) | (native.FLAG_TF32 if tf32 else 0) | _flags)
    record_launch(ctx, family, cfg, grid, launched, kcfg)
