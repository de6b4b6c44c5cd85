"""Batched GEMM: ``gemm_batched`` and ``gemm_strided_batched``
(pkg/src/tunedblas/routines/extras.py:116-122, 175-348 of the reference).

The reference validated every instance in a Python loop, copied and padded
each instance on the host and then ran all work-groups in one launch
(~86 µs of Python per instance).  Here validation is vectorised
over the batch (same checks, same error text naming the first failing
instance, no partial writes) and the whole batch is ONE persistent kernel
launch over (instance, tile) work items:

* strided batched → ``tb_gemm_strided_batched`` (arithmetic offsets; HGEMM
  uses 3-D TMA tensor maps with the batch as the outer dimension);
* generic batched → ``tb_gemm_batched`` with device arrays of per-instance
  offsets and alpha/beta.

Each instance runs exactly the per-element arithmetic of a single ``gemm``
call of the same shape and configuration, so batched == looped bitwise.
"""

from __future__ import annotations

import numpy as np

from ..core import Buffer, Context, Layout, Precision, Transpose, matrix_span
from ..errors import UsageError
from ..kernels import native
from ..kernels.dispatch import b200_config, gemm_batched_native, gemm_strided_batched_native, prec_code
from ..kernels.engine import WorkGrid, pre_launch, record_launch, reference_grid
from .common import check_precision, get_store, scalars, stored_dims
from .level3 import route_family

__all__ = ["gemm_batched", "gemm_strided_batched"]


def _default_lds(layout, trans_a, trans_b, m, n, k, lda, ldb, ldc):
    col = layout is Layout.COL_MAJOR
    lda = lda if lda is not None else ((m if trans_a is Transpose.NO else k) if col
                                       else (k if trans_a is Transpose.NO else m))
    ldb = ldb if ldb is not None else ((k if trans_b is Transpose.NO else n) if col
                                       else (n if trans_b is Transpose.NO else k))
    ldc = ldc if ldc is not None else (m if col else n)
    return lda, ldb, ldc


def _storage_shape(layout: Layout, rows: int, cols: int) -> tuple[int, int]:
    """Column-major (rows, cols) of a logical matrix in ``layout``."""
    return (rows, cols) if layout is Layout.COL_MAJOR else (cols, rows)


def _first_instance_error(operands) -> tuple[int, str] | None:
    """Vectorised per-instance view checks (extras.py:175-185 + core.py:345-355).

    ``operands`` = [(buf, offsets, stored_rows, stored_cols, ld)] in the
    reference's check order A, B, C.  ``offsets`` is an int64 array, or a
    (base, stride, count) triple for strided batches (checked in O(1): the
    offsets are monotone, so only the extremes can fail first).  Returns
    (instance, message) of the first instance that fails, naming the first
    failing operand."""
    first = None
    for buf, offs, rows, cols, ld in operands:
        if rows == 0 or cols == 0:
            continue
        if ld < rows:
            cand = (0, f"leading dimension {ld} < row count {rows}")
        else:
            span = ld * (cols - 1) + rows
            if isinstance(offs, tuple):
                base, stride, count = offs
                lo, hi = (base, base + (count - 1) * stride)
                if min(lo, hi) >= 0 and max(lo, hi) + span <= buf.length:
                    continue
                offs = base + np.arange(count, dtype=np.int64) * stride
            bad = (offs < 0) | (offs + span > buf.length)
            if not bad.any():
                continue
            i = int(np.argmax(bad))
            off = int(offs[i])
            cand = (i, f"access [{off}, {off + span}) outside buffer of length {buf.length}")
        if first is None or cand[0] < first[0]:
            first = cand
    return first


def _check_no_overlap(starts: np.ndarray, span: int, what: str) -> None:
    """extras.py:116-122: sort by start, neighbours must not overlap."""
    if len(starts) < 2 or span == 0:
        return
    order = np.argsort(starts, kind="stable")
    s = starts[order]
    bad = (s[:-1] + span) > s[1:]
    if bad.any():
        j = int(np.argmax(bad))
        raise UsageError(
            f"batched {what} ranges overlap between instances {int(order[j])} and {int(order[j + 1])}")


def _validate(ctx, layout, trans_a, trans_b, m, n, k, a, a_offs, lda, b, b_offs, ldb,
              c, c_offs, ldc, batch_count):
    precision = a.precision
    check_precision(ctx, precision, a, b, c)
    if batch_count < 1:
        raise UsageError("batch_count must be >= 1")
    if m < 0 or n < 0 or k < 0:
        raise UsageError("gemm dimensions must be >= 0")
    prec_code(precision)
    lda, ldb, ldc = _default_lds(layout, trans_a, trans_b, m, n, k, lda, ldb, ldc)
    ar, ac = _storage_shape(layout, *stored_dims(trans_a, m, k))
    br, bc = _storage_shape(layout, *stored_dims(trans_b, k, n))
    cr, cc = _storage_shape(layout, m, n)
    err = _first_instance_error([(a, a_offs, ar, ac, lda), (b, b_offs, br, bc, ldb),
                                 (c, c_offs, cr, cc, ldc)])
    if err is not None:
        raise UsageError(f"batched gemm instance {err[0]}: {err[1]}")
    return lda, ldb, ldc, matrix_span(cr, cc, ldc) if m and n else 0


def _launch_family(ctx, precision, m, n, k):
    store = get_store(ctx)
    cfg, _ = store.resolve("gemm", precision, ctx.device, (m, n, k))
    route = route_family(m, n, k, store.direct_threshold, None)
    family = "gemm_direct" if route == "direct" else "gemm"
    return cfg, family, b200_config(store, precision, ctx.device, (m, n, k))


def gemm_batched(ctx: Context, layout: Layout, trans_a: Transpose, trans_b: Transpose,
                 m: int, n: int, k: int, alphas, a: Buffer, a_offsets, b: Buffer, b_offsets,
                 betas, c: Buffer, c_offsets, batch_count: int, *,
                 lda: int | None = None, ldb: int | None = None, ldc: int | None = None) -> None:
    """batch_count GEMMs with per-instance offsets and scalars (extras.py:289-306)."""
    alphas = list(alphas) if not isinstance(alphas, np.ndarray) else alphas
    betas = list(betas) if not isinstance(betas, np.ndarray) else betas
    a_offs = np.asarray(a_offsets, dtype=np.int64).reshape(-1)
    b_offs = np.asarray(b_offsets, dtype=np.int64).reshape(-1)
    c_offs = np.asarray(c_offsets, dtype=np.int64).reshape(-1)
    lengths = {len(alphas), len(betas), len(a_offs), len(b_offs), len(c_offs)}
    if lengths != {batch_count}:
        raise UsageError("scalar and offset arrays must all have length batch_count")
    lda, ldb, ldc, c_span = _validate(ctx, layout, trans_a, trans_b, m, n, k, a, a_offs, lda,
                                      b, b_offs, ldb, c, c_offs, ldc, batch_count)
    precision = a.precision
    al = scalars(alphas, precision)
    be = scalars(betas, precision)
    _check_no_overlap(c_offs, c_span, "gemm output")
    if m == 0 or n == 0:
        return
    cfg, family, ncfg = _launch_family(ctx, precision, m, n, k)
    grid1 = reference_grid(family, m, n, cfg)
    grid = WorkGrid((batch_count,) + grid1.work_groups, grid1.work_group_size)
    computes = k != 0 and bool(np.any(al != 0))
    if computes:
        pre_launch(ctx, family, cfg, grid, precision)
    launched = gemm_batched_native(ctx, precision, layout, trans_a, trans_b, m, n, k, al,
                                   a, a_offs, lda, b, b_offs, ldb, be, c, c_offs, ldc, ncfg)
    if computes:
        # All-alpha-zero batches make no launch in the reference
        # (extras.py:281-286), so last_launch is left unchanged then.
        record_launch(ctx, family, cfg, grid, launched, ncfg)


def gemm_strided_batched(ctx: Context, layout: Layout, trans_a: Transpose, trans_b: Transpose,
                         m: int, n: int, k: int, alpha, a: Buffer, stride_a: int, b: Buffer,
                         stride_b: int, beta, c: Buffer, stride_c: int, batch_count: int, *,
                         a_offset: int = 0, b_offset: int = 0, c_offset: int = 0,
                         lda: int | None = None, ldb: int | None = None,
                         ldc: int | None = None, tf32: bool = False, _validate_only: bool = False):
    """Instance i uses base offset + i*stride per matrix (extras.py:309-348).
    ``tf32=True`` opts in to the TF32 tensor-core kernel (see ``gemm``);
    ``_validate_only`` as for ``gemm`` (internal, netlib layer)."""
    if batch_count < 1:
        raise UsageError("batch_count must be >= 1")
    lda_e, ldb_e, ldc_e = _default_lds(layout, trans_a, trans_b, m, n, k, lda, ldb, ldc)
    for name, stride, ld, (rows, cols) in (
        ("a", stride_a, lda_e, stored_dims(trans_a, m, k)),
        ("b", stride_b, ldb_e, stored_dims(trans_b, k, n)),
        ("c", stride_c, ldc_e, (m, n)),
    ):
        if layout is Layout.ROW_MAJOR:
            rows, cols = cols, rows
        extent = ld * (cols - 1) + rows if rows and cols else 0
        if batch_count > 1 and stride < extent:
            raise UsageError(f"stride_{name} = {stride} smaller than one instance extent {extent}")
    a_offs = (a_offset, stride_a, batch_count)
    b_offs = (b_offset, stride_b, batch_count)
    c_offs = (c_offset, stride_c, batch_count)
    lda_e, ldb_e, ldc_e, c_span = _validate(ctx, layout, trans_a, trans_b, m, n, k, a, a_offs, lda,
                                            b, b_offs, ldb, c, c_offs, ldc, batch_count)
    precision = a.precision
    if tf32 and precision is not Precision.S:
        raise UsageError("tf32 applies to Precision.S only")
    al = scalars([alpha], precision)[0]
    be = scalars([beta], precision)[0]
    # stride_c >= one instance extent was checked above, so strided outputs
    # never overlap (extras.py:116-122 would find no pair).
    if m == 0 or n == 0:
        return False if _validate_only else None
    if _validate_only:
        return True
    cfg, family, ncfg = _launch_family(ctx, precision, m, n, k)
    grid1 = reference_grid(family, m, n, cfg)
    grid = WorkGrid((batch_count,) + grid1.work_groups, grid1.work_group_size)
    computes = k != 0 and al != 0
    if computes:
        pre_launch(ctx, family, cfg, grid, precision)
    launched = gemm_strided_batched_native(
        ctx, precision, layout, trans_a, trans_b, m, n, k, float(al),
        a, a_offset, lda_e, stride_a, b, b_offset, ldb_e, stride_b, float(be),
        c, c_offset, ldc_e, stride_c, batch_count, ncfg, native.FLAG_TF32 if tf32 else 0)
    if computes:
        record_launch(ctx, family, cfg, grid, launched, ncfg)
