"""Shared argument handling for the routine layer (routines/common.py:38-103
of the reference): parameter store access, precision/context checks, scalar
coercion, and the storage view rules for layouts.

All routines canonicalise to column-major: a row-major (rows, cols) matrix
is the column-major (cols, rows) matrix over the same bytes (common.py:1-7).
"""

from __future__ import annotations

import numpy as np

from ..core import Buffer, Context, Layout, Precision, Transpose, check_matrix
from ..errors import UsageError
from ..tuningdb import ParameterStore

__all__ = ["get_store", "check_precision", "scalar", "scalars", "stored_dims",
           "default_ld", "check_logical"]


def get_store(ctx: Context) -> ParameterStore:
    """The context's parameter-resolution store (created on first use)."""
    store = getattr(ctx, "params", None)
    if store is None:
        store = ParameterStore()
        ctx.params = store
    return store


def check_precision(ctx: Context, precision: Precision, *bufs: Buffer) -> None:
    ctx.check_owns(*bufs)
    for i, buf in enumerate(bufs):
        if buf.precision is not precision:
            raise UsageError(
                f"operand {i} has precision {buf.precision.value}, expected {precision.value}")


_F32 = np.float32


def scalar(value, precision: Precision):
    """Coerce a routine scalar to the compute dtype (common.py:68-76)."""
    if (precision is Precision.S or precision is Precision.H) and type(value) in (float, int):
        return _F32(value)
    if precision.is_complex:
        return precision.compute_dtype.type(complex(value))
    if isinstance(value, complex):
        if value.imag != 0:
            raise UsageError("complex scalar passed to a real-precision routine")
        value = value.real
    return precision.compute_dtype.type(value)


def scalars(values, precision: Precision) -> np.ndarray:
    """Vectorised :func:`scalar` for per-instance alpha/beta arrays."""
    arr = np.asarray(list(values) if not isinstance(values, np.ndarray) else values)
    if np.iscomplexobj(arr):
        if np.any(arr.imag != 0):
            raise UsageError("complex scalar passed to a real-precision routine")
        arr = arr.real
    return arr.astype(precision.compute_dtype)


def stored_dims(trans: Transpose, rows: int, cols: int) -> tuple[int, int]:
    """Stored (rows, cols) of an operand whose op() is (rows, cols)."""
    return (rows, cols) if trans is Transpose.NO else (cols, rows)


def default_ld(layout: Layout, rows: int, cols: int) -> int:
    """Default leading dimension of a stored (rows, cols) matrix
    (level3.py:116-118)."""
    return rows if layout is Layout.COL_MAJOR else cols


def check_logical(buf: Buffer, offset: int, rows: int, cols: int, ld: int, layout: Layout) -> None:
    """Checks of the reference's _logical view (level3.py:41-45)."""
    if layout is Layout.COL_MAJOR:
        check_matrix(buf, offset, rows, cols, ld)
    else:
        check_matrix(buf, offset, cols, rows, ld)
