"""Netlib-style host-array layer for the GEMM path (routines/netlib.py:23-155
of the reference): ``netlib_call("sgemm" | "hgemm", ...)`` allocates device
buffers, copies the host arrays in, runs the device routine and copies the
in/out arrays back.  Device results are the ones ``gemm`` produces for the
same inputs (bitwise: tests/test_netlib_gpu.py).
"""

from __future__ import annotations

import inspect
import threading

import numpy as np

from ..core import Context, Layout, Precision, buffer_alloc, buffer_read, buffer_write, \
    context_create, host_device
from ..errors import UsageError
from . import extras, level3

__all__ = ["netlib_call", "default_context"]

_PRECISIONS = {"h": Precision.H, "s": Precision.S}

# base routine -> (function, {buffer parameter: role})
_ROUTINES = {
    "gemm": (level3.gemm, {"a": "in", "b": "in", "c": "inout"}),
    "gemm_strided_batched": (extras.gemm_strided_batched, {"a": "in", "b": "in", "c": "inout"}),
}

_session_lock = threading.Lock()
_session_ctx: Context | None = None


def default_context() -> Context:
    """The lazily created context netlib_call uses when none is passed."""
    global _session_ctx
    with _session_lock:
        if _session_ctx is None:
            _session_ctx = context_create(host_device())
        return _session_ctx


def _storage(arr: np.ndarray, layout) -> np.ndarray:
    if arr.ndim == 1:
        return arr
    if arr.ndim == 2:
        return arr.reshape(-1, order="F" if layout is Layout.COL_MAJOR else "C")
    raise UsageError("host arrays must be 1-D or 2-D")


def netlib_call(routine_id: str, *args, ctx: Context | None = None, **kwargs):
    """Invoke a GEMM routine by Netlib name on host NumPy arrays."""
    rid = routine_id.lower()
    if len(rid) < 2 or rid[0] not in "hsdcz":
        raise UsageError(f"unknown routine id {routine_id!r}")
    if rid[0] not in _PRECISIONS or rid[1:] not in _ROUTINES:
        raise UsageError(f"routine {routine_id!r} is not part of the B200 GEMM path "
                         "(sgemm / hgemm / [sh]gemm_strided_batched)")
    precision = _PRECISIONS[rid[0]]
    fn, roles = _ROUTINES[rid[1:]]
    ctx = ctx or default_context()
    bound = inspect.signature(fn).bind(ctx, *args, **kwargs)
    bound.apply_defaults()
    layout = bound.arguments.get("layout", Layout.COL_MAJOR)
    writebacks = []
    for name, role in roles.items():
        arr = bound.arguments.get(name)
        if arr is None:
            continue
        arr = np.asanyarray(arr)
        if arr.dtype != precision.dtype:
            raise UsageError(f"array {name!r} has dtype {arr.dtype}, routine {routine_id!r} "
                             f"expects {precision.dtype}")
        flat = _storage(arr, layout)
        buf = buffer_alloc(ctx, precision, flat.size)
        if role in ("in", "inout"):
            buffer_write(buf, 0, flat)
        bound.arguments[name] = buf
        if role in ("inout", "out"):
            writebacks.append((arr, buf, layout))
    result = fn(*bound.args, **bound.kwargs)
    for arr, buf, lay in writebacks:
        host = buffer_read(buf, 0, buf.length)
        if arr.ndim == 1:
            arr[:] = host
        else:
            arr[:] = host.reshape(arr.shape, order="F" if lay is Layout.COL_MAJOR else "C")
    return result
