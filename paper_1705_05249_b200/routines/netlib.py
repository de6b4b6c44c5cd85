"""Netlib-style host-array layer for the GEMM path (routines/netlib.py:23-155
of the reference): ``netlib_call("sgemm" | "hgemm" | "[sh]gemm_strided_batched",
...)`` takes host NumPy arrays in the buffer positions, runs the device
routine and writes the in/out arrays back — bitwise what ``gemm`` /
``gemm_strided_batched`` produce for the same inputs
(tests/test_netlib_gpu.py; reference tests/test_netlib.py:19-36).

The reference copies every array into a fresh buffer, calls the routine and
copies back (netlib.py:131-155).  Here one call is a pipeline over three CUDA
streams (H2D copy engine, the context's compute stream, D2H copy engine):

* the operand every sub-problem needs (B for a row-major C, A for a
  column-major C) goes over first, whole;
* the other operand and C are cut into sub-blocks along C's contiguous axis
  (rows of a row-major C, columns of a column-major C, instances of a
  strided batch); sub-block i's H2D copy overlaps sub-block i-1's GEMM and
  sub-block i-2's D2H copy;
* host arrays already in pinned memory (``pinned_empty``) are copied
  directly; pageable ones are staged through a pinned double buffer
  (multi-threaded host copies by torch) overlapped with the transfers;
* C is uploaded only where the kernel reads it (beta != 0) or where its span
  has gaps (ld > rows), so every element outside the written matrix returns
  unchanged, as in the reference.

Every sub-block runs the kernel configuration resolved for the WHOLE problem
(``gemm(..., _config_args=)``); an HGEMM is cut only when neither the
whole problem nor a sub-block would take the cluster split-K route (whose
reduction order depends on the call's shape — hgemm.cu hgemm_split_ks), an
SGEMM only when its whole problem cannot split (sgemm_tma.cu sgemm_split_ks)
and its sub-blocks then run unsplit (TB_FLAG_NO_SPLITK), so the result
equals the single device call bitwise.
"""

from __future__ import annotations

import inspect
import threading

import numpy as np

from ..core import Context, Layout, Precision, Transpose, buffer_from_tensor, context_create, host_device
from ..errors import UsageError
from ..kernels import native
from . import extras, level3
from .common import default_ld, stored_dims

__all__ = ["netlib_call", "default_context", "pinned_empty"]

_PRECISIONS = {"h": Precision.H, "s": Precision.S}

# base routine -> (function, {buffer parameter: role})
_ROUTINES = {
    "gemm": (level3.gemm, {"a": "in", "b": "in", "c": "inout"}),
    "gemm_strided_batched": (extras.gemm_strided_batched, {"a": "in", "b": "in", "c": "inout"}),
}

#: Sub-blocks aim at this many bytes of the cut operand (and at most 8).
# Sub-block size of the pipelined calls.  8192^3 HGEMM on pinned arrays
# (tools/pcie_probe.py): 32 MB x 4 sub-blocks 6.2 ms, 16 MB x 8 6.05 ms,
# 8 MB x 16 6.3 ms per call — the last sub-block's GEMM + D2H is the tail
# after the final H2D, while below ~16 MB the interleaved H2D / D2H copies
# lose rate (gaps between copies on the H2D stream).  Cutting B into column
# blocks so the D2H could start during B's upload would need 2-D copies.
CHUNK_BYTES = 16 << 20
MAX_CHUNKS = 16

_session_lock = threading.Lock()
_session_ctx: Context | None = None


def default_context() -> Context:
    """The lazily created context netlib_call uses when none is passed."""
    global _session_ctx
    with _session_lock:
        if _session_ctx is None:
            _session_ctx = context_create(host_device())
        return _session_ctx


def pinned_empty(count: int, precision: Precision) -> np.ndarray:
    """A 1-D host array in page-locked memory (keeps its torch storage
    alive); netlib_call copies such arrays without staging."""
    import torch

    return torch.empty(int(count), dtype=precision.torch_dtype, pin_memory=True).numpy()


def _storage(arr: np.ndarray, layout) -> np.ndarray:
    if arr.ndim == 1:
        return arr
    if arr.ndim == 2:
        return arr.reshape(-1, order="F" if layout is Layout.COL_MAJOR else "C")
    raise UsageError("host arrays must be 1-D or 2-D")


_SIGNATURES: dict = {}
_SM_COUNTS: dict = {}


def _signature(fn):
    """inspect.signature, cached (it costs tens of microseconds per call)."""
    sig = _SIGNATURES.get(fn)
    if sig is None:
        sig = _SIGNATURES[fn] = inspect.signature(fn)
    return sig


def _sm_count(device) -> int:
    import torch

    key = str(device)
    n = _SM_COUNTS.get(key)
    if n is None:
        n = _SM_COUNTS[key] = torch.cuda.get_device_properties(device).multi_processor_count
    return n


def _is_pinned(flat: np.ndarray) -> bool:
    import torch

    if not flat.flags["C_CONTIGUOUS"] or flat.size == 0:
        return False
    try:
        return bool(torch.from_numpy(flat).is_pinned())
    except (TypeError, RuntimeError):
        return False


def _sgemm_may_split(m: int, n: int, sms: int) -> bool:
    """Whether the built-in S route may split K for a (canonical column-
    major) m x n problem: sgemm_tma.cu sgemm_split_ks returns 1 whenever the
    128 x 64 tiles fill more than half the SMs, and the 64 x 32 split needs
    fewer still."""
    return 2 * (-(-m // 128)) * (-(-n // 64)) <= sms


def _hgemm_split_ks(m: int, n: int, k: int, sms: int) -> int:
    """Mirror of hgemm.cu hgemm_split_ks (canonical column-major m, n)."""
    t1 = -(-m // 128) * -(-n // 128)
    nkb = -(-k // 64)
    ks = 1
    while ks < 8 and t1 * ks * 2 <= sms and nkb >= 32 * ks and (ks < 4 or 4 * t1 * ks <= sms):
        ks *= 2
    return ks


class _Pipeline:
    """Per-context streams and pinned staging blocks (reused across calls;
    every call ends synchronised, so a block is free when the next starts)."""

    def __init__(self, ctx: Context):
        import torch

        dev = ctx.torch_device
        self.h2d = torch.cuda.Stream(dev)
        self.d2h = torch.cuda.Stream(dev)
        self.staging: dict = {}

    def stage(self, key, count: int, dtype):
        import torch

        buf = self.staging.get(key)
        if buf is None or buf.numel() < count or buf.dtype != dtype:
            buf = torch.empty(max(count, 1), dtype=dtype, pin_memory=True)
            self.staging[key] = buf
        return buf[:count]


_pipelines: dict = {}


def _pipeline(ctx: Context) -> _Pipeline:
    key = id(ctx)
    p = _pipelines.get(key)
    if p is None or p[0] is not ctx:
        p = (ctx, _Pipeline(ctx))
        _pipelines[key] = p
    return p[1]


class _Transfer:
    """One host array <-> one device buffer over element spans."""

    def __init__(self, ctx, pipe, name, host_flat, precision):
        import torch

        self.name, self.host = name, host_flat
        self.pinned = _is_pinned(host_flat)
        self.host_t = torch.from_numpy(np.ascontiguousarray(host_flat)) if self.pinned else None
        self.dev = torch.empty(host_flat.size, dtype=precision.torch_dtype, device=ctx.torch_device)
        self.buf = buffer_from_tensor(ctx, precision, self.dev)
        self.pipe, self.precision = pipe, precision

    def upload(self, lo: int, hi: int, slot: int, done_with_slot=None):
        """Async H2D of host[lo:hi] on the H2D stream (staged when pageable)."""
        import torch

        if hi <= lo:
            return
        if self.pinned:
            src = self.host_t[lo:hi]
        else:
            if done_with_slot is not None:
                done_with_slot.synchronize()
            src = self.pipe.stage((self.name, "in", slot), hi - lo, self.precision.torch_dtype)
            src.copy_(torch.from_numpy(self.host[lo:hi]))
        with torch.cuda.stream(self.pipe.h2d):
            self.dev[lo:hi].copy_(src, non_blocking=True)

    def download(self, lo: int, hi: int, slot: int):
        """Async D2H of dev[lo:hi] on the D2H stream; returns a finisher that
        lands the data in the host array (a no-op for pinned arrays)."""
        import torch

        if hi <= lo:
            return None
        if self.pinned:
            dst = self.host_t[lo:hi]
        else:
            dst = self.pipe.stage((self.name, "out", slot), hi - lo, self.precision.torch_dtype)
        with torch.cuda.stream(self.pipe.d2h):
            dst.copy_(self.dev[lo:hi], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(self.pipe.d2h)
        if self.pinned:
            return ev, None
        host = self.host

        def land():
            ev.synchronize()
            torch.from_numpy(host[lo:hi]).copy_(dst)
        return ev, land


def _span(layout, rows: int, cols: int, off: int, ld: int, u0: int = 0, count: int | None = None):
    """Element span [lo, hi) of stored units [u0, u0 + count) of a (rows x
    cols) matrix: units are rows of row-major storage, columns of
    column-major storage (unit u starts at off + u*ld)."""
    units, inner = (rows, cols) if layout is Layout.ROW_MAJOR else (cols, rows)
    count = units - u0 if count is None else count
    if count <= 0 or inner == 0:
        return off, off
    return off + u0 * ld, off + (u0 + count - 1) * ld + inner


def _download(finishers: list, C, lo: int, hi: int, slot: int) -> None:
    """Queue the D2H of C[lo:hi] through staging slot ``slot``.  The landing
    of the sub-block two back used the same slot, so it completes first
    (pageable C only: a pinned C is copied into directly and nothing is
    reused, so the host does not wait)."""
    if len(finishers) >= 2 and not C.pinned:
        finishers.pop(0)()
    fin = C.download(lo, hi, slot)
    if fin is not None:
        ev, land = fin
        finishers.append(land if land is not None else ev.synchronize)


def _gemm_pipelined(ctx, precision, xfers, bound) -> None:
    import torch

    A, B, C = xfers["a"], xfers["b"], xfers["c"]
    args = bound.arguments
    layout, ta, tb = args["layout"], args["trans_a"], args["trans_b"]
    m, n, k = args["m"], args["n"], args["k"]
    alpha, beta = args["alpha"], args["beta"]
    a_off, b_off, c_off = args["a_offset"], args["b_offset"], args["c_offset"]
    a_rows, a_cols = stored_dims(ta, m, k)
    b_rows, b_cols = stored_dims(tb, k, n)
    lda = args["lda"] if args["lda"] is not None else default_ld(layout, a_rows, a_cols)
    ldb = args["ldb"] if args["ldb"] is not None else default_ld(layout, b_rows, b_cols)
    ldc = args["ldc"] if args["ldc"] is not None else (m if layout is Layout.COL_MAJOR else n)
    row = layout is Layout.ROW_MAJOR
    pipe = A.pipe
    cur = torch.cuda.current_stream(ctx.torch_device)
    pipe.h2d.wait_stream(cur)
    pipe.d2h.wait_stream(cur)
    # Cut along C's stored units (rows of a row-major C, columns of a
    # column-major one); the operand sharing that axis must be untransposed
    # so its units are the same stored units: A for row-major, B for
    # column-major.  The other operand goes over whole, first.
    units = m if row else n
    cuttable = (ta if row else tb) is Transpose.NO
    chunks = 1
    if cuttable and units > 1 and k > 0:
        chunks = int(max(1, min(MAX_CHUNKS, units, units * k * precision.elemsize // CHUNK_BYTES)))
        if precision is Precision.S and alpha != 0:
            # The S route splits K only with at most half the SMs' worth of
            # 128 x 64 tiles (sgemm_tma.cu sgemm_split_ks / the 64 x 32 split):
            # cut only a call whose whole problem cannot split, and run its
            # sub-blocks unsplit (FLAG_NO_SPLITK) — every unsplit S kernel
            # runs the same sequential-k chains, so bitwise the whole call.
            cm, cn = (n, m) if row else (m, n)          # canonical column-major (m, n)
            if _sgemm_may_split(cm, cn, _sm_count(ctx.torch_device)):
                chunks = 1
        if precision is Precision.H and alpha != 0:
            sms = _sm_count(ctx.torch_device)
            cm, cn = (n, m) if row else (m, n)          # canonical column-major (m, n)
            size = -(-units // chunks)
            last = units - size * (chunks - 1)
            sub = (cm, size) if row else (cm, size)
            lsub = (cm, last) if row else (cm, last)
            if max(_hgemm_split_ks(cm, cn, k, sms), _hgemm_split_ks(*sub, k, sms),
                   _hgemm_split_ks(*lsub, k, sms)) > 1:
                chunks = 1
    if row:
        cut, cut_dims, cut_off, cut_ld = A, (a_rows, a_cols), a_off, lda
        whole, whole_span = B, _span(layout, b_rows, b_cols, b_off, ldb)
    else:
        cut, cut_dims, cut_off, cut_ld = B, (b_rows, b_cols), b_off, ldb
        whole, whole_span = A, _span(layout, a_rows, a_cols, a_off, lda)
    whole.upload(*whole_span, 0)
    c_dense = ldc == (n if row else m)
    base, rem = divmod(units, chunks)
    finishers, slot_events = [], [None, None]
    u0 = 0
    for i in range(chunks):
        size = base + (1 if i < rem else 0)
        slot = i & 1
        if chunks == 1:
            cut_span = _span(layout, *cut_dims, cut_off, cut_ld)
        else:
            cut_span = _span(layout, *cut_dims, cut_off, cut_ld, u0, size)
        c_span = _span(layout, m, n, c_off, ldc, u0, size)
        cut.upload(*cut_span, slot, slot_events[slot])
        if beta != 0 or not c_dense:
            C.upload(*c_span, slot, slot_events[slot])
        ev_in = torch.cuda.Event()
        ev_in.record(pipe.h2d)
        slot_events[slot] = ev_in
        cur.wait_event(ev_in)
        common = dict(lda=lda, ldb=ldb, ldc=ldc, kernel=args.get("kernel"), tf32=args.get("tf32", False),
                      _config_args=(m, n, k), _flags=native.FLAG_NO_SPLITK if chunks > 1 else 0)
        if row:
            level3.gemm(ctx, layout, ta, tb, size, n, k, alpha, A.buf, B.buf, beta, C.buf,
                        a_offset=a_off + u0 * lda, b_offset=b_off, c_offset=c_off + u0 * ldc, **common)
        else:
            level3.gemm(ctx, layout, ta, tb, m, size, k, alpha, A.buf, B.buf, beta, C.buf,
                        a_offset=a_off, b_offset=b_off + u0 * ldb, c_offset=c_off + u0 * ldc, **common)
        pipe.d2h.wait_stream(cur)
        _download(finishers, C, *c_span, slot)
        u0 += size
    for f in finishers:
        f()
    cur.synchronize()
    pipe.h2d.synchronize()
    pipe.d2h.synchronize()


def _strided_pipelined(ctx, precision, xfers, bound) -> None:
    """gemm_strided_batched over host arrays: instance blocks pipelined."""
    import torch

    A, B, C = xfers["a"], xfers["b"], xfers["c"]
    a_host, b_host, c_host = A.host, B.host, C.host
    args = bound.arguments
    layout, ta, tb = args["layout"], args["trans_a"], args["trans_b"]
    m, n, k = args["m"], args["n"], args["k"]
    batch = args["batch_count"]
    sa, sb, sc = args["stride_a"], args["stride_b"], args["stride_c"]
    a_off, b_off, c_off = args["a_offset"], args["b_offset"], args["c_offset"]
    pipe = A.pipe
    cur = torch.cuda.current_stream(ctx.torch_device)
    pipe.h2d.wait_stream(cur)
    pipe.d2h.wait_stream(cur)
    esz = precision.elemsize
    chunks = int(max(1, min(MAX_CHUNKS, batch, (batch * (sa + sb) * esz) // CHUNK_BYTES)))
    base, rem = divmod(batch, chunks)
    # one instance's extent in each operand (the routine checked it <= stride)
    ldc = args["ldc"] if args["ldc"] is not None else (m if layout is Layout.COL_MAJOR else n)
    c_ext = ldc * ((n if layout is Layout.COL_MAJOR else m) - 1) + (m if layout is Layout.COL_MAJOR else n)
    gaps = sc != c_ext or ldc != (m if layout is Layout.COL_MAJOR else n)
    finishers, slot_events = [], [None, None]
    start = 0
    for i in range(chunks):
        size = base + (1 if i < rem else 0)
        z0 = start
        start += size
        slot = i & 1
        if chunks == 1:
            spans = [(A, a_off, a_host.size), (B, b_off, b_host.size)]
        else:
            spans = [(A, a_off + z0 * sa, a_off + (z0 + size) * sa), (B, b_off + z0 * sb, b_off + (z0 + size) * sb)]
        for X, lo, hi in spans:
            X.upload(lo, min(hi, X.host.size), slot, slot_events[slot])
        c_lo, c_hi = c_off + z0 * sc, min(c_off + (z0 + size - 1) * sc + c_ext, c_host.size)
        if args["beta"] != 0 or gaps:
            C.upload(c_lo, c_hi, slot, slot_events[slot])
        ev_in = torch.cuda.Event()
        ev_in.record(pipe.h2d)
        slot_events[slot] = ev_in
        cur.wait_event(ev_in)
        extras.gemm_strided_batched(ctx, layout, ta, tb, m, n, k, args["alpha"], A.buf, sa, B.buf, sb,
                                    args["beta"], C.buf, sc, size, a_offset=a_off + z0 * sa,
                                    b_offset=b_off + z0 * sb, c_offset=c_off + z0 * sc,
                                    lda=args["lda"], ldb=args["ldb"], ldc=args["ldc"],
                                    tf32=args.get("tf32", False))
        pipe.d2h.wait_stream(cur)
        _download(finishers, C, c_lo, c_hi, slot)
    for f in finishers:
        f()
    cur.synchronize()
    pipe.h2d.synchronize()
    pipe.d2h.synchronize()


def netlib_call(routine_id: str, *args, ctx: Context | None = None, **kwargs):
    """Invoke a GEMM routine by Netlib name on host NumPy arrays (in/out
    arrays updated in place; returns None like the device routines)."""
    rid = routine_id.lower()
    if len(rid) < 2 or rid[0] not in "hsdcz":
        raise UsageError(f"unknown routine id {routine_id!r}")
    if rid[0] not in _PRECISIONS or rid[1:] not in _ROUTINES:
        raise UsageError(f"routine {routine_id!r} is not part of the B200 GEMM path "
                         "(sgemm / hgemm / [sh]gemm_strided_batched)")
    precision = _PRECISIONS[rid[0]]
    fn, roles = _ROUTINES[rid[1:]]
    ctx = ctx or default_context()
    bound = _signature(fn).bind(ctx, *args, **kwargs)
    bound.apply_defaults()
    layout = bound.arguments.get("layout", Layout.COL_MAJOR)
    flats, views = {}, {}
    for name in roles:
        arr = bound.arguments.get(name)
        if arr is None:
            continue
        arr = np.asanyarray(arr)
        if arr.dtype != precision.dtype:
            raise UsageError(f"array {name!r} has dtype {arr.dtype}, routine {routine_id!r} "
                             f"expects {precision.dtype}")
        flats[name], views[name] = _storage(arr, layout), arr
    from ..kernels.dispatch import require_gpu

    require_gpu(ctx)
    pipe = _pipeline(ctx)
    xfers = {name: _Transfer(ctx, pipe, name, flat, precision) for name, flat in flats.items()}
    # Validate the whole call first, exactly as the device routine does (same
    # errors in the same order, before any copy), on the device buffers the
    # pipeline will use.
    for name, x in xfers.items():
        bound.arguments[name] = x.buf
    bound.arguments["_validate_only"] = True
    if not fn(*bound.args, **bound.kwargs):
        return None                                  # m == 0 or n == 0: a no-op
    bound.arguments["_validate_only"] = False
    if rid[1:] == "gemm":
        _gemm_pipelined(ctx, precision, xfers, bound)
    else:
        _strided_pipelined(ctx, precision, xfers, bound)
    for name, arr in views.items():
        if roles[name] in ("inout", "out"):
            flat = flats[name]
            if not np.shares_memory(flat, arr):
                arr[...] = flat.reshape(arr.shape, order="F" if layout is Layout.COL_MAJOR else "C")
    return None
