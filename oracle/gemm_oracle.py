"""oracle/gemm_oracle.py — TEST INFRASTRUCTURE ONLY.

CPU restatement of the reference GEMM hot path, used (a) as the parity
checker in tests/, (b) by ``__graft_entry__.smoke()`` and (c) as the CPU
baseline leg of bench.py (``cpu_baseline.kind = "port"``; also the
``--impl reference`` arm).  Nothing in the product package imports this.

Contents (each function cites what it restates):

* ``ref_gemm`` / ``gemm_tolerance`` / ``allclose_tol`` — the reference's
  naive oracle and tolerance model (pkg/src/tunedblas/reference.py:52-99).
* ``port_gemm`` — the reference routine ``gemm`` on host arrays with its
  tiled algorithm: route by ``direct_threshold`` (level3.py:57-59), pad to
  tile multiples with B transposed (level3.py:71-82), per-tile
  ``_tile_product`` = KWG chunks x KWI slabs multiplied with one np.matmul
  and summed pairwise over slabs then chunks (compute.py:360-381), FP32
  epilogue (compute.py:408-412), one rounding on unpad (level3.py:91); the
  direct path's bounds-checked tiles (compute.py:432-471).  Tiles run on a
  thread pool like the reference's parallel backend (engine.py:134-137).
* ``port_gemm_strided_batched`` — the per-instance loop of
  _gemm_batched_core (extras.py:188-286) on the sequential backend.
* ``seqk_gemm`` — ctypes wrapper of oracle/gemm_seqk.c (sequential-k FMA
  chain; bit-exact checker for the GPU SGEMM contract); ``seqk_gemm_split``
  — the same chain cut into the GPU's split-K ranges and summed in rank
  order (bit-exact checker for the split-K SGEMM route).
* ``port_im2col`` — the reference's ``im2col`` gather (extras.py:56-109):
  index grids per (channel, ky, kx) row and (oy, ox) column, zero outside the
  image, written column-major with ld = rows.  Pinned bitwise to
  tests/golden/im2col_golden.* (made by running the reference).

Parity anchor: tests/golden/ holds outputs of the reference itself
(tests/golden/make_golden.py imports /root/reference); tests/test_oracle.py
pins this port to them.
"""

from __future__ import annotations

import ctypes
import os
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

import numpy as np

EPS = {"H": 2.0 ** -10, "S": 2.0 ** -23}
DTYPE = {"H": np.float16, "S": np.float32}

#: The reference's built-in gemm configuration (params.py:424, 130-143).
REFERENCE_DEFAULT = dict(MWG=64, NWG=64, KWG=16, KWI=8, MDIMA=8, NDIMB=8,
                         SA=1, SB=1, STRM=0, STRN=0)
DIRECT_THRESHOLD = 128  # tuningdb.py:303


# ---------------------------------------------------------------------------
# Naive oracle and tolerance (reference.py:52-99)
# ---------------------------------------------------------------------------

def ref_gemm(alpha, a, b, beta, c, prec: str) -> np.ndarray:
    """One matmul in the FP32 compute dtype, epilogue, one rounding."""
    prod = a.astype(np.float32) @ b.astype(np.float32)
    alpha, beta = np.float32(alpha), np.float32(beta)
    out = alpha * prod if beta == 0 else alpha * prod + beta * c.astype(np.float32)
    return out.astype(DTYPE[prec])


def gemm_tolerance(a, b, prec: str, row_block: int = 64) -> np.ndarray:
    """4 * eps * K * max_k |a_ik| |b_kj| per element (reference.py:68-83)."""
    k = a.shape[1]
    absa = np.abs(a).astype(np.float64)
    absb = np.abs(b).astype(np.float64)
    bound = np.empty((absa.shape[0], absb.shape[1]))
    for r0 in range(0, absa.shape[0], row_block):
        r1 = min(r0 + row_block, absa.shape[0])
        bound[r0:r1] = np.max(absa[r0:r1, :, None] * absb[None, :, :], axis=1)
    return 4.0 * EPS[prec] * max(k, 1) * bound


def allclose_tol(actual, expected, tol, scale=1.0) -> bool:
    diff = np.abs(np.asarray(actual, np.float64) - np.asarray(expected, np.float64))
    return bool(np.all(diff <= scale * np.asarray(tol, np.float64) + 1e-300))


def wide_oracle(alpha, a_op, b_op, beta, c) -> np.ndarray:
    """float64 alpha*op(A)op(B) + beta*C (tests/oracles.py:44-51 style)."""
    out = float(alpha) * (a_op.astype(np.float64) @ b_op.astype(np.float64))
    if beta != 0:
        out = out + float(beta) * c.astype(np.float64)
    return out


# ---------------------------------------------------------------------------
# Port of the tiled algorithm (compute.py:338-471, level3.py:48-91)
# ---------------------------------------------------------------------------

def _ceil_to(x: int, step: int) -> int:
    return -(-x // step) * step


def _slab_product(a_tile, bt_tile, kwg, kwi):
    """(Tm, Tn) tile: K split in KWG chunks of KWI-wide slabs, each slab one
    matmul, summed over slabs then over chunks (compute.py:360-381).  The
    SA/SB staging copies and STRM/STRN permutations change no values."""
    tm, k = a_tile.shape
    tn = bt_tile.shape[0]
    nchunk, ns = k // kwg, kwg // kwi
    a4 = np.ascontiguousarray(a_tile.reshape(tm, nchunk, kwg).transpose(1, 0, 2))
    b4 = np.ascontiguousarray(bt_tile.reshape(tn, nchunk, kwg).transpose(1, 0, 2))
    a_s = a4.reshape(nchunk, tm, ns, kwi).transpose(0, 2, 1, 3)
    b_s = b4.reshape(nchunk, tn, ns, kwi).transpose(0, 2, 3, 1)
    return np.matmul(a_s, b_s).sum(axis=1).sum(axis=0)


def _indirect(alpha, beta, a_arr, bt_arr, c_view, cfg, pool, out_dtype):
    m, k = a_arr.shape
    n = bt_arr.shape[0]
    mwg, nwg, kwg, kwi = cfg["MWG"], cfg["NWG"], cfg["KWG"], cfg["KWI"]
    mp, np_, kp = _ceil_to(max(m, 1), mwg), _ceil_to(max(n, 1), nwg), _ceil_to(max(k, 1), kwg)
    aw = np.zeros((mp, kp), np.float32)
    aw[:m, :k] = a_arr
    btw = np.zeros((np_, kp), np.float32)
    btw[:n, :k] = bt_arr
    cw = np.zeros((mp, np_), np.float32)
    if beta != 0:
        cw[:m, :n] = c_view.astype(np.float32)

    def task(i0, j0):
        acc = _slab_product(aw[i0:i0 + mwg], btw[j0:j0 + nwg], kwg, kwi)
        out = cw[i0:i0 + mwg, j0:j0 + nwg]
        if beta == 0:
            out[...] = alpha * acc
        else:
            out[...] = alpha * acc + beta * out

    tiles = [(i0, j0) for i0 in range(0, mp, mwg) for j0 in range(0, np_, nwg)]
    if pool is None:
        for t in tiles:
            task(*t)
    else:
        list(pool.map(lambda t: task(*t), tiles))
    c_view[...] = cw[:m, :n].astype(out_dtype)


def _direct(alpha, beta, a_arr, bt_arr, c_view, cfg, pool, out_dtype):
    m, k = a_arr.shape
    n = bt_arr.shape[0]
    mwg, nwg, kwg, kwi = cfg["MWG"], cfg["NWG"], cfg["KWG"], cfg["KWI"]

    def task(i0, j0):
        i1, j1 = min(i0 + mwg, m), min(j0 + nwg, n)
        at, bt = a_arr[i0:i1], bt_arr[j0:j1]
        acc = np.zeros((i1 - i0, j1 - j0), np.float32)
        for k0 in range(0, k, kwg):
            k1 = min(k0 + kwg, k)
            if k1 - k0 == kwg and kwg % kwi == 0:
                acc += _slab_product(at[:, k0:k1], bt[:, k0:k1], kwg, kwi)
            else:
                acc += at[:, k0:k1] @ bt[:, k0:k1].T
        out = c_view[i0:i1, j0:j1]
        if beta == 0:
            out[...] = (alpha * acc).astype(out_dtype)
        else:
            out[...] = (alpha * acc + beta * out.astype(np.float32)).astype(out_dtype)

    tiles = [(i0, j0) for i0 in range(0, m, mwg) for j0 in range(0, n, nwg)]
    if pool is None:
        for t in tiles:
            task(*t)
    else:
        list(pool.map(lambda t: task(*t), tiles))


def logical(buf: np.ndarray, offset: int, rows: int, cols: int, ld: int, row_major: bool):
    """Logical (rows, cols) strided view over a flat array (core.py:345-362,
    level3.py:41-45)."""
    if rows == 0 or cols == 0:
        return np.empty((rows, cols), buf.dtype)
    if not row_major:
        v = np.lib.stride_tricks.as_strided(buf[offset:], shape=(cols, ld),
                                            strides=(ld * buf.itemsize, buf.itemsize))
        return v.T[:rows, :]
    v = np.lib.stride_tricks.as_strided(buf[offset:], shape=(rows, ld),
                                        strides=(ld * buf.itemsize, buf.itemsize))
    return v[:, :cols]


def port_gemm(prec: str, row_major: bool, trans_a: bool, trans_b: bool, m, n, k, alpha,
              a: np.ndarray, b: np.ndarray, beta, c: np.ndarray, *, a_offset=0, lda=None,
              b_offset=0, ldb=None, c_offset=0, ldc=None, kernel=None, cfg=None,
              pool: ThreadPoolExecutor | None = None) -> None:
    """The reference ``gemm`` routine on flat host arrays (level3.py:94-149)."""
    cfg = dict(REFERENCE_DEFAULT if cfg is None else cfg)
    if m == 0 or n == 0:
        return
    a_rows, a_cols = (m, k) if not trans_a else (k, m)
    b_rows, b_cols = (k, n) if not trans_b else (n, k)
    lda = lda if lda is not None else (a_cols if row_major else a_rows)
    ldb = ldb if ldb is not None else (b_cols if row_major else b_rows)
    ldc = ldc if ldc is not None else (n if row_major else m)
    av = logical(a, a_offset, a_rows, a_cols, lda, row_major)
    bv = logical(b, b_offset, b_rows, b_cols, ldb, row_major)
    cv = logical(c, c_offset, m, n, ldc, row_major)
    alpha, beta = np.float32(alpha), np.float32(beta)
    out_dtype = c.dtype
    if k == 0 or alpha == 0:
        cv[...] = 0 if beta == 0 else (beta * cv.astype(np.float32)).astype(out_dtype)
        return
    a_arr = np.ascontiguousarray(av if not trans_a else av.T, dtype=np.float32)
    bt_arr = np.ascontiguousarray(bv.T if not trans_b else bv, dtype=np.float32)
    route = kernel or ("direct" if max(m, n, k) < DIRECT_THRESHOLD else "indirect")
    if route == "direct":
        _direct(alpha, beta, a_arr, bt_arr, cv, cfg, pool, out_dtype)
    else:
        _indirect(alpha, beta, a_arr, bt_arr, cv, cfg, pool, out_dtype)


def port_gemm_strided_batched(prec, row_major, trans_a, trans_b, m, n, k, alpha, a, stride_a,
                              b, stride_b, beta, c, stride_c, batch, *, a_offset=0, b_offset=0,
                              c_offset=0, lda=None, ldb=None, ldc=None, pool=None):
    """Per-instance loop of _gemm_batched_core (extras.py:188-286)."""
    for z in range(batch):
        port_gemm(prec, row_major, trans_a, trans_b, m, n, k, alpha, a, b, beta, c,
                  a_offset=a_offset + z * stride_a, lda=lda, b_offset=b_offset + z * stride_b,
                  ldb=ldb, c_offset=c_offset + z * stride_c, ldc=ldc, pool=pool)


def make_pool(threads: int | None = None) -> ThreadPoolExecutor:
    """The reference's parallel backend: os.cpu_count() workers (core.py:210-255)."""
    return ThreadPoolExecutor(max_workers=threads or os.cpu_count() or 1)


# ---------------------------------------------------------------------------
# C restatement (oracle/gemm_seqk.c)
# ---------------------------------------------------------------------------

_C = None


def c_library_path() -> Path:
    return Path(__file__).resolve().parent / "_build" / "liboracle.so"


def c_lib():
    global _C
    if _C is None:
        path = c_library_path()
        if not path.exists():
            import subprocess

            subprocess.run(["make", "-C", str(path.parent.parent)], check=True,
                           stdout=subprocess.DEVNULL)
        so = ctypes.CDLL(str(path))
        i32, i64, f32, vp = ctypes.c_int, ctypes.c_int64, ctypes.c_float, ctypes.c_void_p
        so.oracle_gemm.restype = i32
        so.oracle_gemm.argtypes = [i32, i32, i32, i32, i64, i64, i64, f32, vp, i64, i64,
                                   vp, i64, i64, f32, vp, i64, i64]
        so.oracle_gemm_strided_batched.restype = i32
        so.oracle_gemm_strided_batched.argtypes = [i32, i32, i32, i32, i64, i64, i64, f32,
                                                   vp, i64, i64, i64, vp, i64, i64, i64, f32,
                                                   vp, i64, i64, i64, i64]
        so.oracle_h2f.restype = ctypes.c_float
        so.oracle_h2f.argtypes = [ctypes.c_uint16]
        so.oracle_f2h.restype = ctypes.c_uint16
        so.oracle_f2h.argtypes = [ctypes.c_float]
        _C = so
    return _C


def _ptr(arr: np.ndarray) -> int:
    assert arr.flags["C_CONTIGUOUS"]
    return arr.ctypes.data


def seqk_gemm(prec: str, row_major: bool, trans_a: bool, trans_b: bool, m, n, k, alpha,
              a: np.ndarray, a_offset, lda, b: np.ndarray, b_offset, ldb, beta, c: np.ndarray,
              c_offset, ldc) -> None:
    """Sequential-k FMA GEMM in place on flat host arrays (C oracle)."""
    rc = c_lib().oracle_gemm(0 if prec == "H" else 1, 1 if row_major else 0, int(trans_a),
                             int(trans_b), m, n, k, float(alpha), _ptr(a), a_offset, lda,
                             _ptr(b), b_offset, ldb, float(beta), _ptr(c), c_offset, ldc)
    if rc:
        raise ValueError("oracle_gemm rejected its arguments")


def seqk_gemm_strided_batched(prec, row_major, trans_a, trans_b, m, n, k, alpha, a, a_offset,
                              lda, stride_a, b, b_offset, ldb, stride_b, beta, c, c_offset, ldc,
                              stride_c, batch) -> None:
    rc = c_lib().oracle_gemm_strided_batched(
        0 if prec == "H" else 1, 1 if row_major else 0, int(trans_a), int(trans_b), m, n, k,
        float(alpha), _ptr(a), a_offset, lda, stride_a, _ptr(b), b_offset, ldb, stride_b,
        float(beta), _ptr(c), c_offset, ldc, stride_c, batch)
    if rc:
        raise ValueError("oracle_gemm_strided_batched rejected its arguments")


def seqk_gemm_split(prec: str, row_major: bool, trans_a: bool, trans_b: bool, m, n, k, alpha,
                    a: np.ndarray, a_offset, lda, b: np.ndarray, b_offset, ldb, beta, c: np.ndarray,
                    c_offset, ldc, ks: int, stage: int = 32) -> None:
    """The GPU's deterministic split-K SGEMM (csrc/sgemm_tma.cuh, KS > 1):
    rank r runs the sequential-k chain over K stages [r*kt, (r+1)*kt) of
    `stage` elements (kt = ceil(ceil(k/stage)/ks)), the partials are added in
    rank order with FP32 roundings, then the reference epilogue (alpha*acc,
    + beta*C as separately rounded FP32 ops; compute.py:408-412).  Any layout
    and transposition (the K slices are cut from the logical op(A), op(B))."""
    assert prec == "S"
    kt = -(-(-(-k // stage)) // ks)
    ar, ac = (k, m) if trans_a else (m, k)
    br, bc = (n, k) if trans_b else (k, n)
    A = logical(a, a_offset, ar, ac, lda, row_major)
    B = logical(b, b_offset, br, bc, ldb, row_major)
    A = A.T if trans_a else A
    B = B.T if trans_b else B
    total = None
    for r in range(ks):
        k0, k1 = min(k, r * kt * stage), min(k, (r + 1) * kt * stage)
        part = np.zeros(m * n, np.float32)
        if k1 > k0:
            a_s = np.ascontiguousarray(A[:, k0:k1], np.float32).ravel()
            b_s = np.ascontiguousarray(B[k0:k1, :], np.float32).ravel()
            seqk_gemm("S", True, False, False, m, n, k1 - k0, 1.0, a_s, 0, k1 - k0, b_s, 0, n, 0.0, part, 0, n)
        total = part if total is None else (total + part).astype(np.float32)
    cv = logical(c, c_offset, m, n, ldc, row_major)
    al, be = np.float32(alpha), np.float32(beta)
    acc = total.reshape(m, n)
    out = (al * acc).astype(np.float32)
    if be != 0:
        out = (out + (be * cv.astype(np.float32)).astype(np.float32)).astype(np.float32)
    cv[...] = out


def port_im2col(image_flat: np.ndarray, im_offset: int, channels: int, height: int, width: int,
                kernel_h: int, kernel_w: int, pad_h: int, pad_w: int, stride_h: int, stride_w: int,
                dilation_h: int, dilation_w: int, col_flat: np.ndarray, col_offset: int) -> np.ndarray:
    """extras.py:56-109 on host arrays: writes the (C*KH*KW) x (OH*OW)
    column-major patch matrix into ``col_flat`` at ``col_offset`` and returns
    ``col_flat``.  Same index arithmetic as the reference (y = ky*dh + oy*sh -
    ph, x = kx*dw + ox*sw - pw; zero where outside the image)."""
    span_h = dilation_h * (kernel_h - 1) + 1
    span_w = dilation_w * (kernel_w - 1) + 1
    out_h = (height + 2 * pad_h - span_h) // stride_h + 1
    out_w = (width + 2 * pad_w - span_w) // stride_w + 1
    image = image_flat[im_offset:im_offset + channels * height * width].reshape(channels, height, width)
    y = np.arange(kernel_h)[:, None] * dilation_h + np.arange(out_h)[None, :] * stride_h - pad_h
    x = np.arange(kernel_w)[:, None] * dilation_w + np.arange(out_w)[None, :] * stride_w - pad_w
    y_ok, x_ok = (y >= 0) & (y < height), (x >= 0) & (x < width)
    g = image[:, np.clip(y, 0, height - 1)[:, None, :, None], np.clip(x, 0, width - 1)[None, :, None, :]]
    mask = (y_ok[:, None, :, None] & x_ok[None, :, None, :])[None, ...]
    mat = np.where(mask, g, 0).astype(col_flat.dtype).reshape(channels * kernel_h * kernel_w, out_h * out_w)
    rows, cols = mat.shape
    col_flat[col_offset:col_offset + rows * cols] = mat.reshape(-1, order="F")
    return col_flat
