"""The numerical tolerance model (pkg/src/tunedblas/reference.py:68-99) and a
device-side verification helper used by the tuner and the bench clients.

Tolerance: per element 4 * eps * K * max_k |a_ik| |b_kj| with eps the storage
unit roundoff (2^-23 for S, 2^-10 for H); two implementations are compared at
2x that (tests/test_level3.py:84-85 of the reference).

This module computes no GEMM results for the routines.  ``device_expected``
produces the float64 product that candidates are *checked* against (the
reference's tuner checks every candidate against ``ref_gemm``,
tuner.py:267-269); it runs on the GPU in float64 and is never used as a
result path.
"""

from __future__ import annotations

import numpy as np

from .core import Precision

__all__ = ["gemm_tolerance", "allclose_tol", "gemm_tolerance_device", "device_expected",
           "device_within_tol"]


def gemm_tolerance(a: np.ndarray, b: np.ndarray, precision: Precision,
                   row_block: int = 64) -> np.ndarray:
    """Per-element bound 4*eps*K*max_k |a_ik|*|b_kj| for C = a@b (exact)."""
    eps = precision.eps
    k = a.shape[1]
    absa = np.abs(a).astype(np.float64)
    absb = np.abs(b).astype(np.float64)
    m, n = absa.shape[0], absb.shape[1]
    bound = np.empty((m, n))
    for r0 in range(0, m, row_block):
        r1 = min(r0 + row_block, m)
        bound[r0:r1] = np.max(absa[r0:r1, :, None] * absb[None, :, :], axis=1)
    return 4.0 * eps * max(k, 1) * bound


def allclose_tol(actual, expected, tol, scale: float = 1.0) -> bool:
    """Elementwise |actual - expected| <= scale*tol (+ tiny absolute floor)."""
    diff = np.abs(np.asarray(actual, dtype=np.complex128) - np.asarray(expected, dtype=np.complex128))
    limit = scale * np.asarray(tol, dtype=np.float64) + 1e-300
    return bool(np.all(diff <= limit))


def gemm_tolerance_device(a, b, precision: Precision, budget_bytes: int = 1 << 28):
    """The same exact bound evaluated on the GPU (a: m x k, b: k x n tensors)."""
    import torch

    absa = a.abs().to(torch.float64)
    absb = b.abs().to(torch.float64)
    m, k = absa.shape
    n = absb.shape[1]
    out = torch.empty((m, n), dtype=torch.float64, device=a.device)
    rows = max(1, budget_bytes // max(1, 8 * k * n))
    for r0 in range(0, m, rows):
        r1 = min(m, r0 + rows)
        out[r0:r1] = (absa[r0:r1, :, None] * absb[None, :, :]).amax(dim=1)
    return out * (4.0 * precision.eps * max(k, 1))


def device_expected(a, b, alpha=1.0, beta=0.0, c=None):
    """float64 alpha*a@b (+ beta*c) on the device — a checker, not a result path."""
    import torch

    out = alpha * (a.to(torch.float64) @ b.to(torch.float64))
    if beta != 0 and c is not None:
        out = out + beta * c.to(torch.float64)
    return out


def device_within_tol(actual, expected, tol, scale: float = 1.0) -> bool:
    diff = (actual.to(expected.dtype) - expected).abs()
    return bool((diff <= scale * tol + 1e-300).all().item())
