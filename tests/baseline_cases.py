"""Shared helpers for the BASELINE-configuration golden cases
(tests/golden/make_golden_baseline.py ran the reference to make them)."""

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

GOLDEN_DIR = Path(__file__).resolve().parent / "golden"
sys.path.insert(0, str(GOLDEN_DIR))

from make_golden_baseline import operands  # noqa: E402  (pure NumPy; no reference import)

EPS = {"H": 2.0 ** -10, "S": 2.0 ** -23}


def load():
    with open(GOLDEN_DIR / "baseline_golden.json") as fh:
        meta = json.load(fh)
    return meta["cases"], np.load(GOLDEN_DIR / "baseline_golden.npz")


def digest(arr: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(arr).tobytes()).hexdigest()


def case_operands(case):
    return operands(case["prec"], case["m"], case["n"], case["k"], case["batch"], case["seed"])


def instance_views(case, a, b, c):
    """Per-instance logical (A, B, C) views of row-major packed flat arrays."""
    m, n, k = case["m"], case["n"], case["k"]
    for z in range(case["batch"]):
        yield (a[z * m * k:(z + 1) * m * k].reshape(m, k), b[z * k * n:(z + 1) * k * n].reshape(k, n),
               c[z * m * n:(z + 1) * m * n].reshape(m, n))


def tolerance(prec: str, a: np.ndarray, b: np.ndarray, wide: np.ndarray, rows: int = 16) -> np.ndarray:
    """The reference bound 4*eps*K*max_k |a_ik||b_kj| (reference.py:68-83),
    evaluated in row blocks small enough for (4096, 128, 9216), plus 2^-11 |C|
    for the FP16 output rounding."""
    k = a.shape[1]
    absa, absb = np.abs(a.astype(np.float32)), np.abs(b.astype(np.float32))
    bound = np.empty((a.shape[0], b.shape[1]), np.float64)
    for r0 in range(0, a.shape[0], rows):
        bound[r0:r0 + rows] = np.max(absa[r0:r0 + rows, :, None] * absb[None, :, :], axis=1)
    tol = 4.0 * EPS[prec] * max(k, 1) * bound
    if prec == "H":
        tol = tol + 2.0 ** -11 * np.abs(wide) + 2.0 ** -24
    return tol + 1e-30


def max_ratio(got, want, tol) -> float:
    return float(np.max(np.abs(np.asarray(got, np.float64) - want) / tol))
