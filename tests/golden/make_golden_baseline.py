"""Golden outputs of the REFERENCE at the BASELINE.json configurations.

Run in the build container (needs /root/reference, which does not exist on
the GPU box):

    python tests/golden/make_golden_baseline.py

Cases (SURVEY §8 naming):
* C1  1024^3 row-major NN alpha=1 beta=0, S and H
* C3a (64, 3136, 576) and C3b (4096, 128, 9216) row-major NN, S and H
* C4  256-instance prefixes of the 16384 x 32^3 and x 64^3 strided batches,
      row-major NN packed strides, S and H

Inputs are NOT stored: every operand is ``default_rng(seed).uniform(-1, 1,
size).astype(dtype)`` (PCG64 streams are stable across NumPy versions) and
the JSON records a SHA-256 of each generated operand so the GPU-side test
proves it regenerated the same bytes.  Only the reference's outputs are
stored (tests/golden/baseline_golden.npz), produced by ``tunedblas.gemm`` /
``tunedblas.gemm_strided_batched`` on the sequential backend with the
built-in configuration.
"""

import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

OUT = Path(__file__).resolve().parent

CASES = [
    # name, kind, prec, m, n, k, batch, seed
    ("C1_S", "gemm", "S", 1024, 1024, 1024, 1, 101),
    ("C1_H", "gemm", "H", 1024, 1024, 1024, 1, 102),
    ("C3a_S", "gemm", "S", 64, 3136, 576, 1, 103),
    ("C3a_H", "gemm", "H", 64, 3136, 576, 1, 104),
    ("C3b_S", "gemm", "S", 4096, 128, 9216, 1, 105),
    ("C3b_H", "gemm", "H", 4096, 128, 9216, 1, 106),
    ("C4_32_S", "strided", "S", 32, 32, 32, 256, 107),
    ("C4_32_H", "strided", "H", 32, 32, 32, 256, 108),
    ("C4_64_S", "strided", "S", 64, 64, 64, 256, 109),
    ("C4_64_H", "strided", "H", 64, 64, 64, 256, 110),
]


def operands(prec: str, m: int, n: int, k: int, batch: int, seed: int):
    """The case's A and B (flat, row-major packed), shared with the tests."""
    dt = np.float16 if prec == "H" else np.float32
    rng = np.random.default_rng(seed)
    a = rng.uniform(-1, 1, m * k * batch).astype(dt)
    b = rng.uniform(-1, 1, k * n * batch).astype(dt)
    return a, b


def digest(arr: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(arr).tobytes()).hexdigest()


def main():
    sys.path.insert(0, "/root/reference/pkg/src")
    import tunedblas as tb  # the reference, read-only

    ctx = tb.context_create(tb.host_device())
    P = {"S": tb.Precision.S, "H": tb.Precision.H}
    R, N = tb.Layout.ROW_MAJOR, tb.Transpose.NO
    meta, arrays = [], {}
    for name, kind, prec, m, n, k, batch, seed in CASES:
        a, b = operands(prec, m, n, k, batch, seed)
        ab = tb.buffer_alloc(ctx, P[prec], a.size)
        ab.data[:] = a
        bb = tb.buffer_alloc(ctx, P[prec], b.size)
        bb.data[:] = b
        cb = tb.buffer_alloc(ctx, P[prec], m * n * batch)
        t0 = time.perf_counter()
        if kind == "gemm":
            tb.gemm(ctx, R, N, N, m, n, k, 1.0, ab, bb, 0.0, cb)
        else:
            tb.gemm_strided_batched(ctx, R, N, N, m, n, k, 1.0, ab, m * k, bb, k * n, 0.0, cb,
                                    m * n, batch)
        dt = time.perf_counter() - t0
        arrays[name] = cb.data.copy()
        meta.append(dict(name=name, kind=kind, prec=prec, m=m, n=n, k=k, batch=batch, seed=seed,
                         layout="row", ta="n", tb="n", alpha=1.0, beta=0.0,
                         sha_a=digest(a), sha_b=digest(b), sha_c=digest(arrays[name]),
                         family=ctx.last_launch.family if ctx.last_launch else None,
                         reference_seconds=round(dt, 3)))
        print(f"{name}: {dt:.2f} s", flush=True)
    np.savez_compressed(OUT / "baseline_golden.npz", **arrays)
    with open(OUT / "baseline_golden.json", "w") as fh:
        json.dump({"generator": "tests/golden/make_golden_baseline.py",
                   "reference": "tunedblas (pkg/src) sequential backend, built-in config",
                   "inputs": "default_rng(seed).uniform(-1, 1, size).astype(dtype): A then B, "
                             "row-major packed (see operands())",
                   "numpy": np.__version__, "cases": meta}, fh, indent=1)


if __name__ == "__main__":
    main()
