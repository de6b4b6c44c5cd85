"""Generate golden GEMM vectors by running the REFERENCE implementation.

Run in the build container (needs /root/reference, which does not exist on
the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes tests/golden/gemm_golden.npz + gemm_golden.json: for every case the
flat input buffers, the routine arguments, and the output buffer the
reference's own ``tunedblas.gemm`` / ``gemm_batched`` /
``gemm_strided_batched`` produced (sequential backend, built-in config).
"""

import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import tunedblas as tb  # noqa: E402  (the reference, read-only)

OUT = Path(__file__).resolve().parent


def buf(ctx, prec, arr):
    b = tb.buffer_alloc(ctx, prec, arr.size)
    b.data[:] = arr
    return b


def main():
    ctx = tb.context_create(tb.host_device())
    rng = np.random.default_rng(20240521)
    cases, arrays = [], {}
    P = {"S": tb.Precision.S, "H": tb.Precision.H}
    L = {"col": tb.Layout.COL_MAJOR, "row": tb.Layout.ROW_MAJOR}
    T = {"n": tb.Transpose.NO, "t": tb.Transpose.YES}

    def add_gemm(prec, lay, ta, tbn, m, n, k, alpha, beta, a_off=0, b_off=0, c_off=0,
                 lda=None, ldb=None, ldc=None, c_fill=None, kernel=None):
        dt = P[prec].dtype
        a_rows, a_cols = (m, k) if ta == "n" else (k, m)
        b_rows, b_cols = (k, n) if tbn == "n" else (n, k)
        col = lay == "col"
        lda_ = lda if lda is not None else (a_rows if col else a_cols)
        ldb_ = ldb if ldb is not None else (b_rows if col else b_cols)
        ldc_ = ldc if ldc is not None else (m if col else n)
        def span(rows, cols, ld):
            r, c = (rows, cols) if col else (cols, rows)
            return ld * (c - 1) + r if r and c else 0
        la = a_off + span(a_rows, a_cols, lda_) + 3
        lb = b_off + span(b_rows, b_cols, ldb_) + 3
        lc = c_off + span(m, n, ldc_) + 3
        a = rng.uniform(-1, 1, la).astype(dt)
        b = rng.uniform(-1, 1, lb).astype(dt)
        c = rng.uniform(-1, 1, lc).astype(dt) if c_fill is None else np.full(lc, c_fill, dt)
        ab, bb, cb = buf(ctx, P[prec], a), buf(ctx, P[prec], b), buf(ctx, P[prec], c)
        tb.gemm(ctx, L[lay], T[ta], T[tbn], m, n, k, alpha, ab, bb, beta, cb,
                a_offset=a_off, lda=lda, b_offset=b_off, ldb=ldb, c_offset=c_off, ldc=ldc,
                kernel=kernel)
        i = len(cases)
        arrays[f"c{i}_a"], arrays[f"c{i}_b"], arrays[f"c{i}_c_in"] = a, b, c
        arrays[f"c{i}_c_out"] = cb.data.copy()
        cases.append(dict(kind="gemm", prec=prec, layout=lay, ta=ta, tb=tbn, m=m, n=n, k=k,
                          alpha=alpha, beta=beta, a_off=a_off, b_off=b_off, c_off=c_off,
                          lda=lda, ldb=ldb, ldc=ldc, kernel=kernel,
                          family=ctx.last_launch.family if ctx.last_launch else None))

    def add_strided(prec, lay, m, n, k, batch, alpha, beta):
        dt = P[prec].dtype
        ea, eb, ec = m * k, k * n, m * n
        a = rng.uniform(-1, 1, batch * ea).astype(dt)
        b = rng.uniform(-1, 1, batch * eb).astype(dt)
        c = rng.uniform(-1, 1, batch * ec).astype(dt)
        ab, bb, cb = buf(ctx, P[prec], a), buf(ctx, P[prec], b), buf(ctx, P[prec], c)
        tb.gemm_strided_batched(ctx, L[lay], tb.Transpose.NO, tb.Transpose.NO, m, n, k, alpha,
                                ab, ea, bb, eb, beta, cb, ec, batch)
        i = len(cases)
        arrays[f"c{i}_a"], arrays[f"c{i}_b"], arrays[f"c{i}_c_in"] = a, b, c
        arrays[f"c{i}_c_out"] = cb.data.copy()
        cases.append(dict(kind="strided", prec=prec, layout=lay, ta="n", tb="n", m=m, n=n, k=k,
                          batch=batch, alpha=alpha, beta=beta, stride_a=ea, stride_b=eb, stride_c=ec))

    def add_batched(prec, m, n, k, batch):
        dt = P[prec].dtype
        ea, eb, ec = m * k, k * n, m * n
        alphas = [float(x) for x in rng.uniform(0.5, 2, batch)]
        betas = [float(x) for x in rng.uniform(-1, 1, batch)]
        alphas[1] = 0.0  # an instance the reference finishes without the kernel
        a = rng.uniform(-1, 1, batch * ea).astype(dt)
        b = rng.uniform(-1, 1, batch * eb).astype(dt)
        c = rng.uniform(-1, 1, batch * ec).astype(dt)
        ao = [i * ea for i in range(batch)][::-1]
        bo = [i * eb for i in range(batch)]
        co = [i * ec for i in range(batch)]
        ab, bb, cb = buf(ctx, P[prec], a), buf(ctx, P[prec], b), buf(ctx, P[prec], c)
        tb.gemm_batched(ctx, tb.Layout.COL_MAJOR, tb.Transpose.NO, tb.Transpose.NO, m, n, k,
                        alphas, ab, ao, bb, bo, betas, cb, co, batch)
        i = len(cases)
        arrays[f"c{i}_a"], arrays[f"c{i}_b"], arrays[f"c{i}_c_in"] = a, b, c
        arrays[f"c{i}_c_out"] = cb.data.copy()
        cases.append(dict(kind="batched", prec=prec, layout="col", ta="n", tb="n", m=m, n=n, k=k,
                          batch=batch, alphas=alphas, betas=betas, a_offs=ao, b_offs=bo, c_offs=co))

    for prec in ("S", "H"):
        for lay in ("col", "row"):
            for ta in ("n", "t"):
                for tbn in ("n", "t"):
                    add_gemm(prec, lay, ta, tbn, 37, 29, 23, 1.25, 0.5)        # direct
        for lay, ta, tbn in (("col", "n", "n"), ("row", "t", "t"), ("col", "t", "n"), ("row", "n", "t")):
            add_gemm(prec, lay, ta, tbn, 129, 130, 131, 1.0, 0.0)                # indirect, odd
        add_gemm(prec, "col", "n", "n", 6, 5, 4, 1.0, 0.0, c_off=2, ldc=9)    # canary layout
        add_gemm(prec, "col", "n", "n", 64, 48, 40, 1.0, 0.0, c_fill=np.nan)   # beta=0 over NaN
        add_gemm(prec, "row", "t", "n", 20, 30, 0, 1.0, 0.75)                  # k == 0
        add_gemm(prec, "col", "n", "t", 33, 17, 70, 0.0, -1.5)                 # alpha == 0
        add_gemm(prec, "col", "t", "t", 100, 100, 100, 1.0, 0.0, kernel="direct")
        add_gemm(prec, "col", "t", "t", 100, 100, 100, 1.0, 0.0, kernel="indirect")
        add_gemm(prec, "row", "n", "n", 150, 130, 140, 0.5, 2.0, a_off=3, b_off=5, c_off=7,
                 lda=141, ldb=133, ldc=131)
        add_strided(prec, "col", 32, 32, 32, 16, 1.0, 0.0)
        add_strided(prec, "row", 24, 20, 16, 5, 1.5, 0.5)
        add_batched(prec, 16, 12, 8, 6)
    np.savez_compressed(OUT / "gemm_golden.npz", **arrays)
    with open(OUT / "gemm_golden.json", "w") as fh:
        json.dump({"generator": "tests/golden/make_golden.py",
                   "reference": "tunedblas (pkg/src) sequential backend, built-in config",
                   "numpy": np.__version__, "cases": cases}, fh, indent=1)
    print(f"{len(cases)} cases, {sum(a.nbytes for a in arrays.values())/1e6:.2f} MB raw")


if __name__ == "__main__":
    main()
