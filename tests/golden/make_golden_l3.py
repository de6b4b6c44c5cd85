"""Generate golden vectors for the structured level-3 routines by running the
REFERENCE (pkg/src/tunedblas/routines/level3.py:152-537).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_l3.py

Writes tests/golden/l3_golden.npz + l3_golden.json: per case the routine,
its arguments, the flat input buffers and the reference's output buffer
(symm / syrk / syr2k: C; trmm / trsm: B), for S and H.
"""

import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import tunedblas as tb  # noqa: E402  (the reference, read-only)

OUT = Path(__file__).resolve().parent


def main():
    ctx = tb.context_create(tb.host_device())
    rng = np.random.default_rng(20240612)
    P = {"S": tb.Precision.S, "H": tb.Precision.H}
    L = {"col": tb.Layout.COL_MAJOR, "row": tb.Layout.ROW_MAJOR}
    SIDE = {"L": tb.Side.LEFT, "R": tb.Side.RIGHT}
    TRI = {"U": tb.Triangle.UPPER, "L": tb.Triangle.LOWER}
    TR = {"n": tb.Transpose.NO, "t": tb.Transpose.YES}
    DG = {"N": tb.Diagonal.NON_UNIT, "U": tb.Diagonal.UNIT}
    cases, arrays = [], {}

    def buf(prec, arr):
        b = tb.buffer_alloc(ctx, P[prec], arr.size)
        b.data[:] = arr
        return b

    def mat(prec, rows, cols, layout, extra=0):
        v = rng.uniform(-1, 1, (rows, cols)).astype(P[prec].dtype)
        flat = v.reshape(-1, order="F" if layout == "col" else "C")
        return np.concatenate([flat, rng.uniform(-1, 1, extra).astype(P[prec].dtype)])

    def save(case, ins, out):
        i = len(cases)
        for name, arr in ins.items():
            arrays[f"l{i}_{name}"] = arr
        arrays[f"l{i}_out"] = out
        cases.append(case)

    for prec in ("S", "H"):
        for _ in range(10):   # symm
            lay, side, tri = rng.choice(["col", "row"]), rng.choice(["L", "R"]), rng.choice(["U", "L"])
            m, n = int(rng.integers(1, 40)), int(rng.integers(1, 40))
            na = m if side == "L" else n
            a, b, c = mat(prec, na, na, lay), mat(prec, m, n, lay), mat(prec, m, n, lay)
            alpha, beta = float(rng.uniform(-1.5, 1.5)), float(rng.uniform(-1.5, 1.5))
            cb = buf(prec, c)
            tb.symm(ctx, L[lay], SIDE[side], TRI[tri], m, n, alpha, buf(prec, a), buf(prec, b), beta, cb)
            save(dict(fn="symm", prec=prec, layout=lay, side=side, tri=tri, m=m, n=n, alpha=alpha, beta=beta),
                 {"a": a, "b": b, "c": c}, cb.data.copy())
        for fn in ("syrk", "syr2k"):
            for _ in range(10):
                lay, tri, tr = rng.choice(["col", "row"]), rng.choice(["U", "L"]), rng.choice(["n", "t"])
                n, k = int(rng.integers(1, 36)), int(rng.integers(0, 36))
                shape = (n, k) if tr == "n" else (k, n)
                a, b, c = mat(prec, *shape, lay), mat(prec, *shape, lay), mat(prec, n, n, lay)
                alpha, beta = float(rng.uniform(-1.5, 1.5)), float(rng.uniform(-1.5, 1.5))
                cb = buf(prec, c)
                if fn == "syrk":
                    tb.syrk(ctx, L[lay], TRI[tri], TR[tr], n, k, alpha, buf(prec, a), beta, cb)
                else:
                    tb.syr2k(ctx, L[lay], TRI[tri], TR[tr], n, k, alpha, buf(prec, a), buf(prec, b), beta, cb)
                save(dict(fn=fn, prec=prec, layout=lay, tri=tri, trans=tr, n=n, k=k, alpha=alpha, beta=beta),
                     {"a": a, "b": b, "c": c}, cb.data.copy())
        for fn in ("trmm", "trsm"):
            for i in range(12):
                lay, side = rng.choice(["col", "row"]), rng.choice(["L", "R"])
                tri, tr, dg = rng.choice(["U", "L"]), rng.choice(["n", "t"]), rng.choice(["N", "U"])
                big = i >= 10
                m = int(rng.integers(60, 140)) if big else int(rng.integers(1, 40))
                n = int(rng.integers(20, 70)) if big else int(rng.integers(1, 24))
                na = m if side == "L" else n
                av = rng.uniform(-1, 1, (na, na))
                if fn == "trsm":   # well-conditioned diagonal (routine_cases.py:749-751)
                    ii = np.arange(na)
                    av[ii, ii] += np.sign(av[ii, ii] + 0.1) * 2
                    av = av / np.sqrt(na)   # keep growth bounded
                    av[ii, ii] = np.sign(av[ii, ii]) * (np.abs(av[ii, ii]) + 1.0)
                av = av.astype(P[prec].dtype)
                a = av.reshape(-1, order="F" if lay == "col" else "C")
                b = mat(prec, m, n, lay)
                alpha = float(rng.uniform(-1.5, 1.5))
                bb = buf(prec, b)
                bs = int(rng.choice([4, 8, 16, 32]))
                if fn == "trmm":
                    tb.trmm(ctx, L[lay], SIDE[side], TRI[tri], TR[tr], DG[dg], m, n, alpha, buf(prec, a), bb)
                else:
                    tb.trsm(ctx, L[lay], SIDE[side], TRI[tri], TR[tr], DG[dg], m, n, alpha, buf(prec, a), bb,
                            block_size=bs)
                save(dict(fn=fn, prec=prec, layout=lay, side=side, tri=tri, trans=tr, diag=dg, m=m, n=n,
                          alpha=alpha, block_size=bs), {"a": a, "b": b}, bb.data.copy())

    np.savez_compressed(OUT / "l3_golden.npz", **arrays)
    (OUT / "l3_golden.json").write_text(json.dumps({"cases": cases}, indent=1))
    print(f"wrote {len(cases)} structured level-3 cases")


if __name__ == "__main__":
    main()
