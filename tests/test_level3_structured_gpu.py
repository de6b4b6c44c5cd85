"""GPU parity of the structured level-3 routines (symm / syrk / syr2k / trmm
/ trsm over the sm_100a GEMM).  Each golden case (tests/golden/l3_golden.*,
made by running the reference) is checked against the float64 product with
the reference's own tolerance model (tests/routine_cases.py:616-767 of the
reference) and against the reference's output within 2x that tolerance; the
rank-k updates must leave the other triangle bitwise untouched."""

import json

import numpy as np
import pytest

import paper_1705_05249_b200 as tb
from paper_1705_05249_b200 import Diagonal, Layout, Precision, Side, Transpose, Triangle
from conftest import GOLDEN_DIR

pytestmark = pytest.mark.gpu

META = json.loads((GOLDEN_DIR / "l3_golden.json").read_text())
CASES = META["cases"]
ARR = np.load(GOLDEN_DIR / "l3_golden.npz")
P = {"S": Precision.S, "H": Precision.H}
EPS = {"S": 2.0 ** -23, "H": 2.0 ** -10}
L = {"col": Layout.COL_MAJOR, "row": Layout.ROW_MAJOR}
SIDE = {"L": Side.LEFT, "R": Side.RIGHT}
TRI = {"U": Triangle.UPPER, "L": Triangle.LOWER}
TR = {"n": Transpose.NO, "t": Transpose.YES}
DG = {"N": Diagonal.NON_UNIT, "U": Diagonal.UNIT}


def logical(flat, rows, cols, layout):
    f = np.asarray(flat, dtype=np.float64)[:rows * cols]
    return f.reshape(cols, rows).T if layout == "col" else f.reshape(rows, cols)


def tri_mask(n, tri):
    ii, jj = np.arange(n)[:, None], np.arange(n)[None, :]
    return (ii <= jj) if tri == "U" else (ii >= jj)


def sym_full(a, tri):
    mask = tri_mask(a.shape[0], tri)
    return np.where(mask, a, a.T)


def tri_full(a, tri, dg):
    full = np.where(tri_mask(a.shape[0], tri), a, 0.0)
    if dg == "U":
        np.fill_diagonal(full, 1.0)
    return full


def _buf(ctx, prec, arr):
    b = tb.buffer_alloc(ctx, prec, arr.size)
    tb.buffer_write(b, 0, arr)
    return b


@pytest.mark.parametrize("i", range(len(CASES)), ids=[f"{c['fn']}{i}{c['prec']}" for i, c in enumerate(CASES)])
def test_structured_parity(ctx, i):
    cs = CASES[i]
    prec, fn, lay = P[cs["prec"]], cs["fn"], cs["layout"]
    eps = EPS[cs["prec"]]
    a_in, b_in = ARR[f"l{i}_a"], ARR[f"l{i}_b"]
    ref_out = ARR[f"l{i}_out"].astype(np.float64)
    if fn == "symm":
        m, n, side = cs["m"], cs["n"], cs["side"]
        na = m if side == "L" else n
        c_in = ARR[f"l{i}_c"]
        c = _buf(ctx, prec, c_in)
        tb.symm(ctx, L[lay], SIDE[side], TRI[cs["tri"]], m, n, cs["alpha"], _buf(ctx, prec, a_in),
                _buf(ctx, prec, b_in), cs["beta"], c)
        got = logical(tb.buffer_read(c, 0, m * n), m, n, lay)
        full = sym_full(logical(a_in, na, na, lay), cs["tri"])
        B, C0 = logical(b_in, m, n, lay), logical(c_in, m, n, lay)
        prod = full @ B if side == "L" else B @ full
        want = cs["alpha"] * prod + cs["beta"] * C0
        tol = abs(cs["alpha"]) * 4 * eps * na * (np.abs(prod) + na / 4 + 1) + 4 * eps * np.abs(cs["beta"] * C0) + 1e-30
        ref = logical(ref_out, m, n, lay)
        assert np.all(np.abs(got - want) <= tol)
        assert np.all(np.abs(got - ref) <= 2 * tol)
    elif fn in ("syrk", "syr2k"):
        n, k, tr, tri = cs["n"], cs["k"], cs["trans"], cs["tri"]
        shape = (n, k) if tr == "n" else (k, n)
        c_in = ARR[f"l{i}_c"]
        c = _buf(ctx, prec, c_in)
        a = _buf(ctx, prec, a_in)
        if fn == "syrk":
            tb.syrk(ctx, L[lay], TRI[tri], TR[tr], n, k, cs["alpha"], a, cs["beta"], c)
        else:
            tb.syr2k(ctx, L[lay], TRI[tri], TR[tr], n, k, cs["alpha"], a, _buf(ctx, prec, b_in), cs["beta"], c)
        got = logical(tb.buffer_read(c, 0, n * n), n, n, lay)
        A, B, C0 = logical(a_in, *shape, lay), logical(b_in, *shape, lay), logical(c_in, n, n, lay)
        opa = A if tr == "n" else A.T
        opb = B if tr == "n" else B.T
        prod = cs["alpha"] * (opa @ opa.T if fn == "syrk" else opa @ opb.T + opb @ opa.T)
        want = prod + cs["beta"] * C0
        mask = tri_mask(n, tri)
        tol = 8 * eps * max(k, 1) * (np.abs(prod) + np.abs(cs["beta"] * C0) + k / 2 + 1)
        ref = logical(ref_out, n, n, lay)
        assert np.all(np.abs(got - want)[mask] <= tol[mask])
        assert np.all(np.abs(got - ref)[mask] <= 2 * tol[mask])
        assert np.array_equal(got[~mask], C0[~mask])   # other triangle untouched
    else:
        m, n, side, tri, tr, dg = cs["m"], cs["n"], cs["side"], cs["tri"], cs["trans"], cs["diag"]
        na = m if side == "L" else n
        b = _buf(ctx, prec, b_in)
        args = (ctx, L[lay], SIDE[side], TRI[tri], TR[tr], DG[dg], m, n, cs["alpha"], _buf(ctx, prec, a_in), b)
        full = tri_full(logical(a_in, na, na, lay), tri, dg)
        op = full if tr == "n" else full.T
        B = logical(b_in, m, n, lay)
        if fn == "trmm":
            tb.trmm(*args)
            got = logical(tb.buffer_read(b, 0, m * n), m, n, lay)
            want = cs["alpha"] * (op @ B if side == "L" else B @ op)
            tol = 4 * eps * max(na, 1) * (np.abs(want) + abs(cs["alpha"]) * na + 4)
            assert np.all(np.abs(got - want) <= tol)
            assert np.all(np.abs(got - logical(ref_out, m, n, lay)) <= 2 * tol)
        else:
            tb.trsm(*args, block_size=cs["block_size"])
            x = logical(tb.buffer_read(b, 0, m * n), m, n, lay)
            lhs = op @ x if side == "L" else x @ op
            rhs = cs["alpha"] * B
            limit = 8 * eps * max(na, 1) * max(np.abs(rhs).max(), np.abs(x).max(), 1e-3)
            assert np.abs(lhs - rhs).max() <= limit, "trsm residual too large"
            xr = logical(ref_out, m, n, lay)
            assert np.abs(x - xr).max() <= 2 * limit * max(1.0, np.abs(xr).max())


def test_trsm_singular_raises(ctx):
    a = _buf(ctx, Precision.S, np.array([[2.0, 1.0], [0.0, 0.0]], np.float32).ravel(order="F"))
    b = _buf(ctx, Precision.S, np.ones(4, np.float32))
    with pytest.raises(tb.SingularMatrixError) as info:
        tb.trsm(ctx, Layout.COL_MAJOR, Side.LEFT, Triangle.UPPER, Transpose.NO, Diagonal.NON_UNIT, 2, 2, 1.0, a, b)
    assert info.value.index == 1


@pytest.mark.parametrize("prec", ["S", "H"])
def test_structured_large_on_tensor_and_ffma_paths(ctx, prec):
    """Larger sizes route through the tcgen05 / 128x256 kernels."""
    rng = np.random.default_rng(3)
    n, k = 640, 384
    dt = np.float16 if prec == "H" else np.float32
    A = rng.uniform(-1, 1, (n, k)).astype(dt)
    C0 = rng.uniform(-1, 1, (n, n)).astype(dt)
    a = _buf(ctx, P[prec], A.ravel(order="F"))
    c = _buf(ctx, P[prec], C0.ravel(order="F"))
    tb.syrk(ctx, Layout.COL_MAJOR, Triangle.LOWER, Transpose.NO, n, k, 0.75, a, -0.5, c)
    got = tb.buffer_read(c, 0, n * n).reshape(n, n).T.astype(np.float64)
    Af, Cf = A.astype(np.float64), C0.astype(np.float64)
    want = 0.75 * Af @ Af.T - 0.5 * Cf
    mask = tri_mask(n, "L")
    tol = 8 * EPS[prec] * k * (np.abs(0.75 * Af @ Af.T) + np.abs(0.5 * Cf) + k / 2 + 1)
    assert np.all(np.abs(got - want)[mask] <= tol[mask])
    assert np.array_equal(got[~mask], Cf[~mask])
