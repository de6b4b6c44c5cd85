"""Seeded random sweep over the public ``gemm`` surface: shapes drawn to hit
every shape-routed kernel (small packed instances, single-CTA tcgen05, CTA
pair, cluster split-K, TMA-fed and register-staged FFMA2, S split-K),
random layouts, transpositions, offsets, padded leading dimensions (which
also exercise the unaligned / LDG routes), alpha and beta.  C lives inside
a larger buffer whose other elements must come back untouched.

S: bitwise against the sequential-k oracle (`oracle/gemm_seqk.c`), or
against the split oracle (`oracle.seqk_gemm_split`) when the launched kernel
is a split-K one.  H: within the reference tolerance (4·eps·k·max|a|·max|b|,
eps = 2^-10, plus the final FP16 rounding) against a float64 product of the
FP16 inputs (reference `tests/oracles.py:62-73`)."""

import re

import numpy as np
import pytest

import paper_1705_05249_b200 as tb
from paper_1705_05249_b200 import Layout, Precision, Transpose
from oracle import gemm_oracle as orc

pytestmark = pytest.mark.gpu


def _draw(rng, i):
    kind = i % 6
    if kind == 0:      # small: packed instances / direct kernels
        m, n, k = (int(x) for x in rng.integers(1, 80, 3))
    elif kind == 1:    # medium, ragged
        m, n, k = (int(x) for x in rng.integers(100, 700, 3))
    elif kind == 2:    # few tiles, long K: split-K routes
        m, n, k = int(rng.integers(100, 600)), int(rng.integers(60, 260)), int(rng.integers(2000, 5000))
    elif kind == 3:    # wide enough for the CTA pair (H) / 128x64 tiles (S)
        m, n, k = int(rng.integers(1200, 2400)), int(rng.integers(1200, 2400)), int(rng.integers(64, 200))
    elif kind == 4:    # tall-skinny
        m, n, k = int(rng.integers(2000, 5000)), int(rng.integers(1, 40)), int(rng.integers(10, 300))
    else:              # mid-size, longer K (S split-K)
        m, n, k = int(rng.integers(300, 700)), int(rng.integers(300, 700)), int(rng.integers(1000, 2500))
    prec = "H" if rng.random() < 0.5 else "S"
    layout = Layout.ROW_MAJOR if rng.random() < 0.5 else Layout.COL_MAJOR
    ta, tbn = bool(rng.random() < 0.4), bool(rng.random() < 0.4)
    # aligned: leading dimensions rounded up to 8 elements and offsets in
    # 8-element steps (the TMA / vector routes); else ragged (LDG / general)
    aligned = rng.random() < 0.7
    pad = (lambda: -8) if aligned else (lambda: int(rng.integers(1, 6)))
    off = (lambda: 8 * int(rng.integers(0, 3))) if aligned else (lambda: int(rng.integers(1, 8)))
    alpha = float(rng.choice([1.0, -0.5, 0.75]))
    beta = float(rng.choice([0.0, 0.0, 0.5]))
    return dict(prec=prec, layout=layout, ta=ta, tb=tbn, m=m, n=n, k=k, pad=(pad(), pad(), pad()),
                off=(off(), off(), off()), alpha=alpha, beta=beta)


RNG = np.random.default_rng(20261019)
CASES = [_draw(RNG, i) for i in range(60)]


def _ids(cs):
    return (f"{cs['prec']}{'r' if cs['layout'] is Layout.ROW_MAJOR else 'c'}{'t' if cs['ta'] else 'n'}"
            f"{'t' if cs['tb'] else 'n'}_{cs['m']}x{cs['n']}x{cs['k']}")


@pytest.mark.parametrize("cs", CASES, ids=[_ids(c) for c in CASES])
def test_random_route(ctx, cs):
    prec = Precision.H if cs["prec"] == "H" else Precision.S
    dt = orc.DTYPE[cs["prec"]]
    row = cs["layout"] is Layout.ROW_MAJOR
    m, n, k = cs["m"], cs["n"], cs["k"]
    ar, ac = (k, m) if cs["ta"] else (m, k)
    br, bc = (n, k) if cs["tb"] else (k, n)
    ld_of = lambda base, pad: -(-base // 8) * 8 if pad < 0 else base + pad  # noqa: E731
    lda = ld_of(ac if row else ar, cs["pad"][0])
    ldb = ld_of(bc if row else br, cs["pad"][1])
    ldc = ld_of(n if row else m, cs["pad"][2])
    oa, ob, oc = cs["off"]
    span = lambda rows, cols, ld: (rows - 1) * ld + cols if row else (cols - 1) * ld + rows  # noqa: E731
    rng = np.random.default_rng(m * 7919 + n * 104729 + k)
    a = rng.uniform(-1, 1, oa + span(ar, ac, lda) + 9).astype(dt)
    b = rng.uniform(-1, 1, ob + span(br, bc, ldb) + 9).astype(dt)
    c0 = rng.uniform(-1, 1, oc + span(m, n, ldc) + 9).astype(dt)
    bufs = []
    for arr in (a, b, c0):
        buf = tb.buffer_alloc(ctx, prec, arr.size)
        tb.buffer_write(buf, 0, arr)
        bufs.append(buf)
    T = {False: Transpose.NO, True: Transpose.YES}
    tb.gemm(ctx, cs["layout"], T[cs["ta"]], T[cs["tb"]], m, n, k, cs["alpha"], bufs[0], bufs[1], cs["beta"],
            bufs[2], a_offset=oa, lda=lda, b_offset=ob, ldb=ldb, c_offset=oc, ldc=ldc)
    kern = ctx.last_launch.native["kernel"] if ctx.last_launch.native else ""
    got = tb.buffer_read(bufs[2], 0, c0.size)
    if prec is Precision.S:
        want = c0.copy()
        mt = re.search(r"_splitk(\d+)", kern)
        if mt:
            orc.seqk_gemm_split("S", row, cs["ta"], cs["tb"], m, n, k, cs["alpha"], a, oa, lda, b, ob, ldb,
                                cs["beta"], want, oc, ldc, int(mt.group(1)))
        else:
            orc.seqk_gemm("S", row, cs["ta"], cs["tb"], m, n, k, cs["alpha"], a, oa, lda, b, ob, ldb,
                          cs["beta"], want, oc, ldc)
        assert got.tobytes() == want.tobytes(), kern
        return
    # H: untouched outside C, tolerance inside
    cview = orc.logical(got, oc, m, n, ldc, row).astype(np.float64)
    inside = np.zeros(c0.size, bool)
    orc.logical(inside, oc, m, n, ldc, row)[...] = True
    assert got[~inside].tobytes() == c0[~inside].tobytes(), kern
    A = orc.logical(a, oa, ar, ac, lda, row).astype(np.float64)
    B = orc.logical(b, ob, br, bc, ldb, row).astype(np.float64)
    A = A.T if cs["ta"] else A
    B = B.T if cs["tb"] else B
    C0 = orc.logical(c0, oc, m, n, ldc, row).astype(np.float64)
    want = cs["alpha"] * (A @ B) + cs["beta"] * C0
    eps = 2.0 ** -10
    tol = 4 * eps * k * abs(cs["alpha"]) * np.abs(A).max(1, keepdims=True) * np.abs(B).max(0, keepdims=True) \
        + 2.0 ** -10 * np.abs(want) + 1e-3 * abs(cs["beta"])
    assert np.all(np.abs(cview - want) <= tol), (kern, float(np.max(np.abs(cview - want) - tol)))
