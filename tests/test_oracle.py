"""Pin the CPU oracle (oracle/) to the reference's own outputs.

tests/golden/gemm_golden.npz was produced by running the reference
``tunedblas`` routines (tests/golden/make_golden.py).  Before any GPU result
is judged against the oracle, the oracle itself must reproduce those
vectors: the NumPy port within the reference tolerance (bitwise where the
arithmetic has no summation), the C sequential-k restatement within 2x the
tolerance (the reference's pairwise rule, test_level3.py:84-85).
"""

import numpy as np
import pytest

from conftest import load_golden
from oracle import gemm_oracle as orc

CASES, ARR = load_golden()


def _views(case, flat_c):
    """Logical (m, n) C from a flat buffer for a golden gemm case."""
    row = case["layout"] == "row"
    m, n = case["m"], case["n"]
    ldc = case.get("ldc") or (n if row else m)
    return orc.logical(flat_c, case.get("c_off", 0), m, n, ldc, row)


def _ops(case, i):
    row = case["layout"] == "row"
    m, n, k = case["m"], case["n"], case["k"]
    ta, tbn = case["ta"] == "t", case["tb"] == "t"
    a_rows, a_cols = (k, m) if ta else (m, k)
    b_rows, b_cols = (n, k) if tbn else (k, n)
    lda = case.get("lda") or (a_cols if row else a_rows)
    ldb = case.get("ldb") or (b_cols if row else b_rows)
    av = orc.logical(ARR[f"c{i}_a"], case.get("a_off", 0), a_rows, a_cols, lda, row)
    bv = orc.logical(ARR[f"c{i}_b"], case.get("b_off", 0), b_rows, b_cols, ldb, row)
    return (av.T if ta else av), (bv.T if tbn else bv)


def _tol(case, a_op, b_op, c_in_view):
    tol = abs(case["alpha"]) * orc.gemm_tolerance(a_op, b_op, case["prec"])
    if case["beta"] != 0:
        tol = tol + 4 * orc.EPS[case["prec"]] * np.abs(case["beta"] * c_in_view.astype(np.float64))
    if case["prec"] == "H":  # final FP16 rounding of the result
        tol = tol + 2.0 ** -11 * np.abs(orc.wide_oracle(case["alpha"], a_op, b_op, case["beta"],
                                                        c_in_view))
    return tol + 1e-30


GEMM_CASES = [(i, c) for i, c in enumerate(CASES) if c["kind"] == "gemm"]


@pytest.mark.parametrize("i,case", GEMM_CASES, ids=[f"g{i}" for i, _ in GEMM_CASES])
def test_golden_is_sane(i, case):
    """The reference output itself is within tolerance of the float64 product."""
    a_op, b_op = _ops(case, i)
    c_in = _views(case, ARR[f"c{i}_c_in"])
    got = _views(case, ARR[f"c{i}_c_out"])
    if case["k"] == 0 or case["alpha"] == 0:
        want = np.zeros_like(c_in) if case["beta"] == 0 else (
            np.float32(case["beta"]) * c_in.astype(np.float32)).astype(c_in.dtype)
        assert np.array_equal(got, want, equal_nan=True)
        return
    want = orc.wide_oracle(case["alpha"], a_op, b_op, case["beta"], c_in)
    assert orc.allclose_tol(got, want, _tol(case, a_op, b_op, c_in))


@pytest.mark.parametrize("i,case", GEMM_CASES, ids=[f"g{i}" for i, _ in GEMM_CASES])
def test_port_reproduces_reference(i, case):
    c = ARR[f"c{i}_c_in"].copy()
    orc.port_gemm(case["prec"], case["layout"] == "row", case["ta"] == "t", case["tb"] == "t",
                  case["m"], case["n"], case["k"], case["alpha"], ARR[f"c{i}_a"], ARR[f"c{i}_b"],
                  case["beta"], c, a_offset=case["a_off"], lda=case["lda"], b_offset=case["b_off"],
                  ldb=case["ldb"], c_offset=case["c_off"], ldc=case["ldc"], kernel=case["kernel"])
    gold = ARR[f"c{i}_c_out"]
    # untouched elements and the no-summation cases are exact
    if case["k"] == 0 or case["alpha"] == 0:
        assert np.array_equal(c, gold, equal_nan=True)
        return
    a_op, b_op = _ops(case, i)
    c_in = _views(case, ARR[f"c{i}_c_in"])
    assert orc.allclose_tol(_views(case, c), _views(case, gold), _tol(case, a_op, b_op, c_in))
    mask = np.ones(c.shape, bool)
    mask_view = _views(case, mask)
    mask_view[...] = False
    assert np.array_equal(c[mask], gold[mask], equal_nan=True)  # canary: nothing else written


@pytest.mark.parametrize("i,case", GEMM_CASES, ids=[f"g{i}" for i, _ in GEMM_CASES])
def test_c_oracle_matches_reference(i, case):
    c = ARR[f"c{i}_c_in"].copy()
    row = case["layout"] == "row"
    m, n, k = case["m"], case["n"], case["k"]
    ta, tbn = case["ta"] == "t", case["tb"] == "t"
    a_rows, a_cols = (k, m) if ta else (m, k)
    b_rows, b_cols = (n, k) if tbn else (k, n)
    lda = case["lda"] or (a_cols if row else a_rows)
    ldb = case["ldb"] or (b_cols if row else b_rows)
    ldc = case["ldc"] or (n if row else m)
    orc.seqk_gemm(case["prec"], row, ta, tbn, m, n, k, case["alpha"], ARR[f"c{i}_a"],
                  case["a_off"], lda, ARR[f"c{i}_b"], case["b_off"], ldb, case["beta"], c,
                  case["c_off"], ldc)
    gold = ARR[f"c{i}_c_out"]
    if k == 0 or case["alpha"] == 0:
        assert np.array_equal(c, gold, equal_nan=True)
        return
    a_op, b_op = _ops(case, i)
    c_in = _views(case, ARR[f"c{i}_c_in"])
    assert orc.allclose_tol(_views(case, c), _views(case, gold), _tol(case, a_op, b_op, c_in),
                            scale=2.0)
    mask = np.ones(c.shape, bool)
    _views(case, mask)[...] = False
    assert np.array_equal(c[mask], gold[mask], equal_nan=True)


BATCH_CASES = [(i, c) for i, c in enumerate(CASES) if c["kind"] in ("strided", "batched")]


@pytest.mark.parametrize("i,case", BATCH_CASES, ids=[f"b{i}" for i, _ in BATCH_CASES])
def test_batched_oracles_match_reference(i, case):
    m, n, k, batch = case["m"], case["n"], case["k"], case["batch"]
    row = case["layout"] == "row"
    gold = ARR[f"c{i}_c_out"]
    c_port = ARR[f"c{i}_c_in"].copy()
    c_seq = ARR[f"c{i}_c_in"].copy()
    if case["kind"] == "strided":
        orc.port_gemm_strided_batched(case["prec"], row, False, False, m, n, k, case["alpha"],
                                      ARR[f"c{i}_a"], case["stride_a"], ARR[f"c{i}_b"],
                                      case["stride_b"], case["beta"], c_port, case["stride_c"], batch)
        orc.seqk_gemm_strided_batched(case["prec"], row, False, False, m, n, k, case["alpha"],
                                      ARR[f"c{i}_a"], 0, (k if row else m), case["stride_a"],
                                      ARR[f"c{i}_b"], 0, (n if row else k), case["stride_b"],
                                      case["beta"], c_seq, 0, (n if row else m), case["stride_c"],
                                      batch)
        alphas = [case["alpha"]] * batch
        betas = [case["beta"]] * batch
        offs = [(z * case["stride_a"], z * case["stride_b"], z * case["stride_c"]) for z in range(batch)]
    else:
        alphas, betas = case["alphas"], case["betas"]
        offs = list(zip(case["a_offs"], case["b_offs"], case["c_offs"]))
        for z, (ao, bo, co) in enumerate(offs):
            orc.port_gemm(case["prec"], False, False, False, m, n, k, alphas[z], ARR[f"c{i}_a"],
                          ARR[f"c{i}_b"], betas[z], c_port, a_offset=ao, b_offset=bo, c_offset=co)
            orc.seqk_gemm(case["prec"], False, False, False, m, n, k, alphas[z], ARR[f"c{i}_a"], ao, m,
                          ARR[f"c{i}_b"], bo, k, betas[z], c_seq, co, m)
    for z, (ao, bo, co) in enumerate(offs):
        a_rows = b_rows = None  # noqa: F841
        a_op = orc.logical(ARR[f"c{i}_a"], ao, m, k, k if row else m, row)
        b_op = orc.logical(ARR[f"c{i}_b"], bo, k, n, n if row else k, row)
        c_in = orc.logical(ARR[f"c{i}_c_in"], co, m, n, n if row else m, row)
        cs = dict(alpha=alphas[z], beta=betas[z], prec=case["prec"])
        want = orc.logical(gold, co, m, n, n if row else m, row)
        for got_flat, scale in ((c_port, 1.0), (c_seq, 2.0)):
            got = orc.logical(got_flat, co, m, n, n if row else m, row)
            if alphas[z] == 0:
                assert np.array_equal(got, want)
            else:
                assert orc.allclose_tol(got, want, _tol(cs, a_op, b_op, c_in), scale=scale)


def test_half_conversion_exhaustive():
    """C oracle FP16 widening of all 65536 patterns matches IEEE (numpy)."""
    lib = orc.c_lib()
    bits = np.arange(1 << 16, dtype=np.uint16)
    ref = bits.view(np.float16).astype(np.float32)
    got = np.array([lib.oracle_h2f(int(h)) for h in bits], np.float32)
    finite = np.isfinite(ref)
    assert np.array_equal(got[finite], ref[finite])
    assert np.all(np.isnan(got[~finite]) == np.isnan(ref[~finite]))


def test_half_rounding_rne():
    """C oracle FP32->FP16 narrowing is round-to-nearest-even (numpy astype)."""
    lib = orc.c_lib()
    rng = np.random.default_rng(5)
    vals = np.concatenate([
        rng.uniform(-70000, 70000, 4000), rng.uniform(-1e-4, 1e-4, 4000),
        rng.standard_normal(4000), np.array([65504, 65519.99, 65520, 6.1e-5, 5.96e-8, 2.98e-8,
                                             -0.0, 0.0, 1 + 2 ** -11, 1 + 3 * 2 ** -11])]).astype(np.float32)
    want = vals.astype(np.float16).view(np.uint16)
    got = np.array([lib.oracle_f2h(float(v)) for v in vals], np.uint16)
    assert np.array_equal(got, want)


def test_known_answers():
    """Identity operand is exact; beta=0 overwrites NaN; zero sizes are no-ops
    (reference tests/test_level3.py:37-65)."""
    rng = np.random.default_rng(60)
    n = 16
    eye = np.eye(n, dtype=np.float32).reshape(-1, order="F")
    bv = rng.standard_normal((n, n)).astype(np.float32)
    c = np.full(n * n, np.nan, np.float32)
    orc.seqk_gemm("S", False, False, False, n, n, n, 1.0, eye, 0, n, bv.reshape(-1, order="F"), 0,
                  n, 0.0, c, 0, n)
    assert np.array_equal(c.reshape(n, n).T, bv)
    c0 = np.array([7.0], np.float32)
    orc.seqk_gemm("S", False, False, False, 0, 0, 0, 1.0, c0, 0, 1, c0, 0, 1, 0.0, c0, 0, 1)
    assert c0.tolist() == [7.0]


def test_seqk_split_oracle():
    """oracle.seqk_gemm_split: KS = 1 is the sequential-k chain bitwise; a
    split is the rank-order sum of the chains over the K ranges, within the
    reference tolerance of the float64 product."""
    rng = np.random.default_rng(9)
    m, n, k = 7, 9, 300
    a = rng.uniform(-1, 1, m * k).astype(np.float32)
    b = rng.uniform(-1, 1, k * n).astype(np.float32)
    one = np.zeros(m * n, np.float32)
    orc.seqk_gemm_split("S", True, False, False, m, n, k, 1.5, a, 0, k, b, 0, n, 0.0, one, 0, n, 1)
    seq = np.zeros(m * n, np.float32)
    orc.seqk_gemm("S", True, False, False, m, n, k, 1.5, a, 0, k, b, 0, n, 0.0, seq, 0, n)
    assert one.tobytes() == seq.tobytes()
    A, B = a.reshape(m, k), b.reshape(k, n)
    want = 1.5 * (A.astype(np.float64) @ B.astype(np.float64))
    for ks in (2, 4):
        got = np.zeros(m * n, np.float32)
        orc.seqk_gemm_split("S", True, False, False, m, n, k, 1.5, a, 0, k, b, 0, n, 0.0, got, 0, n, ks)
        # manual: chains over [0,160) / [160,300) for ks=2 (5 stages of 32 per rank)
        assert orc.allclose_tol(got.reshape(m, n), want, 1.5 * orc.gemm_tolerance(A, B, "S"))
    p0 = np.zeros(m * n, np.float32)
    p1 = np.zeros(m * n, np.float32)
    orc.seqk_gemm("S", True, False, False, m, n, 160, 1.0, a, 0, k, b, 0, n, 0.0, p0, 0, n)
    orc.seqk_gemm("S", True, False, False, m, n, 140, 1.0, a, 160, k, b, 160 * n, n, 0.0, p1, 0, n)
    two = np.zeros(m * n, np.float32)
    orc.seqk_gemm_split("S", True, False, False, m, n, k, 1.0, a, 0, k, b, 0, n, 0.0, two, 0, n, 2)
    assert two.tobytes() == (p0 + p1).astype(np.float32).tobytes()
