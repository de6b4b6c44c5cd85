"""Pin the oracle at the BASELINE configurations (C1, C3, C4 prefixes).

tests/golden/baseline_golden.npz holds the REFERENCE's own outputs
(``tunedblas.gemm`` / ``gemm_strided_batched``, sequential backend, built-in
configuration) for operands regenerated here from seeds.  These CPU tests
check (1) that the operands regenerate to the bytes the reference saw,
(2) that the reference outputs sit within the reference tolerance of the
float64 product, and (3) that the oracle port (oracle/gemm_oracle.py)
reproduces them — so the GPU tests (tests/test_baseline_gpu.py) compare
against a pinned checker.
"""

import numpy as np
import pytest

from baseline_cases import case_operands, digest, instance_views, load, max_ratio, tolerance
from oracle import gemm_oracle as orc

CASES, GOLD = load()
IDS = [c["name"] for c in CASES]


@pytest.mark.parametrize("case", CASES, ids=IDS)
def test_operands_regenerate(case):
    a, b = case_operands(case)
    assert digest(a) == case["sha_a"] and digest(b) == case["sha_b"]
    assert digest(GOLD[case["name"]]) == case["sha_c"]


@pytest.mark.parametrize("case", CASES, ids=IDS)
def test_reference_output_within_tolerance(case):
    a, b = case_operands(case)
    worst = 0.0
    for av, bv, cv in instance_views(case, a, b, GOLD[case["name"]]):
        wide = av.astype(np.float64) @ bv.astype(np.float64)
        worst = max(worst, max_ratio(cv, wide, tolerance(case["prec"], av, bv, wide)))
    assert worst <= 1.0, worst


@pytest.mark.parametrize("case", CASES, ids=IDS)
def test_port_reproduces_reference(case):
    """The oracle port runs the reference's tiled algorithm: bitwise on this
    image (same NumPy/OpenBLAS), and within 2x tol as the portable bar."""
    a, b = case_operands(case)
    m, n, k, batch = case["m"], case["n"], case["k"], case["batch"]
    c = np.zeros(m * n * batch, a.dtype)
    if case["kind"] == "gemm":
        orc.port_gemm(case["prec"], True, False, False, m, n, k, 1.0, a, b, 0.0, c, pool=orc.make_pool())
    else:
        orc.port_gemm_strided_batched(case["prec"], True, False, False, m, n, k, 1.0, a, m * k, b, k * n,
                                      0.0, c, m * n, batch)
    gold = GOLD[case["name"]]
    if c.tobytes() == gold.tobytes():
        return
    for (av, bv, cv), (_, _, gv) in zip(instance_views(case, a, b, c), instance_views(case, a, b, gold)):
        wide = av.astype(np.float64) @ bv.astype(np.float64)
        assert max_ratio(cv, gv.astype(np.float64), tolerance(case["prec"], av, bv, wide)) <= 2.0
