"""GPU parity of ``gemm`` (sm_100a kernels through the C-ABI).

Bars:
* against the reference's own outputs (tests/golden): within 2x the
  reference tolerance 4*eps*K*max|a||b| (test_level3.py:84-85);
* SGEMM against the C sequential-k oracle: BITWISE (the kernels' contract);
* HGEMM against the float64 product: within the K-scaled FP16 tolerance;
* no writes outside the declared C range (test_level3.py:141-159).
"""

import re

import numpy as np
import pytest

import paper_1705_05249_b200 as tb
from paper_1705_05249_b200 import Layout, Precision, Transpose
from conftest import load_golden, make_buffer, rand_array, read_mat
from oracle import gemm_oracle as orc

pytestmark = pytest.mark.gpu

P = {"S": Precision.S, "H": Precision.H}
L = {"col": Layout.COL_MAJOR, "row": Layout.ROW_MAJOR}
T = {"n": Transpose.NO, "t": Transpose.YES}
CASES, ARR = load_golden()


def flat_buffer(ctx, arr, prec):
    buf = tb.buffer_alloc(ctx, prec, arr.size)
    tb.buffer_write(buf, 0, arr)
    return buf


def run_case_gpu(ctx, case, i):
    prec = P[case["prec"]]
    a = flat_buffer(ctx, ARR[f"c{i}_a"], prec)
    b = flat_buffer(ctx, ARR[f"c{i}_b"], prec)
    c = flat_buffer(ctx, ARR[f"c{i}_c_in"], prec)
    tb.gemm(ctx, L[case["layout"]], T[case["ta"]], T[case["tb"]], case["m"], case["n"], case["k"],
            case["alpha"], a, b, case["beta"], c, a_offset=case["a_off"], lda=case["lda"],
            b_offset=case["b_off"], ldb=case["ldb"], c_offset=case["c_off"], ldc=case["ldc"],
            kernel=case["kernel"])
    return tb.buffer_read(c, 0, c.length)


def case_ops(case, i):
    row = case["layout"] == "row"
    m, n, k = case["m"], case["n"], case["k"]
    ta, tbn = case["ta"] == "t", case["tb"] == "t"
    a_rows, a_cols = (k, m) if ta else (m, k)
    b_rows, b_cols = (n, k) if tbn else (k, n)
    lda = case["lda"] or (a_cols if row else a_rows)
    ldb = case["ldb"] or (b_cols if row else b_rows)
    ldc = case["ldc"] or (n if row else m)
    av = orc.logical(ARR[f"c{i}_a"], case["a_off"], a_rows, a_cols, lda, row)
    bv = orc.logical(ARR[f"c{i}_b"], case["b_off"], b_rows, b_cols, ldb, row)
    return (av.T if ta else av), (bv.T if tbn else bv), lda, ldb, ldc


def full_tol(prec, alpha, beta, a_op, b_op, c_in):
    tol = abs(alpha) * orc.gemm_tolerance(a_op, b_op, prec)
    if beta != 0:
        tol = tol + 4 * orc.EPS[prec] * np.abs(beta * c_in.astype(np.float64))
    if prec == "H":
        tol = tol + 2.0 ** -11 * np.abs(orc.wide_oracle(alpha, a_op, b_op, beta, c_in)) + 2.0 ** -24
    return tol + 1e-30


GEMM_CASES = [(i, c) for i, c in enumerate(CASES) if c["kind"] == "gemm"]


@pytest.mark.parametrize("i,case", GEMM_CASES, ids=[f"g{i}" for i, _ in GEMM_CASES])
def test_golden_parity(ctx, i, case):
    got = run_case_gpu(ctx, case, i)
    gold = ARR[f"c{i}_c_out"]
    row = case["layout"] == "row"
    a_op, b_op, lda, ldb, ldc = case_ops(case, i)
    view = lambda flat: orc.logical(flat, case["c_off"], case["m"], case["n"], ldc, row)  # noqa: E731
    # canary: everything outside the declared C range is untouched
    mask = np.ones(got.shape, bool)
    view(mask)[...] = False
    assert np.array_equal(got[mask], ARR[f"c{i}_c_in"][mask], equal_nan=True)
    if case["k"] == 0 or case["alpha"] == 0:
        assert np.array_equal(got, gold, equal_nan=True)       # no summation: exact
        return
    c_in = view(ARR[f"c{i}_c_in"])
    tol = full_tol(case["prec"], case["alpha"], case["beta"], a_op, b_op, c_in)
    assert orc.allclose_tol(view(got), view(gold), tol, scale=2.0), "vs reference output"
    want = orc.wide_oracle(case["alpha"], a_op, b_op, case["beta"], c_in)
    assert orc.allclose_tol(view(got), want, tol), "vs float64 oracle"
    if case["prec"] == "S":
        seq = ARR[f"c{i}_c_in"].copy()
        orc.seqk_gemm("S", row, case["ta"] == "t", case["tb"] == "t", case["m"], case["n"],
                      case["k"], case["alpha"], ARR[f"c{i}_a"], case["a_off"], lda,
                      ARR[f"c{i}_b"], case["b_off"], ldb, case["beta"], seq, case["c_off"], ldc)
        assert got.tobytes() == seq.tobytes(), "SGEMM must equal the sequential-k oracle bitwise"


SHAPES = [(64, 48, 40), (256, 384, 320), (129, 130, 131), (300, 520, 200), (1, 1, 1), (7, 300, 2)]


@pytest.mark.parametrize("prec", ["S", "H"])
@pytest.mark.parametrize("layout", ["col", "row"])
@pytest.mark.parametrize("ta", ["n", "t"])
@pytest.mark.parametrize("tbn", ["n", "t"])
@pytest.mark.parametrize("shape", SHAPES, ids=[f"{m}x{n}x{k}" for m, n, k in SHAPES])
def test_layout_trans_matrix(ctx, prec, layout, ta, tbn, shape):
    m, n, k = shape
    precision = P[prec]
    rng = np.random.default_rng(hash((prec, layout, ta, tbn, shape)) % 2 ** 31)
    a_shape = (m, k) if ta == "n" else (k, m)
    b_shape = (k, n) if tbn == "n" else (n, k)
    av, bv, cv = rand_array(rng, a_shape, precision), rand_array(rng, b_shape, precision), \
        rand_array(rng, (m, n), precision)
    alpha, beta = 1.5, -0.5
    a = make_buffer(ctx, av, precision, L[layout])
    b = make_buffer(ctx, bv, precision, L[layout])
    c = make_buffer(ctx, cv, precision, L[layout])
    tb.gemm(ctx, L[layout], T[ta], T[tbn], m, n, k, alpha, a, b, beta, c)
    got = read_mat(c, (m, n), L[layout])
    a_op = av if ta == "n" else av.T
    b_op = bv if tbn == "n" else bv.T
    want = orc.wide_oracle(alpha, a_op, b_op, beta, cv)
    assert orc.allclose_tol(got, want, full_tol(prec, alpha, beta, a_op, b_op, cv))
    if prec == "S":
        order = "F" if layout == "col" else "C"
        af, bf = av.reshape(-1, order=order), bv.reshape(-1, order=order)
        cf = cv.reshape(-1, order=order).copy()
        lda = a_shape[0] if layout == "col" else a_shape[1]
        ldb = b_shape[0] if layout == "col" else b_shape[1]
        ldc = m if layout == "col" else n
        orc.seqk_gemm("S", layout == "row", ta == "t", tbn == "t", m, n, k, alpha, af, 0, lda,
                      bf, 0, ldb, beta, cf, 0, ldc)
        assert tb.buffer_read(c, 0, m * n).tobytes() == cf.tobytes()


@pytest.mark.parametrize("prec", ["S", "H"])
def test_direct_and_indirect_bitwise_equal(ctx, prec):
    """The reference allows 2x tol between its two routes (test_level3.py:68-85);
    here the bounds-checked producers and the TMA/vector ones agree bitwise."""
    precision = P[prec]
    for (m, n, k) in ((100, 100, 100), (256, 512, 192), (512, 256, 1024)):
        rng = np.random.default_rng(m + n + k)
        for ta in ("n", "t"):
            for tbn in ("n", "t"):
                av = rand_array(rng, (m, k) if ta == "n" else (k, m), precision)
                bv = rand_array(rng, (k, n) if tbn == "n" else (n, k), precision)
                a, b = make_buffer(ctx, av, precision), make_buffer(ctx, bv, precision)
                outs, kernels = [], []
                for kernel in ("direct", "indirect"):
                    c = tb.buffer_alloc(ctx, precision, m * n)
                    tb.gemm(ctx, Layout.COL_MAJOR, T[ta], T[tbn], m, n, k, 1.0, a, b, 0.0, c,
                            kernel=kernel)
                    outs.append(tb.buffer_read(c, 0, m * n))
                    kernels.append(ctx.last_launch.native["kernel"])
                ks = re.search(r"_splitk(\d+)", kernels[1])
                if ks is not None and prec == "S":
                    # the TMA route splits K (S split-K: sgemm_tma.cu sgemm_split_ks);
                    # each route then matches its own oracle bitwise
                    order = "F"
                    lda, ldb = av.shape[0], bv.shape[0]
                    for out, split in ((outs[0], None), (outs[1], int(ks.group(1)))):
                        want = np.zeros(m * n, np.float32)
                        args = ("S", False, ta == "t", tbn == "t", m, n, k, 1.0, av.reshape(-1, order=order), 0,
                                lda, bv.reshape(-1, order=order), 0, ldb, 0.0, want, 0, m)
                        if split is None:
                            orc.seqk_gemm(*args)
                        else:
                            orc.seqk_gemm_split(*args, split)
                        assert out.tobytes() == want.tobytes(), kernels
                    continue
                assert outs[0].tobytes() == outs[1].tobytes(), kernels
                if prec == "H" and m % 8 == 0 and k % 8 == 0 and n % 8 == 0:
                    assert "ldg" in kernels[0] and "tma" in kernels[1], kernels


def test_identity_exact(ctx):
    rng = np.random.default_rng(60)
    for prec in (Precision.S, Precision.H):
        for n in (16, 256):
            eye = make_buffer(ctx, np.eye(n), prec)
            bv = rand_array(rng, (n, n), prec)
            c = tb.buffer_alloc(ctx, prec, n * n)
            tb.gemm(ctx, Layout.COL_MAJOR, Transpose.NO, Transpose.NO, n, n, n, 1.0, eye,
                    make_buffer(ctx, bv, prec), 0.0, c)
            assert np.array_equal(read_mat(c, (n, n)), bv)


def test_beta_zero_overwrites_nan_and_alpha_zero_skips_ab(ctx):
    for prec in (Precision.S, Precision.H):
        n = 64
        a = make_buffer(ctx, np.full((n, n), np.nan), prec)   # never read when alpha == 0
        b = make_buffer(ctx, np.ones((n, n)), prec)
        c = make_buffer(ctx, np.full((n, n), np.nan), prec)
        tb.gemm(ctx, Layout.COL_MAJOR, Transpose.NO, Transpose.NO, n, n, n, 0.0, a, b, 0.0, c)
        assert np.all(read_mat(c, (n, n)) == 0)
        c2 = make_buffer(ctx, np.full((n, n), 2.0), prec)
        tb.gemm(ctx, Layout.COL_MAJOR, Transpose.NO, Transpose.NO, n, n, n, 0.0, a, b, 0.5, c2)
        assert np.all(read_mat(c2, (n, n)) == 1.0)
        eye = make_buffer(ctx, np.eye(n), prec)
        c3 = make_buffer(ctx, np.full((n, n), np.nan), prec)
        tb.gemm(ctx, Layout.COL_MAJOR, Transpose.NO, Transpose.NO, n, n, n, 1.0, eye, b, 0.0, c3)
        assert np.all(np.isfinite(read_mat(c3, (n, n))))
        c4 = make_buffer(ctx, np.full((n, n), 3.0), prec)
        tb.gemm(ctx, Layout.COL_MAJOR, Transpose.NO, Transpose.NO, n, n, 0, 1.0, a, b, 2.0, c4)
        assert np.all(read_mat(c4, (n, n)) == 6.0)


def test_canary_regions(ctx):
    rng = np.random.default_rng(65)
    for prec in (Precision.S, Precision.H):
        m, n, k, ldc = 6, 5, 4, 9
        av, bv = rand_array(rng, (m, k), prec), rand_array(rng, (k, n), prec)
        canary = -777.0
        c = tb.buffer_alloc(ctx, prec, 2 + ldc * n + 3)
        tb.buffer_write(c, 0, np.full(c.length, canary))
        tb.gemm(ctx, Layout.COL_MAJOR, Transpose.NO, Transpose.NO, m, n, k, 1.0,
                make_buffer(ctx, av, prec), make_buffer(ctx, bv, prec), 0.0, c, c_offset=2, ldc=ldc)
        data = tb.buffer_read(c, 0, c.length)
        for j in range(n):
            data[2 + j * ldc: 2 + j * ldc + m] = canary
        assert np.all(data == np.float32(canary).astype(prec.dtype))


def test_routing_family_and_launch_record(ctx):
    rng = np.random.default_rng(62)
    for size, family in ((32, "gemm_direct"), (200, "gemm")):
        a = make_buffer(ctx, rand_array(rng, (size, size), Precision.S), Precision.S)
        b = make_buffer(ctx, rand_array(rng, (size, size), Precision.S), Precision.S)
        c = tb.buffer_alloc(ctx, Precision.S, size * size)
        tb.gemm(ctx, Layout.COL_MAJOR, Transpose.NO, Transpose.NO, size, size, size, 1.0, a, b, 0.0, c)
        rec = ctx.last_launch
        assert rec.family == family
        assert rec.native["launches"] == 1 and rec.native["kernel"].startswith("sgemm_")


def test_override_is_recorded_and_applied(ctx):
    store = tb.routines.common.get_store(ctx)
    override = tb.GemmParams(MWG=32, NWG=32, KWG=16, MDIMC=8, NDIMC=8, MDIMA=8, NDIMB=8,
                             KWI=8).to_config()
    tb.override_parameters(store, "gemm", Precision.S, ctx.device, (40, 40, 40), override)
    a = tb.buffer_alloc(ctx, Precision.S, 1600)
    tb.gemm(ctx, Layout.COL_MAJOR, Transpose.NO, Transpose.NO, 40, 40, 40, 1.0, a, a, 0.0,
            tb.buffer_alloc(ctx, Precision.S, 1600))
    assert ctx.last_launch.params == override.as_dict()
    a2 = tb.buffer_alloc(ctx, Precision.S, 48 * 48)
    tb.gemm(ctx, Layout.COL_MAJOR, Transpose.NO, Transpose.NO, 48, 48, 48, 1.0, a2, a2, 0.0,
            tb.buffer_alloc(ctx, Precision.S, 48 * 48))
    assert ctx.last_launch.params != override.as_dict()
    store.clear_overrides()


def test_parameter_robustness(ctx):
    """200 random valid configurations on 96x80x64 (test_acceptance.py:62-97):
    every one recorded verbatim; SGEMM results bitwise identical across all."""
    import random

    from paper_1705_05249_b200.kernels import random_configuration, validate_gemm_params

    m, n, k = 96, 80, 64
    rng = np.random.default_rng(2024)
    av = rng.uniform(-1, 1, (m, k)).astype(np.float32)
    bv = rng.uniform(-1, 1, (k, n)).astype(np.float32)
    tol = orc.gemm_tolerance(av, bv, "S")
    want = orc.wide_oracle(1.0, av, bv, 0.0, None)
    sampler = random.Random(77)
    store = tb.routines.common.get_store(ctx)
    a, b = make_buffer(ctx, av, Precision.S), make_buffer(ctx, bv, Precision.S)
    first = None
    count = 0
    while count < 200:
        cfg = random_configuration("gemm", sampler)
        if not validate_gemm_params(cfg, ctx.device, Precision.S):
            continue
        count += 1
        store.set_override("gemm", Precision.S, ctx.device, (m, n, k), cfg)
        c = tb.buffer_alloc(ctx, Precision.S, m * n)
        tb.gemm(ctx, Layout.COL_MAJOR, Transpose.NO, Transpose.NO, m, n, k, 1.0, a, b, 0.0, c,
                kernel="indirect")
        assert ctx.last_launch.params == cfg.as_dict()
        got = tb.buffer_read(c, 0, m * n)
        assert orc.allclose_tol(got.reshape(n, m).T, want, tol)
        first = got if first is None else first
        assert got.tobytes() == first.tobytes()
    store.clear_overrides()


def test_repeat_determinism(ctx):
    rng = np.random.default_rng(6)
    for prec in (Precision.S, Precision.H):
        n = 512
        a = make_buffer(ctx, rand_array(rng, (n, n), prec), prec)
        b = make_buffer(ctx, rand_array(rng, (n, n), prec), prec)
        outs = []
        for _ in range(3):
            c = tb.buffer_alloc(ctx, prec, n * n)
            tb.gemm(ctx, Layout.ROW_MAJOR, Transpose.NO, Transpose.YES, n, n, n, 1.0, a, b, 0.0, c)
            outs.append(tb.buffer_read(c, 0, n * n).tobytes())
        assert outs[0] == outs[1] == outs[2]


@pytest.mark.parametrize("prec", ["S", "H"])
def test_large_sampled_parity(ctx, prec):
    """4096^3 row-major NN: sampled rows/cols vs the C oracle (bitwise for S)
    and the float64 product (tolerance) — the full-size property test."""
    import torch

    precision = P[prec]
    N = 4096
    g = torch.Generator(device="cuda").manual_seed(7)
    at = (torch.rand(N * N, device="cuda", generator=g) * 2 - 1).to(precision.torch_dtype)
    bt = (torch.rand(N * N, device="cuda", generator=g) * 2 - 1).to(precision.torch_dtype)
    a = tb.buffer_from_tensor(ctx, precision, at)
    b = tb.buffer_from_tensor(ctx, precision, bt)
    c = tb.buffer_alloc(ctx, precision, N * N)
    tb.gemm(ctx, Layout.ROW_MAJOR, Transpose.NO, Transpose.NO, N, N, N, 1.0, a, b, 0.0, c)
    rows = np.sort(np.random.default_rng(1).choice(N, 24, replace=False))
    cols = np.sort(np.random.default_rng(2).choice(N, 24, replace=False))
    A = at.view(N, N)[torch.from_numpy(rows).cuda()].cpu().numpy()
    B = bt.view(N, N)[:, torch.from_numpy(cols).cuda()].cpu().numpy()
    C = c.device_tensor().view(N, N)[torch.from_numpy(rows).cuda()][:, torch.from_numpy(cols).cuda()]
    got = C.cpu().numpy()
    want = orc.wide_oracle(1.0, A, B, 0.0, None)
    assert orc.allclose_tol(got, want, full_tol(prec, 1.0, 0.0, A, B, None))
    if prec == "S":
        sub = np.zeros(len(rows) * len(cols), np.float32)
        Ar, Br = np.ascontiguousarray(A).reshape(-1), np.ascontiguousarray(B).reshape(-1)
        orc.seqk_gemm("S", True, False, False, len(rows), len(cols), N, 1.0, Ar, 0, N, Br, 0,
                      len(cols), 0.0, sub, 0, len(cols))
        assert sub.reshape(len(rows), len(cols)).tobytes() == np.ascontiguousarray(got).tobytes()


@pytest.mark.parametrize("layout", ["col", "row"])
@pytest.mark.parametrize("ta", ["n", "t"])
@pytest.mark.parametrize("tbn", ["n", "t"])
def test_cta_pair_kernel_bitwise_equals_single_cta(ctx, layout, ta, tbn):
    """The 2-SM (tcgen05 cta_group::2) kernel — with and without its wave
    barrier — agrees bitwise with the single-CTA kernel, and all with the
    float64 product within tolerance."""
    import torch

    from paper_1705_05249_b200.kernels import native
    from paper_1705_05249_b200.kernels.dispatch import gemm_native

    m, n, k = 4096, 4352, 576
    prec = Precision.H
    g = torch.Generator(device="cuda").manual_seed(3)
    at = (torch.rand(m * k, device="cuda", generator=g) * 2 - 1).half()
    bt = (torch.rand(k * n, device="cuda", generator=g) * 2 - 1).half()
    a, b = tb.buffer_from_tensor(ctx, prec, at), tb.buffer_from_tensor(ctx, prec, bt)
    a_rows, a_cols = (m, k) if ta == "n" else (k, m)
    b_rows, b_cols = (k, n) if tbn == "n" else (n, k)
    lda = a_rows if layout == "col" else a_cols
    ldb = b_rows if layout == "col" else b_cols
    ldc = m if layout == "col" else n
    cfg = None  # built-in shape routing (gemm_b200 configurations select kernels)
    outs, kernels = [], []
    for flags in (0, native.FLAG_NO_2SM, native.FLAG_WAVE_SYNC):
        c = tb.buffer_alloc(ctx, prec, m * n)
        rec = gemm_native(ctx, prec, L[layout], T[ta], T[tbn], m, n, k, 1.0, a, 0, lda, b, 0, ldb, 0.0,
                          c, 0, ldc, cfg, flags)
        outs.append(c.device_tensor().clone())
        kernels.append(rec["kernel"])
    assert "2sm" in kernels[0] and "2sm" not in kernels[1] and "2sm" in kernels[2], kernels
    assert torch.equal(outs[0], outs[1]) and torch.equal(outs[0], outs[2]), kernels
    # sampled rows against the float64 product
    A = at.view(a_rows, a_cols).double() if layout == "row" else at.view(a_cols, a_rows).t().double()
    B = bt.view(b_rows, b_cols).double() if layout == "row" else bt.view(b_cols, b_rows).t().double()
    A = A if ta == "n" else A.t()
    B = B if tbn == "n" else B.t()
    rows = torch.arange(0, m, 257, device="cuda")
    want = A[rows] @ B
    C = outs[0].view(m, n) if layout == "row" else outs[0].view(n, m).t()
    tol = 4 * 2.0 ** -10 * k * A[rows].abs().amax(1, keepdim=True) * B.abs().amax(0, keepdim=True) \
        + 2.0 ** -11 * want.abs()
    assert bool(((C[rows].double() - want).abs() <= tol).all())


@pytest.mark.parametrize("ta,tbn", [("n", "n"), ("t", "t")])
@pytest.mark.parametrize("alpha,beta,ldc_pad", [(1.0, 0.0, 0), (0.75, 0.0, 0), (0.75, 0.5, 0), (1.0, 0.0, 3)])
def test_pair_256x512_epilogues_bitwise(ctx, ta, tbn, alpha, beta, ldc_pad):
    """The 256 x 512 CTA-pair tile (gemm_b200 NWG = 512, CTA_GROUP = 2) gives
    its single accumulator back before storing full beta == 0 tiles
    (hgemm_tc_2sm.cuh epi_store_early_release); partial tiles, beta != 0 and
    unaligned ldc take the per-block epilogue.  Every case equals the
    256 x 256 pair tile bitwise (same K16 sequence, same rounding)."""
    import torch

    from paper_1705_05249_b200.kernels.dispatch import gemm_native

    m, n, k = 1100, 1300, 320          # ragged in both dimensions: full and partial tiles
    prec = Precision.H
    g = torch.Generator(device="cuda").manual_seed(11)
    at = (torch.rand(m * k, device="cuda", generator=g) * 2 - 1).half()
    bt = (torch.rand(k * n, device="cuda", generator=g) * 2 - 1).half()
    c0 = (torch.rand(m * (n + ldc_pad), device="cuda", generator=g) * 2 - 1).half()
    a, b = tb.buffer_from_tensor(ctx, prec, at), tb.buffer_from_tensor(ctx, prec, bt)
    lda = k if ta == "n" else m
    ldb = n if tbn == "n" else k
    ldc = n + ldc_pad
    outs, kernels = [], []
    for nwg in (256, 512):
        cfg = tb.Configuration.make("gemm_b200", dict(zip(
            ("MWG", "NWG", "KWG", "STAGES", "CTA_GROUP", "SPLIT_K", "GROUP_M"), (256, nwg, 64, 0, 2, 1, 8))))
        c = tb.buffer_from_tensor(ctx, prec, c0.clone())
        rec = gemm_native(ctx, prec, Layout.ROW_MAJOR, T[ta], T[tbn], m, n, k, alpha, a, 0, lda, b, 0, ldb, beta,
                          c, 0, ldc, cfg, 0)
        outs.append(c.device_tensor().clone())
        kernels.append(rec["kernel"])
    assert "256x256" in kernels[0] and "256x512" in kernels[1], kernels
    assert torch.equal(outs[0], outs[1]), kernels
    A = at.view(m, k).double() if ta == "n" else at.view(k, m).t().double()
    B = bt.view(k, n).double() if tbn == "n" else bt.view(n, k).t().double()
    want = alpha * (A @ B) + beta * c0.view(m, ldc)[:, :n].double()
    got = outs[1].view(m, ldc)[:, :n].double()
    tol = 4 * 2.0 ** -10 * k * A.abs().amax(1, keepdim=True) * B.abs().amax(0, keepdim=True) \
        + 2.0 ** -10 * want.abs() + 2.0 ** -10
    assert bool(((got - want).abs() <= tol).all())
    if ldc_pad:
        assert torch.equal(outs[1].view(m, ldc)[:, n:], c0.view(m, ldc)[:, n:])


@pytest.mark.parametrize("layout", ["row", "col"])
@pytest.mark.parametrize("ta,tbn", [("n", "n"), ("t", "n"), ("n", "t"), ("t", "t")])
def test_unaligned_h_repacked_equals_ldg_path(ctx, layout, ta, tbn):
    """H operands with leading dimensions that are not a multiple of 8 are
    copied once into 16-byte aligned scratch and run on the TMA kernels
    (hgemm.cu hgemm_repacked, kernel name "+pack"); the values are the
    operands exactly, so the result equals the LDG-producer path bitwise."""
    from paper_1705_05249_b200.kernels import native
    from paper_1705_05249_b200.kernels.dispatch import gemm_native

    m, n, k = 700, 520, 333
    prec = Precision.H
    L = Layout.ROW_MAJOR if layout == "row" else Layout.COL_MAJOR
    rng = np.random.default_rng(m + n + k + len(layout) + ord(ta) + ord(tbn))
    ar, ac = (k, m) if ta == "t" else (m, k)
    br, bc = (n, k) if tbn == "t" else (k, n)
    lda = (ac if layout == "row" else ar) + 3
    ldb = (bc if layout == "row" else br) + 5
    ldc = (n if layout == "row" else m) + 1
    span = lambda r, c, ld: (r - 1) * ld + c if layout == "row" else (c - 1) * ld + r  # noqa: E731
    a = make_buffer(ctx, rng.uniform(-1, 1, span(ar, ac, lda) + 1).astype(np.float16), prec)
    b = make_buffer(ctx, rng.uniform(-1, 1, span(br, bc, ldb) + 3).astype(np.float16), prec)
    outs, kernels = [], []
    for flags in (0, native.FLAG_NO_TMA):
        c = tb.buffer_alloc(ctx, prec, span(m, n, ldc))
        rec = gemm_native(ctx, prec, L, T[ta], T[tbn], m, n, k, 1.0, a, 1, lda, b, 3, ldb, 0.0, c, 0, ldc,
                          None, flags)
        outs.append(tb.buffer_read(c, 0, c.length))
        kernels.append(rec["kernel"])
    assert kernels[0].endswith("+pack") and "tma" in kernels[0], kernels
    assert "ldg" in kernels[1], kernels
    assert outs[0].tobytes() == outs[1].tobytes(), kernels
