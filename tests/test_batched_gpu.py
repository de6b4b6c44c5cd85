"""GPU batched GEMM: one persistent launch per batch; bitwise equal to the
looped single calls (reference tests/test_extras.py:213-329,
routine_cases.py:837-880) and to the oracle."""

import numpy as np
import pytest

import paper_1705_05249_b200 as tb
from paper_1705_05249_b200 import Layout, Precision, Transpose
from conftest import load_golden, make_buffer, rand_array
from oracle import gemm_oracle as orc

pytestmark = pytest.mark.gpu
COL, NO = Layout.COL_MAJOR, Transpose.NO
CASES, ARR = load_golden()


def setup(ctx, rng, m, n, k, batch, prec):
    ea, eb, ec = m * k, k * n, m * n
    host = [rand_array(rng, batch * e, prec) for e in (ea, eb, ec)]
    bufs = [make_buffer(ctx, h, prec) for h in host]
    offs = ([i * ea for i in range(batch)], [i * eb for i in range(batch)],
            [i * ec for i in range(batch)])
    return host, bufs, offs


@pytest.mark.parametrize("prec", [Precision.S, Precision.H])
@pytest.mark.parametrize("shape,batch", [((32, 32, 32), 64), ((129, 129, 129), 2),
                                         ((64, 64, 64), 9), ((17, 13, 9), 5), ((256, 128, 64), 3)])
def test_batched_equals_loop_bitwise(ctx, prec, shape, batch):
    m, n, k = shape
    rng = np.random.default_rng(89 + m)
    alphas = [float(x) for x in rng.uniform(0.5, 2, batch)]
    betas = [float(x) for x in rng.uniform(-1, 1, batch)]
    host, (a, b, c), (ao, bo, co) = setup(ctx, rng, m, n, k, batch, prec)
    tb.gemm_batched(ctx, COL, NO, NO, m, n, k, alphas, a, ao, b, bo, betas, c, co, batch)
    got = tb.buffer_read(c, 0, c.length)
    assert ctx.last_launch.work_groups[0] == batch
    a2, b2, c2 = (make_buffer(ctx, h, prec) for h in host)
    for i in range(batch):
        tb.gemm(ctx, COL, NO, NO, m, n, k, alphas[i], a2, b2, betas[i], c2,
                a_offset=ao[i], b_offset=bo[i], c_offset=co[i])
    assert got.tobytes() == tb.buffer_read(c2, 0, c2.length).tobytes()


@pytest.mark.parametrize("prec", [Precision.S, Precision.H])
@pytest.mark.parametrize("layout", [Layout.COL_MAJOR, Layout.ROW_MAJOR])
def test_strided_equals_generic_and_loop(ctx, prec, layout):
    rng = np.random.default_rng(91)
    for (m, n, k), batch in (((16, 16, 16), 8), ((64, 48, 32), 6), ((128, 256, 64), 2)):
        ea, eb, ec = m * k, k * n, m * n
        host, (a, b, c), (ao, bo, co) = setup(ctx, rng, m, n, k, batch, prec)
        tb.gemm_strided_batched(ctx, layout, NO, Transpose.YES, m, n, k, 1.5, a, ea, b, eb,
                                0.5, c, ec, batch)
        got = tb.buffer_read(c, 0, c.length)
        a2, b2, c2 = (make_buffer(ctx, h, prec) for h in host)
        tb.gemm_batched(ctx, layout, NO, Transpose.YES, m, n, k, [1.5] * batch, a2, ao, b2, bo,
                        [0.5] * batch, c2, co, batch)
        assert got.tobytes() == tb.buffer_read(c2, 0, c2.length).tobytes()
        a3, b3, c3 = (make_buffer(ctx, h, prec) for h in host)
        for i in range(batch):
            tb.gemm(ctx, layout, NO, Transpose.YES, m, n, k, 1.5, a3, b3, 0.5, c3,
                    a_offset=ao[i], b_offset=bo[i], c_offset=co[i])
        assert got.tobytes() == tb.buffer_read(c3, 0, c3.length).tobytes()


def test_single_instance_equals_plain(ctx):
    rng = np.random.default_rng(93)
    for prec in (Precision.S, Precision.H):
        m = n = k = 12
        host, (a, b, c), _ = setup(ctx, rng, m, n, k, 1, prec)
        tb.gemm_strided_batched(ctx, COL, NO, NO, m, n, k, 1.0, a, m * k, b, k * n, 0.0, c, m * n, 1)
        a2, b2, c2 = (make_buffer(ctx, h, prec) for h in host)
        tb.gemm(ctx, COL, NO, NO, m, n, k, 1.0, a2, b2, 0.0, c2)
        assert tb.buffer_read(c, 0, c.length).tobytes() == tb.buffer_read(c2, 0, c2.length).tobytes()


def test_alpha_zero_instances_and_record(ctx):
    rng = np.random.default_rng(94)
    m = n = k = 16
    batch = 4
    host, (a, b, c), (ao, bo, co) = setup(ctx, rng, m, n, k, batch, Precision.S)
    tb.gemm_batched(ctx, COL, NO, NO, m, n, k, [1.0] * batch, a, ao, b, bo, [0.0] * batch, c, co,
                    batch)
    rec = ctx.last_launch
    assert rec.work_groups[0] == batch
    prev = tb.buffer_read(c, 0, c.length)
    # every instance alpha == 0: C = beta*C and the reference makes no launch
    # (extras.py:281-286), so last_launch is unchanged
    tb.gemm_batched(ctx, COL, NO, NO, m, n, k, [0.0] * batch, a, ao, b, bo, [2.0] * batch, c, co,
                    batch)
    assert ctx.last_launch is rec
    assert tb.buffer_read(c, 0, c.length).tobytes() == (np.float32(2.0) * prev).tobytes()
    # a mixed batch: alpha == 0 instances are scaled only, NaN in A never read
    a_nan = make_buffer(ctx, np.full(batch * m * k, np.nan, np.float32), Precision.S)
    c2 = make_buffer(ctx, np.ones(batch * m * n, np.float32), Precision.S)
    tb.gemm_batched(ctx, COL, NO, NO, m, n, k, [0.0, 0.0, 0.0, 0.0], a_nan, ao, b, bo,
                    [0.5, 0.0, 2.0, 1.0], c2, co, batch)
    out = tb.buffer_read(c2, 0, c2.length).reshape(batch, -1)
    assert np.all(out[0] == 0.5) and np.all(out[1] == 0) and np.all(out[2] == 2) and np.all(out[3] == 1)


@pytest.mark.parametrize("i,case", [(i, c) for i, c in enumerate(CASES)
                                    if c["kind"] in ("strided", "batched")],
                         ids=lambda v: str(v) if isinstance(v, int) else "")
def test_golden_batched_parity(ctx, i, case):
    prec = {"S": Precision.S, "H": Precision.H}[case["prec"]]
    m, n, k, batch = case["m"], case["n"], case["k"], case["batch"]
    row = case["layout"] == "row"
    layout = Layout.ROW_MAJOR if row else COL
    a = make_buffer(ctx, ARR[f"c{i}_a"], prec)
    b = make_buffer(ctx, ARR[f"c{i}_b"], prec)
    c = make_buffer(ctx, ARR[f"c{i}_c_in"], prec)
    if case["kind"] == "strided":
        tb.gemm_strided_batched(ctx, layout, NO, NO, m, n, k, case["alpha"], a, case["stride_a"],
                                b, case["stride_b"], case["beta"], c, case["stride_c"], batch)
        alphas, betas = [case["alpha"]] * batch, [case["beta"]] * batch
        offs = [(z * case["stride_a"], z * case["stride_b"], z * case["stride_c"]) for z in range(batch)]
    else:
        tb.gemm_batched(ctx, layout, NO, NO, m, n, k, case["alphas"], a, case["a_offs"], b,
                        case["b_offs"], case["betas"], c, case["c_offs"], batch)
        alphas, betas = case["alphas"], case["betas"]
        offs = list(zip(case["a_offs"], case["b_offs"], case["c_offs"]))
    got = tb.buffer_read(c, 0, c.length)
    gold = ARR[f"c{i}_c_out"]
    lda, ldb, ldc = (k, n, n) if row else (m, k, m)
    for z, (ao, bo, co) in enumerate(offs):
        A = orc.logical(ARR[f"c{i}_a"], ao, m, k, lda, row)
        B = orc.logical(ARR[f"c{i}_b"], bo, k, n, ldb, row)
        Cin = orc.logical(ARR[f"c{i}_c_in"], co, m, n, ldc, row)
        g = orc.logical(got, co, m, n, ldc, row)
        w = orc.logical(gold, co, m, n, ldc, row)
        if alphas[z] == 0:
            assert np.array_equal(g, w)
            continue
        tol = abs(alphas[z]) * orc.gemm_tolerance(A, B, case["prec"]) + \
            4 * orc.EPS[case["prec"]] * np.abs(betas[z] * Cin.astype(np.float64)) + 1e-30
        if case["prec"] == "H":
            tol = tol + 2.0 ** -11 * np.abs(w.astype(np.float64))
        assert orc.allclose_tol(g, w, tol, scale=2.0)


@pytest.mark.parametrize("prec", ["S", "H"])
@pytest.mark.parametrize("size", [32, 64])
def test_full_size_batch_16384(ctx, prec, size):
    """BASELINE config C4 at full size: sampled instances vs the C oracle
    (bitwise for S, tolerance for H)."""
    import torch

    precision = {"S": Precision.S, "H": Precision.H}[prec]
    batch, m = 16384, size
    e = m * m
    g = torch.Generator(device="cuda").manual_seed(11)
    at = (torch.rand(batch * e, device="cuda", generator=g) * 2 - 1).to(precision.torch_dtype)
    bt = (torch.rand(batch * e, device="cuda", generator=g) * 2 - 1).to(precision.torch_dtype)
    a, b = tb.buffer_from_tensor(ctx, precision, at), tb.buffer_from_tensor(ctx, precision, bt)
    c = tb.buffer_alloc(ctx, precision, batch * e)
    tb.gemm_strided_batched(ctx, Layout.ROW_MAJOR, NO, NO, m, m, m, 1.0, a, e, b, e, 0.0, c, e, batch)
    for z in (0, 1, 4097, 9999, batch - 1):
        A = at[z * e:(z + 1) * e].cpu().numpy()
        B = bt[z * e:(z + 1) * e].cpu().numpy()
        got = c.device_tensor()[z * e:(z + 1) * e].cpu().numpy()
        want = np.zeros(e, precision.dtype)
        orc.seqk_gemm(prec, True, False, False, m, m, m, 1.0, A, 0, m, B, 0, m, 0.0, want, 0, m)
        if prec == "S":
            assert got.tobytes() == want.tobytes()
        else:
            tol = orc.gemm_tolerance(A.reshape(m, m), B.reshape(m, m), "H").reshape(-1)
            assert orc.allclose_tol(got, want, tol, scale=2.0)


@pytest.mark.parametrize("prec", [Precision.S, Precision.H])
@pytest.mark.parametrize("layout", [Layout.COL_MAJOR, Layout.ROW_MAJOR])
@pytest.mark.parametrize("ta", [Transpose.NO, Transpose.YES])
@pytest.mark.parametrize("tbt", [Transpose.NO, Transpose.YES])
@pytest.mark.parametrize("shape", [(32, 32, 32), (64, 64, 64), (20, 50, 77), (64, 17, 300), (8, 64, 1),
                                   (48, 40, 64), (64, 32, 40)])
def test_small_path_bitwise_equals_general_path(ctx, prec, layout, ta, tbt, shape):
    """The small-instance kernels (packed tcgen05 for H, TMA-fed FFMA2 tiles
    for S) give the same bits as the general kernels forced via flags."""
    from paper_1705_05249_b200.kernels import native
    from paper_1705_05249_b200.kernels.dispatch import gemm_strided_batched_native

    m, n, k = shape
    batch = 37
    rng = np.random.default_rng(m * 7 + n + k)
    ea, eb, ec = m * k, k * n, m * n
    host = [rand_array(rng, batch * e, prec) for e in (ea, eb, ec)]
    lda = (m if ta is NO else k) if layout is COL else (k if ta is NO else m)
    ldb = (k if tbt is NO else n) if layout is COL else (n if tbt is NO else k)
    ldc = m if layout is COL else n
    outs, kernels = [], []
    general = native.FLAG_NO_PACK if prec is Precision.H else native.FLAG_SIMT_GENERAL
    for flags in (0, general):
        a, b, c = (make_buffer(ctx, h, prec) for h in host)
        rec = gemm_strided_batched_native(ctx, prec, layout, ta, tbt, m, n, k, 1.25, a, 0, lda, ea,
                                          b, 0, ldb, eb, -0.5, c, 0, ldc, ec, batch, None, flags)
        outs.append(tb.buffer_read(c, 0, c.length))
        kernels.append(rec["kernel"])
    assert "small" not in kernels[1], kernels
    aligned = (prec is Precision.S and all(v % 4 == 0 for v in (ea, eb, lda, ldb))) or \
        (prec is Precision.H and all(v % 8 == 0 for v in (ea, eb, lda, ldb)))
    if prec is Precision.H:
        assert "small" in kernels[0], kernels
        if aligned and max(m, n, k) <= 64:   # one TMA box per operand per tile (32- or 64-wide kernel)
            assert kernels[0].endswith("_tma"), kernels
    elif aligned and m <= 32 and n <= 32:
        # strided S batches of <= 32x32 instances: one TMA-fed 32x32 tile each
        assert kernels[0].startswith("sgemm_tma_32x32"), kernels
    assert outs[0].tobytes() == outs[1].tobytes(), kernels


def test_batched_beats_looped_launches_10x(ctx):
    """North star / acceptance criterion (test_acceptance.py:168-204 asks >= 1.2x
    on the host): one batched launch vs one gemm call per instance, >= 10x."""
    import time

    import torch

    rng = np.random.default_rng(3)
    s, batch = 32, 512
    e = s * s
    host, (a, b, c), _ = setup(ctx, rng, s, s, s, batch, Precision.S)
    c2 = tb.buffer_alloc(ctx, Precision.S, batch * e)

    def batched():
        tb.gemm_strided_batched(ctx, COL, NO, NO, s, s, s, 1.0, a, e, b, e, 0.0, c, e, batch)

    def looped():
        for i in range(batch):
            tb.gemm(ctx, COL, NO, NO, s, s, s, 1.0, a, b, 0.0, c2, a_offset=i * e, b_offset=i * e,
                    c_offset=i * e)

    def best(fn, reps=3):
        fn()
        torch.cuda.synchronize()
        out = float("inf")
        for _ in range(reps):
            t0 = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            out = min(out, time.perf_counter() - t0)
        return out

    speedup = best(looped) / best(batched)
    assert tb.buffer_read(c, 0, batch * e).tobytes() == tb.buffer_read(c2, 0, batch * e).tobytes()
    assert speedup >= 10.0, speedup
