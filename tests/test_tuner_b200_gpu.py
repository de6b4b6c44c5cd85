"""The B200-native tuning family ``gemm_b200`` (kernels/params.py;
include/tbgemm.h tb_gemm_config) on the GPU: every configuration selects the
kernel it names, results keep the bitwise contracts (S: every tile equals
the sequential-k oracle; H: single-CTA tiles, ring depths and the CTA pair
agree bitwise, split-K within tolerance), the tuner explores distinct
kernels with the built-in route as a candidate, and a tuned DB entry is
selected at call time for its exact shape only."""

import numpy as np
import pytest

import paper_1705_05249_b200 as tb
from paper_1705_05249_b200 import Layout, Precision, Transpose
from paper_1705_05249_b200.kernels.params import b200_variants, curated_b200, is_b200_auto
from paper_1705_05249_b200.tuner import TuningTask, tune
from conftest import make_buffer, rand_array
from oracle import gemm_oracle as orc

pytestmark = pytest.mark.gpu

NAMES = ("MWG", "NWG", "KWG", "STAGES", "CTA_GROUP", "SPLIT_K", "GROUP_M")


def cfg_of(v, group_m=0):
    return tb.Configuration.make("gemm_b200", dict(zip(NAMES, tuple(v) + (group_m,))))


def run_with(ctx, cfg, prec, layout, ta, tbn, m, n, k, a, b):
    store = tb.routines.common.get_store(ctx)
    store.clear_overrides()
    if cfg is not None:
        store.set_override("gemm_b200", prec, ctx.device, (m, n, k), cfg)
    c = tb.buffer_alloc(ctx, prec, m * n)
    tb.gemm(ctx, layout, ta, tbn, m, n, k, 1.0, a, b, 0.0, c)
    rec = ctx.last_launch
    store.clear_overrides()
    return tb.buffer_read(c, 0, m * n), rec


@pytest.mark.parametrize("layout", [Layout.COL_MAJOR, Layout.ROW_MAJOR])
@pytest.mark.parametrize("ta,tbn", [("n", "n"), ("t", "n"), ("n", "t"), ("t", "t")])
def test_sgemm_every_tile_equals_seqk(ctx, layout, ta, tbn):
    T = {"n": Transpose.NO, "t": Transpose.YES}
    m, n, k = 300, 520, 200
    prec = Precision.S
    rng = np.random.default_rng(41)
    av = rand_array(rng, (m, k) if ta == "n" else (k, m), prec)
    bv = rand_array(rng, (k, n) if tbn == "n" else (n, k), prec)
    a, b = make_buffer(ctx, av, prec, layout), make_buffer(ctx, bv, prec, layout)
    order = "F" if layout is Layout.COL_MAJOR else "C"
    seq = np.zeros(m * n, np.float32)
    lda = av.shape[0] if layout is Layout.COL_MAJOR else av.shape[1]
    ldb = bv.shape[0] if layout is Layout.COL_MAJOR else bv.shape[1]
    orc.seqk_gemm("S", layout is Layout.ROW_MAJOR, ta == "t", tbn == "t", m, n, k, 1.0,
                  av.reshape(-1, order=order), 0, lda, bv.reshape(-1, order=order), 0, ldb, 0.0,
                  seq, 0, m if layout is Layout.COL_MAJOR else n)
    kernels = set()
    for v in b200_variants(prec):
        got, rec = run_with(ctx, cfg_of(v, 4), prec, layout, T[ta], T[tbn], m, n, k, a, b)
        assert rec.kernel_config == cfg_of(v, 4).as_dict()
        kern = rec.native["kernel"]
        kernels.add(kern)
        if "splitk" in kern:   # the chain cut at the rank boundaries, partials summed in rank order
            assert v[5] > 1 and f"splitk{v[5]}" in kern, (v, kern)
            want = np.zeros(m * n, np.float32)
            orc.seqk_gemm_split("S", layout is Layout.ROW_MAJOR, ta == "t", tbn == "t", m, n, k, 1.0,
                                av.reshape(-1, order=order), 0, lda, bv.reshape(-1, order=order), 0, ldb, 0.0,
                                want, 0, m if layout is Layout.COL_MAJOR else n, v[5])
            assert got.tobytes() == want.tobytes(), (v, kern)
        else:
            assert got.tobytes() == seq.tobytes(), (v, kern)
    assert len(kernels) >= 8, kernels


def test_hgemm_configurations(ctx):
    import torch

    m, n, k = 1024, 768, 4096
    prec = Precision.H
    g = torch.Generator(device="cuda").manual_seed(5)
    at = (torch.rand(m * k, device="cuda", generator=g) * 2 - 1).half()
    bt = (torch.rand(k * n, device="cuda", generator=g) * 2 - 1).half()
    a, b = tb.buffer_from_tensor(ctx, prec, at), tb.buffer_from_tensor(ctx, prec, bt)
    A, B = at.view(m, k).double(), bt.view(k, n).double()
    want = (A @ B).cpu().numpy()
    tol = (4 * 2.0 ** -10 * k * A.abs().amax(1, keepdim=True) * B.abs().amax(0, keepdim=True)).cpu().numpy() \
        + 2.0 ** -11 * np.abs(want)
    unsplit, kernels = None, set()
    for v in b200_variants(prec):
        got, rec = run_with(ctx, cfg_of(v, 8), prec, Layout.ROW_MAJOR, Transpose.NO, Transpose.NO,
                            m, n, k, a, b)
        kern = rec.native["kernel"]
        kernels.add(kern)
        if v[5] > 1:
            assert f"splitk{v[5]}" in kern, (v, kern)
        elif v[4] == 2:
            assert "2sm" in kern, (v, kern)
        else:
            assert f"128x{v[1]}" in kern, (v, kern)
        assert np.all(np.abs(got.reshape(m, n).astype(np.float64) - want) <= tol), (v, kern)
        if v[5] == 1:   # every unsplit H kernel issues the same MMA sequence per element
            unsplit = got if unsplit is None else unsplit
            assert got.tobytes() == unsplit.tobytes(), (v, kern)
    assert len(kernels) == len(b200_variants(prec)), kernels


@pytest.mark.parametrize("prec", [Precision.H, Precision.S])
def test_tune_b200_distinct_kernels_and_db_selection(ctx, tmp_path, prec):
    m, n, k = 4096, 128, 9216
    task = TuningTask("gemm_b200", prec, {"m": m, "n": n, "k": k}, ctx.device, timed_runs=2)
    run = tune(task, ctx)
    ok = [x for x in run.measurements if x.status == "ok"]
    assert len(run.measurements) == len(curated_b200(prec))
    assert is_b200_auto(run.measurements[0].configuration)
    assert len({x.kernel for x in ok}) >= 4
    auto_time = run.measurements[0].mean_time
    best = min(ok, key=lambda x: x.mean_time)
    assert best.configuration == run.best and best.mean_time <= auto_time
    db = tb.Database()
    tb.db_insert(db, run)
    path = tmp_path / "db.json"
    db.save(path)
    store = tb.routines.common.get_store(ctx)
    store.database = tb.Database.load(path)
    try:
        a = tb.buffer_alloc(ctx, prec, m * k)
        b = tb.buffer_alloc(ctx, prec, k * n)
        tb.gemm(ctx, Layout.COL_MAJOR, Transpose.NO, Transpose.NO, m, n, k, 1.0, a, b, 0.0,
                tb.buffer_alloc(ctx, prec, m * n))
        rec = ctx.last_launch
        if is_b200_auto(run.best):
            assert rec.kernel_config is None
        else:
            assert rec.kernel_config == run.best.as_dict()
        assert rec.native["kernel"] == best.kernel
        # another shape: exact-only lookup -> the built-in route
        tb.gemm(ctx, Layout.COL_MAJOR, Transpose.NO, Transpose.NO, 512, 128, 9216, 1.0, a, b, 0.0,
                tb.buffer_alloc(ctx, prec, 512 * 128))
        assert ctx.last_launch.kernel_config is None
    finally:
        store.database = None
