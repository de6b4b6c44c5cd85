"""Search space, curated set and constraint filter (reference tests/test_params.py)."""

import random

import pytest

import paper_1705_05249_b200 as tb
from paper_1705_05249_b200 import GemmParams, Precision
from paper_1705_05249_b200.kernels import (curated_configurations, default_config,
                                          enumerate_search_space, full_grid_size,
                                          local_mem_usage, random_configuration,
                                          validate_gemm_params)

DEV = tb.DeviceSpec(max_work_group_size=1024, local_mem_bytes=49152)
B200 = tb.b200_device()


def test_full_gemm_grid_size():
    assert full_grid_size("gemm") == 1_327_104


def test_curated_set_size_and_determinism():
    first = curated_configurations("gemm")
    assert len(first) == 512
    assert first == curated_configurations("gemm")
    assert list(enumerate_search_space("gemm", "curated")) == first


def test_random_enumeration_seeded():
    a = list(enumerate_search_space("gemm", "random", n=20, seed=3))
    b = list(enumerate_search_space("gemm", "random", n=20, seed=3))
    assert a == b and len(a) == 20
    with pytest.raises(tb.UsageError):
        list(enumerate_search_space("gemm", "random", n=-1))
    with pytest.raises(tb.UsageError):
        list(enumerate_search_space("gemm", "bogus"))


def test_validate_examples():
    p = GemmParams(MWG=64, NWG=64, KWG=16, MDIMC=16, NDIMC=16, MDIMA=16, NDIMB=16, KWI=2,
                   VWM=2, VWN=2, SA=1, SB=1)
    assert validate_gemm_params(p, DEV, Precision.S).valid
    v = validate_gemm_params(GemmParams(MDIMC=32, NDIMC=32), tb.DeviceSpec(max_work_group_size=512),
                             Precision.S)
    assert not v.valid and any("work-group too large" in s for s in v.violations)
    v = validate_gemm_params(GemmParams(MWG=128, NWG=128, KWG=32, SA=1, SB=1),
                             tb.DeviceSpec(local_mem_bytes=16384), Precision.S)
    assert any("local memory" in s for s in v.violations)
    assert not validate_gemm_params(GemmParams(MWG=16, MDIMC=16, VWM=2), DEV, Precision.S).valid
    assert not validate_gemm_params(GemmParams(KWG=16, KWI=12), DEV, Precision.S).valid


def test_every_rejection_names_a_constraint():
    rng = random.Random(7)
    for _ in range(2000):
        v = validate_gemm_params(random_configuration("gemm", rng), DEV, Precision.S)
        if not v.valid:
            assert v.violations


def test_local_mem_usage_examples():
    assert local_mem_usage(GemmParams(SA=0, SB=0), Precision.S) == 0
    assert local_mem_usage(GemmParams(SA=1, SB=0, KWG=16, MWG=64), Precision.S) == 4096
    assert local_mem_usage(GemmParams(SA=1, SB=1, KWG=32, MWG=128, NWG=128), Precision.D) == 65536


def test_b200_default_is_valid_and_distinct():
    for prec in (Precision.S, Precision.H):
        cfg = default_config("gemm", B200, prec)
        assert validate_gemm_params(cfg, B200, prec).valid
        assert cfg["MWG"] == 128 and cfg["NWG"] == 128
    # the reference host profile keeps the reference built-in (params.py:424)
    host_cfg = default_config("gemm", DEV, Precision.S)
    assert host_cfg.as_dict() == GemmParams(MWG=64, NWG=64, KWG=16, KWI=8).as_dict()


def test_b200_accepts_all_curated():
    for prec in (Precision.S, Precision.H):
        valid = [c for c in curated_configurations("gemm") if validate_gemm_params(c, B200, prec)]
        assert len(valid) > 300


def test_configuration_make_requires_exact_names():
    with pytest.raises(tb.UsageError):
        tb.Configuration.make("gemm", {"MWG": 64})
    with pytest.raises(tb.UsageError):
        tb.Configuration.make("axpy", {"WGS": 64})
    cfg = GemmParams().to_config()
    assert str(cfg).startswith("gemm[MWG=64")
    assert cfg["KWI"] == 2


def test_launch_grid_examples():
    cfg = GemmParams(MWG=64, NWG=64, MDIMC=16, NDIMC=16).to_config()
    grid = tb.launch_grid("gemm", (1024, 1024), cfg)
    assert grid.work_groups == (16, 16) and grid.work_group_size == 256
    with pytest.raises(tb.UsageError):
        tb.launch_grid("gemm", (100, 128), cfg)
    assert tb.launch_grid("gemm_direct", (100, 70), cfg).work_groups == (2, 2)


def test_gemm_b200_family():
    """The sm_100a tuning family: instantiated kernels only, the all-zero
    built-in route first in the curated list, sm_100 devices only."""
    from paper_1705_05249_b200.kernels.params import (b200_auto, b200_variants, curated_b200,
                                                      is_b200_auto, validate_config)

    B200 = tb.b200_device()
    for prec in (Precision.H, Precision.S):
        cur = curated_b200(prec)
        assert is_b200_auto(cur[0]) and len(set(cur)) == len(cur)
        assert all(validate_config(c, B200, prec) for c in cur)
        assert len(cur) == 1 + 4 * len(b200_variants(prec))
    assert validate_config(b200_auto(), B200, Precision.S)
    bad = tb.Configuration.make("gemm_b200", dict(MWG=256, NWG=256, KWG=64, STAGES=0, CTA_GROUP=2,
                                                  SPLIT_K=1, GROUP_M=0))
    assert validate_config(bad, B200, Precision.H) and not validate_config(bad, B200, Precision.S)
    host = tb.DeviceSpec()
    assert not validate_config(b200_auto(), host, Precision.S)


def test_gemm_b200_exact_only_resolution():
    """gemm_b200 DB entries apply to their exact shape only (tuningdb.py
    EXACT_ONLY_FAMILIES); other shapes fall back to the built-in route."""
    from paper_1705_05249_b200.kernels.params import curated_b200, is_b200_auto
    from paper_1705_05249_b200.tuningdb import DbEntry, DbKey

    B200 = tb.b200_device()
    cfg = curated_b200(Precision.H)[5]
    db = tb.Database()
    key = DbKey.for_task("gemm_b200", Precision.H, B200, (4096, 128, 9216))
    db.insert(DbEntry(key=key, measurements=[{"params": cfg.as_dict(), "per_run_times_s": [1e-5],
                                              "mean_time_s": 1e-5, "status": "ok"}], best=cfg))
    store = tb.ParameterStore(database=db)
    assert store.resolve("gemm_b200", Precision.H, B200, (4096, 128, 9216)) == (cfg, "device")
    got, src = store.resolve("gemm_b200", Precision.H, B200, (1024, 1024, 1024))
    assert is_b200_auto(got) and src == "builtin"
