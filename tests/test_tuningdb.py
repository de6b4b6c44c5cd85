"""Tuning database, defaults hierarchy and overrides (reference tests/test_tuningdb.py)."""

import math

import pytest

import paper_1705_05249_b200 as tb
from paper_1705_05249_b200 import GemmParams, Precision
from paper_1705_05249_b200.tuningdb import Database, DbEntry, DbKey, compute_defaults, db_lookup


def _cfg(mwg):
    return GemmParams(MWG=mwg, NWG=mwg).to_config()


def _entry(device, args, timings, prec=Precision.S):
    key = DbKey.for_task("gemm", prec, device, args)
    meas = [{"params": c.as_dict(), "per_run_times_s": [t], "mean_time_s": t, "status": "ok"}
            for c, t in timings]
    best = min(timings, key=lambda ct: ct[1])[0]
    return DbEntry(key=key, measurements=meas, best=best)


DEV_A = tb.b200_device(name="gpu-a")
DEV_B = tb.b200_device(name="gpu-b")
DEV_C = tb.DeviceSpec(name="cpu-c", vendor="x", architecture="y")


def test_insert_lookup_and_keep_faster():
    db = Database()
    db.insert(_entry(DEV_A, (64, 64, 64), [(_cfg(64), 2.0), (_cfg(32), 1.0)]))
    cfg, level = db_lookup(db, DEV_A, "gemm", Precision.S, (64, 64, 64))
    assert cfg == _cfg(32) and level == "device"
    db.insert(_entry(DEV_A, (64, 64, 64), [(_cfg(128), 5.0)]))  # slower: ignored
    assert db_lookup(db, DEV_A, "gemm", Precision.S, (64, 64, 64))[0] == _cfg(32)


def test_fallback_chain():
    db = Database()
    db.insert(_entry(DEV_A, (1024, 1024, 1024), [(_cfg(64), 1.0)]))
    db.insert(_entry(DEV_A, (8, 8, 8), [(_cfg(16), 1.0)]))
    assert db_lookup(db, DEV_A, "gemm", Precision.S, (5, 5, 5)) == (_cfg(64), "device_any_args")
    cfg, level = db_lookup(db, DEV_B, "gemm", Precision.S, (5, 5, 5))
    assert level == "architecture"
    cfg, level = db_lookup(db, DEV_C, "gemm", Precision.S, (5, 5, 5))
    assert level == "global"
    with pytest.raises(tb.DbLookupError):
        db_lookup(Database(), DEV_A, "gemm", Precision.S, (1, 1, 1))
    with pytest.raises(tb.DbLookupError):
        db_lookup(db, DEV_A, "gemm", Precision.H, (1, 1, 1))


def test_defaults_geometric_mean():
    db = Database()
    db.insert(_entry(DEV_A, (1, 1, 1), [(_cfg(64), 1.0), (_cfg(32), 1.1)]))
    db.insert(_entry(DEV_B, (1, 1, 1), [(_cfg(64), 3.0), (_cfg(32), 1.0)]))
    d = compute_defaults(db)
    # relative: 64 -> (1, 3), 32 -> (1.1, 1): geomean favours 32
    assert d[("architecture", "sm_100a", "gemm", "S")] == _cfg(32)
    assert math.isclose(len(d), 4)


def test_json_roundtrip(tmp_path):
    db = Database()
    db.insert(_entry(DEV_A, (256, 256, 256), [(_cfg(64), 1.0)]))
    path = tmp_path / "db.json"
    db.save(path)
    loaded = Database.load(path)
    assert db_lookup(loaded, DEV_A, "gemm", Precision.S, (256, 256, 256)) == \
        db_lookup(db, DEV_A, "gemm", Precision.S, (256, 256, 256))
    doc = db.to_json()
    assert doc["schema_version"] == 1
    doc["entries"][0]["future_field"] = 1          # unknown fields ignored on read
    Database.from_json(doc)


def test_parameter_store_resolution():
    store = tb.ParameterStore()
    cfg, level = store.resolve("gemm", Precision.S, DEV_A, (40, 40, 40))
    assert level == "builtin" and cfg["MWG"] == 128
    override = GemmParams(MWG=32, NWG=32, KWG=16, KWI=8).to_config()
    tb.override_parameters(store, "gemm", Precision.S, DEV_A, (40, 40, 40), override)
    assert store.resolve("gemm", Precision.S, DEV_A, (40, 40, 40)) == (override, "override")
    assert store.resolve("gemm", Precision.S, DEV_A, (48, 48, 48))[1] == "builtin"
    bad = GemmParams(MDIMC=32, NDIMC=32, MWG=32, NWG=32).to_config()
    with pytest.raises(tb.ValidationError):
        store.set_override("gemm", Precision.S, tb.DeviceSpec(max_work_group_size=512), (1, 1, 1), bad)
    store.clear_overrides()
    assert store.resolve("gemm", Precision.S, DEV_A, (40, 40, 40))[1] == "builtin"
