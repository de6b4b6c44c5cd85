import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(Path(__file__).resolve().parent))

import paper_1705_05249_b200 as tb  # noqa: E402


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")


def _has_gpu() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:  # noqa: BLE001
        return False


HAS_GPU = _has_gpu()


def pytest_collection_modifyitems(config, items):
    if HAS_GPU:
        return
    skip = pytest.mark.skip(reason="no CUDA device visible")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture
def ctx():
    return tb.context_create(tb.host_device())


def make_buffer(ctx, arr, precision, layout=tb.Layout.COL_MAJOR):
    """Buffer holding ``arr`` in BLAS storage order (conftest.py:22-28 of the reference)."""
    arr = np.asarray(arr, dtype=precision.dtype)
    buf = tb.buffer_alloc(ctx, precision, arr.size)
    if arr.ndim == 2:
        order = "F" if layout is tb.Layout.COL_MAJOR else "C"
        flat = arr.reshape(-1, order=order)
    else:
        flat = arr.reshape(-1)
    tb.buffer_write(buf, 0, flat)
    return buf


def read_mat(buf, shape, layout=tb.Layout.COL_MAJOR):
    m, n = shape
    data = tb.buffer_read(buf, 0, m * n)
    if layout is tb.Layout.COL_MAJOR:
        return data.reshape((n, m)).T.copy()
    return data.reshape((m, n)).copy()


def rand_array(rng, shape, precision, scale=1.0):
    return rng.uniform(-scale, scale, size=shape).astype(precision.dtype)


GOLDEN_DIR = Path(__file__).resolve().parent / "golden"


def load_golden():
    with open(GOLDEN_DIR / "gemm_golden.json") as fh:
        meta = json.load(fh)
    arrays = np.load(GOLDEN_DIR / "gemm_golden.npz")
    return meta["cases"], arrays
