"""Core types, buffers and the host mirror (reference tests/test_core.py).

Buffers live on the context's device (CUDA on the GPU box, host memory when
no GPU is visible — compute entry points then raise, see test_routines_cpu)."""

import numpy as np
import pytest

import paper_1705_05249_b200 as tb
from paper_1705_05249_b200 import Precision


def test_precision_element_sizes():
    assert [p.elemsize for p in (Precision.H, Precision.S, Precision.D, Precision.C, Precision.Z)] == \
        [2, 4, 8, 8, 16]
    assert Precision.H.compute_dtype == np.float32
    assert Precision.H.eps == 2.0 ** -10 and Precision.S.eps == 2.0 ** -23


def test_buffer_alloc_zero_and_roundtrip(ctx):
    b = tb.buffer_alloc(ctx, Precision.S, 10)
    assert b.nbytes == 40
    assert np.all(tb.buffer_read(b, 0, 10) == 0)
    tb.buffer_write(b, 3, [1, 2, 3])
    assert tb.buffer_read(b, 2, 5).tolist() == [0, 1, 2, 3, 0]
    h = tb.buffer_alloc(ctx, Precision.H, 17)
    assert h.nbytes * 2 == tb.buffer_alloc(ctx, Precision.S, 17).nbytes


def test_buffer_range_errors(ctx):
    b = tb.buffer_alloc(ctx, Precision.S, 8)
    with pytest.raises(tb.RangeError):
        tb.buffer_read(b, 5, 4)
    with pytest.raises(tb.RangeError):
        tb.buffer_write(b, -1, [1.0])
    with pytest.raises(tb.UsageError):
        tb.buffer_alloc(ctx, Precision.S, -1)


def test_data_mirror_semantics(ctx):
    b = tb.buffer_alloc(ctx, Precision.S, 6)
    b.data[:] = np.arange(6)           # host write ...
    assert tb.buffer_read(b, 0, 6).tolist() == [0, 1, 2, 3, 4, 5]   # ... reaches the device
    tb.buffer_write(b, 0, [9, 9])      # device write ...
    assert b.data[:3].tolist() == [9, 9, 2]                         # ... reaches the mirror
    d = b.data
    d[5] = 42
    assert tb.buffer_read(b, 5, 1).tolist() == [42]


def test_roundtrip_bit_identical(ctx):
    rng = np.random.default_rng(1)
    for prec in (Precision.H, Precision.S):
        vals = rng.standard_normal(33).astype(prec.dtype)
        b = tb.buffer_alloc(ctx, prec, 33)
        tb.buffer_write(b, 0, vals)
        assert tb.buffer_read(b, 0, 33).tobytes() == vals.tobytes()


def test_context_isolation():
    c1 = tb.context_create(tb.host_device())
    c2 = tb.context_create(tb.host_device())
    b = tb.buffer_alloc(c1, Precision.S, 4)
    assert c1.owns(b) and not c2.owns(b)
    with pytest.raises(tb.UsageError):
        c2.check_owns(b)


def test_device_spec_validation_and_json():
    spec = tb.b200_device()
    assert spec.is_b200 and spec.compute_units == 148 and spec.local_mem_bytes == 232448
    assert tb.DeviceSpec.from_dict(spec.to_dict()) == spec
    with pytest.raises(tb.ConfigurationError):
        tb.context_create(tb.DeviceSpec(compute_units=0))
    with pytest.raises(tb.ConfigurationError):
        tb.DeviceSpec.from_dict({"device_type": "TPU"})


def test_half_encodings():
    assert tb.half_from_f32(1.0) == 0x3C00
    assert tb.half_from_f32(65504.0) == 0x7BFF
    assert tb.half_from_f32(1e6) == 0x7C00
    assert tb.half_to_f32(0x3555) == pytest.approx(0.33325195)
    assert tb.half_from_f32(1 + 2 ** -11) == 0x3C00    # tie to even
    with pytest.raises(tb.UsageError):
        tb.half_to_f32(0x10000)
