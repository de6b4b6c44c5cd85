"""Multi-GPU sharding logic on one GPU: every rank's shard is computed in
turn (no collective), and the assembled C must equal the unsharded call
(shards are independent output blocks — SURVEY §8e).

Bitwise equality holds when every shard takes the same per-element
arithmetic as the unsharded call: always for S (sequential-k chain), and for
H unless the cluster split-K factor changes with the shard's (m, n) (it is a
pure function of the CALL's shape, tbgemm.cu hgemm_split_ks).  The shapes of
the bitwise tests never split (K < 32 K blocks); the split case is checked
against the tolerance instead (test_split_k_shards_within_tolerance)."""

import numpy as np
import pytest

import paper_1705_05249_b200 as tb
from paper_1705_05249_b200 import Layout, Precision, Transpose
from paper_1705_05249_b200.distributed import gemm_sharded, gemm_strided_batched_sharded
from conftest import make_buffer, rand_array

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("prec", [Precision.S, Precision.H])
@pytest.mark.parametrize("layout", [Layout.COL_MAJOR, Layout.ROW_MAJOR])
@pytest.mark.parametrize("world", [2, 3, 8])
def test_column_row_shards_assemble_bitwise(ctx, prec, layout, world):
    rng = np.random.default_rng(world)
    m, n, k = 640, 520, 300
    av, bv = rand_array(rng, (m, k), prec), rand_array(rng, (k, n), prec)
    a, b = make_buffer(ctx, av, prec, layout), make_buffer(ctx, bv, prec, layout)
    full = tb.buffer_alloc(ctx, prec, m * n)
    tb.gemm(ctx, layout, Transpose.NO, Transpose.NO, m, n, k, 1.0, a, b, 0.0, full)
    sharded = tb.buffer_alloc(ctx, prec, m * n)
    for rank in range(world):
        gemm_sharded(ctx, layout, Transpose.NO, Transpose.NO, m, n, k, 1.0, a, b, 0.0, sharded,
                     rank=rank, world=world)
    assert tb.buffer_read(sharded, 0, m * n).tobytes() == tb.buffer_read(full, 0, m * n).tobytes()


@pytest.mark.parametrize("prec", [Precision.S, Precision.H])
def test_batch_shards_assemble_bitwise(ctx, prec):
    rng = np.random.default_rng(5)
    s, batch, world = 32, 1000, 8
    e = s * s
    av, bv = rand_array(rng, batch * e, prec), rand_array(rng, batch * e, prec)
    a, b = make_buffer(ctx, av, prec), make_buffer(ctx, bv, prec)
    full = tb.buffer_alloc(ctx, prec, batch * e)
    tb.gemm_strided_batched(ctx, Layout.ROW_MAJOR, Transpose.NO, Transpose.NO, s, s, s, 1.0, a, e,
                            b, e, 0.0, full, e, batch)
    sharded = tb.buffer_alloc(ctx, prec, batch * e)
    for rank in range(world):
        gemm_strided_batched_sharded(ctx, Layout.ROW_MAJOR, Transpose.NO, Transpose.NO, s, s, s, 1.0,
                                     a, e, b, e, 0.0, sharded, e, batch, rank=rank, world=world)
    assert tb.buffer_read(sharded, 0, batch * e).tobytes() == tb.buffer_read(full, 0, batch * e).tobytes()


def test_split_k_shards_within_tolerance(ctx):
    """(4096, 128, 9216) H row-sharded over 2 ranks: each 2048-row shard picks
    its own split-K factor, so the assembled C differs from the unsharded call
    in summation order only — within 2x the FP16 tolerance of it."""
    import torch

    prec = Precision.H
    m, n, k, world = 4096, 128, 9216, 2
    g = torch.Generator(device="cuda").manual_seed(11)
    at = (torch.rand(m * k, device="cuda", generator=g) * 2 - 1).half()
    bt = (torch.rand(k * n, device="cuda", generator=g) * 2 - 1).half()
    a, b = tb.buffer_from_tensor(ctx, prec, at), tb.buffer_from_tensor(ctx, prec, bt)
    full = tb.buffer_alloc(ctx, prec, m * n)
    tb.gemm(ctx, Layout.ROW_MAJOR, Transpose.NO, Transpose.NO, m, n, k, 1.0, a, b, 0.0, full)
    sharded = tb.buffer_alloc(ctx, prec, m * n)
    for rank in range(world):
        gemm_sharded(ctx, Layout.ROW_MAJOR, Transpose.NO, Transpose.NO, m, n, k, 1.0, a, b, 0.0,
                     sharded, rank=rank, world=world)
    A, B = at.view(m, k).double(), bt.view(k, n).double()
    want = A @ B
    tol = 4 * 2.0 ** -10 * k * A.abs().amax(1, keepdim=True) * B.abs().amax(0, keepdim=True) \
        + 2.0 ** -11 * want.abs()
    x = sharded.device_tensor().view(m, n).double()
    y = full.device_tensor().view(m, n).double()
    assert bool(((x - y).abs() <= 2 * tol).all())
    assert bool(((x - want).abs() <= tol).all())
