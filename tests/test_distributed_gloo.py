"""Multi-rank sharding logic on CPU with world_size 2 over gloo.

The GEMM itself needs the GPU; here each rank fills its shard of C from the
oracle (the value a rank's local GEMM produces) and the collective path
(plan, in-place / staged all-gather, layout of the slabs) is checked.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1705_05249_b200 import Layout
from paper_1705_05249_b200.distributed import gather_shards, plan_gemm_shards, shard_range


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shard_range_partitions():
    for total in (0, 1, 7, 8, 8192, 16385):
        for world in (1, 2, 3, 8):
            ranges = [shard_range(total, world, r) for r in range(world)]
            assert sum(c for _, c in ranges) == total
            pos = 0
            for s, c in ranges:
                assert s == pos
                pos += c
            assert max(c for _, c in ranges) - min(c for _, c in ranges) <= 1


def test_plan_axis_follows_layout():
    assert plan_gemm_shards(Layout.COL_MAJOR, 10, 12, 4).axis == "n"
    assert plan_gemm_shards(Layout.ROW_MAJOR, 10, 12, 4).axis == "m"
    p = plan_gemm_shards(Layout.COL_MAJOR, 10, 13, 4)
    assert p.counts == (4, 3, 3, 3) and not p.equal


def _worker(rank, world, port, n_cols, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m, k = 6, 5
        rng = np.random.default_rng(0)
        A = rng.standard_normal((m, k)).astype(np.float32)
        B = rng.standard_normal((k, n_cols)).astype(np.float32)
        full_expected = (A @ B).reshape(-1, order="F")     # column-major C
        plan = plan_gemm_shards(Layout.COL_MAJOR, m, n_cols, world)
        s0, cnt = plan.of(rank)
        c = torch.zeros(m * n_cols, dtype=torch.float32)
        # this rank's local GEMM result: columns [s0, s0+cnt)
        c[s0 * m:(s0 + cnt) * m] = torch.from_numpy(full_expected[s0 * m:(s0 + cnt) * m])
        gather_shards(c, plan, rank, m)
        q.put((rank, bool(np.array_equal(c.numpy(), full_expected))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n_cols", [8, 7])   # equal (in-place) and unequal (staged) shards
def test_gather_replicates_c_world2(n_cols):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n_cols, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert results == {0: True, 1: True}


def _chunk_worker(rank, world, port, n_rows, chunks, q):
    """Row-major C (M shards): each rank fills its rows sub-block by sub-block
    and replicates every sub-block with send_chunk as soon as it is 'computed'
    (the overlapped replicate_c path of gemm_sharded)."""
    from paper_1705_05249_b200.distributed import chunk_ranges, send_chunk

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, k = 5, 4
        rng = np.random.default_rng(1)
        A = rng.standard_normal((n_rows, k)).astype(np.float32)
        B = rng.standard_normal((k, n)).astype(np.float32)
        want = (A @ B).reshape(-1)                         # row-major C
        plan = plan_gemm_shards(Layout.ROW_MAJOR, n_rows, n, world)
        s0, cnt = plan.of(rank)
        c = torch.full((n_rows * n,), -1.0, dtype=torch.float32)
        works = []
        parts = chunk_ranges(cnt, chunks)
        for j, (o, sz) in enumerate(parts):
            u0 = s0 + o
            c[u0 * n:(u0 + sz) * n] = torch.from_numpy(want[u0 * n:(u0 + sz) * n])
            works += send_chunk(c, plan, rank, n, j, chunks)
        for j in range(len(parts), max(len(chunk_ranges(pc, chunks)) for pc in plan.counts)):
            works += send_chunk(c, plan, rank, n, j, chunks)
        for w in works:
            w.wait()
        q.put((rank, bool(np.array_equal(c.numpy(), want))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n_rows,chunks", [(2, 8, 2), (2, 7, 3), (3, 7, 4), (3, 2, 2)])
def test_chunked_replication(world, n_rows, chunks):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_chunk_worker, args=(r, world, port, n_rows, chunks, q))
             for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert results == {r: True for r in range(world)}
