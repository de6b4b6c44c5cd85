"""Two ranks over NCCL, one GPU each (skipped with fewer than 2 GPUs): the
sharded GEMM with a replicated C — one all-gather after the GEMM, and the
overlapped per-sub-block send/recv path — leaves every rank holding exactly
the C a single-GPU call produces (bitwise: shapes whose per-sub-block route
issues the same per-element arithmetic, see test_sharding_gpu.py)."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _gpus() -> int:
    try:
        import torch

        return torch.cuda.device_count()
    except Exception:  # noqa: BLE001
        return 0


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    import paper_1705_05249_b200 as tb
    from paper_1705_05249_b200.distributed import gemm_sharded, gemm_strided_batched_sharded

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    out = {}
    try:
        ctx = tb.context_create(tb.host_device())
        ctx.device_index = rank
        for prec in (tb.Precision.S, tb.Precision.H):
            for layout in (tb.Layout.ROW_MAJOR, tb.Layout.COL_MAJOR):
                m, n, k = 1000, 1200, 320
                g = torch.Generator(device="cuda").manual_seed(9)
                at = (torch.rand(m * k, device="cuda", generator=g) * 2 - 1).to(prec.torch_dtype)
                bt = (torch.rand(k * n, device="cuda", generator=g) * 2 - 1).to(prec.torch_dtype)
                a, b = tb.buffer_from_tensor(ctx, prec, at), tb.buffer_from_tensor(ctx, prec, bt)
                ref = tb.buffer_alloc(ctx, prec, m * n)
                tb.gemm(ctx, layout, tb.Transpose.NO, tb.Transpose.NO, m, n, k, 1.0, a, b, 0.0, ref)
                for chunks in (1, 3):
                    c = tb.buffer_alloc(ctx, prec, m * n)
                    gemm_sharded(ctx, layout, tb.Transpose.NO, tb.Transpose.NO, m, n, k, 1.0, a, b, 0.0,
                                 c, rank=rank, world=world, replicate_c=True, chunks=chunks)
                    torch.cuda.synchronize()
                    out[(prec.value, layout.name, chunks)] = bool(
                        torch.equal(c.device_tensor(), ref.device_tensor()))
            s, batch = 32, 1001
            e = s * s
            g = torch.Generator(device="cuda").manual_seed(4)
            at = (torch.rand(batch * e, device="cuda", generator=g) * 2 - 1).to(prec.torch_dtype)
            bt = (torch.rand(batch * e, device="cuda", generator=g) * 2 - 1).to(prec.torch_dtype)
            a, b = tb.buffer_from_tensor(ctx, prec, at), tb.buffer_from_tensor(ctx, prec, bt)
            ref = tb.buffer_alloc(ctx, prec, batch * e)
            tb.gemm_strided_batched(ctx, tb.Layout.ROW_MAJOR, tb.Transpose.NO, tb.Transpose.NO, s, s, s, 1.0,
                                    a, e, b, e, 0.0, ref, e, batch)
            for chunks in (1, 4):
                c = tb.buffer_alloc(ctx, prec, batch * e)
                gemm_strided_batched_sharded(ctx, tb.Layout.ROW_MAJOR, tb.Transpose.NO, tb.Transpose.NO, s, s,
                                             s, 1.0, a, e, b, e, 0.0, c, e, batch, rank=rank, world=world,
                                             replicate_c=True, chunks=chunks)
                torch.cuda.synchronize()
                out[(prec.value, "batched", chunks)] = bool(torch.equal(c.device_tensor(), ref.device_tensor()))
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.skipif(_gpus() < 2, reason="needs 2 GPUs")
def test_replicated_c_two_ranks_nccl():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=120)
    for rank, res in results.items():
        assert res and all(res.values()), (rank, {k: v for k, v in res.items() if not v})
