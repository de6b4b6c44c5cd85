"""Multi-GPU sharding of the GEMM path (BASELINE configs C4/C5).

One process per GPU (torch.distributed, NCCL over NVLink 5 / NVSwitch).  The
GEMM shards with no reduction — output units are independent — so there is
no collective on the data path:

* large GEMM: shard the output along N for column-major C (a column block of
  C is one contiguous ``ldc * n_r`` slab when ldc == m) and along M for
  row-major C (a row block is contiguous when ldc == n).  Every rank reads
  all of A (B for row-major) and only its slice of the other operand;
* batched GEMM: shard the instances; instance blocks are contiguous for
  strided batched.

Only when the caller asks for a replicated C does a collective run
(``replicate_c=True``).  With ``chunks=1`` it is one ``all_gather`` after
the GEMM: in place when the shards are equal and contiguous, through a
staging buffer otherwise.  With ``chunks=c > 1`` the rank's block is
computed as c sub-blocks along the sharded axis and each sub-block is sent
to every peer (grouped NCCL send/recv, straight into the peers' final C
positions — no staging) as soon as its GEMM is queued, so the transfer of
sub-block j overlaps the GEMM of sub-block j+1 (SURVEY §7 hard part 7).
NCCL runs on its own stream, ordered after the work queued before each
issue; the caller's stream waits for every transfer before the call returns.
Caveat: the persistent GEMM kernels size their grid to the SM count, so the
NCCL kernels of sub-block j start when SMs free up at the end of GEMM j+1's
last wave at the latest — the overlap is bounded by that.
The reference has no distributed code; this is the
B200-native scaling axis.
"""

from __future__ import annotations

from dataclasses import dataclass

from .core import Buffer, Context, Layout, Transpose
from .errors import UsageError
from .routines import gemm, gemm_strided_batched

__all__ = ["shard_range", "ShardPlan", "plan_gemm_shards", "gemm_sharded",
           "gemm_strided_batched_sharded", "gather_shards", "chunk_ranges", "send_chunk"]


def shard_range(total: int, world: int, rank: int) -> tuple[int, int]:
    """(start, count) of rank's even share; the first total % world ranks get +1."""
    if world < 1 or not 0 <= rank < world:
        raise UsageError("invalid world size / rank")
    base, rem = divmod(total, world)
    start = rank * base + min(rank, rem)
    return start, base + (1 if rank < rem else 0)


@dataclass(frozen=True)
class ShardPlan:
    """How a GEMM's output is split across ranks."""

    axis: str            # "n" (column blocks) or "m" (row blocks) or "batch"
    total: int
    world: int
    starts: tuple
    counts: tuple

    def of(self, rank: int) -> tuple[int, int]:
        return self.starts[rank], self.counts[rank]

    @property
    def equal(self) -> bool:
        return len(set(self.counts)) == 1


def plan_gemm_shards(layout: Layout, m: int, n: int, world: int) -> ShardPlan:
    """N-blocks for column-major C, M-blocks for row-major C (contiguous slabs)."""
    axis, total = ("n", n) if layout is Layout.COL_MAJOR else ("m", m)
    ranges = [shard_range(total, world, r) for r in range(world)]
    return ShardPlan(axis, total, world, tuple(s for s, _ in ranges), tuple(c for _, c in ranges))


def _dist():
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized():
        raise UsageError("torch.distributed is not initialised")
    return dist


def gather_shards(full, plan: ShardPlan, rank: int, slab: int, group=None) -> None:
    """Replicate a sharded flat tensor ``full`` on every rank.

    Rank r owns elements [starts[r]*slab, (starts[r]+counts[r])*slab) of
    ``full`` (slab = elements per unit of the sharded axis).  Equal shards
    gather in place; unequal ones go through a padded staging tensor.
    """
    import torch

    dist = _dist()
    s0, cnt = plan.of(rank)
    if plan.equal:
        out = full[: plan.total * slab]
        mine = out[s0 * slab: (s0 + cnt) * slab]
        dist.all_gather_into_tensor(out, mine, group=group)
        return
    width = max(plan.counts) * slab
    staging = torch.zeros(plan.world * width, dtype=full.dtype, device=full.device)
    send = torch.zeros(width, dtype=full.dtype, device=full.device)
    send[: cnt * slab].copy_(full[s0 * slab: (s0 + cnt) * slab])
    dist.all_gather_into_tensor(staging, send, group=group)
    for r in range(plan.world):
        rs, rc = plan.of(r)
        full[rs * slab: (rs + rc) * slab].copy_(staging[r * width: r * width + rc * slab])


def chunk_ranges(count: int, chunks: int) -> list:
    """(offset, size) of each sub-block of a rank's ``count`` units, in order."""
    chunks = max(1, min(chunks, count)) if count > 0 else 1
    return [shard_range(count, chunks, j) for j in range(chunks)]


def send_chunk(full, plan: ShardPlan, rank: int, slab: int, j: int, chunks: int, group=None) -> list:
    """Issue the grouped send/recv that replicates sub-block ``j`` of every
    rank's shard of the flat tensor ``full`` (rank r's sub-block j lives at
    units [starts[r] + off_j(r), + size_j(r)) of the sharded axis, ``slab``
    elements per unit).  Returns the pending works (wait before reading)."""
    dist = _dist()
    ops = []
    s0, cnt = plan.of(rank)
    mine = chunk_ranges(cnt, chunks)
    if j < len(mine) and mine[j][1] > 0:
        o, sz = mine[j]
        src = full[(s0 + o) * slab:(s0 + o + sz) * slab]
        for peer in range(plan.world):
            if peer != rank:
                ops.append(dist.P2POp(dist.isend, src, peer, group))
    for peer in range(plan.world):
        if peer == rank:
            continue
        ps, pc = plan.of(peer)
        theirs = chunk_ranges(pc, chunks)
        if j < len(theirs) and theirs[j][1] > 0:
            o, sz = theirs[j]
            ops.append(dist.P2POp(dist.irecv, full[(ps + o) * slab:(ps + o + sz) * slab], peer, group))
    return dist.batch_isend_irecv(ops) if ops else []


def gemm_sharded(ctx: Context, layout: Layout, trans_a: Transpose, trans_b: Transpose,
                 m: int, n: int, k: int, alpha, a: Buffer, b: Buffer, beta, c: Buffer, *,
                 rank: int, world: int, replicate_c: bool = False, chunks: int = 1, group=None,
                 lda: int | None = None, ldb: int | None = None) -> ShardPlan:
    """This rank's block of C = alpha*op(A)op(B) + beta*C (full-size buffers,
    C packed: ldc = m col-major / n row-major).  Returns the plan used.

    ``replicate_c`` makes every rank hold all of C afterwards; ``chunks`` > 1
    overlaps that replication with the GEMM (module docstring)."""
    plan = plan_gemm_shards(layout, m, n, world)
    s0, cnt = plan.of(rank)
    col = layout is Layout.COL_MAJOR
    a_rows, a_cols = (m, k) if trans_a is Transpose.NO else (k, m)
    b_rows, b_cols = (k, n) if trans_b is Transpose.NO else (n, k)
    lda = lda if lda is not None else (a_rows if col else a_cols)
    ldb = ldb if ldb is not None else (b_rows if col else b_cols)
    slab = m if col else n
    overlap = replicate_c and chunks > 1 and world > 1
    parts = chunk_ranges(cnt, chunks if overlap else 1)
    works = []
    for j, (o, sz) in enumerate(parts):
        u0 = s0 + o
        if sz > 0:
            if col:
                # columns [u0, u0+sz) of op(B): element offset of column u0
                b_off = u0 * ldb if trans_b is Transpose.NO else u0
                gemm(ctx, layout, trans_a, trans_b, m, sz, k, alpha, a, b, beta, c,
                     lda=lda, b_offset=b_off, ldb=ldb, c_offset=u0 * m, ldc=m)
            else:
                # rows [u0, u0+sz) of op(A) in row-major storage
                a_off = u0 * lda if trans_a is Transpose.NO else u0
                gemm(ctx, layout, trans_a, trans_b, sz, n, k, alpha, a, b, beta, c,
                     a_offset=a_off, lda=lda, ldb=ldb, c_offset=u0 * n, ldc=n)
        if overlap:
            works += send_chunk(c.device_tensor(), plan, rank, slab, j, chunks, group)
    if overlap:
        # peers' ranks may hold more sub-blocks than this one (uneven counts)
        for j in range(len(parts), max(len(chunk_ranges(pc, chunks)) for pc in plan.counts)):
            works += send_chunk(c.device_tensor(), plan, rank, slab, j, chunks, group)
        for w in works:
            w.wait()
        c.mark_device_written()
    elif replicate_c:
        gather_shards(c.device_tensor(), plan, rank, slab, group)
        c.mark_device_written()
    return plan


def gemm_strided_batched_sharded(ctx: Context, layout: Layout, trans_a: Transpose,
                                 trans_b: Transpose, m: int, n: int, k: int, alpha,
                                 a: Buffer, stride_a: int, b: Buffer, stride_b: int, beta,
                                 c: Buffer, stride_c: int, batch_count: int, *, rank: int,
                                 world: int, replicate_c: bool = False, chunks: int = 1,
                                 group=None) -> ShardPlan:
    """This rank's contiguous block of instances of a strided batched GEMM
    (``replicate_c`` / ``chunks`` as for :func:`gemm_sharded`)."""
    ranges = [shard_range(batch_count, world, r) for r in range(world)]
    plan = ShardPlan("batch", batch_count, world, tuple(s for s, _ in ranges),
                     tuple(c_ for _, c_ in ranges))
    s0, cnt = plan.of(rank)
    overlap = replicate_c and chunks > 1 and world > 1
    parts = chunk_ranges(cnt, chunks if overlap else 1)
    works = []
    for j, (o, sz) in enumerate(parts):
        u0 = s0 + o
        if sz > 0:
            gemm_strided_batched(ctx, layout, trans_a, trans_b, m, n, k, alpha, a, stride_a, b,
                                 stride_b, beta, c, stride_c, sz, a_offset=u0 * stride_a,
                                 b_offset=u0 * stride_b, c_offset=u0 * stride_c)
        if overlap:
            works += send_chunk(c.device_tensor(), plan, rank, stride_c, j, chunks, group)
    if overlap:
        for j in range(len(parts), max(len(chunk_ranges(pc, chunks)) for pc in plan.counts)):
            works += send_chunk(c.device_tensor(), plan, rank, stride_c, j, chunks, group)
        for w in works:
            w.wait()
        c.mark_device_written()
    elif replicate_c:
        gather_shards(c.device_tensor(), plan, rank, stride_c, group)
        c.mark_device_written()
    return plan
