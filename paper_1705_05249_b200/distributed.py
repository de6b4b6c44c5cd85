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

Only when the caller asks for a replicated C does one ``all_gather`` run
(``replicate_c=True``): in place when the shards are equal and contiguous,
through a staging buffer otherwise.  The reference has no distributed code
(SURVEY §2.2); this is the B200-native scaling axis.
"""

from __future__ import annotations

from dataclasses import dataclass

from .core import Buffer, Context, Layout, Transpose
from .errors import UsageError
from .routines import gemm, gemm_strided_batched

__all__ = ["shard_range", "ShardPlan", "plan_gemm_shards", "gemm_sharded",
           "gemm_strided_batched_sharded", "gather_shards"]


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


def gemm_sharded(ctx: Context, layout: Layout, trans_a: Transpose, trans_b: Transpose,
                 m: int, n: int, k: int, alpha, a: Buffer, b: Buffer, beta, c: Buffer, *,
                 rank: int, world: int, replicate_c: bool = False, group=None,
                 lda: int | None = None, ldb: int | None = None) -> ShardPlan:
    """This rank's block of C = alpha*op(A)op(B) + beta*C (full-size buffers,
    C packed: ldc = m col-major / n row-major).  Returns the plan used."""
    plan = plan_gemm_shards(layout, m, n, world)
    s0, cnt = plan.of(rank)
    col = layout is Layout.COL_MAJOR
    a_rows, a_cols = (m, k) if trans_a is Transpose.NO else (k, m)
    b_rows, b_cols = (k, n) if trans_b is Transpose.NO else (n, k)
    lda = lda if lda is not None else (a_rows if col else a_cols)
    ldb = ldb if ldb is not None else (b_rows if col else b_cols)
    if cnt > 0:
        if col:
            # columns [s0, s0+cnt) of op(B): element offset of column s0
            b_off = s0 * ldb if trans_b is Transpose.NO else s0
            gemm(ctx, layout, trans_a, trans_b, m, cnt, k, alpha, a, b, beta, c,
                 lda=lda, b_offset=b_off, ldb=ldb, c_offset=s0 * m, ldc=m)
        else:
            # rows [s0, s0+cnt) of op(A) in row-major storage
            a_off = s0 * lda if trans_a is Transpose.NO else s0
            gemm(ctx, layout, trans_a, trans_b, cnt, n, k, alpha, a, b, beta, c,
                 a_offset=a_off, lda=lda, ldb=ldb, c_offset=s0 * n, ldc=n)
    if replicate_c:
        gather_shards(c.device_tensor(), plan, rank, m if col else n, group)
        c.mark_device_written()
    return plan


def gemm_strided_batched_sharded(ctx: Context, layout: Layout, trans_a: Transpose,
                                 trans_b: Transpose, m: int, n: int, k: int, alpha,
                                 a: Buffer, stride_a: int, b: Buffer, stride_b: int, beta,
                                 c: Buffer, stride_c: int, batch_count: int, *, rank: int,
                                 world: int, replicate_c: bool = False, group=None) -> ShardPlan:
    """This rank's contiguous block of instances of a strided batched GEMM."""
    ranges = [shard_range(batch_count, world, r) for r in range(world)]
    plan = ShardPlan("batch", batch_count, world, tuple(s for s, _ in ranges),
                     tuple(c_ for _, c_ in ranges))
    s0, cnt = plan.of(rank)
    if cnt > 0:
        gemm_strided_batched(ctx, layout, trans_a, trans_b, m, n, k, alpha, a, stride_a, b,
                             stride_b, beta, c, stride_c, cnt, a_offset=s0 * stride_a,
                             b_offset=s0 * stride_b, c_offset=s0 * stride_c)
    if replicate_c:
        gather_shards(c.device_tensor(), plan, rank, stride_c, group)
        c.mark_device_written()
    return plan
