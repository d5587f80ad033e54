"""Multi-GPU slice partitioning and the single NCCL reduce (SURVEY.md §8 e).

Slices are independent sub-tasks ("these sub-tasks are
independent of each other and can be parallelly implemented on different
computing devices"); "each A100 GPU executed partial sub-tasks independently,
and the final outcome was the sum of the resulting tensors" (L497).  Rank r of
P contracts the contiguous range ``partition(S, P, r)`` into its own fp64
accumulator; one ``all_reduce(SUM)`` of the complex128 amplitude vector over
NCCL (NVLink 5 / NVSwitch) produces the total.  No other data crosses GPUs.
"""
from __future__ import annotations


def partition(n_slices: int, world: int, rank: int):
    """Contiguous, balanced range [b, e) of slices for ``rank`` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    q, r = divmod(n_slices, world)
    b = rank * q + min(rank, r)
    e = b + q + (1 if rank < r else 0)
    return b, e


def coverage_audit(n_slices: int, world: int) -> bool:
    """Every slice index is assigned to exactly one rank (bit-exact bookkeeping)."""
    seen = [0] * n_slices
    for r in range(world):
        b, e = partition(n_slices, world, r)
        for t in range(b, e):
            seen[t] += 1
    return all(x == 1 for x in seen)


def reduce_amplitudes(ctx, world: int, group=None, device=None):
    """Gather this rank's slice sum (tn_sum_slices, device) and SUM it across ranks.
    Returns a complex128 CUDA tensor (identical on every rank)."""
    import torch
    import torch.distributed as dist
    out = torch.zeros(ctx.n_out, dtype=torch.complex128,
                      device=device or torch.device("cuda", torch.cuda.current_device()))
    ctx.sum_slices(out)
    if world > 1:
        v = torch.view_as_real(out)
        dist.all_reduce(v, op=dist.ReduceOp.SUM, group=group)
    return out


def contract_partitioned(ctx, world: int, rank: int, precision="extended", mixed_topk=10,
                         group=None):
    """Contract this rank's share of all slices and return the global amplitudes."""
    b, e = partition(ctx.n_slices, world, rank)
    ctx.reset_accumulator()
    if e > b:
        ctx.contract(b, e, precision, mixed_topk)
    return reduce_amplitudes(ctx, world, group)
