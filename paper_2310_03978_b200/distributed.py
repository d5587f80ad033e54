"""Multi-GPU slice partitioning and the single reduce of the slice sums (SURVEY.md §8 e).

Slices are independent sub-tasks ("these sub-tasks are
independent of each other and can be parallelly implemented on different
computing devices"); "each A100 GPU executed partial sub-tasks independently,
and the final outcome was the sum of the resulting tensors" (L497).  Rank r of
P contracts the contiguous range ``partition(S, P, r)`` into its own fp64
accumulator; one collective over NCCL (NVLink 5 / NVSwitch) produces the total.
No other data crosses GPUs.

Stream ordering.  The library enqueues everything on the stream its context was
created with (``Contraction.stream``), which need not be torch's current stream.
``reduce_amplitudes`` allocates the output, gathers the rank's sum into it and runs
the collective all on that stream (ProcessGroupNCCL orders its kernels after the
current stream), then makes the caller's current stream wait for it.

Determinism.  SPEC L390 sums slices in a fixed order; with an NCCL ``all_reduce``
the order of the cross-rank additions is NCCL's.  The default reduce is therefore
an ``all_gather`` of the per-rank fp64 partial sums followed by their addition in
rank order on every rank: bit-identical on every rank and across runs for a fixed
world size (a different world size changes which slices share a partial sum, so
results then agree to rounding only).  ``deterministic=False`` uses
one ``all_reduce(SUM)`` instead.
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


def _sum_collective(v, world, group, deterministic):
    """Sum the float64 view ``v`` over ranks in place (see module docstring)."""
    import torch
    import torch.distributed as dist
    if world <= 1:
        return v
    if not deterministic:
        dist.all_reduce(v, op=dist.ReduceOp.SUM, group=group)
        return v
    parts = [torch.empty_like(v) for _ in range(world)]
    dist.all_gather(parts, v, group=group)
    v.copy_(parts[0])
    for p in parts[1:]:
        v.add_(p)
    return v


def reduce_amplitudes(ctx, world: int, group=None, deterministic: bool = True):
    """Gather this rank's slice sum (tn_sum_slices) and sum it across ranks.

    ``ctx`` is a ``Contraction`` (or any object with ``n_out``, ``sum_slices(out)``,
    ``torch_device`` and ``stream``).  Returns a complex128 tensor on ctx's device,
    identical on every rank, ready on the caller's current stream."""
    import torch
    dev = ctx.torch_device
    stream = ctx.stream if dev.type == "cuda" else None
    if stream is None:
        out = torch.empty(ctx.n_out, dtype=torch.complex128, device=dev)
        ctx.sum_slices(out)        # writes every element (gather in caller order)
        _sum_collective(torch.view_as_real(out), world, group, deterministic)
        return out
    caller = torch.cuda.current_stream(dev)
    with torch.cuda.stream(stream):
        out = torch.empty(ctx.n_out, dtype=torch.complex128, device=dev)
        ctx.sum_slices(out)
        _sum_collective(torch.view_as_real(out), world, group, deterministic)
    caller.wait_stream(stream)
    out.record_stream(caller)
    return out


def contract_partitioned(ctx, world: int, rank: int, precision="extended", mixed_topk=10,
                         group=None, deterministic: bool = True):
    """Contract this rank's share of all slices and return the global amplitudes."""
    b, e = partition(ctx.n_slices, world, rank)
    ctx.reset_accumulator()
    if e > b:
        ctx.contract(b, e, precision, mixed_topk)
    return reduce_amplitudes(ctx, world, group, deterministic)
