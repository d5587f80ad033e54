"""Multi-process (world_size 2, gloo, CPU) tests of the slice partition and the
single reduce of the N>1 path (SURVEY.md §8 e).  The coverage audit is
bit-exact; the reduced sum is compared with the oracle's total, computed
per-rank on that rank's slice range (the CPU stands in for the GPU ranks here:
only the partition / reduction logic is under test)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2310_03978_b200.distributed import partition, coverage_audit


def test_partition_covers_every_slice_once():
    for S in [1, 2, 7, 64, 1000, 4096]:
        for P in [1, 2, 3, 4, 8]:
            assert coverage_audit(S, P)
            sizes = [partition(S, P, r)[1] - partition(S, P, r)[0] for r in range(P)]
            assert max(sizes) - min(sizes) <= 1 and sum(sizes) == S


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import oracle
    from tnworkloads import configs
    w = configs.small(grid=(3, 3), cycles=6, mode="sparse", n_samples=16, n_slices=8, seed=9)
    b, e = partition(w.n_slices, world, rank)
    local = oracle.contract(w.net, w.path, w.sliced, w.samples, slice_ids=range(b, e))
    v = torch.from_numpy(np.ascontiguousarray(local)).view(torch.float64).clone()
    dist.all_reduce(v, op=dist.ReduceOp.SUM)
    if rank == 0:
        out.put(v.view(torch.complex128).numpy().copy())
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_slice_sum_equals_total():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    import oracle
    from tnworkloads import configs
    w = configs.small(grid=(3, 3), cycles=6, mode="sparse", n_samples=16, n_slices=8, seed=9)
    ref = oracle.contract(w.net, w.path, w.sliced, w.samples)
    assert np.abs(got - ref).max() < 1e-12
