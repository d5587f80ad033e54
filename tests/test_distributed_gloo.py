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


class OracleContext:
    """Stand-in for ``Contraction`` on CPU ranks (tests only): the same method surface
    that ``distributed.contract_partitioned`` / ``reduce_amplitudes`` use, with the
    slice contraction done by the oracle, so the partition -> per-rank accumulate ->
    collective logic runs exactly as on GPUs (gloo instead of NCCL)."""

    def __init__(self, w):
        import torch
        self.w = w
        self.n_slices = w.n_slices
        self.acc = None
        self.torch_device = torch.device("cpu")
        self.stream = None
        self.contracted = []

    @property
    def n_out(self):
        return len(self.w.samples)

    def reset_accumulator(self):
        self.acc = np.zeros(self.n_out, np.complex128)

    def contract(self, b, e, precision="extended", mixed_topk=10):
        import oracle
        self.contracted.extend(range(b, e))
        for t in range(b, e):
            self.acc = self.acc + oracle.contract_slice(self.w.net, self.w.path, self.w.sliced, t,
                                                        self.w.samples)

    def sum_slices(self, out):
        out.copy_(torch.from_numpy(self.acc))


def _worker_partitioned(rank, world, port, det, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from tnworkloads import configs
    from paper_2310_03978_b200.distributed import contract_partitioned
    w = configs.small(grid=(3, 3), cycles=6, mode="sparse", n_samples=16, n_slices=8, seed=9)
    ctx = OracleContext(w)
    amps = contract_partitioned(ctx, world, rank, deterministic=det)
    out.put((rank, ctx.contracted, amps.numpy().copy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("det", [True, False])
def test_contract_partitioned_over_gloo(world, det):
    """distributed.contract_partitioned itself (not a re-implementation): every rank
    contracts its contiguous range, every slice exactly once, and every rank ends with
    the same total = the oracle's sum over all slices; the deterministic (all_gather,
    rank-order) reduce gives bit-identical results on every rank."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_partitioned, args=(r, world, port, det, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    import oracle
    from tnworkloads import configs
    w = configs.small(grid=(3, 3), cycles=6, mode="sparse", n_samples=16, n_slices=8, seed=9)
    ref = oracle.contract(w.net, w.path, w.sliced, w.samples)
    covered = sorted(t for _, ts, _ in res for t in ts)
    assert covered == list(range(w.n_slices))
    for _, _, amps in res:
        assert np.abs(amps - ref).max() < 1e-12
    if det:
        for _, _, amps in res[1:]:
            assert np.array_equal(amps, res[0][2])


def test_bench_self_spawns_ranks_for_gpus_n():
    """``bench.py --gpus 2`` without torchrun re-launches itself as 2 ranks (weak #4 of
    round 1): exercised with the reference arm, where rank 0 times the oracle and
    prints the one JSON line and rank 1 exits 0 without work."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--workload", "c2", "--steps", "1", "--warmup", "0", "--cpu-flops", "3e9"],
                       capture_output=True, text=True, timeout=600, env=env, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1
    assert lines[0]["impl"] == "reference" and lines[0]["n_gpus"] == 2
