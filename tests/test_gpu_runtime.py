"""GPU tests of the runtime around the kernels (``-m gpu``): device memory through
the caller's allocator (tn_allocator, SURVEY.md §8 b), the stream ordering of the
cross-rank reduce (distributed.reduce_amplitudes, §8 e) and the delayed-scaling
history across tensor uploads.  Values are checked against the CPU
oracle on the same seeded inputs."""
import ctypes as C
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle                                          # noqa: E402
from tnworkloads import configs                        # noqa: E402
from paper_2310_03978_b200 import Contraction, TNError, tn as tnlib   # noqa: E402
from paper_2310_03978_b200.distributed import reduce_amplitudes, contract_partitioned  # noqa: E402

EXT_TOL = 1e-5
TC = {"TN_TC_MIN_BIG": "8", "TN_TC_MIN_SMALL": "2", "TN_TC_MIN_K": "2"}


def rel_l2(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def _small(seed=6):
    return configs.small(grid=(3, 4), cycles=8, mode="sparse", n_samples=64, n_slices=8, seed=seed)


def test_plan_memory_comes_from_torch_allocator(monkeypatch):
    """With the torch allocator every device block of the plan is torch-managed:
    torch.cuda.memory_allocated grows by the plan's device bytes and returns to its
    previous value when the context is destroyed."""
    for k, v in TC.items():
        monkeypatch.setenv(k, v)
    w = _small()
    torch.cuda.synchronize()
    base = torch.cuda.memory_allocated(0)
    c = Contraction(device=0, stream=torch.cuda.current_stream(), allocator="torch")
    c.setup(w.net, w.samples, w.path, w.sliced)
    held = torch.cuda.memory_allocated(0) - base
    assert held >= c.info()["device_bytes"] > 0, (held, c.info()["device_bytes"])
    c.contract(0, c.n_slices)
    got = c.sum_slices_host()
    c.close()
    torch.cuda.synchronize()
    assert torch.cuda.memory_allocated(0) == base
    assert rel_l2(got, oracle.contract(w.net, w.path, w.sliced, w.samples)) <= EXT_TOL
    # the cudaMalloc context gives the same amplitudes and no torch memory
    d = Contraction(device=0, stream=torch.cuda.current_stream(), allocator="cuda")
    d.setup(w.net, w.samples, w.path, w.sliced)
    assert torch.cuda.memory_allocated(0) == base
    d.contract(0, d.n_slices)
    assert rel_l2(d.sum_slices_host(), got) <= 1e-12
    d.close()


def test_failing_allocator_is_a_resource_error():
    """An allocator returning NULL makes planning fail with TN_ERR_RESOURCE, and the
    library returns every block it did obtain (alloc/free calls balance)."""
    w = _small()
    live = {}
    nxt = [0x10000]

    def alloc(nbytes, dev, stream, user):
        if len(live) >= 3:
            return None
        p = torch.cuda.caching_allocator_alloc(int(nbytes), device=int(dev), stream=int(stream or 0))
        live[p] = nbytes
        return p

    def free(ptr, nbytes, dev, stream, user):
        assert live.pop(ptr) == nbytes
        torch.cuda.caching_allocator_delete(ptr)

    a = tnlib.Allocator(tnlib.ALLOC_FN(alloc), tnlib.FREE_FN(free), None)
    L = tnlib.lib()
    h = C.c_void_p()
    assert L.tn_create(C.byref(h), 0, C.byref(a), C.c_void_p(torch.cuda.current_stream().cuda_stream)) == 0
    ranks, labels, dims, data, opens = w.net.flat()
    ranks = np.ascontiguousarray(ranks, np.int32)
    labels = np.ascontiguousarray(labels, np.int64)
    dims = np.ascontiguousarray(dims, np.int64)
    data = np.ascontiguousarray(np.asarray(data, np.complex128)).view(np.float64)
    opens = np.ascontiguousarray(opens, np.int64)
    smp = np.ascontiguousarray(w.samples, np.uint8)
    P = lambda x: x.ctypes.data_as(C.c_void_p)   # noqa: E731
    assert L.tn_load_network(h, len(ranks), P(ranks), P(labels), P(dims), P(data), len(opens), P(opens),
                             smp.shape[0], P(smp)) == 0
    pairs = np.ascontiguousarray(np.asarray(w.path, np.int32).reshape(-1, 2))
    assert L.tn_set_path(h, pairs.shape[0], P(pairs)) == 0
    sl = np.ascontiguousarray(np.asarray(list(w.sliced), np.int64))
    n = C.c_int64()
    st = L.tn_set_slices(h, len(sl), P(sl), C.byref(n))
    assert st == 3, (st, L.tn_last_error())
    assert b"allocator returned NULL" in L.tn_last_error()
    L.tn_destroy(h)
    assert live == {}


def test_reduce_amplitudes_on_a_non_current_stream(monkeypatch):
    """The context runs on its own (non-blocking) stream, not torch's current one:
    reduce_amplitudes must order allocation, gather and collective on that stream and
    hand a ready tensor to the caller's stream.  World 1 and a 1-rank NCCL group (the
    all_gather path) both equal tn_sum_slices_host and the oracle."""
    import torch.distributed as dist
    for k, v in TC.items():
        monkeypatch.setenv(k, v)
    w = _small(7)
    ref = oracle.contract(w.net, w.path, w.sliced, w.samples)
    side = torch.cuda.Stream()
    c = Contraction(device=0, stream=side)
    c.setup(w.net, w.samples, w.path, w.sliced)
    host = None
    for rep in range(3):                       # repeated: a race would show up as a mismatch
        c.reset_accumulator()
        c.contract(0, c.n_slices)
        out = reduce_amplitudes(c, 1)
        got = out.cpu().numpy()                 # on the current stream, after the wait
        host = c.sum_slices_host()
        assert np.array_equal(got, host), rep
    assert rel_l2(host, ref) <= EXT_TOL
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        for det in (True, False):
            out = contract_partitioned(c, 1, 0, deterministic=det)
            assert np.array_equal(out.cpu().numpy(), host)
    finally:
        dist.destroy_process_group()
    c.close()


def test_upload_after_large_shrink_restarts_delayed_scaling(monkeypatch):
    """after tensors 2^-20 smaller are uploaded, a stale delayed-scaling
    history would put the fused fp16 planes' exponent ~20 too low (lo plane, then hi,
    in subnormals).  A >2x change of any leaf's absmax restarts the history, so the
    result scales exactly; changes within 2x keep the history and the CUDA graph."""
    for k, v in TC.items():
        monkeypatch.setenv(k, v)
    w = _small(6)
    ref = oracle.contract(w.net, w.path, w.sliced, w.samples)
    c = Contraction(device=0, stream=torch.cuda.current_stream())
    c.setup(w.net, w.samples, w.path, w.sliced)
    assert any(s["planes_out"] for s in c.plan_json()["steps"])
    for t in range(c.n_slices):
        c.contract(t, t + 1)
    assert rel_l2(c.sum_slices_host(), ref) <= EXT_TOL
    _, _, _, data, _ = w.net.flat()
    size0 = int(np.prod([w.net.dims[x] for x in w.net.labels[0]]))
    for f, kept in ((1.0, True), (0.75, True), (2.0 ** -20, False), (1.0, False), (2.0 ** 20, False)):
        d2 = data.copy()
        d2[:size0] *= f
        c.upload_tensors(d2)
        c.reset_accumulator()
        r0 = c.info()["graph_replays"]
        for t in range(c.n_slices):
            c.contract(t, t + 1)
        replays = c.info()["graph_replays"] - r0
        assert replays == (c.n_slices if kept else c.n_slices - 1), (f, replays)
        assert not c.overflow()
        assert rel_l2(c.sum_slices_host(), ref * f) <= EXT_TOL, f
    c.close()


def test_sum_slices_device_is_asynchronous_and_flags_overflow(monkeypatch):
    """tn_sum_slices no longer synchronises; its result (device buffer) equals the
    host variant.  tn_last_overflow reports no saturation on a normal run."""
    for k, v in TC.items():
        monkeypatch.setenv(k, v)
    w = _small(8)
    c = Contraction(device=0, stream=torch.cuda.current_stream())
    c.setup(w.net, w.samples, w.path, w.sliced)
    c.contract(0, c.n_slices)
    out = torch.empty(c.n_out, dtype=torch.complex128, device="cuda")
    c.sum_slices(out)
    assert np.array_equal(out.cpu().numpy(), c.sum_slices_host())
    assert c.overflow() is False
    c.close()
