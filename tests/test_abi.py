"""CPU tests of the C-ABI library: it loads, exports every symbol include/tn.h
declares, and its host-side planner (path replay, Eq. 3 set rule, Eq. 4/5
bookkeeping, Eq. 7 merge tables, slice validation) agrees bit-exactly with the
oracle's independent derivation.  No GPU needed (host-only context, device -1)."""
import os
import re

import numpy as np
import pytest

import oracle
from tnworkloads import configs, grid_layout, random_circuit, circuit_to_network, greedy_path
from tnworkloads.paths import slice_greedy
from paper_2310_03978_b200 import tn as tnlib
from paper_2310_03978_b200 import Contraction, TNError

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "tn.h")).read()
    return sorted(set(re.findall(r"^TN_API\s+[\w\s\*]+?\b(tn_\w+)\s*\(", src, flags=re.M)))


def test_library_exports_every_declared_symbol():
    L = tnlib.lib()
    declared = header_symbols()
    assert len(declared) >= 15
    for s in declared:
        assert hasattr(L, s), s
    assert sorted(tnlib.SYMBOLS) == declared
    assert b"sm_100a" in L.tn_version()


def _check_plan(w):
    c = Contraction(device=-1)
    ns = c.setup(w.net, w.samples, w.path, w.sliced)
    assert ns == w.n_slices
    pj = c.plan_json()
    bk = oracle.plan_bookkeeping(w.net, w.path, w.sliced, w.samples)
    assert len(pj["steps"]) == len(bk)
    for a, b in zip(pj["steps"], bk):
        for key in ["i", "j", "J", "m", "n", "k", "tcc", "tmc"]:
            assert a[key] == b[key], (key, a, b)
        assert a["ia"] == b["ia"] and a["ib"] == b["ib"]
    info = c.info()
    assert info["flops_per_slice"] == sum(r["tcc"] for r in bk)
    return c, pj


@pytest.mark.parametrize("mode", ["sparse", "full", "single", "subspace"])
@pytest.mark.parametrize("seed", [0, 1])
def test_plan_bookkeeping_matches_oracle(mode, seed):
    w = configs.small(grid=(3, 3), cycles=6, mode=mode, n_samples=24, n_slices=4, seed=seed)
    _check_plan(w)


def test_plan_bookkeeping_raw_network_and_output_positions():
    w = configs.small(grid=(2, 4), cycles=5, mode="sparse", n_samples=40, n_slices=2, seed=3,
                      simplify=False)
    c, pj = _check_plan(w)
    # a9: root table is sorted unique samples; out_pos maps caller order onto it
    s = w.samples.astype(np.int64)
    packed = (s << (s.shape[1] - 1 - np.arange(s.shape[1]))[None, :]).sum(1)
    uniq = np.unique(packed)
    assert pj["out_pos"] == [int(np.searchsorted(uniq, v)) for v in packed]


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_grouped_merge_tables(seed, monkeypatch):
    """Slab-grouped merges: the gathered rows of every
    grouped step cover each output row (j, q) exactly once, padding rows are -1, and
    every 128-row block reads a single X slab, the one Eq. 7's table gives its j."""
    for k, v in {"TN_TC_MIN_BIG": "2", "TN_TC_MIN_SMALL": "1", "TN_TC_MIN_K": "2",
                 "TN_GROUP": "2"}.items():
        monkeypatch.setenv(k, v)
    w = configs.small(grid=(3, 4), cycles=8, mode="sparse", n_samples=64, n_slices=8, seed=seed)
    c, pj = _check_plan(w)
    grouped = [s for s in pj["steps"] if s["grouped"]]
    assert grouped
    for s in grouped:
        Q = s["n"] if s["swap"] else s["m"]          # Y = tensor-core M side
        sx = s["ia"] if s["swap"] else s["ib"]       # X slab of each merged config j
        rm, blk = np.array(s["g_rowmap"]), np.array(s["g_blk"])
        assert len(rm) == s["gathered_rows"] and len(rm) % 128 == 0 and len(blk) == len(rm) // 128
        real = rm[rm >= 0]
        assert np.array_equal(np.sort(real), np.arange(s["J"] * Q))
        r = np.nonzero(rm >= 0)[0]
        assert np.array_equal(np.array(sx)[rm[r] // Q], blk[r // 128])


def test_c2_plan_matches_oracle_bookkeeping():
    w = configs.c2()
    c, pj = _check_plan(w)
    assert c.info()["n_slices"] == 64
    assert c.info()["n_out"] == 1024


def test_c5_m20_plan_matches_oracle_bookkeeping():
    """C5 (m=20, 430 fsim tensors): the cached order's plan at full size, bit-exact."""
    w = configs.c5()
    c, pj = _check_plan(w)
    assert len(pj["steps"]) == len(w.net.labels) - 1
    assert pj["peak_elements"] <= 2.0 ** 32


def test_error_codes():
    w = configs.small(grid=(2, 3), cycles=4, mode="sparse", n_samples=8, n_slices=1, seed=5)
    ranks, labels, dims, data, opens = w.net.flat()
    c = Contraction(device=-1)
    with pytest.raises(TNError) as e:
        c.set_path(w.path)                       # wrong call order
    assert e.value.status == 1
    c.load_network(ranks, labels, dims, data, opens, w.samples)
    bad = list(w.path)
    bad[1] = (bad[0][1], bad[1][1])              # references a retired id
    with pytest.raises(TNError) as e:
        c.set_path(bad)
    assert e.value.status == 2
    with pytest.raises(TNError) as e:
        c.set_path(w.path[:-1])                  # not N-1 steps
    assert e.value.status == 2
    c.set_path(w.path)
    with pytest.raises(TNError) as e:
        c.set_slices([opens[0]])                 # open bond cannot be sliced
    assert e.value.status == 2
    closed = [x for x in labels if x not in set(opens)]
    with pytest.raises(TNError) as e:
        c.set_slices([closed[0], closed[0]])     # repeated
    assert e.value.status == 2
    with pytest.raises(TNError) as e:
        c.set_slices([10 ** 9])                  # unknown
    assert e.value.status == 2
    assert c.set_slices([closed[0]]) == 2
    with pytest.raises(TNError) as e:
        c.contract(0, 1)                         # host-only context cannot execute
    assert e.value.status == 1
    # malformed networks
    c2 = Contraction(device=-1)
    lab2 = labels.copy()
    lab2[0] = lab2[1] if ranks[0] > 1 else lab2[0]
    if ranks[0] > 1:
        with pytest.raises(TNError) as e:        # label repeated inside a tensor
            c2.load_network(ranks, lab2, dims, data, opens, w.samples)
        assert e.value.status == 2
    smp = w.samples.copy()
    smp[0, 0] = 2
    with pytest.raises(TNError) as e:
        c2.load_network(ranks, labels, dims, data, opens, smp)
    assert e.value.status == 2


def test_create_rejects_incomplete_allocator():
    """tn_create validates the tn_allocator (SURVEY.md §8 b) before touching a device:
    an allocator without a free callback is a usage error."""
    import ctypes as C
    L = tnlib.lib()
    h = C.c_void_p()
    half = tnlib.Allocator(tnlib.ALLOC_FN(lambda n, d, s, u: None), tnlib.FREE_FN(), None)
    assert L.tn_create(C.byref(h), -1, C.byref(half), None) == 1
    assert b"alloc and free" in L.tn_last_error()
    full = tnlib.Allocator(tnlib.ALLOC_FN(lambda n, d, s, u: None),
                           tnlib.FREE_FN(lambda p, n, d, s, u: None), None)
    assert L.tn_create(C.byref(h), -1, C.byref(full), None) == 0
    L.tn_destroy(h)
    assert L.tn_last_overflow(None) == -1


@pytest.mark.parametrize("topk", [1, 3, 10, 1000])
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_paper_reorder_selection_matches_oracle(topk, seed, monkeypatch):
    """f3: the library's TN_REORDER=1 pass (§4.1 top-k rule) selects and marks
    exactly the steps the oracle's plain implementation of the rule does, on T_cc the
    oracle re-derives itself (Eq. 4)."""
    from oracle.reorder import paper_topk_reorder
    monkeypatch.setenv("TN_REORDER", "1")
    monkeypatch.setenv("TN_REORDER_TOPK", str(topk))
    w = configs.small(grid=(3, 4), cycles=8, mode=["sparse", "single", "full"][seed], n_samples=64,
                      n_slices=4, seed=seed)
    c, pj = _check_plan(w)
    bk = oracle.plan_bookkeeping(w.net, w.path, w.sliced, w.samples)
    sel, mod = paper_topk_reorder(w.path, len(w.net.labels), [r["tcc"] for r in bk], topk)
    assert pj["reorder"]["mode"] == 1
    assert pj["reorder"]["selected"] == sel and pj["reorder"]["modified"] == mod
    assert sel, "the rule selects at least the top contraction"


def test_paper_reorder_selection_c4(monkeypatch):
    from oracle.reorder import paper_topk_reorder
    monkeypatch.setenv("TN_REORDER", "1")
    w = configs.c4("single", 32, "a64")
    c = Contraction(device=-1)
    c.setup(w.net, w.samples, w.path, w.sliced)
    pj = c.plan_json()
    tcc = [s["tcc"] for s in pj["steps"]]
    sel, mod = paper_topk_reorder(w.path, len(w.net.labels), tcc, 10)
    assert pj["reorder"]["selected"] == sel and pj["reorder"]["modified"] == mod
    # the reordered producers are exactly the associated contractions: only they write
    # the consumer's order (out_gen); in mode 0 no producer does
    assert 1 <= len(sel) <= 10


def test_reorder_modes_change_layout_not_bookkeeping(monkeypatch):
    w = configs.small(grid=(3, 4), cycles=8, mode="sparse", n_samples=64, n_slices=4, seed=0)
    for k, v in {"TN_TC_MIN_BIG": "8", "TN_TC_MIN_SMALL": "2", "TN_TC_MIN_K": "2"}.items():
        monkeypatch.setenv(k, v)
    gens = {}
    for mode in (0, 1, 2):
        monkeypatch.setenv("TN_REORDER", str(mode))
        c, pj = _check_plan(w)
        gens[mode] = sum(1 for s in pj["steps"] if s["out_gen"])
    assert gens[0] == 0 and gens[0] <= gens[1] <= gens[2] and gens[2] > 0


def test_skinny_chains_c4_sparse(monkeypatch):
    """Fused skinny chains on the headline plan: stem chains are found
    (263 -> 264 -> 266 among them); every member is a skinny (mode 1)
    SIMT step whose big operand is the previous member's output; only the last member of a
    chain is launched (the others are marked chained)."""
    w = configs.c4("sparse16", 32)
    monkeypatch.setenv("TN_CHAIN_MIN_SAVE_LOG2", "0")    # every eligible chain
    c = Contraction(device=-1)
    c.setup(w.net, w.samples, w.path, w.sliced)
    steps = c.plan_json()["steps"]
    runs = {}
    for i, s in enumerate(steps):
        if s["chain"] >= 0:
            runs.setdefault(s["chain"], []).append(i)
    assert [263, 264, 266] in runs.values(), runs
    assert any(283 in r for r in runs.values()), runs
    assert len(runs) >= 5
    for run in runs.values():
        assert len(run) >= 2
        assert [steps[t]["chained"] for t in run] == [True] * (len(run) - 1) + [False]
        for a, b in zip(run, run[1:]):
            assert a in (_producer(steps, b, steps[b]["i"]), _producer(steps, b, steps[b]["j"]))
        for t in run:
            assert steps[t]["route"] == "simt" and steps[t]["mode"] == 1 and not steps[t]["folded"]


def _producer(steps, s, tid):
    """Step that produced live tensor id `tid` before step s (stable ids: result keeps i)."""
    for q in range(s - 1, -1, -1):
        if steps[q]["i"] == tid:
            return q
    return -1


def test_skinny_chains_off_keeps_bookkeeping(monkeypatch):
    w = configs.c4("sparse16", 32)
    monkeypatch.setenv("TN_CHAIN", "0")
    c0 = Contraction(device=-1)
    c0.setup(w.net, w.samples, w.path, w.sliced)
    s0 = c0.plan_json()["steps"]
    monkeypatch.setenv("TN_CHAIN", "1")
    c1 = Contraction(device=-1)
    c1.setup(w.net, w.samples, w.path, w.sliced)
    s1 = c1.plan_json()["steps"]
    assert not any(s["chain"] >= 0 or s["chained"] for s in s0)
    assert any(s["chained"] for s in s1)
    for a, b in zip(s0, s1):
        for key in ["i", "j", "J", "m", "n", "k", "tcc", "tmc", "route", "mode"]:
            assert a[key] == b[key]
