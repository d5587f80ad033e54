"""Pins for the CPU oracle (``-m "not gpu"``): the oracle is checked against
things other than itself — closed forms, a brute-force state vector, invariants
and the paper's worked Eq. 7 example — so that a dropped term, wrong sign,
wrong index or transposed operand anywhere in it fails at least one test."""
import json
import os

import numpy as np
import pytest

import oracle
from oracle.contract import _contract_pair, _Tensor
from tnworkloads import (random_circuit, grid_layout, circuit_to_network, gate_matrix,
                         uniform_samples, single_amplitude, subspace_samples, greedy_path)
from tnworkloads.circuits import Gate, Circuit, fsim, PAULI
from tnworkloads.paths import slice_greedy, bisection_path
from tnworkloads.samples import all_bitstrings
from tnworkloads import configs

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# ----------------------------------------------------------------------------- gates (closed forms)

@pytest.mark.parametrize("k,p", [("sx", "x"), ("sy", "y"), ("sw", "w")])
def test_sqrt_gates_square_to_pauli(k, p):
    g = gate_matrix(Gate(k, (0,)))
    assert np.allclose(g @ g, PAULI[p], atol=1e-15)
    assert np.allclose(g @ g.conj().T, np.eye(2), atol=1e-15)


def test_sqrtx_matrix_spec_l72():
    g = gate_matrix(Gate("sx", (0,)))
    assert np.allclose(g, 0.5 * np.array([[1 + 1j, 1 - 1j], [1 - 1j, 1 + 1j]]))


def test_fsim_pi2_0_maps_01_to_minus_i_10():
    u = fsim(np.pi / 2, 0.0)
    v = np.zeros(4, complex)
    v[0b01] = 1
    out = u @ v
    assert np.allclose(out, -1j * np.eye(4)[0b10])
    assert np.allclose(fsim(0, 0), np.eye(4))


# ----------------------------------------------------------------------------- state vector (textbook)

def test_statevector_small_cases():
    c = Circuit(1, [[Gate("sx", (0,))]])
    psi = oracle.statevector(c, gate_matrix)
    assert np.allclose(psi, [(1 + 1j) / 2, (1 - 1j) / 2])
    c = Circuit(2, [])
    assert np.allclose(oracle.statevector(c, gate_matrix), [1, 0, 0, 0])
    # |01> via X on qubit 1 (built from sqrt X twice), then fsim(pi/2,0) -> -i|10>
    c = Circuit(2, [[Gate("sx", (1,))], [Gate("sx", (1,))], [Gate("fsim", (0, 1), (np.pi / 2, 0.0))]])
    assert np.allclose(oracle.statevector(c, gate_matrix), [0, 0, -1j, 0])


def test_bit_order_qubit0_is_msb():
    c = Circuit(3, [[Gate("sx", (0,))], [Gate("sx", (0,))]])   # X on qubit 0
    psi = oracle.statevector(c, gate_matrix)
    assert abs(psi[0b100]) == pytest.approx(1.0)


# ----------------------------------------------------------------------------- oracle vs state vector

@pytest.mark.parametrize("rows,cols,cyc,seed", [(2, 2, 3, 0), (2, 3, 5, 1), (3, 3, 6, 2), (3, 4, 8, 3)])
@pytest.mark.parametrize("simplify", [True, False])
def test_oracle_full_state_matches_statevector(rows, cols, cyc, seed, simplify):
    c = random_circuit(grid_layout(rows, cols), cyc, seed=seed)
    net = circuit_to_network(c, simplify=simplify)
    path, _ = greedy_path(net, None, seed=seed)
    amps = oracle.contract(net, path, (), None)
    psi = oracle.statevector(c, gate_matrix)
    assert np.abs(amps - psi).max() < 1e-12
    assert np.sum(np.abs(amps) ** 2) == pytest.approx(1.0, abs=1e-12)


@pytest.mark.parametrize("mode", ["sparse", "single", "subspace"])
def test_oracle_sparse_state_matches_statevector(mode):
    n = 9
    c = random_circuit(grid_layout(3, 3), 6, seed=11)
    net = circuit_to_network(c)
    if mode == "sparse":
        smp = uniform_samples(n, 24, seed=5)
        smp[3] = smp[7]                     # duplicates are re-expanded on output
    elif mode == "single":
        smp = single_amplitude(n, seed=6)
    else:
        smp = subspace_samples(n, [5, 6, 7, 8], seed=7)
    path, _ = greedy_path(net, smp, seed=3)
    sl, _ = slice_greedy(net, smp, path, n_slices=4)
    amps = oracle.contract(net, path, sl, smp)
    ref = oracle.amplitudes_for(oracle.statevector(c, gate_matrix), smp)
    assert np.abs(amps - ref).max() < 1e-12


def test_path_independence_and_slicing_identity():
    c = random_circuit(grid_layout(3, 3), 7, seed=21)
    net = circuit_to_network(c)
    smp = uniform_samples(9, 32, seed=22)
    p1, _ = greedy_path(net, smp, seed=0)
    p2 = bisection_path(net, smp, seed=1, leaf_size=4)
    a1 = oracle.contract(net, p1, (), smp)
    a2 = oracle.contract(net, p2, (), smp)
    assert np.abs(a1 - a2).max() < 1e-12
    sl, _ = slice_greedy(net, smp, p1, n_slices=8)
    parts = [oracle.contract_slice(net, p1, sl, t, smp) for t in range(8)]
    assert np.abs(np.sum(parts, axis=0) - a1).max() < 1e-12
    # each slice on its own is not the full answer (slicing really fixes bonds)
    assert np.abs(parts[0] - a1).max() > 1e-6


def test_sparse_equals_dense_then_pick():
    c = random_circuit(grid_layout(2, 4), 6, seed=31)
    net = circuit_to_network(c)
    smp = uniform_samples(8, 20, seed=32)
    pd, _ = greedy_path(net, None, seed=1)
    dense = oracle.contract(net, pd, (), None)
    ps, _ = greedy_path(net, smp, seed=2)
    sparse = oracle.contract(net, ps, (), smp)
    idx = (smp.astype(np.int64) << (7 - np.arange(8))[None, :]).sum(1)
    assert np.abs(sparse - dense[idx]).max() < 1e-12


# ----------------------------------------------------------------------------- exact width pins

def test_echo_circuit_exact():
    w = configs.echo(grid_layout(3, 4), 4, seed=41, mode="sparse", n_samples=16, n_slices=4)
    amps = oracle.contract(w.net, w.path, w.sliced, w.samples)
    is0 = ~w.samples.any(axis=1)
    assert np.abs(amps[is0] - 1).max() < 1e-12
    assert np.abs(amps[~is0]).max() < 1e-12


def test_clifford_probabilities_are_dyadic():
    c = random_circuit(grid_layout(3, 3), 5, seed=51, theta=np.pi / 2, phi=0.0,
                       one_qubit=("sx", "sy"))
    net = circuit_to_network(c)
    path, _ = greedy_path(net, None, seed=0)
    p = np.abs(oracle.contract(net, path, (), None)) ** 2
    nz = p[p > 1e-9]
    k = np.log2(1 / nz)
    assert np.allclose(k, np.round(k), atol=1e-9)
    assert len(set(np.round(k))) == 1          # stabilizer state: uniform on its support
    assert np.sum(p) == pytest.approx(1.0, abs=1e-12)


# ----------------------------------------------------------------------------- Eq. 7 worked example

def test_eq7_fig1c_merge_table():
    g = json.load(open(os.path.join(GOLDEN, "eq7_fig1c.json")))
    smp = np.array([[int(ch) for ch in s] for s in g["samples"]], np.uint8)
    q, table, ia, ib = oracle.merge_table(smp, [g["c_qubit"]], [g["e_qubit"]])
    assert ["".join(map(str, r)) for r in table] == g["expected_merged_configs"]
    ta = oracle.unique_projection(smp, [g["c_qubit"]])
    tb = oracle.unique_projection(smp, [g["e_qubit"]])
    assert [int(ta[i][0]) for i in ia] == g["expected_c_values"]
    assert [int(tb[i][0]) for i in ib] == g["expected_e_values"]


def test_eq7_fig1c_values():
    """L_fab = concat(Σ_d F[c=0,a,b,d] H[e=0,d], Σ_d F[c=0,a,b,d] H[e=1,d])."""
    g = json.load(open(os.path.join(GOLDEN, "eq7_fig1c.json")))
    smp = np.array([[int(ch) for ch in s] for s in g["samples"]], np.uint8)
    rng = np.random.default_rng(0)
    F = rng.normal(size=(2, 2, 3, 2)) + 1j * rng.normal(size=(2, 2, 3, 2))   # (c, a, b, d)
    H = rng.normal(size=(2, 2)) + 1j * rng.normal(size=(2, 2))               # (e, d)
    # group tables of the single open legs: c = qubit 1 takes {0}, e = qubit 2 takes {0,1}
    tc = oracle.unique_projection(smp, [1])
    te = oracle.unique_projection(smp, [2])
    A = _Tensor(F[tc[:, 0]], ["a", "b", "d"], [1], tc)
    B = _Tensor(H[te[:, 0]], ["d"], [2], te)
    L = _contract_pair(A, B, smp)
    expect = np.stack([np.einsum("abd,d->ab", F[0], H[0]), np.einsum("abd,d->ab", F[0], H[1])])
    assert L.group == [1, 2]
    assert L.labels == ["a", "b"]
    assert np.abs(L.data - expect).max() < 1e-14


# ----------------------------------------------------------------------------- bookkeeping

def test_slice_digits_mixed_radix():
    assert oracle.slice_digits(3, [2, 2]) == [1, 1]
    assert oracle.slice_digits(0, [2]) == [0]
    assert oracle.slice_digits(5, [2, 3]) == [1, 2]      # 5 = 1*3 + 2, last fastest
    assert oracle.slice_digits(1, [3, 2]) == [0, 1]
    with pytest.raises(ValueError):
        oracle.slice_digits(4, [2, 2])


def _naive_step(A, la, B, lb, dims):
    """Explicit nested-loop einsum that counts complex multiplications."""
    K = [x for x in la if x in lb]
    out = [x for x in la if x not in K] + [x for x in lb if x not in K]
    allx = out + K
    C = np.zeros([dims[x] for x in out], complex)
    count = 0
    for idx in np.ndindex(*[dims[x] for x in allx]):
        v = dict(zip(allx, idx))
        C[tuple(v[x] for x in out)] += A[tuple(v[x] for x in la)] * B[tuple(v[x] for x in lb)]
        count += 1
    return C, count


def test_tcc_equals_instrumented_mac_count():
    c = random_circuit(grid_layout(2, 3), 3, seed=61)
    net = circuit_to_network(c)
    smp = single_amplitude(6, bits=[0] * 6)
    # close the network: contract pairs with the naive loop and count MACs
    path, _ = greedy_path(net, smp, seed=0)
    bk = oracle.plan_bookkeeping(net, path, (), smp)
    # leaves with open legs restricted to the (single) sample value -> dense closed tensors
    T = {}
    qubit_of = {l: q for q, l in enumerate(net.open_labels)}
    for t, (d, ls) in enumerate(zip(net.tensors, net.labels)):
        for x in [x for x in ls if x in qubit_of]:
            ax = ls.index(x)
            d = np.take(d, smp[0][qubit_of[x]], axis=ax)
            ls = [y for y in ls if y != x]
        T[t] = (d, list(ls))
    total = 0
    for (i, j), rec in zip(path, bk):
        (A, la), (B, lb) = T[i], T[j]
        C, cnt = _naive_step(A, la, B, lb, net.dims)
        assert rec["tcc"] == 8 * cnt
        total += cnt
        K = [x for x in la if x in lb]
        T[i] = (C, [x for x in la if x not in K] + [x for x in lb if x not in K])
        del T[j]
    (root, _), = T.values()
    ref = oracle.amplitudes_for(oracle.statevector(c, gate_matrix), smp)
    assert abs(complex(root) - ref[0]) < 1e-12
    assert sum(r["tcc"] for r in bk) == 8 * total


def test_tcc_tmc_spec_example():
    """C_mn = Σ_k A_mk B_kn, all dims 4, complex64 -> T_cc 512, T_mc 384."""
    from tnworkloads.network import Network
    net = Network([np.zeros((4, 4), complex), np.zeros((4, 4), complex)], [[0, 1], [1, 2]],
                  {0: 4, 1: 4, 2: 4}, [], 0)
    net.labels = [[0, 1], [1, 2]]
    # treat 0 and 2 as free (uncontracted) labels of a 2-tensor network
    bk = oracle.plan_bookkeeping(net, [(0, 1)], (), np.zeros((1, 0), np.uint8))
    assert bk[0]["tcc"] == 512 and bk[0]["tmc"] == 384


def _naive_sparse_pass(net, path, samples):
    """Sparse-state contraction written as plain loops (independent of the oracle's
    Eq. 7 code): a live tensor is a dict {open-leg configuration: dense array over its
    closed labels}, with the configurations that actually occur in the samples
    (only sampled bitstrings are kept).  A step loops over the
    output configurations and over every (free A, free B, contracted) index tuple,
    counting one complex multiply-add per innermost iteration.  Returns the per-step
    records (configs, MAC count, stored sizes, A/B config of each output config) and
    the amplitudes of the samples."""
    qubit_of = {l: q for q, l in enumerate(net.open_labels)}
    rows = [tuple(int(b) for b in s) for s in samples]
    live = {}
    for t, (d, ls) in enumerate(zip(net.tensors, net.labels)):
        opens = sorted([x for x in ls if x in qubit_of], key=lambda x: qubit_of[x])
        closed = [x for x in ls if x not in qubit_of]
        qs = [qubit_of[x] for x in opens]
        cfgs = sorted({tuple(r[q] for q in qs) for r in rows})
        table = {}
        for cf in cfgs:
            sub = d
            for x, bit in sorted(zip(opens, cf), key=lambda p: -ls.index(p[0])):
                sub = np.take(sub, bit, axis=ls.index(x))
            table[cf] = sub.reshape([net.dims[x] for x in closed])
        live[t] = (qs, closed, table)
    recs = []
    for i, j in path:
        qa, la, ta = live[i]
        qb, lb, tb = live[j]
        K = [x for x in la if x in lb]
        fa = [x for x in la if x not in K]
        fb = [x for x in lb if x not in K]
        out_l = fa + fb
        q = sorted(qa + qb)
        cfgs = sorted({tuple(r[x] for x in q) for r in rows})
        sa, sb = sorted(ta), sorted(tb)
        res, macs, ia, ib = {}, 0, [], []
        for cf in cfgs:
            ca = tuple(cf[q.index(x)] for x in qa)
            cb = tuple(cf[q.index(x)] for x in qb)
            ia.append(sa.index(ca))
            ib.append(sb.index(cb))
            A, B = ta[ca], tb[cb]
            C = np.zeros([net.dims[x] for x in out_l], complex)
            for idx in np.ndindex(*[net.dims[x] for x in out_l + K]):
                v = dict(zip(out_l + K, idx))
                C[tuple(v[x] for x in out_l)] += A[tuple(v[x] for x in la)] * B[tuple(v[x] for x in lb)]
                macs += 1
            res[cf] = C
        size = lambda tab, ls_: len(tab) * int(np.prod([net.dims[x] for x in ls_]))   # noqa: E731
        recs.append({"configs": len(cfgs), "merge": bool(qa) and bool(qb), "macs": macs,
                     "sizes": (size(ta, la), size(tb, lb), size(res, out_l)), "ia": ia, "ib": ib})
        live[i] = (q, out_l, res)
        del live[j]
    (q, ls, tab), = live.values()
    amps = np.array([complex(tab[tuple(r[x] for x in q)]) for r in rows])
    return recs, amps


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_sparse_merge_bookkeeping_equals_naive_loop_count(seed):
    """Round-1 gap: plan_bookkeeping's sparse-merge branch (J > 1: T_cc, T_mc and the
    Eq. 7 gather tables) pinned against an instrumented loop over the sampled
    configurations, whose amplitudes are themselves pinned by the state vector."""
    c = random_circuit(grid_layout(2, 3), 4, seed=70 + seed)
    net = circuit_to_network(c)
    smp = uniform_samples(6, 12, seed=80 + seed)
    path, _ = greedy_path(net, smp, seed=seed)
    bk = oracle.plan_bookkeeping(net, path, (), smp)
    recs, amps = _naive_sparse_pass(net, path, smp)
    ref = oracle.amplitudes_for(oracle.statevector(c, gate_matrix), smp)
    assert np.abs(amps - ref).max() < 1e-12
    n_merge = 0
    for rec, nv in zip(bk, recs):
        assert rec["tcc"] == 8 * nv["macs"]
        assert rec["tmc"] == 8 * sum(nv["sizes"])
        if nv["merge"]:
            n_merge += rec["J"] > 1
            assert rec["J"] == nv["configs"]
            assert rec["ia"] == nv["ia"] and rec["ib"] == nv["ib"]
    assert n_merge >= 2, n_merge          # the J > 1 branch is exercised
    assert oracle.plan_bookkeeping(net, path, (), smp)[-1]["J"] == len(np.unique(smp, axis=0))


# ----------------------------------------------------------------------------- §4.1 reorder rule (f3)
# Hand-worked cases of the Fig. 3 rule on the Fig. 1(b)-shaped tree
# M = einsum(I, J) [s0], N = einsum(K, L) [s1], O = einsum(M, N) [s2], final (O, P) [s3];
# expected sets derived by hand from the four steps of the rule, not by running it.
_FIG1B_PATH = [(0, 1), (2, 3), (0, 2), (0, 4)]


def test_reorder_producers_follow_stable_ids():
    from oracle.reorder import producers
    assert producers(_FIG1B_PATH, 5) == [(None, None), (None, None), (0, 1), (2, None)]


@pytest.mark.parametrize("tcc,k,selected,modified", [
    # O ranks first: O and its associated M, N are reordered; the final step's associated
    # contraction O is modified -> skipped; M and N are modified -> skipped
    ([10, 20, 100, 50], 4, [2], [0, 1, 2]),
    # N first (leaf inputs only); O's associated N is modified -> skipped; the final step's
    # associated O is untouched -> reordered (O modified); M has leaf inputs -> reordered
    ([10, 200, 100, 50], 4, [0, 1, 3], [0, 1, 2, 3]),
    # top-2 group {N, O}: only N
    ([10, 200, 100, 50], 2, [1], [1]),
    # equal T_cc: earlier step first (reading R18): s0, s1, then s2 blocked, s3 reordered
    ([5, 5, 5, 5], 4, [0, 1, 3], [0, 1, 2, 3]),
    # k = 0: nothing
    ([10, 20, 100, 50], 0, [], []),
])
def test_reorder_rule_hand_worked(tcc, k, selected, modified):
    from oracle.reorder import paper_topk_reorder
    assert paper_topk_reorder(_FIG1B_PATH, 5, tcc, k) == (selected, modified)


def test_reorder_rule_chain_blocks_consumers_of_reordered_steps():
    # chain X=(0,1) s0, Y=(0,2) s1, Z=(0,3) s2: Y ranks first -> Y, X modified; Z's
    # associated Y is modified -> skipped; X is modified -> skipped
    from oracle.reorder import paper_topk_reorder
    assert paper_topk_reorder([(0, 1), (0, 2), (0, 3)], 4, [1, 9, 5], 3) == ([1], [0, 1])
    # Z first -> Z, Y modified; then Y skipped; X: its inputs are leaves -> reordered
    assert paper_topk_reorder([(0, 1), (0, 2), (0, 3)], 4, [1, 5, 9], 3) == ([0, 2], [0, 1, 2])
