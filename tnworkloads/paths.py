"""Contraction-path and slice-set *generators* (workload tooling, not the method).

The path is an input of the hot path (BASELINE.json north_star: "executing a
given contraction path"); PAPER.md's own path finder (SA, §3.2) and
dynamic slicing (L296) are out of scope (SURVEY.md §8 f).  These heuristics
only manufacture reasonable synthetic workloads:

* ``greedy_path``     — randomised greedy on "size(out) - size(A) - size(B)".
* ``bisection_path``  — recursive Kernighan-Lin bisection (networkx) with a
                         greedy finish inside small parts (the graph-partitioning
                         family cited at L112/L270).
* ``slice_greedy``    — pick bonds to slice (L292-295) greedily by total cost.

Path format (L259-262): a list of N-1 pairs (i, j) of *stable* tensor ids; the
result of each step "is indexed by the first tensor" i, and j retires.

Size model: all closed labels carry their dims; the open legs of a tensor form
one merged group whose extent is U(Q) = number of distinct projections of the
samples onto the group's qubits (full state: 2^|Q|).  Cost per step follows
Eq. 4 (L232-237): 8 * prod(dims of A) * prod(dims of B) / prod(contracted),
with the merged sample dimension J replacing the product of the two open
groups for a sparse merge.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np


class SampleModel:
    """U(Q): distinct projections of the sample set onto a qubit set."""

    def __init__(self, n_qubits: int, samples):
        self.n = n_qubits
        self.samples = samples
        self.cache = {}
        if samples is not None:
            s = np.asarray(samples, dtype=np.uint64)
            w = (np.uint64(1) << np.arange(n_qubits - 1, -1, -1, dtype=np.uint64))
            self.packed = (s * w[None, :]).sum(axis=1, dtype=np.uint64) if n_qubits <= 64 else None

    def log2U(self, qubits: frozenset) -> float:
        if not qubits:
            return 0.0
        if self.samples is None:
            return float(len(qubits))
        key = qubits
        v = self.cache.get(key)
        if v is None:
            mask = np.uint64(0)
            for q in qubits:
                mask |= np.uint64(1) << np.uint64(self.n - 1 - q)
            u = np.unique(self.packed & mask).size
            v = math.log2(u)
            self.cache[key] = v
        return v


@dataclass
class StepInfo:
    i: int
    j: int
    J: float          # merged sample extent (1 if no sparse merge)
    m: float
    n: float
    k: float
    flops: float      # Eq. 4 with ops_per_element = 8
    out_log2: float   # log2 elements of the result


@dataclass
class PathCost:
    steps: list = field(default_factory=list)
    flops_per_slice: float = 0.0
    peak_log2: float = 0.0
    n_slices: int = 1

    @property
    def total_flops(self):
        return self.flops_per_slice * self.n_slices


def _leaf_state(net, sliced=frozenset()):
    qubit_of = {lab: q for q, lab in enumerate(net.open_labels)}
    st = {}
    for t, ls in enumerate(net.labels):
        L = frozenset(x for x in ls if x not in qubit_of and x not in sliced)
        Q = frozenset(qubit_of[x] for x in ls if x in qubit_of)
        st[t] = (L, Q)
    return st


def _lsize(L, dims):
    return sum(math.log2(dims[x]) for x in L)


def _step(a, b, dims, sm):
    (LA, QA), (LB, QB) = a, b
    K = LA & LB
    out = (LA | LB) - K
    Q = QA | QB
    lk = _lsize(K, dims)
    lm = _lsize(LA - K, dims)
    ln = _lsize(LB - K, dims)
    if QA and QB:
        lJ = sm.log2U(Q)
    else:
        lJ = 0.0
        if QA:
            lm += sm.log2U(QA)
        if QB:
            ln += sm.log2U(QB)
    flops = 8.0 * 2.0 ** (lJ + lm + ln + lk)
    out_log2 = _lsize(out, dims) + sm.log2U(Q)
    return (out, Q), StepInfo(0, 0, 2 ** lJ, 2 ** lm, 2 ** ln, 2 ** lk, flops, out_log2)


def path_cost(net, samples, path, sliced=()) -> PathCost:
    sm = samples if isinstance(samples, SampleModel) else SampleModel(net.n_qubits, samples)
    st = _leaf_state(net, frozenset(sliced))
    pc = PathCost(n_slices=int(np.prod([net.dims[x] for x in sliced])) if sliced else 1)
    peak = max((_lsize(L, net.dims) + sm.log2U(Q) for L, Q in st.values()), default=0.0)
    for i, j in path:
        res, info = _step(st[i], st[j], net.dims, sm)
        info.i, info.j = i, j
        st[i] = res
        del st[j]
        pc.steps.append(info)
        pc.flops_per_slice += info.flops
        peak = max(peak, info.out_log2)
    pc.peak_log2 = peak
    return pc


# ----------------------------------------------------------------------------- greedy

def greedy_path(net, samples=None, seed: int = 0, temperature: float = 0.0,
                subset=None, sm=None):
    """Randomised greedy; returns (path, representative id of the final tensor)."""
    rng = np.random.default_rng(seed)
    sm = sm or SampleModel(net.n_qubits, samples)
    st_all = _leaf_state(net)
    ids = sorted(subset) if subset is not None else sorted(st_all)
    st = {t: st_all[t] for t in ids}
    by_label = {}
    for t in ids:
        for x in st[t][0]:
            by_label.setdefault(x, set()).add(t)

    def size(s):
        return 2.0 ** (_lsize(s[0], net.dims) + sm.log2U(s[1]))

    def cost(a, b):
        res, _ = _step(st[a], st[b], net.dims, sm)
        return size(res) - size(st[a]) - size(st[b])

    cand = {}
    for x, ts in by_label.items():
        ts = sorted(ts)
        for p in range(len(ts)):
            for q in range(p + 1, len(ts)):
                cand[(ts[p], ts[q])] = None
    for key in cand:
        cand[key] = cost(*key)
    path = []
    alive = set(ids)
    while len(alive) > 1:
        if not cand:   # disconnected pieces: outer products, smallest first
            order = sorted(alive, key=lambda t: size(st[t]))
            a, b = min(order[0], order[1]), max(order[0], order[1])
        else:
            keys = list(cand)
            c = np.array([cand[k] for k in keys])
            if temperature > 0:
                # Boltzmann choice on the cost relative to the best candidate
                cmin = c.min()
                rel = (c - cmin) / max(abs(cmin), 1.0)
                g = -np.log(-np.log(rng.random(len(c)) + 1e-300) + 1e-300)
                k = int(np.argmin(rel - temperature * g))
            else:
                k = int(np.argmin(c))
            a, b = keys[k]
        res, _ = _step(st[a], st[b], net.dims, sm)
        path.append((a, b))
        for key in [k for k in cand if a in k or b in k]:
            del cand[key]
        for x in st[b][0]:
            by_label[x].discard(b)
        for x in st[a][0]:
            by_label[x].discard(a)
        st[a] = res
        del st[b]
        alive.discard(b)
        for x in res[0]:
            by_label.setdefault(x, set()).add(a)
        nb = set()
        for x in res[0]:
            nb |= by_label[x]
        nb.discard(a)
        for t in nb:
            key = (min(a, t), max(a, t))
            cand[key] = cost(*key)
    return path, (ids[0] if len(ids) == 1 else path[-1][0])


# ----------------------------------------------------------------------------- bisection

def bisection_path(net, samples=None, seed: int = 0, leaf_size: int = 12,
                   temperature: float = 0.0, time_weight: float | None = None,
                   kl: bool = True):
    """Recursive bisection; greedy inside parts of <= leaf_size tensors.

    With ``time_weight`` set and ``net.coords`` present, each level first splits
    geometrically (median cut along the widest of row / col / time*time_weight)
    and then refines the cut with Kernighan-Lin; otherwise KL starts from a
    random balanced partition."""
    import networkx as nx
    from networkx.algorithms.community import kernighan_lin_bisection

    sm = SampleModel(net.n_qubits, samples)
    rng = np.random.default_rng(seed)
    coords = np.asarray(net.coords, dtype=float) if (net.coords is not None and
                                                      time_weight is not None) else None
    owners = {}
    for t, ls in enumerate(net.labels):
        for x in ls:
            owners.setdefault(x, []).append(t)
    G = nx.Graph()
    G.add_nodes_from(range(net.n_tensors))
    for x, ts in owners.items():
        if len(ts) == 2:
            a, b = ts
            w = math.log2(net.dims[x])
            if G.has_edge(a, b):
                G[a][b]["weight"] += w
            else:
                G.add_edge(a, b, weight=w)

    path = []

    def rec(nodes):
        if len(nodes) <= leaf_size:
            p, rep = greedy_path(net, None, int(rng.integers(1 << 30)), temperature,
                                 subset=nodes, sm=sm)
            path.extend(p)
            return rep
        sub = G.subgraph(nodes)
        init = None
        if coords is not None:
            xs = coords[nodes] * np.array([1.0, 1.0, time_weight])
            ax = int(np.argmax(xs.max(axis=0) - xs.min(axis=0)))
            order = [nodes[p] for p in np.argsort(xs[:, ax], kind="stable")]
            init = (set(order[: len(order) // 2]), set(order[len(order) // 2:]))
        if init is not None and not kl:
            A, B = init
        else:
            A, B = kernighan_lin_bisection(sub, partition=init, weight="weight",
                                           seed=int(rng.integers(1 << 30)))
        if not A or not B:
            A, B = set(sorted(nodes)[: len(nodes) // 2]), set(sorted(nodes)[len(nodes) // 2:])
        ra = rec(sorted(A))
        rb = rec(sorted(B))
        a, b = min(ra, rb), max(ra, rb)
        path.append((a, b))
        return a

    rec(list(range(net.n_tensors)))
    return path


# ----------------------------------------------------------------------------- slicing

def slice_greedy(net, samples, path, n_slices: int | None = None,
                 peak_log2: float | None = None, candidates_top: int = 4, initial=()):
    """Greedily slice closed bonds (L292-295) until ``n_slices`` is reached and/or the
    largest intermediate is <= 2**peak_log2, starting from the ``initial`` slice
    list.  Returns the ordered sliced-label list (the last one is the
    fastest-varying digit of the slice index)."""
    sm = SampleModel(net.n_qubits, samples)
    open_set = set(net.open_labels)
    sliced = list(initial)

    def done(pc):
        ok = True
        if n_slices is not None:
            ok &= pc.n_slices >= n_slices
        if peak_log2 is not None:
            ok &= pc.peak_log2 <= peak_log2 + 1e-9
        return ok

    pc = path_cost(net, sm, path, sliced)
    while not done(pc):
        # candidate labels: those of the largest intermediates
        st = _leaf_state(net, frozenset(sliced))
        outs, costly = [], []
        for i, j in path:
            labs = st[i][0] | st[j][0]
            res, info = _step(st[i], st[j], net.dims, sm)
            st[i] = res
            del st[j]
            outs.append((info.out_log2, res[0]))
            costly.append((info.flops, labs))
        outs.sort(key=lambda t: -t[0])
        costly.sort(key=lambda t: -t[0])
        cands = set()
        for _, L in outs[:candidates_top]:
            cands |= set(L)
        for _, L in costly[:candidates_top]:     # bonds of the most expensive steps
            cands |= set(L)
        cands -= open_set
        cands -= set(sliced)
        if not cands:
            raise RuntimeError("slice_greedy: no sliceable bond left")
        best = None
        for x in sorted(cands):
            c = path_cost(net, sm, path, sliced + [x])
            key = (c.peak_log2 if peak_log2 is not None and c.peak_log2 > peak_log2 else 0.0,
                   c.total_flops)
            if best is None or key < best[0]:
                best = (key, x, c)
        sliced.append(best[1])
        pc = best[2]
    return sliced, pc


def best_path(net, samples, trials: int = 8, seed: int = 0, method: str = "bisection",
              n_slices=None, peak_log2=None, leaf_size: int = 12):
    """Try several seeds, keep the (sliced) path with the smallest total flops."""
    best = None
    rng = np.random.default_rng(seed)
    for t in range(trials):
        s = int(rng.integers(1 << 30))
        if method == "bisection":
            p = bisection_path(net, samples, s, leaf_size=leaf_size, temperature=0.3 if t else 0.0)
        else:
            p, _ = greedy_path(net, samples, s, temperature=0.3 if t else 0.0)
        if n_slices or peak_log2 is not None:
            sl, pc = slice_greedy(net, samples, p, n_slices=n_slices, peak_log2=peak_log2)
        else:
            sl, pc = [], path_cost(net, samples, p)
        if best is None or pc.total_flops < best[2].total_flops:
            best = (p, sl, pc)
    return best
