"""Circuit -> tensor network, §2.1 L142.

"Quantum gates and initial quantum states can be mathematically represented by
tensors and vectors ... The interconnection and ordering of quantum gates ...
can be mapped to the bonds between tensors ... the tensor network input is
closed in the initial state section and opened in the final state section."

Two builders:

* ``simplify=False`` — one tensor per |0⟩ input vector, per 1q gate and per 2q
  gate (the raw gate-level network of Fig. 1(a)).
* ``simplify=True`` (default) — single-qubit gates are fused into the adjacent
  two-qubit gate *matrix* before tensors are formed (the 4x4 product
  U·(P_a⊗P_b), circuit-level gate fusion), and the |0⟩ input leg of the first
  2q gate on a wire is fixed to 0 by index selection.  This is the
  "1q gates absorbed into fsim" network of SURVEY.md §8 (N = #fsim tensors).

Tensor layout: row-major over the tensor's label list; a 2q gate tensor is
(out_a, out_b, in_a, in_b) = U.reshape(2,2,2,2) (q_a = MSB of the basis index);
a 1q gate tensor is (out, in).  ``open_labels[q]`` is qubit q's final leg.
"""
from __future__ import annotations

from dataclasses import dataclass
import numpy as np

from .circuits import Circuit, gate_matrix

_ZERO = np.array([1.0, 0.0], dtype=np.complex128)


@dataclass
class Network:
    tensors: list           # list[np.ndarray complex128], one axis per label
    labels: list            # list[list[int]]
    dims: dict              # label -> extent
    open_labels: list       # open_labels[q] = open leg of qubit q
    n_qubits: int
    coords: list | None = None  # optional (row, col, time) per tensor (path tooling only)

    @property
    def n_tensors(self) -> int:
        return len(self.tensors)

    def flat(self):
        """Flattened arrays in the layout ``tn_load_network`` takes (include/tn.h)."""
        ranks = np.array([len(l) for l in self.labels], dtype=np.int32)
        labels = np.array([x for l in self.labels for x in l], dtype=np.int64)
        dims = np.array([self.dims[x] for l in self.labels for x in l], dtype=np.int64)
        data = np.concatenate([np.ascontiguousarray(t, dtype=np.complex128).ravel()
                               for t in self.tensors]) if self.tensors else np.zeros(0, np.complex128)
        opens = np.array(self.open_labels, dtype=np.int64)
        return ranks, labels, dims, data, opens

    def label_counts(self):
        cnt = {}
        for ls in self.labels:
            for x in ls:
                cnt[x] = cnt.get(x, 0) + 1
        return cnt


def fix_bonds(net: Network, values: dict) -> Network:
    """Sub-network with closed bonds fixed to given values (index selection on the
    two tensors carrying each bond; tensor ids unchanged, so a path stays valid).
    Used to carve oracle-sized samples out of a large workload for parity tests."""
    tensors, labels = [], []
    for t, ls in zip(net.tensors, net.labels):
        t = np.asarray(t)
        ls = list(ls)
        for x in [x for x in ls if x in values]:
            ax = ls.index(x)
            t = np.take(t, values[x], axis=ax)
            ls.pop(ax)
        tensors.append(np.ascontiguousarray(t))
        labels.append(ls)
    dims = {x: d for x, d in net.dims.items() if x not in values}
    return Network(tensors, labels, dims, list(net.open_labels), net.n_qubits, net.coords)


def circuit_to_network(c: Circuit, simplify: bool = True) -> Network:
    if simplify:
        return _simplified(c)
    return _raw(c)


class _Labels:
    def __init__(self):
        self.next = 0

    def new(self):
        self.next += 1
        return self.next - 1


def _raw(c: Circuit) -> Network:
    lab = _Labels()
    tensors, labels = [], []
    wire = []
    for q in range(c.n_qubits):
        w = lab.new()
        wire.append(w)
        tensors.append(_ZERO.copy())
        labels.append([w])
    site = c.sites or [(0, q) for q in range(c.n_qubits)]
    coords = [(site[q][0], site[q][1], -1) for q in range(c.n_qubits)]
    for t, g in c.timed_gates():
        m = gate_matrix(g)
        coords.append((float(np.mean([site[q][0] for q in g.qubits])),
                       float(np.mean([site[q][1] for q in g.qubits])), t))
        if len(g.qubits) == 1:
            q, = g.qubits
            o = lab.new()
            tensors.append(m.copy())
            labels.append([o, wire[q]])
            wire[q] = o
        else:
            a, b = g.qubits
            oa, ob = lab.new(), lab.new()
            tensors.append(m.reshape(2, 2, 2, 2).copy())
            labels.append([oa, ob, wire[a], wire[b]])
            wire[a], wire[b] = oa, ob
    dims = {x: 2 for ls in labels for x in ls}
    return Network(tensors, labels, dims, list(wire), c.n_qubits, coords)


def _simplified(c: Circuit) -> Network:
    n = c.n_qubits
    eye = np.eye(2, dtype=np.complex128)
    pending = [eye.copy() for _ in range(n)]
    wire = [None] * n               # None while the wire still carries |0>
    lab = _Labels()
    twoq = []                       # [U, (a,b), (in_a,in_b), (out_a,out_b), time]
    last = [None] * n
    for tm, g in c.timed_gates():
        m = gate_matrix(g)
        if len(g.qubits) == 1:
            q, = g.qubits
            pending[q] = m @ pending[q]
        else:
            a, b = g.qubits
            u = m @ np.kron(pending[a], pending[b])
            pending[a], pending[b] = eye.copy(), eye.copy()
            oa, ob = lab.new(), lab.new()
            twoq.append([u, (a, b), (wire[a], wire[b]), (oa, ob), tm])
            last[a] = last[b] = len(twoq) - 1
            wire[a], wire[b] = oa, ob
    # fuse trailing single-qubit gates into the last 2q gate on each wire
    for q in range(n):
        if last[q] is not None and not np.array_equal(pending[q], eye):
            rec = twoq[last[q]]
            a, b = rec[1]
            rec[0] = (np.kron(pending[q], eye) if q == a else np.kron(eye, pending[q])) @ rec[0]
    tensors, labels, coords = [], [], []
    site = c.sites or [(0, q) for q in range(n)]
    for u, (a, b), (ia, ib), (oa, ob), tm in twoq:
        coords.append(((site[a][0] + site[b][0]) / 2, (site[a][1] + site[b][1]) / 2, tm))
        t = u.reshape(2, 2, 2, 2)
        ls = [oa, ob, ia, ib]
        # fix |0> inputs by index selection (drop the leg)
        if ib is None:
            t = t[:, :, :, 0]
            ls = ls[:3]
        if ia is None:
            t = t[:, :, 0]
            ls = ls[:2] + ls[3:]
        tensors.append(np.ascontiguousarray(t))
        labels.append(ls)
    opens = []
    for q in range(n):
        if wire[q] is None:         # qubit without any 2q gate: product state vector
            o = lab.new()
            tensors.append(pending[q] @ _ZERO)
            labels.append([o])
            coords.append((site[q][0], site[q][1], len(c.layers)))
            opens.append(o)
        else:
            opens.append(wire[q])
    dims = {x: 2 for ls in labels for x in ls}
    return Network(tensors, labels, dims, opens, n, coords)
