"""ORACLE (test infrastructure only) — sliced sparse-state contraction in fp64.

Follows PAPER.md step by step, in the paper's order:

* Eq. 3 (L219-229): a pairwise contraction sums the shared indices
  δ = α ∩ β and keeps γ = (α ∪ β) \\ δ.  Executed with ``np.tensordot``
  (complex128) — a library primitive used as one step, no fusion.
* Path semantics (L259-262): N-1 pairs; "the contracted tensor resulting from
  each step is indexed by the first tensor".  Stable ids: (i, j) -> i, j retires.
* Slicing (L292-295): a sliced bond is fixed to one value on every tensor that
  carries it; the slice index t decodes in mixed radix over the sliced bonds in
  the order given, last = fastest.  The sum
  over slices is accumulated in fp64 in ascending t.
* Sparse-state contraction (§3.3, Eq. 7): the open legs of a tensor form
  one merged group indexed by the *unique projections of the sample bitstrings*
  onto the group's qubits (lexicographically sorted, reading R9).  When
  two tensors that both carry a group are contracted, the merged group ranges over
  the unique projections onto the union and, per Eq. 7, the result is the
  concatenation over merged configurations f of Σ_d A[c(f), ...] B[e(f), ...].
  Leaves carrying several open legs merge them at load by index selection.
* Unification (App. A.1): full state = all 2^n strings, single
  amplitude = one string, subspace = 2^k strings with the others fixed.

Bookkeeping (``plan_bookkeeping``) re-derives, independently of the CUDA
library's planner, each step's shape and T_cc (Eq. 4, ops_per_element = 8,
L232-237) and T_mc (Eq. 5, sizeof_data = 8 for complex64, L240-244), plus the
merge index tables, so the library's plan dump can be compared bit-exactly.
"""
from __future__ import annotations

import numpy as np


# ----------------------------------------------------------------------------- helpers

def slice_digits(t: int, dims) -> list:
    """Mixed-radix digits of slice index t over ``dims``; the last digit is fastest."""
    total = 1
    for d in dims:
        total *= int(d)
    if not 0 <= t < total:
        raise ValueError(f"slice index {t} out of range [0, {total})")
    out = [0] * len(dims)
    for p in range(len(dims) - 1, -1, -1):
        out[p] = t % int(dims[p])
        t //= int(dims[p])
    return out


def unique_projection(samples: np.ndarray, qubits) -> np.ndarray:
    """Sorted unique rows of samples[:, qubits] (lexicographic, qubits ascending)."""
    qubits = list(qubits)
    if len(qubits) == 0:
        return np.zeros((1, 0), dtype=np.uint8)
    return np.unique(np.asarray(samples)[:, qubits], axis=0)


def _row_index(table: np.ndarray, rows: np.ndarray) -> np.ndarray:
    """Position of each row of ``rows`` inside ``table`` (every row must be present)."""
    lookup = {tuple(r): p for p, r in enumerate(table.tolist())}
    return np.array([lookup[tuple(r)] for r in rows.tolist()], dtype=np.int64)


def merge_table(samples, qa, qb):
    """Eq. 7 merge of open groups with qubits ``qa`` and ``qb``.

    Returns (q, table, ia, ib): q = sorted union, table = unique projections onto q,
    ia[f] / ib[f] = index of configuration f's projection in A's / B's own table.
    """
    q = sorted(set(qa) | set(qb))
    if set(qa) & set(qb):
        raise ValueError("overlapping open groups")
    table = unique_projection(samples, q)
    ta = unique_projection(samples, sorted(qa))
    tb = unique_projection(samples, sorted(qb))
    pa = [q.index(x) for x in sorted(qa)]
    pb = [q.index(x) for x in sorted(qb)]
    ia = _row_index(ta, table[:, pa])
    ib = _row_index(tb, table[:, pb])
    return q, table, ia, ib


class _Tensor:
    """Oracle tensor: axis 0 is the open group (if any), then ``labels`` in order."""

    def __init__(self, data, labels, group=None, table=None):
        self.data = data
        self.labels = list(labels)
        self.group = group          # sorted list of qubits, or None
        self.table = table          # [G, len(group)] uint8


def _all_bitstrings(n):
    idx = np.arange(1 << n, dtype=np.int64)
    return ((idx[:, None] >> (n - 1 - np.arange(n))[None, :]) & 1).astype(np.uint8)


def _prepare_leaves(net, sliced, digits, samples):
    qubit_of = {lab: q for q, lab in enumerate(net.open_labels)}
    fixed = dict(zip(sliced, digits))
    leaves = {}
    for tid, (data, labels) in enumerate(zip(net.tensors, net.labels)):
        data = np.asarray(data, dtype=np.complex128)
        labels = list(labels)
        # slicing: fix sliced bonds by index selection
        for lab in [x for x in labels if x in fixed]:
            ax = labels.index(lab)
            data = np.take(data, fixed[lab], axis=ax)
            labels.pop(ax)
        opens = [x for x in labels if x in qubit_of]
        if not opens:
            leaves[tid] = _Tensor(data, labels)
            continue
        # open legs -> one group indexed by unique sample projections (Eq. 7 at load)
        opens.sort(key=lambda x: qubit_of[x])
        q = [qubit_of[x] for x in opens]
        table = unique_projection(samples, q)
        axes = [labels.index(x) for x in opens]
        moved = np.moveaxis(data, axes, list(range(len(axes))))
        g = moved[tuple(table[:, c].astype(np.int64) for c in range(len(q)))]
        rest = [x for x in labels if x not in opens]
        leaves[tid] = _Tensor(np.ascontiguousarray(g), rest, q, table)
    return leaves


def _contract_pair(A: _Tensor, B: _Tensor, samples):
    K = [x for x in A.labels if x in B.labels]
    offA = 1 if A.group is not None else 0
    offB = 1 if B.group is not None else 0
    axA = [offA + A.labels.index(x) for x in K]
    axB = [offB + B.labels.index(x) for x in K]
    freeA = [x for x in A.labels if x not in K]
    freeB = [x for x in B.labels if x not in K]
    if A.group is not None and B.group is not None:
        # Eq. 7: concat over merged configurations f of sum_d A[c(f)...] B[e(f)...]
        q, table, ia, ib = merge_table(samples, A.group, B.group)
        axA1 = [a - 1 for a in axA]
        axB1 = [b - 1 for b in axB]
        parts = [np.tensordot(A.data[ia[f]], B.data[ib[f]], axes=(axA1, axB1))
                 for f in range(len(table))]
        data = np.stack(parts, axis=0)
        return _Tensor(data, freeA + freeB, q, table)
    data = np.tensordot(A.data, B.data, axes=(axA, axB))
    if A.group is not None:
        return _Tensor(data, freeA + freeB, A.group, A.table)
    if B.group is not None:
        # tensordot order is [freeA..., G, freeB...]; the group goes to axis 0
        data = np.moveaxis(data, len(freeA), 0)
        return _Tensor(data, freeA + freeB, B.group, B.table)
    return _Tensor(data, freeA + freeB)


def _validate_path(n, path):
    if len(path) != max(n - 1, 0):
        raise ValueError(f"path must have N-1 = {n - 1} steps, got {len(path)}")
    alive = set(range(n))
    for i, j in path:
        if i == j or i not in alive or j not in alive:
            raise ValueError(f"path step ({i},{j}) references a retired/unknown id")
        alive.discard(j)


def contract_slice(net, path, sliced, t, samples=None) -> np.ndarray:
    """Contribution of slice t: amplitudes (caller sample order) of the network with
    the sliced bonds fixed to the digits of t."""
    n_open = len(net.open_labels)
    full = samples is None
    smp = _all_bitstrings(n_open) if full else np.asarray(samples, dtype=np.uint8)
    dims = [net.dims[x] for x in sliced]
    digits = slice_digits(t, dims)
    _validate_path(net.n_tensors, path)
    T = _prepare_leaves(net, list(sliced), digits, smp)
    for i, j in path:
        T[i] = _contract_pair(T[i], T[j], smp)
        del T[j]
    (root,) = T.values()
    if root.labels:
        raise ValueError(f"closed labels left uncontracted: {root.labels}")
    if root.group is None:
        return np.array([complex(root.data)], dtype=np.complex128)
    if root.group != list(range(n_open)):
        raise ValueError("final group does not cover all open qubits")
    pos = _row_index(root.table, smp)
    return root.data[pos].astype(np.complex128)


def contract(net, path, sliced=(), samples=None, slice_ids=None) -> np.ndarray:
    """Σ over slices (ascending t, fp64) of ``contract_slice``."""
    total = 1
    for x in sliced:
        total *= net.dims[x]
    ids = range(total) if slice_ids is None else sorted(slice_ids)
    acc = None
    for t in ids:
        v = contract_slice(net, path, sliced, t, samples)
        acc = v.copy() if acc is None else acc + v
    return acc


# ----------------------------------------------------------------------------- bookkeeping

def plan_bookkeeping(net, path, sliced=(), samples=None):
    """Independent per-step bookkeeping: shapes, T_cc (Eq. 4), T_mc (Eq. 5), merges.

    For step s: J = merged configurations (1 if no sparse merge), m = elements of
    A's free part (its group included when only A carries one), n likewise for B,
    k = elements of the contracted indices.  T_cc = 8*J*m*n*k, T_mc = 8*(|A|+|B|+|C|).
    """
    n_open = len(net.open_labels)
    smp = _all_bitstrings(n_open) if samples is None else np.asarray(samples, dtype=np.uint8)
    qubit_of = {lab: q for q, lab in enumerate(net.open_labels)}
    sl = set(sliced)
    st = {}
    for tid, labels in enumerate(net.labels):
        ls = [x for x in labels if x not in sl]
        opens = sorted((x for x in ls if x in qubit_of), key=lambda x: qubit_of[x])
        q = [qubit_of[x] for x in opens]
        G = len(unique_projection(smp, q)) if q else None
        st[tid] = ([x for x in ls if x not in qubit_of], q if q else None, G)

    def prod(ls):
        p = 1
        for x in ls:
            p *= int(net.dims[x])
        return p

    out = []
    for i, j in path:
        (LA, QA, GA), (LB, QB, GB) = st[i], st[j]
        K = [x for x in LA if x in LB]
        fA = [x for x in LA if x not in K]
        fB = [x for x in LB if x not in K]
        rec = {"i": i, "j": j, "k": prod(K)}
        sizeA = prod(LA) * (GA or 1)
        sizeB = prod(LB) * (GB or 1)
        if QA is not None and QB is not None:
            q, table, ia, ib = merge_table(smp, QA, QB)
            J = len(table)
            rec.update(J=J, m=prod(fA), n=prod(fB), ia=ia.tolist(), ib=ib.tolist())
            st[i] = (fA + fB, q, J)
        else:
            rec.update(J=1, m=prod(fA) * (GA or 1), n=prod(fB) * (GB or 1), ia=None, ib=None)
            q = QA if QA is not None else QB
            st[i] = (fA + fB, q, GA if QA is not None else GB)
        del st[j]
        sizeC = prod(st[i][0]) * (st[i][2] or 1)
        rec["tcc"] = 8 * rec["J"] * rec["m"] * rec["n"] * rec["k"]
        rec["tmc"] = 8 * (sizeA + sizeB + sizeC)
        out.append(rec)
    return out
