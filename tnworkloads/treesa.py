"""Contraction-tree simulated annealing with dynamic slicing (workload tooling).

Follows the path-finding recipe PAPER.md describes as prior art (§3.2):
a contraction tree is improved by *local updates* that exchange the descendants
of one ancestor among its three nearest descendants (L280-281, Fig. 1(d)),
accepted with a Metropolis rule on a cost score; slicing adds one bond at a time
and re-tunes the tree after each cut ("dynamic slicing", L296).  This module only
manufactures synthetic workloads for the executor (the path and slices are
inputs of the hot path); the score is the sliced total flop count of Eq. 4 with
a hard cap on the largest intermediate (the paper's α/β are unstated).

Bond dims are assumed 2 (circuit networks); label sets are Python int bitmasks.
"""
from __future__ import annotations

import math

import numpy as np

from .paths import SampleModel


class Tree:
    def __init__(self, net, samples, path):
        self.net = net
        self.sm = samples if isinstance(samples, SampleModel) else SampleModel(net.n_qubits, samples)
        qubit_of = {lab: q for q, lab in enumerate(net.open_labels)}
        closed = sorted({x for ls in net.labels for x in ls if x not in qubit_of})
        self.bit = {x: i for i, x in enumerate(closed)}
        self.label_of = closed
        N = net.n_tensors
        self.N = N
        size = 2 * N - 1
        self.left = [-1] * size
        self.right = [-1] * size
        self.parent = [-1] * size
        self.L = [0] * size
        self.Q = [0] * size
        for t, ls in enumerate(net.labels):
            m = 0
            q = 0
            for x in ls:
                if x in qubit_of:
                    q |= 1 << qubit_of[x]
                else:
                    m |= 1 << self.bit[x]
            self.L[t], self.Q[t] = m, q
        rep = list(range(N))
        nxt = N
        for i, j in path:
            v = nxt
            nxt += 1
            a, b = rep[i], rep[j]
            self.left[v], self.right[v] = a, b
            self.parent[a] = self.parent[b] = v
            self.L[v] = self.L[a] ^ self.L[b]
            self.Q[v] = self.Q[a] | self.Q[b]
            rep[i] = v
        self.root = nxt - 1
        self._ucache = {}

    # ----------------------------------------------------------------- costs
    def log2U(self, qmask):
        if qmask == 0:
            return 0.0
        v = self._ucache.get(qmask)
        if v is None:
            qs = frozenset(i for i in range(self.net.n_qubits) if qmask >> i & 1)
            v = self.sm.log2U(qs)
            self._ucache[qmask] = v
        return v

    alpha = 0.0     # Eq. 6 memory weight: flop-equivalents per byte of T_mc (8 B/element)
    # balanced-index feedback (App. A.2): a GEMM with k < 64 or min(m, n) < 32
    # under-uses the tensor cores ("k should be equal to or greater than 64 ... m or n
    # should be greater than or equal to 32"); beta weights the lost tensor time,
    # T_cc * (1/u - 1) with u = min(1, k/64) * min(1, min(m, n)/32), into the score
    beta = 0.0

    def pair_cost(self, La, Qa, Lb, Qb, keep):
        """(cost, log2 out size) of contracting (La,Qa) with (Lb,Qb); keep = ~sliced.
        cost = T_cc + alpha * T_mc (the argument of the log in Eq. 6)."""
        La &= keep
        Lb &= keep
        K = La & Lb
        lk = K.bit_count()
        lm = (La & ~K).bit_count()
        ln = (Lb & ~K).bit_count()
        ua, ub = self.log2U(Qa), self.log2U(Qb)
        if Qa and Qb:
            lj = self.log2U(Qa | Qb)
        else:
            lj = 0.0
            lm += ua
            ln += ub
        out = (La ^ Lb).bit_count() + self.log2U(Qa | Qb)
        cost = 2.0 ** (lj + lm + ln + lk + 3.0)
        if self.beta and min(lm, ln) >= 4.0 and lk >= 4.0 and max(lm, ln) >= 7.0:
            # only GEMM-shaped steps (the executor's tensor-core routing thresholds): small
            # gate absorptions are HBM-bound either way and carry alpha's T_mc term
            lu = min(0.0, lk - 6.0) + min(0.0, min(lm, ln) - 5.0)   # log2 u
            if lu < 0.0:
                cost += self.beta * cost * (2.0 ** -lu - 1.0)
        if self.alpha:
            cost += self.alpha * 8.0 * (2.0 ** (La.bit_count() + ua) + 2.0 ** (Lb.bit_count() + ub)
                                        + 2.0 ** out)
        return cost, out

    def node_cost(self, v, keep):
        a, b = self.left[v], self.right[v]
        return self.pair_cost(self.L[a], self.Q[a], self.L[b], self.Q[b], keep)

    def internal(self):
        return range(self.N, 2 * self.N - 1)

    def totals(self, keep):
        tot = 0.0
        peak = 0.0
        for v in self.internal():
            f, s = self.node_cost(v, keep)
            tot += f
            peak = max(peak, s)
        return tot, peak

    # ----------------------------------------------------------------- SA
    def anneal(self, keep, sweeps, t0, t1, peak_cap, rng):
        nodes = list(self.internal())
        flops = {}
        tot = 0.0
        for v in nodes:
            f, _ = self.node_cost(v, keep)
            flops[v] = f
            tot += flops[v]
        for sw in range(sweeps):
            T = t0 * (t1 / t0) ** (sw / max(sweeps - 1, 1))
            order = rng.permutation(nodes)
            for X in order:
                X = int(X)
                kids = [c for c in (self.left[X], self.right[X]) if c >= self.N]
                if not kids:
                    continue
                Y = kids[int(rng.integers(len(kids)))]
                Z = self.right[X] if self.left[X] == Y else self.left[X]
                r = int(rng.integers(2))
                Y1, Y2 = (self.left[Y], self.right[Y]) if r == 0 else (self.right[Y], self.left[Y])
                # new: Y' = (Y1, Z), X = (Y', Y2)
                fy, sy = self.pair_cost(self.L[Y1], self.Q[Y1], self.L[Z], self.Q[Z], keep)
                if peak_cap is not None and sy > peak_cap + 1e-9:
                    continue
                Ly, Qy = self.L[Y1] ^ self.L[Z], self.Q[Y1] | self.Q[Z]
                fx, _ = self.pair_cost(Ly, Qy, self.L[Y2], self.Q[Y2], keep)
                new = fy + fx
                old = flops[X] + flops[Y]
                tot_new = tot - old + new
                dE = math.log2(tot_new) - math.log2(tot)
                if dE <= 0 or rng.random() < math.exp(-dE / T):
                    # apply rotation
                    self.left[Y], self.right[Y] = Y1, Z
                    self.parent[Y1] = Y
                    self.parent[Z] = Y
                    self.left[X], self.right[X] = Y, Y2
                    self.parent[Y2] = X
                    self.L[Y], self.Q[Y] = Ly, Qy
                    flops[Y] = fy
                    flops[X] = fx
                    tot = tot_new
        return tot

    # ----------------------------------------------------------------- output
    def to_path(self):
        pairs = []

        def rec(v):
            if v < self.N:
                return v
            a = rec(self.left[v])
            b = rec(self.right[v])
            i, j = (a, b) if a < b else (b, a)
            pairs.append((i, j))
            return i

        import sys
        lim = sys.getrecursionlimit()
        sys.setrecursionlimit(max(lim, 10 * self.N))
        rec(self.root)
        sys.setrecursionlimit(lim)
        return pairs


def refine_slices(net, samples, path, sliced, target_flops: float, max_extra: int = 40):
    """Keep ``path`` fixed and append bonds to ``sliced`` (greedy, min per-slice flops)
    until one sub-slice costs <= target_flops.  Sub-slices of coarse slice t are
    t*2^e .. (t+1)*2^e - 1 (the new bonds are the fastest digits).  Used to size
    oracle-checkable samples of a large workload."""
    tr = Tree(net, samples, path)
    keep = (1 << len(tr.label_of)) - 1
    for x in sliced:
        keep &= ~(1 << tr.bit[x])
    extra = []
    tot, _ = tr.totals(keep)
    while tot > target_flops and len(extra) < max_extra:
        best = None
        b = keep
        while b:
            low = b & -b
            bit = low.bit_length() - 1
            b ^= low
            t2, _ = tr.totals(keep & ~(1 << bit))
            if best is None or t2 < best[1]:
                best = (bit, t2)
        if best is None or best[1] >= tot:
            break
        keep &= ~(1 << best[0])
        extra.append(tr.label_of[best[0]])
        tot = best[1]
    return list(sliced) + extra, tot


def optimize(net, samples, path0, peak_log2: float, seed: int = 0, sweeps: int = 40,
             fine_sweeps: int = 6, t0: float = 0.3, t1: float = 0.01, max_slices: int = 64,
             cand_top: int = 48, log=None, alpha: float = 0.0, beta: float = 0.0):
    """SA on the unsliced tree, then dynamic slicing down to ``peak_log2`` with a
    short low-temperature re-tune after every cut.  The score is Eq. 6's
    T_cc + alpha*T_mc (alpha in flop per byte), plus the App. A.2 balance term with
    weight beta (Tree.beta).  Returns (path, sliced labels,
    per-slice cost, peak log2)."""
    rng = np.random.default_rng(seed)
    tr = Tree(net, samples, path0)
    tr.alpha = alpha
    tr.beta = beta
    full = (1 << len(tr.label_of)) - 1
    tr.anneal(full, sweeps, t0, t1, None, rng)
    sliced_bits = []
    keep = full
    tot, peak = tr.totals(keep)
    if log:
        log(f"unsliced: flops {tot:.3g} peak 2^{peak:.1f}")
    while peak > peak_log2 + 1e-9:
        if len(sliced_bits) >= max_slices:
            raise RuntimeError("dynamic slicing: slice limit reached")
        # candidate bonds: those on the largest intermediates
        big = []
        for v in tr.internal():
            _, s = tr.node_cost(v, keep)
            big.append((s, tr.L[tr.left[v]] ^ tr.L[tr.right[v]]))
        big.sort(key=lambda x: -x[0])
        cand = 0
        for s, m in big[:cand_top]:
            if s > peak_log2:
                cand |= m
        cand &= keep
        best = None
        b = cand
        while b:
            low = b & -b
            bit = low.bit_length() - 1
            b ^= low
            k2 = keep & ~(1 << bit)
            t2, p2 = tr.totals(k2)
            key = (p2, t2)
            if best is None or (t2 * 2 ** (len(sliced_bits) + 1), p2) < (best[1], best[2]):
                best = (bit, t2 * 2 ** (len(sliced_bits) + 1), p2)
        bit = best[0]
        sliced_bits.append(bit)
        keep &= ~(1 << bit)
        tr.anneal(keep, fine_sweeps, t1 * 3, t1, best[2], rng)
        tot, peak = tr.totals(keep)
        if log:
            log(f"slice {len(sliced_bits)}: per-slice flops {tot:.3g} total {tot * 2 ** len(sliced_bits):.3g} peak 2^{peak:.1f}")
    sliced = [tr.label_of[b] for b in sliced_bits]
    return tr.to_path(), sliced, tot, peak
