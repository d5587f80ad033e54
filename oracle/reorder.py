"""ORACLE (test infrastructure only) — the paper's top-k index-reordering rule.

PAPER.md §4.1 (L324-338, Fig. 3 "Reorder indices for top-k contractions"),
followed step by step in the paper's order:

1. *Rank contractions* (L335): rank all contractions by computing complexity
   (T_cc, Eq. 4) and take the top-k group.  Ties: the earlier path step first
   (the paper is silent; reading R18).
2. *Check current contraction* (L336): starting from the most expensive, the
   contraction qualifies when (1) it has not been modified by another reordering
   step and (2) it can form a GEMM by modifying only its input index order,
   without modifying its own output order.  In this framework every contraction
   that no reordering has touched keeps the GEMM-form output [J][P][Q] (Eq. 3's
   γ = A-free then B-free), so (2) holds exactly when (1) does (reading R18).
3. *Check associated contractions* (L337): the contractions that produced the
   current contraction's two input tensors ("if O = einsum(M, N) is determined
   to reorder, check M = einsum(I, J) and N = einsum(K, L)").  Neither may have
   been modified by another reordering step.  An input that is a network leaf
   has no associated contraction and imposes no condition.
4. *Reorder indices* (L338): the current contraction's input orders and the
   associated contractions' output orders are replaced; all of them count as
   modified from now on (reading R18: the current contraction's output order must
   stay fixed, so a later step may not reorder it either).

Returns (selected, modified): the contractions reordered as "current" and every
contraction whose index order was replaced, both as sorted step lists.
"""
from __future__ import annotations


def producers(path, n_leaves):
    """For each step s, the steps that produced its two inputs (None for a leaf).
    Stable-id path semantics (L259-262): step (i, j) -> result keeps id i."""
    last = {t: None for t in range(n_leaves)}
    out = []
    for s, (i, j) in enumerate(path):
        out.append((last[i], last[j]))
        last[i] = s
        del last[j]
    return out


def paper_topk_reorder(path, n_leaves, tcc, k):
    """The §4.1 rule over a path with per-step T_cc; k = size of the top-k group."""
    prod = producers(path, n_leaves)
    # 1. rank all contractions by T_cc (descending), ties by step index
    ranked = sorted(range(len(path)), key=lambda s: (-tcc[s], s))
    top = ranked[:k]
    modified = set()
    selected = []
    for s in top:
        # 2. current contraction: not modified by another reordering step
        if s in modified:
            continue
        # 3. associated contractions: the producers of its two inputs
        assoc = [p for p in prod[s] if p is not None]
        if any(p in modified for p in assoc):
            continue
        # 4. reorder: current + associated contractions are now modified
        selected.append(s)
        modified.add(s)
        modified.update(assoc)
    return sorted(selected), sorted(modified)
