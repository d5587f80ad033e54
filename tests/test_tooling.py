"""CPU tests of the workload tooling (not the hot path): the App. A.2 balanced-index
term of the path score (R19)."""
from tnworkloads import configs
from tnworkloads.treesa import Tree


def _bits(lo, n):
    return ((1 << n) - 1) << lo


def test_balance_term_penalises_unbalanced_gemms_only():
    w = configs.small(grid=(3, 4), cycles=8, mode="single", n_slices=1, seed=0)
    t = Tree(w.net, w.samples, w.path)
    assert len(t.label_of) >= 24
    keep = (1 << len(t.label_of)) - 1
    # GEMM-shaped: m = 2^7, n = 2^4, k = 2^4 -> u = (16/64) * (16/32) = 1/8
    La, Lb = _bits(0, 7) | _bits(7, 4), _bits(11, 4) | _bits(7, 4)
    t.beta = 0.0
    c0, _ = t.pair_cost(La, 0, Lb, 0, keep)
    t.beta = 1.0
    c1, _ = t.pair_cost(La, 0, Lb, 0, keep)
    assert c0 == 2.0 ** (7 + 4 + 4 + 3)
    assert c1 == c0 * 8.0
    # balanced (m, n >= 32, k >= 64): no penalty
    La, Lb = _bits(0, 6) | _bits(12, 6), _bits(6, 6) | _bits(12, 6)
    t.beta = 0.0
    b0, _ = t.pair_cost(La, 0, Lb, 0, keep)
    t.beta = 1.0
    assert t.pair_cost(La, 0, Lb, 0, keep)[0] == b0
    # gate absorption (k = 2, n = 2): not GEMM-shaped, left to alpha's memory term
    La, Lb = _bits(0, 10) | _bits(10, 1), _bits(11, 1) | _bits(10, 1)
    t.beta = 0.0
    g0, _ = t.pair_cost(La, 0, Lb, 0, keep)
    t.beta = 1.0
    assert t.pair_cost(La, 0, Lb, 0, keep)[0] == g0
