"""LXEB (Eq. 2) and the Porter-Thomas histogram (Fig. 7b) on
amplitudes; pinned against the oracle's state vector (exact sampling gives F = 1,
uniform sampling F = 0, within the statistical error)."""
import numpy as np
import pytest

import oracle
from paper_2310_03978_b200 import verify
from tnworkloads import configs
from tnworkloads.circuits import gate_matrix


def _psi():
    w = configs.c1("full")
    return oracle.statevector(w.circuit, gate_matrix), w.circuit.n_qubits


def test_lxeb_exact_and_uniform_sampling():
    psi, n = _psi()
    p = np.abs(psi) ** 2
    rng = np.random.default_rng(11)
    m = 20000
    exact = rng.choice(p.size, size=m, p=p / p.sum())
    uniform = rng.integers(0, p.size, size=m)
    f_exact = verify.lxeb(psi[exact], n)
    f_unif = verify.lxeb(psi[uniform], n)
    assert abs(f_exact - 1.0) < 5 * verify.lxeb_stderr(psi[exact], n)
    assert abs(f_unif) < 5 * verify.lxeb_stderr(psi[uniform], n)
    # the full-space identity behind Eq. 1: 2^N sum_x p(x)^2 - 1 for the ideal circuit
    assert abs(2.0 ** n * np.sum(p ** 2) - 2.0) < 0.3          # Porter-Thomas: 2^N sum p^2 ~ 2


def test_porter_thomas_histogram_matches_theory():
    psi, n = _psi()
    p = np.abs(psi) ** 2
    rng = np.random.default_rng(12)
    x = rng.choice(p.size, size=40000, p=p / p.sum())
    c, obs, exp, f = verify.porter_thomas_histogram(psi[x], n, bins=16, x_max=6.0)
    assert abs(f - 1.0) < 0.1
    assert np.max(np.abs(obs - exp)) < 0.12
    assert np.all(np.isfinite(verify.porter_thomas_pdf(c, 0.5)))


def test_lxeb_rejects_empty():
    with pytest.raises(ValueError):
        verify.lxeb([], 3)
