"""Verification statistics of computed amplitudes: the linear
cross-entropy benchmark and the Porter-Thomas histogram of the sampled
probabilities.  Plain host arithmetic on the amplitudes ``tn_sum_slices``
returns; nothing here contracts anything.

* Eq. 2 (sampled LXEB): F_l = 2^N * sum_i p_U(x_i) / m - 1, with
  p_U(x_i) = |amp(x_i)|^2 of the ideal circuit and x_i the m sampled bitstrings.
* Fig. 7(b) (L528): the histogram of 2^N p_U(x) over bitstrings sampled from a
  circuit with fidelity f follows (f x + 1 - f) e^{-x} (Porter-Thomas, x = 2^N p,
  mixed with the uniform distribution); f = 1 for exact sampling, 0 for uniform.
"""
from __future__ import annotations

import numpy as np


def lxeb(amplitudes, n_qubits: int) -> float:
    """Sampled linear XEB (Eq. 2) of the amplitudes of m sampled bitstrings."""
    p = np.abs(np.asarray(amplitudes, dtype=np.complex128)) ** 2
    if p.size == 0:
        raise ValueError("no amplitudes")
    return float(2.0 ** n_qubits * p.mean() - 1.0)


def lxeb_stderr(amplitudes, n_qubits: int) -> float:
    """Standard error of the sampled LXEB estimate (sample std of 2^N p / sqrt(m))."""
    x = 2.0 ** n_qubits * np.abs(np.asarray(amplitudes, dtype=np.complex128)) ** 2
    return float(x.std(ddof=1) / np.sqrt(x.size)) if x.size > 1 else float("inf")


def porter_thomas_pdf(x, fidelity: float):
    """Density of x = 2^N p_U(x_i) over bitstrings sampled at the given fidelity."""
    x = np.asarray(x, dtype=np.float64)
    return (fidelity * x + 1.0 - fidelity) * np.exp(-x)


def porter_thomas_histogram(amplitudes, n_qubits: int, bins: int = 40, x_max: float = 8.0):
    """Histogram (density) of 2^N p over the samples and the f-matched theory curve.
    Returns (bin_centres, observed_density, expected_density, fidelity_estimate)."""
    x = 2.0 ** n_qubits * np.abs(np.asarray(amplitudes, dtype=np.complex128)) ** 2
    edges = np.linspace(0.0, x_max, bins + 1)
    obs, _ = np.histogram(x, bins=edges, density=False)
    width = edges[1] - edges[0]
    obs = obs / (x.size * width)
    centres = 0.5 * (edges[:-1] + edges[1:])
    f = float(x.mean() - 1.0)
    return centres, obs, porter_thomas_pdf(centres, f), f
