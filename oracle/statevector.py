"""ORACLE (test infrastructure only) — brute-force state vector, fp64.

Textbook simulation used as an independent pin for the tensor-network oracle
(§1 "state vector based methods").  Qubit 0 is
the most significant bit of the basis index.  Each gate is applied
by reshaping the 2^n vector to (2,)*n and contracting the gate matrix into the
target axes.
"""
from __future__ import annotations

import numpy as np


def statevector(circuit, gate_matrix) -> np.ndarray:
    """Final state U|0^n> of ``circuit``; ``gate_matrix(g)`` supplies unitaries."""
    n = circuit.n_qubits
    if n > 30:
        raise ValueError("statevector oracle limited to n <= 30")
    psi = np.zeros((2,) * n, dtype=np.complex128)
    psi[(0,) * n] = 1.0
    for g in circuit.gates():
        u = np.asarray(gate_matrix(g), dtype=np.complex128)
        qs = list(g.qubits)
        k = len(qs)
        u = u.reshape((2,) * (2 * k))
        # new[o...] = sum_i U[o..., i...] psi[... i ...]
        psi = np.tensordot(u, psi, axes=(list(range(k, 2 * k)), qs))
        # tensordot puts the k output axes first; move them back to the qubit slots
        psi = np.moveaxis(psi, list(range(k)), qs)
    return psi.reshape(-1)


def amplitudes_for(psi: np.ndarray, samples) -> np.ndarray:
    """Entries of the state vector at the given bitstrings (rows of 0/1, q0 = MSB)."""
    if samples is None:
        return psi.copy()
    s = np.asarray(samples, dtype=np.int64)
    n = s.shape[1]
    idx = (s << (n - 1 - np.arange(n))[None, :]).sum(axis=1)
    return psi[idx]
