"""Sparse-state boundary conditions, App. A.1 L618-636 and §3.3 L305.

All four simulation modes are sample sets over the open legs (qubit order,
qubit 0 first = MSB):

* full state      -> ``None`` (all 2^n bitstrings, index order)        L620
* single amplitude-> one bitstring                                     L619
* subspace        -> 2^k strings: k open qubits, the rest fixed        L621-623
* sparse          -> m sampled bitstrings (uniform stand-in for the    L305, L501
                     experiment's samples; near-uniform at F≈0.2 %, L167)

Returned as uint8 arrays of shape [n_samples, n_qubits].
"""
from __future__ import annotations

import numpy as np


def full_state(n: int):
    return None


def all_bitstrings(n: int) -> np.ndarray:
    idx = np.arange(1 << n, dtype=np.int64)
    return ((idx[:, None] >> (n - 1 - np.arange(n))[None, :]) & 1).astype(np.uint8)


def single_amplitude(n: int, seed: int | None = None, bits=None) -> np.ndarray:
    if bits is None:
        rng = np.random.default_rng(seed)
        bits = rng.integers(0, 2, size=n)
    return np.asarray(bits, dtype=np.uint8).reshape(1, n)


def subspace_samples(n: int, open_qubits, seed: int) -> np.ndarray:
    """2^k bitstrings: ``open_qubits`` free (lexicographic), the rest a seeded fixed string."""
    rng = np.random.default_rng(seed)
    fixed = rng.integers(0, 2, size=n).astype(np.uint8)
    open_qubits = sorted(open_qubits)
    k = len(open_qubits)
    sub = all_bitstrings(k)
    out = np.repeat(fixed[None, :], 1 << k, axis=0)
    out[:, open_qubits] = sub
    return out


def uniform_samples(n: int, m: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return rng.integers(0, 2, size=(m, n)).astype(np.uint8)
