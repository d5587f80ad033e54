"""ORACLE — test infrastructure, NOT part of the product path.

A plain, slow, obviously-correct CPU fp64 implementation of what the sliced
tensor-network contraction of arXiv 2310.03978 computes.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it.  It shares no code with
``paper_2310_03978_b200`` (the CUDA library) and never imports it; the only
shared module is the seeded input generator ``tnworkloads`` (no contraction
arithmetic there).

Modules
  contract.py    path-following sliced sparse-state contraction (Eq. 3, Eq. 7,
                 L259-262, L292-295), fp64; per-step bookkeeping (Eq. 4/5).
  statevector.py brute-force state-vector simulation (textbook pin).

Parity status: every function here is pinned by
``tests/test_oracle_*.py`` against closed forms, a brute-force state vector,
invariants or the paper's worked example.  Nothing is "parity unpinned".
"""
from .contract import (contract, contract_slice, slice_digits, plan_bookkeeping,
                       merge_table, unique_projection)
from .statevector import statevector, amplitudes_for

__all__ = ["contract", "contract_slice", "slice_digits", "plan_bookkeeping",
           "merge_table", "unique_projection", "statevector", "amplitudes_for"]
