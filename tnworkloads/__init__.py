"""Seeded synthetic input generators shared by the oracle and the CUDA path.

This package produces the *inputs* of the sliced tensor-network contraction
(arXiv 2310.03978 §3): random quantum circuits (§2.2), the
tensor network they map to (§2.1), sparse-state sample sets (§3.3
L303-309, App. A.1), contraction paths (§3.1) and slice
sets (§3.2).  It holds none of the method's contraction arithmetic:
no pairwise einsum, no sparse merge, no precision split — those live
independently in ``oracle/`` (CPU fp64 reference) and in
``paper_2310_03978_b200/`` (the CUDA library).  Gate fusion while building the
network multiplies 2x2/4x4 gate *matrices* (circuit-level preprocessing, A1 in
SURVEY.md §2.1), never tensors of the network.
"""

from .circuits import (Circuit, Gate, gate_matrix, grid_layout, sycamore53_layout,
                       random_circuit, echo_circuit)
from .network import Network, circuit_to_network
from .samples import full_state, single_amplitude, subspace_samples, uniform_samples
from .paths import (greedy_path, bisection_path, path_cost, slice_greedy, PathCost,
                    best_path)

__all__ = [
    "Circuit", "Gate", "gate_matrix", "grid_layout", "sycamore53_layout",
    "random_circuit", "echo_circuit", "Network", "circuit_to_network",
    "full_state", "single_amplitude", "subspace_samples", "uniform_samples",
    "greedy_path", "bisection_path", "path_cost", "slice_greedy", "PathCost",
    "best_path",
]
