"""Random-circuit-sampling (RCS) circuits, §2.2 L147-149.

"each sequence composed of a single-qubit gate layer, followed by a two-qubit
gate layer" with single-qubit gates "selected randomly from the √X, √Y, and √W
gates" and fsim two-qubit gates.  The paper prints no matrices, layout or
coupler sequence; the readings adopted (DESIGN.md
"Readings"):

* fsim(θ,φ) = [[1,0,0,0],[0,cosθ,-i sinθ,0],[0,-i sinθ,cosθ,0],[0,0,0,e^{-iφ}]]
  (SPEC.md L90), θ=π/2, φ=π/6 on every coupler.
* √P = principal square root = ((1+i)/2)·I + ((1-i)/2)·P for P ∈ {X, Y, W},
  W = (X+Y)/√2, so (√P)² = P exactly.
* initial state |0…0⟩ (L142 "separable initial state"); qubit 0 = MSB.
* couplers: A = vertical with (r+c) even, B = vertical odd, C = horizontal odd,
  D = horizontal even; cycle sequence ABCDCDAB; a final 1q layer.
* no single-qubit gate repeats on the same qubit in consecutive cycles.
"""
from __future__ import annotations

from dataclasses import dataclass, field
import numpy as np

_SQ2 = np.sqrt(0.5)

PAULI = {
    "x": np.array([[0, 1], [1, 0]], dtype=np.complex128),
    "y": np.array([[0, -1j], [1j, 0]], dtype=np.complex128),
    "w": np.array([[0, (1 - 1j) * _SQ2], [(1 + 1j) * _SQ2, 0]], dtype=np.complex128),
}


def _sqrt_pauli(p: np.ndarray) -> np.ndarray:
    return 0.5 * (1 + 1j) * np.eye(2, dtype=np.complex128) + 0.5 * (1 - 1j) * p


def fsim(theta: float, phi: float) -> np.ndarray:
    c, s = np.cos(theta), np.sin(theta)
    return np.array([[1, 0, 0, 0],
                     [0, c, -1j * s, 0],
                     [0, -1j * s, c, 0],
                     [0, 0, 0, np.exp(-1j * phi)]], dtype=np.complex128)


@dataclass(frozen=True)
class Gate:
    kind: str                 # "sx" | "sy" | "sw" | "fsim" | "u"
    qubits: tuple
    params: tuple = ()
    matrix: np.ndarray | None = field(default=None, compare=False, hash=False)


def gate_matrix(g: Gate) -> np.ndarray:
    """Unitary of a gate; 2-qubit basis index = 2*b(q0) + b(q1) (q0 = MSB)."""
    if g.kind == "sx":
        return _sqrt_pauli(PAULI["x"])
    if g.kind == "sy":
        return _sqrt_pauli(PAULI["y"])
    if g.kind == "sw":
        return _sqrt_pauli(PAULI["w"])
    if g.kind == "fsim":
        return fsim(*g.params)
    if g.kind == "u":
        return np.asarray(g.matrix, dtype=np.complex128)
    raise ValueError(f"unknown gate kind {g.kind}")


@dataclass
class Circuit:
    n_qubits: int
    layers: list            # list[list[Gate]]; gates in a layer act on disjoint qubits
    sites: list | None = None   # optional (row, col) per qubit, for geometric path tooling

    def gates(self):
        for layer in self.layers:
            yield from layer

    def timed_gates(self):
        for t, layer in enumerate(self.layers):
            for g in layer:
                yield t, g

    def validate(self):
        for li, layer in enumerate(self.layers):
            seen = set()
            for g in layer:
                for q in g.qubits:
                    if not 0 <= q < self.n_qubits:
                        raise ValueError(f"layer {li}: qubit {q} out of range")
                    if q in seen:
                        raise ValueError(f"layer {li}: qubit {q} used twice")
                    seen.add(q)


# ----------------------------------------------------------------------------- layouts

def grid_layout(rows: int, cols: int):
    """Rectangular grid: sites (r,c) -> qubit r*cols+c."""
    return [(r, c) for r in range(rows) for c in range(cols)]


_SYC_ROWS = {0: (5, 6), 1: (4, 7), 2: (3, 8), 3: (2, 9), 4: (1, 9), 5: (0, 8),
             6: (1, 7), 7: (2, 6), 8: (3, 5), 9: (4, 4)}


def sycamore53_layout():
    """54-site diamond grid (SURVEY.md App. A conventions) with site (3,2) dropped."""
    sites = []
    for r in range(10):
        lo, hi = _SYC_ROWS[r]
        for c in range(lo, hi + 1):
            if (r, c) != (3, 2):
                sites.append((r, c))
    return sites


def coupler_patterns(sites):
    """A/B/C/D coupler matchings over site coordinates; returns dict name -> [(qa,qb)]."""
    index = {s: i for i, s in enumerate(sites)}
    pats = {"A": [], "B": [], "C": [], "D": []}
    for (r, c), q in index.items():
        if (r + 1, c) in index:
            pats["A" if (r + c) % 2 == 0 else "B"].append((q, index[(r + 1, c)]))
        if (r, c + 1) in index:
            pats["C" if (r + c) % 2 == 1 else "D"].append((q, index[(r, c + 1)]))
    return pats


# ----------------------------------------------------------------------------- generators

def random_circuit(sites, cycles: int, seed: int, sequence: str = "ABCDCDAB",
                   theta: float = np.pi / 2, phi: float = np.pi / 6,
                   one_qubit=("sx", "sy", "sw"), final_layer: bool = True) -> Circuit:
    """Seeded RCS circuit: per cycle a 1q layer (no repeats per qubit) then fsim on
    the cycle's coupler pattern; optional final 1q layer (Sycamore convention)."""
    rng = np.random.default_rng(seed)
    n = len(sites)
    pats = coupler_patterns(sites)
    prev = [None] * n
    layers = []

    def one_q_layer():
        layer = []
        for q in range(n):
            choices = [k for k in one_qubit if k != prev[q]]
            k = choices[int(rng.integers(len(choices)))]
            prev[q] = k
            layer.append(Gate(k, (q,)))
        return layer

    for cyc in range(cycles):
        layers.append(one_q_layer())
        pat = pats[sequence[cyc % len(sequence)]]
        layers.append([Gate("fsim", (a, b), (theta, phi)) for a, b in pat])
    if final_layer:
        layers.append(one_q_layer())
    c = Circuit(n, layers, list(sites))
    c.validate()
    return c


def echo_circuit(c: Circuit) -> Circuit:
    """U followed by U† (reverse order, daggered gates): amp(0^n) = 1 exactly."""
    inv_layers = []
    for layer in reversed(c.layers):
        inv_layers.append([Gate("u", g.qubits, (), gate_matrix(g).conj().T) for g in layer])
    out = Circuit(c.n_qubits, [list(l) for l in c.layers] + inv_layers, c.sites)
    out.validate()
    return out
