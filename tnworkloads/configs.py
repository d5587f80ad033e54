"""Named synthetic workloads (BASELINE.json ``configs``; recipe in DESIGN.md §Inputs).

Seeds follow SURVEY.md §8 d: circuit = 1000+c, samples = 2000+c, path = 3000+c
for config c.  Paths for the large configs are cached as order files under
``tnworkloads/orders/`` (JSON: path pairs + sliced labels + the seeds and the
generator settings that produced them), so every process sees the same
workload without re-running the path search.
"""
from __future__ import annotations

import json
import os
from dataclasses import dataclass

import numpy as np

from .circuits import random_circuit, grid_layout, sycamore53_layout, echo_circuit
from .network import circuit_to_network
from .samples import single_amplitude, subspace_samples, uniform_samples, all_bitstrings
from .paths import best_path, greedy_path, path_cost, slice_greedy, bisection_path

ORDERS = os.path.join(os.path.dirname(__file__), "orders")


@dataclass
class Workload:
    name: str
    circuit: object
    net: object
    samples: object          # uint8 [S, n] or None (full state)
    path: list
    sliced: list
    meta: dict

    @property
    def n_slices(self):
        p = 1
        for x in self.sliced:
            p *= self.net.dims[x]
        return p

    def cost(self):
        return path_cost(self.net, self.samples, self.path, self.sliced)


def _order_file(name):
    return os.path.join(ORDERS, f"{name}.json")


def _load_or_make(name, make):
    fn = _order_file(name)
    if os.path.exists(fn):
        with open(fn) as f:
            d = json.load(f)
        return [tuple(p) for p in d["path"]], list(d["sliced"]), d.get("meta", {})
    path, sliced, meta = make()
    os.makedirs(ORDERS, exist_ok=True)
    with open(fn, "w") as f:
        json.dump({"path": [list(map(int, p)) for p in path],
                   "sliced": [int(x) for x in sliced], "meta": meta}, f)
    return path, sliced, meta


def c1(mode: str = "single", simplify: bool = True) -> Workload:
    """C1: 3x4 grid, 12 qubits, 8 cycles, unsliced; single amplitude or full state."""
    circ = random_circuit(grid_layout(3, 4), 8, seed=1001)
    net = circuit_to_network(circ, simplify=simplify)
    samples = None if mode == "full" else single_amplitude(12, seed=2001)
    path, _ = greedy_path(net, samples, seed=3001)
    return Workload(f"c1_{mode}", circ, net, samples, path, [],
                    {"grid": "3x4", "cycles": 8, "mode": mode, "simplify": simplify})


def c2(n_slices: int = 64) -> Workload:
    """C2: 5x6 grid, 30 qubits, 14 cycles; 2^10 correlated amplitudes (last 10 qubits
    open, the other 20 fixed to a seeded bitstring); greedy path, 64 slices."""
    circ = random_circuit(grid_layout(5, 6), 14, seed=1002)
    net = circuit_to_network(circ)
    samples = subspace_samples(30, list(range(20, 30)), seed=2002)

    def make():
        path, _ = greedy_path(net, samples, seed=3002)
        sliced, pc = slice_greedy(net, samples, path, n_slices=n_slices)
        return path, sliced, {"flops_per_slice": pc.flops_per_slice, "peak_log2": pc.peak_log2}

    path, sliced, meta = _load_or_make(f"c2_s{n_slices}", make)
    return Workload("c2", circ, net, samples, path, sliced,
                    dict(meta, grid="5x6", cycles=14, open_qubits=10, n_slices=n_slices))


def c4_base(boundary: str = "single", cycles: int = 18):
    """Sycamore-53 m=18 circuit + boundary (no path): single amplitude, a 2^10
    correlated subspace, or 2^k uniform samples ("sparse<k>")."""
    circ = random_circuit(sycamore53_layout(), cycles, seed=1004)
    net = circuit_to_network(circ)
    if boundary == "single":
        samples = single_amplitude(53, seed=2004)
    elif boundary == "subspace":
        samples = subspace_samples(53, list(range(43, 53)), seed=2004)
    elif boundary.startswith("sparse"):
        samples = uniform_samples(53, 1 << int(boundary[6:]), seed=2004)
    else:
        raise ValueError(boundary)
    return Workload(f"c4_m{cycles}_{boundary}", circ, net, samples, [], [],
                    {"layout": "sycamore53", "cycles": cycles, "boundary": boundary})


def c4(boundary: str = "single", peak: int = 32, tag: str = "a64") -> Workload:
    """C4: Sycamore-53 m=18 with a cached SA + dynamic-slicing order file
    (tools/make_orders.py; tag "a64" = Eq. 6 score with alpha = 64 flop/B); the
    bench times a subset of its slices and extrapolates (L542)."""
    w = c4_base(boundary)
    fn = _order_file(f"c4_{boundary}_p{peak}{tag}")
    if not os.path.exists(fn):
        raise FileNotFoundError(f"{fn} missing: run tools/make_orders.py c4 --peak {peak} "
                                f"--boundary {boundary} --alpha ... --tag {tag}")
    with open(fn) as f:
        d = json.load(f)
    w.path = [tuple(p) for p in d["path"]]
    w.sliced = list(d["sliced"])
    w.meta.update(d.get("meta", {}))
    w.name = f"c4_sycamore53_m18_{boundary}_p{peak}{tag}"
    return w


def c5(boundary: str = "single", peak: int = 32, tag: str = "a64") -> Workload:
    """C5: Sycamore-53 m=20 (the paper's largest circuit, Table 5: per-slice
    peak 2^32 elements = 32 GB complex64, L556) with a cached SA + dynamic-slicing order
    file (tools/make_orders.py c5 --cycles 20 ...)."""
    w = c4_base(boundary, cycles=20)
    fn = _order_file(f"c5_{boundary}_p{peak}{tag}")
    if not os.path.exists(fn):
        raise FileNotFoundError(f"{fn} missing: run tools/make_orders.py c5 --cycles 20 --peak {peak} "
                                f"--boundary {boundary} --alpha 64 --tag {tag}")
    with open(fn) as f:
        d = json.load(f)
    w.path = [tuple(p) for p in d["path"]]
    w.sliced = list(d["sliced"])
    w.meta.update(d.get("meta", {}))
    w.name = f"c5_sycamore53_m20_{boundary}_p{peak}{tag}"
    return w


def c3(samples_log2: int = 16, peak: int = 30, tag: str = "a64") -> Workload:
    """C3: Sycamore-53 m=14 with a sparse-state boundary of 2^samples_log2 uniform
    random bitstrings (stand-ins for experiment samples, L501) — the sparse einsum
    (Eq. 7) at scale: gather-batched merges with J up to ~2^16.  Cached order file
    from tools/make_orders.py (sparse-aware U(Q) size model)."""
    w = c4_base(f"sparse{samples_log2}", cycles=14)
    fn = _order_file(f"c3_sparse{samples_log2}_p{peak}{tag}")
    if not os.path.exists(fn):
        raise FileNotFoundError(f"{fn} missing: run tools/make_orders.py c3 --cycles 14 "
                                f"--boundary sparse{samples_log2} --peak {peak} --tag {tag}")
    with open(fn) as f:
        d = json.load(f)
    w.path = [tuple(p) for p in d["path"]]
    w.sliced = list(d["sliced"])
    w.meta.update(d.get("meta", {}))
    w.name = f"c3_sycamore53_m14_sparse{samples_log2}_p{peak}{tag}"
    return w


def small(grid=(3, 3), cycles=6, mode="sparse", n_samples=16, n_slices=4, seed=0,
          simplify=True) -> Workload:
    """Small seeded case for parity tests (oracle finishes in well under a second)."""
    rows, cols = grid
    n = rows * cols
    circ = random_circuit(grid_layout(rows, cols), cycles, seed=1100 + seed)
    net = circuit_to_network(circ, simplify=simplify)
    if mode == "full":
        samples = None
    elif mode == "single":
        samples = single_amplitude(n, seed=2100 + seed)
    elif mode == "subspace":
        samples = subspace_samples(n, list(range(n - min(n, 4), n)), seed=2100 + seed)
    else:
        samples = uniform_samples(n, n_samples, seed=2100 + seed)
    path, _ = greedy_path(net, samples, seed=3100 + seed)
    sliced = []
    if n_slices > 1:
        sliced, _ = slice_greedy(net, samples, path, n_slices=n_slices)
    return Workload(f"small_{rows}x{cols}_m{cycles}_{mode}", circ, net, samples, path, sliced,
                    {"grid": f"{rows}x{cols}", "cycles": cycles, "mode": mode})


def echo(sites, cycles, seed, mode="single", n_slices=1, n_samples=8, simplify=True):
    """Echo circuit U†U: amp(0^n) = 1 and every other amplitude is 0 (exact pin)."""
    base = random_circuit(sites, cycles, seed=seed)
    circ = echo_circuit(base)
    net = circuit_to_network(circ, simplify=simplify)
    n = circ.n_qubits
    if mode == "single":
        samples = np.zeros((1, n), np.uint8)
    else:
        samples = uniform_samples(n, n_samples, seed=seed + 1)
        samples[0] = 0
    path, _ = greedy_path(net, samples, seed=seed + 2)
    sliced = []
    if n_slices > 1:
        sliced, _ = slice_greedy(net, samples, path, n_slices=n_slices)
    return Workload(f"echo_{n}q_m{cycles}", circ, net, samples, path, sliced, {"mode": mode})
