"""LXEB / Porter-Thomas report of GPU-computed amplitudes.

    python tools/lxeb_report.py [--grid 4 5] [--cycles 12] [--samples 65536]

Full output state of a grid circuit on the GPU; bitstrings drawn from the
computed |amp|^2 (ideal sampling) and uniformly; prints F_l (Eq. 2) for both and
the Porter-Thomas histogram against (f x + 1 - f) e^{-x} (Fig. 7b)."""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_03978_b200 import Contraction, verify  # noqa: E402
from tnworkloads import configs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", type=int, nargs=2, default=[4, 5])
    ap.add_argument("--cycles", type=int, default=12)
    ap.add_argument("--samples", type=int, default=65536)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    w = configs.small(grid=tuple(a.grid), cycles=a.cycles, mode="full", n_slices=4, seed=21)
    c = Contraction(device=0, stream=torch.cuda.current_stream())
    c.setup(w.net, w.samples, w.path, w.sliced)
    c.contract(0, c.n_slices)
    amps = c.sum_slices_host()
    c.close()
    n = w.circuit.n_qubits
    p = np.abs(amps) ** 2
    rng = np.random.default_rng(7)
    ideal = rng.choice(p.size, size=a.samples, p=p / p.sum())
    unif = rng.integers(0, p.size, size=a.samples)
    centres, obs, exp, f = verify.porter_thomas_histogram(amps[ideal], n, bins=16, x_max=8.0)
    res = {"n_qubits": n, "cycles": a.cycles, "norm": float(p.sum()),
           "lxeb_ideal": verify.lxeb(amps[ideal], n), "lxeb_ideal_stderr": verify.lxeb_stderr(amps[ideal], n),
           "lxeb_uniform": verify.lxeb(amps[unif], n), "porter_thomas_2N_sum_p2": float(2.0 ** n * (p ** 2).sum()),
           "histogram": {"x": centres.tolist(), "observed": obs.tolist(), "expected": exp.tolist()}}
    print(json.dumps({k: v for k, v in res.items() if k != "histogram"}))
    if a.out:
        json.dump(res, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
