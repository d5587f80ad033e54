"""Gate-folding debug: small networks, GPU vs oracle with different fold limits."""
import os
import subprocess
import sys

CODE = r'''
import os, sys, numpy as np, torch
sys.path.insert(0, os.environ["ROOT"])
import oracle
from paper_2310_03978_b200 import Contraction
from tnworkloads import configs
for mode in ["sparse", "single"]:
    w = configs.small(grid=(3, 4), cycles=8, mode=mode, n_samples=64, n_slices=8, seed=2)
    ref = oracle.contract(w.net, w.path, w.sliced, w.samples)
    c = Contraction(device=0, stream=torch.cuda.current_stream())
    c.setup(w.net, w.samples, w.path, w.sliced)
    folds = [(s, p["n"], p["m"], p["k"]) for s, p in enumerate(c.plan_json()["steps"]) if p["folded"]]
    c.contract(0, c.n_slices)
    out = c.sum_slices_host()
    c.close()
    print(mode, "folds", folds, "rel_l2 %.3e" % (np.linalg.norm(out - ref) / np.linalg.norm(ref)))
'''
base = {"TN_TC_MIN_BIG": "8", "TN_TC_MIN_SMALL": "2", "TN_TC_MIN_K": "8", "TN_SKINNY_MIN_BIG": "2",
        "ROOT": os.path.dirname(os.path.dirname(os.path.abspath(__file__)))}
for extra in [{"TN_FOLD_GATES": "0"}, {"TN_FOLD_GATES": "1"}]:
    env = dict(os.environ, **base, **extra)
    r = subprocess.run([sys.executable, "-c", CODE], env=env, capture_output=True, text=True)
    print(extra, r.stdout.strip(), r.stderr[-400:])
