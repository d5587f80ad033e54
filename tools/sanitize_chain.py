"""compute-sanitizer driver for the round-2 SIMT kernels on a full-width C4-sparse16
sub-network slice: the fused skinny chains (TN_CHAIN_MIN_SAVE_LOG2=0: every eligible chain)
and the slab-staged final merge, checked against the oracle.

    compute-sanitizer --tool memcheck python tools/sanitize_chain.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("TN_CHAIN_MIN_SAVE_LOG2", "0")
os.environ.setdefault("TN_GRAPHS", "0")
import oracle  # noqa: E402
from tnworkloads import configs  # noqa: E402
from tnworkloads.network import Network, fix_bonds  # noqa: E402
from tnworkloads.treesa import refine_slices  # noqa: E402
from paper_2310_03978_b200 import Contraction  # noqa: E402

w = configs.c4("sparse16", 32)
fine, _ = refine_slices(w.net, w.samples, w.path, w.sliced, 2e11, max_extra=48)
sub = fix_bonds(w.net, {x: 0 for x in fine[len(w.sliced):]})
ref0 = oracle.contract_slice(sub, w.path, w.sliced, 0, w.samples)
c_ = float(np.abs(ref0).max()) ** (-1.0 / sub.n_tensors)
sub = Network([t * c_ for t in sub.tensors], sub.labels, sub.dims, sub.open_labels, sub.n_qubits, sub.coords)
ref = ref0 * c_ ** sub.n_tensors
ctx = Contraction(0, torch.cuda.current_stream())
ctx.setup(sub, w.samples, w.path, w.sliced)
steps = ctx.plan_json()["steps"]
ctx.contract(0, 1)
got = ctx.sum_slices_host()
ctx.close()
print("chained steps", sum(s["chained"] for s in steps), "wd_staged", sum(s["wd_staged"] for s in steps),
      "rel", float(np.linalg.norm(got - ref) / np.linalg.norm(ref)), flush=True)
