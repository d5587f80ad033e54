"""C5 sub-slice precision diagnosis: the seeded-digit sub-slice of
test_c5_m20_sampled_subslice under the routing given in the environment."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from tnworkloads import configs  # noqa: E402
from tnworkloads.network import Network, fix_bonds  # noqa: E402
from tnworkloads.treesa import refine_slices  # noqa: E402
from paper_2310_03978_b200 import Contraction  # noqa: E402

w = configs.c5()
fine, _ = refine_slices(w.net, w.samples, w.path, w.sliced, 3e11, max_extra=48)
extra = fine[len(w.sliced):]
rng = np.random.default_rng(102)
digit = {x: int(rng.integers(w.net.dims[x])) for x in fine}
sub = fix_bonds(w.net, {x: digit[x] for x in extra})
t = 0
for x in w.sliced:
    t = t * w.net.dims[x] + digit[x]
ref0 = oracle.contract_slice(sub, w.path, w.sliced, t, w.samples)
c_ = float(np.abs(ref0).max()) ** (-1.0 / sub.n_tensors)
sub = Network([tt * c_ for tt in sub.tensors], sub.labels, sub.dims, sub.open_labels, sub.n_qubits, sub.coords)
ref = ref0 * c_ ** sub.n_tensors
c = Contraction(device=0, stream=torch.cuda.current_stream())
c.setup(sub, w.samples, w.path, w.sliced)
for rep in range(2):
    c.reset_accumulator()
    c.contract(t, t + 1, os.environ.get("PREC", "extended"))
    got = c.sum_slices_host()
    print(os.environ.get("TAG", ""), rep, "rel", float(np.linalg.norm(got - ref) / np.linalg.norm(ref)), flush=True)
