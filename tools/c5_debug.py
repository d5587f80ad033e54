"""C5 sub-slice diagnosis: the scaled sub-network of test_c5_m20_sampled_subslice under
several routing settings (one process per setting, env given on the command line)."""
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
sub = fix_bonds(w.net, {x: 0 for x in fine[len(w.sliced):]})
ref0 = oracle.contract_slice(sub, w.path, w.sliced, 0, w.samples)
c_ = float(np.abs(ref0).max()) ** (-1.0 / sub.n_tensors)
sub = Network([t * c_ for t in sub.tensors], sub.labels, sub.dims, sub.open_labels, sub.n_qubits, sub.coords)
ref = ref0 * c_ ** sub.n_tensors
c = Contraction(device=0, stream=torch.cuda.current_stream())
c.setup(sub, w.samples, w.path, w.sliced)
c.contract(0, 1)
got = c.sum_slices_host()
print(os.environ.get("TAG", ""), "got", got, "ref", ref, "rel", float(np.linalg.norm(got - ref) / np.linalg.norm(ref)))
