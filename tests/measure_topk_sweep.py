"""Mixed-precision top-k sweep on B200 (§4.3, Table 3 L471-490 analogue).

For k in {0, 1, 10, 50, all}: the k tensor-core steps with the largest T_cc run
1-pass fp16, the rest 3-pass (TN_PREC_MIXED).  Reports, per k:
  * replaced T_cc ratio (Table 3 column 2),
  * time per C4 slice relative to all-1-pass (Table 3 column 3),
  * relative L2 and eps_L2^2 (Eq. 9) against the CPU oracle on a
    full-width C4 sample (sub-network with extra bonds fixed).
    python tests/measure_topk_sweep.py [out.json]   (lives under tests/: it runs the oracle)
"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402  (test/measurement infrastructure)
from paper_2310_03978_b200 import Contraction  # noqa: E402
from tnworkloads import configs  # noqa: E402
from tnworkloads.network import fix_bonds  # noqa: E402
from tnworkloads.treesa import refine_slices  # noqa: E402


def main(out):
    w = configs.c4()
    stream = torch.cuda.current_stream()
    # --- timing on the full C4 slice
    ctx = Contraction(0, stream)
    ctx.setup(w.net, w.samples, w.path, w.sliced)
    steps = ctx.plan_json()["steps"]
    tc = sorted([s["tcc"] for s in steps if s["route"] == "tcgen05"], reverse=True)
    total = sum(s["tcc"] for s in steps)
    ks = sorted({k for k in (0, 1, 10, 50, len(tc)) if k <= len(tc)})
    res = []
    for k in ks:
        prec = "extended" if k == 0 else "mixed"
        ctx.contract(0, 1, prec, k)            # warm-up
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for t in range(3):
            ctx.contract(t, t + 1, prec, k)
        e1.record(stream)
        torch.cuda.synchronize()
        res.append({"k": k, "tcc_ratio": sum(tc[:k]) / total, "ms_per_slice": e0.elapsed_time(e1) / 3})
    ctx.close()
    # --- accuracy on a full-width sample
    fine, _ = refine_slices(w.net, w.samples, w.path, w.sliced, 3e11, max_extra=48)
    sub = fix_bonds(w.net, {x: 0 for x in fine[len(w.sliced):]})
    ref = oracle.contract_slice(sub, w.path, w.sliced, 0, w.samples)
    ctx = Contraction(0, stream)
    ctx.setup(sub, w.samples, w.path, w.sliced)
    for r in res:
        ctx.reset_accumulator()
        ctx.contract(0, 1, "extended" if r["k"] == 0 else "mixed", r["k"])
        got = ctx.sum_slices_host()
        r["rel_l2"] = float(np.linalg.norm(got - ref) / np.linalg.norm(ref))
        l2, l2p = float(np.sum(np.abs(ref) ** 2)), float(np.sum(np.abs(got) ** 2))
        r["eps_l2sq"] = abs(l2 - l2p) / l2
    ctx.close()
    t_all = res[-1]["ms_per_slice"]
    for r in res:
        r["relative_time"] = r["ms_per_slice"] / t_all
    doc = {"workload": w.name, "flops_per_slice": total, "n_tc_steps": len(tc), "rows": res,
           "note": "Table 3 analogue: k top tensor-core steps by T_cc in 1-pass fp16, rest 3-pass; "
                   "accuracy on a C4 sub-network sample vs the fp64 oracle"}
    print(json.dumps(doc, indent=1))
    with open(out, "w") as f:
        json.dump(doc, f, indent=1)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/topk_sweep.json")
