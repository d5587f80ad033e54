"""Per-step device-time breakdown of one workload (profiling events per launch).

    python tools/step_profile.py [--workload c4] [--slices 2] [--out file.json]

Writes every path step with its route, shape, Eq. 4/5 cost and the GEMM / prep /
SIMT milliseconds per slice, sorted by time."""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_03978_b200 import Contraction  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c4")
    ap.add_argument("--slices", type=int, default=2)
    ap.add_argument("--precision", default="extended")
    ap.add_argument("--boundary", default="single", help="c4 boundary: single | sparse16")
    ap.add_argument("--peak", type=int, default=32)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    from tnworkloads import configs
    if a.workload == "c4":
        w = configs.c4(a.boundary, a.peak)
    else:
        w = {"c3": configs.c3, "c2": configs.c2}[a.workload]()
    stream = torch.cuda.Stream()
    ctx = Contraction(0, stream)
    ctx.setup(w.net, w.samples, w.path, w.sliced)
    with torch.cuda.stream(stream):
        ctx.contract(0, 1, a.precision)
        stream.synchronize()
        ctx.reset_kernel_stats()
        ctx.set_profiling(True)
        ctx.contract(1, 1 + a.slices, a.precision)
        stream.synchronize()
    fam = {f: ctx.step_stats(f) / a.slices for f in (0, 1, 2)}
    steps = ctx.plan_json()["steps"]
    rows = []
    for s, p in enumerate(steps):
        t = fam[0][s] + fam[1][s] + fam[2][s]
        rows.append({"step": s, "route": p["route"] + ("/grouped" if p.get("grouped") else ""),
                     "mode": p["mode"], "swap": p["swap"], "J": p["J"], "m": p["m"], "n": p["n"],
                     "k": p["k"], "tcc": p["tcc"], "tmc": p["tmc"], "ms": t,
                     "gemm_ms": fam[0][s], "prep_ms": fam[1][s], "simt_ms": fam[2][s],
                     "tflops": p["tcc"] / max(t, 1e-9) / 1e9,
                     "gbs": p["tmc"] / max(t, 1e-9) / 1e6})
    rows.sort(key=lambda r: -r["ms"])
    tot = {k: float(sum(r[k] for r in rows)) for k in ("ms", "gemm_ms", "prep_ms", "simt_ms")}
    res = {"workload": w.name, "precision": a.precision, "per_slice": tot, "steps": rows}
    print(json.dumps(tot))
    for r in rows[:40]:
        print("%4d %-16s J=%-6d m=%-9d n=%-9d k=%-6d ms=%7.2f (g %6.2f p %6.2f s %6.2f) %6.1f TF %6.0f GB/s"
              % (r["step"], r["route"], r["J"], r["m"], r["n"], r["k"], r["ms"], r["gemm_ms"],
                 r["prep_ms"], r["simt_ms"], r["tflops"], r["gbs"]))
    if a.out:
        with open(a.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
