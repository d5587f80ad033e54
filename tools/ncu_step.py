"""Profile one path step's kernels of a steady slice under ncu.

    ncu --profile-from-start off -k regex:cgemm --launch-skip N --launch-count 1 \
        --set full -o gpurun_out/x python tools/ncu_step.py --boundary sparse16 --step 217

Runs the first slices unprofiled (absmax seeding, autotuning), then brackets one
slice with cudaProfilerStart/Stop.  Prints, for --step S, how many launches of each
kernel family precede S's launches inside one slice (the --launch-skip value).
CUDA graphs are disabled so every launch is a plain kernel launch."""
import argparse
import os
import sys

os.environ.setdefault("TN_GRAPHS", "0")
import torch  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_03978_b200 import Contraction  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c4")
    ap.add_argument("--boundary", default="sparse16")
    ap.add_argument("--peak", type=int, default=32)
    ap.add_argument("--tag", default="a64")
    ap.add_argument("--step", type=int, default=-1)
    ap.add_argument("--precision", default="extended")
    a = ap.parse_args()
    from tnworkloads import configs
    w = configs.c4(a.boundary, a.peak, a.tag) if a.workload == "c4" else getattr(configs, a.workload)()
    ctx = Contraction(0, torch.cuda.current_stream())
    ctx.setup(w.net, w.samples, w.path, w.sliced)
    steps = ctx.plan_json()["steps"]
    if a.step >= 0:
        gemm_before = sum(1 for s in steps[:a.step] if s["route"] == "tcgen05")
        gate_before = sum(p.count(5) for s in steps[:a.step] if s["route"] == "tcgen05"
                          for p in [s["prep"]])
        print(f"step {a.step}: {steps[a.step]['route']} J={steps[a.step]['J']} m={steps[a.step]['m']} "
              f"n={steps[a.step]['n']} k={steps[a.step]['k']} prep={steps[a.step]['prep']}; in a slice, "
              f"cgemm launches before it: {gemm_before}, prep_gate launches before it: {gate_before}",
              flush=True)
    ctx.contract(0, 3, a.precision)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    ctx.contract(3, 4, a.precision)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    ctx.close()


if __name__ == "__main__":
    main()
