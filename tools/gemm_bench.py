"""Stand-alone timing of the tcgen05 complex GEMM (tn_cgemm) on one GPU.

    python tools/gemm_bench.py [m n k] [--passes 3] [--reps 5]

Reports useful TFLOPS (8·m·n·k per launch / CUDA-event duration of the GEMM
launch only, via tn_set_profiling) and the relative L2 error on a sampled
block against an fp64 product."""
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
    ap.add_argument("shape", nargs="*", type=int, default=[8192, 8192, 16384])
    ap.add_argument("--passes", type=int, default=3)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    m, n, k = a.shape
    torch.manual_seed(0)
    A = torch.randn(1, m, k, dtype=torch.complex64, device="cuda")
    B = torch.randn(1, n, k, dtype=torch.complex64, device="cuda")
    C = torch.empty(1, m, n, dtype=torch.complex64, device="cuda")
    ctx = Contraction(0, torch.cuda.current_stream())
    ctx.cgemm(A, B, C, 1, m, n, k, passes=a.passes)       # warm-up
    ctx.reset_kernel_stats()
    ctx.set_profiling(True)
    for _ in range(a.reps):
        ctx.cgemm(A, B, C, 1, m, n, k, passes=a.passes)
    st = ctx.kernel_stats()["gemm_tcgen05"]
    tflops = st["flops"] / (st["ms"] / 1e3) / 1e12
    # accuracy on a 64x64 block
    Ab = A[0, :64].cpu().numpy().astype(np.complex128)
    Bb = B[0, :64].cpu().numpy().astype(np.complex128)
    ref = Ab @ Bb.T
    err = float(np.linalg.norm(C[0, :64, :64].cpu().numpy() - ref) / np.linalg.norm(ref))
    res = {"m": m, "n": n, "k": k, "passes": a.passes, "ms_per_launch": st["ms"] / st["launches"],
           "tflops_useful": tflops, "tensor_tflops": tflops * a.passes, "rel_l2_block": err,
           "env": {x: os.environ.get(x) for x in ("TN_KCHUNK3", "TN_GEMM_GROUP", "TN_GEMM_PAIR_MIN_M") if os.environ.get(x)}}
    print(json.dumps(res))
    if a.out:
        with open(a.out, "a") as f:
            f.write(json.dumps(res) + "\n")


if __name__ == "__main__":
    main()
