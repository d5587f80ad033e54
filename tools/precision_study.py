"""Precision micro-study (the Fig. 4 analogue):
complex dot products (as 128 x 128 x K GEMMs on the tensor cores) of data with
magnitudes 1e-7 .. 1e3, relative error vs an fp64 product for
  - 3xFP16 with power-of-two rescaling (this library's extended mode),
  - 1xFP16 with rescaling (mixed mode),
  - fp32 SIMT (this library's CUDA-core path, fp64 accumulation),
  - fp32 matmul with fp32 accumulation (numpy float32, the paper's FP32 baseline).

    python tools/precision_study.py [--k 16384] [--out file.json]"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_03978_b200 import Contraction  # noqa: E402


def rel(x, ref):
    return float(np.linalg.norm(x - ref) / np.linalg.norm(ref))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--k", type=int, default=16384)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    m = n = 128
    ctx = Contraction(0, torch.cuda.current_stream())
    rng = np.random.default_rng(5)
    rows = []
    for e in range(-7, 4):
        scale = 10.0 ** e
        A = (rng.standard_normal((m, a.k)) + 1j * rng.standard_normal((m, a.k))) * scale
        B = (rng.standard_normal((n, a.k)) + 1j * rng.standard_normal((n, a.k))) * scale
        A32, B32 = A.astype(np.complex64), B.astype(np.complex64)
        ref = A32.astype(np.complex128) @ B32.astype(np.complex128).T     # exact on the fp32 inputs
        res = {"magnitude": scale}
        for tag, passes, simt in (("3xfp16", 3, False), ("1xfp16", 1, False), ("fp32_simt", 3, True)):
            tA = torch.from_numpy(A32).cuda().reshape(1, m, a.k)
            tB = torch.from_numpy(B32).cuda().reshape(1, n, a.k)
            tC = torch.empty(1, m, n, dtype=torch.complex64, device="cuda")
            ctx.cgemm(tA, tB, tC, 1, m, n, a.k, passes=passes, force_simt=simt)
            res[tag] = rel(tC[0].cpu().numpy().astype(np.complex128), ref)
        res["fp32_numpy"] = rel((A32 @ B32.T).astype(np.complex128), ref)
        rows.append(res)
        print(json.dumps(res))
    ctx.close()
    if a.out:
        json.dump({"k": a.k, "rows": rows}, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
