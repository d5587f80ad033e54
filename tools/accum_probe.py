"""Accumulator-rounding probe for tcgen05 kind::f16 with an fp32 TMEM accumulator
(SURVEY.md §7 M4).  Known-answer products, all exactly representable in fp16
after the library's power-of-two rescale, pushed through tn_cgemm (1 pass).
Writes a JSON summary (argv[1]) with, per case, the result in units of fp32 ulp(1)."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2310_03978_b200 import Contraction  # noqa: E402

ULP = 2.0 ** -23


def run(ctx, a, b):
    k = 128
    A = np.zeros((1, 128, k), np.complex64)
    B = np.zeros((1, 128, k), np.complex64)
    A[0, 0, : len(a)] = a
    B[0, 0, : len(b)] = b
    C = torch.zeros((1, 128, 128), dtype=torch.complex64, device="cuda")
    ctx.cgemm(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), C, 1, 128, 128, k, passes=1)
    v = float(C[0, 0, 0].real.item())
    return v


def main(out):
    ctx = Contraction(0, torch.cuda.current_stream())
    res = {}
    # (i) intra-instruction: 1 + 3 * 0.25ulp... products 2^-25 each -> exact 1 + 0.75 ulp
    for sgn in (1, -1):
        a = [sgn * 1.0] + [sgn * 2.0 ** -13] * 3
        b = [1.0] + [2.0 ** -12] * 3
        v = run(ctx, a, b)
        res[f"intra_0.75ulp_sign{sgn}"] = (abs(v) - 1) / ULP
    # (iii) alignment: 1 + 4 products of 0.25 ulp in one MMA: exact 1 + 1 ulp
    for sgn in (1, -1):
        a = [sgn * 1.0] + [sgn * 2.0 ** -13] * 4
        b = [1.0] + [2.0 ** -12] * 4
        res[f"align_4x0.25ulp_sign{sgn}"] = (abs(run(ctx, a, b)) - 1) / ULP
    # (ii) inter-instruction: 1 at k=0, then 0.75 ulp at k=16,32,48,64 (separate MMAs)
    for sgn in (1, -1):
        a = np.zeros(80)
        b = np.zeros(80)
        a[0], b[0] = sgn, 1.0
        for kk in (16, 32, 48, 64):
            a[kk], b[kk] = sgn * 3 * 2.0 ** -13, 2.0 ** -12
        res[f"inter_4x0.75ulp_sign{sgn}"] = (abs(run(ctx, a, b)) - 1) / ULP
    res["expect"] = {"intra exact": 0.75, "intra RN": 1, "intra RZ": 0,
                     "align exact": 1, "align truncating-alignment": 0,
                     "inter exact": 3, "inter RN-per-MMA": 4, "inter RZ-per-MMA": 0}
    print(json.dumps(res, indent=1))
    json.dump(res, open(out, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/accum_probe.json")
