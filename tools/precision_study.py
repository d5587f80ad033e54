"""Precision micro-study (the Fig. 4 analogue):
complex dot products (as 128 x 128 x K GEMMs) of data with magnitudes 1e-7 .. 1e3
(one row per magnitude, plus a row whose entries are log-uniform over the whole
"FP16 range"), relative error vs the fp64 product of the same fp32 inputs, for the
Fig. 4 set on B200:
  - FP32: CUDA-core fp32 GEMM (torch.matmul, TF32 off) and numpy float32,
  - 1xTF32 / 3xTF32 (Eq. 8 as printed; tcgen05 kind::tf32, RN split),
  - 1xBF16 / 3xBF16 (kind::f16 with bf16 operands, RN split),
  - 1xFP16 / 3xFP16 with power-of-two rescaling (this library's mixed / extended mode),
  - the library's SIMT path (fp32 products, fp64 sums),
  - an Ozaki-scheme emulation on the same tensor cores: every row of A and B is split
    into 8 slices of 4-bit integers under a per-row power of two; the slice products
    with i + j <= 7 (36 one-pass fp16 GEMMs through tn_cgemm) are exact, because their
    integer sums stay below 2^24 and the fp32 TMEM accumulator then never rounds; they
    are combined in fp64 on the host (an error-free transformation up to the dropped
    slices).

    python tools/precision_study.py [--k 16384] [--out file.json]"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_03978_b200 import Contraction  # noqa: E402

SCHEMES = [("1xtf32", 1, "tf32"), ("3xtf32", 3, "tf32"), ("1xbf16", 1, "bf16"),
           ("3xbf16", 3, "bf16"), ("1xfp16", 1, "fp16"), ("3xfp16", 3, "fp16")]


def rel(x, ref):
    return float(np.linalg.norm(x - ref) / np.linalg.norm(ref))


def operands(rng, m, n, k, magnitude):
    """Complex normal data at one magnitude, or (magnitude None) entries whose moduli
    are log-uniform over [1e-7, 1e3] with uniform phases."""
    def one(r):
        if magnitude is None:
            mod = 10.0 ** rng.uniform(-7, 3, (r, k))
            return mod * np.exp(2j * np.pi * rng.random((r, k)))
        return (rng.standard_normal((r, k)) + 1j * rng.standard_normal((r, k))) * magnitude
    return one(m).astype(np.complex64), one(n).astype(np.complex64)


OZ_BITS, OZ_SLICES = 4, 8


def ozaki_split(X):
    """Row-wise split X[r] = 2^e_r * sum_s S_s[r] * 2^(-4 (s+1)), S_s complex with integer
    parts |.| < 16 (exact in fp16), 8 slices; the remainder is below 2^-32 of the row max."""
    X = X.astype(np.complex128)
    amax = np.maximum(np.abs(X.real), np.abs(X.imag)).max(axis=1)
    e = np.floor(np.log2(np.where(amax > 0, amax, 1.0))) + 1.0      # |X / 2^e| < 1
    Y = X / 2.0 ** e[:, None]
    slices = []
    for _ in range(OZ_SLICES):
        Y = Y * 2.0 ** OZ_BITS
        S = np.trunc(Y.real) + 1j * np.trunc(Y.imag)
        slices.append(S.astype(np.complex64))
        Y = Y - S
    return e, slices


def ozaki_gemm(ctx, A32, B32):
    """C = A B^T from exact one-pass fp16 tensor-core products of 4-bit slices (k <= 2^14:
    each complex slice product sums < 2 * 2^8 * 2^14 = 2^23 < 2^24, so the fp32
    accumulator holds the integers exactly)."""
    m, k = A32.shape
    n = B32.shape[0]
    assert k <= 1 << 14
    ea, sa = ozaki_split(A32)
    eb, sb = ozaki_split(B32)
    C = np.zeros((m, n), np.complex128)
    for i in range(OZ_SLICES):
        tA = torch.from_numpy(sa[i]).cuda().reshape(1, m, k)
        for j in range(OZ_SLICES - i):     # i + j <= OZ_SLICES - 1
            tB = torch.from_numpy(sb[j]).cuda().reshape(1, n, k)
            tC = torch.empty(1, m, n, dtype=torch.complex64, device="cuda")
            ctx.cgemm(tA, tB, tC, 1, m, n, k, passes=1, fmt="fp16")
            C += tC[0].cpu().numpy().astype(np.complex128) * 2.0 ** (-OZ_BITS * (i + j + 2))
    return C * 2.0 ** ea[:, None] * 2.0 ** eb[None, :]


def study(ctx, k=16384, m=128, n=128, magnitudes=tuple(10.0 ** e for e in range(-7, 4)) + (None,),
          seed=5):
    rng = np.random.default_rng(seed)
    rows = []
    for mag in magnitudes:
        A32, B32 = operands(rng, m, n, k, mag)
        ref = A32.astype(np.complex128) @ B32.astype(np.complex128).T     # exact on the fp32 inputs
        tA = torch.from_numpy(A32).cuda().reshape(1, m, k)
        tB = torch.from_numpy(B32).cuda().reshape(1, n, k)
        res = {"magnitude": "log-uniform 1e-7..1e3" if mag is None else mag}
        for tag, passes, fmt in SCHEMES:
            tC = torch.empty(1, m, n, dtype=torch.complex64, device="cuda")
            ctx.cgemm(tA, tB, tC, 1, m, n, k, passes=passes, fmt=fmt)
            res[tag] = rel(tC[0].cpu().numpy().astype(np.complex128), ref)
        tC = torch.empty(1, m, n, dtype=torch.complex64, device="cuda")
        ctx.cgemm(tA, tB, tC, 1, m, n, k, force_simt=True)
        res["simt"] = rel(tC[0].cpu().numpy().astype(np.complex128), ref)
        prev = torch.backends.cuda.matmul.allow_tf32
        torch.backends.cuda.matmul.allow_tf32 = False
        res["fp32_cuda_core"] = rel((tA[0] @ tB[0].T).cpu().numpy().astype(np.complex128), ref)
        torch.backends.cuda.matmul.allow_tf32 = prev
        res["fp32_numpy"] = rel((A32 @ B32.T).astype(np.complex128), ref)
        res["ozaki_fp16"] = rel(ozaki_gemm(ctx, A32, B32), ref)
        rows.append(res)
    return rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--k", type=int, default=16384)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    ctx = Contraction(0, torch.cuda.current_stream())
    rows = study(ctx, a.k)
    for r in rows:
        print(json.dumps(r))
    ctx.close()
    if a.out:
        json.dump({"k": a.k, "m": 128, "n": 128, "rows": rows}, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
