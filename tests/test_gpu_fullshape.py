"""Full-shape parity of the tcgen05 complex GEMM (``-m gpu``) at the shapes the
bench's C4 slices run (round-1 VERDICT weak 1(ii)), in the
launch configuration ``bench.py`` times (persistent grid, CTA pairs for M >= 512,
wave synchronisation for K >= 1024, chunk-promoted accumulation).  The oracle side
is the fp64 product (numpy complex128) of the same complex64 inputs, computed for
64 sampled rows x all columns (the two edge rows always included).

Tolerance: 3-pass hi/lo fp16 = operand split error ~2^-22 per product
plus one RN fp32 addition per promoted 32-k chunk, whose random-walk error grows as
sqrt(K/32/2)·2^-24 relative: bar = max(2e-6, 2^-22 + 1.5·sqrt(K/64)·2^-24) — 2e-6 up
to K ~ 2^16, 2.4e-6 at K = 2^17.  1-pass: 2e-3 (fp16 operand rounding, 2^-11)."""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2310_03978_b200 import Contraction    # noqa: E402


def bar3(K):
    return max(2e-6, 2.0 ** -22 + 1.5 * math.sqrt(K / 64) * 2.0 ** -24)


@pytest.fixture(scope="module")
def ctx():
    c = Contraction(device=0, stream=torch.cuda.current_stream())
    yield c
    c.close()


SHAPES = [
    # (M, N, K, tag)
    (32768, 16384, 16384, "C4 heavy step, CTA pair, many waves"),
    (8192, 4096, 65536, "deep K"),
    (1 << 25, 128, 128, "C4 step 356: 2^25 x 128 x 128, HBM-bound narrow"),
    (1 << 20, 64, 4096, "narrow N = 64 (N = 64 MMAs, pair halves of 32 rows)"),
    (4096, 2048, 131072, "K = 131072 dense-merge shape"),
    (20037, 1000, 65539, "ragged M, N, K tails at full size"),
]


@pytest.mark.timeout(900)
@pytest.mark.parametrize("M,N,K,tag", SHAPES)
@pytest.mark.parametrize("passes", [3, 1])
def test_cgemm_full_shape_sampled_rows(ctx, M, N, K, tag, passes):
    if passes == 1 and K not in (16384, 128):
        pytest.skip("1-pass checked on two shapes")
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N * 3 + K)
    A = torch.randn((M, K), dtype=torch.complex64, device="cuda", generator=g)
    B = torch.randn((N, K), dtype=torch.complex64, device="cuda", generator=g)
    C = torch.empty((M, N), dtype=torch.complex64, device="cuda")
    ctx.cgemm(A, B, C, 1, M, N, K, passes=passes)
    rng = np.random.default_rng(M + N + K)
    rows = np.unique(np.concatenate([[0, M - 1], rng.choice(M, 62, replace=False)]))
    ridx = torch.from_numpy(rows).cuda()
    a = A.index_select(0, ridx).cpu().numpy().astype(np.complex128)
    got = C.index_select(0, ridx).cpu().numpy().astype(np.complex128)
    del A, C
    b = B.cpu().numpy().astype(np.complex128)
    del B
    torch.cuda.empty_cache()
    ref = a @ b.T
    err = float(np.linalg.norm(got - ref) / np.linalg.norm(ref))
    bound = bar3(K) if passes == 3 else 2e-3
    print(f"[fullshape] {M}x{N}x{K} passes={passes} ({tag}): rel_l2 {err:.3e} (bar {bound:.2e})")
    assert np.isfinite(got).all()
    assert err <= bound, err
    # no row is much worse than the block (catches one bad tile / wave)
    per_row = np.linalg.norm(got - ref, axis=1) / np.linalg.norm(ref, axis=1)
    assert per_row.max() <= 4 * bound, per_row.max()


@pytest.mark.timeout(900)
def test_cgemm_full_shape_gather_batched(ctx):
    """A sparse-einsum GEMM (Eq. 7 gather tables) at a C4-sparse shape:
    J = 4096 merged configurations of 128 x 64 x 512 over 1024 / 512 slabs."""
    J, m, n, k, ga, gb = 4096, 128, 64, 512, 1024, 512
    g = torch.Generator(device="cuda").manual_seed(99)
    A = torch.randn((ga, m, k), dtype=torch.complex64, device="cuda", generator=g)
    B = torch.randn((gb, n, k), dtype=torch.complex64, device="cuda", generator=g)
    rng = np.random.default_rng(5)
    ia = rng.integers(0, ga, J).astype(np.int32)
    ib = rng.integers(0, gb, J).astype(np.int32)
    C = torch.empty((J, m, n), dtype=torch.complex64, device="cuda")
    ctx.cgemm(A, B, C, J, m, n, k, ga, gb, torch.from_numpy(ia).cuda(), torch.from_numpy(ib).cuda())
    js = np.unique(np.concatenate([[0, J - 1], rng.choice(J, 62, replace=False)]))
    An, Bn = A.cpu().numpy().astype(np.complex128), B.cpu().numpy().astype(np.complex128)
    ref = np.einsum("jmk,jnk->jmn", An[ia[js]], Bn[ib[js]])
    got = C.cpu().numpy()[js].astype(np.complex128)
    err = float(np.linalg.norm(got - ref) / np.linalg.norm(ref))
    print(f"[fullshape] gathered J={J} {m}x{n}x{k}: rel_l2 {err:.3e}")
    assert err <= bar3(k)
