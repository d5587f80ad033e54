"""Fig. 4 ordering on B200: relative error of complex
dot products over the "FP16 range" 1e-7..1e3 for the operand formats of tn_cgemm,
against the fp64 product of the same fp32 inputs.  The paper's finding:
err(1xTF32) > err(3xBF16) > err(3xTF32) ~ err(3xFP16) ~ err(FP32); the Ozaki-scheme
emulation (exact one-pass fp16 slice products, tools/precision_study.py) beats all of them."""
import os
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
from paper_2310_03978_b200 import Contraction   # noqa: E402


@pytest.fixture(scope="module")
def rows():
    import precision_study
    c = Contraction(device=0, stream=torch.cuda.current_stream())
    r = precision_study.study(c, k=4096, magnitudes=(1e-7, 1e-2, 1.0, 1e3, None))
    c.close()
    return r


def test_fig4_ordering(rows):
    for r in rows:
        # 1xTF32: 2^-11 operand rounding; 3xBF16: 2 x 8-bit halves (~2^-16); 3xTF32 / 3xFP16:
        # 2 x 11-bit halves (~2^-22) plus fp32 accumulation, the FP32 level
        assert r["1xtf32"] > 5 * r["3xbf16"], r
        assert r["3xbf16"] > 5 * r["3xtf32"], r
        assert r["3xtf32"] <= 2e-6 and r["3xfp16"] <= 2e-6, r
        assert r["3xfp16"] <= 3 * r["3xtf32"] and r["3xtf32"] <= 3 * r["3xfp16"], r
        assert r["3xtf32"] <= 5 * r["fp32_cuda_core"], r
        assert r["3xbf16"] < 2e-4, r
        # 1-pass formats: fp16 and tf32 share the 10-bit mantissa, bf16 has 7
        assert r["1xbf16"] > 3 * r["1xtf32"], r
        assert r["1xtf32"] < 2e-3 and r["1xfp16"] < 2e-3, r


def test_scaled_formats_are_range_independent(rows):
    """Power-of-two rescaling (L403) makes the 3-pass error independent of the data's
    magnitude across the FP16 range."""
    e = [r["3xfp16"] for r in rows if not isinstance(r["magnitude"], str)]
    assert max(e) < 2 * min(e), e


def test_ozaki_emulation_is_exact_up_to_the_slicing(rows):
    """Ozaki scheme on the fp16 tensor cores: exact slice products leave
    only the slicing remainder (< 2^-28 of a row's largest entry), so the error sits well
    below the fp32 level on every row of the study, including the log-uniform one."""
    for r in rows:
        assert r["ozaki_fp16"] < 0.1 * r["3xfp16"], r
        assert r["ozaki_fp16"] < 0.5 * r["fp32_numpy"], r
