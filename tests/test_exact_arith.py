"""Host-side proofs of the exact-arithmetic shortcuts the CUDA kernels take.

grey_value (csrc/lk_fastpath.cu, k_refine_exact): k / 255.0 as
q0 = RN(k * RN(1/255)), q = RN(q0 + RN(k - q0 * 255) * RN(1/255)) with both
steps fused multiply-adds. It must equal the reference's k / 255.0
(image_io.hpp:147, the value every stage reads) for all 256 grey levels.
"""
from fractions import Fraction


def _fma(a, b, c):
    return float(Fraction(a) * Fraction(b) + Fraction(c))


def test_grey_value_markstein_is_exact_for_every_grey_level():
    y = 1.0 / 255.0
    plain_off = 0
    for k in range(256):
        x = float(k)
        q0 = x * y
        plain_off += q0 != x / 255.0
        q = _fma(_fma(-q0, 255.0, x), y, q0)
        assert q == x / 255.0, k
    assert plain_off == 24  # the correction step is needed: the bare product is off for 24 levels
