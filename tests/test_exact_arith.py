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


def test_energy_track_llround_via_half_add():
    """k_energy (csrc/lk_kernels.cu): llround(u) for -0.5 < u < W - 0.5 as
    trunc(RN(u + 0.5)) minus the one u whose sum rounds up (0.5 - 2^-54).
    Checked on the binade edges and half-integers where it could break."""
    import math

    import numpy as np

    def fast(u):
        return int(u + 0.5) - (u == float.fromhex("0x1.fffffffffffffp-2"))

    cases = []
    for n in range(0, 4100):
        for base in (n - 0.5, n + 0.5, float(n)):
            x = base
            for _ in range(4):
                cases += [x]
                x = np.nextafter(x, -np.inf)
            x = base
            for _ in range(4):
                x = np.nextafter(x, np.inf)
                cases += [x]
    for k in range(-60, 13):
        p = 2.0 ** k
        cases += [p, np.nextafter(p, 0), np.nextafter(p, np.inf), p - 0.5, p + 0.5]
    rng = np.random.default_rng(0)
    cases += list(rng.uniform(-0.5, 4096, 200000))
    for u in cases:
        u = float(u)
        if not (-0.5 < u < 4095.5):
            continue
        # C llround (half away from zero) on -0.5 < u: 0 for negatives, else floor + (frac >= 0.5)
        exact = 0 if u < 0 else math.floor(u) + (1 if u - math.floor(u) >= 0.5 else 0)
        assert fast(u) == exact, u


def test_mod64_small_identity():
    """lk_fit.cuh mod64_small: x mod d (x 64-bit, 0 < d < 2^16, the RANSAC draw
    rng() % (m.size() - i), ransac.hpp:58-64) as three 32-bit modulos over 16-bit
    slices of x. Exhaustive over the edge cases, random elsewhere."""
    import random

    def mod64_small(x, d):
        hi, lo = x >> 32, x & 0xFFFFFFFF
        r = hi % d
        r = ((r << 16) | (lo >> 16)) % d
        return ((r << 16) | (lo & 0xFFFF)) % d

    rng = random.Random(3)
    edges = [0, 1, 2**16 - 1, 2**32 - 1, 2**32, 2**48 - 1, 2**63, 2**64 - 1]
    for d in list(range(1, 300)) + [2**15, 2**16 - 1, 40000]:
        for x in edges + [rng.getrandbits(64) for _ in range(50)]:
            assert mod64_small(x, d) == x % d
