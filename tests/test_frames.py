"""8-bit observed frames (LSB_OBS_U8): the device decodes u to u / 255.0
without a division (common.cuh u8_unit: q = u * RN(1/255), then one fma
residual correction).  This restates that formula with exactly rounded fma
(fractions) and checks it against read_ppm's u / 255.0 (raster.py:541) for
every byte value, so the GPU's frames equal the reference's bit for bit."""
from fractions import Fraction


def _fma(a, b, c):
    return float(Fraction(a) * Fraction(b) + Fraction(c))      # one rounding, like the hardware fma


def test_u8_unit_is_exact_for_every_byte():
    r = 1.0 / 255.0
    for u in range(256):
        q = float(u) * r
        assert _fma(_fma(-q, 255.0, float(u)), r, q) == u / 255.0, u


def test_plain_reciprocal_multiply_is_not_exact():
    """Why the correction step exists: u * RN(1/255) alone misses some bytes."""
    r = 1.0 / 255.0
    assert any(float(u) * r != u / 255.0 for u in range(256))
