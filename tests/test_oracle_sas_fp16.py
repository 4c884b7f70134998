"""Pins of the oracle's FP16 SAS variant (sas_fp16, reading R-30; the
polynomial of Sec. 4 evaluated "in FP16").  -m "not gpu".

R-30: dist = m - x (binary32, as R-12), the threshold, floor and exact fraction f as
in the binary32 SAS; then f and the printed coefficients rounded to binary16
(nearest even), POLY by Horner with binary16 fused multiply-adds (one rounding each),
and the LUT factor e^-i times POLY in binary32.

The reference below re-derives every binary16 rounding from exact rational arithmetic
(fractions.Fraction) and numpy's float16 value set -- nothing is shared with the C oracle.
"""
from fractions import Fraction

import numpy as np
import pytest

from oracle import oracle as O

C3, C2, C1, C0 = (np.float32(c) for c in (-0.1025, 0.4626, -0.9922, 0.9996))


def f16_round(v: Fraction) -> Fraction:
    """The binary16 value nearest to v (ties to the even significand), by exact comparison
    of the two float16 neighbours around a first guess."""
    if v == 0:
        return Fraction(0)
    g = np.float16(float(v))
    cands = {g, np.nextafter(g, np.float16(np.inf)), np.nextafter(g, np.float16(-np.inf))}
    cands = sorted((c for c in cands if np.isfinite(c)), key=lambda c: Fraction(float(c)))
    best = None
    for c in cands:
        d = abs(Fraction(float(c)) - v)
        if best is None or d < best[0] or (d == best[0] and (c.view(np.uint16) & 1) == 0):
            best = (d, c)
    return Fraction(float(best[1]))


def poly_fp16_ref(f: np.float32) -> float:
    fh = f16_round(Fraction(float(f)))
    c3, c2, c1, c0 = (f16_round(Fraction(float(c))) for c in (C3, C2, C1, C0))
    p = f16_round(c3 * fh + c2)
    p = f16_round(p * fh + c1)
    p = f16_round(p * fh + c0)
    return float(p)


def test_coefficients_and_closed_forms():
    # fp16 coefficients: the binary16 neighbours of the binary32 constants
    assert O.sas_poly_fp16(0.0) == np.float32(np.float16(C0)) == np.float32(0.99951171875)
    lut = O.sas_lut(-6)
    for k in range(7):  # f = 0: POLY = fp16(C0) exactly, SAS = fl32(LUT[k] fp16(C0))
        assert O.sas_fp16(float(k)) == np.float32(lut[k] * np.float32(0.99951171875))
    assert O.sas_fp16(6.0) > 0 and O.sas_fp16(float(np.nextafter(np.float32(6), np.float32(7)))) == 0
    assert O.sas_fp16(7.5) == 0
    assert O.sas_fp16(6.0, nr=-3) == 0 and O.sas_fp16(3.0, nr=-3) > 0


def test_poly_fp16_exhaustive_over_binary16_fractions():
    """POLY_fp16 depends on f only through fh = fp16(f): every binary16 fh in [0, 1) (15360
    values) against the exact-rational Horner -- a complete check of the three binary16 FMAs
    (it separates them from binary32 FMAs rounded to binary16, which differ on 3 of them)."""
    fhs = np.arange(0, 0x3C00, dtype=np.uint16).view(np.float16)
    for fh in fhs:
        assert O.sas_poly_fp16(float(fh)) == np.float32(poly_fp16_ref(np.float32(fh))), fh


def test_poly_fp16_rounds_the_fraction():
    rng = np.random.default_rng(30)
    fs = np.concatenate([rng.random(2000, dtype=np.float32),
                         np.float32(2.0) ** -rng.integers(1, 30, 200).astype(np.float32)])  # tiny f
    fs = fs[fs < 1]
    for f in fs:
        assert O.sas_poly_fp16(float(f)) == np.float32(poly_fp16_ref(f)), f


def test_sas_fp16_from_parts_and_error_bound():
    rng = np.random.default_rng(31)
    d = np.concatenate([rng.random(4000, dtype=np.float32) * 6, np.arange(0, 6, 1 / 64, dtype=np.float32)])
    lut = O.sas_lut(-6)
    worst = 0.0
    for x in d:
        i = int(np.floor(x))
        f = np.float32(x - np.float32(i))
        want = np.float32(lut[i] * np.float32(poly_fp16_ref(f)))
        got = O.sas_fp16(float(x))
        assert got == want, x
        worst = max(worst, abs(float(got) / np.exp(-float(x)) - 1))
    # the cubic's own relative error (1.0314e-3) plus the binary16 roundings of f
    # (|df| <= 2^-12 -> <= 6.7e-4 of POLY >= 0.3675) and of three Horner steps (each <= 2^-12 of
    # an intermediate <= 1 -> <= 3 x 6.7e-4): <= 3.7e-3 relative
    assert worst <= 3.7e-3
    assert worst > 1.0314e-3  # and it is really coarser than the binary32 SAS


def test_attention_sas_fp16_close_to_binary32_sas():
    rng = np.random.default_rng(32)
    n, d = 200, 64
    q, k, v = (rng.standard_normal((n, d)).astype(np.float32) for _ in range(3))
    o32, l32 = O.prefill_head(O.params(d=d), q, k, v)
    o16, l16 = O.prefill_head(O.params(d=d, sas_fp16=1), q, k, v)
    assert not np.array_equal(o16, o32)
    rel = np.linalg.norm(o16 - o32) / np.linalg.norm(o32)
    assert rel < 1e-2
    assert np.abs(l16 - l32).max() < 1e-2


def test_alpha_uses_the_fp16_sas():
    """Two key tiles of identical scores (alpha mode 0): every P~ = SAS_fp16(0) = fp16(C0) and
    alpha = SAS_fp16(m - m) = fp16(C0), so L = m + ln(fp16(C0) (64 fp16(C0) + 64)) with m the
    tile max recomputed here from the stage-1 operands (R-18 rounding order)."""
    rng = np.random.default_rng(34)
    n, d = 128, 64
    q = np.tile(rng.standard_normal((1, d)).astype(np.float32), (n, 1))
    k = np.tile(rng.standard_normal((1, d)).astype(np.float32), (n, 1))
    v = rng.standard_normal((n, d)).astype(np.float32)
    p = O.params(d=d, sas_fp16=1, alpha_mode=0)
    _, lse = O.prefill_head(p, q, k, v, causal=False)
    q1, sq = O.quant_sym8(q[:64])
    k1, sk = O.quant_sym8(k[:64])
    s_int = int(q1[0].astype(np.int64) @ k1[0].astype(np.int64))
    c = np.float32(np.float32(np.float32(sq) * np.float32(sk)) * np.float32(p.softmax_scale))
    m = np.float32(np.float32(s_int) * c)
    c0h = 0.99951171875
    want = float(m) + np.log(c0h * (64 * c0h + 64))
    assert abs(float(lse[0]) - want) < 2e-6, (float(lse[0]), want)
    assert abs(float(m) + np.log(c0h * (64 * 0.9996 + 64)) - want) > 1e-5  # a binary32 alpha is separable


@pytest.mark.parametrize("alpha_mode", [0, 1])
def test_decode_sas_fp16_one_key_closed_form(alpha_mode):
    """One cached token: P~ = SAS_fp16(0) = fp16(C0), code 119, O = s_V v1 (the closed form
    does not depend on the polynomial's value) -- the variant changes no other step."""
    rng = np.random.default_rng(33)
    d = 64
    p = O.params(d=d, sas_fp16=1, alpha_mode=alpha_mode)
    kx, vx = rng.standard_normal((1, d)).astype(np.float32), rng.standard_normal((1, d)).astype(np.float32)
    ks, vs = O.Slot(p, 4, 2), O.Slot(p, 4, 2)
    ks.prefill(kx)
    vs.prefill(vx)
    o, lse = O.decode_head(p, rng.standard_normal(d).astype(np.float32), ks, vs, 0, 0, True)
    s_v = np.float32(np.abs(vx).max() / np.float32(119))
    np.testing.assert_allclose(o, s_v * vs.buf[0].astype(np.float32), rtol=1e-6, atol=1e-7)
