"""Exhaustive check of the division-free stage-2 rounding used by the CUDA
quantiser (quantize.cu:stage2_column): for every INT8 range and scale,
trunc(fl(a * fl(1/(2s)) + 2^-10)) == floor(a / (2s)) with a = 2(v - z) + s,
i.e. round_half_up((v - z)/s) of R-6.  Float32 arithmetic is
emulated exactly (single rounding of the fused multiply-add)."""
import numpy as np


def test_division_free_round_half_up_is_exact():
    for bits in (2, 4):
        L = (1 << bits) - 1
        for s in range(1, 81):
            inv = np.float32(1.0) / np.float32(2 * s)
            diff = np.arange(0, min(238, L * s) + 1, dtype=np.int64)   # v - z for groups with this s
            a = 2 * diff + s
            fused = (a.astype(np.float64) * np.float64(inv) + 2.0 ** -10).astype(np.float32)
            np.testing.assert_array_equal(np.trunc(fused).astype(np.int64), a // (2 * s))


def test_mulhi_round_half_up_is_exact():
    """quantize.cu:quant_prefill_kernel: code = umulhi(a, M), M = floor((2^32 - 1) / 2s) + 1
    = ceil(2^32 / 2s), equals floor(a / (2s)) for every a = 2(v - z) + s a stage-2 group can
    produce (v - z <= 238, s <= 80) -- the multiply-high form of R-6's round half up."""
    for s in range(1, 81):
        D = 2 * s
        M = (0xFFFFFFFF // D) + 1
        assert M < 2 ** 32
        a = np.arange(0, 2 * 238 + 80 + 1, dtype=np.uint64)
        np.testing.assert_array_equal((a * np.uint64(M)) >> np.uint64(32), a // np.uint64(D))


def test_packed_float_round_half_up_is_exact():
    """quantize.cu:quant_prefill_kernel (packed form): code2 = floor(fl(y * fl(1/s) + (0.5 + 2^-10)))
    with y = v - z, the floor taken by add.rm against 2^23, equals floor((2 y + s) / (2 s)) -- R-6's
    round half up -- for every y and s a stage-2 group can produce (y <= min(238, (2^b - 1) s))."""
    for bits in (2, 4):
        L = (1 << bits) - 1
        for s in range(1, 81):
            invs = np.float32(1.0) / np.float32(s)  # correctly rounded, as __frcp_rn
            y = np.arange(0, min(238, L * s) + 1, dtype=np.int64)
            # the product and sum are exact in float64 (8 + 24 significant bits); one rounding to float32
            r = (y.astype(np.float64) * np.float64(invs) + (0.5 + 2.0 ** -10)).astype(np.float32)
            np.testing.assert_array_equal(np.floor(r).astype(np.int64), (2 * y + s) // (2 * s))


def test_stage1_fp16_magic_is_exact():
    """quantize.cu: fma(x, inv, C1) with C1 = 1.5 2^23 + 0x6480 rounds x * inv half-even to an integer
    (C1 is even and its ulp is 1), and the low 16 bits of the result are the binary16 pattern of
    1152 + code for every code in [-119, 119]; subtracting 1152 in binary16 is exact."""
    c1 = 12582912 + 0x6480
    assert c1 % 2 == 0 and float(np.float32(c1)) == c1
    for code in range(-119, 120):
        bits = int(np.array([c1 + code], dtype=np.float32).view(np.uint32)[0])
        h = np.array([bits & 0xFFFF], dtype=np.uint16).view(np.float16)[0]
        assert float(h) == 1152 + code
        assert float(np.float16(h - np.float16(1152))) == code
    # half-even ties: x * inv = k + 0.5 rounds to the even neighbour
    for k in range(-119, 119):
        t = np.float32(c1) + np.float32(k + 0.5)  # exact sum rounded once (k + 0.5 is exact in float32)
        assert int(t) - c1 == (k if k % 2 == 0 else k + 1)
