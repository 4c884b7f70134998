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
