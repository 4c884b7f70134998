"""Pins for the oracle's *quantized* Alg. 2 decode and the
rounding rules (-m "not gpu").

The decode's own steps -- integer dequantisation K^q1 = K^q2 s^int + z^int
(P:966-967), the parent (stage-1) scale of each flushed block, the INT8
buffer block with the universal scale a_univ/119, the per-row P scale
 and the alpha chain -- are checked against routines that
share none of that code:

* a *lossless* cache (every channel of every block is an arithmetic progression
  z + s k, k in [0, 2^bits-1] with both ends present, so stage 2 reproduces the
  stage-1 codes exactly) whose buffered tail holds the global max |x|: then the
  decode of one query equals, bit for bit, Alg. 1 (the chunked-prefill core) for
  that single query row at the last position over the stage-1 operands that
  ``tq_quant_sym8`` produced from the raw K/V;
* closed forms: q = 0 makes every score equal, so O is the (alpha-weighted) mean
  of the stage-1 dequantised V rows; a one-token cache gives O = s_V v^q1;
* ties: FP -> INT codes round half to even (R-2) and stage-2 codes round half up
  (R-6), discriminated by inputs that sit exactly on .5.

tests/test_oracle_mutations.py re-runs these pins against deliberately broken
oracles and requires each mutation to be caught.
"""
import numpy as np
import pytest

from paper_2412_08585_b200 import synth

BC = 64


def lossless_stream(rng, n, d, bits, amax_code=119):
    """[n][d] float32 values v * 2^-e_blk with integer v: every B_c block has channel 0
    reaching +119, so its stage-1 scale is exactly 2^-e_blk (e_blk drawn per block from
    {5, 6, 7}, so parent scales differ across blocks and between streams) and its codes
    are v; every channel of a block is z + s k with k = 2^bits - 1 at the block's first
    token and k = 0 at its second, so stage 2 is lossless.  The tail (the INT8 buffer)
    takes the smallest exponent: its max |x| is the universal max (R-9)."""
    L = (1 << bits) - 1
    v = np.zeros((n, d), np.int32)
    nfull = n // BC
    exps = rng.integers(5, 8, nfull + 1)
    if nfull:
        exps[nfull] = exps[:nfull].min()
    scale = np.zeros((n, 1))
    for bi, b0 in enumerate(range(0, n, BC)):
        m = min(BC, n - b0)
        scale[b0:b0 + m] = 2.0 ** -int(exps[bi])
        for c in range(d):
            s = int(rng.integers(1, 238 // L + 1))
            if c == 0:
                z = amax_code - s * L
            else:
                z = int(rng.integers(-119, 119 - s * L + 1))
            k = rng.integers(0, L + 1, m)
            k[0] = L
            if m > 1:
                k[1] = 0
            v[b0:b0 + m, c] = z + s * k
    return (v * scale).astype(np.float16).astype(np.float32)


def _cache(O, p, k, v, kbits, vbits):
    ks, vs = O.Slot(p, kbits, len(k) // BC + 2), O.Slot(p, vbits, len(k) // BC + 2)
    k1, sk = ks.prefill(k)
    v1, sv = vs.prefill(v)
    return ks, vs, k1, sk, v1, sv


@pytest.mark.parametrize("kbits,vbits", [(4, 4), (2, 4), (4, 2), (2, 2)])
@pytest.mark.parametrize("n", [5 * BC + 17, 3 * BC, 40])
@pytest.mark.parametrize("alpha_mode", [0, 1])
def test_lossless_decode_equals_single_row_prefill(oracle, kbits, vbits, n, alpha_mode):
    d = 128
    p = oracle.params(d=d, alpha_mode=alpha_mode)
    rng = np.random.default_rng(1000 * kbits + 10 * vbits + n + alpha_mode)
    k = lossless_stream(rng, n, d, kbits)
    v = lossless_stream(rng, n, d, vbits)
    ks, vs, k1, sk, v1, sv = _cache(oracle, p, k, v, kbits, vbits)
    nb = n // BC
    # the construction really is lossless and the buffer holds stage-1 codes
    kp, skp = ks.stage1_prefix(nb)
    vp, svp = vs.stage1_prefix(nb)
    np.testing.assert_array_equal(kp, k1[:nb * BC])
    np.testing.assert_array_equal(vp, v1[:nb * BC])
    np.testing.assert_array_equal(ks.buf[:ks.n_buf], k1[nb * BC:])
    np.testing.assert_array_equal(vs.buf[:vs.n_buf], v1[nb * BC:])
    for seed in range(3):
        q = synth.qkv(77 + seed, 1, 1, 1, 1, d)[0][0, 0, 0].astype(np.float32)
        o, l = oracle.decode_head(p, q, ks, vs)
        o_ref, l_ref = oracle.prefill_chunk_head(p, q[None], k1, sk, v1, sv, causal=True)
        np.testing.assert_array_equal(o, o_ref[0])
        assert l == l_ref[0]
        # one tap: q1 / s_q / S_int of the first block equal the single-row prefill's
        o2, l2, tap = oracle.decode_head(p, q, ks, vs, tap=0 if nb else -1)
        assert tap["hit"]
        s_int = k1[:min(BC, n)].astype(np.int32) @ tap["q1"].astype(np.int32)
        np.testing.assert_array_equal(tap["s_int"][:min(BC, n)], s_int)


@pytest.mark.parametrize("alpha_mode", [0, 1])
def test_decode_zero_query_is_weighted_mean_of_v(oracle, alpha_mode):
    """q = 0: every score is 0, every P~ = SAS(0) = c0 = 0.9996 and every P code 119,
    so O = sum_j w_j s_V,j sum_t v1_t / sum_j w_j n_j with w_j = alpha^(T-1-j):
    alpha = SAS(0) = 0.9996 in mode 0 (P:916 literally), 1 in mode 1 (R-15)."""
    d, n = 64, 7 * BC + 23
    p = oracle.params(d=d, alpha_mode=alpha_mode)
    rng = np.random.default_rng(3)
    k = lossless_stream(rng, n, d, 4)
    v = lossless_stream(rng, n, d, 2)
    ks, vs, k1, sk, v1, sv = _cache(oracle, p, k, v, 4, 2)
    o, l = oracle.decode_head(p, np.zeros(d, np.float32), ks, vs)
    T = -(-n // BC)
    a = np.float64(np.float32(0.9996)) if alpha_mode == 0 else 1.0
    num = np.zeros(d)
    den = 0.0
    for j in range(T):
        w = a ** (T - 1 - j)
        blk = v1[j * BC:(j + 1) * BC].astype(np.float64)
        num += w * np.float64(sv[j]) * blk.sum(0)
        den += w * len(blk)
    np.testing.assert_allclose(o, num / den, rtol=2e-6, atol=1e-7)
    # L = m + log(l) with m = 0 and l = c0 sum_j w_j n_j
    assert abs(l - np.log(np.float64(np.float32(0.9996)) * den)) < 2e-6


def test_decode_one_token_cache(oracle):
    """One cached token (buffer only): P~ = c0, P code 119, O = s_V v^q1 where
    (v^q1, s_V) = tq_quant_sym8(v) -- the buffer's universal scale a_univ/119 is the
    token's own stage-1 scale."""
    d = 128
    p = oracle.params(d=d)
    rng = np.random.default_rng(4)
    for _ in range(5):
        k, v, q = (rng.standard_normal((1, d)).astype(np.float16).astype(np.float32) for _ in range(3))
        ks, vs = oracle.Slot(p, 4, 2), oracle.Slot(p, 2, 2)
        ks.prefill(k)
        vs.prefill(v)
        o, l = oracle.decode_head(p, q[0], ks, vs)
        v1, s = oracle.quant_sym8(v[0])
        np.testing.assert_allclose(o, np.float64(s) * v1.astype(np.float64), rtol=3e-7, atol=1e-9)


def test_decode_buffer_after_appends_uses_universal_scale(oracle):
    """Appended tokens are coded with the universal scale and clamped at
    +-119: a token that doubles the prefill max saturates; the decode over a buffer-only
    cache equals the single-row Alg. 1 over those buffer codes with block scale
    a_univ/119, which is checked against the prefill's own stage-1 scale of a block
    holding the max."""
    d = 64
    p = oracle.params(d=d)
    rng = np.random.default_rng(6)
    x = lossless_stream(rng, 10, d, 4)  # channel 0 of token 0 = 119/64: the prefill max
    ks, vs = oracle.Slot(p, 4, 4), oracle.Slot(p, 4, 4)
    _, sk0 = ks.prefill(x)
    _, sv0 = vs.prefill(x[::-1].copy())
    assert sk0[0] == np.float32(ks.a_univ / np.float32(119))  # the block's own stage-1 scale
    extra = rng.standard_normal((5, d)).astype(np.float16).astype(np.float32)
    extra[2, 3] = 2 * ks.a_univ  # outlier: clamps to 119
    for t in extra:
        ks.append(t)
        vs.append(t)
    assert ks.buf[12, 3] == 119 and ks.n_buf == 15 and ks.n_blocks == 0
    codes_k = ks.buf[:15].copy()
    codes_v = vs.buf[:15].copy()
    sc = np.array([sk0[0]], np.float32)
    q = rng.standard_normal(d).astype(np.float16).astype(np.float32)
    o, l = oracle.decode_head(p, q, ks, vs)
    o_ref, l_ref = oracle.prefill_chunk_head(p, q[None], codes_k, sc, codes_v, sc, causal=True)
    np.testing.assert_array_equal(o, o_ref[0])
    assert l == l_ref[0]


def test_rounding_ties_half_even_and_half_up(oracle):
    """R-2: FP -> INT codes round half to EVEN (x 119/a with a = 119 is x itself:
    2.5 -> 2, -2.5 -> -2, 3.5 -> 4, 0.5 -> 0, 1.5 -> 2; half-away would give 3, -3, 4,
    1, 2).  R-6: stage-2 codes round half UP ((v - z)/s = 0.5 -> 1, 2.5 -> 3 where
    half-even gives 0 and 2)."""
    codes, s = oracle.quant_sym8(np.array([119, 2.5, -2.5, 3.5, 0.5, -0.5, 1.5, -119], np.float32))
    assert s == np.float32(1.0)
    assert codes.tolist() == [119, 2, -2, 4, 0, 0, 2, -119]
    c2, s2, z2 = oracle.quant_asym(np.array([0, 1, 5, 6], np.int8), 2)
    assert (s2, z2) == (2, 0)
    assert c2.tolist() == [0, 1, 3, 3]
    c4, s4, z4 = oracle.quant_asym(np.array([-30, -29, 0], np.int8), 4)  # s = ceil(30/15) = 2
    assert (s4, z4) == (2, -30) and c4.tolist() == [0, 1, 15]


@pytest.mark.parametrize("alpha_mode", [0, 1])
def test_prefill_row_p_scale_equals_decode(oracle, alpha_mode):
    """NEXT-2 variant p_row (P scale per row x B_c block, the granularity of Alg. 2,
    P:976-977): with every query row of the B_r block holding the block's max |q| (so
    the block's s_Q and codes are each row's own) and a lossless cache, non-causal Alg. 1
    with p_row = 1 gives every row exactly the decode of that row; with the paper's
    per-tile scale it does not."""
    d, n, nq = 128, 4 * BC + 9, 64
    rng = np.random.default_rng(11 + alpha_mode)
    k = lossless_stream(rng, n, d, 4)
    v = lossless_stream(rng, n, d, 2)
    q = (rng.standard_normal((nq, d)) * 0.5).clip(-1.9, 1.9)
    for r in range(nq):
        q[r, (5 * r) % d] = 2.0 if r % 2 else -2.0  # the same max |q| in every row
    q = q.astype(np.float16).astype(np.float32)
    rows_equal = {}
    for p_row in (1, 0):
        p = oracle.params(d=d, alpha_mode=alpha_mode, p_row=p_row)
        ks, vs, k1, sk, v1, sv = _cache(oracle, p, k, v, 4, 2)
        o, l = oracle.prefill_chunk_head(p, q, k1, sk, v1, sv, causal=False)
        rows_equal[p_row] = 0
        for r in range(nq):
            od, ld = oracle.decode_head(p, q[r], ks, vs)
            if p_row:
                np.testing.assert_array_equal(o[r], od)
                assert l[r] == ld
            rows_equal[p_row] += int(np.array_equal(o[r], od))
    assert rows_equal[0] < nq // 2
