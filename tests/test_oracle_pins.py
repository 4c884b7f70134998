"""Pins for the CPU oracle (-m "not gpu").

Each test checks the oracle against something other than itself: values of a
worked example (tests/golden), closed forms, invariants, brute force, the exact
FP64 attention of Eq. 2 under the exact-mode switches, or
exhaustive enumeration.  Citations: PAPER.md line numbers.
"""
import json
import os
from decimal import Decimal, getcontext
from fractions import Fraction

import numpy as np
import pytest

from paper_2412_08585_b200 import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_example.json")))


def rel_l2(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


# ---------------------------------------------------------------- SAS
def _nearest_f32(x: Decimal) -> np.float32:
    f = np.float32(float(x))
    cands = [f, np.nextafter(f, np.float32(np.inf)), np.nextafter(f, np.float32(-np.inf))]
    return min(cands, key=lambda c: abs(Fraction(float(c)) - Fraction(x)))


def test_lut_is_correctly_rounded_exp(oracle):
    """LUT[i] = e^{-i} vs 60-digit Decimal exp."""
    getcontext().prec = 60
    lut = oracle.sas_lut(-6)
    for i in range(7):
        assert lut[i] == _nearest_f32(Decimal(-i).exp()), i


def test_poly_closed_form_values(oracle):
    """POLY(x) = -0.1025x^3 + 0.4626x^2 - 0.9922x + 0.9996."""
    assert oracle.sas_poly(0.0) == np.float32(0.9996)
    assert abs(float(oracle.sas_poly(1.0)) - (-0.1025 + 0.4626 - 0.9922 + 0.9996)) < 1e-6
    assert abs(float(oracle.sas_poly(0.5)) - (-0.1025 / 8 + 0.4626 / 4 - 0.9922 / 2 + 0.9996)) < 1e-6


def test_sas_vs_exact_exp_over_domain(oracle):
    """SAS error bound against e^{-x} on [0, |n_r|] (closed-form analysis of the
    cubic: max rel err 1.0314e-3 at f->1, max abs 4.0e-4 at f=0)."""
    for d in np.linspace(0.0, 6.0, 6001, dtype=np.float32):
        s = float(oracle.sas(d))
        e = float(np.exp(-np.float64(d)))
        assert abs(s / e - 1.0) <= 1.04e-3, d
        assert abs(s - e) <= 4.0e-4 + 1e-7, d


def test_sas_threshold_and_integer_points(oracle):
    """Zero iff x - m < n_r (strict), LUT x POLY(0) at integers."""
    lut = oracle.sas_lut(-6)
    assert oracle.sas(6.0) > 0
    assert oracle.sas(np.nextafter(np.float32(6.0), np.float32(7))) == 0
    assert oracle.sas(10.0) == 0
    for k in range(7):
        assert oracle.sas(float(k)) == np.float32(lut[k] * np.float32(0.9996))
    # POLY(1) < e^{-1}*POLY(0)/LUT ratio -> SAS jumps *up* at each integer (not monotone).
    for k in range(1, 7):
        below = np.nextafter(np.float32(k), np.float32(0))
        assert oracle.sas(float(k)) > oracle.sas(float(below))
    # smallest kept value (PAPER.md:493 sparsity): LUT[5] * POLY(1^-)
    assert 2.47e-3 < float(oracle.sas(5.999999)) < 2.48e-3


def test_appendix_b_row_softmax(oracle):
    """Appendix B: integer-spaced rows reproduce the exact
    softmax (c0 cancels), far-apart rows are pruned to one-hot."""
    out = oracle.sas_softmax_rows(np.array([[0.0, -1.0], [5.0, -5.0], [0.0, -2.0]], np.float32))
    e = np.exp([0.0, -1.0])
    np.testing.assert_allclose(out[0], e / e.sum(), rtol=1e-6)
    np.testing.assert_array_equal(out[1], [1.0, 0.0])
    e = np.exp([0.0, -2.0])
    np.testing.assert_allclose(out[2], e / e.sum(), rtol=1e-6)


# ---------------------------------------------------------------- stage 1
def test_stage1_spec_example_and_edges(oracle):
    codes, s = oracle.quant_sym8(np.array([1.0, -2.0, 3.0]))
    assert s == np.float32(3.0) / np.float32(119.0)
    assert codes.tolist() == [40, -79, 119]
    codes, s = oracle.quant_sym8(np.zeros(16))
    assert s == 0 and not codes.any()
    codes, s = oracle.quant_sym8(np.array([119.0, -5.0]))
    assert s == 1.0 and codes.tolist() == [119, -5]


def test_stage1_round_trip_bound(oracle):
    """|x - s code| <= s (1/2 + 2^-15); codes in [-119, 119]; the max-abs element
    maps to +-119 (invariants of round-to-nearest with the 119 divisor)."""
    rng = np.random.default_rng(7)
    for it in range(300):
        scale = 10.0 ** rng.uniform(-3, 3)
        x = (rng.standard_normal((64, 16)) * scale).astype(np.float16).astype(np.float32)
        codes, s = oracle.quant_sym8(x)
        assert codes.min() >= -119 and codes.max() <= 119
        err = np.abs(x.astype(np.float64) - float(s) * codes.astype(np.float64))
        assert err.max() <= float(s) * (0.5 + 2.0 ** -15)
        i = np.unravel_index(np.argmax(np.abs(x)), x.shape)
        assert abs(int(codes[i])) == 119


# ---------------------------------------------------------------- stage 2
@pytest.mark.parametrize("bits", [2, 4])
def test_stage2_exhaustive(oracle, bits):
    """All 28,680 (min, max) INT8 ranges, every value: no code overflow, error <=
    floor(s/2), reconstruction stays in INT8 ([-119, 127]) so dequant is linear."""
    L = (1 << bits) - 1
    for mn in range(-119, 120):
        for mx in range(mn, 120):
            g = np.arange(mn, mx + 1, dtype=np.int8)
            codes, s, z = oracle.quant_asym(g, bits)
            assert z == mn and 1 <= s <= 80
            assert codes.max() <= L
            rec = codes.astype(np.int32) * s + z
            assert rec.min() >= -119 and rec.max() <= 127
            assert np.abs(rec - g.astype(np.int32)).max() <= s // 2


def test_stage2_worked_examples(oracle):
    for case in GOLD["W0_stage2"]:
        codes, s, z = oracle.quant_asym(np.array(case["group"], np.int8), case["bits"])
        assert (s, z, codes.tolist()) == (case["s_int"], case["z_int"], case["codes"])
        assert [oracle.dequant_q2(c, s, z) for c in codes] == case["dequant"]


def test_stage2_mse_monotone_in_bits(oracle):
    rng = np.random.default_rng(3)
    for _ in range(200):
        g = np.clip(np.rint(rng.standard_normal(64) * 40), -119, 119).astype(np.int8)
        errs = []
        for bits in (2, 4):
            c, s, z = oracle.quant_asym(g, bits)
            errs.append(np.mean((c.astype(np.int32) * s + z - g.astype(np.int32)) ** 2))
        assert errs[0] >= errs[1]


def test_eq5_fold_identity(oracle):
    """Eq. 5 (with the inner-dim factor K on z_a z_b) and the
    decode fold: sum q1 (code s + z) == sum (q1 s) code + sum q1 z, exactly."""
    rng = np.random.default_rng(5)
    for _ in range(50):
        d = 128
        g = rng.integers(-119, 120, (64, d)).astype(np.int8)
        q1 = rng.integers(-119, 120, d).astype(np.int64)
        codes = np.zeros((64, d), np.int64)
        s = np.zeros(d, np.int64)
        z = np.zeros(d, np.int64)
        for c in range(d):
            cc, s[c], z[c] = oracle.quant_asym(g[:, c], 4)
            codes[:, c] = cc
        deq = np.array([[oracle.dequant_q2(codes[t, c], s[c], z[c]) for c in range(d)] for t in range(4)])
        lhs = deq @ q1
        rhs = codes[:4] @ (q1 * s) + (q1 * z).sum()
        np.testing.assert_array_equal(lhs, rhs)
    a, sa, za, b, sb, zb = 3, 1.0, 2.0, 4, 1.0, 1.0  # SPEC-style 1x1 four-term check
    assert (a * sa + za) * (b * sb + zb) == sa * sb * a * b + sa * zb * a + sb * za * b + 1 * za * zb == 25


# ---------------------------------------------------------------- cache
def test_cache_prefill_tail_append_flush(oracle):
    p = oracle.params(d=64)
    rng = np.random.default_rng(11)
    x = rng.standard_normal((200, 64)).astype(np.float16).astype(np.float32)
    sl = oracle.Slot(p, 4, 8)
    x1, sc = sl.prefill(x)
    assert sl.n_blocks == 3 and sl.n_buf == 8 and len(sc) == 4
    a = np.float32(np.abs(x).max())
    assert sl.a_univ == a
    # tail tokens re-quantised with the universal scale (R-11)
    inv = np.float32(119.0) / a
    np.testing.assert_array_equal(sl.buf[:8], np.rint(x[192:].astype(np.float64) * np.float64(inv)).astype(np.int8))
    # full blocks: parent scale = block stage-1 scale, codes == stage-2 of x1
    for j in range(3):
        assert sl.s_parent[j] == sc[j]
        for c in range(0, 64, 7):
            codes, s, z = oracle.quant_asym(x1[j * 64:(j + 1) * 64, c], 4)
            np.testing.assert_array_equal(sl.codes[j, :, c], codes)
            assert (sl.s_int[j, c], sl.z_int[j, c]) == (s, z)
    # appends: outliers clamp to +-119, flush at n_b = B_c with parent s_univ
    for t in range(56):
        tok = x[t] * (20.0 if t == 0 else 1.0)
        sl.append(tok)
    assert sl.n_blocks == 4 and sl.n_buf == 0
    assert sl.s_parent[3] == a / np.float32(119.0)
    buf_block = sl.dequant_block(3)
    assert buf_block.min() >= -119 and buf_block.max() <= 127


def test_compression_ratio(oracle):
    """KV size reduction > 4.4x for the mixed 2/4-bit plan at
    B_c = 64, d = 128: bytes/token/kv-head K+V = 136.125 (4b), 72.125 (2b)."""
    d, bc = 128, 64
    p = oracle.params(d=d)
    per_tok = {}
    for bits in (2, 4):
        sl = oracle.Slot(p, bits, 1)
        meta = sl.s_int[0].nbytes + sl.z_int[0].nbytes + sl.s_parent[:1].nbytes
        per_tok[bits] = 2 * (sl.codes[0].size * bits / 8 + meta) / bc
    assert per_tok[4] == 136.125 and per_tok[2] == 72.125
    mixed = (per_tok[4] + per_tok[2]) / 2
    assert 2 * d * 2 / mixed > 4.4
    assert abs(2 * d * 2 / mixed - 4.917) < 1e-3


# ---------------------------------------------------------------- attention
def test_worked_example_W1_W2_W3(oracle):
    """tests/golden/worked_example.json (Alg. 1 by hand)."""
    q = np.array([[1, 0]] * 3, np.float32)
    k = np.array(GOLD["setup"]["K"], np.float32)
    v = np.array(GOLD["setup"]["V"], np.float32)
    p = oracle.params(d=2, block_kv=64)
    o, l, tap = oracle.prefill_head(p, q, k, v, causal=False, tap=(0, 0))
    w1 = GOLD["W1_Bc64"]
    assert tap["q1"][0].tolist() == w1["q1"]
    assert tap["s_int"][0, :3].tolist() == w1["S_int"]
    np.testing.assert_allclose(tap["p_tilde"][0, :3], w1["p_tilde"], rtol=2e-7)
    assert tap["p_codes"][0, :3].tolist() == w1["p_codes"]
    assert tap["pv_int"][0].tolist() == w1["pv_int"]
    np.testing.assert_allclose(o[0], w1["O"], atol=2e-7)
    assert abs(l[0] - w1["L"]) < 2e-7
    for key, bc, am in (("W2_Bc2_alpha0", 2, 0), ("W3_Bc2_alpha1", 2, 1)):
        p = oracle.params(d=2, block_kv=bc, alpha_mode=am)
        o, l = oracle.prefill_head(p, q, k, v, causal=False)
        np.testing.assert_allclose(o[0], GOLD[key]["O"], atol=3e-7)
        assert abs(l[0] - GOLD[key]["L"]) < 2e-7
    oref, lref = oracle.reference_attention(q[:1], k, v, causal=False)
    np.testing.assert_allclose(oref[0], GOLD["exact_softmax"]["O"], atol=1e-7)


@pytest.mark.parametrize("bq,bk", [(64, 64), (64, 128), (128, 64), (128, 128)])
@pytest.mark.parametrize("causal", [True, False])
def test_exact_mode_reduces_to_fp64_attention(oracle, bq, bk, causal):
    """Pin P5: with quantisation off and SAS -> exp, the tiled online recurrence
    (tiling, masking, alpha chaining, scale placement) equals Eq. 2 in FP64."""
    for n in (1, 63, 64, 65, 256):
        q, k, v = synth.qkv(100 + n, 1, n, 1, 1, 64)
        q, k, v = (a[0, :, 0].astype(np.float32) for a in (q, k, v))
        p = oracle.params(d=64, block_q=bq, block_kv=bk, quant=0, sas=0)
        o, l = oracle.prefill_head(p, q, k, v, causal=causal)
        oref, lref = oracle.reference_attention(q, k, v, causal=causal, scale=float(p.softmax_scale))
        assert rel_l2(o, oref) < 1e-5, n
        np.testing.assert_allclose(l, lref, rtol=1e-6, atol=1e-6)


def test_exact_mode_decode_splits_and_combine(oracle):
    """Pin P5 for Alg. 2 + the split-KV combine: any split of the cache blocks,
    combined by log-sum-exp, equals FP64 attention of the query over all keys."""
    d, bc = 128, 64
    q, k, v = synth.qkv(9, 1, 1000, 1, 1, d)
    k, v = k[0, :, 0].astype(np.float32), v[0, :, 0].astype(np.float32)
    q = q[0, 0, 0].astype(np.float32)
    p = oracle.params(d=d, block_kv=bc, quant=0, sas=0)
    ks, vs = oracle.Slot(p, 4, 32), oracle.Slot(p, 4, 32)
    ks.prefill(k)
    vs.prefill(v)
    oref, lref = oracle.reference_attention(q[None], k, v, causal=False, scale=float(p.softmax_scale))
    nb = ks.n_blocks
    for bounds in ([0, nb], [0, 5, nb], [0, 1, 7, 8, nb], [0, 3, 3, nb]):
        parts, lses = [], []
        for s in range(len(bounds) - 1):
            last = s == len(bounds) - 2
            o, l = oracle.decode_head(p, q, ks, vs, bounds[s], bounds[s + 1], last, k_raw=k, v_raw=v)
            parts.append(o)
            lses.append(l)
        o, l = oracle.combine(np.stack(parts), np.array(lses))
        assert rel_l2(o, oref[0]) < 1e-5
        assert abs(l - lref[0]) < 1e-5


def test_closed_form_one_key_and_uniform_scores(oracle):
    """(i) one key: O = s_V v1; (ii) q = 0 -> all scores equal -> O = mean of the
    dequantised V rows (P~ constant, all P codes 119)."""
    d = 64
    p = oracle.params(d=d)
    rng = np.random.default_rng(1)
    k = rng.standard_normal((1, d)).astype(np.float16).astype(np.float32)
    v = rng.standard_normal((1, d)).astype(np.float16).astype(np.float32)
    q = rng.standard_normal((1, d)).astype(np.float16).astype(np.float32)
    o, l = oracle.prefill_head(p, q, k, v, causal=True)
    v1, sv = oracle.quant_sym8(v)
    np.testing.assert_allclose(o[0], sv * v1[0].astype(np.float64), rtol=1e-6, atol=1e-7)
    n = 50
    v = rng.standard_normal((n, d)).astype(np.float16).astype(np.float32)
    k = rng.standard_normal((n, d)).astype(np.float16).astype(np.float32)
    q = np.zeros((n, d), np.float32)
    o, l, tap = oracle.prefill_head(p, q, k, v, causal=False, tap=(0, 0))
    assert (tap["p_codes"][:n, :n] == 119).all()
    v1, sv = oracle.quant_sym8(v)
    np.testing.assert_allclose(o[7], sv * v1.astype(np.float64).mean(0), rtol=1e-5, atol=1e-7)


def test_threshold_sparsity_invariant(oracle):
    """Pin P2: P~ == 0 exactly where x - m_new < n_r or the key is masked, and
    every kept P~ >= LUT[5] POLY(1^-)."""
    d, n = 64, 256
    q, k, v = synth.qkv(21, 1, n, 1, 1, d)
    q, k, v = (a[0, :, 0].astype(np.float32) * 3 for a in (q, k, v))
    p = oracle.params(d=d)
    k1s = oracle.Slot(p, 4, 8).prefill(k)[1]
    for (i, j) in ((3, 1), (3, 3), (2, 0)):
        o, l, tap = oracle.prefill_head(p, q, k, v, causal=True, tap=(i, j))
        cqk = np.float32(np.float32(tap["s_q"][0] * k1s[j]) * p.softmax_scale)
        x = tap["s_int"].astype(np.float32) * cqk
        rows = np.arange(64)[:, None] + 64 * i
        cols = np.arange(64)[None, :] + 64 * j
        pruned = (tap["m_new"][:, None] - x > 6) | (cols > rows)
        pt = tap["p_tilde"]
        np.testing.assert_array_equal(pt == 0, pruned)
        assert pt[~pruned].min() >= 2.47e-3
        assert pruned.sum() > 0 or i == 2


def test_config1_error_vs_exact_attention(oracle):
    """Pin P7 (config 1: B=1, N=128, d=64, causal): the approximation's distance
    from FP64 softmax attention, frozen bound (parity of the approximation
    itself is unpinned by the paper -- DESIGN.md §5)."""
    q, k, v = synth.qkv(1001, 1, 128, 1, 1, 64)
    q, k, v = (a[0, :, 0].astype(np.float32) for a in (q, k, v))
    p = oracle.params(d=64)
    o, l = oracle.prefill_head(p, q, k, v, causal=True)
    oref, lref = oracle.reference_attention(q, k, v, causal=True, scale=float(p.softmax_scale))
    # frozen after the first verified run: 4.30e-2 / 0.151 on this seed (outlier head)
    assert rel_l2(o, oref) < 5e-2
    assert np.abs(l - lref).max() < 0.2


def test_block_size_robustness(oracle):
    """Pin P10 (block-size table): error vs exact within 3x
    across (B_r, B_c) in {64,128}^2."""
    q, k, v = synth.qkv(1002, 1, 512, 1, 1, 64)
    q, k, v = (a[0, :, 0].astype(np.float32) for a in (q, k, v))
    errs = []
    oref, _ = oracle.reference_attention(q, k, v, causal=True)
    for bq in (64, 128):
        for bk in (64, 128):
            p = oracle.params(d=64, block_q=bq, block_kv=bk)
            o, _ = oracle.prefill_head(p, q, k, v, causal=True)
            errs.append(rel_l2(o, oref))
    assert max(errs) < 3 * min(errs)


def test_causal_independence(oracle):
    """Pin P11: changing K/V in blocks after the last block a query block can see
    leaves that query block bit-identical."""
    d, n = 64, 320
    q, k, v = synth.qkv(31, 1, n, 1, 1, d)
    q, k, v = (a[0, :, 0].astype(np.float32) for a in (q, k, v))
    p = oracle.params(d=d)
    o1, l1 = oracle.prefill_head(p, q, k, v, causal=True)
    k2, v2 = k.copy(), v.copy()
    k2[192:] *= -3.0
    v2[192:] += 1.0
    o2, l2 = oracle.prefill_head(p, q, k2, v2, causal=True)
    np.testing.assert_array_equal(o1[:192], o2[:192])
    np.testing.assert_array_equal(l1[:192], l2[:192])
    assert not np.array_equal(o1[192:], o2[192:])


def test_split_deviation_alpha_modes(oracle):
    """Pin P12 (trend-V probe, V = position/N + noise): splitting the cache into
    4 ranges + LSE combine moves the decode output by less than half of the
    method's own distance from exact attention, in both alpha modes."""
    d, n = 128, 4096 + 17
    q, k, _ = synth.qkv(41, 1, n, 1, 1, d)
    k = k[0, :, 0].astype(np.float32)
    q = q[0, 0, 0].astype(np.float32)
    rng = np.random.default_rng(0)
    v = (np.arange(n)[:, None] / n + 0.1 * rng.standard_normal((n, d))).astype(np.float16).astype(np.float32)
    oref, _ = oracle.reference_attention(q[None], k, v, causal=False)
    for mode in (0, 1):
        p = oracle.params(d=d, alpha_mode=mode)
        ks, vs = oracle.Slot(p, 4, 80), oracle.Slot(p, 2, 80)
        ks.prefill(k)
        vs.prefill(v)
        full, _ = oracle.decode_head(p, q, ks, vs)
        cuts = [0, 16, 32, 48, 64]
        parts = [oracle.decode_head(p, q, ks, vs, cuts[s], cuts[s + 1], s == 3) for s in range(4)]
        o, _ = oracle.combine(np.stack([a for a, _ in parts]), np.array([b for _, b in parts]))
        assert rel_l2(o, full) < 0.5 * rel_l2(full, oref[0])


def test_head_priority_planner(oracle):
    """priority = gap x std of channel gaps: equal channel
    ranges -> std 0 -> lowest priority -> 2 bits."""
    rng = np.random.default_rng(2)
    flat = np.tile(np.array([[-1.0], [1.0]], np.float32), (1, 8))
    outl = rng.standard_normal((16, 8)).astype(np.float32)
    outl[:, 3] *= 10
    pr = [oracle.head_priority(flat), oracle.head_priority(outl)]
    assert pr[0] == 0.0 and pr[1] > 0
    g = outl.max(0) - outl.min(0)
    assert abs(pr[1] - (outl.max() - outl.min()) * g.std()) < 1e-4 * pr[1]
    assert oracle.plan_bits([3.0, 1.0, 1.0, 5.0], 2).tolist() == [4, 2, 2, 4]


def test_prefill_query_block_subset(oracle):
    """Alg. 1's outer loop over query blocks is independent: running
    only blocks [i0, i1) reproduces those rows of the full run bit-for-bit and
    leaves the others untouched (used by the full-size sampled GPU parity)."""
    for causal in (True, False):
        q, k, v = synth.qkv(31, 1, 64 * 5 + 17, 1, 1, 64)
        p = oracle.params(d=64)
        full, lf = oracle.prefill_head(p, q[0, :, 0], k[0, :, 0], v[0, :, 0], causal=causal)
        part, lp = oracle.prefill_head(p, q[0, :, 0], k[0, :, 0], v[0, :, 0], causal=causal, blocks=(2, 6))
        np.testing.assert_array_equal(part[128:], full[128:])
        np.testing.assert_array_equal(lp[128:], lf[128:])
        assert not part[:128].any() and not lp[:128].any()


def test_scale_fp16_variant_rounds_every_first_stage_scale(oracle):
    """NEXT-2 variant scale_fp16 (P:297 FP16 first-stage scales, R-29): each stored block scale is
    the binary16 round-to-nearest-even of the FP32 scale max|x|/119 -- checked against numpy's own
    float16 conversion over blocks whose scales span normal and subnormal binary16 (amax 2^-20 ...
    2^10) -- the codes are unchanged, the parent scales and the buffer scale a_univ/119 follow."""
    rng = np.random.default_rng(5)
    d = 64
    for e in range(-20, 11, 3):
        x = (rng.standard_normal((64 * 3 + 17, d)) * 2.0 ** e).astype(np.float16).astype(np.float32)
        p32, p16 = oracle.params(d=d), oracle.params(d=d, scale_fp16=1)
        s32, s16 = oracle.Slot(p32, 4, 8), oracle.Slot(p16, 4, 8)
        x1a, sca = s32.prefill(x)
        x1b, scb = s16.prefill(x)
        np.testing.assert_array_equal(x1a, x1b)  # codes unchanged
        np.testing.assert_array_equal(scb, sca.astype(np.float16).astype(np.float32))
        np.testing.assert_array_equal(s16.s_parent[:3], scb[:3])
        assert np.abs(scb - sca).max() <= np.abs(sca).max() * 2.0 ** -11 + 2.0 ** -25
        # a flushed buffer block takes fp16(a_univ / 119) as its parent scale
        for t in range(64 - 17):
            s16.append(x[t])
        assert s16.n_blocks == 4 and s16.n_buf == 0
        parent = np.float32(s16.a_univ) / np.float32(119.0)
        assert s16.s_parent[3] == np.float32(np.float16(parent))


def test_scale_fp16_variant_attention_changes_little(oracle):
    """The FP16 scales move the prefill and the decode outputs by far less than the method's own
    distance from exact attention (the variant is a storage-format choice, not a different
    method), and they do move them (the flag is live)."""
    d, n = 128, 200
    q, k, v = synth.qkv(6, 1, n, 1, 1, d)
    q, k, v = (x[0, :, 0].astype(np.float32) for x in (q, k, v))
    o32, _ = oracle.prefill_head(oracle.params(d=d), q, k, v)
    o16, _ = oracle.prefill_head(oracle.params(d=d, scale_fp16=1), q, k, v)
    ex, _ = oracle.reference_attention(q, k, v, causal=True)
    assert 0 < rel_l2(o16, o32) < 0.1 * rel_l2(o32, ex)
    res = {}
    for f in (0, 1):
        p = oracle.params(d=d, scale_fp16=f)
        ks, vs = oracle.Slot(p, 4, 8), oracle.Slot(p, 2, 8)
        ks.prefill(k)
        vs.prefill(v)
        res[f] = oracle.decode_head(p, q[-1], ks, vs)[0]
    assert 0 < rel_l2(res[1], res[0]) < 1e-2


def test_scale_fp16_variant_ties_to_even(oracle):
    """R-29's binary16 rounding on exact ties: block maxima chosen so that fl(max/119) lies exactly
    halfway between two binary16 values; the stored scale must be the even one (numpy float16)."""
    d, hits = 64, 0
    p16 = oracle.params(d=d, scale_fp16=1)
    for k, q in ((1024, -12), (1536, -10), (2046, -8), (1110, -14), (1300, -20), (1998, -6)):
        # k even (11 bits): k + 1/2 is halfway between two binary16 values; ties-to-even keeps k,
        # rounding half away from zero would give k + 1
        s_tie = np.float32(np.ldexp(k + 0.5, q))
        a = np.float32(s_tie * np.float32(119.0))
        for _ in range(64):  # nudge a until fl(a / 119) is exactly the tie
            if np.float32(a / np.float32(119.0)) == s_tie:
                break
            a = np.nextafter(a, np.float32(np.inf) if np.float32(a / np.float32(119.0)) < s_tie else np.float32(0))
        if np.float32(a / np.float32(119.0)) != s_tie:
            continue
        x = np.zeros((64, d), np.float32)
        x[3, 5] = a
        x[10, 7] = -a / 3
        sl = oracle.Slot(p16, 4, 2)
        _, sc = sl.prefill(x)
        assert sc[0] == np.float32(np.float16(s_tie)) == np.float32(np.ldexp(k, q)), (k, q)
        hits += 1
    assert hits >= 4
