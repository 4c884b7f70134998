"""GPU parity at the edges of the parameter space and of the data (-m gpu).

* the SAS threshold n_r over the whole accepted range (LUT lanes
  up to 30) for prefill and decode;
* all-zero K / V / Q blocks (stage-1 s = 0 branch, R-5) and a zero decode query
  (every P code 119);
* appended tokens beyond the universal max (the +-119 clamp);
* alpha_mode = 1 and B_r = 128 at N >= 2048, d = 64 at N = 4096 (sampled heads);
* the per-row prefill P scale (NEXT-2 variant p_scale_rows, oracle flag p_row).
Same bar as tests/test_gpu_parity.py.
"""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2412_08585_b200 import synth
from tests import cache_layout
from tests.test_gpu_parity import _oracle_decode, assert_out_close

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ta():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2412_08585_b200 import binding

    binding.lib()
    return binding


def _prefill(ta, p, q, k, v, bits, causal=True):
    B, N, Hq, d = q.shape
    Hkv = k.shape[2]
    cache = ta.KVCache(B, Hkv, d, max_blocks=N // 64 + 2, bits=bits)
    qt, kt, vt = (torch.from_numpy(x).cuda() for x in (q, k, v))
    k1, v1t, k1s, v1s = ta.turbo_quantize_kv(p, cache, kt, vt)
    o, lse = ta.turbo_attention_prefill(p, qt, k1, v1t, k1s, v1s, causal=causal)
    torch.cuda.synchronize()
    return cache, k1, o.cpu().numpy(), lse.cpu().numpy()


def _check_prefill_heads(op, q, k, v, o, lse, heads, causal=True, blocks=None):
    G = q.shape[2] // k.shape[2]
    for b, h in heads:
        oref, lref = O.prefill_head(op, q[b, :, h], k[b, :, h // G], v[b, :, h // G], causal=causal, blocks=blocks)
        r0 = 0 if blocks is None else blocks[0] * op.block_q
        assert_out_close(o[b, r0:, h], oref[r0:], f"b{b} h{h}")
        np.testing.assert_allclose(lse[b, h, r0:], lref[r0:], atol=1e-4, rtol=1e-5)


@pytest.mark.parametrize("nr", [-1, -3, -6, -12, -30])
def test_prefill_sas_threshold_range(ta, nr):
    B, N, Hq, Hkv, d = 1, 333, 4, 2, 128
    q, k, v = synth.qkv(4100 - nr, B, N, Hq, Hkv, d)
    bits = synth.head_bits_alternating(Hkv)
    p = ta.params(head_dim=d, sas_nr=nr)
    _, _, o, lse = _prefill(ta, p, q, k, v, bits)
    _check_prefill_heads(O.params(d=d, sas_nr=nr), q, k, v, o, lse, [(0, h) for h in range(Hq)])


def _decode_setup(ta, p, op, q, k, v, bits, appends=()):
    B, N, Hkv, d = k.shape
    maxb = (N + len(appends)) // 64 + 2
    cache = ta.KVCache(B, Hkv, d, max_blocks=maxb, bits=bits)
    ta.turbo_quantize_kv(p, cache, torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda())
    ref = O.build_cache(op, k.astype(np.float32), v.astype(np.float32), bits, maxb)
    for kt, vt in appends:
        ta.turbo_quantize_kv(p, cache, torch.from_numpy(kt).cuda(), torch.from_numpy(vt).cuda(), mode=1)
        for b in range(B):
            for h in range(Hkv):
                ref["slots"][b][h][0].append(kt[b, h].astype(np.float32))
                ref["slots"][b][h][1].append(vt[b, h].astype(np.float32))
    return cache, ref


def _check_decode(ta, p, op, cache, ref, qd, G, S=1):
    o, _, lse = ta.turbo_attention_decode(p, cache, torch.from_numpy(qd).cuda(), n_splits=S)
    torch.cuda.synchronize()
    o, lse = o.cpu().numpy(), lse.cpu().numpy()
    nb = ref["slots"][0][0][0].n_blocks
    per = -(-nb // S)
    bounds = [(min(s * per, nb), min(s * per + per, nb)) for s in range(S)]
    for b in range(qd.shape[0]):
        ro, rl = _oracle_decode(op, qd[b].astype(np.float32), ref["slots"][b], G, bounds)
        assert_out_close(o[b], ro, f"decode b{b}")
        np.testing.assert_allclose(lse[b], rl, atol=1e-4, rtol=1e-5)


@pytest.mark.parametrize("nr", [-1, -3, -12, -30])
def test_decode_sas_threshold_range(ta, nr):
    B, N, Hq, Hkv, d = 2, 64 * 6 + 21, 8, 2, 128
    q, k, v = synth.qkv(4200 - nr, B, N, Hq, Hkv, d)
    bits = synth.head_bits_alternating(Hkv)
    p, op = ta.params(head_dim=d, sas_nr=nr), O.params(d=d, sas_nr=nr)
    cache, ref = _decode_setup(ta, p, op, q, k, v, bits)
    qd, _, _ = synth.decode_token(4300, B, Hq, Hkv, d)
    _check_decode(ta, p, op, cache, ref, qd, Hq // Hkv, S=2)


def test_zero_blocks_prefill_and_decode(ta):
    """All-zero K block, V block and Q rows: stage-1 s = 0, codes 0 (R-5); a zero
    decode query: every score 0, every P code 119."""
    B, N, Hq, Hkv, d = 1, 64 * 5 + 10, 4, 2, 128
    q, k, v = synth.qkv(4400, B, N, Hq, Hkv, d)
    k[0, 64:128, 0] = 0
    v[0, 128:192, 1] = 0
    v[0, 256:, 0] = 0          # zero tail (buffer) of one V stream
    q[0, 64:128, 1] = 0        # a zero Q block (one B_r block of head 1)
    bits = synth.head_bits_alternating(Hkv)
    p = ta.params(head_dim=d)
    op = O.params(d=d)
    cache, k1, o, lse = _prefill(ta, p, q, k, v, bits)
    assert not k1[0, 0, 64:128].any()
    _check_prefill_heads(op, q, k, v, o, lse, [(0, h) for h in range(Hq)])
    cache, ref = _decode_setup(ta, p, op, q, k, v, bits)
    recs = cache.records().cpu().numpy()
    for h in range(Hkv):
        for kind, sl in enumerate(ref["slots"][0][h]):
            for j in range(sl.n_blocks):
                codes, s_int, z_int = cache_layout.unpack_record(recs[0, h, kind, j], d, int(bits[h][kind]), kind)
                np.testing.assert_array_equal(codes, sl.codes[j])
                np.testing.assert_array_equal(s_int, sl.s_int[j])
                np.testing.assert_array_equal(z_int, sl.z_int[j])
    qd, _, _ = synth.decode_token(4401, B, Hq, Hkv, d)
    qd[0, 2] = 0
    _check_decode(ta, p, op, cache, ref, qd, Hq // Hkv, S=1)
    tap = ta.DebugTap(0, 2, 0, 1, d, decode=True)
    pt = ta.params(head_dim=d, debug_tap=tap)
    ta.turbo_attention_decode(pt, cache, torch.from_numpy(qd).cuda(), n_splits=1)
    torch.cuda.synchronize()
    assert (tap.p_codes.cpu().numpy()[0] == 119).all()


def test_append_clamp_beyond_universal_scale(ta):
    """Appended tokens with |x| up to 8x the prefill distribution: codes clamp at +-119;
    the cache (buffer and the flushed block) and the decode match the oracle."""
    B, N, Hq, Hkv, d = 2, 64 * 3 + 50, 8, 2, 128
    q, k, v = synth.qkv(4500, B, N, Hq, Hkv, d)
    bits = synth.head_bits_alternating(Hkv)
    p, op = ta.params(head_dim=d), O.params(d=d)
    apps = []
    for t in range(20):
        _, kt, vt = synth.decode_token(4600 + t, B, Hq, Hkv, d)
        if t % 3 == 0:
            kt = (kt.astype(np.float32) * 8).astype(np.float16)
            vt = (vt.astype(np.float32) * 8).astype(np.float16)
        apps.append((kt, vt))
    cache, ref = _decode_setup(ta, p, op, q, k, v, bits, apps)
    assert sum((np.abs(sl.buf[:sl.n_buf]) == 119).sum() for r in ref["slots"] for hh in r for sl in hh) > 8
    buf = cache.buf.view(B, Hkv, 2, 64 * d).cpu().numpy()
    cnt = cache.counters.view(B, 2).cpu().numpy()
    recs = cache.records().cpu().numpy()
    for b in range(B):
        for h in range(Hkv):
            for kind, sl in enumerate(ref["slots"][b][h]):
                assert tuple(cnt[b]) == (sl.n_blocks, sl.n_buf)
                bb = buf[b, h, kind].reshape(64, d) if kind == 0 else buf[b, h, kind].reshape(d, 64).T
                np.testing.assert_array_equal(bb[:sl.n_buf], sl.buf[:sl.n_buf])
                j = sl.n_blocks - 1  # the block flushed from the buffer during the appends
                codes, s_int, z_int = cache_layout.unpack_record(recs[b, h, kind, j], d, int(bits[h][kind]), kind)
                np.testing.assert_array_equal(codes, sl.codes[j])
                np.testing.assert_array_equal(s_int, sl.s_int[j])
                np.testing.assert_array_equal(z_int, sl.z_int[j])
    qd, _, _ = synth.decode_token(4700, B, Hq, Hkv, d)
    _check_decode(ta, p, op, cache, ref, qd, Hq // Hkv, S=2)


@pytest.mark.parametrize("N,d,bq,am", [(2048, 128, 64, 1), (2048, 128, 128, 0), (2304, 128, 128, 1),
                                       (4096, 64, 64, 0)])
def test_prefill_long_sampled(ta, N, d, bq, am):
    """Long sequences for the configurations the small cases reach only at N <= 333:
    alpha_mode 1, B_r = 128, d = 64 (its own swizzle) -- two sampled heads, last query
    blocks (the longest key walks) against the oracle."""
    B, Hq, Hkv = 1, 4, 2
    q, k, v = synth.qkv(4800 + N + d, B, N, Hq, Hkv, d)
    bits = synth.head_bits_alternating(Hkv)
    p = ta.params(head_dim=d, block_q=bq, alpha_mode=am)
    _, _, o, lse = _prefill(ta, p, q, k, v, bits)
    op = O.params(d=d, block_q=bq, alpha_mode=am)
    nblk = N // bq
    _check_prefill_heads(op, q, k, v, o, lse, [(0, 0), (0, Hq - 1)], blocks=(nblk - 2, nblk))


PROW_CASES = [  # (B, N, Hq, Hkv, d, causal, block_q, alpha_mode)
    (1, 128, 1, 1, 64, True, 64, 0),
    (2, 200, 8, 2, 128, True, 64, 0),
    (1, 333, 4, 4, 128, False, 64, 1),
    (1, 256, 2, 1, 64, True, 128, 0),
    (1, 520, 6, 2, 128, True, 64, 1),
]


@pytest.mark.parametrize("case", PROW_CASES)
def test_prefill_row_p_scale_parity(ta, case):
    """NEXT-2 variant: P scale per row x B_c block in the prefill (p_scale_rows = 1)."""
    B, N, Hq, Hkv, d, causal, bq, am = case
    q, k, v = synth.qkv(5100 + N, B, N, Hq, Hkv, d)
    bits = synth.head_bits_alternating(Hkv)
    p = ta.params(head_dim=d, block_q=bq, alpha_mode=am, p_scale_rows=1)
    _, _, o, lse = _prefill(ta, p, q, k, v, bits, causal=causal)
    op = O.params(d=d, block_q=bq, alpha_mode=am, p_row=1)
    _check_prefill_heads(op, q, k, v, o, lse, [(b, h) for b in range(B) for h in range(Hq)], causal=causal)


def test_prefill_row_p_scale_tap(ta):
    B, N, Hq, Hkv, d = 1, 300, 4, 2, 128
    q, k, v = synth.qkv(5200, B, N, Hq, Hkv, d)
    bits = synth.head_bits_alternating(Hkv)
    b, h, i, j = 0, 3, 3, 2
    tap = ta.DebugTap(b, h, i, j, d)
    p = ta.params(head_dim=d, debug_tap=tap, p_scale_rows=1)
    _prefill(ta, p, q, k, v, bits)
    _, _, rt = O.prefill_head(O.params(d=d, p_row=1), q[b, :, h], k[b, :, h // 2], v[b, :, h // 2], causal=True,
                              tap=(i, j))
    rows = min(64, N - 64 * i)
    np.testing.assert_array_equal(tap.s_int.cpu().numpy()[:rows], rt["s_int"][:rows])
    np.testing.assert_array_equal(tap.p_codes.cpu().numpy()[:rows], rt["p_codes"][:rows])
    np.testing.assert_array_equal(tap.pv_int.cpu().numpy()[:rows], rt["pv_int"][:rows])
    assert tap.s_p.item() == rt["s_p"][0]


@pytest.mark.parametrize("d,bq", [(128, 64), (64, 128)])
def test_scale_fp16_variant_prefill(ta, d, bq):
    """NEXT-2 variant scale_fp16 (R-29): stage-1 K/V scales and parent scales bit-exact
    binary16 values, codes identical to the FP32 build, prefill output within tolerance of the
    oracle with the same flag; Q's scale too (through the output)."""
    B, N, Hq, Hkv = 2, 64 * 5 + 29, 4, 2
    q, k, v = synth.qkv(5300 + d, B, N, Hq, Hkv, d)
    k[:, :, 1] *= 1e-3  # small scales: binary16 near its subnormal range
    bits = synth.head_bits_alternating(Hkv)
    p = ta.params(head_dim=d, block_q=bq, scale_fp16=1)
    cache, k1, o, lse = _prefill(ta, p, q, k, v, bits)
    op = O.params(d=d, block_q=bq, scale_fp16=1)
    ref = O.build_cache(op, k.astype(np.float32), v.astype(np.float32), bits, N // 64 + 2)
    np.testing.assert_array_equal(k1.cpu().numpy(), ref["k1"])
    sp = cache.s_parent.view(B, Hkv, 2, -1).cpu().numpy()
    for b in range(B):
        for h in range(Hkv):
            for kind, sl in enumerate(ref["slots"][b][h]):
                np.testing.assert_array_equal(sp[b, h, kind, :sl.n_blocks], sl.s_parent[:sl.n_blocks])
                assert (sp[b, h, kind, :sl.n_blocks] == sp[b, h, kind, :sl.n_blocks].astype(np.float16)).all()
    _check_prefill_heads(op, q, k, v, o, lse, [(b, h) for b in range(B) for h in range(Hq)])


def test_scale_fp16_variant_decode_with_flush(ta):
    """scale_fp16 through appends that flush the buffer (parent fp16(a_univ / 119)) and the buffer
    block's scales, equal splits and the default schedule."""
    B, N, Hq, Hkv, d = 2, 64 * 4 + 50, 8, 2, 128
    q, k, v = synth.qkv(5400, B, N, Hq, Hkv, d)
    bits = synth.head_bits_alternating(Hkv)
    p, op = ta.params(head_dim=d, scale_fp16=1), O.params(d=d, scale_fp16=1)
    apps = [synth.decode_token(5500 + t, B, Hq, Hkv, d)[1:] for t in range(20)]
    cache, ref = _decode_setup(ta, p, op, q, k, v, bits, apps)
    sp = cache.s_parent.view(B, Hkv, 2, -1).cpu().numpy()
    sl = ref["slots"][1][1][1]
    np.testing.assert_array_equal(sp[1, 1, 1, :sl.n_blocks], sl.s_parent[:sl.n_blocks])
    qd, _, _ = synth.decode_token(5600, B, Hq, Hkv, d)
    _check_decode(ta, p, op, cache, ref, qd, Hq // Hkv, S=1)
    _check_decode(ta, p, op, cache, ref, qd, Hq // Hkv, S=3)


SF_CASES = [  # (B, N, Hq, Hkv, d, causal, block_q, alpha_mode, block_kv)
    (2, 200, 8, 2, 128, True, 64, 0, 64),
    (1, 333, 4, 4, 128, False, 64, 1, 64),
    (1, 256, 2, 1, 64, True, 128, 0, 64),
    (2, 700, 3, 3, 128, True, 64, 0, 64),
    (1, 300, 8, 2, 128, True, 64, 1, 128),
]


@pytest.mark.parametrize("case", SF_CASES)
def test_sas_fp16_variant_prefill(ta, case):
    """NEXT-2 variant sas_fp16 (R-30): the SAS polynomial with binary16 FMAs in the
    prefill (P~ and alpha), O / LSE against the oracle run with the same flag."""
    B, N, Hq, Hkv, d, causal, bq, am, bc = case
    q, k, v = synth.qkv(5700 + N, B, N, Hq, Hkv, d)
    bits = synth.head_bits_alternating(Hkv)
    p = ta.params(head_dim=d, block_q=bq, block_kv=bc, alpha_mode=am, sas_fp16=1)
    cache = ta.KVCache(B, Hkv, d, max_blocks=N // bc + 2, bits=bits, block_kv=bc)
    qt, kt, vt = (torch.from_numpy(x).cuda() for x in (q, k, v))
    k1, v1t, k1s, v1s = ta.turbo_quantize_kv(p, cache, kt, vt)
    o, lse = ta.turbo_attention_prefill(p, qt, k1, v1t, k1s, v1s, causal=causal)
    torch.cuda.synchronize()
    op = O.params(d=d, block_q=bq, block_kv=bc, alpha_mode=am, sas_fp16=1)
    _check_prefill_heads(op, q, k, v, o.cpu().numpy(), lse.cpu().numpy(),
                         [(b, h) for b in range(B) for h in range(Hq)], causal=causal)


@pytest.mark.parametrize("ij", [(3, 2), (4, 4)])
def test_sas_fp16_variant_prefill_tap(ta, ij):
    """Bit-exact P codes, s_P, m and PV_int under sas_fp16 (P~ from binary16 Horner)."""
    B, N, Hq, Hkv, d = 1, 300, 4, 2, 128
    q, k, v = synth.qkv(5800, B, N, Hq, Hkv, d)
    bits = synth.head_bits_alternating(Hkv)
    b, h = 0, 3
    i, j = ij
    tap = ta.DebugTap(b, h, i, j, d)
    p = ta.params(head_dim=d, debug_tap=tap, sas_fp16=1)
    _prefill(ta, p, q, k, v, bits)
    _, _, rt = O.prefill_head(O.params(d=d, sas_fp16=1), q[b, :, h], k[b, :, h // 2], v[b, :, h // 2], causal=True,
                              tap=(i, j))
    rows = min(64, N - 64 * i)
    np.testing.assert_array_equal(tap.m_new.cpu().numpy()[:rows], rt["m_new"][:rows])
    np.testing.assert_array_equal(tap.p_codes.cpu().numpy()[:rows], rt["p_codes"][:rows])
    np.testing.assert_array_equal(tap.pv_int.cpu().numpy()[:rows], rt["pv_int"][:rows])
    assert tap.s_p.item() == rt["s_p"][0]


@pytest.mark.parametrize("Hq,S", [(8, 1), (8, 3), (16, 2), (16, 1)])
def test_sas_fp16_variant_decode(ta, Hq, S):
    """sas_fp16 in the decode (packed G = 4 and general G = 8 paths, equal splits),
    through appends that flush the buffer."""
    B, N, Hkv, d = 2, 64 * 4 + 50, 2, 128
    q, k, v = synth.qkv(5900, B, N, Hq, Hkv, d)
    bits = synth.head_bits_alternating(Hkv)
    p, op = ta.params(head_dim=d, sas_fp16=1), O.params(d=d, sas_fp16=1)
    apps = [synth.decode_token(6000 + t, B, Hq, Hkv, d)[1:] for t in range(20)]
    cache, ref = _decode_setup(ta, p, op, q, k, v, bits, apps)
    qd, _, _ = synth.decode_token(6100, B, Hq, Hkv, d)
    _check_decode(ta, p, op, cache, ref, qd, Hq // Hkv, S=S)


def test_sas_fp16_variant_decode_tap(ta):
    B, N, Hq, Hkv, d = 2, 64 * 5 + 37, 8, 2, 128
    q, k, v = synth.qkv(6200, B, N, Hq, Hkv, d)
    bits = synth.head_bits_alternating(Hkv)
    b, h, jb = 1, 5, 3
    tap = ta.DebugTap(b, h, 0, jb, d, decode=True)
    p = ta.params(head_dim=d, debug_tap=tap, sas_fp16=1)
    cache = ta.KVCache(B, Hkv, d, max_blocks=8, bits=bits)
    ta.turbo_quantize_kv(p, cache, torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda())
    qd, _, _ = synth.decode_token(6300, B, Hq, Hkv, d)
    ta.turbo_attention_decode(p, cache, torch.from_numpy(qd).cuda(), n_splits=1)
    torch.cuda.synchronize()
    op = O.params(d=d, sas_fp16=1)
    ref = O.build_cache(op, k.astype(np.float32), v.astype(np.float32), bits, 8)
    ks, vs = ref["slots"][b][h // (Hq // Hkv)]
    _, _, rt = O.decode_head(op, qd[b, h].astype(np.float32), ks, vs, 0, ks.n_blocks, True, tap=jb)
    assert rt["hit"]
    assert tap.m_new.item() == rt["m_new"][0]
    np.testing.assert_array_equal(tap.p_codes.cpu().numpy()[0], rt["p_codes"])
    assert tap.s_p.item() == rt["s_p"][0]
    np.testing.assert_array_equal(tap.pv_int.cpu().numpy()[0], rt["pv_int"])
