"""GPU parity at B_c = 128 (turbo_params_t.block_kv = 128; the block-size ablation of
Table 3): the K/V stage-1 block, the stage-2 group, the decode
buffer and the prefill key tile are 128 tokens.  Same bar as tests/test_gpu_parity.py:
codes, scales, records, counters and the tapped exact-set values bit-exact; FP16
outputs within max-abs 2e-3 / rel-L2 1e-3 of the oracle run with block_kv = 128.
"""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2412_08585_b200 import synth
from tests import cache_layout
from tests.test_gpu_parity import _oracle_decode, assert_out_close, balanced_bounds

pytestmark = pytest.mark.gpu

BC = 128


@pytest.fixture(scope="module")
def ta():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2412_08585_b200 import binding

    binding.lib()
    return binding


CASES = [  # (B, N, Hq, Hkv, d, causal, block_q, alpha_mode)
    (1, 128, 1, 1, 64, True, 64, 0),      # one block
    (2, 300, 8, 2, 128, True, 64, 0),     # GQA, ragged tail (44 tokens to the buffer)
    (1, 333, 4, 4, 128, False, 64, 1),    # non-causal, ragged, alpha mode 1
    (1, 520, 2, 1, 64, True, 128, 0),     # B_r = 128, d = 64
    (2, 700, 3, 3, 128, True, 64, 0),     # MHA: adjacent query-tile pairs
    (1, 1100, 6, 2, 128, True, 64, 1),    # odd G = 3, several tiles
]


def _check_cache(ta, cache, ref, B, Hkv, d, bits):
    recs = cache.records().cpu().numpy()
    mb = cache.max_blocks
    spar = cache.s_parent[: B * Hkv * 2 * mb].view(B, Hkv, 2, mb).cpu().numpy()
    buf = cache.buf.view(B, Hkv, 2, BC * d).cpu().numpy()
    a_univ = cache.a_univ.view(B, Hkv, 2).cpu().numpy()
    cnt = cache.counters.view(B, 2).cpu().numpy()
    for b in range(B):
        for h in range(Hkv):
            for kind, sl in enumerate(ref["slots"][b][h]):
                assert cnt[b, 0] == sl.n_blocks and cnt[b, 1] == sl.n_buf
                assert a_univ[b, h, kind] == sl.a_univ
                for j in range(sl.n_blocks):
                    codes, s_int, z_int = cache_layout.unpack_record(recs[b, h, kind, j], d, int(bits[h][kind]),
                                                                     kind, bc=BC)
                    np.testing.assert_array_equal(codes, sl.codes[j])
                    np.testing.assert_array_equal(s_int, sl.s_int[j])
                    np.testing.assert_array_equal(z_int, sl.z_int[j])
                    assert spar[b, h, kind, j] == sl.s_parent[j]
                bb = buf[b, h, kind].reshape(BC, d) if kind == 0 else buf[b, h, kind].reshape(d, BC).T
                np.testing.assert_array_equal(bb[: sl.n_buf], sl.buf[: sl.n_buf])


@pytest.mark.parametrize("case", CASES)
def test_bc128_quantize_kv_bit_exact(ta, case):
    B, N, Hq, Hkv, d, causal, bq, am = case
    q, k, v = synth.qkv(1500 + N, B, N, Hq, Hkv, d)
    bits = synth.head_bits_alternating(Hkv)
    p = ta.params(head_dim=d, block_q=bq, block_kv=BC, alpha_mode=am)
    mb = N // BC + 2
    cache = ta.KVCache(B, Hkv, d, max_blocks=mb, bits=bits, block_kv=BC)
    k1, v1t, k1s, v1s = ta.turbo_quantize_kv(p, cache, torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda())
    torch.cuda.synchronize()
    ref = O.build_cache(O.params(d=d, block_q=bq, block_kv=BC, alpha_mode=am), k.astype(np.float32),
                        v.astype(np.float32), bits, mb)
    np.testing.assert_array_equal(k1.cpu().numpy(), ref["k1"])
    np.testing.assert_array_equal(k1s.cpu().numpy(), ref["k1s"])
    np.testing.assert_array_equal(v1s.cpu().numpy(), ref["v1s"])
    tc = -(-N // BC)
    v1t = v1t.float().cpu().numpy()
    assert v1t.shape == (B, Hkv, tc, d, BC) and (v1t == np.rint(v1t)).all()
    v1 = v1t.astype(np.int8).transpose(0, 1, 2, 4, 3).reshape(B, Hkv, tc * BC, d)
    np.testing.assert_array_equal(v1[:, :, :N], ref["v1"])
    assert not v1[:, :, N:].any()
    _check_cache(ta, cache, ref, B, Hkv, d, bits)


@pytest.mark.parametrize("case", CASES)
def test_bc128_prefill_parity(ta, case):
    B, N, Hq, Hkv, d, causal, bq, am = case
    q, k, v = synth.qkv(1700 + N, B, N, Hq, Hkv, d)
    bits = synth.head_bits_alternating(Hkv)
    p = ta.params(head_dim=d, block_q=bq, block_kv=BC, alpha_mode=am)
    cache = ta.KVCache(B, Hkv, d, max_blocks=N // BC + 2, bits=bits, block_kv=BC)
    qt, kt, vt = (torch.from_numpy(x).cuda() for x in (q, k, v))
    k1, v1t, k1s, v1s = ta.turbo_quantize_kv(p, cache, kt, vt)
    o, lse = ta.turbo_attention_prefill(p, qt, k1, v1t, k1s, v1s, causal=causal)
    torch.cuda.synchronize()
    o, lse = o.cpu().numpy(), lse.cpu().numpy()
    op = O.params(d=d, block_q=bq, block_kv=BC, alpha_mode=am)
    G = Hq // Hkv
    for b in range(B):
        for h in range(Hq):
            oref, lref = O.prefill_head(op, q[b, :, h], k[b, :, h // G], v[b, :, h // G], causal=causal)
            assert_out_close(o[b, :, h], oref, f"b{b} h{h}")
            np.testing.assert_allclose(lse[b, h], lref, atol=1e-4, rtol=1e-5)


@pytest.mark.parametrize("case", [CASES[1], CASES[2], CASES[5]])
def test_bc128_prefill_exact_set_tap(ta, case):
    """Bit-exact q1, s_Q, S_int, m_new, P codes, s_P and PV_int of chosen 64 x 128 tiles."""
    B, N, Hq, Hkv, d, causal, bq, am = case
    q, k, v = synth.qkv(1900 + N, B, N, Hq, Hkv, d)
    bits = synth.head_bits_alternating(Hkv)
    qt, kt, vt = (torch.from_numpy(x).cuda() for x in (q, k, v))
    G = Hq // Hkv
    op = O.params(d=d, block_q=bq, block_kv=BC, alpha_mode=am)
    Ti, Tj = -(-N // 64), -(-N // BC)
    for (b, h, i, j) in sorted({(B - 1, Hq - 1, Ti - 1, Tj - 1), (0, 0, 2, 1), (0, Hq // 2, Ti - 1, 0)}):
        tap = ta.DebugTap(b, h, i, j, d, block_kv=BC)
        p = ta.params(head_dim=d, block_q=bq, block_kv=BC, alpha_mode=am, debug_tap=tap)
        cache = ta.KVCache(B, Hkv, d, max_blocks=N // BC + 2, bits=bits, block_kv=BC)
        k1, v1t, k1s, v1s = ta.turbo_quantize_kv(p, cache, kt, vt)
        ta.turbo_attention_prefill(p, qt, k1, v1t, k1s, v1s, causal=causal)
        torch.cuda.synchronize()
        _, _, rt = O.prefill_head(op, q[b, :, h], k[b, :, h // G], v[b, :, h // G], causal=causal, tap=(i, j))
        assert rt["hit"]
        rows = min(64, N - 64 * i)
        np.testing.assert_array_equal(tap.q1.cpu().numpy()[:rows], rt["q1"][:rows])
        assert tap.s_q.item() == rt["s_q"][0]
        np.testing.assert_array_equal(tap.s_int.cpu().numpy()[:rows], rt["s_int"][:rows])
        np.testing.assert_array_equal(tap.m_new.cpu().numpy()[:rows], rt["m_new"][:rows])
        np.testing.assert_array_equal(tap.p_codes.cpu().numpy()[:rows], rt["p_codes"][:rows])
        assert tap.s_p.item() == rt["s_p"][0]
        np.testing.assert_array_equal(tap.pv_int.cpu().numpy()[:rows], rt["pv_int"][:rows])


DEC_CASES = [  # (B, N_prefill, n_append, Hq, Hkv, d, n_splits, alpha_mode)
    (1, 128, 128, 1, 1, 64, 1, 0),        # one block + 128 appends (one flush)
    (2, 700, 70, 8, 2, 128, 1, 0),        # G = 4 packed path, buffer crosses a flush
    (2, 700, 5, 8, 2, 128, 3, 1),         # equal splits + combine
    (3, 128 * 9 + 5, 3, 8, 2, 128, 0, 1),  # balanced schedule
    (2, 128 * 5 + 17, 3, 16, 2, 128, 2, 0),  # G = 8 general path
    (1, 128 * 6 + 5, 0, 8, 1, 64, 0, 0),  # G = 8, d = 64, balanced
    (1, 128 * 5 + 9, 5, 6, 2, 128, 2, 0),  # G = 3
]


@pytest.mark.parametrize("case", DEC_CASES)
def test_bc128_append_and_decode_parity(ta, case):
    B, N, n_app, Hq, Hkv, d, S, am = case
    G = Hq // Hkv
    q, k, v = synth.qkv(2300 + N, B, N, Hq, Hkv, d)
    bits = synth.head_bits_alternating(Hkv)
    maxb = (N + n_app) // BC + 1
    p = ta.params(head_dim=d, block_kv=BC, alpha_mode=am)
    cache = ta.KVCache(B, Hkv, d, max_blocks=maxb, bits=bits, block_kv=BC)
    ta.turbo_quantize_kv(p, cache, torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda())
    op = O.params(d=d, block_kv=BC, alpha_mode=am)
    ref = O.build_cache(op, k.astype(np.float32), v.astype(np.float32), bits, maxb)
    for t in range(n_app):
        _, kt, vt = synth.decode_token(6000 + t, B, Hq, Hkv, d)
        ta.turbo_quantize_kv(p, cache, torch.from_numpy(kt).cuda(), torch.from_numpy(vt).cuda(), mode=1)
        for b in range(B):
            for h in range(Hkv):
                ref["slots"][b][h][0].append(kt[b, h].astype(np.float32))
                ref["slots"][b][h][1].append(vt[b, h].astype(np.float32))
    qd, _, _ = synth.decode_token(9100, B, Hq, Hkv, d)
    o, _, lse = ta.turbo_attention_decode(p, cache, torch.from_numpy(qd).cuda(), n_splits=S)
    torch.cuda.synchronize()
    o, lse = o.cpu().numpy(), lse.cpu().numpy()
    _check_cache(ta, cache, ref, B, Hkv, d, bits)
    nb = ref["slots"][0][0][0].n_blocks
    if S > 0:
        per = -(-nb // S)
        bounds = [(min(s * per, nb), min(s * per + per, nb)) for s in range(S)]
    else:
        bal = balanced_bounds(ta, ref["slots"], Hq, Hkv, d)
    for b in range(B):
        ro, rl = _oracle_decode(op, qd[b].astype(np.float32), ref["slots"][b], G, bounds if S > 0 else bal[b])
        assert_out_close(o[b], ro, f"decode b{b}")
        np.testing.assert_allclose(lse[b], rl, atol=1e-4, rtol=1e-5)


@pytest.mark.parametrize("j_block", [0, 2, -1])
@pytest.mark.parametrize("Hq", [8, 16])  # G = 4 (packed IMMA path) and G = 8 (general path)
def test_bc128_decode_exact_set_tap(ta, j_block, Hq):
    B, N, Hkv, d = 2, 128 * 3 + 37, 2, 128
    q, k, v = synth.qkv(79, B, N, Hq, Hkv, d)
    bits = synth.head_bits_alternating(Hkv)
    b, h = 1, 5
    tap = ta.DebugTap(b, h, 0, j_block, d, decode=True, block_kv=BC)
    p = ta.params(head_dim=d, block_kv=BC, debug_tap=tap)
    cache = ta.KVCache(B, Hkv, d, max_blocks=5, bits=bits, block_kv=BC)
    ta.turbo_quantize_kv(p, cache, torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda())
    qd, _, _ = synth.decode_token(33, B, Hq, Hkv, d)
    ta.turbo_attention_decode(p, cache, torch.from_numpy(qd).cuda(), n_splits=1)
    torch.cuda.synchronize()
    op = O.params(d=d, block_kv=BC)
    ref = O.build_cache(op, k.astype(np.float32), v.astype(np.float32), bits, 5)
    ks, vs = ref["slots"][b][h // (Hq // Hkv)]
    _, _, rt = O.decode_head(op, qd[b, h].astype(np.float32), ks, vs, 0, ks.n_blocks, True, tap=j_block)
    assert rt["hit"]
    np.testing.assert_array_equal(tap.q1.cpu().numpy()[0], rt["q1"])
    assert tap.s_q.item() == rt["s_q"][0]
    np.testing.assert_array_equal(tap.s_int.cpu().numpy()[0], rt["s_int"])
    assert tap.m_new.item() == rt["m_new"][0]
    np.testing.assert_array_equal(tap.p_codes.cpu().numpy()[0], rt["p_codes"])
    assert tap.s_p.item() == rt["s_p"][0]
    np.testing.assert_array_equal(tap.pv_int.cpu().numpy()[0], rt["pv_int"])


def test_bc128_chunked_prefill(ta):
    """NEXT-3 at B_c = 128: a prefix prefill, the cache's stage-1 reconstruction
    (turbo_dequantize_cache) and a chunk at a 128-token boundary (R-28)."""
    B, P, Nc, Hq, Hkv, d = 1, 256, 300, 8, 2, 128
    Nk = P + Nc
    q, k, v = synth.qkv(4242, B, Nk, Hq, Hkv, d)
    bits = synth.head_bits_alternating(Hkv)
    p = ta.params(head_dim=d, block_kv=BC)
    maxb = Nk // BC + 2
    cache = ta.KVCache(B, Hkv, d, max_blocks=maxb, bits=bits, block_kv=BC)
    dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()  # noqa: E731
    ta.turbo_quantize_kv(p, cache, dev(k[:, :P]), dev(v[:, :P]))
    ops = ta.turbo_dequantize_cache(p, cache, Nk)
    ta.turbo_quantize_kv(p, cache, dev(k[:, P:]), dev(v[:, P:]), mode=2, out=ops)
    o, lse = ta.turbo_attention_prefill_chunk(p, dev(q[:, P:]), *ops)
    torch.cuda.synchronize()
    o, lse = o.cpu().numpy(), lse.cpu().numpy()
    op = O.params(d=d, block_kv=BC)
    G = Hq // Hkv
    for h in range(Hkv):
        ops_ref = []
        for kind, x in ((0, k), (1, v)):
            sl = O.Slot(op, int(bits[h][kind]), maxb)
            sl.prefill(x[0, :P, h].astype(np.float32))
            xp, sp = sl.stage1_prefix(P // BC)
            xc, sc = sl.prefill_append(x[0, P:, h].astype(np.float32))
            ops_ref.append((np.concatenate([xp, xc]), np.concatenate([sp, sc])))
        (k1r, skr), (v1r, svr) = ops_ref
        for hq in range(h * G, (h + 1) * G):
            oref, lref = O.prefill_chunk_head(op, q[0, P:, hq], k1r, skr, v1r, svr, causal=True)
            assert_out_close(o[0, :, hq], oref, f"h{hq}")
            np.testing.assert_allclose(lse[0, hq], lref, atol=1e-4, rtol=1e-5)


def test_bc128_with_fp16_scales_and_fp16_sas(ta):
    """B_c = 128 together with both NEXT-2 arithmetic variants (scale_fp16: R-29, sas_fp16: R-30):
    records / parent scales bit-exact, prefill and decode against the oracle run with the same flags."""
    B, N, Hq, Hkv, d = 2, 128 * 3 + 40, 8, 2, 128
    q, k, v = synth.qkv(7777, B, N, Hq, Hkv, d)
    bits = synth.head_bits_alternating(Hkv)
    p = ta.params(head_dim=d, block_kv=BC, scale_fp16=1, sas_fp16=1)
    op = O.params(d=d, block_kv=BC, scale_fp16=1, sas_fp16=1)
    mb = N // BC + 2
    cache = ta.KVCache(B, Hkv, d, max_blocks=mb, bits=bits, block_kv=BC)
    qt, kt, vt = (torch.from_numpy(x).cuda() for x in (q, k, v))
    k1, v1t, k1s, v1s = ta.turbo_quantize_kv(p, cache, kt, vt)
    o, lse = ta.turbo_attention_prefill(p, qt, k1, v1t, k1s, v1s)
    qd, _, _ = synth.decode_token(7778, B, Hq, Hkv, d)
    od, _, ld = ta.turbo_attention_decode(p, cache, torch.from_numpy(qd).cuda(), n_splits=2)
    torch.cuda.synchronize()
    ref = O.build_cache(op, k.astype(np.float32), v.astype(np.float32), bits, mb)
    _check_cache(ta, cache, ref, B, Hkv, d, bits)
    o, lse, od, ld = (x.cpu().numpy() for x in (o, lse, od, ld))
    G = Hq // Hkv
    for b in range(B):
        for h in range(Hq):
            oref, lref = O.prefill_head(op, q[b, :, h], k[b, :, h // G], v[b, :, h // G])
            assert_out_close(o[b, :, h], oref, f"b{b} h{h}")
            np.testing.assert_allclose(lse[b, h], lref, atol=1e-4, rtol=1e-5)
        nb = ref["slots"][b][0][0].n_blocks
        per = -(-nb // 2)
        ro, rl = _oracle_decode(op, qd[b].astype(np.float32), ref["slots"][b], G,
                                [(0, min(per, nb)), (min(per, nb), nb)])
        assert_out_close(od[b], ro, f"decode b{b}")
        np.testing.assert_allclose(ld[b], rl, atol=1e-4, rtol=1e-5)
