"""GPU parity: the CUDA path through the C-ABI vs the CPU oracle (-m gpu).

Bar (BASELINE.json north_star): bit-exact codes, scales and INT32 S; the other
exact-set values (m, P codes, s_P, PV_int) bit-exact too; FP16
outputs within max-abs 2e-3 and rel-L2 1e-3 of the oracle's FP32 output.
"""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2412_08585_b200 import synth
from tests import cache_layout

pytestmark = pytest.mark.gpu

MAX_ABS, REL_L2 = 2e-3, 1e-3


@pytest.fixture(scope="module")
def ta():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2412_08585_b200 import binding

    binding.lib()
    return binding


def rel_l2(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def assert_out_close(gpu_fp16, ref_f32, what=""):
    g = gpu_fp16.astype(np.float32)
    err = np.abs(g - ref_f32).max()
    rl = rel_l2(g, ref_f32)
    assert err <= MAX_ABS and rl <= REL_L2, f"{what}: max-abs {err:.3e} rel-L2 {rl:.3e}"


CASES = [  # (B, N, Hq, Hkv, d, causal, block_q, alpha_mode)
    (1, 128, 1, 1, 64, True, 64, 0),      # config 1 (BASELINE.json configs[0])
    (2, 200, 8, 2, 128, True, 64, 0),     # GQA, ragged tail, several tiles
    (1, 333, 4, 4, 128, False, 64, 1),    # non-causal, ragged, alpha mode 1
    (1, 256, 2, 1, 64, True, 128, 0),     # B_r = 128
    (2, 700, 3, 3, 128, True, 64, 0),     # MHA (G = 1): adjacent query-tile pairs, ragged last pair
    (1, 520, 6, 2, 128, True, 64, 1),     # odd G = 3: tile pairs of one head
]


def _oracle_params(d, block_q, alpha_mode):
    return O.params(d=d, block_q=block_q, block_kv=64, alpha_mode=alpha_mode)


@pytest.mark.parametrize("case", CASES)
def test_quantize_kv_prefill_bit_exact(ta, case):
    B, N, Hq, Hkv, d, causal, bq, am = case
    q, k, v = synth.qkv(500 + N, B, N, Hq, Hkv, d)
    bits = synth.head_bits_alternating(Hkv)
    p = ta.params(head_dim=d, block_q=bq, alpha_mode=am)
    mb = N // 64 + 2
    cache = ta.KVCache(B, Hkv, d, max_blocks=mb, bits=bits)
    k1, v1t, k1s, v1s = ta.turbo_quantize_kv(p, cache, torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda())
    torch.cuda.synchronize()
    ref = O.build_cache(_oracle_params(d, bq, am), k.astype(np.float32), v.astype(np.float32), bits, mb)
    np.testing.assert_array_equal(k1.cpu().numpy(), ref["k1"])
    np.testing.assert_array_equal(k1s.cpu().numpy(), ref["k1s"])
    np.testing.assert_array_equal(v1s.cpu().numpy(), ref["v1s"])
    tc = -(-N // 64)
    v1t = v1t.float().cpu().numpy()
    assert (v1t == np.rint(v1t)).all()  # integer codes carried exactly in FP16
    v1 = v1t.astype(np.int8).transpose(0, 1, 2, 4, 3).reshape(B, Hkv, tc * 64, d)
    np.testing.assert_array_equal(v1[:, :, :N], ref["v1"])
    assert not v1[:, :, N:].any()
    recs = cache.records().cpu().numpy()
    spar = cache.s_parent[: B * Hkv * 2 * mb].view(B, Hkv, 2, mb).cpu().numpy()
    buf = cache.buf.view(B, Hkv, 2, 64 * d).cpu().numpy()
    a_univ = cache.a_univ.view(B, Hkv, 2).cpu().numpy()
    cnt = cache.counters.view(B, 2).cpu().numpy()
    for b in range(B):
        for h in range(Hkv):
            for kind, sl in enumerate(ref["slots"][b][h]):
                assert cnt[b, 0] == sl.n_blocks and cnt[b, 1] == sl.n_buf
                assert a_univ[b, h, kind] == sl.a_univ
                for j in range(sl.n_blocks):
                    codes, s_int, z_int = cache_layout.unpack_record(recs[b, h, kind, j], d, int(bits[h][kind]), kind)
                    np.testing.assert_array_equal(codes, sl.codes[j])
                    np.testing.assert_array_equal(s_int, sl.s_int[j])
                    np.testing.assert_array_equal(z_int, sl.z_int[j])
                    assert spar[b, h, kind, j] == sl.s_parent[j]
                bb = buf[b, h, kind].reshape(64, d) if kind == 0 else buf[b, h, kind].reshape(d, 64).T
                np.testing.assert_array_equal(bb[: sl.n_buf], sl.buf[: sl.n_buf])


@pytest.mark.parametrize("case", CASES)
def test_prefill_parity(ta, case):
    B, N, Hq, Hkv, d, causal, bq, am = case
    q, k, v = synth.qkv(700 + N, B, N, Hq, Hkv, d)
    bits = synth.head_bits_alternating(Hkv)
    p = ta.params(head_dim=d, block_q=bq, alpha_mode=am)
    cache = ta.KVCache(B, Hkv, d, max_blocks=N // 64 + 2, bits=bits)
    qt, kt, vt = (torch.from_numpy(x).cuda() for x in (q, k, v))
    k1, v1t, k1s, v1s = ta.turbo_quantize_kv(p, cache, kt, vt)
    o, lse = ta.turbo_attention_prefill(p, qt, k1, v1t, k1s, v1s, causal=causal)
    torch.cuda.synchronize()
    o, lse = o.cpu().numpy(), lse.cpu().numpy()
    op = _oracle_params(d, bq, am)
    G = Hq // Hkv
    for b in range(B):
        for h in range(Hq):
            oref, lref = O.prefill_head(op, q[b, :, h], k[b, :, h // G], v[b, :, h // G], causal=causal)
            assert_out_close(o[b, :, h], oref, f"b{b} h{h}")
            np.testing.assert_allclose(lse[b, h], lref, atol=1e-4, rtol=1e-5)


@pytest.mark.parametrize("case", CASES[:3])
def test_prefill_exact_set_tap(ta, case):
    """Bit-exact q1, s_Q, S_int, m_new, P codes, s_P and PV_int of chosen tiles."""
    B, N, Hq, Hkv, d, causal, bq, am = case
    q, k, v = synth.qkv(900 + N, B, N, Hq, Hkv, d)
    bits = synth.head_bits_alternating(Hkv)
    qt, kt, vt = (torch.from_numpy(x).cuda() for x in (q, k, v))
    G = Hq // Hkv
    op = _oracle_params(d, bq, am)
    T = -(-N // 64)
    for (b, h, i, j) in sorted({(B - 1, Hq - 1, T - 1, T - 1), (0, 0, 1, 0), (0, Hq // 2, T - 1, 0)}):
        tap = ta.DebugTap(b, h, i, j, d)
        p = ta.params(head_dim=d, block_q=bq, alpha_mode=am, debug_tap=tap)
        cache = ta.KVCache(B, Hkv, d, max_blocks=N // 64 + 2, bits=bits)
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
    (1, 128, 64, 1, 1, 64, 1, 0),       # config 1 + 64 appends (one flush)
    (2, 700, 70, 8, 2, 128, 1, 0),      # GQA, mixed 2/4 bit, buffer + flush
    (2, 700, 5, 8, 2, 128, 3, 1),       # in-GPU split-KV + combine
    (1, 64 * 9, 0, 4, 1, 128, 4, 0),    # G = 4, empty buffer
    # balanced schedule (n_splits = 0): chunks of >= 8 units cut across (b, kv head) ranges
    (2, 700, 70, 8, 2, 128, 0, 0),      # pieces incl. a buffer-only piece
    (3, 64 * 20 + 5, 3, 8, 2, 128, 0, 1),
    (1, 128, 64, 1, 1, 64, 0, 0),       # d = 64, one piece
    (1, 64 * 9, 0, 4, 1, 128, 0, 0),    # G = 4, empty buffer
    # G = 8: the general (unpacked) IMMA path, separate hi / lo B fragments
    (2, 64 * 6 + 17, 3, 16, 2, 128, 2, 0),
    (1, 64 * 9 + 5, 0, 8, 1, 128, 0, 1),
    (1, 300, 2, 8, 1, 64, 1, 0),
    # odd / small groups on the packed path (rows >= G absent): G = 3 split, G = 2 balanced at d = 64
    (1, 64 * 5 + 9, 5, 6, 2, 128, 2, 0),
    (2, 64 * 20 + 5, 3, 4, 2, 64, 0, 0),
    # G = 6 (general path) through n_splits=None, which selects the balanced schedule over the
    # fixed reference worker count (device-independent) for G > 4
    (1, 64 * 7 + 3, 2, 6, 1, 128, None, 0),
    # balanced schedule over an explicit worker count (n_splits = -W), a G <= 4 default (None)
    (3, 64 * 20 + 5, 3, 8, 2, 128, -7, 1),
    (2, 64 * 40 + 9, 4, 8, 2, 128, None, 0),
]


def _oracle_decode(op, q, slots, G, splits_bounds):
    """Per q head: oracle decode over explicit split ranges + combine.
    splits_bounds: [(a, e)] (buffer with the last) or, per kv head,
    {kvh: [(a, e, with_buffer)]}."""
    Hq = q.shape[0]
    outs, lses = np.zeros((Hq, op.d), np.float32), np.zeros(Hq, np.float32)
    for h in range(Hq):
        ks, vs = slots[h // G]
        if isinstance(splits_bounds, dict):
            pieces = splits_bounds[h // G]
        else:
            pieces = [(a, e, s == len(splits_bounds) - 1) for s, (a, e) in enumerate(splits_bounds)]
        parts, ls = [], []
        for a, e, wb in pieces:
            o, l = O.decode_head(op, q[h], ks, vs, a, e, wb)
            parts.append(o)
            ls.append(l)
        if len(parts) == 1:
            outs[h], lses[h] = parts[0], ls[0]
        else:
            outs[h], lses[h] = O.combine(np.stack(parts), np.array(ls))
    return outs, lses


def balanced_bounds(ta, slots_by_b, Hq, Hkv, d, workers=None):
    """{b: {kvh: [(a, e, with_buffer)]}} of the balanced schedule, from the
    documented partition (include/turbo_attention.h) and the oracle's counters."""
    units = [sl[0][0].n_blocks + (1 if sl[0][0].n_buf > 0 else 0) for sl in slots_by_b]
    rng = ta.balanced_ranges(units, Hkv, workers or ta.turbo_decode_workers(Hq, Hkv, d))
    out = {}
    for b, sl in enumerate(slots_by_b):
        nb = sl[0][0].n_blocks
        out[b] = {h: [(u0, min(u1, nb), u1 > nb) for u0, u1 in rng[(b, h)]] for h in range(Hkv)}
    return out


@pytest.mark.parametrize("case", DEC_CASES)
def test_append_and_decode_parity(ta, case):
    B, N, n_app, Hq, Hkv, d, S, am = case
    G = Hq // Hkv
    q, k, v = synth.qkv(1300 + N, B, N, Hq, Hkv, d)
    bits = synth.head_bits_alternating(Hkv)
    maxb = (N + n_app) // 64 + 1
    p = ta.params(head_dim=d, alpha_mode=am)
    cache = ta.KVCache(B, Hkv, d, max_blocks=maxb, bits=bits)
    ta.turbo_quantize_kv(p, cache, torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda())
    op = O.params(d=d, alpha_mode=am)
    ref = O.build_cache(op, k.astype(np.float32), v.astype(np.float32), bits, maxb)
    for t in range(n_app):
        _, kt, vt = synth.decode_token(5000 + t, B, Hq, Hkv, d)
        ta.turbo_quantize_kv(p, cache, torch.from_numpy(kt).cuda(), torch.from_numpy(vt).cuda(), mode=1)
        for b in range(B):
            for h in range(Hkv):
                ref["slots"][b][h][0].append(kt[b, h].astype(np.float32))
                ref["slots"][b][h][1].append(vt[b, h].astype(np.float32))
    qd, _, _ = synth.decode_token(9000, B, Hq, Hkv, d)
    o, _, lse = ta.turbo_attention_decode(p, cache, torch.from_numpy(qd).cuda(), n_splits=S)
    torch.cuda.synchronize()
    o, lse = o.cpu().numpy(), lse.cpu().numpy()
    nb = ref["slots"][0][0][0].n_blocks
    if S is None:  # the binding's default, recomputed from its documented rule
        S = ta.reference_workers(Hq, Hkv, d)
        S = -S if G > 4 else ta.auto_splits(B, Hkv, nb, S)
    if S > 0:
        per = -(-nb // S)
        bounds = [(min(s * per, nb), min(s * per + per, nb)) for s in range(S)]
    else:
        bal = balanced_bounds(ta, ref["slots"], Hq, Hkv, d, -S if S < 0 else None)
        assert B * Hkv == 1 or sum(len(v) for x in bal.values() for v in x.values()) > B * Hkv  # really split
    # cache state after the appends is bit-exact
    recs = cache.records().cpu().numpy()
    cnt = cache.counters.view(B, 2).cpu().numpy()
    for b in range(B):
        for h in range(Hkv):
            for kind, sl in enumerate(ref["slots"][b][h]):
                assert tuple(cnt[b]) == (sl.n_blocks, sl.n_buf)
                for j in range(sl.n_blocks):
                    codes, s_int, z_int = cache_layout.unpack_record(recs[b, h, kind, j], d, int(bits[h][kind]), kind)
                    np.testing.assert_array_equal(codes, sl.codes[j])
                    np.testing.assert_array_equal(s_int, sl.s_int[j])
                    np.testing.assert_array_equal(z_int, sl.z_int[j])
        ro, rl = _oracle_decode(op, qd[b].astype(np.float32), ref["slots"][b], G, bounds if S > 0 else bal[b])
        assert_out_close(o[b], ro, f"decode b{b}")
        np.testing.assert_allclose(lse[b], rl, atol=1e-4, rtol=1e-5)


@pytest.mark.parametrize("j_block", [0, 3, -1])
@pytest.mark.parametrize("n_splits", [1, 0])
@pytest.mark.parametrize("Hq", [8, 16])  # G = 4 (packed IMMA path) and G = 8 (general path)
def test_decode_exact_set_tap(ta, j_block, n_splits, Hq):
    B, N, Hkv, d = 2, 64 * 5 + 37, 2, 128
    q, k, v = synth.qkv(77, B, N, Hq, Hkv, d)
    bits = synth.head_bits_alternating(Hkv)
    b, h = 1, 5
    tap = ta.DebugTap(b, h, 0, j_block, d, decode=True)
    p = ta.params(head_dim=d, debug_tap=tap)
    cache = ta.KVCache(B, Hkv, d, max_blocks=8, bits=bits)
    ta.turbo_quantize_kv(p, cache, torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda())
    qd, _, _ = synth.decode_token(31, B, Hq, Hkv, d)
    ta.turbo_attention_decode(p, cache, torch.from_numpy(qd).cuda(), n_splits=n_splits)
    torch.cuda.synchronize()
    op = O.params(d=d)
    ref = O.build_cache(op, k.astype(np.float32), v.astype(np.float32), bits, 8)
    kvh = h // (Hq // Hkv)
    ks, vs = ref["slots"][b][kvh]
    a_, e_, wb = 0, ks.n_blocks, True
    if n_splits == 0:  # the tapped block's piece of the balanced partition (its m, l start there)
        unit = ks.n_blocks if j_block < 0 else j_block
        pieces = balanced_bounds(ta, ref["slots"], Hq, Hkv, d)[b][kvh]
        a_, e_, wb = next(x for x in pieces if x[0] <= unit < (x[1] + (1 if x[2] else 0)))
    _, _, rt = O.decode_head(op, qd[b, h].astype(np.float32), ks, vs, a_, e_, wb, tap=j_block)
    assert rt["hit"]
    np.testing.assert_array_equal(tap.q1.cpu().numpy()[0], rt["q1"])
    assert tap.s_q.item() == rt["s_q"][0]
    np.testing.assert_array_equal(tap.s_int.cpu().numpy()[0], rt["s_int"])
    assert tap.m_new.item() == rt["m_new"][0]
    np.testing.assert_array_equal(tap.p_codes.cpu().numpy()[0], rt["p_codes"])
    assert tap.s_p.item() == rt["s_p"][0]
    np.testing.assert_array_equal(tap.pv_int.cpu().numpy()[0], rt["pv_int"])


# part counts covering 1-8 warps per row, the 8-parts-in-flight loop and its remainder (S = 300, 101)
@pytest.mark.parametrize("S,rows,d", [(5, 37, 128), (40, 9, 64), (1, 3, 128), (300, 7, 128), (101, 5, 64)])
def test_combine_lse_parity(ta, S, rows, d):
    rng = np.random.default_rng(S)
    o_parts = rng.standard_normal((S, rows, d)).astype(np.float32)
    lse_parts = (rng.standard_normal((S, rows)) * 3).astype(np.float32)
    lse_parts[min(2, S - 1), :2] = -np.inf
    lse_parts[:, rows - 2] = -np.inf  # a row with no part at all: O = 0, L = -inf
    o16, _, lse = ta.turbo_combine_lse(torch.from_numpy(o_parts).cuda(), torch.from_numpy(lse_parts).cuda())
    torch.cuda.synchronize()
    for r in range(rows):
        ro, rl = O.combine(o_parts[:, r], lse_parts[:, r])
        np.testing.assert_allclose(o16[r].float().cpu().numpy(), ro, atol=2e-3, rtol=1e-3)
        if np.isfinite(rl):
            assert abs(lse[r].item() - rl) < 1e-5
        else:
            assert lse[r].item() == -np.inf


def test_combine_lse_rejects_other_head_dims(ta):
    o_parts = torch.zeros(2, 3, 96, device="cuda")
    with pytest.raises(ta.TurboError):
        ta.turbo_combine_lse(o_parts, torch.zeros(2, 3, device="cuda"))


def test_validation_errors(ta):
    p = ta.params(head_dim=96)
    cache_ok = ta.KVCache(1, 1, 64, 4, [[4, 4]])
    with pytest.raises(ta.TurboError) as e:
        ta.turbo_attention_prefill(p, torch.zeros(1, 64, 1, 96, dtype=torch.float16, device="cuda"),
                                   torch.zeros(1, 1, 64, 96, dtype=torch.int8, device="cuda"),
                                   torch.zeros(1, 1, 1, 96, 64, dtype=torch.int8, device="cuda"),
                                   torch.zeros(1, 1, 1, device="cuda"), torch.zeros(1, 1, 1, device="cuda"))
    assert e.value.code == ta.TURBO_ERR_UNSUPPORTED
    p = ta.params(head_dim=64)
    with pytest.raises(ta.TurboError) as e:  # decode on an empty cache
        ta.turbo_attention_decode(p, cache_ok, torch.zeros(1, 1, 64, dtype=torch.float16, device="cuda"))
    assert e.value.code == ta.TURBO_ERR_INVALID_ARG
    with pytest.raises(ta.TurboError) as e:  # capacity
        kk = torch.zeros(1, 64 * 5, 1, 64, dtype=torch.float16, device="cuda")
        ta.turbo_quantize_kv(p, cache_ok, kk, kk)
    assert e.value.code == ta.TURBO_ERR_CAPACITY


def test_seq_sharded_decode_emulated_ranks(ta):
    """configs[4]-style long-context decode on one GPU with W emulated ranks:
    each shard's cache decodes with o_part (FP32, normalised) + L, the
    partials merge with turbo_combine_lse in rank order."""
    from paper_2412_08585_b200 import parallel

    B, N, Hq, Hkv, d, W = 2, 64 * 11 + 9, 8, 2, 128, 3
    G = Hq // Hkv
    q, k, v = synth.qkv(4242, B, N, Hq, Hkv, d)
    qd, _, _ = synth.decode_token(4243, B, Hq, Hkv, d)
    bits = synth.head_bits_alternating(Hkv)
    p = ta.params(head_dim=d, alpha_mode=1)
    op = O.params(d=d, alpha_mode=1)
    parts, lses, ref_parts, ref_lses = [], [], [], []
    for r in range(W):
        t0, t1 = parallel.seq_shard_tokens(N, W, r)
        cache = ta.KVCache(B, Hkv, d, max_blocks=8, bits=bits)
        ta.turbo_quantize_kv(p, cache, torch.from_numpy(np.ascontiguousarray(k[:, t0:t1])).cuda(),
                             torch.from_numpy(np.ascontiguousarray(v[:, t0:t1])).cuda())
        _, op32, l_ = ta.turbo_attention_decode(p, cache, torch.from_numpy(qd).cuda(), with_buffer=(r == W - 1),
                                                n_splits=2, want_fp16=False, want_f32=True)
        parts.append(op32.reshape(B * Hq, d))
        lses.append(l_.reshape(B * Hq))
        ref = O.build_cache(op, k[:, t0:t1].astype(np.float32), v[:, t0:t1].astype(np.float32), bits, 8)
        rp, rl = np.zeros((B, Hq, d), np.float32), np.zeros((B, Hq), np.float32)
        for b in range(B):
            nb = ref["slots"][b][0][0].n_blocks
            per = -(-nb // 2)
            bounds = [(min(s * per, nb), min(s * per + per, nb)) for s in range(2)]
            for h in range(Hq):
                ks, vs = ref["slots"][b][h // G]
                pp = [O.decode_head(op, qd[b, h].astype(np.float32), ks, vs, a_, e_, (s == 1) and (r == W - 1))
                      for s, (a_, e_) in enumerate(bounds)]
                rp[b, h], rl[b, h] = O.combine(np.stack([x for x, _ in pp]), np.array([y for _, y in pp]))
        ref_parts.append(rp.reshape(B * Hq, d))
        ref_lses.append(rl.reshape(B * Hq))
    o16, _, L = ta.turbo_combine_lse(torch.stack(parts), torch.stack(lses))
    torch.cuda.synchronize()
    ref_p, ref_l = np.stack(ref_parts), np.stack(ref_lses)
    for r in range(W):
        np.testing.assert_allclose(parts[r].cpu().numpy(), ref_p[r], atol=2e-3, rtol=1e-3)
        np.testing.assert_allclose(lses[r].cpu().numpy(), ref_l[r], atol=1e-4, rtol=1e-5)
    for row in range(B * Hq):
        ro, rl = O.combine(ref_p[:, row], ref_l[:, row])
        assert np.abs(o16[row].float().cpu().numpy() - ro).max() <= MAX_ABS
        assert abs(L[row].item() - rl) < 1e-4


@pytest.mark.parametrize("shape", [(2, 300, 8, 128), (1, 128, 1, 64)])
def test_head_priority_planner_parity(ta, shape):
    """NEXT-1: per-slot priority (gap x std of channel gaps)
    bit-exact against the oracle; the plan (n_h lowest -> 2 bits) identical."""
    B, N, Hkv, d = shape
    _, k, v = synth.qkv(606 + N, B, N, Hkv, Hkv, d)
    pr = ta.turbo_head_priority(torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda())
    torch.cuda.synchronize()
    pr = pr.cpu().numpy()
    ref = np.zeros((Hkv, 2))
    for h in range(Hkv):
        for kind, x in enumerate((k, v)):
            ref[h, kind] = O.head_priority(x[:, :, h].reshape(B * N, d).astype(np.float32))
    np.testing.assert_array_equal(pr, ref)
    n2 = Hkv
    bits = ta.turbo_plan_bits(torch.from_numpy(pr), n2).numpy()
    np.testing.assert_array_equal(bits.reshape(-1), O.plan_bits(ref.reshape(-1), n2))


def test_planner_drives_the_cache_end_to_end(ta):
    """NEXT-1 end to end: the on-device plan (turbo_head_priority -> turbo_plan_bits, half of the
    slots at 2 bits) configures the cache that turbo_quantize_kv fills; records and the
    decode match the oracle run with the oracle's own plan over the same K/V."""
    B, N, Hq, Hkv, d = 2, 64 * 6 + 21, 16, 4, 128
    q, k, v = synth.qkv(808, B, N, Hq, Hkv, d)
    kt, vt = torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda()
    bits = ta.turbo_plan_bits(ta.turbo_head_priority(kt, vt), Hkv).numpy().reshape(Hkv, 2)
    ref_pr = np.array([[O.head_priority(x[:, :, h].reshape(B * N, d).astype(np.float32)) for x in (k, v)]
                       for h in range(Hkv)])
    ref_bits = O.plan_bits(ref_pr.reshape(-1), Hkv).reshape(Hkv, 2)
    np.testing.assert_array_equal(bits, ref_bits)
    assert (bits == 2).sum() == Hkv and len(set(bits.reshape(-1))) == 2
    p = ta.params(head_dim=d)
    maxb = N // 64 + 2
    cache = ta.KVCache(B, Hkv, d, max_blocks=maxb, bits=bits)
    ta.turbo_quantize_kv(p, cache, kt, vt)
    qd, _, _ = synth.decode_token(809, B, Hq, Hkv, d)
    o, _, lse = ta.turbo_attention_decode(p, cache, torch.from_numpy(qd).cuda(), n_splits=1)
    torch.cuda.synchronize()
    op = O.params(d=d)
    ref = O.build_cache(op, k.astype(np.float32), v.astype(np.float32), ref_bits, maxb)
    recs = cache.records().cpu().numpy()
    for b in range(B):
        for h in range(Hkv):
            for kind, sl in enumerate(ref["slots"][b][h]):
                for j in range(sl.n_blocks):
                    codes, s_int, z_int = cache_layout.unpack_record(recs[b, h, kind, j], d, int(ref_bits[h][kind]),
                                                                     kind)
                    np.testing.assert_array_equal(codes, sl.codes[j])
                    np.testing.assert_array_equal(s_int, sl.s_int[j])
        ro, rl = _oracle_decode(op, qd[b].astype(np.float32), ref["slots"][b], Hq // Hkv, [(0, N // 64)])
        assert_out_close(o[b].cpu().numpy(), ro, f"b{b}")
        np.testing.assert_allclose(lse[b].cpu().numpy(), rl, atol=1e-4, rtol=1e-5)


@pytest.mark.parametrize("which,lo,hi", [(0, 0x04000000, 0x7F7FFFFF), (1, 0x03800000, 0x7E800000)])
def test_fast_division_exhaustive(ta, which, lo, hi):
    """The fast correctly rounded a/119 and 119/a used for the stage-1 and P
    scales equal IEEE division for every binary32 in the domain: a/119 for all
    positive normals with a normal quotient (a >= 2^-119); 119/a for
    2^-120 <= a <= 2^126 (above 2^126 the reciprocal estimate is subnormal and
    flushed).  Every scale the path forms is in range: P maxima are <= 1 and
    FP16 inputs are <= 65504."""
    bad, first = ta.turbo_selftest_div(which, lo, hi)
    assert bad == 0, f"{bad} mismatches, first at bits {first:#010x}"


@pytest.mark.parametrize("Hq,Hkv,d", [(8, 2, 128), (16, 2, 128), (8, 2, 64), (16, 2, 64)])
def test_reference_workers_match_b200(ta, Hq, Hkv, d):
    """The deterministic default schedule assumes the B200's resident decode warps; on a B200 the
    device's own count must equal it (so the default keeps the measured-fastest schedule)."""
    if torch.cuda.get_device_properties(0).multi_processor_count != ta.B200_SMS:
        pytest.skip("not a 148-SM B200")
    assert ta.turbo_decode_workers(Hq, Hkv, d) == ta.reference_workers(Hq, Hkv, d)


def test_combine_at_the_part_bound(ta):
    """turbo_combine_lse at n_parts = 12000 (the documented maximum): the weights need > 48 KB of
    shared memory with the static part, which the launch raises explicitly."""
    S, rows, d = 12000, 2, 64
    rng = np.random.default_rng(7)
    parts = rng.standard_normal((S, rows, d)).astype(np.float32)
    lses = rng.standard_normal((S, rows)).astype(np.float32)
    o, _, lse = ta.turbo_combine_lse(torch.from_numpy(parts).cuda(), torch.from_numpy(lses).cuda())
    torch.cuda.synchronize()
    for r in range(rows):
        ro, rl = O.combine(parts[:, r], lses[:, r])
        np.testing.assert_allclose(o[r].float().cpu().numpy(), ro, atol=2e-3, rtol=0)
        assert abs(lse[r].item() - rl) < 1e-4


def test_seq_sharded_prefill_global_universal_scale(ta):
    """Sequence-sharded cache construction (parallel.prefill_seq_sharded, emulated ranks on one GPU):
    every rank quantises its whole blocks, the per-rank a_univ are reduced by MAX (the all-reduce),
    then the last rank quantises the tail with the global scale (turbo_quantize_kv mode 2).  The
    blocks, the universal scales and the buffer equal the single-device cache bit for bit (R-9)."""
    from paper_2412_08585_b200 import parallel

    B, N, Hkv, d, W = 2, 64 * 11 + 37, 2, 128, 3
    _, k, v = synth.qkv(4250, B, N, Hkv, Hkv, d)
    k[1, 40, 1] *= 6.0   # the largest |K| of (b=1, kv head 1) on rank 0: the tail must use it
    v[0, N - 5, 0] *= 3.0  # the largest |V| of (b=0, kv head 0) in the tail itself
    bits = synth.head_bits_alternating(Hkv)
    p = ta.params(head_dim=d)
    kt, vt = torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda()
    whole = ta.KVCache(B, Hkv, d, max_blocks=16, bits=bits)
    ta.turbo_quantize_kv(p, whole, kt, vt)
    caches, amax = [], []
    for r in range(W):
        t0, t1 = parallel.seq_shard_tokens(N, W, r)
        c = ta.KVCache(B, Hkv, d, max_blocks=16, bits=bits)
        amax.append(parallel.prefill_shard_blocks(p, c, kt[:, t0:t1], vt[:, t0:t1]))
        caches.append((c, t0, t1))
    a_glob = torch.stack(amax).amax(0)
    for c, t0, t1 in caches:
        parallel.prefill_shard_tail(p, c, kt[:, t0:t1], vt[:, t0:t1], a_glob)
    torch.cuda.synchronize()
    nau = B * Hkv * 2
    last = caches[-1][0]
    np.testing.assert_array_equal(last.a_univ[:nau].cpu().numpy(), whole.a_univ[:nau].cpu().numpy())
    np.testing.assert_array_equal(last.buf.cpu().numpy(), whole.buf.cpu().numpy())
    np.testing.assert_array_equal(last.counters.view(B, 2)[:, 1].cpu().numpy(),
                                  whole.counters.view(B, 2)[:, 1].cpu().numpy())
    rw = whole.records().cpu().numpy()
    for c, t0, t1 in caches:
        nb = (t1 - t0) // 64
        np.testing.assert_array_equal(c.records().cpu().numpy()[:, :, :, :nb], rw[:, :, :, t0 // 64:t0 // 64 + nb])


@pytest.mark.parametrize("Hq,Hkv,d,S", [(32, 2, 128, 1), (32, 2, 128, 3), (24, 2, 128, 2), (18, 2, 64, 1),
                                        (32, 2, 128, 0)])
def test_decode_large_gqa_groups(ta, Hq, Hkv, d, S):
    """G > 8 query rows per KV head (G = 16, 12, 9): each KV head runs as r virtual heads of G / r <= 8
    rows (include/turbo_attention.h) over the same cache; equal splits and the balanced schedule."""
    B, N, n_app = 2, 64 * 5 + 21, 3
    G = Hq // Hkv
    q, k, v = synth.qkv(8800 + Hq, B, N, Hq, Hkv, d)
    bits = synth.head_bits_alternating(Hkv)
    p, op = ta.params(head_dim=d), O.params(d=d)
    maxb = (N + n_app) // 64 + 2
    cache = ta.KVCache(B, Hkv, d, max_blocks=maxb, bits=bits)
    ta.turbo_quantize_kv(p, cache, torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda())
    ref = O.build_cache(op, k.astype(np.float32), v.astype(np.float32), bits, maxb)
    for t in range(n_app):
        _, kt, vt = synth.decode_token(8900 + t, B, Hq, Hkv, d)
        ta.turbo_quantize_kv(p, cache, torch.from_numpy(kt).cuda(), torch.from_numpy(vt).cuda(), mode=1)
        for b in range(B):
            for h in range(Hkv):
                ref["slots"][b][h][0].append(kt[b, h].astype(np.float32))
                ref["slots"][b][h][1].append(vt[b, h].astype(np.float32))
    qd, _, _ = synth.decode_token(8999, B, Hq, Hkv, d)
    o, _, lse = ta.turbo_attention_decode(p, cache, torch.from_numpy(qd).cuda(), n_splits=S)
    torch.cuda.synchronize()
    o, lse = o.cpu().numpy(), lse.cpu().numpy()
    nb = ref["slots"][0][0][0].n_blocks
    r = ta.decode_row_groups(G)
    Gv, Hv = G // r, Hkv * r
    if S > 0:
        per = -(-nb // S)
        bounds = [(min(s * per, nb), min(s * per + per, nb)) for s in range(S)]
    else:  # the balanced partition over the virtual heads
        units = [ref["slots"][b][0][0].n_blocks + (1 if ref["slots"][b][0][0].n_buf > 0 else 0) for b in range(B)]
        rng = ta.balanced_ranges(units, Hv, ta.turbo_decode_workers(Hq, Hkv, d))
    for b in range(B):
        for hq in range(Hq):
            ks, vs = ref["slots"][b][hq // G]
            pieces = ([(a_, e_, s == len(bounds) - 1) for s, (a_, e_) in enumerate(bounds)] if S > 0 else
                      [(u0, min(u1, nb), u1 > nb) for u0, u1 in rng[(b, hq // Gv)]])
            parts = [O.decode_head(op, qd[b, hq].astype(np.float32), ks, vs, a_, e_, wb) for a_, e_, wb in pieces]
            if len(parts) == 1:
                ro, rl = parts[0]
            else:
                ro, rl = O.combine(np.stack([x[0] for x in parts]), np.array([x[1] for x in parts]))
            assert_out_close(o[b, hq], ro, f"b{b} h{hq}")
            np.testing.assert_allclose(lse[b, hq], rl, atol=1e-4, rtol=1e-5)


@pytest.mark.parametrize("d", [64, 128])
def test_prefill_whole_blocks_resets_a_used_cache(ta, d):
    """A PREFILL of a whole number of B_c blocks writes the buffer and the counters inside
    quant_prefill_kernel (no memset, no tail launch): on a cache that already holds a buffered
    tail and appended tokens, the buffer must come back all zero, the counters (N / B_c, 0), the
    universal scales and records those of the new prefill, and an append + decode must match the
    oracle (Alg. 2)."""
    B, Hq, Hkv = 2, 8, 2
    G = Hq // Hkv
    bits = synth.head_bits_alternating(Hkv)
    p = ta.params(head_dim=d)
    op = O.params(d=d)
    cache = ta.KVCache(B, Hkv, d, max_blocks=8, bits=bits)
    _, k0, v0 = synth.qkv(41, B, 200, Hq, Hkv, d)  # 3 blocks + an 8-token buffered tail
    ta.turbo_quantize_kv(p, cache, torch.from_numpy(k0).cuda(), torch.from_numpy(v0).cuda())
    for t in range(5):
        _, kt, vt = synth.decode_token(600 + t, B, Hq, Hkv, d)
        ta.turbo_quantize_kv(p, cache, torch.from_numpy(kt).cuda(), torch.from_numpy(vt).cuda(), mode=1)
    torch.cuda.synchronize()
    assert cache.buf.abs().sum().item() > 0
    N = 256
    q, k, v = synth.qkv(43, B, N, Hq, Hkv, d)
    ta.turbo_quantize_kv(p, cache, torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda())
    torch.cuda.synchronize()
    assert not cache.buf.any().item()
    np.testing.assert_array_equal(cache.counters.view(B, 2).cpu().numpy(), [[N // 64, 0]] * B)
    ref = O.build_cache(op, k.astype(np.float32), v.astype(np.float32), bits, 8)
    a_univ = cache.a_univ.view(B, Hkv, 2).cpu().numpy()
    recs = cache.records().cpu().numpy()
    for b in range(B):
        for h in range(Hkv):
            for kind, sl in enumerate(ref["slots"][b][h]):
                assert a_univ[b, h, kind] == sl.a_univ and sl.n_buf == 0
                for j in range(sl.n_blocks):
                    codes, s_int, z_int = cache_layout.unpack_record(recs[b, h, kind, j], d, int(bits[h][kind]), kind)
                    np.testing.assert_array_equal(codes, sl.codes[j])
    _, kt, vt = synth.decode_token(700, B, Hq, Hkv, d)
    ta.turbo_quantize_kv(p, cache, torch.from_numpy(kt).cuda(), torch.from_numpy(vt).cuda(), mode=1)
    for b in range(B):
        for h in range(Hkv):
            ref["slots"][b][h][0].append(kt[b, h].astype(np.float32))
            ref["slots"][b][h][1].append(vt[b, h].astype(np.float32))
    qd, _, _ = synth.decode_token(701, B, Hq, Hkv, d)
    o, _, lse = ta.turbo_attention_decode(p, cache, torch.from_numpy(qd).cuda(), n_splits=1)
    torch.cuda.synchronize()
    o, lse = o.cpu().numpy(), lse.cpu().numpy()
    nb = ref["slots"][0][0][0].n_blocks
    for b in range(B):
        ro, rl = _oracle_decode(op, qd[b].astype(np.float32), ref["slots"][b], G, [(0, nb)])
        assert_out_close(o[b], ro, f"decode b{b}")
        np.testing.assert_allclose(lse[b], rl, atol=1e-4, rtol=1e-5)


@pytest.mark.parametrize("bc", [64, 128])
@pytest.mark.parametrize("d", [64, 128])
def test_quantize_kv_fallback_kernel_matches_tma_kernel(ta, bc, d):
    """turbo_quantize_kv runs the persistent TMA kernel (channel-pair body); the per-block kernel (16-byte LDG
    staging, thread = channel) is the fallback for inputs a tensor map cannot describe (TURBO_QUANT_NOTMA=1
    forces it).  Both must write the same stage-1 operands, records, scales, universal scales, buffer and
    counters, bit for bit -- for a PREFILL with a ragged tail and for a chunk that starts inside a block and
    continues over whole blocks (mode 2 after appends, R-31)."""
    import os

    B, N, Hkv = 2, 64 * 5 + 17, 4
    _, k, v = synth.qkv(77 + d, B, N, Hkv, Hkv, d)
    _, kc, vc = synth.qkv(78 + d, B, 3 * bc + 9, Hkv, Hkv, d)
    bits = synth.head_bits_alternating(Hkv)
    p = ta.params(head_dim=d, block_kv=bc)
    kt, vt, kct, vct = (torch.from_numpy(x).cuda() for x in (k, v, kc, vc))
    outs = []
    for force in (False, True):
        cache = ta.KVCache(B, Hkv, d, max_blocks=(N + kc.shape[1]) // bc + 4, bits=bits, block_kv=bc)
        if force:
            os.environ["TURBO_QUANT_NOTMA"] = "1"
        try:
            ops = ta.turbo_quantize_kv(p, cache, kt, vt)
            torch.cuda.synchronize()
            got = [x.cpu() for x in ops]
            Nk = N + kc.shape[1]
            buf = ta.turbo_dequantize_cache(p, cache, Nk)
            ops2 = ta.turbo_quantize_kv(p, cache, kct, vct, mode=2, out=buf)
            torch.cuda.synchronize()
            got += [x.cpu() for x in ops2]
        finally:
            os.environ.pop("TURBO_QUANT_NOTMA", None)
        outs.append(got + [t.cpu() for t in (cache.block_rec, cache.s_parent, cache.buf, cache.a_univ,
                                             cache.counters)])
    for a, b in zip(*outs):
        assert torch.equal(a, b)
