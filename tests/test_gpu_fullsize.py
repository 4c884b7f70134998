"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py
times (-m gpu): the GPU runs the whole problem, the oracle recomputes sampled
(batch, head) units -- or sampled query blocks of Alg. 1's independent outer
loop -- one by one on the same seeded inputs (synth.qkv_torch with
bench.py's seeds, copied back to the host).

Bar as in test_gpu_parity.py: codes / scales / records bit-exact, FP16 O within
max-abs 2e-3 and rel-L2 1e-3 of the oracle's FP32 O, LSE within 1e-4.
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


def _close(gpu, ref, what):
    g = np.asarray(gpu, np.float32)
    err = float(np.abs(g - ref).max())
    rl = float(np.linalg.norm((g - ref).astype(np.float64)) / max(np.linalg.norm(ref.astype(np.float64)), 1e-30))
    assert err <= MAX_ABS and rl <= REL_L2, f"{what}: max-abs {err:.3e} rel-L2 {rl:.3e}"


def _host(x):
    return x.float().cpu().numpy()


def test_fullsize_prefill_configs1(ta):
    """configs[1] (bench.py's step): B=8, N=4096, 32/8 heads, d=128, causal, B_r=64, alpha_mode 0."""
    B, N, Hq, Hkv, d = 8, 4096, 32, 8, 128
    G = Hq // Hkv
    bits = synth.head_bits_alternating(Hkv)
    p = ta.params(head_dim=d, block_q=64, alpha_mode=0)
    q, k, v = synth.qkv_torch(1002, B, N, Hq, Hkv, d)
    cache = ta.KVCache(B, Hkv, d, max_blocks=N // 64 + 2, bits=bits)
    k1, v1t, k1s, v1s = ta.turbo_quantize_kv(p, cache, k, v)
    o, lse = ta.turbo_attention_prefill(p, q, k1, v1t, k1s, v1s)
    torch.cuda.synchronize()
    op = O.params(d=d, block_q=64, alpha_mode=0)
    tc = N // 64
    for b, kvh in ((0, 0), (5, 3), (7, 7)):
        kh, vh = _host(k[b, :, kvh]), _host(v[b, :, kvh])
        ks, vs = O.Slot(op, int(bits[kvh][0]), N // 64 + 2), O.Slot(op, int(bits[kvh][1]), N // 64 + 2)
        rk1, rk1s = ks.prefill(kh)
        rv1, rv1s = vs.prefill(vh)
        np.testing.assert_array_equal(k1[b, kvh].cpu().numpy(), rk1)
        np.testing.assert_array_equal(k1s[b, kvh].cpu().numpy(), rk1s)
        np.testing.assert_array_equal(v1s[b, kvh].cpu().numpy(), rv1s)
        gv1 = v1t[b, kvh].float().cpu().numpy().astype(np.int8).transpose(0, 2, 1).reshape(tc * 64, d)
        np.testing.assert_array_equal(gv1, rv1)
        recs = cache.records()[b, kvh].cpu().numpy()
        for kind, sl in enumerate((ks, vs)):
            for j in (0, 1, sl.n_blocks // 2, sl.n_blocks - 1):
                codes, s_int, z_int = cache_layout.unpack_record(recs[kind, j], d, int(bits[kvh][kind]), kind)
                np.testing.assert_array_equal(codes, sl.codes[j])
                np.testing.assert_array_equal(s_int, sl.s_int[j])
                np.testing.assert_array_equal(z_int, sl.z_int[j])
        # one query head of the group in full, the others on sampled query blocks
        for i, h in enumerate(range(kvh * G, kvh * G + G)):
            blocks = None if i == 0 else ((0, 2), (31, 33), (62, 64))[i - 1]
            ro, rl = O.prefill_head(op, _host(q[b, :, h]), kh, vh, causal=True, blocks=blocks)
            r0, r1 = (0, N) if blocks is None else (blocks[0] * 64, blocks[1] * 64)
            _close(_host(o[b, r0:r1, h]), ro[r0:r1], f"b{b} h{h} rows {r0}:{r1}")
            np.testing.assert_allclose(lse[b, h, r0:r1].cpu().numpy(), rl[r0:r1], atol=1e-4, rtol=1e-5)


def test_fullsize_prefill_configs3(ta):
    """configs[3]: Llama-3-70B shape, B=1, N=32k, 64/8 heads (the single-GPU launch
    of bench.py --workload prefill_70b); sampled query blocks of sampled heads."""
    B, N, Hq, Hkv, d = 1, 32768, 64, 8, 128
    G = Hq // Hkv
    bits = synth.head_bits_alternating(Hkv)
    p = ta.params(head_dim=d, block_q=64, alpha_mode=0)
    q, k, v = synth.qkv_torch(5005, B, N, Hq, Hkv, d)
    cache = ta.KVCache(B, Hkv, d, max_blocks=N // 64 + 2, bits=bits)
    k1, v1t, k1s, v1s = ta.turbo_quantize_kv(p, cache, k, v)
    o, lse = ta.turbo_attention_prefill(p, q, k1, v1t, k1s, v1s)
    torch.cuda.synchronize()
    op = O.params(d=d, block_q=64, alpha_mode=0)
    for h, blocks in ((0, (0, 1)), (37, (255, 256)), (63, (511, 512))):
        kvh = h // G
        ro, rl = O.prefill_head(op, _host(q[0, :, h]), _host(k[0, :, kvh]), _host(v[0, :, kvh]), causal=True,
                                blocks=blocks)
        r0, r1 = blocks[0] * 64, blocks[1] * 64
        _close(_host(o[0, r0:r1, h]), ro[r0:r1], f"h{h} rows {r0}:{r1}")
        np.testing.assert_allclose(lse[0, h, r0:r1].cpu().numpy(), rl[r0:r1], atol=1e-4, rtol=1e-5)


def _decode_fullsize(ta, B, N, Hq, Hkv, d, seed_kv, seed_tok, alpha_mode, samples, S):
    """Cache build + one APPEND + split-KV decode in bench.py's configuration
    (S > 1: equal splits, bench.py's auto_splits; S = 0: the balanced schedule); the oracle rebuilds
    sampled (b, kv_head) slots and decodes their G query heads over the same
    sub-ranges, then combines."""
    G = Hq // Hkv
    bits = synth.head_bits_alternating(Hkv)
    p = ta.params(head_dim=d, alpha_mode=alpha_mode)
    cache = ta.KVCache(B, Hkv, d, max_blocks=N // 64 + 4, bits=bits)
    _, k, v = synth.qkv_torch(seed_kv, B, N, Hkv, Hkv, d)
    ta.turbo_quantize_kv(p, cache, k, v)
    qd, kd, vd = (x[:, 0].contiguous() for x in synth.qkv_torch(seed_tok, B, 1, Hq, Hkv, d))
    ta.turbo_quantize_kv(p, cache, kd, vd, mode=1)
    o, _, lse = ta.turbo_attention_decode(p, cache, qd, n_splits=S)
    torch.cuda.synchronize()
    op = O.params(d=d, alpha_mode=alpha_mode)
    nb = N // 64
    if S > 0:
        per = -(-nb // S)
        pieces = {key: [(min(s * per, nb), min(s * per + per, nb), s == S - 1) for s in range(S)] for key in samples}
    else:  # every sequence: nb blocks + the 1-token buffer block
        rng = ta.balanced_ranges([nb + 1] * B, Hkv, ta.turbo_decode_workers(Hq, Hkv, d))
        pieces = {key: [(u0, min(u1, nb), u1 > nb) for u0, u1 in rng[key]] for key in samples}
        assert max(len(x) for x in pieces.values()) > 1
    for b, kvh in samples:
        ks, vs = O.Slot(op, int(bits[kvh][0]), nb + 4), O.Slot(op, int(bits[kvh][1]), nb + 4)
        ks.prefill(_host(k[b, :, kvh]))
        vs.prefill(_host(v[b, :, kvh]))
        ks.append(_host(kd[b, kvh]))
        vs.append(_host(vd[b, kvh]))
        recs = cache.records()[b, kvh].cpu().numpy()
        for kind, sl in enumerate((ks, vs)):
            for j in (0, nb // 3, nb - 1):
                codes, s_int, z_int = cache_layout.unpack_record(recs[kind, j], d, int(bits[kvh][kind]), kind)
                np.testing.assert_array_equal(codes, sl.codes[j])
                np.testing.assert_array_equal(s_int, sl.s_int[j])
                np.testing.assert_array_equal(z_int, sl.z_int[j])
        for h in range(kvh * G, kvh * G + G):
            qh = _host(qd[b, h])
            parts = [O.decode_head(op, qh, ks, vs, a_, e_, wb) for a_, e_, wb in pieces[(b, kvh)]]
            if len(parts) == 1:
                ro, rl = parts[0]
            else:
                ro, rl = O.combine(np.stack([x for x, _ in parts]), np.array([y for _, y in parts], np.float32))
            _close(_host(o[b, h]), ro, f"decode b{b} h{h}")
            assert abs(float(lse[b, h]) - float(rl)) <= 1e-4


def test_fullsize_decode_configs2(ta):
    """configs[2] (bench.py's decode object): Phi-3-medium 40/10 heads, B=64, 32k, mixed bits."""
    _decode_fullsize(ta, 64, 32768, 40, 10, 128, 3003, 6000, 0, ((0, 0), (37, 5), (63, 9)),
                     ta.auto_splits(64, 10, 512, ta.turbo_decode_workers(40, 10, 128)))


def test_fullsize_decode_configs2_balanced(ta):
    """configs[2] with the balanced schedule (n_splits = 0), the other schedule."""
    _decode_fullsize(ta, 64, 32768, 40, 10, 128, 3003, 6000, 0, ((37, 5),), 0)


def test_fullsize_decode_configs4(ta):
    """configs[4] on one rank (bench.py --workload decode_long): 128k context, B=16, 32/8 heads, alpha_mode 1."""
    _decode_fullsize(ta, 16, 131072, 32, 8, 128, 9009, 7000, 1, ((0, 0), (15, 7)),
                     ta.auto_splits(16, 8, 2048, ta.turbo_decode_workers(32, 8, 128)))
