"""Chunked prefill (NEXT-3, reading R-28) on the GPU against the oracle, through the
C-ABI: a prefix prefill, the stage-1 reconstruction of its cached blocks
(turbo_dequantize_cache), a further chunk (turbo_quantize_kv mode 2) and
turbo_attention_prefill_chunk.  Bit-exact: the stage-1 operands of prefix and
chunk, every cache record, the universal scales, the buffer and the counters;
tolerance set: O and L."""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2412_08585_b200 import synth
from tests import cache_layout
from tests.test_gpu_parity import assert_out_close, ta  # noqa: F401  (fixture)

pytestmark = pytest.mark.gpu

CASES = [  # (B, P, Nq, Hq, Hkv, d, causal, B_c)
    (2, 128, 64, 8, 2, 128, True, 64),
    (1, 256, 100, 4, 1, 128, True, 64),    # ragged chunk: its tail goes to the buffer
    (2, 64, 1, 8, 2, 128, True, 64),       # one-token chunk
    (1, 192, 130, 2, 2, 64, True, 64),     # d = 64
    (1, 128, 70, 4, 2, 128, False, 64),    # non-causal: every query sees all P + Nq keys
    (1, 128, 300, 2, 2, 128, True, 64),    # MHA: query-tile pairs with a prefix offset
    # R-31: the cache ends inside a block (buffered tail) -- the chunk completes it as appends do
    (1, 100, 20, 4, 2, 128, True, 64),     # the chunk stays inside the boundary block
    (2, 100, 200, 8, 2, 128, True, 64),    # boundary block flushed, then aligned blocks + tail
    (1, 200, 1, 4, 1, 128, True, 64),      # one token into the buffer
    (1, 70, 60, 2, 2, 64, False, 64),      # d = 64, non-causal, exactly fills the block
    (1, 130, 300, 4, 2, 128, True, 128),   # B_c = 128
    (1, 37, 150, 6, 2, 128, True, 64),     # prefix shorter than one block (buffer only)
]


@pytest.mark.parametrize("case", CASES)
def test_chunked_prefill_parity(ta, case):  # noqa: F811
    B, P, Nq, Hq, Hkv, d, causal, bc = case
    G, Nk = Hq // Hkv, P + Nq
    q, k, v = synth.qkv(4100 + Nk, B, Nk, Hq, Hkv, d)
    bits = synth.head_bits_alternating(Hkv)
    p = ta.params(head_dim=d, block_kv=bc)
    maxb = Nk // bc + 2
    cache = ta.KVCache(B, Hkv, d, max_blocks=maxb, bits=bits, block_kv=bc)
    dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()  # noqa: E731
    ta.turbo_quantize_kv(p, cache, dev(k[:, :P]), dev(v[:, :P]))
    ops = ta.turbo_dequantize_cache(p, cache, Nk)
    ta.turbo_quantize_kv(p, cache, dev(k[:, P:]), dev(v[:, P:]), mode=2, out=ops)
    o, lse = ta.turbo_attention_prefill_chunk(p, dev(q[:, P:]), *ops, causal=causal)
    torch.cuda.synchronize()
    assert cache.n_tokens == Nk
    k1, v1t, k1s, v1s = (x.cpu().numpy() for x in ops)
    o, lse = o.cpu().numpy(), lse.cpu().numpy()
    recs = cache.records().cpu().numpy()
    cnt = cache.counters.view(B, 2).cpu().numpy()
    a_univ = cache.a_univ.view(B, Hkv, 2).cpu().numpy()
    buf = cache.buf.view(B, Hkv, 2, bc * d).cpu().numpy()
    op = O.params(d=d, block_kv=bc)
    for b in range(B):
        for h in range(Hkv):
            ops_ref = []
            for kind, x in ((0, k), (1, v)):
                sl = O.Slot(op, int(bits[h][kind]), maxb)
                sl.prefill(x[b, :P, h].astype(np.float32))
                xp, sp = sl.stage1_prefix(P // bc, with_buffer=True)
                xc, sc = sl.prefill_append(x[b, P:, h].astype(np.float32))
                ops_ref.append((np.concatenate([xp, xc]), np.concatenate([sp, sc])))
                # cache state after both chunks
                assert tuple(cnt[b]) == (sl.n_blocks, sl.n_buf)
                assert a_univ[b, h, kind] == sl.a_univ
                for j in range(sl.n_blocks):
                    codes, s_int, z_int = cache_layout.unpack_record(recs[b, h, kind, j], d, int(bits[h][kind]), kind,
                                                                     bc=bc)
                    np.testing.assert_array_equal(codes, sl.codes[j])
                    np.testing.assert_array_equal(s_int, sl.s_int[j])
                    np.testing.assert_array_equal(z_int, sl.z_int[j])
                bb = buf[b, h, kind].reshape(bc, d) if kind == 0 else buf[b, h, kind].reshape(d, bc).T
                np.testing.assert_array_equal(bb[:sl.n_buf], sl.buf[:sl.n_buf])
            (K1, SK), (V1, SV) = ops_ref
            # stage-1 operands: prefix reconstruction + chunk, bit-exact
            np.testing.assert_array_equal(k1[b, h], K1)
            np.testing.assert_array_equal(k1s[b, h], SK)
            np.testing.assert_array_equal(v1s[b, h], SV)
            vt = v1t[b, h].astype(np.float32)  # [Tk][d][B_c] codes
            for j in range(-(-Nk // bc)):
                rows = min(bc, Nk - bc * j)
                np.testing.assert_array_equal(vt[j][:, :rows].T, V1[bc * j:bc * j + rows])
                assert not vt[j][:, rows:].any()  # keys past Nk: zero codes
            for hq in range(h * G, h * G + G):
                ro, rl = O.prefill_chunk_head(op, q[b, P:, hq].astype(np.float32), K1, SK, V1, SV, causal=causal)
                assert_out_close(o[b, :, hq], ro, f"chunk b{b} h{hq}")
                np.testing.assert_allclose(lse[b, hq], rl, atol=1e-4, rtol=1e-5)


def test_chunk_needs_the_prefix_operands(ta):  # noqa: F811
    B, N, Hkv, d = 1, 100, 1, 128
    _, k, v = synth.qkv(3, B, N + 64, Hkv, Hkv, d)
    p = ta.params(head_dim=d)
    cache = ta.KVCache(B, Hkv, d, max_blocks=8, bits=[[4, 4]])
    ta.turbo_quantize_kv(p, cache, torch.from_numpy(k[:, :N].copy()).cuda(), torch.from_numpy(v[:, :N].copy()).cuda())
    with pytest.raises(ta.TurboError):  # the buffered tail needs Nk >= the cached length
        ta.turbo_dequantize_cache(p, cache, N - 1)
    with pytest.raises(ValueError):  # the binding requires the prefix operands for mode 2
        ta.turbo_quantize_kv(p, cache, torch.from_numpy(k[:, N:].copy()).cuda(),
                             torch.from_numpy(v[:, N:].copy()).cuda(), mode=2)


def test_two_chunks_after_a_prefix(ta):  # noqa: F811
    """prefix 128 -> chunk 64 -> chunk 100: block offsets and the running universal scale
    across several chunks; the second chunk's attention and the final cache vs the oracle."""
    B, P, N1, N2, Hq, Hkv, d = 1, 128, 64, 100, 4, 2, 128
    G, Nk = Hq // Hkv, P + N1 + N2
    q, k, v = synth.qkv(4321, B, Nk, Hq, Hkv, d)
    k[:, P + 10] *= 3.0  # the second and third segments carry the largest magnitudes (universal scale grows)
    v[:, P + N1 + 5] *= 2.0
    bits = synth.head_bits_alternating(Hkv)
    p = ta.params(head_dim=d)
    maxb = Nk // 64 + 2
    cache = ta.KVCache(B, Hkv, d, max_blocks=maxb, bits=bits)
    dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()  # noqa: E731
    ta.turbo_quantize_kv(p, cache, dev(k[:, :P]), dev(v[:, :P]))
    ops1 = ta.turbo_dequantize_cache(p, cache, P + N1)
    ta.turbo_quantize_kv(p, cache, dev(k[:, P:P + N1]), dev(v[:, P:P + N1]), mode=2, out=ops1)
    ops2 = ta.turbo_dequantize_cache(p, cache, Nk)
    ta.turbo_quantize_kv(p, cache, dev(k[:, P + N1:]), dev(v[:, P + N1:]), mode=2, out=ops2)
    o, lse = ta.turbo_attention_prefill_chunk(p, dev(q[:, P + N1:]), *ops2)
    torch.cuda.synchronize()
    o, lse = o.cpu().numpy(), lse.cpu().numpy()
    recs = cache.records().cpu().numpy()
    cnt = cache.counters.view(B, 2).cpu().numpy()
    a_univ = cache.a_univ.view(B, Hkv, 2).cpu().numpy()
    buf = cache.buf.view(B, Hkv, 2, 64 * d).cpu().numpy()
    op = O.params(d=d)
    for h in range(Hkv):
        ops_ref = []
        for kind, x in ((0, k), (1, v)):
            sl = O.Slot(op, int(bits[h][kind]), maxb)
            sl.prefill(x[0, :P, h].astype(np.float32))
            sl.prefill_append(x[0, P:P + N1, h].astype(np.float32))
            xp, sp = sl.stage1_prefix((P + N1) // 64)
            xc, sc = sl.prefill_append(x[0, P + N1:, h].astype(np.float32))
            ops_ref.append((np.concatenate([xp, xc]), np.concatenate([sp, sc])))
            assert tuple(cnt[0]) == (sl.n_blocks, sl.n_buf)
            assert a_univ[0, h, kind] == sl.a_univ
            for j in range(sl.n_blocks):
                codes, s_int, z_int = cache_layout.unpack_record(recs[0, h, kind, j], d, int(bits[h][kind]), kind)
                np.testing.assert_array_equal(codes, sl.codes[j])
                np.testing.assert_array_equal(s_int, sl.s_int[j])
            # buffer: K token-major, V channel-major
            bref = sl.buf[:sl.n_buf]
            bgpu = buf[0, h, kind].reshape(64, d)[:sl.n_buf] if kind == 0 else buf[0, h, kind].reshape(d, 64)[:, :sl.n_buf].T
            np.testing.assert_array_equal(bgpu, bref)
        (K1, SK), (V1, SV) = ops_ref
        np.testing.assert_array_equal(ops2[0][0, h].cpu().numpy(), K1)
        for hq in range(h * G, h * G + G):
            ro, rl = O.prefill_chunk_head(op, q[0, P + N1:, hq].astype(np.float32), K1, SK, V1, SV)
            assert_out_close(o[0, :, hq], ro, f"chunk 2 h{hq}")
            np.testing.assert_allclose(lse[0, hq], rl, atol=1e-4, rtol=1e-5)
