"""Pins of the oracle's chunked-prefill path (R-28, NEXT-3; CPU): the core it shares
with the plain prefill, the row independence of Alg. 1's outer loop, and
the cache built chunk by chunk against the cache built in one prefill."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2412_08585_b200 import synth


def _qkv(seed, n, d):
    q, k, v = synth.qkv(seed, 1, n, 1, 1, d)
    return (x[0, :, 0].astype(np.float32) for x in (q, k, v))


@pytest.mark.parametrize("n,causal", [(64, True), (200, True), (130, False)])
def test_chunk_without_prefix_is_the_prefill(n, causal):
    d = 64
    p = O.params(d=d)
    q, k, v = _qkv(11 + n, n, d)
    ks, vs = O.Slot(p, 4, n // 64 + 1), O.Slot(p, 4, n // 64 + 1)
    k1, sk = ks.prefill(k)
    v1, sv = vs.prefill(v)
    o_ref, l_ref = O.prefill_head(p, q, k, v, causal=causal)
    o, l = O.prefill_chunk_head(p, q, k1, sk, v1, sv, causal=causal)
    np.testing.assert_array_equal(o, o_ref)
    np.testing.assert_array_equal(l, l_ref)


@pytest.mark.parametrize("prefix,nq", [(64, 64), (128, 100), (192, 1)])
def test_chunk_rows_equal_the_full_prefill_rows(prefix, nq):
    """Given the same stage-1 operands, the chunk's rows are the full prefill's rows
    (the query blocks of the chunk coincide with the full call's when prefix % B_r == 0)."""
    d = 128
    p = O.params(d=d, block_q=64)
    n = prefix + nq
    q, k, v = _qkv(7 + n, n, d)
    ks, vs = O.Slot(p, 2, n // 64 + 1), O.Slot(p, 4, n // 64 + 1)
    k1, sk = ks.prefill(k)
    v1, sv = vs.prefill(v)
    i0 = prefix // 64
    o_ref, l_ref = O.prefill_head(p, q, k, v, causal=True, blocks=(i0, 10 ** 6))
    o, l = O.prefill_chunk_head(p, q[prefix:], k1, sk, v1, sv, causal=True)
    np.testing.assert_array_equal(o, o_ref[prefix:])
    np.testing.assert_array_equal(l, l_ref[prefix:])


@pytest.mark.parametrize("bits", [2, 4])
def test_cache_built_by_chunks_equals_one_prefill(bits):
    d, n1, n2 = 64, 128, 150
    p = O.params(d=d)
    _, k, _ = _qkv(3, n1 + n2, d)
    a = O.Slot(p, bits, 8)
    a.prefill(k)
    b = O.Slot(p, bits, 8)
    b.prefill(k[:n1])
    x1, sc = b.prefill_append(k[n1:])
    assert (a.n_blocks, a.n_buf) == (b.n_blocks, b.n_buf) == ((n1 + n2) // 64, (n1 + n2) % 64)
    assert a.a_univ == b.a_univ
    for arr in ("codes", "s_int", "z_int", "s_parent"):
        np.testing.assert_array_equal(getattr(a, arr)[:a.n_blocks], getattr(b, arr)[:b.n_blocks])
    np.testing.assert_array_equal(a.buf[:a.n_buf], b.buf[:b.n_buf])
    full_x1, full_sc = O.Slot(p, bits, 8).prefill(k)
    np.testing.assert_array_equal(x1, full_x1[n1:])
    np.testing.assert_array_equal(sc, full_sc[n1 // 64:])
    with pytest.raises(ValueError):  # a buffered tail first: the chunk would not start a block
        c = O.Slot(p, bits, 8)
        c.prefill(k[:100])
        c.prefill_append(k[100:])


def test_chunk_over_a_lossless_compressed_prefix():
    """Prefix channels spanning <= 3 stage-1 codes per block: stage 2 is lossless at 2 and
    4 bits, so the stage-1 reconstruction of the cache equals the prefix's stage-1
    codes and the chunked prefill equals the full prefill's chunk rows."""
    d, prefix, nq = 64, 128, 64
    p = O.params(d=d)
    rng = np.random.default_rng(5)
    n = prefix + nq
    q, k, v = (np.float32(x) for x in _qkv(9, n, d))
    for x in (k, v):  # per block: a channel-wise constant pattern, every token equal -> 1 code per channel
        for j in range(prefix // 64):
            x[j * 64:(j + 1) * 64] = np.float16(rng.standard_normal(d)).astype(np.float32)
    ks, vs = O.Slot(p, 2, n // 64 + 1), O.Slot(p, 4, n // 64 + 1)
    k_pre1, _ = ks.prefill(k[:prefix])
    v_pre1, _ = vs.prefill(v[:prefix])
    kc1, skc = ks.prefill_append(k[prefix:])
    vc1, svc = vs.prefill_append(v[prefix:])
    kp, skp = ks.stage1_prefix(prefix // 64)
    vp, svp = vs.stage1_prefix(prefix // 64)
    np.testing.assert_array_equal(kp, k_pre1)
    np.testing.assert_array_equal(vp, v_pre1)
    o, l = O.prefill_chunk_head(p, q[prefix:], np.concatenate([kp, kc1]), np.concatenate([skp, skc]),
                                np.concatenate([vp, vc1]), np.concatenate([svp, svc]))
    o_ref, l_ref = O.prefill_head(p, q, k, v, causal=True)
    np.testing.assert_array_equal(o, o_ref[prefix:])
    np.testing.assert_array_equal(l, l_ref[prefix:])
