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


# ---- R-31: a chunk that starts inside a block (the cache ends with a buffered tail)

@pytest.mark.parametrize("n", [1, 20, 28])
def test_mid_block_chunk_within_the_block_is_appends(n):
    """A chunk that does not leave the boundary block is exactly n decode appends:
    same buffer, counters, universal scale and flushes; its operands are the buffer codes."""
    d, P = 64, 100
    p = O.params(d=d)
    _, k, _ = _qkv(21, P + n, d)
    a, b = O.Slot(p, 4, 4), O.Slot(p, 4, 4)
    a.prefill(k[:P])
    b.prefill(k[:P])
    x1, sc = a.prefill_append(k[P:])
    for t in range(n):
        b.append(k[P + t])
    assert (a.n_blocks, a.n_buf, a.a_univ) == (b.n_blocks, b.n_buf, b.a_univ)
    for arr in ("codes", "s_int", "z_int", "s_parent"):
        np.testing.assert_array_equal(getattr(a, arr)[:a.n_blocks], getattr(b, arr)[:b.n_blocks])
    np.testing.assert_array_equal(a.buf, b.buf)
    assert sc.size == 0
    if P % 64 + n < 64:  # the operands are the buffer rows (n = 28 fills and flushes the block)
        np.testing.assert_array_equal(x1, a.buf[P % 64:P % 64 + n])


def _lossless_inputs(seed, n, d, P, bc, small=3):
    """Integer-valued Q/K/V whose every block max is 119 (channel 0 == 119): every stage-1 scale,
    the universal scale and every Q block scale are 1 and the codes are the values, whatever the
    block alignment; flushed prefix blocks are constant per channel (stage 2 lossless)."""
    rng = np.random.default_rng(seed)
    q, k, v = (rng.integers(-small, small + 1, (n, d)).astype(np.float32) for _ in range(3))
    for x in (q, k, v):
        x[:, 0] = 119.0
    for x in (k, v):
        for j in range(P // bc):
            x[j * bc:(j + 1) * bc] = x[j * bc]
    return q, k, v


@pytest.mark.parametrize("bc,P,nq,p_row", [(128, 192, 200, 0), (64, 100, 90, 1), (64, 100, 20, 1), (128, 130, 300, 1)])
def test_mid_block_chunk_lossless_equals_one_shot_prefill(bc, P, nq, p_row):
    """With lossless quantisation (every scale 1, codes = values, stage 2 exact on the flushed prefix)
    the chunk's rows -- prefix blocks reconstructed, the boundary block from the buffer at s_univ,
    the chunk's own blocks at stage 1 -- equal the one-shot prefill's rows bit for bit.  (Rows are
    independent under the per-row P scale; with the tile P scale the chunk starts a B_r block.)"""
    d = 64
    n = P + nq
    p = O.params(d=d, block_kv=bc, p_row=p_row, softmax_scale=1.0 / 64)
    q, k, v = _lossless_inputs(40 + P + nq, n, d, P, bc)
    ops = []
    for bits, x in ((2, k), (4, v)):
        sl = O.Slot(p, bits, n // bc + 2)
        x_pre1, _ = sl.prefill(x[:P])
        np.testing.assert_array_equal(x_pre1, x[:P].astype(np.int8))
        xp, sp = sl.stage1_prefix(P // bc, with_buffer=True)
        xc, sc = sl.prefill_append(x[P:])
        ops.append((np.concatenate([xp, xc]), np.concatenate([sp, sc])))
        assert sl.n_blocks * bc + sl.n_buf == n
    (k1, sk), (v1, sv) = ops
    np.testing.assert_array_equal(k1, k.astype(np.int8))
    assert (sk == 1).all() and sk.size == -(-n // bc)
    o, l = O.prefill_chunk_head(p, q[P:], k1, sk, v1, sv, causal=True)
    o_ref, l_ref = O.prefill_head(p, q, k, v, causal=True)
    np.testing.assert_array_equal(o, o_ref[P:])
    np.testing.assert_array_equal(l, l_ref[P:])


def test_mid_block_chunk_universal_scale_and_clamp():
    """The boundary tokens use the universal scale from before the chunk (clamped to +-119 when they
    exceed it); the chunk's aligned part then raises a_univ to its own max (R-28)."""
    d, P, n, bc = 64, 100, 60, 64
    p = O.params(d=d)
    _, k, _ = _qkv(23, P + n, d)
    k = k.copy()
    k[P + 2, 5] = 8 * np.abs(k[:P]).max()  # a boundary token beyond a_univ: clamped code
    k[P + 40, 7] = 4 * np.abs(k[:P]).max()  # in the aligned part: raises a_univ
    sl = O.Slot(p, 4, 4)
    sl.prefill(k[:P])
    a0 = sl.a_univ
    x1, sc = sl.prefill_append(k[P:])
    assert x1[2, 5] == 119
    assert sl.a_univ == np.float32(np.abs(k[P + bc - P % bc:]).max()) and sl.a_univ > a0
    assert sc.size == 1  # one aligned block (tokens 128..159 -> 32 in the buffer)
