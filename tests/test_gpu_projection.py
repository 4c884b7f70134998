"""The Q projection with the stage-1 Q quantisation fused into its epilogue (NEXT-3)
and the prefill that reads the quantised query (-m gpu).

Parity: with integer-valued X and W_q the product is exact in both fp32 accumulation and the
oracle's float64, so Q (fp16), its codes and scales are compared bit for bit; with Gaussian inputs
the fp16 projection is within one binary16 ulp of the float64 product and every B_r block whose fp16
Q max agrees carries the same scale and codes that differ only where the fp16 Q does (by one).  The prefill on the fused query equals the prefill on
the FP16 query bit for bit and the oracle within the usual tolerance."""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2412_08585_b200 import synth
from tests.test_gpu_parity import assert_out_close, ta  # noqa: F401  (fixture)

pytestmark = pytest.mark.gpu


def _oracle_q1(q16, Hq, d, bq):
    """Stage-1 codes and scales of the oracle's fp16 Q per (b, head, B_r block)."""
    B, N = q16.shape[:2]
    q = q16.reshape(B, N, Hq, d).astype(np.float32)
    nb = -(-N // bq)
    codes = np.zeros((B, N, Hq, d), np.int8)
    sc = np.zeros((B, Hq, nb), np.float32)
    for b in range(B):
        for h in range(Hq):
            for i in range(nb):
                c, s = O.quant_sym8(q[b, i * bq:(i + 1) * bq, h])
                codes[b, i * bq:(i + 1) * bq, h] = c
                sc[b, h, i] = s
    return codes, sc


@pytest.mark.parametrize("B,N,D,Hq,d,bq", [(2, 200, 256, 4, 128, 64), (1, 300, 512, 8, 64, 128), (1, 64, 128, 2, 128, 64)])
def test_q_projection_integer_exact(ta, B, N, D, Hq, d, bq):  # noqa: F811
    rng = np.random.default_rng(N + D)
    x = rng.integers(-3, 4, (B, N, D)).astype(np.float16)
    w = rng.integers(-2, 3, (Hq * d, D)).astype(np.float16)
    p = ta.params(head_dim=d, block_q=bq)
    q1, sq, q16 = ta.turbo_q_projection(p, torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda(), Hq, want_q16=True)
    torch.cuda.synchronize()
    qref = O.project_q(x, w)
    np.testing.assert_array_equal(q16.cpu().numpy().reshape(B, N, Hq * d), qref)
    codes, sc = _oracle_q1(qref, Hq, d, bq)
    np.testing.assert_array_equal(q1.cpu().numpy(), codes)
    np.testing.assert_array_equal(sq.cpu().numpy(), sc)


def test_q_projection_gaussian(ta):  # noqa: F811
    B, N, D, Hq, d, bq = 2, 256, 1024, 8, 128, 64
    rng = np.random.default_rng(7)
    x = (rng.standard_normal((B, N, D)) * 0.5).astype(np.float16)
    w = (rng.standard_normal((Hq * d, D)) / np.sqrt(D)).astype(np.float16)
    p = ta.params(head_dim=d, block_q=bq)
    q1, sq, q16 = ta.turbo_q_projection(p, torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda(), Hq, want_q16=True)
    torch.cuda.synchronize()
    qref = O.project_q(x, w).reshape(B, N, Hq, d)
    g = q16.cpu().numpy()
    # any fp32 summation order: |fl32(sum) - sum| <= D 2^-24 sum |x w| (Higham), then one binary16 rounding
    absdot = (np.abs(x.astype(np.float64)) @ np.abs(w.astype(np.float64)).T).reshape(B, N, Hq, d)
    bound = np.abs(np.spacing(qref.astype(np.float16))).astype(np.float64) + D * 2.0 ** -24 * absdot
    err = np.abs(g.astype(np.float64) - qref.astype(np.float64))
    assert (err <= bound).all()
    assert (err == 0).mean() > 0.99  # nearly every element is the correctly rounded product
    codes, sc = _oracle_q1(qref, Hq, d, bq)
    q1, sq = q1.cpu().numpy(), sq.cpu().numpy()
    # blocks whose max |Q| agrees have the same scale; their codes differ only where the fp16 Q does,
    # and there by at most one
    same_scale = 0
    for b in range(B):
        for h in range(Hq):
            for i in range(N // bq):
                rows = slice(i * bq, (i + 1) * bq)
                if sq[b, h, i] != sc[b, h, i]:
                    continue
                same_scale += 1
                diff = q1[b, rows, h].astype(np.int32) - codes[b, rows, h].astype(np.int32)
                assert (np.abs(diff) <= 1).all()
                assert not diff[g[b, rows, h] == qref[b, rows, h]].any()
    assert same_scale >= 0.9 * B * Hq * (N // bq)


@pytest.mark.parametrize("N,Hq,Hkv,d,bq", [(200, 8, 2, 128, 64), (333, 4, 4, 128, 128), (256, 8, 2, 64, 64)])
def test_prefill_on_the_fused_query(ta, N, Hq, Hkv, d, bq):  # noqa: F811
    B, D = 2, 256
    rng = np.random.default_rng(N)
    x = rng.integers(-3, 4, (B, N, D)).astype(np.float16)
    w = (rng.integers(-2, 3, (Hq * d, D)) * 0.0625).astype(np.float16)  # exact: multiples of 1/16
    _, k, v = synth.qkv(33 + N, B, N, Hq, Hkv, d)
    bits = synth.head_bits_alternating(Hkv)
    p = ta.params(head_dim=d, block_q=bq)
    cache = ta.KVCache(B, Hkv, d, max_blocks=N // 64 + 2, bits=bits)
    k1, v1t, k1s, v1s = ta.turbo_quantize_kv(p, cache, torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda())
    q1, sq, q16 = ta.turbo_q_projection(p, torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda(), Hq, want_q16=True)
    o1, l1 = ta.turbo_attention_prefill_q1(p, q1, sq, k1, v1t, k1s, v1s)
    o2, l2 = ta.turbo_attention_prefill(p, q16, k1, v1t, k1s, v1s)
    torch.cuda.synchronize()
    assert torch.equal(o1, o2) and torch.equal(l1, l2)
    qref = O.project_q(x, w).reshape(B, N, Hq, d)
    np.testing.assert_array_equal(q16.cpu().numpy(), qref)
    op = O.params(d=d, block_q=bq)
    o1, l1 = o1.cpu().numpy(), l1.cpu().numpy()
    G = Hq // Hkv
    for b in range(B):
        for h in range(Hq):
            oref, lref = O.prefill_head(op, qref[b, :, h].astype(np.float32), k[b, :, h // G], v[b, :, h // G])
            assert_out_close(o1[b, :, h], oref, f"b{b} h{h}")
            np.testing.assert_allclose(l1[b, h], lref, atol=1e-4, rtol=1e-5)


def test_q_projection_validation(ta):  # noqa: F811
    p = ta.params(head_dim=128)
    x = torch.zeros((1, 64, 100), dtype=torch.float16, device="cuda")  # D % 64 != 0
    w = torch.zeros((256, 100), dtype=torch.float16, device="cuda")
    with pytest.raises(ta.TurboError) as e:
        ta.turbo_q_projection(p, x, w, 2)
    assert e.value.code == ta.TURBO_ERR_UNSUPPORTED


def test_q_projection_fp16_scales(ta):  # noqa: F811
    """scale_fp16 (R-29) in the projection epilogue: the block scales are the binary16 roundings."""
    B, N, D, Hq, d, bq = 2, 128, 256, 2, 128, 64
    rng = np.random.default_rng(99)
    x = rng.integers(-3, 4, (B, N, D)).astype(np.float16)
    w = (rng.integers(-2, 3, (Hq * d, D)) * 0.03125).astype(np.float16)
    p = ta.params(head_dim=d, block_q=bq, scale_fp16=1)
    q1, sq, _ = ta.turbo_q_projection(p, torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda(), Hq)
    torch.cuda.synchronize()
    codes, sc = _oracle_q1(O.project_q(x, w), Hq, d, bq)
    np.testing.assert_array_equal(q1.cpu().numpy(), codes)  # codes do not depend on the scale's format
    np.testing.assert_array_equal(sq.cpu().numpy(), sc.astype(np.float16).astype(np.float32))
