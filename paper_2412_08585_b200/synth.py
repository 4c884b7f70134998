"""Seeded synthetic attention inputs (DESIGN.md §4 "input recipe").

This module holds none of the method's arithmetic: it only draws Q/K/V with
the shapes and value structure of the paper's workloads, and is the single
input source shared by the CUDA path's tests/bench and the oracle.

Structure ("certain heads in query and key have a number of
large-magnitude channels"; PAPER.md:1060 value-channel outliers in Phi-3):
  * Q, K ~ N(0, 1); in every 4th KV head the K channels OUTLIER_K are scaled
    x8 and the matching Q channels (of the query heads in that group) x2.
  * V ~ 0.25 N(0, 1); in every 5th KV head the channels OUTLIER_V are scaled
    x4; V is clipped to +-3.9 so |O| < 4 (FP16 output ulp).
All values are rounded to FP16 (the paper's activation format).
"""
from __future__ import annotations

import numpy as np

OUTLIER_K = {128: (3, 17, 64, 100), 64: (3, 17, 40)}
OUTLIER_V = (5, 77)
V_CLIP = 3.9


def _outlier_k(d):
    return OUTLIER_K.get(d, tuple(c for c in (3, 17) if c < d))


def _structure_np(q, k, v, n_kv_heads):
    """In-place structure on [.., H, d] arrays (last two axes head, channel)."""
    d = k.shape[-1]
    hq = q.shape[-2]
    g = hq // n_kv_heads
    ok = list(_outlier_k(d))
    ov = [c for c in OUTLIER_V if c < d]
    for h in range(n_kv_heads):
        if h % 4 == 0:
            k[..., h, ok] *= 8.0
            q[..., h * g:(h + 1) * g, ok] *= 2.0
        if h % 5 == 0:
            v[..., h, ov] *= 4.0
    np.clip(v, -V_CLIP, V_CLIP, out=v)


def qkv(seed: int, B: int, N: int, Hq: int, Hkv: int, d: int):
    """Prefill inputs: Q [B,N,Hq,d], K/V [B,N,Hkv,d] float16 numpy arrays."""
    rng = np.random.default_rng(seed)
    q = rng.standard_normal((B, N, Hq, d), dtype=np.float32)
    k = rng.standard_normal((B, N, Hkv, d), dtype=np.float32)
    v = 0.25 * rng.standard_normal((B, N, Hkv, d), dtype=np.float32)
    _structure_np(q, k, v, Hkv)
    return q.astype(np.float16), k.astype(np.float16), v.astype(np.float16)


def decode_token(seed: int, B: int, Hq: int, Hkv: int, d: int):
    """One decode step: q [B,Hq,d], k/v [B,Hkv,d] float16 numpy arrays."""
    q, k, v = qkv(seed, B, 1, Hq, Hkv, d)
    return q[:, 0], k[:, 0], v[:, 0]


def qkv_torch(seed: int, B: int, N: int, Hq: int, Hkv: int, d: int, device="cuda"):
    """Same recipe drawn directly on the device (bench-size inputs).  Returns
    fp16 torch tensors; a different RNG stream than ``qkv`` (the oracle only
    ever sees the tensors actually produced here, copied back to the host)."""
    import torch

    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    q = torch.randn((B, N, Hq, d), generator=gen, device=device, dtype=torch.float32)
    k = torch.randn((B, N, Hkv, d), generator=gen, device=device, dtype=torch.float32)
    v = 0.25 * torch.randn((B, N, Hkv, d), generator=gen, device=device, dtype=torch.float32)
    g = Hq // Hkv
    ok = list(_outlier_k(d))
    ov = [c for c in OUTLIER_V if c < d]
    for h in range(Hkv):
        if h % 4 == 0:
            k[..., h, ok] *= 8.0
            q[..., h * g:(h + 1) * g, ok] *= 2.0
        if h % 5 == 0:
            v[..., h, ov] *= 4.0
    v.clamp_(-V_CLIP, V_CLIP)
    return q.half(), k.half(), v.half()


def head_bits_alternating(n_kv_heads: int):
    """A fixed headwise plan with half of the 2*Hkv (K,V) slots at 2 bits
    ("half of the heads' KV cache to 2-bit"): slot (h, V) gets 2
    bits for even h, slot (h, K) for odd h.  Returned as [Hkv][2] int32."""
    bits = np.full((n_kv_heads, 2), 4, np.int32)
    for h in range(n_kv_heads):
        bits[h, 1 if h % 2 == 0 else 0] = 2
    return bits
