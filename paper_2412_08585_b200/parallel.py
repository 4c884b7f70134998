"""Multi-GPU partitioning of the TurboAttention hot path.

* Prefill and moderate-context decode: independent (batch, KV head) units,
  split across ranks with no collective (`head_shard`, `batch_shard`).
* Long-context decode: the compressed cache of every (batch, KV head) is
  sharded by contiguous whole-block ranges of the sequence (`seq_shard_tokens`);
  the last rank owns the tail and the INT8 decode buffer, quantised with the
  GLOBAL universal scale (one all-reduce(MAX) at cache construction,
  `prefill_seq_sharded`).  Each rank runs
  Alg. 2 over its shard (`turbo_attention_decode`, FP32 normalised partial O
  and L) and the partials are merged by ONE all-gather plus the log-sum-exp
  combine in rank order (`turbo_combine_lse`) -- the only collective of the
  path (R-23).

Communication uses torch.distributed (NCCL on GPUs; gloo in the CPU tests).
"""
from __future__ import annotations

import torch
import torch.distributed as dist

BC = 64


def contiguous_range(n: int, world: int, rank: int):
    """[begin, end) of rank's contiguous share of n units (first n % world ranks get one more)."""
    base, rem = divmod(n, world)
    begin = rank * base + min(rank, rem)
    return begin, begin + base + (1 if rank < rem else 0)


def head_shard(n_q_heads: int, n_kv_heads: int, world: int, rank: int):
    """KV heads [k0, k1) and their query heads [h0, h1) on `rank` (GQA groups stay whole)."""
    if n_kv_heads % world:
        raise ValueError("n_kv_heads must be divisible by the world size")
    g = n_q_heads // n_kv_heads
    k0, k1 = contiguous_range(n_kv_heads, world, rank)
    return (k0, k1), (k0 * g, k1 * g)


def batch_shard(batch: int, world: int, rank: int):
    return contiguous_range(batch, world, rank)


def seq_shard_tokens(n_tokens: int, world: int, rank: int, block: int = BC):
    """Token range [t0, t1) of rank's sequence shard: whole B_c blocks split
    contiguously, the N mod B_c tail (decode buffer) on the last rank."""
    n_full = n_tokens // block
    b0, b1 = contiguous_range(n_full, world, rank)
    t0, t1 = b0 * block, b1 * block
    if rank == world - 1:
        t1 = n_tokens
    return t0, t1


def gather_along(x: torch.Tensor, dim: int, group=None):
    """All-gather every rank's shard of x along `dim` (shards may differ in size by the
    contiguous_range rule: padded to the largest, trimmed after) and concatenate them in rank
    order.  NCCL uses all_gather_into_tensor; gloo (CPU tests) the list form."""
    world = dist.get_world_size(group)
    n = torch.tensor([x.shape[dim]], dtype=torch.int64, device=x.device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    sizes = [int(t.item()) for t in sizes]
    xm = x.movedim(dim, 0).contiguous()
    if xm.shape[0] < max(sizes):
        pad = torch.zeros((max(sizes) - xm.shape[0],) + tuple(xm.shape[1:]), dtype=x.dtype, device=x.device)
        xm = torch.cat([xm, pad]).contiguous()
    out = torch.empty((world,) + tuple(xm.shape), dtype=x.dtype, device=x.device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, xm, group=group)
    else:
        dist.all_gather(list(out.unbind(0)), xm, group=group)
    return torch.cat([out[r, :sizes[r]] for r in range(world)]).movedim(0, dim).contiguous()


def prefill_head_sharded(p, q, k, v, group=None, causal=True, run=None, gather=True, bits=None):
    """Prefill partitioned by KV head (configs[3]): this rank takes the KV heads
    head_shard() gives it with their GQA query heads, runs the whole hot path on them
    (turbo_quantize_kv + turbo_attention_prefill with the layer's bit plan `bits` [Hkv][2], or
    `run(p, q, k, v, causal)` -> (o, lse)),
    with no data-path collective; `gather` all-gathers O [B, N, Hq, d] and LSE [B, Hq, N] in
    head order (for checking / a following projection).  Heads are independent, so the result
    is bit-identical to one device's (tests/test_parallel_gloo.py, tests/test_gpu_multi.py)."""
    from . import binding as ta

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    Hq, Hkv = q.shape[2], k.shape[2]
    (k0, k1), (h0, h1) = head_shard(Hq, Hkv, world, rank)
    ql, kl, vl = q[:, :, h0:h1].contiguous(), k[:, :, k0:k1].contiguous(), v[:, :, k0:k1].contiguous()
    if run is None:
        B, N, _, d = q.shape
        hb = [[4, 2]] * Hkv if bits is None else [list(map(int, r)) for r in bits]  # [Hkv][K, V] plan
        cache = ta.KVCache(B, k1 - k0, d, max_blocks=N // BC + 1, bits=hb[k0:k1], device=q.device)
        k1_, v1t, k1s, v1s = ta.turbo_quantize_kv(p, cache, kl, vl)
        o, lse = ta.turbo_attention_prefill(p, ql, k1_, v1t, k1s, v1s, causal=causal)
    else:
        o, lse = run(p, ql, kl, vl, causal)
    if not gather:
        return o, lse
    return gather_along(o, 2, group), gather_along(lse, 1, group)


def decode_batch_sharded(decode_local, q, group=None, gather=True):
    """Moderate-context decode partitioned by batch (configs[2]): this rank holds the caches of
    its contiguous batch range batch_shard(); `decode_local(q_local)` -> (o [b, Hq, d], lse [b, Hq])
    runs Alg. 2 on them (turbo_attention_decode); no data-path collective.  `gather` returns the
    full batch in order."""
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    b0, b1 = batch_shard(q.shape[0], world, rank)
    o, lse = decode_local(q[b0:b1].contiguous())
    if not gather:
        return o, lse
    return gather_along(o, 0, group), gather_along(lse, 0, group)


def prefill_shard_blocks(p, cache, k, v):
    """Step 1 of the sequence-sharded cache construction: this rank's whole B_c blocks (stage 1 +
    stage 2 are per block, R-21).  Returns the rank's universal-scale candidates a_univ
    [B, Hkv, 2] (max |x| over its full-block tokens, R-9)."""
    from . import binding as ta

    n = k.shape[1] // BC * BC
    if n:
        ta.turbo_quantize_kv(p, cache, k[:, :n].contiguous(), v[:, :n].contiguous())
    return cache.a_univ[: cache.batch * cache.n_kv_heads * 2].view(cache.batch, cache.n_kv_heads, 2).clone()


def prefill_shard_tail(p, cache, k, v, a_global):
    """Step 2: every rank stores the global universal scale (R-9: max over ALL prefill tokens);
    the last rank then quantises its N mod B_c tail into the INT8 buffer with
    turbo_quantize_kv mode 2 (a_univ = max(a_global, tail max)), exactly as one device would."""
    from . import binding as ta

    cache.a_univ[: a_global.numel()].copy_(a_global.reshape(-1))
    n = k.shape[1] // BC * BC
    if k.shape[1] > n:
        B, _, H, d = k.shape
        nk = n + (k.shape[1] - n)
        tc = -(-nk // BC)
        out = (torch.empty((B, H, nk, d), dtype=torch.float16, device=k.device),
               torch.empty((B, H, tc, d, BC), dtype=torch.float16, device=k.device),
               torch.empty((B, H, tc), dtype=torch.float32, device=k.device),
               torch.empty((B, H, tc), dtype=torch.float32, device=k.device))  # prefill operands: unused
        ta.turbo_quantize_kv(p, cache, k[:, n:].contiguous(), v[:, n:].contiguous(), mode=2, out=out)


def prefill_seq_sharded(p, cache, k, v, group=None):
    """Sequence-sharded cache construction for long-context decode (configs[4]): k, v fp16
    [B, n, Hkv, d] is this rank's token shard (seq_shard_tokens: whole blocks, the tail on the
    last rank).  One all-reduce(MAX) of the per-rank a_univ makes the universal scale global, so
    the buffer, later appends and flushes match the single-device cache."""
    a = prefill_shard_blocks(p, cache, k, v)
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(a, op=dist.ReduceOp.MAX, group=group)
    prefill_shard_tail(p, cache, k, v, a)


def gather_partials(o_part: torch.Tensor, lse: torch.Tensor, group=None):
    """All-gather every rank's (O_part [rows, d] f32, L [rows] f32) into
    ([world, rows, d], [world, rows]) in rank order."""
    world = dist.get_world_size(group)
    rows, d = o_part.shape
    packed = torch.cat([o_part.reshape(rows, d), lse.reshape(rows, 1)], dim=1).contiguous()
    out = torch.empty((world, rows, d + 1), dtype=packed.dtype, device=packed.device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, packed, group=group)
    else:
        dist.all_gather(list(out.unbind(0)), packed, group=group)
    return out[:, :, :d].contiguous(), out[:, :, d].contiguous()


def decode_seq_sharded(p, cache, q, group=None, n_splits_local: int = 4, local_decode=None, combine=None):
    """Alg. 2 over a sequence-sharded cache: local split-KV decode on this
    rank's blocks (buffer on the last rank), one all-gather, LSE combine.
    Returns (O fp16 [B, Hq, d], L f32 [B, Hq]) on every rank."""
    from . import binding as ta

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    last = rank == world - 1
    B, Hq, d = q.shape
    if local_decode is None:
        _, o_part, lse = ta.turbo_attention_decode(p, cache, q, with_buffer=last, n_splits=n_splits_local,
                                                   want_fp16=False, want_f32=True)
    else:
        o_part, lse = local_decode(p, cache, q, last)
    parts, lses = gather_partials(o_part.reshape(B * Hq, d), lse.reshape(B * Hq), group)
    if combine is None:
        o, _, L = ta.turbo_combine_lse(parts, lses)
    else:
        o, L = combine(parts, lses)
    return o.reshape(B, Hq, d), L.reshape(B, Hq)
