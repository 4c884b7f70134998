"""Multi-GPU partitioning of the TurboAttention hot path.

* Prefill and moderate-context decode: independent (batch, KV head) units,
  split across ranks with no collective (`head_shard`, `batch_shard`).
* Long-context decode: the compressed cache of every (batch, KV head) is
  sharded by contiguous whole-block ranges of the sequence (`seq_shard_tokens`);
  the last rank owns the tail and the INT8 decode buffer.  Each rank runs
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
