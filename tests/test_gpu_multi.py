"""Multi-GPU parity (-m gpu, skipped below 2 visible GPUs): two NCCL ranks run the
head-sharded prefill, the batch-sharded decode and the sequence-sharded decode (global
universal scale, all_gather_into_tensor of the partials, LSE combine) and compare them with
one device's run of the same inputs: bit-identical for the head / batch partitions (independent
units), the oracle's split semantics for the sequence partition."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

WORLD = 2


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    torch.distributed.init_process_group("nccl", rank=rank, world_size=WORLD,
                                         device_id=torch.device("cuda", rank))
    from paper_2412_08585_b200 import binding as ta
    from paper_2412_08585_b200 import parallel, synth

    B, N, Hq, Hkv, d = 2, 64 * 9 + 21, 8, 4, 128
    bits = synth.head_bits_alternating(Hkv)
    q, k, v = (torch.from_numpy(x).cuda() for x in synth.qkv(6100, B, N, Hq, Hkv, d))
    p = ta.params(head_dim=d)
    o, lse = parallel.prefill_head_sharded(p, q, k, v, bits=bits)
    res = {"prefill_o": o.cpu().numpy(), "prefill_lse": lse.cpu().numpy()}
    # batch-sharded decode: each rank builds the caches of its batch range
    b0, b1 = parallel.batch_shard(B, WORLD, rank)
    cache = ta.KVCache(b1 - b0, Hkv, d, max_blocks=N // 64 + 2, bits=bits)
    ta.turbo_quantize_kv(p, cache, k[b0:b1].contiguous(), v[b0:b1].contiguous())
    qd = torch.from_numpy(synth.decode_token(6101, B, Hq, Hkv, d)[0]).cuda()
    od, lsed = parallel.decode_batch_sharded(
        lambda ql: (lambda r: (r[0], r[2]))(ta.turbo_attention_decode(p, cache, ql, n_splits=2)), qd)
    res.update(decode_o=od.cpu().numpy(), decode_lse=lsed.cpu().numpy())
    # sequence-sharded long-context decode
    t0, t1 = parallel.seq_shard_tokens(N, WORLD, rank)
    sc = ta.KVCache(B, Hkv, d, max_blocks=N // 64 + 2, bits=bits)
    parallel.prefill_seq_sharded(p, sc, k[:, t0:t1].contiguous(), v[:, t0:t1].contiguous())
    os_, ls_ = parallel.decode_seq_sharded(p, sc, qd, n_splits_local=1)
    res.update(seq_o=os_.cpu().numpy(), seq_lse=ls_.cpu().numpy())
    if rank == 0:
        np.savez(out, **res)
    torch.distributed.barrier()
    torch.distributed.destroy_process_group()


def test_two_rank_partitions_match_one_device(tmp_path):
    if torch.cuda.device_count() < WORLD:
        pytest.skip(f"needs {WORLD} GPUs")
    from paper_2412_08585_b200 import binding as ta
    from paper_2412_08585_b200 import synth

    out = str(tmp_path / "multi.npz")
    ctx = mp.get_context("spawn")
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, port, out)) for r in range(WORLD)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(timeout=300)
        assert pr.exitcode == 0
    res = np.load(out)
    B, N, Hq, Hkv, d = 2, 64 * 9 + 21, 8, 4, 128
    bits = synth.head_bits_alternating(Hkv)
    q, k, v = (torch.from_numpy(x).cuda() for x in synth.qkv(6100, B, N, Hq, Hkv, d))
    p = ta.params(head_dim=d)
    cache = ta.KVCache(B, Hkv, d, max_blocks=N // 64 + 2, bits=bits)
    k1, v1t, k1s, v1s = ta.turbo_quantize_kv(p, cache, k, v)
    o, lse = ta.turbo_attention_prefill(p, q, k1, v1t, k1s, v1s)
    np.testing.assert_array_equal(res["prefill_o"], o.cpu().numpy())
    np.testing.assert_array_equal(res["prefill_lse"], lse.cpu().numpy())
    qd = torch.from_numpy(synth.decode_token(6101, B, Hq, Hkv, d)[0]).cuda()
    od, _, lsed = ta.turbo_attention_decode(p, cache, qd, n_splits=2)
    np.testing.assert_array_equal(res["decode_o"], od.cpu().numpy())
    np.testing.assert_array_equal(res["decode_lse"], lsed.cpu().numpy())
    # the sequence partition = split decode over the rank ranges (blocks [0, nb0), [nb0, nb) + buffer)
    from paper_2412_08585_b200 import parallel

    nb0 = parallel.seq_shard_tokens(N, WORLD, 0)[1] // 64
    parts = [ta.turbo_attention_decode(p, cache, qd, blk_begin=a, blk_end=e, with_buffer=wb, n_splits=1,
                                       want_fp16=False, want_f32=True) for a, e, wb in
             ((0, nb0, False), (nb0, -1, True))]
    ref_o, _, ref_l = ta.turbo_combine_lse(torch.stack([x[1].reshape(B * Hq, d) for x in parts]),
                                           torch.stack([x[2].reshape(B * Hq) for x in parts]))
    np.testing.assert_array_equal(res["seq_o"].reshape(B * Hq, d), ref_o.cpu().numpy())
    np.testing.assert_array_equal(res["seq_lse"].reshape(B * Hq), ref_l.cpu().numpy())
