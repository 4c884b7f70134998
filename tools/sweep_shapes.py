"""Throughput across shapes beyond the BASELINE configs (profiles/r1_shape_sweep.txt):
prefill TOPS vs sequence length (causal / non-causal, GQA 32/8 and 64/8, d = 64 / 128) and
decode KV GB/s vs context length, batch and GQA group (packed G <= 4 and general G = 8 IMMA
paths).  Kernel-only CUDA-event timings, inputs resident, auto split counts."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2412_08585_b200 import binding as ta  # noqa: E402
from paper_2412_08585_b200 import synth  # noqa: E402


def timeit(fn, iters):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


print("# prefill: B, N, Hq, Hkv, d, causal -> us, TOPS (4 d x unmasked pairs)")
for B, N, Hq, Hkv, d, causal in ((32, 1024, 32, 8, 128, True), (16, 2048, 32, 8, 128, True),
                                 (8, 4096, 32, 8, 128, True), (4, 8192, 32, 8, 128, True),
                                 (2, 16384, 32, 8, 128, True), (8, 4096, 32, 8, 128, False),
                                 (8, 4096, 64, 8, 128, True), (8, 4096, 32, 32, 128, True),
                                 (8, 4096, 32, 8, 64, True)):
    p = ta.params(head_dim=d)
    q, k, v = synth.qkv_torch(11, B, N, Hq, Hkv, d)
    cache = ta.KVCache(B, Hkv, d, max_blocks=N // 64 + 2, bits=synth.head_bits_alternating(Hkv))
    ops_ = ta.turbo_quantize_kv(p, cache, k, v)
    o = torch.empty_like(q)
    lse = torch.empty((B, Hq, N), dtype=torch.float32, device="cuda")
    ms = timeit(lambda: ta.turbo_attention_prefill(p, q, *ops_, causal=causal, o=o, lse=lse), 5)
    ops = bench.prefill_ops(B, N, Hq, d, causal)
    print(f"prefill B={B:3d} N={N:6d} Hq={Hq} Hkv={Hkv} d={d:3d} causal={int(causal)}  {ms * 1e3:9.1f} us  "
          f"{ops / ms / 1e9:7.1f} TOPS", flush=True)
    del q, k, v, cache, ops_, o, lse
    torch.cuda.empty_cache()

print("# decode: B, context, Hq, Hkv -> splits, us, KV GB/s (algorithmic bytes), tokens/s per layer")
for B, N, Hq, Hkv in ((64, 4096, 40, 10), (64, 16384, 40, 10), (64, 32768, 40, 10), (16, 65536, 32, 8),
                      (16, 131072, 32, 8), (8, 32768, 64, 8), (16, 32768, 64, 8), (128, 8192, 32, 8),
                      (1, 131072, 32, 8), (1, 131072, 64, 8)):
    d = 128
    bits = synth.head_bits_alternating(Hkv)
    p = ta.params(head_dim=d)
    cache = ta.KVCache(B, Hkv, d, max_blocks=N // 64 + 2, bits=bits)
    _, k, v = synth.qkv_torch(3, B, N, Hkv, Hkv, d)
    ta.turbo_quantize_kv(p, cache, k, v)
    del k, v
    torch.cuda.empty_cache()
    qd = synth.qkv_torch(7, B, 1, Hq, Hkv, d)[0][:, 0].contiguous()
    S = ta.resolve_splits(None, B, Hq, cache)  # the binding's deterministic default (balanced for G > 4)
    ws = torch.empty(max(ta.turbo_decode_workspace_bytes(B, Hq, Hkv, d, S), 16), dtype=torch.uint8, device="cuda")
    o = torch.empty_like(qd)
    lse = torch.empty((B, Hq), dtype=torch.float32, device="cuda")
    ms = timeit(lambda: ta.turbo_attention_decode(p, cache, qd, n_splits=S, workspace=ws, o=o, lse=lse), 20)
    byt = bench.decode_bytes(B, Hkv, d, N // 64, 0, bits, Hq)
    print(f"decode B={B:3d} ctx={N:7d} Hq={Hq} Hkv={Hkv} (G={Hq // Hkv}) S={S:5d}  {ms * 1e3:8.1f} us  "
          f"{byt / ms / 1e6:7.1f} GB/s  {B / ms * 1e3:9.0f} tok/s", flush=True)
    del cache, qd, ws
    torch.cuda.empty_cache()
