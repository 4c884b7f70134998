"""Compare auto_splits (task count nearest 4.5 waves) with an alternative rule (about 32
blocks per task, at least 2.5 waves) on a set of decode shapes (kernel time, GB/s)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2412_08585_b200 import binding as ta  # noqa: E402
from paper_2412_08585_b200 import synth  # noqa: E402


def alt_splits(bh, nb, W):
    best = None
    for s in range(1, max(1, nb // 8) + 1):
        per = -(-nb // s)
        last = nb - per * (s - 1)
        if s > 1 and (last <= 0 or 4 * last < 3 * per):
            continue
        if bh * s >= 2.5 * W and per <= 32:
            return s
        best = s
    return best


def run(B, N, Hq, Hkv, d=128):
    bits = synth.head_bits_alternating(Hkv)
    p = ta.params(head_dim=d)
    cache = ta.KVCache(B, Hkv, d, max_blocks=N // 64 + 4, bits=bits)
    _, k, v = synth.qkv_torch(3003, B, N, Hkv, Hkv, d)
    ta.turbo_quantize_kv(p, cache, k, v)
    del k, v
    torch.cuda.empty_cache()
    qd = synth.qkv_torch(7, B, 1, Hq, Hkv, d)[0][:, 0].contiguous()
    byt = bench.decode_bytes(B, Hkv, d, N // 64, 0, bits, Hq)
    W = ta.turbo_decode_workers(Hq, Hkv, d)
    s_old = ta.auto_splits(B, Hkv, N // 64, W)
    s_new = alt_splits(B * Hkv, N // 64, W)
    res = {}
    for S in sorted({s_old, s_new}):
        ws = torch.empty(max(ta.turbo_decode_workspace_bytes(B, Hq, Hkv, d, S), 16), dtype=torch.uint8, device="cuda")
        for _ in range(3):
            ta.turbo_attention_decode(p, cache, qd, n_splits=S, workspace=ws)
        ms = []
        for rep in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(20):
                ta.turbo_attention_decode(p, cache, qd, n_splits=S, workspace=ws)
            e1.record()
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1) / 20)
        res[S] = min(ms)
    print(f"B={B:3d} N={N:6d} {Hq}/{Hkv}: old S={s_old:3d} {byt / res[s_old] / 1e6:7.1f} GB/s | "
          f"new S={s_new:3d} {byt / res[s_new] / 1e6:7.1f} GB/s", flush=True)


for shp in ((64, 32768, 40, 10), (16, 131072, 32, 8), (64, 16384, 40, 10), (128, 8192, 32, 8), (64, 4096, 40, 10),
            (16, 65536, 32, 8), (4, 32768, 32, 8), (1, 131072, 32, 8), (32, 16384, 32, 8), (8, 65536, 40, 10)):
    run(*shp)
