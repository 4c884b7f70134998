"""Sweep the split count of configs[2] / configs[4] decode (kernel time, GB/s)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2412_08585_b200 import binding as ta  # noqa: E402
from paper_2412_08585_b200 import synth  # noqa: E402
import bench  # noqa: E402

SPL3 = tuple(int(x) for x in os.environ.get("SPL3", "0,8,12").split(","))
SPL5 = tuple(int(x) for x in os.environ.get("SPL5", "0,32").split(","))
SHAPES = [("cfg3", (64, 32768, 40, 10, 128), SPL3), ("cfg5", (16, 131072, 32, 8, 128), SPL5)]
if os.environ.get("DEC_SHAPES"):  # "B,N,Hq,Hkv,d;..." with split list SPLX (e.g. the G = 8 shapes)
    SPLX = tuple(int(x) for x in os.environ.get("SPLX", "0").split(","))
    SHAPES = [("G%d" % (int(t.split(",")[2]) // int(t.split(",")[3])), tuple(int(x) for x in t.split(",")), SPLX)
              for t in os.environ["DEC_SHAPES"].split(";")]
BC = int(os.environ.get("TP_BC", "64"))  # block_kv
for name, (B, N, Hq, Hkv, d), splits in SHAPES:
    bits = synth.head_bits_alternating(Hkv)
    p = ta.params(head_dim=d, block_kv=BC)
    cache = ta.KVCache(B, Hkv, d, max_blocks=N // BC + 4, bits=bits, block_kv=BC)
    _, k, v = synth.qkv_torch(3003, B, N, Hkv, Hkv, d)
    ta.turbo_quantize_kv(p, cache, k, v)
    del k, v
    torch.cuda.empty_cache()
    qd = synth.qkv_torch(7, B, 1, Hq, Hkv, d)[0][:, 0].contiguous()
    byt = bench.decode_bytes(B, Hkv, d, N // BC, 0, bits, Hq, BC)
    for S in splits:
        ws = torch.empty(max(ta.turbo_decode_workspace_bytes(B, Hq, Hkv, d, S), 16), dtype=torch.uint8, device="cuda")
        for _ in range(3):
            ta.turbo_attention_decode(p, cache, qd, n_splits=S, workspace=ws)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            ta.turbo_attention_decode(p, cache, qd, n_splits=S, workspace=ws)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 20
        print(f"{name} BC={BC} B={B} N={N} S={S:3d} {ms * 1e3:8.1f} us  {byt / ms / 1e6:8.1f} GB/s", flush=True)
    del cache
    torch.cuda.empty_cache()
