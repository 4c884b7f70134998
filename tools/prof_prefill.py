"""Per-phase cycle breakdown of the prefill kernel (library built with -DTURBO_PROFILE)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2412_08585_b200 import binding as ta  # noqa: E402
from paper_2412_08585_b200 import synth  # noqa: E402

B, N, Hq, Hkv, d = 8, 4096, 32, 8, 128
p = ta.params(head_dim=d)
q, k, v = synth.qkv_torch(1002, B, N, Hq, Hkv, d)
cache = ta.KVCache(B, Hkv, d, max_blocks=N // 64 + 2, bits=synth.head_bits_alternating(Hkv))
k1, v1t, k1s, v1s = ta.turbo_quantize_kv(p, cache, k, v)
o, lse = ta.turbo_attention_prefill(p, q, k1, v1t, k1s, v1s)
torch.cuda.synchronize()
buf = (C.c_ulonglong * 32)()
ta.lib().turbo_debug_prof(buf, 1)
ta.turbo_attention_prefill(p, q, k1, v1t, k1s, v1s, o=o, lse=lse)
torch.cuda.synchronize()
ta.lib().turbo_debug_prof(buf, 1)
tiles, ctas = buf[20], buf[21]
NSW = int(os.environ.get("NSW", "8"))  # softmax warps per CTA (16 with SP = 2)
names = {0: "sm wait S", 1: "sm pass1 x/max", 2: "sm pass2 SAS", 3: "sm wait PV", 4: "sm O update",
         5: "sm wait pmax", 6: "sm quant+P", 7: "sm prologue (per CTA)", 8: "sm epilogue (per CTA)", 10: "mma wait KV", 11: "mma wait S free", 12: "mma wait P",
         13: "mma wait PV free", 16: "tma wait KV empty"}
print(f"CTAs {ctas} KV tiles {tiles}  CTA lifetime {buf[22] / ctas:.0f} cycles = {buf[22] / tiles:.0f} per tile")
for i, n in names.items():
    if i in (7, 8):
        print(f"{n:24s} {buf[i] / (NSW * ctas):10.1f} cycles per (warp, CTA)")
        continue
    per = buf[i] / (NSW * tiles if i < 10 else (2 * tiles if i in (11, 12, 13) else tiles))
    print(f"{n:24s} {per:10.1f} cycles per (warp, tile)")
