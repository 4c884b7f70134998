"""Run configs[2] decode (Phi-3-medium shape, B=64, 32k context, mixed bits) a few
times -- a short driver for ncu captures of decode_kernel."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2412_08585_b200 import binding as ta  # noqa: E402
from paper_2412_08585_b200 import synth  # noqa: E402

B, N, Hq, Hkv, d = 64, 32768, 40, 10, 128
if os.environ.get("DEC_SHAPE"):  # "B,N,Hq,Hkv,d" (e.g. the G = 8 shape 16,32768,64,8,128)
    B, N, Hq, Hkv, d = (int(x) for x in os.environ["DEC_SHAPE"].split(","))
S = int(sys.argv[1]) if len(sys.argv) > 1 else 8
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 5
p = ta.params(head_dim=d)
cache = ta.KVCache(B, Hkv, d, max_blocks=N // 64 + 4, bits=synth.head_bits_alternating(Hkv))
_, k, v = synth.qkv_torch(3003, B, N, Hkv, Hkv, d)
ta.turbo_quantize_kv(p, cache, k, v)
del k, v
qd = synth.qkv_torch(7, B, 1, Hq, Hkv, d)[0][:, 0].contiguous()
for _ in range(iters):
    ta.turbo_attention_decode(p, cache, qd, n_splits=S)
torch.cuda.synchronize()
print("ok")
