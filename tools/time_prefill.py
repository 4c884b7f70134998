"""Time turbo_attention_prefill on configs[1] (B=8, N=4096, 32/8 heads, d=128,
causal) for the library in $TURBO_LIB (A/B of kernel variants)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2412_08585_b200 import binding as ta  # noqa: E402
from paper_2412_08585_b200 import synth  # noqa: E402

B, N, Hq, Hkv, d = (1, 32768, 64, 8, 128) if os.environ.get("TP_CFG") == "70b" else (8, 4096, 32, 8, 128)
if os.environ.get("TP_SHAPE"):  # "B,N,Hq,Hkv,d" (e.g. MHA: 8,4096,32,32,128)
    B, N, Hq, Hkv, d = (int(x) for x in os.environ["TP_SHAPE"].split(","))
p = ta.params(head_dim=d, p_scale_rows=int(os.environ.get("TP_PROW", "0")),
              alpha_mode=int(os.environ.get("TP_ALPHA", "0")), block_q=int(os.environ.get("TP_BQ", "64")),
              block_kv=int(os.environ.get("TP_BC", "64")), sas_fp16=int(os.environ.get("TP_SF16", "0")))
q, k, v = synth.qkv_torch(1002, B, N, Hq, Hkv, d)
cache = ta.KVCache(B, Hkv, d, max_blocks=N // p.block_kv + 2, bits=synth.head_bits_alternating(Hkv),
                   block_kv=p.block_kv)
k1, v1t, k1s, v1s = ta.turbo_quantize_kv(p, cache, k, v)
o, lse = ta.turbo_attention_prefill(p, q, k1, v1t, k1s, v1s)
for _ in range(3):
    ta.turbo_attention_prefill(p, q, k1, v1t, k1s, v1s, o=o, lse=lse)
ITERS = 5 if os.environ.get("TP_CFG") == "70b" else 20
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(ITERS):
    ta.turbo_attention_prefill(p, q, k1, v1t, k1s, v1s, o=o, lse=lse)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / ITERS
ops = 4.0 * d * N * (N + 1) / 2 * B * Hq
print(f"{os.environ.get('TURBO_LIB', 'in-tree')} sf16={p.sas_fp16} bc={p.block_kv} {B},{N},{Hq},{Hkv},{d}: {ms * 1e3:8.1f} us  {ops / ms / 1e9:7.1f} TOPS  "
      f"checksum {o.float().abs().sum().item():.6e}")
