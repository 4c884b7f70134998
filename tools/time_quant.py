"""Time turbo_quantize_kv on configs[1] (B=8, N=4096, 8 KV heads, d=128) for the
library in $TURBO_LIB (A/B of kernel variants)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2412_08585_b200 import binding as ta  # noqa: E402
from paper_2412_08585_b200 import synth  # noqa: E402

B, N, Hq, Hkv, d = 8, 4096, 32, 8, 128
BC = int(os.environ.get("TP_BC", "64"))
p = ta.params(head_dim=d, block_kv=BC)
q, k, v = synth.qkv_torch(1002, B, N, Hq, Hkv, d)
cache = ta.KVCache(B, Hkv, d, max_blocks=N // BC + 2, bits=synth.head_bits_alternating(Hkv), block_kv=BC)
outs = ta.turbo_quantize_kv(p, cache, k, v)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
rd = torch.ones(64 << 20, dtype=torch.float32, device="cuda")  # 256 MB read by the 'clean' flush
FLUSH = os.environ.get("TQ_FLUSH", "write")  # write: zero 256 MB (L2 left dirty); clean: + read 256 MB; none
ts = []
for i in range(23):
    if FLUSH != "none":
        flush.zero_()
    if FLUSH == "clean":
        rd.sum()  # evicts the dirty flush lines (written back here, outside the timed region)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(2_000_000)  # ~1 ms of GPU work: the host enqueues the timed launches before they run
    e0.record()
    ta.turbo_quantize_kv(p, cache, k, v)
    e1.record()
    torch.cuda.synchronize()
    if i >= 3:
        ts.append(e0.elapsed_time(e1))
ms = sorted(ts)[len(ts) // 2]
nbytes = 2 * k.numel() * 2 + k.numel() + 2 * v.numel() + cache.records().numel()
print(f"{os.environ.get('TURBO_LIB', 'in-tree')} flush={FLUSH}: {ms * 1e3:8.1f} us  {nbytes / ms / 1e6:7.1f} GB/s  "
      f"checksum {sum(int(x.double().abs().sum().item()) for x in outs[:2])} {int(cache.records().double().sum().item())}")
