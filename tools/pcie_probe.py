"""H2D / D2H / concurrent copy bandwidth from pinned host memory (e2e diagnostics)."""
import torch
n = 400 << 20
h = torch.empty(n, dtype=torch.uint8).pin_memory()
h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
def both():
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)
for _ in range(2):
    th = t(lambda: d.copy_(h, non_blocking=True))
    td = t(lambda: h2.copy_(d2, non_blocking=True))
    tb = t(both)
    print(f"H2D {n / th / 1e6:.1f} GB/s  D2H {n / td / 1e6:.1f} GB/s  both {2 * n / tb / 1e6:.1f} GB/s total")
