"""Pinned host <-> device copy bandwidth alone and concurrent (the e2e
bound of bench.py's HostPipeline leg).  GPU only."""
import torch
n = 402653184 // 2
h = torch.empty(n, dtype=torch.bfloat16).pin_memory()
ho = torch.empty(268435456 // 2, dtype=torch.bfloat16).pin_memory()
d = torch.empty(n, dtype=torch.bfloat16, device="cuda")
do = torch.empty(268435456 // 2, dtype=torch.bfloat16, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ms = []
    for _ in range(reps):
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ms.append(a.elapsed_time(b))
    return min(ms)
h2d = t(lambda: d.copy_(h, non_blocking=True))
d2h = t(lambda: ho.copy_(do, non_blocking=True))
def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur); s2.wait_stream(cur)
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): ho.copy_(do, non_blocking=True)
    cur.wait_stream(s1); cur.wait_stream(s2)
bo = t(both)
print(f"H2D 402 MB: {h2d:.2f} ms ({402.65/h2d:.1f} GB/s); D2H 268 MB: {d2h:.2f} ms ({268.4/d2h:.1f} GB/s); "
      f"concurrent: {bo:.2f} ms")
