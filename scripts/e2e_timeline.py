"""Timeline of bench.py's e2e leg (HostPipeline, Llama 32K): per-chunk H2D,
compute and D2H start/end on the device clock.  GPU only."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2502_18137_b200 import inputs, sparge
cfg = bench.workload_cfg(sys.argv[1] if len(sys.argv) > 1 else "llama31_8b_32k")
q, k, v = bench.gen_inputs(cfg, 1000)
qh, kh, vh = (inputs.to_device(a).cpu().pin_memory() for a in (q, k, v))
oh = torch.empty_like(qh).pin_memory()
Hq, Hkv, N, d = cfg["Hq"], cfg["Hkv"], cfg["N"], cfg["d"]
chunks = int(sys.argv[2]) if len(sys.argv) > 2 else max(c for c in (1, 2, 3, 4, 6, 8) if Hkv % c == 0)
pipe = sparge.HostPipeline(1, Hq, Hkv, N, d, causal=cfg["causal"], dtype=qh.dtype, chunks=chunks)
tl = []
orig = torch.cuda.Event
def ev_factory(*a, **kw):
    e = orig(enable_timing=True); tl.append(e); return e
def run():
    pipe(qh, kh, vh, oh, cfg["tau"], cfg["theta"], cfg["lam"])
run(); run(); torch.cuda.synchronize()
a, b = orig(enable_timing=True), orig(enable_timing=True)
ms = []
for _ in range(5):
    a.record(); run(); b.record(); torch.cuda.synchronize(); ms.append(a.elapsed_time(b))
print(f"chunks {chunks}: e2e ms {min(ms):.3f} (all {[round(x, 3) for x in ms]})")
# instrumented run: events at every stage boundary
torch.cuda.Event = ev_factory
t0 = orig(enable_timing=True); t0.record()
run(); torch.cuda.synchronize()
torch.cuda.Event = orig
# pipeline records ev_in (after H2D) and ev_out (after compute) per chunk
for c, pl in enumerate(pipe.plan):
    print(f"chunk {c} q-heads {pl[0]}-{pl[1] - 1}{' +K/V' if pl[4] else ''}: H2D done {t0.elapsed_time(tl[2 * c]):7.3f}  "
          f"compute done {t0.elapsed_time(tl[2 * c + 1]):7.3f}")
