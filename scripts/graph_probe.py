"""Step time eager vs CUDA-graph replay (GPU only): how much of a step is
host enqueue latency?  usage: python scripts/graph_probe.py [workload]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
w = sys.argv[1] if len(sys.argv) > 1 else "flux"
cfg = bench.hyper(bench.workload_cfg(w), w, "tuned")
dev = torch.device("cuda", 0)
prob = bench.Problem(cfg, 1, 0, dev, "heads", pin=False)
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
prob.step(); torch.cuda.synchronize()
o_eager = prob.o.clone()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    for _ in range(2):
        prob.step()
torch.cuda.current_stream().wait_stream(s)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    prob.step()
torch.cuda.synchronize()
prob.o.zero_(); g.replay(); torch.cuda.synchronize()
same = torch.equal(prob.o, o_eager)
def timed(fn, n=30):
    ts = []
    for _ in range(n):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record()
        torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    return np.median(ts) * 1e3
t0 = time.perf_counter()
for _ in range(50): prob.step()
torch.cuda.synchronize()
host = (time.perf_counter() - t0) / 50 * 1e6
t1 = time.perf_counter()
for _ in range(20): prob.step(); torch.cuda.synchronize()
print(w, "step us: eager", round(timed(prob.step), 1), "| graph replay", round(timed(g.replay), 1),
      "| O equal", same, "| eager back-to-back wall per step", round(host, 1))
