"""Attention-kernel time under three L2 states (GPU only): back-to-back
calls (operands L2-resident), right after the 512 MB L2 flush, and inside
the full step after the flush (as bench.py times it).
usage: python scripts/attn_l2_probe.py [workload]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2502_18137_b200 import sparge
w = sys.argv[1] if len(sys.argv) > 1 else "flux"
cfg = bench.hyper(bench.workload_cfg(w), w, "tuned")
dev = torch.device("cuda", 0)
prob = bench.Problem(cfg, 1, 0, dev, "heads", pin=False)
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
bf, sh = prob.bf, prob.shape
def attn():
    sparge.sparge_attn_fwd_ex(sh, bf.qq, bf.dq, bf.kq, bf.dk, prob.v, bf.lut, bf.cnt, cfg["lam"],
                              prob.perm, prob.o, None, bf.workspace, sparge.SPARGE_ATTN_SKIP_VPREP)
def timed(pre, fn, n=20):
    ts = []
    for _ in range(n):
        pre()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record()
        torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    return np.median(ts) * 1e3
prob.step(); torch.cuda.synchronize()
print(w, "attention (+k_order) us: back-to-back", round(timed(lambda: None, attn), 1),
      "| after flush", round(timed(flush.zero_, attn), 1),
      "| after flush + quant/predict/V", round(timed(lambda: (flush.zero_(), prob.step()), attn), 1),
      "| flush then a 2nd flush", round(timed(lambda: (flush.zero_(), flush.zero_()), attn), 1))
print(w, "whole step us: after flush", round(timed(flush.zero_, prob.step), 1),
      "| back-to-back", round(timed(lambda: None, prob.step), 1))
