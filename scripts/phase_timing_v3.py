"""Run the attention kernel of a bench workload with the instrumented
library (SPARGE_PHASE_TIMING) and print the per-phase cycle split of the
softmax warps.  GPU only.  usage: python scripts/phase_timing.py [workload]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("SPARGE_LIB", "libsparge_sparge_phase_timing.so")
import numpy as np, torch
import bench
from paper_2502_18137_b200 import inputs, sparge
w = sys.argv[1] if len(sys.argv) > 1 else "llama31_8b_32k"
cfg = bench.workload_cfg(w)
q, k, v = (inputs.to_device(a) for a in bench.gen_inputs(cfg, 1000))
perm_np = bench.hilbert_perm(cfg)
perm = None if perm_np is None else torch.from_numpy(perm_np).cuda()
o, bf = sparge.sparge_forward(q, k, v, cfg["tau"], cfg["theta"], cfg["lam"], causal=cfg["causal"], perm=perm)
torch.cuda.synchronize()
bf.workspace[:256].zero_()
sparge.sparge_attn_fwd_ex(bf.shape, bf.qq, bf.dq, bf.kq, bf.dk, v, bf.lut, bf.cnt, cfg["lam"], perm, o,
                          None, bf.workspace, sparge.SPARGE_ATTN_SKIP_VPREP)
torch.cuda.synchronize()
ph = bf.workspace[32:32 + 64].view(torch.int64).cpu().numpy()
tiles = ph[7]
order = [(0, "loop top (LUT chunk, shfl)"), (1, "wait s_full (QK done)"), (6, "LDTM S + wait::ld"),
         (2, "mask + row max + gate votes"), (4, "[pair: bar.sync] exp2 + row sum"),
         (3, "(rare) O rescale"), (5, "P~ STTM + fence + arrive")]
tot = ph[:7].sum()
print(f"{os.environ['SPARGE_LIB']} {w}: tiles {tiles}, cycles per tile per softmax warp {tot / tiles / 4:.0f}")
for k, n in order:
    print(f"  {n:36s} {ph[k] / tiles / 4:8.0f} cyc  {100 * ph[k] / tot:5.1f}%")
