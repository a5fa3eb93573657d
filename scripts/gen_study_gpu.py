"""GPU study of the llm_rope generator knobs: for each knob set
and sequence length, the largest sparsity whose relative L1 against full
attention (the f1 kernel, filters off: tuner reading R25) stays under the
paper's Llama bound l1 = 0.08, over a tau x theta grid with
lambda = -inf -- stage 1 of the §3.6 tuner on a few heads.  Used to
pick knobs under which Table 8's shape holds (sparsity rising with N at a
constant bound).  GPU only.

    python scripts/gen_study_gpu.py '[{}, {"sink": 0.0}]' [--causal] [--ns 8192,32768]
"""
import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2502_18137_b200 import inputs, tuner  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("variants")
ap.add_argument("--causal", action="store_true")
ap.add_argument("--ns", default="8192,16384,32768,65536,131072")
ap.add_argument("--heads", type=int, default=4)
ap.add_argument("--seeds", type=int, default=2)
ap.add_argument("--l1", type=float, default=0.08)
args = ap.parse_args()
TAUS = [0.5, 0.6, 0.7, 0.75, 0.8, 0.84, 0.88, 0.9, 0.92, 0.94, 0.96, 0.98, 0.99, 1.0]
THETAS = [-1.0, 0.2, 0.5]
for kw in json.loads(args.variants):
    for N in (int(x) for x in args.ns.split(",")):
        t0 = time.time()
        Hq = args.heads
        Hkv = 1 if args.causal else Hq
        cal = [tuple(inputs.to_device(a) for a in inputs.llm_rope(2000 + s, N, Hq=Hq, Hkv=Hkv, **kw))
               for s in range(args.seeds)]
        ev = tuner.GpuEvaluator(cal, causal=args.causal)
        rows = [(t, th) + ev(t, th, -math.inf) for t in TAUS for th in THETAS]
        pick = tuner.select_stage1(rows, args.l1)
        fixed = ev(0.9, 0.5, -5.0)
        print(json.dumps({"kw": kw, "N": N, "causal": args.causal, "best": pick,
                          "fixed_0.9_0.5_-5": fixed,
                          "at_tau": {str(t): [round(e, 4), round(s, 3)] for t, th, e, s in rows
                                     if th == 0.5},
                          "secs": round(time.time() - t0, 1)}), flush=True)
        del ev, cal
        torch.cuda.empty_cache()
