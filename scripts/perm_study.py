"""Scope row f3: permutation and self-similarity-judge study (§4.5 Table 6,
P:L595-618; App. A.2 Tables 13-14; App. A.3 Table 15,
P:L773-801) on the synthetic smooth-3D video workloads, through the GPU path.

For each token order (random / rowmajor / columnmajor / timemajor / hilbert):
Sim-q, Sim-k = mean block CosSim of Q (b_q = 128) and K (b_k = 64) blocks
(a1 statistics), L1 vs full attention without quantisation (the f1 kernel,
filters off; the paper uses FlashAttention2), sparsity per R16 --
averaged over five seeded inputs, with one (tau, theta, lambda) per workload:
the f2 tuner's result at (l1, l2) = (0.05, 0.06) ("pre-searched
hyperparameters with l1=0.05, l2=0.06") from profiles/r01_f2_tuned.json.
The judge ablation reruns with theta = -1 (self-similarity judge off).

usage: python scripts/perm_study.py [--out profiles/r01_f3_perm_study.json] [workload ...]
"""
import argparse, json, math, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import bench
from paper_2502_18137_b200 import inputs, permutations, tuner

ap = argparse.ArgumentParser()
ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01_f3_perm_study.json"))
ap.add_argument("--tuned", default=os.path.join(ROOT, "profiles", "r01_f2_tuned.json"))
ap.add_argument("--seeds", type=int, default=5)
ap.add_argument("workloads", nargs="*", default=["cogvideox_2b", "mochi"])
args = ap.parse_args()
tuned = json.load(open(args.tuned)) if os.path.exists(args.tuned) else {}
report = {}
for w in args.workloads:
    cfg = bench.workload_cfg(w)
    tp = tuned.get(w, {"tau": cfg["tau"], "theta": cfg["theta"], "lambda": cfg["lam"]})
    tau, theta = float(tp["tau"]), float(tp["theta"])
    lam = -math.inf if tp["lambda"] == "-inf" else float(tp["lambda"])
    cal = [tuple(inputs.to_device(a) for a in bench.gen_inputs(cfg, 3000 + s))
           for s in range(args.seeds)]
    rows = {}
    for kind in permutations.KINDS:
        perm = torch.from_numpy(permutations.make_perm(kind, cfg["T"], cfg["H"], cfg["W"],
                                                       cfg["text_prefix"], seed=7)).cuda()
        ev = tuner.GpuEvaluator(cal, causal=False, perm=perm)
        sim_q = float(np.mean([it[2].q_sim.mean().item() for it in ev.items]))
        sim_k = float(np.mean([it[2].k_sim.mean().item() for it in ev.items]))
        err, sp = ev(tau, theta, lam)
        err_nj, sp_nj = ev(tau, -1.0, lam)
        rows[kind] = {"sim_q": sim_q, "sim_k": sim_k, "l1": err, "sparsity": sp,
                      "no_judge": {"l1": err_nj, "sparsity": sp_nj}}
        print(w, kind, json.dumps(rows[kind]), flush=True)
        del ev
        torch.cuda.empty_cache()
    report[w] = {"params": {"tau": tau, "theta": theta, "lambda": tp["lambda"]},
                 "seeds": args.seeds, "l1_is": "max over seeds", "sparsity_is": "mean over seeds",
                 "rows": rows}
os.makedirs(os.path.dirname(args.out), exist_ok=True)
json.dump(report, open(args.out, "w"), indent=1)
