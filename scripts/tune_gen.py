"""Pick generator knobs so the oracle's stage-1 mask at tau=.9/theta=.5 lands
in the paper's Llama sparsity band (0.36-0.54).  CPU only."""
import math, sys, time
import numpy as np, torch
sys.path.insert(0, '.')
import oracle as O
from paper_2502_18137_b200 import inputs

def bf(x): return torch.from_numpy(x).bfloat16().double().numpy()

def study(N, causal, **kw):
    q, k, v = inputs.llm_local(1000, N, d=128, Hq=4, Hkv=1, heads=[0], **kw)
    qs, ks, vs = bf(q[0, 0]), bf(k[0, 0]), bf(v[0, 0])
    M, near, st = O.predict_mask(qs, ks, 0.9, 0.5, causal=causal, return_stats=True)
    tm, tn = M.shape
    live = sum(O.causal_live(i, j, N, 128, 64) or not causal for i in range(tm) for j in range(tn))
    kept = M.sum() / live
    qb = [1, tm // 2, tm - 1]
    o, cnt = O.sparse_attention(qs, ks, vs, M, -5.0, causal=causal, qblocks=qb, quant=None, pv_round=None)
    rows = np.concatenate([np.arange(i*128, min((i+1)*128, N)) for i in qb])
    od = O.dense_attention(qs, ks, vs, causal=causal, rows=rows)
    l1 = np.abs(o[rows] - od).sum() / np.abs(od).sum()
    print(f"N={N} {kw} kept={kept:.3f} s_q<th={np.mean(st['s_q']<0.5):.2f} s_k<th={np.mean(st['s_k']<0.5):.2f} "
          f"sim_q={st['s_q'].mean():.2f} sim_k={st['s_k'].mean():.2f} L1(dense)={l1:.3f}", flush=True)

for kw in ([] if len(sys.argv) > 1 else [dict(gamma=0.7)]):
    study(8192, True, **kw)
if len(sys.argv) > 1:
    for kw in eval(sys.argv[1]):
        study(int(sys.argv[2]) if len(sys.argv) > 2 else 8192, True, **kw)
