"""Generator study for the C2/C5 llm_rope recipe, oracle only,
CPU: for each N, the largest stage-1 sparsity whose relative L1 against
dense attention stays under the paper's Llama bound l1 = 0.08 on a
fine tau grid (theta fixed, lambda = -inf), with INT8 quantisation and bf16
P~ as in the product.  Table 8's claim is the target shape:
sparsity at a constant accuracy bound rises with N.

    python scripts/tune_gen_rope.py "dict(gamma=0.9)" CAUSAL "[8192, 32768]" [SEED]
"""
import math
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
from paper_2502_18137_b200 import inputs  # noqa: E402


def bf(x):
    return torch.from_numpy(np.ascontiguousarray(x)).bfloat16().double().numpy()


def scan(N, causal, seed=1000, theta=0.5, taus=tuple(np.round(np.arange(0.6, 1.0, 0.02), 2)),
         head=0, **kw):
    q, k, v = inputs.llm_rope(seed, N, Hq=4, Hkv=1, heads=[head], **kw)
    q, k, v = bf(q[0, 0]), bf(k[0, 0]), bf(v[0, 0])
    tm, tn = -(-N // 128), -(-N // 64)
    qbar, kbar = O.block_mean(q, 128), O.block_mean(k, 64)
    s_q, s_k = O.block_sims(q, 128), O.block_sims(k, 64)
    S, P, fl = O.compressed_map(qbar, kbar, s_k, theta, N, 128, 64, causal)
    qb = sorted(set([1, tm // 4, tm // 2, 3 * tm // 4, tm - 1]))
    rows = np.concatenate([np.arange(i * 128, min((i + 1) * 128, N)) for i in qb])
    od = O.dense_attention(q, k, v, causal=causal, rows=rows)
    quant = O.quantize_blocks(q, 128) + O.quantize_blocks(k, 64)
    live = np.array([[O.causal_live(i, j, N, 128, 64) or not causal for j in range(tn)]
                     for i in range(tm)])
    out = []
    for tau in taus:
        M = np.zeros((tm, tn), bool)
        for i in range(tm):
            if not fl[i]:
                M[i] = O.top_cdf(P[i], tau)
        M[s_q < theta, :] = True
        M[:, s_k < theta] = True
        M[fl] = True
        if causal:
            M &= live
            for i in range(tm):
                M[i, (i * 128) // 64] = True
        o, _ = O.sparse_attention(q, k, v, M.astype(np.uint8), -math.inf, causal=causal,
                                  qblocks=qb, quant=quant, pv_round="bf16")
        l1 = np.abs(o[rows] - od).sum() / np.abs(od).sum()
        out.append((tau, 1 - M.sum() / live.sum(), l1))
    return out, float(s_q.mean()), float(s_k.mean())


if __name__ == "__main__":
    kw = eval(sys.argv[1])
    causal = bool(int(sys.argv[2]))
    Ns = eval(sys.argv[3])
    seed = int(sys.argv[4]) if len(sys.argv) > 4 else 1000
    for N in Ns:
        t0 = time.time()
        res, sq, sk = scan(N, causal, seed=seed, **kw)
        best = max([r for r in res if r[2] < 0.08], key=lambda r: r[1], default=None)
        print(f"{kw} causal={int(causal)} N={N} seed={seed}: sim_q {sq:.2f} sim_k {sk:.2f}; "
              f"best at l1<0.08: tau={best and best[0]} sparsity={best and round(best[1], 3)} "
              f"L1={best and round(best[2], 4)}  ({time.time() - t0:.0f}s)", flush=True)
