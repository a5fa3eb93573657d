import math, sys
import numpy as np, torch
sys.path.insert(0, 'tests'); sys.path.insert(0, '.')
import oracle as O
from helpers import bf16_np, oracle_forward, rel_l1
from paper_2502_18137_b200 import inputs, sparge as lib

def case(N, d, H, tau, theta, lam, seeds=(1,2,3), gen='gauss'):
    if gen == 'gauss':
        qn, kn, vn = (inputs.gaussian(s, 1, H, N, d) for s in seeds)
    else:
        qn, kn, vn = inputs.llm_local(5, N, d=d, Hq=H, Hkv=H, gamma=1.5)
    q, k, v = (inputs.to_device(a) for a in (qn, kn, vn))
    o, bf = lib.sparge_forward(q, k, v, tau, theta, lam)
    lib.sparge_attn_status(bf.workspace)
    ref = oracle_forward(bf16_np(q)[0], bf16_np(k)[0], bf16_np(v)[0], tau, theta, lam)
    og = bf16_np(o)[0]
    for h in range(H):
        e = np.abs(og[h] - ref[h]['o']).sum(1) / np.abs(ref[h]['o']).sum(1)
        blocks = [float(e[i*128:(i+1)*128].mean()) for i in range(math.ceil(N/128))]
        warps = [float(e[w*32:(w+1)*32].mean()) for w in range(4)]
        print(f"N={N} d={d} tau={tau} lam={lam} {gen} h={h} L1={rel_l1(og[h], ref[h]['o']):.3e} "
              f"blocks={np.round(blocks,4).tolist()} cnt={bf.counters.cpu().numpy()[0,h].tolist()} ref={ref[h]['cnt']}")
        bad = np.where(e > 0.02)[0]
        print("   bad rows:", bad[:40].tolist(), len(bad))

case(900, 128, 2, 1.0, -1.0, -math.inf)
case(900, 128, 2, 1.0, -1.0, -5.0)
case(1024, 128, 1, 1.0, -1.0, -math.inf)
case(900, 128, 1, 0.9, 0.5, -math.inf)
case(900, 128, 1, 1.0, -1.0, -math.inf, gen='llm')
case(900, 64, 1, 1.0, -1.0, -math.inf)
case(256, 128, 1, 1.0, -1.0, -math.inf)
