"""Kernel speed versus sparsity (the analogue of the paper's Fig. 7, P:L526,
P:L533; SURVEY.md §8(d) "secondary"): N = 22528, d = 128, 32 heads,
non-causal, random Gaussian Q/K/V, forced uniform-random block masks at
densities 1.0 ... 0.1 with lambda = -inf, so the measurement isolates kernel
efficiency from the data.  Both kernels: SpargeAttn+Sage (INT8 QK^T, the
default) and SpargeAttn+FA2 (bf16 QK^T, row f1).  Times the attention launch
alone (CUDA events on the launching stream, L2 flushed, median of 7).

usage: python scripts/fig7_sweep.py [--out profiles/r01_fig7_sweep.json]
"""
import argparse, json, math, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
from paper_2502_18137_b200 import inputs, sparge

ap = argparse.ArgumentParser()
ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01_fig7_sweep.json"))
ap.add_argument("--N", type=int, default=22528)
ap.add_argument("--heads", type=int, default=32)
args = ap.parse_args()
N, d, H = args.N, 128, args.heads
tm, tn = math.ceil(N / 128), math.ceil(N / 64)
q, k, v = (inputs.to_device(inputs.gaussian(s, 1, H, N, d)) for s in (1, 2, 3))
o = torch.empty_like(q)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
dense_ops = 4.0 * N * N * d * H
peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
bf16_peak = float(peaks.get("bf16_tflops", 1590.0))

rows = []
for qk in (sparge.SPARGE_QK_INT8, sparge.SPARGE_QK_INPUT):
    shape = sparge.make_shape(1, H, H, N, d, False, q.dtype, qk_dtype=qk)
    bf = sparge.Buffers(shape)
    sparge.sparge_quantize(shape, q, 0, None, bf.qq, bf.dq, bf.q_pooled, bf.q_sim)
    sparge.sparge_quantize(shape, k, 1, None, bf.kq, bf.dk, bf.k_pooled, bf.k_sim)
    sparge.sparge_attn_fwd_ex(shape, bf.qq, bf.dq, bf.kq, bf.dk, v, bf.lut, bf.cnt, -math.inf,
                              None, o, None, bf.workspace, sparge.SPARGE_ATTN_VPREP_ONLY)
    rng = np.random.default_rng(0)
    for dens in (1.0, 0.9, 0.8, 0.7, 0.6, 0.5, 0.4, 0.3, 0.2, 0.1):
        nk = max(1, int(round(dens * tn)))
        lut = np.zeros((H, tm, tn), np.int32)
        for h in range(H):
            for i in range(tm):
                lut[h, i, :nk] = np.sort(rng.choice(tn, nk, replace=False))
        bf.lut.copy_(torch.from_numpy(lut).view(1, H, tm, tn))
        bf.cnt.fill_(nk)
        ts = []
        for it in range(10):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            sparge.sparge_attn_fwd_ex(shape, bf.qq, bf.dq, bf.kq, bf.dk, v, bf.lut, bf.cnt,
                                      -math.inf, None, o, None, bf.workspace,
                                      sparge.SPARGE_ATTN_SKIP_VPREP)
            b.record()
            torch.cuda.synchronize()
            if it >= 3:
                ts.append(a.elapsed_time(b))
        ms = float(np.median(ts))
        executed = 4.0 * 128 * 64 * d * nk * tm * H          # QK + PV of every kept tile
        peak = (2 * bf16_peak if qk == sparge.SPARGE_QK_INT8 else bf16_peak)
        mix = executed / (executed / 2 / (2 * bf16_peak if qk == 0 else bf16_peak)
                          + executed / 2 / bf16_peak) if executed else peak
        row = {"kernel": "int8_qk (SpargeAttn+Sage)" if qk == 0 else "bf16_qk (SpargeAttn+FA2, f1)",
               "density": nk / tn, "sparsity": 1 - nk / tn, "attn_ms": ms,
               "effective_tops": dense_ops / (ms * 1e-3) / 1e12,
               "kernel_tops": executed / (ms * 1e-3) / 1e12,
               "tensor_frac": executed / (ms * 1e-3) / 1e12 / mix}
        rows.append(row)
        print(json.dumps(row), flush=True)
    del bf
    torch.cuda.empty_cache()
os.makedirs(os.path.dirname(args.out), exist_ok=True)
json.dump({"N": N, "d": d, "heads": H, "lambda": "-inf", "rows": rows}, open(args.out, "w"), indent=1)
