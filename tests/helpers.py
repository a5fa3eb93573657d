"""Test-side glue between the seeded inputs, the oracle and the C-ABI path."""

import math

import numpy as np

import oracle as O


def bf16_np(t):
    """torch bf16/fp16 tensor -> float64 numpy (exact widening)."""
    return t.detach().float().cpu().double().numpy()


def oracle_forward(q, k, v, tau, theta, lam, causal=False, perm=None, group=1, qblocks=None,
                   heads=None, sim_mode="cosine", quantize=True, pv_round="bf16", smooth=False):
    """Oracle pipeline on fp64 arrays q [Hq, N, d], k/v [Hkv, N, d] (one batch).
    With perm the sequence is permuted first and O inverse-permuted.
    Returns dict of per-head results."""
    tau, theta, lam = O.f32(tau), O.f32(theta), O.f32(lam)
    Hq = q.shape[0]
    out = {}
    for h in (range(Hq) if heads is None else heads):
        g = h // group
        qh, kh, vh = q[h], k[g], v[g]
        sm = O.smooth_k_mean(kh) if smooth else False      # original token order (R28)
        if perm is not None:
            qh, kh, vh = qh[perm], kh[perm], vh[perm]
        o, M, near, cnt, quant = O.spargeattn_head(qh, kh, vh, tau, theta, lam, causal=causal,
                                                   qblocks=qblocks, sim_mode=sim_mode,
                                                   quantize=quantize, pv_round=pv_round,
                                                   smooth=sm)
        if perm is not None:
            inv = np.empty_like(perm)
            inv[perm] = np.arange(perm.size)
            o = o[inv]
        out[h] = dict(o=o, M=M, near=near, cnt=cnt, quant=quant)
    return out


def rows_of_blocks(qblocks, n, bq=128, perm=None):
    rows = np.concatenate([np.arange(i * bq, min((i + 1) * bq, n)) for i in qblocks])
    if perm is not None:
        rows = perm[rows]  # original positions of those permuted rows
    return np.sort(rows)


def rel_l1(a, b):
    return float(np.abs(a - b).sum() / np.abs(b).sum())
