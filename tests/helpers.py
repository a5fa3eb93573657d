"""Test-side glue between the seeded inputs, the oracle and the C-ABI path."""

import math

import numpy as np

import oracle as O


def bf16_np(t):
    """torch bf16/fp16 tensor -> float64 numpy (exact widening)."""
    return t.detach().float().cpu().double().numpy()


def oracle_forward(q, k, v, tau, theta, lam, causal=False, perm=None, group=1, qblocks=None,
                   heads=None, sim_mode="cosine", quantize=True, pv_round="bf16", smooth=False,
                   trace=False):
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
                                                   smooth=sm, trace=trace)
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


HEAD_L1 = 5e-3     # whole-head relative L1 vs the oracle: the bug signal (north star: 2e-2)
ROW_L1 = 2e-2      # every single query row must also be within the north star's 2e-2
# FP8 P~V (row f4, R27): a P~ entry within rounding reach of an E4M3 midpoint
# may round to the other neighbour on the GPU (fp32 exp2) than in the fp64
# oracle -- one E4M3 step is 2^-3 relative, so one such flip on a row's
# dominant key moves that row by up to 2^-3 (R30).  Head L1 stays 5e-3.
ROW_L1_FP8 = 2.0 ** -3


def check_o(o, o_ref, label="", head_tol=HEAD_L1, row_tol=ROW_L1):
    """O parity, element by element summarised two ways: the whole head's
    relative L1 (< head_tol) and EVERY row's relative L1 (< row_tol), so a
    single corrupted row or warp slice cannot hide in the head norm.  Rows
    where o_ref is NaN (not sampled by the oracle) are skipped.  Returns
    (head L1, worst row L1)."""
    o = np.asarray(o, dtype=np.float64)
    o_ref = np.asarray(o_ref, dtype=np.float64)
    rows = ~np.isnan(o_ref).any(axis=1)
    assert rows.any(), f"{label}: no oracle rows"
    a, b = o[rows], o_ref[rows]
    assert np.isfinite(a).all(), f"{label}: non-finite GPU output"
    head = float(np.abs(a - b).sum() / np.abs(b).sum())
    per_row = np.abs(a - b).sum(axis=1) / np.maximum(np.abs(b).sum(axis=1), 1e-300)
    worst = float(per_row.max())
    assert head < head_tol, f"{label}: head relative L1 {head:.3e} >= {head_tol}"
    assert worst < row_tol, (f"{label}: row {int(np.argmax(per_row))} relative L1 {worst:.3e} "
                             f">= {row_tol}")
    return head, worst


def gate_near(gap, mag, lam, tol=1e-5, rel=1e-6):
    """Gate decisions within rounding reach of lambda (SURVEY §8(c) debug
    mode): |g - lambda| < 1e-5, widened by the fp32 rounding of S at its own
    magnitude (|S| up to mag; the kernel's S and running max are fp32,
    DESIGN.md R29)."""
    with np.errstate(invalid="ignore"):
        return np.abs(gap - lam) < tol + rel * mag


def check_gate(mpv_gpu, cnt_ref, lam, gpu_pv_slices=None, qblocks=None, label=""):
    """Lambda-gate decision parity (SURVEY §8(c) debug mode, Alg. 1 line 15,
    P:L214): on every (tile, warp) kept by both sides the GPU's decision
    (2 computed / 1 skipped, sparge_attn_fwd_mpv) equals the oracle's except
    where |g - lambda| is within rounding reach (gate_near).  The GPU's PV
    slice counter must equal its own dumped decisions exactly.  Returns the
    number of near-band disagreements."""
    mpv_gpu = np.asarray(mpv_gpu)
    ref = cnt_ref["mpv"]
    if qblocks is not None:
        sel = np.zeros(ref.shape[0], dtype=bool)
        sel[list(qblocks)] = True
    else:
        sel = np.ones(ref.shape[0], dtype=bool)
    both = (mpv_gpu > 0) & (ref > 0) & sel[:, None, None]
    diff = both & (mpv_gpu != ref)
    near = gate_near(cnt_ref["gap"], cnt_ref["mag"], float(np.float32(lam)))
    bad = diff & ~near
    assert not bad.any(), (f"{label}: {int(bad.sum())} gate decisions differ outside the "
                           f"near-lambda band, first at {np.argwhere(bad)[0].tolist()}")
    if gpu_pv_slices is not None:
        assert int(gpu_pv_slices) == int((mpv_gpu == 2).sum()), label
    return int(diff.sum())
