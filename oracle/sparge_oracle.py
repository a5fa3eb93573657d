"""fp64 SpargeAttn oracle (TEST INFRASTRUCTURE ONLY; see oracle/__init__).

Every function cites the PAPER.md passage it follows (P:Lnnn = line in
/root/reference/PAPER.md).  Readings of silent/ambiguous passages are the R#
items of DESIGN.md §3.  Arrays are numpy; one attention head at a time
(``[N, d]``) unless a function says otherwise.  Inputs are bf16 values that
the caller has widened exactly to float64.

Nothing here is blocked, fused or reordered beyond what the paper's
definitions state: loops follow Algorithm 1 line by line.
"""

import math
from fractions import Fraction

import numpy as np

__all__ = [
    "OracleInvariantError",
    "f32",
    "block_count",
    "quantize_blocks",
    "SMOOTH_CHUNK",
    "smooth_k_mean",
    "smooth_k",
    "block_mean",
    "cos_sim",
    "block_sims",
    "compressed_map",
    "top_cdf",
    "top_cdf_rational",
    "predict_mask",
    "causal_live",
    "E4M3_MAX",
    "round_e4m3",
    "fp8_v_quant",
    "round_bf16",
    "round_fp16",
    "sparse_attention",
    "dense_attention",
    "relative_l1",
    "sparsity_of",
    "spargeattn_head",
]

LOG2E = 1.4426950408889634


class OracleInvariantError(RuntimeError):
    """A valid query row finished Algorithm 1 with l = 0 (reading R8/R9)."""


def f32(v):
    """The fp64 value of a float32-rounded scalar.  The C-ABI passes tau,
    theta and lambda as float32, so the oracle compares against the same
    numbers."""
    return float(np.float32(v))


def block_count(n, b):
    """T = ceil(N / b) blocks (Definition 1; reading R6)."""
    return (n + b - 1) // b


# --------------------------------------------------------------------------
# Alg. 1 line 3: per-block INT8 quantisation "in SageAttention".
# --------------------------------------------------------------------------
def quantize_blocks(x, b):
    """Symmetric per-block INT8 quantisation, emulated in IEEE fp32 (R11).

    For each block of b rows (the last may be partial, R6):
        amax  = max |x|
        amax == 0       -> delta = 1, q = 0
        else inv  = fl32(127 / amax)
             q    = clamp(rne(fl32(x * inv)), -127, 127)
             delta= fl32(amax / 127)
    so that x ~= q * delta (dequantisation of Alg. 1 line 12).
    Returns (q int8 [N, d], delta float32 [T])."""
    x32 = np.asarray(x, dtype=np.float64).astype(np.float32)
    n = x32.shape[0]
    t = block_count(n, b)
    q = np.zeros(x32.shape, dtype=np.int8)
    delta = np.ones(t, dtype=np.float32)
    for i in range(t):
        blk = x32[i * b:min((i + 1) * b, n)]
        amax = np.float32(np.max(np.abs(blk))) if blk.size else np.float32(0)
        if amax == 0:
            continue
        inv = np.float32(127.0) / amax                    # fp32 division, RNE
        scaled = (blk * inv).astype(np.float32)           # fp32 multiply, RNE
        qi = np.clip(np.rint(scaled), -127, 127)          # round half to even
        q[i * b:min((i + 1) * b, n)] = qi.astype(np.int8)
        delta[i] = amax / np.float32(127.0)
    return q, delta


# --------------------------------------------------------------------------
# Row f4, K smoothing (SageAttention, footnote P:L44 "SageAttention2"; the
# paper fixes no arithmetic -- reading R28): K' = K - mean_t K before the
# INT8 quantisation of line 3.  S' = S - q.mu is a per-query-row constant
# shift, so softmax, the lambda gate's m_local - m_new and O are unchanged in
# exact arithmetic; only the INT8 rounding of K improves.  Stage 1 keeps the
# raw K (R14: P^ is shift-invariant, CosSim is not).
# --------------------------------------------------------------------------
SMOOTH_CHUNK = 128


def smooth_k_mean(k):
    """mu = the per-channel token mean of one head's K [N, d], in the fixed
    summation order of reading R28: fp64, tokens in index order within chunks
    of SMOOTH_CHUNK tokens (a sequential sum), chunk sums added in chunk
    order; then / N and rounded to fp32."""
    k = np.asarray(k, dtype=np.float64)
    n, d = k.shape
    total = np.zeros(d)
    for c0 in range(0, n, SMOOTH_CHUNK):
        part = np.cumsum(k[c0:min(c0 + SMOOTH_CHUNK, n)], axis=0)[-1]   # sequential
        total = total + part
    return (total / n).astype(np.float32)


def smooth_k(k, mu):
    """K' = fl32(K - mu) element-wise (fp32 subtraction, RNE), as fp64."""
    k32 = np.asarray(k, dtype=np.float64).astype(np.float32)
    return (k32 - np.asarray(mu, dtype=np.float32)).astype(np.float32).astype(np.float64)


# --------------------------------------------------------------------------
# Alg. 1 line 4 and §3.2: q_i = mean(Q_i, axis=0).
# --------------------------------------------------------------------------
def block_mean(x, b):
    """Mean token of every block, over the block's valid rows only (R6)."""
    x = np.asarray(x, dtype=np.float64)
    n = x.shape[0]
    t = block_count(n, b)
    return np.stack([x[i * b:min((i + 1) * b, n)].mean(axis=0) for i in range(t)])


# --------------------------------------------------------------------------
# §3.2: CosSim(X) = mean(X X^T / |max(X X^T)|).
# --------------------------------------------------------------------------
def cos_sim(X, mode="cosine"):
    """Block self-similarity, evaluated literally as a Gram-matrix mean.

    mode="cosine" (reading R1-A, default): the prose says "mean cosine
    similarity across tokens", so rows are L2-normalised first
    (a zero row stays zero) and the formula is applied to X^ X^T.
    mode="literal" (R1-B): the formula on the raw rows.
    Both: if max(G) == 0 (an all-zero block) the block is treated as
    perfectly self-similar, 1.0."""
    X = np.asarray(X, dtype=np.float64)
    if mode == "cosine":
        norms = np.sqrt((X * X).sum(axis=1))
        Xn = np.zeros_like(X)
        nz = norms > 0
        Xn[nz] = X[nz] / norms[nz, None]
        G = Xn @ Xn.T
    elif mode == "literal":
        G = X @ X.T
    else:
        raise ValueError(mode)
    gmax = np.max(G)
    if gmax == 0:
        return 1.0
    return float(np.mean(G / abs(gmax)))


def block_sims(x, b, mode="cosine"):
    """s[i] = CosSim(X_i) for every block i (Alg. 1 line 5)."""
    x = np.asarray(x, dtype=np.float64)
    n = x.shape[0]
    return np.array([cos_sim(x[i * b:min((i + 1) * b, n)], mode)
                     for i in range(block_count(n, b))])


def causal_live(i, j, n, bq, bk):
    """Tile (i, j) contains at least one key <= query (reading R8-i)."""
    return j * bk <= min((i + 1) * bq, n) - 1


# --------------------------------------------------------------------------
# Alg. 1 lines 5-6, §3.2: the compressed map.
# --------------------------------------------------------------------------
def compressed_map(qbar, kbar, s_k, theta, n, bq, bk, causal=False):
    """S^ = q k^T / sqrt(d) (R2), S^[:, j] = -inf if s_kj < theta (strict, R5),
    -inf on causally dead tiles (R8-i); P^ = row softmax of S^.

    Returns (S_hat, P_hat, all_inf_rows).  A row that is entirely -inf has
    P^ = 0 and is flagged (R7)."""
    qbar = np.asarray(qbar, dtype=np.float64)
    kbar = np.asarray(kbar, dtype=np.float64)
    d = qbar.shape[1]
    tm, tn = qbar.shape[0], kbar.shape[0]
    S = (qbar @ kbar.T) / math.sqrt(d)
    S[:, np.asarray(s_k) < theta] = -np.inf
    if causal:
        for i in range(tm):
            for j in range(tn):
                if not causal_live(i, j, n, bq, bk):
                    S[i, j] = -np.inf
    P = np.zeros_like(S)
    flagged = np.zeros(tm, dtype=bool)
    for i in range(tm):
        row = S[i]
        mx = np.max(row)
        if mx == -np.inf:
            flagged[i] = True
            continue
        e = np.exp(row - mx)
        P[i] = e / e.sum()
    return S, P, flagged


# --------------------------------------------------------------------------
# §3.2 TopCdf (prose P:L253, pseudocode P:L273-281).
# --------------------------------------------------------------------------
def top_cdf(p, tau, near_tol=None):
    """The paper's Top_Cdf, reading R4:
        sort P[i] descending, ties by ascending index;
        cusum = inclusive cumulative sum in that order (sequential fp64);
        keep rank k iff cusum[k] <= tau * cusum[-1]   ("<=");
        always keep rank 0 (top-1 guard).
    Returns a bool row; with near_tol also a bool row of entries whose
    decision lies within near_tol*c_last of the threshold or that tie (within
    near_tol relative) with an entry across the cut."""
    p = np.asarray(p, dtype=np.float64)
    tn = p.size
    order = np.lexsort((np.arange(tn), -p))
    c = np.cumsum(p[order])
    thr = tau * c[-1]
    keep_rank = c <= thr
    keep_rank[0] = True
    m = np.zeros(tn, dtype=bool)
    m[order] = keep_rank
    if near_tol is None:
        return m
    near_rank = np.abs(c - thr) <= near_tol * c[-1]
    near_rank[0] = False  # the guard decides rank 0 regardless
    ps = p[order]
    for k in range(tn - 1):
        if keep_rank[k] != keep_rank[k + 1] and abs(ps[k] - ps[k + 1]) <= near_tol * ps[k]:
            near_rank[k] = near_rank[k + 1] = True
    near = np.zeros(tn, dtype=bool)
    near[order] = near_rank
    return m, near


def top_cdf_rational(p, tau):
    """Sort-free TopCdf in exact rational arithmetic (pin P4).

    j is kept iff the total mass of entries ranked at or ahead of j --
    ranked by (value desc, index asc) -- is <= tau * total, or j is the
    top-ranked entry.  ``p`` and ``tau`` are Fractions (or ints)."""
    p = [Fraction(v) for v in p]
    tau = Fraction(tau)
    total = sum(p, Fraction(0))
    tn = len(p)
    top = min(range(tn), key=lambda k: (-p[k], k))
    out = []
    for j in range(tn):
        ahead = sum((p[k] for k in range(tn) if (-p[k], k) <= (-p[j], j)), Fraction(0))
        out.append(j == top or ahead <= tau * total)
    return out


# --------------------------------------------------------------------------
# Alg. 1 lines 4-6 and Eq. (5): the global mask M_g.
# --------------------------------------------------------------------------
def predict_mask(q, k, tau, theta, bq=128, bk=64, causal=False, sim_mode="cosine",
                 near_tol=1e-6, return_stats=False):
    """M_g for one (q-head, kv-head) pair from the un-quantised Q, K
    (the prediction reads Q_i, K_j; reading R15).

    Steps (O3-O8 in DESIGN.md §4):
      q_i = mean(Q_i), k_j = mean(K_j); s_qi, s_kj = CosSim;
      S^, P^ = compressed_map(...);  M[i,:] = TopCdf(P^[i], tau);
      M[i,:] = 1 if s_qi < theta;  M[:, j] = 1 if s_kj < theta;
      an all -inf row -> all ones (R7);
      causal: M &= live, then M[i, floor(i*bq/bk)] = 1 (R8-iii).
    Returns M (uint8 [T_m, T_n]) and ``near`` (bool [T_m, T_n]): entries
    whose decision lies within near_tol of a threshold (the parity criterion
    of DESIGN.md §5)."""
    n, d = q.shape
    tm, tn = block_count(n, bq), block_count(n, bk)
    qbar, kbar = block_mean(q, bq), block_mean(k, bk)
    s_q, s_k = block_sims(q, bq, sim_mode), block_sims(k, bk, sim_mode)
    S, P, flagged = compressed_map(qbar, kbar, s_k, theta, n, bq, bk, causal)
    M = np.zeros((tm, tn), dtype=bool)
    near = np.zeros((tm, tn), dtype=bool)
    for i in range(tm):
        if flagged[i]:
            continue
        M[i], near[i] = top_cdf(P[i], tau, near_tol)
    M[s_q < theta, :] = True
    M[:, s_k < theta] = True
    M[flagged, :] = True
    # Similarity decisions near theta: a flipped column changes every row's
    # softmax, so the whole head is near; a flipped row changes that row.
    if np.any(np.abs(s_k - theta) < near_tol):
        near[:, :] = True
    near[np.abs(s_q - theta) < near_tol, :] = True
    if causal:
        for i in range(tm):
            for j in range(tn):
                if not causal_live(i, j, n, bq, bk):
                    M[i, j] = False
                    near[i, j] = False
            M[i, (i * bq) // bk] = True
    M = M.astype(np.uint8)
    if return_stats:
        return M, near, dict(qbar=qbar, kbar=kbar, s_q=s_q, s_k=s_k, S_hat=S, P_hat=P,
                             flagged=flagged)
    return M, near


# --------------------------------------------------------------------------
# P~ rounding for the P~V product (R12/R13).
# --------------------------------------------------------------------------
def round_bf16(x):
    """Round fp64 values to the nearest bf16 (8 significant bits), ties to
    even, directly from fp64 (no double rounding).  The exponent range is
    not clamped: values below bf16's normal range are far below the L1
    tolerance."""
    x = np.asarray(x, dtype=np.float64)
    m, e = np.frexp(x)              # x = m * 2**e, 0.5 <= |m| < 1
    return np.ldexp(np.rint(m * 256.0) / 256.0, e)


def round_fp16(x):
    """Round fp64 values to the nearest IEEE binary16 value (11 significant
    bits, normals from 2^-14, subnormals on the 2^-24 grid), ties to even,
    directly from fp64 -- the P~ operand of the P~V product for fp16 inputs
    (R12/R13: P~ is rounded to the input dtype).  P~ <= 1 here, so the
    overflow range (> 65504) is not modelled."""
    x = np.asarray(x, dtype=np.float64)
    a = np.abs(x)
    _, e = np.frexp(a)                   # a = m 2^e, 0.5 <= m < 1
    E = np.maximum(e - 1, -14)           # exponent of the leading bit; subnormals share -14
    q = np.ldexp(1.0, E - 10)            # spacing of representable values around a
    return np.copysign(np.rint(a / q) * q, x)


E4M3_MAX = 448.0


def round_e4m3(x):
    """Round fp64 values to the nearest FP8 E4M3 value (the OCP "fn" format:
    3 mantissa bits, bias 7, normals 2^-6 .. 448, subnormals on the 2^-9
    grid), ties to even, saturating to +-448 -- the P~ and V operands of
    SageAttention2's FP8 P~V product (footnote P:L44; scope row f4, R27).
    Directly from fp64 (no double rounding)."""
    x = np.asarray(x, dtype=np.float64)
    a = np.abs(x)
    _, e = np.frexp(a)                   # a = m 2^e, 0.5 <= m < 1 (e = 0 for a = 0)
    E = np.maximum(e - 1, -6)            # exponent of the leading bit; subnormals share -6
    q = np.ldexp(1.0, E - 3)             # spacing of representable values around a
    r = np.minimum(np.rint(a / q) * q, E4M3_MAX)
    return np.copysign(r, x)


def fp8_v_quant(V):
    """Per-channel FP8 quantisation of V (SageAttention2, R27): over all rows
    of the head, amax_c = max|V[:, c]| (fp32), inv_c = fl32(448 / amax_c),
    s_c = fl32(amax_c / 448), V^ = e4m3(fl32(V * inv_c)); an all-zero column
    has inv_c = s_c = 1.  Returns (V^ fp64 [N, d], s fp32 [d])."""
    V32 = np.asarray(V, dtype=np.float64).astype(np.float32)
    amax = np.abs(V32).max(axis=0)
    nz = amax > 0
    one = np.float32(1.0)
    inv = np.where(nz, np.float32(E4M3_MAX) / np.where(nz, amax, one), one).astype(np.float32)
    sc = np.where(nz, amax / np.float32(E4M3_MAX), one).astype(np.float32)
    return round_e4m3((V32 * inv[None, :]).astype(np.float64)), sc


# --------------------------------------------------------------------------
# Alg. 1 lines 7-21: stage 2, the sparse FlashAttention loop.
# --------------------------------------------------------------------------
def sparse_attention(Q, K, V, M, lam, bq=128, bk=64, cw=4, causal=False, quant=None,
                     pv_round="bf16", qblocks=None, v_fp8=None, trace=False):
    """O for one head, following Algorithm 1 and the online
    softmax of Eq. (1).

    Q, K: fp64 [N, d] (used when quant is None: S = Q K^T / sqrt(d));
    quant = (Qq int8, dq f32, Kq int8, dk f32): S = (Qq_i Kq_j^T) dq_i dk_j
            / sqrt(d) (line 12; 1/sqrt(d) per R3) -- the integer
            product is exact;
    V: fp64 [N, d];  M: [T_m, T_n] mask (line 10);  lam: lambda (natural-log
    units of S, R3; -inf disables);  pv_round: "bf16" / "fp16" round P~ to the
    input dtype before P~V (R12/R13), None keeps fp64, "fp8" is the f4
    product (R27): e4m3(128 P~) times V^ of v_fp8 = fp8_v_quant(V),
    O = acc * s / (128 l).
    trace: also record every gate decision of line 15 -- counters gain
    "mpv" uint8 [T_m, T_n, cw] (2 computed, 1 skipped, 0 block not kept),
    "gap" fp64 [T_m, T_n, cw] (g = max over the group's rows of
    m_local - m_new; NaN where not kept) and "mag" fp64 [T_m, T_n, cw]
    (max |m_local|, |m_new| over the group: the scale of S there).
    qblocks: optional list of q-block indices to compute (sampling); other
    rows of O are NaN.

    Returns (O [N, d], counters dict(qk=#executed QK tiles,
    pv_slices=#executed (tile, warp) P~V slices))."""
    V = np.asarray(V, dtype=np.float64)
    n, d = V.shape
    tm, tn = block_count(n, bq), block_count(n, bk)
    rs = math.sqrt(d)
    if quant is not None:
        Qq, dq, Kq, dk = quant
        Qi64 = np.asarray(Qq, dtype=np.int64)
        Ki64 = np.asarray(Kq, dtype=np.int64)
    else:
        Q = np.asarray(Q, dtype=np.float64)
        K = np.asarray(K, dtype=np.float64)
    O = np.full((n, d), np.nan)
    cnt = dict(qk=0, pv_slices=0)
    if trace:
        cnt["mpv"] = np.zeros((tm, tn, cw), dtype=np.uint8)
        cnt["gap"] = np.full((tm, tn, cw), np.nan)
        cnt["mag"] = np.full((tm, tn, cw), np.nan)
    wrows = bq // cw
    for i in (range(tm) if qblocks is None else qblocks):
        r0, r1 = i * bq, min((i + 1) * bq, n)
        nr = r1 - r0
        m = np.full(nr, -np.inf)                # m_{i,0} = -inf
        l = np.zeros(nr)                        # l_{i,0} = 0
        Oi = np.zeros((nr, d))
        for j in range(tn):
            if not M[i, j]:                     # line 10: skip if M[i,j] = 0
                continue
            c0, c1 = j * bk, min((j + 1) * bk, n)
            cnt["qk"] += 1
            if quant is not None:               # line 12: dequantised scores
                acc = Qi64[r0:r1] @ Ki64[c0:c1].T
                S = acc.astype(np.float64) * float(dq[i]) * float(dk[j]) / rs
            else:
                S = (Q[r0:r1] @ K[c0:c1].T) / rs
            if causal:
                qi = np.arange(r0, r1)[:, None]
                kj = np.arange(c0, c1)[None, :]
                S = np.where(kj > qi, -np.inf, S)
            # line 13: m_local, m_ij, P~, l
            m_loc = S.max(axis=1)
            m_new = np.maximum(m, m_loc)
            with np.errstate(invalid="ignore"):
                P = np.where(np.isneginf(S), 0.0, np.exp(S - m_new[:, None]))
                alpha = np.where(np.isneginf(m_new), 1.0, np.exp(m - m_new))
            l = alpha * l + P.sum(axis=1)
            # lines 14-17: per-warp lambda gate on the P~V product
            with np.errstate(invalid="ignore"):
                gap = np.where(np.isneginf(m_loc), -np.inf, m_loc - m_new)
            for w in range(cw):
                a, b = w * wrows, min((w + 1) * wrows, nr)
                if a >= b:
                    continue                    # warp with no valid rows (R6)
                g = np.max(gap[a:b])
                if trace:
                    cnt["mpv"][i, j, w] = 2 if g > lam else 1
                    cnt["gap"][i, j, w] = g
                    fin = np.concatenate([m_loc[a:b], m_new[a:b]])
                    fin = fin[np.isfinite(fin)]
                    cnt["mag"][i, j, w] = np.max(np.abs(fin)) if fin.size else 0.0
                if g > lam:                     # compute iff > lambda (R5)
                    if pv_round == "fp8":
                        Pw = round_e4m3(P[a:b] * 128.0)
                        Oi[a:b] = alpha[a:b, None] * Oi[a:b] + Pw @ v_fp8[0][c0:c1]
                    else:
                        rnd = {"bf16": round_bf16, "fp16": round_fp16, None: None}[pv_round]
                        Pw = rnd(P[a:b]) if rnd is not None else P[a:b]
                        Oi[a:b] = alpha[a:b, None] * Oi[a:b] + Pw @ V[c0:c1]
                    cnt["pv_slices"] += 1
            m = m_new
        if np.any(l == 0):
            raise OracleInvariantError(f"q-block {i}: a row finished with l = 0")
        if pv_round == "fp8":                   # dequantise: per-channel s, the 128 of P~
            O[r0:r1] = Oi * v_fp8[1].astype(np.float64)[None, :] / (128.0 * l[:, None])
        else:
            O[r0:r1] = Oi / l[:, None]          # line 19: O_i = diag(l)^-1 O_i
    return O, cnt


def dense_attention(Q, K, V, causal=False, rows=None):
    """Two-pass fp64 softmax attention S = QK^T/sqrt(d), P = softmax(S),
    O = PV (§3.1).  ``rows`` optionally restricts the queries."""
    Q = np.asarray(Q, dtype=np.float64)
    K = np.asarray(K, dtype=np.float64)
    V = np.asarray(V, dtype=np.float64)
    n, d = Q.shape
    idx = np.arange(n) if rows is None else np.asarray(rows)
    S = (Q[idx] @ K.T) / math.sqrt(d)
    if causal:
        S = np.where(np.arange(n)[None, :] > idx[:, None], -np.inf, S)
    S = S - S.max(axis=1, keepdims=True)
    E = np.exp(S)
    return (E / E.sum(axis=1, keepdims=True)) @ V


def relative_l1(o, o_ref):
    """L1 = sum|O - O'| / sum|O'| with the reference in the denominator
    (§3.6; reading R17)."""
    o = np.asarray(o, dtype=np.float64)
    o_ref = np.asarray(o_ref, dtype=np.float64)
    den = np.abs(o_ref).sum()
    if den == 0:
        raise ValueError("zero-norm reference")
    return float(np.abs(o - o_ref).sum() / den)


def sparsity_of(qk_exec, pv_slices_exec, live_tiles, cw=4):
    """Sparsity = fraction of the Q_iK_j^T plus P~_ijV_j products skipped
    (§4.1), in tile units (R16): each live tile carries one QK and
    one PV product; a warp slice is 1/c_w of a PV product."""
    total = 2 * live_tiles
    return 1.0 - (qk_exec + pv_slices_exec / cw) / total


def spargeattn_head(q, k, v, tau, theta, lam, bq=128, bk=64, cw=4, causal=False,
                    sim_mode="cosine", quantize=True, pv_round="bf16", qblocks=None,
                    smooth=False, trace=False):
    """The whole of Algorithm 1 for one head: stage 1 (lines 3-6) then the
    sparse loop (lines 7-21).  smooth: K smoothing before the INT8
    quantisation (row f4, R28; stage 1 keeps the raw K, R14) -- True (mu of
    this k) or the fp32 mu itself.  Returns (O, M, near, counters, quant)."""
    q = np.asarray(q, dtype=np.float64)
    k = np.asarray(k, dtype=np.float64)
    M, near = predict_mask(q, k, tau, theta, bq, bk, causal, sim_mode)
    quant = None
    if quantize:
        Qq, dq = quantize_blocks(q, bq)
        if smooth is not False and smooth is not None:
            # mu of the head's K in its ORIGINAL token order (R28): passed in
            # by a caller that permuted k, else computed here
            mu = smooth_k_mean(k) if smooth is True else np.asarray(smooth, dtype=np.float32)
            Kq, dk = quantize_blocks(smooth_k(k, mu), bk)
        else:
            Kq, dk = quantize_blocks(k, bk)
        quant = (Qq, dq, Kq, dk)
    v_fp8 = fp8_v_quant(v) if pv_round == "fp8" else None
    O, cnt = sparse_attention(q, k, v, M, lam, bq, bk, cw, causal, quant, pv_round, qblocks,
                              v_fp8, trace)
    return O, M, near, cnt, quant
