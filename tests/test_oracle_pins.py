"""Pins of the fp64 oracle against what the paper and mathematics fix
(SURVEY.md §8(c) table P).  CPU only.

Each test names the pin (P1..P12) and the passage it checks.  None of them
re-types the oracle's formula: they compare against closed forms, brute
force, exact rationals, textbook routines or invariants, chosen so that a
dropped term, a wrong sign/index or a transposed operand in the oracle fails
at least one of them.
"""

import itertools
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle as O

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def bf16_round(x):
    """Inputs of the method are bf16: round generated fp32 to bf16 (RNE)."""
    import torch
    return torch.from_numpy(np.asarray(x, np.float32)).bfloat16().double().numpy()


def rng(seed):
    return np.random.default_rng(seed)


# ---------------------------------------------------------------- P1 / P3
@pytest.mark.parametrize("n,d,causal", [(64, 16, False), (257, 64, False), (300, 64, True),
                                        (1024, 64, False), (200, 128, True)])
def test_p1_filters_off_equals_dense(n, d, causal):
    """P1 (north star): tau=1, theta=-1, lambda=-inf, no
    quantisation -> the full pipeline equals brute-force softmax attention."""
    g = rng(n + d)
    q, k, v = (bf16_round(g.standard_normal((n, d))) for _ in range(3))
    o, M, near, cnt, _ = O.spargeattn_head(q, k, v, 1.0, -1.0, -math.inf, causal=causal,
                                           quantize=False, pv_round=None)
    # brute force: per-row softmax with an explicit python loop over keys
    ref = np.empty_like(o)
    for r in range(n):
        keys = range(r + 1) if causal else range(n)
        s = np.array([q[r] @ k[c] / math.sqrt(d) for c in keys])
        p = np.exp(s - s.max())
        ref[r] = (p / p.sum()) @ v[list(keys)]
    assert np.max(np.abs(o - ref)) < 1e-12
    if causal:
        live = sum(O.causal_live(i, j, n, 128, 64) for i in range(M.shape[0])
                   for j in range(M.shape[1]))
        assert M.sum() == live
    else:
        assert M.all()


@pytest.mark.parametrize("n,d", [(257, 64), (512, 128)])
def test_p1_quantised_equals_dense_on_dequantised(n, d):
    """P1 (second half): with quantisation on, the filters-off pipeline
    equals dense attention on the dequantised Q^ delta_Q, K^ delta_K."""
    g = rng(7 * n)
    q, k, v = (bf16_round(g.standard_normal((n, d))) for _ in range(3))
    o, _, _, _, (Qq, dq, Kq, dk) = O.spargeattn_head(q, k, v, 1.0, -1.0, -math.inf,
                                                     quantize=True, pv_round=None)
    qd = Qq.astype(np.float64) * np.repeat(dq.astype(np.float64), 128)[:n, None]
    kd = Kq.astype(np.float64) * np.repeat(dk.astype(np.float64), 64)[:n, None]
    ref = O.dense_attention(qd, kd, v)
    assert np.max(np.abs(o - ref)) < 1e-12


def test_p3_masked_online_equals_two_pass_restricted():
    """P3: on any fixed mask with lambda=-inf the online
    recurrence equals a two-pass softmax restricted to the kept blocks."""
    n, d = 640, 32
    g = rng(3)
    q, k, v = (g.standard_normal((n, d)) for _ in range(3))
    tm, tn = 5, 10
    M = (g.random((tm, tn)) < 0.4).astype(np.uint8)
    M[np.arange(tm), g.integers(0, tn, tm)] = 1
    o, cnt = O.sparse_attention(q, k, v, M, -math.inf, quant=None, pv_round=None)
    S = q @ k.T / math.sqrt(d)
    keep = np.repeat(np.repeat(M.astype(bool), 128, 0), 64, 1)[:n, :n]
    S = np.where(keep, S, -np.inf)
    P = np.exp(S - S.max(1, keepdims=True))
    ref = (P / P.sum(1, keepdims=True)) @ v
    assert np.max(np.abs(o - ref)) < 1e-12
    assert cnt["qk"] == M.sum() and cnt["pv_slices"] == 4 * M.sum()


# ---------------------------------------------------------------- P2
@pytest.mark.parametrize("tau,expected", [(0.9, 14), (1.0, 16), (0.5, 8), (0.01, 1)])
def test_p2_uniform_closed_form(tau, expected):
    """P2 (north star): every Q token = q0 and every K token = k0.  Then
    sims = 1, S^ is constant, P^ = 1/T_n and, with the index tie-break, the
    kept set is {0..n_sel-1}, n_sel = max(1, #{k>=1 : k/T_n <= tau})
    (T_n=16, tau=.9 -> 14).  S is constant so every warp computes and O_i
    is the mean of V over the kept tokens."""
    n, d = 1024, 64
    g = rng(11)
    q0 = bf16_round(g.standard_normal(d))
    k0 = bf16_round(g.standard_normal(d))
    q = np.tile(q0, (n, 1))
    k = np.tile(k0, (n, 1))
    v = bf16_round(g.standard_normal((n, d)))
    tau = O.f32(tau)
    o, M, near, cnt, _ = O.spargeattn_head(q, k, v, tau, 0.5, -5.0)
    tn = 16
    n_sel = max(1, sum(1 for kk in range(1, tn + 1) if Fraction(kk, tn) <= Fraction(tau)))
    assert n_sel == expected
    want = np.zeros((8, 16), np.uint8)
    want[:, :n_sel] = 1
    assert (M == want).all()
    ref = v[: n_sel * 64].mean(axis=0)
    # P~ = 1 exactly in every kept tile, so bf16 rounding of P~ is exact
    assert np.max(np.abs(o - ref[None, :])) < 1e-12
    assert cnt["pv_slices"] == 4 * 8 * n_sel


def test_p2_causal_uniform_prefix_mean():
    """P2 causal variant (tau=1): with uniform Q/K, O_r = mean(V[0..r])."""
    n, d = 300, 32
    g = rng(5)
    q = np.tile(bf16_round(g.standard_normal(d)), (n, 1))
    k = np.tile(bf16_round(g.standard_normal(d)), (n, 1))
    v = bf16_round(g.standard_normal((n, d)))
    o, M, _, _, _ = O.spargeattn_head(q, k, v, 1.0, 0.5, -5.0, causal=True, pv_round=None)
    ref = np.cumsum(v, axis=0) / np.arange(1, n + 1)[:, None]
    assert np.max(np.abs(o - ref)) < 1e-12


# ---------------------------------------------------------------- P4
def test_p4_topcdf_exhaustive_rational():
    """P4: the fp64 sort+scan TopCdf equals the sort-free exact
    rational definition on every tiny map, except at exact-threshold hits,
    which it reports as near-threshold."""
    vals = [Fraction(0), Fraction(1, 10), Fraction(1, 5), Fraction(1, 4), Fraction(1, 2)]
    taus = [Fraction(3, 10), Fraction(1, 2), Fraction(4, 5), Fraction(9, 10), Fraction(1)]
    n_cases = n_near = 0
    for tn in range(1, 5):
        for row in itertools.product(vals, repeat=tn):
            if sum(row) == 0:
                continue
            p = np.array([float(x) for x in row])
            for tau in taus:
                exact = O.top_cdf_rational(row, tau)
                got, near = O.top_cdf(p, float(tau), near_tol=1e-9)
                n_cases += 1
                bad = [j for j in range(tn) if bool(got[j]) != exact[j]]
                if bad:
                    assert all(near[j] for j in bad), (row, tau, got, exact)
                    n_near += 1
    assert n_cases > 2000 and n_near < n_cases // 20


def test_p4_topcdf_spec_examples_and_golden():
    """S:L219-221 worked examples (hand traces of the paper's pseudocode)."""
    with open(os.path.join(GOLDEN, "topcdf_examples.json")) as f:
        cases = json.load(f)["cases"]
    for c in cases:
        got = O.top_cdf(np.array(c["p"]), c["tau"])
        assert got.astype(int).tolist() == c["mask"], c


def test_p4_topcdf_random_rows_monotone():
    """10,000 random rows agree with the rational definition, and
    the mask is monotone in tau."""
    g = rng(0)
    for t in range(10000):
        tn = int(g.integers(1, 9))
        num = g.integers(0, 6, tn)
        if num.sum() == 0:
            num[0] = 1
        row = [Fraction(int(x), int(num.sum())) for x in num]
        p = np.array([float(x) for x in row])
        tau = Fraction(int(g.integers(1, 11)), 10)
        got, near = O.top_cdf(p, float(tau), near_tol=1e-9)
        exact = O.top_cdf_rational(row, tau)
        for j in range(tn):
            assert got[j] == exact[j] or near[j]
        lo = O.top_cdf(p, 0.3)
        hi = O.top_cdf(p, 0.95)
        assert np.all(lo <= hi)


# ---------------------------------------------------------------- P5
def test_p5_cossim_examples():
    """identical unit rows -> 1.0; two orthonormal rows -> 0.5,
    under both readings; an all-zero block -> 1.0."""
    e = np.eye(4)
    for mode in ("cosine", "literal"):
        assert O.cos_sim(np.tile(e[1], (5, 1)), mode) == pytest.approx(1.0, abs=1e-15)
        assert O.cos_sim(e[:2], mode) == pytest.approx(0.5, abs=1e-15)
        assert O.cos_sim(np.zeros((3, 4)), mode) == 1.0


def test_p5_cossim_closed_forms():
    """The literal Gram mean equals the O(nd) closed forms
    ||sum_a x^_a||^2 / n^2 (R1-A) and ||sum x||^2 / (n^2 max_a ||x_a||^2)
    (R1-B, max(XX^T) is on the diagonal by Cauchy-Schwarz)."""
    g = rng(1)
    for n, d in [(64, 64), (128, 128), (37, 16)]:
        X = g.standard_normal((n, d)) + 0.7 * g.standard_normal(d)
        X[3] = 0.0
        norms = np.linalg.norm(X, axis=1)
        Xn = np.where(norms[:, None] > 0, X / np.where(norms > 0, norms, 1)[:, None], 0)
        a = np.linalg.norm(Xn.sum(0)) ** 2 / n ** 2
        b = np.linalg.norm(X.sum(0)) ** 2 / (n ** 2 * np.max(norms ** 2))
        assert O.cos_sim(X, "cosine") == pytest.approx(a, rel=1e-12)
        assert O.cos_sim(X, "literal") == pytest.approx(b, rel=1e-12)


def test_p5_planted_block_expectation():
    """Planted tokens x = c + s*eps: E[CosSim] ~ 1/n + (1-1/n) a^2/(a^2+s^2)."""
    g = rng(2)
    n, d, s = 64, 128, 0.5
    vals = [O.cos_sim(g.standard_normal(d)[None, :] + s * g.standard_normal((n, d)))
            for _ in range(20)]
    assert np.mean(vals) == pytest.approx(1 / n + (1 - 1 / n) / (1 + s * s), abs=0.02)


# ---------------------------------------------------------------- P6
def test_p6_quant_examples():
    """zero block -> delta=1, q=0; a constant block 2.54 ->
    delta = 2.54/127 = 0.02, every q = 127."""
    q, dl = O.quantize_blocks(np.zeros((64, 8)), 64)
    assert (q == 0).all() and dl[0] == 1.0
    x = np.full((64, 8), 2.54)
    q, dl = O.quantize_blocks(x, 64)
    assert (q == 127).all()
    assert float(dl[0]) == pytest.approx(0.02, rel=1e-6)


def test_p6_quant_error_bound_and_textbook():
    """|x - q delta| <= delta/2 (+fp32 eps), q in [-127,127], and
    q equals the textbook round(x * 127 / amax) except on exact half-ties."""
    g = rng(4)
    x = bf16_round(g.standard_normal((300, 64)) * 3)
    q, dl = O.quantize_blocks(x, 128)
    for i in range(3):
        blk = x[i * 128:(i + 1) * 128]
        qb = q[i * 128:(i + 1) * 128].astype(np.float64)
        dd = float(dl[i])
        assert np.max(np.abs(blk - qb * dd)) <= dd / 2 * (1 + 1e-5) + 1e-7
        amax = np.max(np.abs(blk))
        tb = np.round(blk * 127.0 / amax)  # fp64 textbook
        frac = np.abs(blk * 127.0 / amax - np.trunc(blk * 127.0 / amax))
        ok = (tb == qb) | (np.abs(frac - 0.5) < 1e-5)
        assert ok.all()
        assert np.abs(qb).max() == 127


# ---------------------------------------------------------------- P7
def test_p7_gate_examples():
    """a tile whose scores are 100 below the running max skips at
    lambda=-50; lambda=-inf computes; a tile that sets a fresh max computes."""
    n, d = 128, 16
    q = np.zeros((n, d)); q[:, 0] = 1.0
    k = np.zeros((n, d)); v = np.ones((n, d))
    k[:64, 0] = 400.0       # block 0: S = 100
    k[64:, 0] = 0.0         # block 1: S = 0 -> 100 below the max
    M = np.ones((1, 2), np.uint8)
    _, cnt = O.sparse_attention(q, k, v, M, -50.0, bq=128, bk=64, quant=None)
    assert cnt["pv_slices"] == 4            # block 1 skipped by all 4 warps
    _, cnt = O.sparse_attention(q, k, v, M, -math.inf, bq=128, bk=64, quant=None)
    assert cnt["pv_slices"] == 8
    k2 = k.copy(); k2[:64, 0] = 0.0; k2[64:, 0] = 400.0   # fresh max in block 1
    _, cnt = O.sparse_attention(q, k2, v, M, -50.0, bq=128, bk=64, quant=None)
    assert cnt["pv_slices"] == 8


@pytest.mark.parametrize("lam,bound", [(-10.0, 1e-3), (-20.0, 1e-6)])
def test_p7_gate_soundness(lam, bound):
    """S:L466 / §3.4: with an all-ones mask, the gated output differs
    from the ungated by < 1e-3 at lambda=-10 and < 1e-6 at -20; the analytic
    per-row bound is b_k e^lambda of dropped mass per skipped tile."""
    n, d = 1024, 64
    g = rng(9)
    u = g.standard_normal(d)
    u *= 8.0 / np.linalg.norm(u)
    q = u[None, :] + 0.3 * g.standard_normal((n, d))
    k = g.standard_normal((n, d))
    # k-block 0 is strongly aligned with every query (S ~ 20-28), so once it
    # has set the running max, most later tiles sit below it by > |lambda|
    k[:64] = u[None, :] * g.uniform(2.5, 3.5, (64, 1))
    v = g.standard_normal((n, d))
    M = np.ones((8, 16), np.uint8)
    a, ca = O.sparse_attention(q, k, v, M, lam, quant=None, pv_round=None)
    b, cb = O.sparse_attention(q, k, v, M, -math.inf, quant=None, pv_round=None)
    assert O.relative_l1(a, b) < bound
    assert ca["pv_slices"] < cb["pv_slices"]      # the gate actually fired
    skipped_tiles = 16
    assert np.max(np.abs(a - b)) <= skipped_tiles * 64 * math.exp(lam) * np.max(np.abs(v)) * 2


# ---------------------------------------------------------------- P8
def test_p8_counter_hand_counts():
    """t_m=t_n=2, one tile mask-skipped, one lambda-skip -> 0.375;
    t_m=2, t_n=4 with only the guard block kept per row -> 0.75."""
    assert O.sparsity_of(qk_exec=3, pv_slices_exec=2 * 4, live_tiles=4) == pytest.approx(0.375)
    assert O.sparsity_of(qk_exec=2, pv_slices_exec=2 * 4, live_tiles=8) == pytest.approx(0.75)


# ---------------------------------------------------------------- P10
def test_p10_degenerate():
    """n=1 -> O = V; identical K rows -> O = mean V;
    n = b_q = b_k -> sparse equals dense for any tau (one block, the guard)."""
    g = rng(6)
    d = 32
    q, k, v = (g.standard_normal((1, d)) for _ in range(3))
    o, *_ = O.spargeattn_head(q, k, v, 0.5, 0.5, -5.0, quantize=False, pv_round=None)
    assert np.allclose(o, v, atol=1e-15)
    n = 200
    q = g.standard_normal((n, d)); k = np.tile(g.standard_normal(d), (n, 1))
    v = g.standard_normal((n, d))
    o, *_ = O.spargeattn_head(q, k, v, 1.0, -1.0, -math.inf, quantize=False, pv_round=None)
    assert np.max(np.abs(o - v.mean(0))) < 1e-12
    n = 64
    q, k, v = (g.standard_normal((n, d)) for _ in range(3))
    for tau in (0.1, 0.5, 0.99):
        o, *_ = O.spargeattn_head(q, k, v, tau, 0.3, -math.inf, bq=64, bk=64,
                                  quantize=False, pv_round=None)
        assert np.max(np.abs(o - O.dense_attention(q, k, v))) < 1e-12


# ---------------------------------------------------------------- P11
@pytest.mark.parametrize("causal", [False, True])
def test_p11_mask_invariants(causal):
    """S:L234-235 forcing completeness and row non-emptiness; R8 causal
    guard -> every valid row has l > 0 (no OracleInvariantError)."""
    g = rng(12)
    n, d = 1100, 64
    base = g.standard_normal((18, d))
    q = np.repeat(base, 64, 0)[:n] + 0.3 * g.standard_normal((n, d))
    k = np.repeat(base[::-1], 64, 0)[:n] + 0.3 * g.standard_normal((n, d))
    q[256:384] = g.standard_normal((128, d))        # non-self-similar Q block 2
    k[640:704] = g.standard_normal((64, d))         # non-self-similar K block 10
    v = g.standard_normal((n, d))
    M, near, st = O.predict_mask(q, k, 0.5, 0.5, causal=causal, return_stats=True)
    assert st["s_q"][2] < 0.5 and st["s_k"][10] < 0.5
    tm, tn = M.shape
    live = np.array([[O.causal_live(i, j, n, 128, 64) or not causal for j in range(tn)]
                     for i in range(tm)])
    assert (M[2][live[2]] == 1).all()
    assert (M[:, 10][live[:, 10]] == 1).all()
    assert (M.sum(1) >= 1).all()
    assert not (M.astype(bool) & ~live).any()
    o, _ = O.sparse_attention(q, k, v, M, -5.0, causal=causal, quant=None)
    assert np.isfinite(o).all()


def test_p11_causal_guard_prevents_empty_rows():
    """R8-iii: without the diagonal guard, q-block 1 keeping only k-block 3
    leaves rows 128..191 with no valid key (l = 0)."""
    n, d = 256, 8
    g = rng(8)
    q, k, v = (g.standard_normal((n, d)) for _ in range(3))
    M = np.zeros((2, 4), np.uint8); M[0, 0] = 1; M[1, 3] = 1
    with pytest.raises(O.OracleInvariantError):
        O.sparse_attention(q, k, v, M, -math.inf, causal=True, quant=None)
    M[1, 2] = 1   # the guard block floor(1*128/64) = 2
    o, _ = O.sparse_attention(q, k, v, M, -math.inf, causal=True, quant=None)
    assert np.isfinite(o).all()


# ---------------------------------------------------------------- sanity of the map
def test_compressed_map_softmax_and_masking():
    """uniform row -> uniform; row [0,-inf] -> [1,0]; rows sum to
    1; S^ uses 1/sqrt(d) (R2): compare with an explicit scalar loop."""
    g = rng(10)
    qbar = g.standard_normal((3, 16)); kbar = g.standard_normal((5, 16))
    s_k = np.array([0.9, 0.1, 0.9, 0.9, 0.9])
    S, P, fl = O.compressed_map(qbar, kbar, s_k, 0.5, 5 * 64, 128, 64)
    for i in range(3):
        for j in range(5):
            want = -np.inf if j == 1 else sum(qbar[i, c] * kbar[j, c] for c in range(16)) / 4.0
            assert S[i, j] == pytest.approx(want, rel=1e-13) if j != 1 else S[i, j] == want
        assert P[i].sum() == pytest.approx(1.0, abs=1e-15)
        assert P[i, 1] == 0.0
    S, P, fl = O.compressed_map(np.zeros((1, 4)), np.ones((2, 4)), np.array([1.0, 0.0]),
                                0.5, 128, 128, 64)
    assert P[0].tolist() == [1.0, 0.0]
