"""Scope row f2 (§3.6 hyper-parameter search): the selection
logic on the CPU, against brute force over the grid and against the oracle
as the evaluator (no GPU)."""

import itertools
import math

import numpy as np
import pytest

import oracle as O
from paper_2502_18137_b200 import tuner


def _analytic(tau, theta, lam):
    """A smooth stand-in evaluator: error grows and density falls as tau
    drops, theta rises and lambda approaches 0."""
    th = 0.0 if theta <= -1 else theta + 1.0
    lg = 0.0 if lam == -math.inf else 1.0 / (-lam)
    err = 0.1 * (1 - tau) + 0.01 * th + 0.05 * lg
    sp = 0.6 * (1 - tau) + 0.05 * th + 0.2 * lg
    return err, sp


def test_select_stage1_ties_and_infeasible():
    rows = [(0.9, 0.2, 0.01, 0.3), (0.95, 0.2, 0.01, 0.3), (0.95, 0.4, 0.01, 0.3),
            (0.5, 0.8, 0.2, 0.9)]
    assert tuner.select_stage1(rows, 0.05) == (0.95, 0.4, 0.01, 0.3)   # larger tau, then theta
    assert tuner.select_stage1(rows, 0.005) is None
    # strict bound: L1 equal to l1 is infeasible
    assert tuner.select_stage1([(0.9, 0.0, 0.05, 0.5)], 0.05) is None


def test_select_stage2_prefers_more_negative_lambda_on_ties():
    rows = [(-math.inf, 0.01, 0.3), (-10.0, 0.02, 0.35), (-5.0, 0.03, 0.35), (-4.0, 0.2, 0.5)]
    assert tuner.select_stage2(rows, 0.06) == (-10.0, 0.02, 0.35)


def test_tune_layer_matches_brute_force():
    l1, l2 = 0.05, 0.06
    res = tuner.tune_layer(_analytic, l1, l2)
    feas = [(t, th) for t, th in itertools.product(tuner.DEFAULT_TAU_GRID, tuner.DEFAULT_THETA_GRID)
            if _analytic(t, th, -math.inf)[0] < l1]
    best_sp = max(_analytic(t, th, -math.inf)[1] for t, th in feas)
    assert res["sparsity_stage1"] == pytest.approx(best_sp)
    assert res["l1_stage1"] < l1 and res["l1_stage2"] < l2
    lam_feas = [lm for lm in tuner.DEFAULT_LAMBDA_GRID
                if _analytic(res["tau"], res["theta"], lm)[0] < l2]
    assert res["sparsity"] == pytest.approx(
        max(_analytic(res["tau"], res["theta"], lm)[1] for lm in lam_feas))
    assert res["sparsity"] >= res["sparsity_stage1"]
    assert not res["fallback"]


def test_tune_layer_monotone_in_l1_and_fallback():
    prev = -1.0
    for l1 in (0.005, 0.01, 0.02, 0.04, 0.08):
        res = tuner.tune_layer(_analytic, l1, l1 + 0.01)
        assert res["sparsity_stage1"] >= prev - 1e-12      # feasible set only grows
        prev = res["sparsity_stage1"]
    # nothing feasible (no dense config in the grid) -> dense fallback, flagged
    res = tuner.tune_layer(_analytic, 1e-4, 2e-4, tau_grid=(0.5,), theta_grid=(0.8,))
    assert res["fallback"] and res["tau"] == 1.0 and res["lambda"] == -math.inf
    with pytest.raises(ValueError):
        tuner.tune_layer(_analytic, 0.06, 0.05)


def test_tune_layer_with_the_oracle_as_evaluator():
    """End to end on the CPU: the oracle (quantised sparse Algorithm 1 vs the
    dense fp64 reference) scores the candidates.  Inputs with one dominant
    key block per query block: the tuner must find tau < 1 with
    positive sparsity, and the returned triple satisfies both bounds when
    re-evaluated."""
    N, d = 512, 64
    cal = []
    for seed in range(3):
        g = np.random.default_rng(seed)
        c = g.standard_normal((N // 64, d))     # one centre per key block
        k = np.repeat(c, 64, axis=0) + 0.5 * g.standard_normal((N, d))
        q = 0.5 * g.standard_normal((N, d))
        for i in range(N // 128):               # q block i attends to k block 2i+1
            q[i * 128:(i + 1) * 128] += 0.45 * c[2 * i + 1]
        v = g.standard_normal((N, d))
        cal.append((q, k, v, O.dense_attention(q, k, v)))

    def evaluate(tau, theta, lam):
        errs, sps = [], []
        for q, k, v, ref in cal:
            o, M, near, cnt, _ = O.spargeattn_head(q, k, v, O.f32(tau), O.f32(theta), O.f32(lam),
                                                   pv_round=None)
            errs.append(O.relative_l1(o, ref))
            sps.append(O.sparsity_of(cnt["qk"], cnt["pv_slices"], M.size))
        return max(errs), float(np.mean(sps))

    grid = dict(tau_grid=(0.5, 0.9, 0.95, 0.98, 0.99, 1.0), theta_grid=(-1.0, 0.5),
                lambda_grid=(-math.inf, -5.0))
    res = tuner.tune_layer(evaluate, 0.05, 0.06, **grid)
    assert not res["fallback"] and res["tau"] < 1.0 and res["sparsity"] > 0.1
    # brute force over the same grid: no feasible pair is sparser
    best = max(sp for t, th, e, sp in res["scan_stage1"] if e < 0.05)
    assert res["sparsity_stage1"] == best
    err, sp = evaluate(res["tau"], res["theta"], res["lambda"])
    assert err < 0.06 and sp == pytest.approx(res["sparsity"])


def test_live_tiles_matches_definition():
    for N, causal in ((1000, True), (1000, False), (64, True), (4096, True)):
        tm, tn = -(-N // 128), -(-N // 64)
        brute = sum(1 for i in range(tm) for j in range(tn)
                    if not causal or j * 64 <= min((i + 1) * 128, N) - 1)
        assert tuner.live_tiles(N, causal) == brute
