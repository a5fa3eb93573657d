"""Pins of the oracle's K smoothing (scope row f4, SageAttention-style
"smooth K", footnote P:L44; reading R28) against things other than itself:
the exact token mean, the shift invariance of softmax attention (a closed-form
property of the definition), the size of the INT8 error it removes, and
stage 1's independence of it (R14)."""

import numpy as np

import oracle as O
from paper_2502_18137_b200 import inputs


def _rng(seed=0):
    return np.random.default_rng(seed)


def test_mean_is_the_exact_mean_to_fp32_rounding():
    for n, d, seed in [(1, 64, 0), (127, 64, 1), (128, 128, 2), (1000, 128, 3)]:
        k = _rng(seed).standard_normal((n, d)) * 3.0 + _rng(seed + 9).standard_normal(d)
        k = O.round_bf16(k)
        mu = O.smooth_k_mean(k).astype(np.float64)
        exact = np.array([float(sum(map(__import__("fractions").Fraction, k[:, c]))) / n
                          for c in range(d)])
        # one fp32 rounding of a value whose fp64 sum error is ~1e-16 relative
        ulp = np.spacing(np.abs(exact).astype(np.float32)).astype(np.float64)
        assert np.all(np.abs(mu - exact) <= ulp)


def test_smoothed_k_is_fp32_difference():
    k = O.round_bf16(_rng(4).standard_normal((200, 64)))
    mu = O.smooth_k_mean(k)
    ks = O.smooth_k(k, mu)
    assert np.array_equal(ks, (k.astype(np.float32) - mu).astype(np.float64))
    # a zero mean leaves K (as fp32) unchanged
    assert np.array_equal(O.smooth_k(k, np.zeros(64, np.float32)), k.astype(np.float32))


def test_unquantised_attention_is_shift_invariant():
    """softmax(q (k - mu)^T) = softmax(q k^T): the definition of smoothing
    does not change attention -- checked on brute-force dense attention."""
    rng = _rng(5)
    n, d = 300, 64
    q, v = (rng.standard_normal((n, d)) for _ in range(2))
    k = O.round_bf16(rng.standard_normal((n, d)) + 3.0)
    # the exact difference K - mu (bf16 minus fp32 is exact in fp64); the
    # smoothed operand fl32(K - mu) differs from it by one fp32 rounding
    mu = O.smooth_k_mean(k).astype(np.float64)
    ks = k - mu
    assert np.abs(O.smooth_k(k, O.smooth_k_mean(k)) - ks).max() <= 4 * np.spacing(np.float32(4.0))
    for causal in (False, True):
        a = O.dense_attention(q, k, v, causal)
        b = O.dense_attention(q, ks, v, causal)
        assert np.abs(a - b).max() < 1e-12


def test_smoothing_removes_the_channel_offset_error():
    """K with a large per-channel offset: per-block INT8 of K loses the
    token-to-token differences, INT8 of K - mu keeps them."""
    rng = _rng(6)
    n, d = 512, 64
    q = rng.standard_normal((n, d))
    k0 = rng.standard_normal((n, d))
    k = O.round_bf16(k0 + 12.0 * rng.standard_normal(d))       # offset >> spread
    v = rng.standard_normal((n, d))
    ref = O.dense_attention(q, k, v)
    common = dict(tau=1.0, theta=-1.0, lam=-np.inf)
    o_plain = O.spargeattn_head(q, k, v, **common)[0]
    o_smooth = O.spargeattn_head(q, k, v, smooth=True, **common)[0]
    e_plain, e_smooth = O.relative_l1(o_plain, ref), O.relative_l1(o_smooth, ref)
    assert e_smooth < 0.25 * e_plain, (e_smooth, e_plain)


def test_stage1_ignores_smoothing():
    """R14: masks (and near-threshold flags) are the same with and without
    smoothing -- stage 1 reads the raw K."""
    q, k, v = (a[0, 0].astype(np.float64) for a in inputs.planted(0))
    a = O.spargeattn_head(q, k, v, 0.9, 0.5, -5.0)
    b = O.spargeattn_head(q, k, v, 0.9, 0.5, -5.0, smooth=True)
    assert np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2])
    assert a[3] == b[3]
    # O stays within the INT8 error level of the unsmoothed path
    c = O.spargeattn_head(q, k, v, 0.9, 0.5, -5.0, quantize=False)
    e_a, e_b = O.relative_l1(a[0], c[0]), O.relative_l1(b[0], c[0])
    assert e_b < 1.5 * e_a + 1e-3, (e_a, e_b)
