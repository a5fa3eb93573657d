"""Pins of the oracle's FP8 P~V path (scope row f4, SageAttention2-style,
footnote P:L44; reading R27) against things other than itself: the FP8 E4M3
format as torch implements it (a library routine), exact closed forms, and
the size of the error the format can introduce."""

import math

import numpy as np
import pytest
import torch

import oracle as O


def _e4m3_grid():
    codes = torch.arange(256, dtype=torch.uint8).view(torch.float8_e4m3fn)
    vals = codes.to(torch.float64).numpy()
    return np.unique(vals[np.isfinite(vals)])


def test_every_e4m3_value_is_a_fixed_point():
    g = _e4m3_grid()
    assert g.max() == 448.0 and g.min() == -448.0 and (g == 0).any()
    assert len(g) == 253                      # 254 finite codes, +0 and -0 merged
    assert np.array_equal(O.round_e4m3(g), g)


def test_rounding_matches_torch_including_ties():
    g = _e4m3_grid()
    g = g[g >= 0]
    mids = (g[:-1] + g[1:]) / 2               # exact ties: round half to even
    rng = np.random.default_rng(0)
    rnd = rng.uniform(-448, 448, 20000) * np.exp2(rng.integers(-14, 1, 20000))
    for x in (mids, -mids, rnd):
        ref = torch.from_numpy(x.astype(np.float32)).to(torch.float8_e4m3fn).to(torch.float64).numpy()
        assert np.array_equal(O.round_e4m3(x.astype(np.float32).astype(np.float64)), ref)


def test_saturation_and_subnormals():
    assert O.round_e4m3(np.array([1000.0, -500.0, 464.0, 470.0]))[:2].tolist() == [448.0, -448.0]
    assert O.round_e4m3(np.array([464.0]))[0] == 448.0          # tie -> even mantissa 1.75
    assert O.round_e4m3(np.array([2.0 ** -9, 2.0 ** -10, 3 * 2.0 ** -11]))[0] == 2.0 ** -9
    assert O.round_e4m3(np.array([2.0 ** -10]))[0] == 0.0        # tie -> 0 (even)
    assert O.round_e4m3(np.array([3 * 2.0 ** -11]))[0] == 2.0 ** -9


def test_v_quant_scales():
    V = np.array([[1.0, 0.0, -3.5], [0.5, 0.0, 7.0]])
    Vh, s = O.fp8_v_quant(V)
    assert s.dtype == np.float32
    assert s[1] == 1.0 and (Vh[:, 1] == 0).all()               # zero column
    assert np.all(np.abs(Vh) <= 448.0)
    assert Vh[0, 0] == 448.0 and Vh[1, 2] == 448.0             # column maxima map to 448
    np.testing.assert_allclose(Vh * s.astype(np.float64), V, rtol=0.0625)


@pytest.mark.parametrize("amax", [448.0, 56.0])
def test_fp8_path_closed_form(amax):
    """Uniform Q, K: every key has P~ = 1 (exact in E4M3 after x128); V on
    the E4M3 grid scaled so that 448/amax is a power of two: V^ is exact,
    and O = the mean of V over the kept keys, exactly (P2 of §4 on the f4
    path)."""
    N, d = 384, 64
    rng = np.random.default_rng(1)
    g = _e4m3_grid()
    g = g[np.abs(g) <= 448.0]
    V = rng.choice(g, size=(N, d)) * (amax / 448.0)
    V[0, :] = amax                                  # column maxima exactly amax
    q = np.ones((N, d))
    k = np.ones((N, d))
    o, M, near, cnt, _ = O.spargeattn_head(q, k, V, O.f32(1.0), O.f32(-1.0), O.f32(-math.inf),
                                           pv_round="fp8")
    assert M.all()
    np.testing.assert_allclose(o, np.broadcast_to(V.mean(axis=0), (N, d)), rtol=1e-13, atol=1e-13)


def test_fp8_path_error_is_format_sized():
    """On Gaussian data the FP8 P~V output stays within the E4M3 format's
    error of the bf16 path (3 mantissa bits: relative L1 a few 1e-2 at most)."""
    rng = np.random.default_rng(2)
    N, d = 512, 64
    q, k, v = (rng.standard_normal((N, d)) for _ in range(3))
    o8, *_ = O.spargeattn_head(q, k, v, O.f32(0.9), O.f32(0.5), O.f32(-5.0), pv_round="fp8")
    ob, *_ = O.spargeattn_head(q, k, v, O.f32(0.9), O.f32(0.5), O.f32(-5.0), pv_round="bf16")
    err = O.relative_l1(o8, ob)
    assert 1e-4 < err < 0.05, err
