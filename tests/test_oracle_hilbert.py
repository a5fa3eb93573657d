"""P9: the oracle's Hilbert permutation against what a Hilbert curve and
attention fix (§3.7; App. A.1).  CPU only."""

import math

import numpy as np
import pytest

import oracle as O


def unit_step_fraction(cells):
    a = np.array(cells)
    return float((np.abs(np.diff(a, axis=0)).sum(1) == 1).mean())


@pytest.mark.parametrize("T,H,W", [(8, 8, 8), (1, 6, 6), (13, 30, 45), (28, 30, 53),
                                   (1, 1, 4), (1, 2, 2), (3, 5, 7), (2, 64, 64)])
def test_bijection_and_inverse(T, H, W):
    for prefix in (0, 226):
        perm, inv = O.hilbert_permutation(T, H, W, prefix)
        n = prefix + T * H * W
        assert sorted(perm.tolist()) == list(range(n))
        assert (perm[inv] == np.arange(n)).all() and (inv[perm] == np.arange(n)).all()
        assert (perm[:prefix] == np.arange(prefix)).all()   # text tokens stay


def test_locality_power_of_two_cube_is_perfect():
    """S:L380 / S:L471: on power-of-two cubes every consecutive pair is a
    unit grid step (the defining property of a Hilbert curve)."""
    for s in (2, 4, 8, 16):
        assert unit_step_fraction(O.gilbert3d(s, s, s)) == 1.0


def test_locality_fig5_geometry():
    """Fig. 5 1x6x6 example: >= 95% unit steps."""
    assert unit_step_fraction(O.gilbert3d(6, 6, 1)) >= 0.95


def test_locality_video_grids():
    """The C3/C4 latent grids keep >= 95% unit steps."""
    assert unit_step_fraction(O.gilbert3d(45, 30, 13)) >= 0.95
    assert unit_step_fraction(O.gilbert3d(53, 30, 28)) >= 0.95


def test_trivial_grids_identity():
    """dims (1,1,4) -> identity; (1,2,2) -> a connected unit-step path."""
    perm, _ = O.hilbert_permutation(1, 1, 4)
    assert perm.tolist() == [0, 1, 2, 3]
    cells = O.gilbert3d(2, 2, 1)
    assert unit_step_fraction(cells) == 1.0 and cells[0] == (0, 0, 0)


def test_curve_starts_at_origin_major_axis_largest():
    """Reading R19: the curve starts at (0,0,0) and first moves along the
    largest extent's half-box."""
    cells = O.gilbert3d(8, 2, 2)
    assert cells[0] == (0, 0, 0)


def test_attention_permutation_invariance():
    """§3.7 "attention is computationally invariant to token
    permutations": inverse_permute(attn(perm Q, perm K, perm V)) = attn(Q,K,V)."""
    g = np.random.default_rng(0)
    perm, inv = O.hilbert_permutation(2, 6, 6, 10)
    n, d = perm.size, 16
    q, k, v = (g.standard_normal((n, d)) for _ in range(3))
    ref = O.dense_attention(q, k, v)
    got = O.dense_attention(q[perm], k[perm], v[perm])[inv]
    assert O.relative_l1(got, ref) < 1e-12


def test_smooth_field_hilbert_beats_rowmajor_direction():
    """Directional Table 6: on a smooth 3-D field, blocks of
    Hilbert-ordered tokens are more self-similar than row-major blocks."""
    g = np.random.default_rng(1)
    T, H, W, d = 4, 16, 16, 32
    t, h, w = np.meshgrid(np.arange(T), np.arange(H), np.arange(W), indexing="ij")
    # the same smoothness per grid step on every axis, as in a video latent
    coords = np.stack([t.ravel(), h.ravel(), w.ravel()], 1) / 16.0
    feats = np.zeros((T * H * W, d))
    for _ in range(8):
        f = g.standard_normal(3) * 3.0
        ph = g.uniform(0, 2 * math.pi)
        feats += np.cos(coords @ f + ph)[:, None] * g.standard_normal(d)[None, :]
    perm, _ = O.hilbert_permutation(T, H, W)
    sim_h = O.block_sims(feats[perm], 64).mean()
    sim_r = O.block_sims(feats, 64).mean()
    assert sim_h > sim_r, (sim_h, sim_r)
