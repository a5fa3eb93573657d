"""Scope row f3: the token orders of App. A.2 (Table 13) on the
CPU -- bijections, their definitions enumerated by hand on tiny grids, and the
locality that makes them differ."""

import numpy as np
import pytest

from paper_2502_18137_b200 import permutations as P


@pytest.mark.parametrize("kind", P.KINDS)
@pytest.mark.parametrize("T,H,W,pre", [(2, 3, 4, 0), (3, 5, 2, 7), (1, 6, 6, 0)])
def test_bijection_and_text_prefix(kind, T, H, W, pre):
    perm = P.make_perm(kind, T, H, W, pre, seed=3)
    L = pre + T * H * W
    assert perm.dtype == np.int32 and perm.shape == (L,)
    assert np.array_equal(np.sort(perm), np.arange(L))
    assert np.array_equal(perm[:pre], np.arange(pre))        # text stays put
    inv = P.inverse(perm)
    assert np.array_equal(inv[perm], np.arange(L))


def test_orders_by_enumeration():
    T, H, W, pre = 2, 3, 4, 5
    def src(t, h, w):
        return pre + (t * H + h) * W + w
    row = [src(t, h, w) for t in range(T) for h in range(H) for w in range(W)]
    col = [src(t, h, w) for t in range(T) for w in range(W) for h in range(H)]
    tim = [src(t, h, w) for h in range(H) for w in range(W) for t in range(T)]
    assert list(P.make_perm("rowmajor", T, H, W, pre)[pre:]) == row
    assert list(P.make_perm("columnmajor", T, H, W, pre)[pre:]) == col
    assert list(P.make_perm("timemajor", T, H, W, pre)[pre:]) == tim


def test_continuity_axes():
    """Consecutive positions differ by one step along W (rowmajor), H
    (columnmajor), T (timemajor) most of the time, per Table 13."""
    T, H, W = 4, 5, 6
    def coords(i):
        return np.stack([i // (H * W), (i // W) % H, i % W], 1)
    for kind, axis in (("rowmajor", 2), ("columnmajor", 1), ("timemajor", 0)):
        c = coords(P.make_perm(kind, T, H, W).astype(np.int64))
        steps = np.abs(np.diff(c, axis=0))
        along = (steps[:, axis] == 1) & (steps.sum(1) == 1)
        assert along.mean() > 0.7, (kind, along.mean())
    with pytest.raises(ValueError):
        P.make_perm("zigzag", 2, 2, 2)
