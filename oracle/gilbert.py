"""Oracle Hilbert-curve permutation (TEST INFRASTRUCTURE ONLY; see oracle/__init__).

Paper: §3.7 "HilbertCurve Permutation": "We use the Hilbert Curve
to fill the 3D space and then flatten tokens along the curve into shape
R^{L x d}, L = T x H x W"; App. A.1: the inverse permutation is
applied to the attention output and, for joint text+visual attention, "we
only permute the visual tokens".

The paper does not say which construction it uses for extents that are not
powers of two (its own Fig. 5 example is 1x6x6).  Reading R19:
the generalised Hilbert curve ("gilbert3d", J. Cervený), started at the
origin with the largest extent as the major axis.  This file is an
independent, recursive transcription of that construction; the product's
C++ ``hilbert_permute`` is a separate implementation and the two are pinned
to each other by integer equality, and each to the locality properties of a
Hilbert curve (tests/test_oracle_hilbert.py).
"""

import numpy as np

__all__ = ["gilbert3d", "hilbert_permutation"]


def _sgn(v):
    return (v > 0) - (v < 0)


def _gen3d(out, x, y, z, ax, ay, az, bx, by, bz, cx, cy, cz):
    """Fill the box spanned by vectors a (major), b, c starting at (x,y,z)."""
    w = abs(ax + ay + az)
    h = abs(bx + by + bz)
    d = abs(cx + cy + cz)
    dax, day, daz = _sgn(ax), _sgn(ay), _sgn(az)
    dbx, dby, dbz = _sgn(bx), _sgn(by), _sgn(bz)
    dcx, dcy, dcz = _sgn(cx), _sgn(cy), _sgn(cz)

    # Degenerate boxes: a straight line along the only non-unit axis.
    if h == 1 and d == 1:
        for _ in range(w):
            out.append((x, y, z))
            x, y, z = x + dax, y + day, z + daz
        return
    if w == 1 and d == 1:
        for _ in range(h):
            out.append((x, y, z))
            x, y, z = x + dbx, y + dby, z + dbz
        return
    if w == 1 and h == 1:
        for _ in range(d):
            out.append((x, y, z))
            x, y, z = x + dcx, y + dcy, z + dcz
        return

    ax2, ay2, az2 = ax // 2, ay // 2, az // 2
    bx2, by2, bz2 = bx // 2, by // 2, bz // 2
    cx2, cy2, cz2 = cx // 2, cy // 2, cz // 2
    w2 = abs(ax2 + ay2 + az2)
    h2 = abs(bx2 + by2 + bz2)
    d2 = abs(cx2 + cy2 + cz2)

    # Prefer even half-lengths so that the sub-curves can chain by unit steps.
    if (w2 % 2) and (w > 2):
        ax2, ay2, az2 = ax2 + dax, ay2 + day, az2 + daz
    if (h2 % 2) and (h > 2):
        bx2, by2, bz2 = bx2 + dbx, by2 + dby, bz2 + dbz
    if (d2 % 2) and (d > 2):
        cx2, cy2, cz2 = cx2 + dcx, cy2 + dcy, cz2 + dcz

    if (2 * w > 3 * h) and (2 * w > 3 * d):
        # Long box: split the major axis only.
        _gen3d(out, x, y, z, ax2, ay2, az2, bx, by, bz, cx, cy, cz)
        _gen3d(out, x + ax2, y + ay2, z + az2,
               ax - ax2, ay - ay2, az - az2, bx, by, bz, cx, cy, cz)
    elif 3 * h > 4 * d:
        # Flat in c: split a and b, keep c whole.
        _gen3d(out, x, y, z, bx2, by2, bz2, cx, cy, cz, ax2, ay2, az2)
        _gen3d(out, x + bx2, y + by2, z + bz2,
               ax, ay, az, bx - bx2, by - by2, bz - bz2, cx, cy, cz)
        _gen3d(out, x + (ax - dax) + (bx2 - dbx),
               y + (ay - day) + (by2 - dby),
               z + (az - daz) + (bz2 - dbz),
               -bx2, -by2, -bz2, cx, cy, cz,
               -(ax - ax2), -(ay - ay2), -(az - az2))
    elif 3 * d > 4 * h:
        # Flat in b: split a and c, keep b whole.
        _gen3d(out, x, y, z, cx2, cy2, cz2, ax2, ay2, az2, bx, by, bz)
        _gen3d(out, x + cx2, y + cy2, z + cz2,
               ax, ay, az, bx, by, bz, cx - cx2, cy - cy2, cz - cz2)
        _gen3d(out, x + (ax - dax) + (cx2 - dcx),
               y + (ay - day) + (cy2 - dcy),
               z + (az - daz) + (cz2 - dcz),
               -cx2, -cy2, -cz2, -(ax - ax2), -(ay - ay2), -(az - az2),
               bx, by, bz)
    else:
        # Regular box: split all three axes into the eight-octant pattern.
        _gen3d(out, x, y, z, bx2, by2, bz2, cx2, cy2, cz2, ax2, ay2, az2)
        _gen3d(out, x + bx2, y + by2, z + bz2,
               cx, cy, cz, ax2, ay2, az2, bx - bx2, by - by2, bz - bz2)
        _gen3d(out, x + (bx2 - dbx) + (cx - dcx),
               y + (by2 - dby) + (cy - dcy),
               z + (bz2 - dbz) + (cz - dcz),
               ax, ay, az, -bx2, -by2, -bz2, -(cx - cx2), -(cy - cy2), -(cz - cz2))
        _gen3d(out, x + (ax - dax) + bx2 + (cx - dcx),
               y + (ay - day) + by2 + (cy - dcy),
               z + (az - daz) + bz2 + (cz - dcz),
               -cx, -cy, -cz, -(ax - ax2), -(ay - ay2), -(az - az2),
               bx - bx2, by - by2, bz - bz2)
        _gen3d(out, x + (ax - dax) + (bx2 - dbx),
               y + (ay - day) + (by2 - dby),
               z + (az - daz) + (bz2 - dbz),
               -bx2, -by2, -bz2, cx2, cy2, cz2, -(ax - ax2), -(ay - ay2), -(az - az2))


def gilbert3d(width, height, depth):
    """List of (x, y, z) cells of a width x height x depth box in curve order.

    x runs along W, y along H, z along T.  The largest extent is the major
    axis (ties: W, then H, then T)."""
    out = []
    if width >= height and width >= depth:
        _gen3d(out, 0, 0, 0, width, 0, 0, 0, height, 0, 0, 0, depth)
    elif height >= width and height >= depth:
        _gen3d(out, 0, 0, 0, 0, height, 0, width, 0, 0, 0, 0, depth)
    else:
        _gen3d(out, 0, 0, 0, 0, 0, depth, width, 0, 0, 0, height, 0)
    return out


def hilbert_permutation(T, H, W, text_prefix=0):
    """(perm, inv) int64 arrays of length text_prefix + T*H*W.

    perm[r] = source token index of position r in the permuted sequence, so
    x_perm = x[perm]; inv is its inverse (x = x_perm[inv]).  Source tokens are
    laid out as [text_prefix tokens, then (t, h, w) row-major]; the text prefix
    maps to itself."""
    cells = gilbert3d(W, H, T)
    vis = np.array([text_prefix + (z * H + y) * W + x for (x, y, z) in cells],
                   dtype=np.int64)
    perm = np.concatenate([np.arange(text_prefix, dtype=np.int64), vis])
    inv = np.empty_like(perm)
    inv[perm] = np.arange(perm.size, dtype=np.int64)
    return perm, inv
