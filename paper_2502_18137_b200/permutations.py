"""Token orders of App. A.2 (Table 13) for scope row f3.

A video latent of T x H x W visual tokens follows `text_prefix` text tokens;
the source layout is [text][(t, h, w) row-major].  `make_perm(kind, ...)`
returns perm (int32) with perm[r] = source index of position r of the
permuted sequence -- the argument sparge_quantize / sparge_attn_fwd take.
Text tokens keep their positions ("we only permute the visual tokens",
P:L724).

  rowmajor     tokens continuous along W (the source order: identity)
  columnmajor  tokens continuous along H: order (t, w, h), h fastest
  timemajor    tokens continuous along T: order (h, w, t), t fastest
  random       a seeded random order of the visual tokens
  hilbert      the generalised 3-D Hilbert curve (a0, `hilbert_permute`)

Pure index arithmetic on the host (numpy); Hilbert comes from the C ABI.
"""

import numpy as np

KINDS = ("random", "rowmajor", "columnmajor", "timemajor", "hilbert")


def make_perm(kind, T, H, W, text_prefix=0, seed=0):
    t, h, w = np.meshgrid(np.arange(T), np.arange(H), np.arange(W), indexing="ij")
    src = (t * H + h) * W + w                       # source index of (t, h, w)
    if kind == "rowmajor":
        vis = src.reshape(-1)
    elif kind == "columnmajor":
        vis = src.transpose(0, 2, 1).reshape(-1)    # (t, w, h)
    elif kind == "timemajor":
        vis = src.transpose(1, 2, 0).reshape(-1)    # (h, w, t)
    elif kind == "random":
        vis = np.random.default_rng(seed).permutation(T * H * W)
    elif kind == "hilbert":
        from . import sparge
        perm, _ = sparge.hilbert_permute(T, H, W, text_prefix)
        return perm.astype(np.int32)
    else:
        raise ValueError(f"unknown permutation kind {kind!r}; one of {KINDS}")
    return np.concatenate([np.arange(text_prefix), text_prefix + vis]).astype(np.int32)


def inverse(perm):
    inv = np.empty_like(perm)
    inv[perm] = np.arange(perm.size, dtype=perm.dtype)
    return inv
