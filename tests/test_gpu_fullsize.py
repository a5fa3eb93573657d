"""GPU parity at BASELINE.json's full sizes.

The CUDA path runs each workload at its full sequence length, head dim, GQA
ratio, causality and Hilbert ordering -- the kernels, tile sizes and launch
configuration bench.py times -- on a subset of heads (all 32 for the Llama
config), and is compared with the oracle on what the oracle can compute one
by one:
  * the full stage-1 mask of sampled heads (bit-exact outside near-threshold);
  * LUT/cnt consistent with the mask (ascending kept j, counts);
  * O on sampled query blocks {0, 1, T_m/2, T_m-1}: head relative L1 < 5e-3
    (the bug threshold; the criterion is 2e-2) and every sampled row < 2e-2;
  * the lambda-gate decision of every (tile, warp) of the sampled blocks
    (sparge_attn_fwd_mpv) equals the oracle's outside the near-lambda band.
"""

import math

import numpy as np
import pytest
import torch

import bench
import oracle as O
from helpers import bf16_np, check_gate, check_o
from paper_2502_18137_b200 import inputs, sparge

pytestmark = pytest.mark.gpu

CASES = {
    # name: (q-heads run on the GPU, q-heads checked against the oracle)
    "llama31_8b_32k": (list(range(32)), [0, 13]),
    "cogvideox_2b": ([0, 1, 2, 3], [0, 3]),
    "mochi": ([0, 1], [1]),
    "sweep_128k": ([0, 1], [0]),
}


def _run_case(name):
    cfg = bench.workload_cfg(name)
    heads, check = CASES[name]
    q, k, v = bench.gen_inputs(cfg, 2024, heads=heads)
    perm = bench.hilbert_perm(cfg)
    qt, kt, vt = (inputs.to_device(a) for a in (q, k, v))
    pt = None if perm is None else torch.from_numpy(perm).cuda()
    tm, tn = math.ceil(cfg["N"] / 128), math.ceil(cfg["N"] / 64)
    mpv = torch.zeros(1, len(heads), tm, tn, 4, dtype=torch.uint8, device="cuda")
    o, bf = sparge.sparge_forward(qt, kt, vt, cfg["tau"], cfg["theta"], cfg["lam"],
                                  causal=cfg["causal"], perm=pt, mpv=mpv)
    sparge.sparge_attn_status(bf.workspace)
    return cfg, heads, check, qt, kt, vt, o, bf, perm, mpv.cpu().numpy()


@pytest.mark.parametrize("name", list(CASES))
def test_fullsize_masks_lut_and_sampled_rows(name):
    cfg, heads, check, qt, kt, vt, o, bf, perm, mpv = _run_case(name)
    N = cfg["N"]
    tm, tn = math.ceil(N / 128), math.ceil(N / 64)
    group = len(heads) // kt.shape[1] if cfg["Hq"] != cfg["Hkv"] else 1
    mask = bf.mask.cpu().numpy()[0]
    lut = bf.lut.cpu().numpy()[0]
    cnt = bf.cnt.cpu().numpy()[0]
    # LUT / cnt consistent with the mask for every head run
    for h in range(len(heads)):
        assert (cnt[h] == mask[h].sum(1)).all()
        for i in (0, tm // 2, tm - 1):
            kept = np.nonzero(mask[h, i])[0]
            assert np.array_equal(lut[h, i, :cnt[h, i]], kept)
    og = bf16_np(o)[0]
    qb = sorted({0, 1, tm // 2, tm - 1})
    for h in check:
        hl = heads.index(h)
        g = hl // group
        qs, ks, vs = bf16_np(qt)[0, hl], bf16_np(kt)[0, g], bf16_np(vt)[0, g]
        if perm is not None:
            qs, ks, vs = qs[perm], ks[perm], vs[perm]
        o_ref, M, near, cnt_ref, _ = O.spargeattn_head(
            qs, ks, vs, O.f32(cfg["tau"]), O.f32(cfg["theta"]), O.f32(cfg["lam"]),
            causal=cfg["causal"], qblocks=qb, trace=True)
        bad = (mask[hl] != M) & ~near
        assert not bad.any(), f"{name} head {h}: {int(bad.sum())} mask mismatches"
        oh = og[hl][perm] if perm is not None else og[hl]
        check_o(oh, o_ref, f"{name} head {h}")       # NaN rows (not sampled) skipped
        check_gate(mpv[0, hl], cnt_ref, cfg["lam"], qblocks=qb, label=f"{name} head {h}")
    c = bf.counters.cpu().numpy()[0]
    assert (c[:, 0] == cnt.sum(1)).all()          # executed QK tiles = kept tiles
    assert (c[:, 2] <= c[:, 0]).all() and (c[:, 1] <= 4 * c[:, 0]).all()
    # PV slices = the dumped computed decisions; kept blocks = the mask
    assert np.array_equal(c[:, 1], (mpv[0] == 2).sum(axis=(1, 2, 3)))
    assert np.array_equal((mpv[0] > 0).any(-1), mask.astype(bool))
