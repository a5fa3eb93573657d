"""Scope row f3 on the GPU: every App. A.2 token order runs the
full path correctly (O returned in the original order, equal to the oracle
under the same permutation), and the orders rank as Table 6 says on a smooth
3-D field: Hilbert has the highest block self-similarity and random the
lowest sparsity."""

import math

import numpy as np
import pytest
import torch

from helpers import check_o, bf16_np, oracle_forward, rel_l1
from paper_2502_18137_b200 import inputs, permutations, tuner

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("kind", ["columnmajor", "timemajor", "random"])
def test_permuted_path_matches_oracle(lib, kind):
    T, H, W, pre, d = 3, 8, 10, 16, 64
    qn, kn, vn = inputs.video(11, T, H, W, d=d, heads=2, text_prefix=pre)
    q, k, v = (inputs.to_device(a) for a in (qn, kn, vn))
    perm = permutations.make_perm(kind, T, H, W, pre, seed=1)
    o, bf = lib.sparge_forward(q, k, v, 0.9, 0.5, -5.0, perm=torch.from_numpy(perm).cuda())
    lib.sparge_attn_status(bf.workspace)
    ref = oracle_forward(bf16_np(q)[0], bf16_np(k)[0], bf16_np(v)[0], 0.9, 0.5, -5.0,
                         perm=perm.astype(np.int64))
    gm = bf.mask.cpu().numpy()[0]
    for h in range(2):
        bad = (gm[h] != ref[h]["M"]) & ~ref[h]["near"]
        assert not bad.any()
        check_o(bf16_np(o)[0, h], ref[h]["o"], "test_gpu_perm_study")


def test_orders_rank_as_table6(lib):
    T, H, W, d = 8, 24, 32, 64
    cal = [tuple(inputs.to_device(a) for a in inputs.video(40 + s, T, H, W, d=d, heads=4))
           for s in range(3)]
    res = {}
    for kind in permutations.KINDS:
        perm = torch.from_numpy(permutations.make_perm(kind, T, H, W, 0, seed=2)).cuda()
        ev = tuner.GpuEvaluator(cal, perm=perm)
        sim_k = float(np.mean([it[2].k_sim.mean().item() for it in ev.items]))
        err, sp = ev(0.9, 0.5, -5.0)
        res[kind] = (sim_k, err, sp)
    assert res["hilbert"][0] >= max(r[0] for r in res.values()) - 1e-12
    assert res["random"][0] <= min(r[0] for r in res.values()) + 1e-12
    assert res["random"][2] < res["hilbert"][2]
