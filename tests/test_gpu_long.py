"""Sequences beyond round 1's 128K limit (T_n <= 2048 then; now T_n <=
SPARGE_MAX_TN = 16384, N <= 2^20): stage-1 masks bit-exact against the
oracle on sampled rows and O on sampled q-blocks, causal and not, through
the C ABI.  Also the causal dead-tile skip of k_shat_dmma (dead Ŝ tiles are
never computed nor read)."""

import math

import numpy as np
import pytest
import torch

import oracle as O
from helpers import bf16_np, check_o
from paper_2502_18137_b200 import inputs, sparge

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("N,causal", [(262144 + 77, False), (200000, True)])
def test_long_sequence_masks_and_rows(N, causal):
    d = 64
    qn, kn, vn = inputs.llm_rope(5, N, d=d, Hq=1, Hkv=1)
    q, k, v = (inputs.to_device(a) for a in (qn, kn, vn))
    tau, theta, lam = 0.9, 0.5, -5.0
    o, bf = sparge.sparge_forward(q, k, v, tau, theta, lam, causal=causal)
    sparge.sparge_attn_status(bf.workspace)
    torch.cuda.synchronize()
    qs, ks, vs = bf16_np(q)[0, 0], bf16_np(k)[0, 0], bf16_np(v)[0, 0]
    M, near = O.predict_mask(qs, ks, O.f32(tau), O.f32(theta), causal=causal)
    gm = bf.mask.cpu().numpy()[0, 0]
    assert gm.shape == M.shape and M.shape[1] > 2048
    bad = (gm != M) & ~near
    assert not bad.any(), int(bad.sum())
    tm = M.shape[0]
    qb = [0, 1, tm // 3, tm - 1]
    o_ref, _ = O.sparse_attention(qs, ks, vs, M, O.f32(lam), causal=causal, qblocks=qb,
                                  quant=O.quantize_blocks(qs, 128) + O.quantize_blocks(ks, 64))
    check_o(bf16_np(o)[0, 0], o_ref, f"N={N}")
    cnt = bf.cnt.cpu().numpy()[0, 0]
    assert np.array_equal(cnt, M.sum(1))
