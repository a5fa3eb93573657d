"""Scope row f4: the FP8 P~V product (SageAttention2-style, footnote P:L44;
reading R27) on INT8 QK, through the C ABI, against the oracle's
`pv_round="fp8"` path (the same E4M3 rounding, pinned against torch in
tests/test_oracle_fp8.py):
  * the staged V^T bytes are exactly the oracle's E4M3 V^, and the dequant
    scales s_c = fl32(amax_c / 448) are bit-exact;
  * masks bit-exact except near-threshold blocks, QK tile counters exact;
  * O within relative L1 2e-2 of the oracle's FP8 output (asserted < 5e-3
    as the bug signal; the FP8 format itself is ~4e-2 away from bf16).
"""

import math

import numpy as np
import pytest
import torch

import oracle as O
from helpers import ROW_L1_FP8, check_o, bf16_np, oracle_forward, rel_l1
from paper_2502_18137_b200 import inputs

pytestmark = pytest.mark.gpu

BUG_L1 = 5e-3


def _dev(x, dtype=torch.bfloat16):
    return inputs.to_device(x, dtype)


def _run(lib, q, k, v, tau, theta, lam, causal, perm=None):
    pt = None if perm is None else torch.from_numpy(perm.astype(np.int32)).cuda()
    o, bf = lib.sparge_forward(q, k, v, tau, theta, lam, causal=causal, perm=pt,
                               pv_dtype=lib.SPARGE_PV_FP8_E4M3)
    lib.sparge_attn_status(bf.workspace)
    return o, bf


def _check_masks(gpu_mask, ref, label):
    bad = (gpu_mask != ref["M"]) & ~ref["near"]
    assert not bad.any(), f"{label}: {int(bad.sum())} mask mismatches outside near-threshold"


def _r256(x):
    return (x + 255) // 256 * 256


@pytest.mark.parametrize("N,d,Hkv", [(1000, 128, 2), (77, 64, 1), (4096, 64, 3)])
def test_fp8_v_staging_bit_exact(lib, N, d, Hkv):
    qn, kn, vn = inputs.llm_local(N + d, N, d=d, Hq=Hkv, Hkv=Hkv)
    q, k, v = _dev(qn), _dev(kn), _dev(vn)
    perm = np.random.default_rng(N).permutation(N).astype(np.int32)
    o, bf = _run(lib, q, k, v, 0.9, 0.5, -5.0, False, perm=perm)
    n_pad = (N + 63) // 64 * 64
    ws = bf.workspace.cpu()
    vt_bytes = _r256(Hkv * d * n_pad)
    vt = ws[256:256 + Hkv * d * n_pad].view(torch.float8_e4m3fn).to(torch.float64).numpy()
    vt = vt.reshape(Hkv, d, n_pad)
    off = 256 + vt_bytes + _r256(Hkv * d * 4)
    sc = ws[off:off + Hkv * d * 4].view(torch.float32).numpy().reshape(Hkv, d)
    vs = bf16_np(v)[0]
    for h in range(Hkv):
        vh, s_ref = O.fp8_v_quant(vs[h][perm])
        assert np.array_equal(sc[h], s_ref)
        assert np.array_equal(vt[h][:, :N], vh.T)
        assert (vt[h][:, N:] == 0).all()


def test_c1_planted_fp8(lib):
    q, k, v = (_dev(a) for a in inputs.planted(0))
    o, bf = _run(lib, q, k, v, 0.9, 0.5, -5.0, False)
    ref = oracle_forward(bf16_np(q)[0], bf16_np(k)[0], bf16_np(v)[0], 0.9, 0.5, -5.0,
                         pv_round="fp8")[0]
    _check_masks(bf.mask.cpu().numpy()[0, 0], ref, "C1")
    err, _ = check_o(bf16_np(o)[0, 0], ref["o"], row_tol=ROW_L1_FP8)
    cnt = bf.counters.cpu().numpy()[0, 0]
    assert cnt[0] == ref["cnt"]["qk"]
    # PV slices: exact per decision in tests/test_gpu_mpv.py


@pytest.mark.parametrize("N,d,Hq,Hkv,causal,dtype", [
    (1000, 128, 4, 2, True, torch.bfloat16), (1000, 64, 2, 2, False, torch.bfloat16),
    (777, 128, 2, 1, False, torch.float16), (2048, 128, 4, 1, True, torch.bfloat16),
    (130, 64, 1, 1, True, torch.float16),
])
def test_fp8_ragged(lib, N, d, Hq, Hkv, causal, dtype):
    qn, kn, vn = inputs.llm_local(N + d + 3, N, d=d, Hq=Hq, Hkv=Hkv, gamma=1.5)
    q, k, v = _dev(qn, dtype), _dev(kn, dtype), _dev(vn, dtype)
    o, bf = _run(lib, q, k, v, 0.9, 0.5, -5.0, causal)
    ref = oracle_forward(bf16_np(q)[0], bf16_np(k)[0], bf16_np(v)[0], 0.9, 0.5, -5.0,
                         causal=causal, group=Hq // Hkv, pv_round="fp8")
    gm = bf.mask.cpu().numpy()[0]
    og = bf16_np(o)[0]
    cnt = bf.counters.cpu().numpy()[0]
    for h in range(Hq):
        _check_masks(gm[h], ref[h], f"head {h}")
        err, _ = check_o(og[h], ref[h]["o"], row_tol=ROW_L1_FP8)
        assert cnt[h, 0] == ref[h]["cnt"]["qk"]


def test_fp8_hilbert_and_filters_off(lib):
    T, H, W, pre, d = 3, 10, 12, 40, 64
    qn, kn, vn = inputs.video(5, T, H, W, d=d, heads=2, text_prefix=pre)
    perm, _ = lib.hilbert_permute(T, H, W, pre)
    q, k, v = (_dev(a) for a in (qn, kn, vn))
    for tau, theta, lam in ((0.9, 0.5, -5.0), (1.0, -1.0, -math.inf)):
        o, bf = _run(lib, q, k, v, tau, theta, lam, False, perm=perm)
        ref = oracle_forward(bf16_np(q)[0], bf16_np(k)[0], bf16_np(v)[0], tau, theta, lam,
                             perm=perm.astype(np.int64), pv_round="fp8")
        for h in range(2):
            _check_masks(bf.mask.cpu().numpy()[0][h], ref[h], f"head {h}")
            check_o(bf16_np(o)[0, h], ref[h]["o"], "test_gpu_f4", row_tol=ROW_L1_FP8)


def test_fp8_with_qk_input_is_not_implemented(lib):
    q = _dev(inputs.gaussian(0, 1, 1, 256, 64))
    with pytest.raises(lib.SpargeError) as e:
        lib.sparge_forward(q, q, q, 0.9, 0.5, -5.0, qk_dtype=lib.SPARGE_QK_INPUT,
                           pv_dtype=lib.SPARGE_PV_FP8_E4M3)
    assert e.value.code == lib.SPARGE_ENOTIMPL
