"""Stage-1 masks of the three TopCdf kernels against the oracle (P:L253-286,
§3.2 TopCdf + Eq. 5; readings R4, R7, R8):
  * k_topcdf_rows   (warp per row,  T_n <= 512),
  * k_topcdf_reg    (CTA per row, keys in registers, radix refinement,
                     512 < T_n <= 2048: U = 8 and U = 16 entries per thread),
  * k_topcdf_cta    (CTA per row, keys in shared memory, T_n > 2048).
Masks bit-exact outside near-threshold blocks; LUT = the kept j ascending;
cnt = row counts.  Row shapes, tau (guard-only 0.01 .. all-selected 1.0),
theta forcing, causal, and the uniform-Q/K closed form (P^ ties everywhere:
the selection is decided by the index tie-break alone, so the radix
refinement descends to the index bits)."""

import numpy as np
import pytest
import torch

import oracle as O
from helpers import bf16_np
from paper_2502_18137_b200 import inputs, sparge

pytestmark = pytest.mark.gpu


def _predict(qn, kn, tau, theta, causal):
    q, k = inputs.to_device(qn), inputs.to_device(kn)
    v = torch.zeros_like(k)
    o, bf = sparge.sparge_forward(q, k, v, tau, theta, -5.0, causal=causal)
    torch.cuda.synchronize()
    return q, k, bf


def _check(q, k, bf, tau, theta, causal, label):
    qs, ks = bf16_np(q)[0, 0], bf16_np(k)[0, 0]
    M, near = O.predict_mask(qs, ks, O.f32(tau), O.f32(theta), causal=causal)
    gm = bf.mask.cpu().numpy()[0, 0].astype(bool)
    bad = (gm != M) & ~near
    assert not bad.any(), f"{label}: {int(bad.sum())} mask mismatches outside near-threshold"
    cnt = bf.cnt.cpu().numpy()[0, 0]
    lut = bf.lut.cpu().numpy()[0, 0]
    assert np.array_equal(cnt, gm.sum(1)), label
    for i in range(gm.shape[0]):
        assert np.array_equal(lut[i, :cnt[i]], np.nonzero(gm[i])[0]), (label, i)
    return int((gm != M).sum()), M.shape


@pytest.mark.parametrize("N", [32768 + 64 * 7, 65536, 131072 - 64 * 3, 131072 + 64 * 5])
@pytest.mark.parametrize("causal", [False, True])
def test_topcdf_kernels_match_oracle(N, causal):
    qn, kn, _ = inputs.llm_rope(17, N, d=64, Hq=1, Hkv=1)
    for tau, theta in [(0.9, 0.5), (0.3, -1.0), (0.01, -1.0), (0.995, 0.6), (1.0, -1.0)]:
        q, k, bf = _predict(qn, kn, tau, theta, causal)
        _, shape = _check(q, k, bf, tau, theta, causal, f"N={N} causal={causal} tau={tau}")
        assert shape[1] == -(-N // 64)


@pytest.mark.parametrize("N", [701 * 64, 1501 * 64, 2501 * 64])
def test_topcdf_uniform_ties(N):
    """Uniform Q/K (north star closed form): S^ is constant, P^ =
    1/T_n, and TopCdf keeps the first n_sel = max(1, #{k >= 1: k/T_n <= tau})
    blocks by the index tie-break -- in every row."""
    d = 64
    rng = np.random.default_rng(3)
    q0, k0 = rng.standard_normal(d), rng.standard_normal(d)
    qn = np.broadcast_to(q0, (1, 1, N, d)).astype(np.float32).copy()
    kn = np.broadcast_to(k0, (1, 1, N, d)).astype(np.float32).copy()
    tn = N // 64
    for tau in (0.9, 0.5, 0.01):
        q, k, bf = _predict(qn, kn, tau, 0.5, False)
        gm = bf.mask.cpu().numpy()[0, 0].astype(bool)
        t32 = float(np.float32(tau))          # the ABI takes tau as fp32
        n_sel = max(1, sum(1 for kk in range(1, tn + 1) if kk <= t32 * tn))
        expect = np.zeros(tn, dtype=bool)
        expect[:n_sel] = True
        # an exact tie at tau * c_last would be near-threshold: not in the sweep
        assert min(abs(kk - t32 * tn) for kk in (n_sel, n_sel + 1)) > 1e-6
        assert (gm == expect[None, :]).all(), (N, tau, int((gm != expect[None, :]).sum()))
