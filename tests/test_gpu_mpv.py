"""Lambda-gate decision parity (SURVEY §8(c) "Debug mode (C1): M_pv decisions
match except where |g - lambda| < 1e-5"; Algorithm 1 lines 14-17,
P:L212-216).

sparge_attn_fwd_mpv dumps, for every kept (q-block i, k-block j) and warp
group w, whether the kernel computed the P~V slice.  The oracle's trace
records its own decision and g = max_{r in I_w}(m_local - m_new) in fp64.
They must agree everywhere except inside the rounding band around lambda
(helpers.gate_near), and the GPU's PV-slice counter must equal its own
dumped decisions -- which replaces round 1's +-2/+-4 counter slack.
"""

import math

import numpy as np
import pytest
import torch

from helpers import ROW_L1, ROW_L1_FP8, bf16_np, check_gate, check_o, oracle_forward
from paper_2502_18137_b200 import inputs

pytestmark = pytest.mark.gpu


def _dev(x, dtype=torch.bfloat16):
    return inputs.to_device(x, dtype)


def _run_mpv(lib, q, k, v, tau, theta, lam, causal=False, perm=None, **kw):
    B, Hq, N, _ = q.shape
    tm, tn = math.ceil(N / 128), math.ceil(N / 64)
    mpv = torch.zeros(B, Hq, tm, tn, 4, dtype=torch.uint8, device="cuda")
    pt = None if perm is None else torch.from_numpy(perm.astype(np.int32)).cuda()
    o, bf = lib.sparge_forward(q, k, v, tau, theta, lam, causal=causal, perm=pt, mpv=mpv, **kw)
    lib.sparge_attn_status(bf.workspace)
    torch.cuda.synchronize()
    return o, bf, mpv.cpu().numpy()


def _sink_input(N=2048, d=128, seed=4):
    g = np.random.default_rng(seed)
    u = g.standard_normal(d)
    u *= 10 / np.linalg.norm(u)
    qn = (u[None, :] + 0.3 * g.standard_normal((N, d)))[None, None].astype(np.float32)
    kn = g.standard_normal((1, 1, N, d)).astype(np.float32)
    kn[0, 0, :64] = u * 2.5
    vn = g.standard_normal((1, 1, N, d)).astype(np.float32)
    return qn, kn, vn


def _compare(lib, q, k, v, tau, theta, lam, causal=False, group=1, perm=None, **kw):
    o, bf, mpv = _run_mpv(lib, q, k, v, tau, theta, lam, causal=causal, perm=perm, **kw)
    okw = {}
    row_tol = ROW_L1
    if kw.get("qk_dtype") == lib.SPARGE_QK_INPUT:
        okw["quantize"] = False
    if kw.get("pv_dtype") == lib.SPARGE_PV_FP8_E4M3:
        okw["pv_round"] = "fp8"
        row_tol = ROW_L1_FP8
    ref = oracle_forward(bf16_np(q)[0], bf16_np(k)[0], bf16_np(v)[0], tau, theta, lam,
                         causal=causal, group=group, trace=True,
                         perm=None if perm is None else perm.astype(np.int64), **okw)
    cnt = bf.counters.cpu().numpy()[0]
    gm = bf.mask.cpu().numpy()[0]
    n_near = 0
    for h in ref:
        assert np.array_equal((mpv[0, h] > 0).any(-1), gm[h].astype(bool))
        assert int(cnt[h, 0]) == int(gm[h].sum())
        n_near += check_gate(mpv[0, h], ref[h]["cnt"], lam, cnt[h, 1], label=f"head {h}")
        check_o(bf16_np(o)[0, h], ref[h]["o"], f"head {h}", row_tol=row_tol)
        if np.array_equal(gm[h], ref[h]["M"]):
            assert abs(int(cnt[h, 1]) - ref[h]["cnt"]["pv_slices"]) <= n_near
    return ref, mpv, n_near


def test_mpv_c1_planted(lib):
    """BASELINE configs[0] at lambda = -5, and at lambda = -1 where the gate
    skips more."""
    q, k, v = (_dev(a) for a in inputs.planted(0))
    for lam in (-5.0, -1.0):
        ref, mpv, _ = _compare(lib, q, k, v, 0.9, 0.5, lam)
        if lam == -1.0:
            assert (mpv == 1).sum() > 0


def test_mpv_sink_input_gate_fires(lib):
    """A sink-dominated input: most tiles sit far below the running max."""
    q, k, v = (_dev(a) for a in _sink_input())
    ref, mpv, _ = _compare(lib, q, k, v, 1.0, -1.0, -5.0)
    skipped = int((mpv == 1).sum())
    assert skipped > 0.5 * int((mpv > 0).sum()), skipped


@pytest.mark.parametrize("N,d,Hq,Hkv,causal", [(1000, 128, 4, 2, True), (777, 64, 2, 2, False),
                                                (2048, 128, 2, 1, True)])
@pytest.mark.parametrize("lam", [-5.0, -2.0])
def test_mpv_ragged_gqa(lib, N, d, Hq, Hkv, causal, lam):
    qn, kn, vn = inputs.llm_local(N + d, N, d=d, Hq=Hq, Hkv=Hkv, gamma=1.5)
    q, k, v = _dev(qn), _dev(kn), _dev(vn)
    _compare(lib, q, k, v, 0.9, 0.5, lam, causal=causal, group=Hq // Hkv)


def test_mpv_fp16_and_f1_and_fp8(lib):
    """The gate in every kernel variant: fp16 P~, the unquantised f1 kernel
    (bf16 QK^T) and FP8 P~V (row f4)."""
    qn, kn, vn = _sink_input(N=1024, d=64, seed=9)
    q, k, v = (_dev(a) for a in (qn, kn, vn))
    _compare(lib, q, k, v, 0.9, 0.5, -4.0, qk_dtype=lib.SPARGE_QK_INPUT)
    _compare(lib, q, k, v, 0.9, 0.5, -4.0, pv_dtype=lib.SPARGE_PV_FP8_E4M3)
    q16, k16, v16 = (_dev(a, torch.float16) for a in (qn, kn, vn))
    o, bf, mpv = _run_mpv(lib, q16, k16, v16, 0.9, 0.5, -4.0)
    ref = oracle_forward(bf16_np(q16)[0], bf16_np(k16)[0], bf16_np(v16)[0], 0.9, 0.5, -4.0,
                         trace=True, pv_round="fp16")[0]
    check_gate(mpv[0, 0], ref["cnt"], -4.0, bf.counters.cpu().numpy()[0, 0, 1])
    check_o(bf16_np(o)[0, 0], ref["o"], "fp16")


def test_mpv_hilbert_video(lib):
    T, H, W, pre, d = 3, 10, 12, 40, 64
    qn, kn, vn = inputs.video(5, T, H, W, d=d, heads=2, text_prefix=pre)
    perm, _ = lib.hilbert_permute(T, H, W, pre)
    q, k, v = _dev(qn), _dev(kn), _dev(vn)
    _compare(lib, q, k, v, 0.9, 0.5, -3.0, perm=perm)


def test_mpv_dump_off_is_default_and_identical(lib):
    """The dump changes nothing: O, mask and counters with and without it are
    bit-identical."""
    q, k, v = (_dev(a) for a in inputs.planted(3))
    o1, bf1 = lib.sparge_forward(q, k, v, 0.9, 0.5, -3.0)
    c1 = bf1.counters.clone()
    o2, bf2, _ = _run_mpv(lib, q, k, v, 0.9, 0.5, -3.0)
    assert torch.equal(o1, o2) and torch.equal(c1, bf2.counters)
