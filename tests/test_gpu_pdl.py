"""Programmatic dependent launch is a scheduling change only:
the kernels wait for their stream predecessor before touching memory, and
within one sparge_attn_fwd call the V stage runs after the launch-order
kernels and overlaps them.  These tests race-check it: the outputs must be
BIT-identical to (a) the split calls (V stage alone, then order + attention,
with a stream sync between) and (b) a process that launches every kernel
plainly (SPARGE_PDL=0), across back-to-back steps on one stream."""

import os
import subprocess
import sys

import numpy as np
import pytest
import torch

from paper_2502_18137_b200 import inputs

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _case(kind):
    if kind == "llm":
        qn, kn, vn = inputs.llm_local(3, 4096 + 77, d=128, Hq=8, Hkv=2)
        return qn, kn, vn, None, True, (0.9, 0.5, -5.0)
    T, H, W, pre = 4, 12, 14, 40
    qn, kn, vn = inputs.video(9, T, H, W, d=64, heads=3, text_prefix=pre)
    from paper_2502_18137_b200 import sparge
    perm, _ = sparge.hilbert_permute(T, H, W, pre)
    return qn, kn, vn, perm, False, (0.9, 0.5, -3.0)


def _steps(lib, kind, n=3, split=False):
    """n back-to-back whole-path steps on one stream (no sync between them);
    returns (O, mask, cnt) of the last."""
    qn, kn, vn, perm, causal, (tau, theta, lam) = _case(kind)
    q, k, v = (inputs.to_device(a) for a in (qn, kn, vn))
    pt = None if perm is None else torch.from_numpy(np.asarray(perm, np.int32)).cuda()
    shape = lib.make_shape(1, q.shape[1], k.shape[1], q.shape[2], q.shape[3], causal, q.dtype)
    bf = lib.Buffers(shape, device="cuda")
    o = torch.empty_like(q)
    for _ in range(n):
        lib.sparge_quantize(shape, q, 0, pt, bf.qq, bf.dq, bf.q_pooled, bf.q_sim)
        lib.sparge_quantize(shape, k, 1, pt, bf.kq, bf.dk, bf.k_pooled, bf.k_sim)
        lib.sparge_predict_mask(shape, bf.q_pooled, bf.q_sim, bf.k_pooled, bf.k_sim, tau, theta,
                                bf.mask, bf.lut, bf.cnt, bf.pred_workspace)
        if split:
            lib.sparge_attn_fwd_ex(shape, bf.qq, bf.dq, bf.kq, bf.dk, v, bf.lut, bf.cnt, lam, pt,
                                   o, None, bf.workspace, lib.SPARGE_ATTN_VPREP_ONLY)
            torch.cuda.synchronize()
            lib.sparge_attn_fwd_ex(shape, bf.qq, bf.dq, bf.kq, bf.dk, v, bf.lut, bf.cnt, lam, pt,
                                   o, None, bf.workspace, lib.SPARGE_ATTN_SKIP_VPREP)
        else:
            lib.sparge_attn_fwd(shape, bf.qq, bf.dq, bf.kq, bf.dk, v, bf.lut, bf.cnt, lam, pt, o,
                                None, bf.workspace)
    lib.sparge_attn_status(bf.workspace)
    torch.cuda.synchronize()
    return o.cpu(), bf.mask.cpu(), bf.cnt.cpu()


@pytest.mark.parametrize("kind", ["llm", "video"])
def test_one_call_equals_split_calls(lib, kind):
    a = _steps(lib, kind)
    b = _steps(lib, kind, split=True)
    for x, y in zip(a, b):
        assert torch.equal(x, y)


@pytest.mark.parametrize("kind", ["llm", "video"])
def test_pdl_equals_plain_launches(lib, kind, tmp_path):
    a = _steps(lib, kind)
    out = tmp_path / "plain.pt"
    code = (f"import sys; sys.path.insert(0, {ROOT!r}); sys.path.insert(0, {os.path.join(ROOT, 'tests')!r});"
            "import torch; from paper_2502_18137_b200 import sparge; import test_gpu_pdl as t;"
            f"torch.save(t._steps(sparge, {kind!r}), {str(out)!r})")
    env = dict(os.environ, SPARGE_PDL="0")
    subprocess.run([sys.executable, "-c", code], check=True, env=env, cwd=ROOT, timeout=600)
    b = torch.load(out)
    for x, y in zip(a, b):
        assert torch.equal(x, y)
