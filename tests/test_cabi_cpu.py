"""CPU-side checks of the C-ABI library: it loads, exports every symbol
include/sparge.h declares, validates arguments without a GPU, and its host
Hilbert builder is integer-identical to the oracle's independent gilbert3d."""

import ctypes
import os
import re

import numpy as np
import pytest

import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def sp():
    from paper_2502_18137_b200 import sparge
    return sparge


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "sparge.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\*?\s+\*?(sparge_\w+|hilbert_\w+)\s*\(",
                                 src, flags=re.M)))


def test_exports_every_declared_symbol(sp):
    names = declared_symbols()
    assert set(names) == set(sp.EXPORTED), names
    lib = ctypes.CDLL(sp.LIB_PATH)
    for n in names:
        assert hasattr(lib, n), n


def test_strerror_and_validation_without_gpu(sp):
    assert sp._lib.sparge_strerror(0) == b"ok"
    assert sp._lib.sparge_strerror(3).startswith(b"internal")
    bad = sp.make_shape(1, 3, 2, 128, 128)          # Hq % Hkv != 0
    assert sp._lib.sparge_attn_workspace(ctypes.byref(bad)) == 0
    bad = sp.make_shape(1, 1, 1, 128, 96)           # d not in {64,128}
    assert sp._lib.sparge_attn_workspace(ctypes.byref(bad)) == 0
    for degenerate in (sp.make_shape(1, 1, 1, 0, 128), sp.make_shape(0, 1, 1, 64, 128),
                       sp.make_shape(1, 0, 1, 64, 64)):   # empty inputs are rejected (N >= 1, B, H >= 1)
        assert sp._lib.sparge_attn_workspace(ctypes.byref(degenerate)) == 0
        assert sp._lib.sparge_predict_mask(ctypes.byref(degenerate), None, None, None, None, 0.9, 0.5,
                                           None, None, None, None, 0, None) == sp.SPARGE_EINVAL
    good = sp.make_shape(2, 4, 2, 1000, 128)
    # status + V^T [B, Hkv, N_pad/64, d, 64] bf16 + launch order of B*Hq*T_m int32 items + its scratch (256-B rounded)
    assert sp._lib.sparge_attn_workspace(ctypes.byref(good)) == 256 + 2 * 2 * 128 * 1024 * 2 + 256 + 512
    with pytest.raises(sp.SpargeError):
        sp.hilbert_permute(0, 4, 4)
    rc = sp._lib.sparge_predict_mask(ctypes.byref(good), None, None, None, None, 0.9, 0.5,
                                     None, None, None, None, 0, None)
    assert rc == sp.SPARGE_EINVAL


@pytest.mark.parametrize("T,H,W,pre", [(8, 8, 8, 0), (1, 6, 6, 0), (13, 30, 45, 226),
                                       (28, 30, 53, 0), (3, 5, 7, 11), (2, 64, 64, 0),
                                       (1, 1, 9, 3), (5, 1, 1, 0), (4, 9, 2, 0)])
def test_hilbert_matches_oracle(sp, T, H, W, pre):
    """Reading R19: two independent gilbert3d implementations agree exactly."""
    perm, inv = sp.hilbert_permute(T, H, W, pre)
    p_ref, i_ref = O.hilbert_permutation(T, H, W, pre)
    assert np.array_equal(perm, p_ref) and np.array_equal(inv, i_ref)


def test_causal_with_permutation_rejected_by_abi(sp):
    """causal masking is defined on token positions (R8), so the C
    ABI refuses a permutation together with causal=1 before touching memory."""
    shape = sp.make_shape(1, 1, 1, 256, 128, causal=True)
    st = sp.Strides(0, 256 * 128, 128)
    fake = ctypes.c_void_p(1 << 20)          # never dereferenced: validation fails first
    ws = sp._lib.sparge_attn_workspace(ctypes.byref(shape))
    rc = sp._lib.sparge_attn_fwd(ctypes.byref(shape), fake, fake, fake, fake, fake, st, fake,
                                 fake, -5.0, fake, fake, st, None, fake, ws, None)
    assert rc == sp.SPARGE_EINVAL
    rc = sp._lib.sparge_attn_fwd_mpv(ctypes.byref(shape), fake, fake, fake, fake, fake, st, fake,
                                     fake, -5.0, None, fake, st, None, fake, ws, None, None)
    assert rc == sp.SPARGE_EINVAL            # mpv NULL


def test_python_binding_validates_inputs(sp):
    """the binding rejects what raw pointers cannot carry (dtype,
    device, shape agreement) instead of handing wrong bytes to the kernels."""
    import torch
    q = torch.zeros(1, 2, 256, 64, dtype=torch.bfloat16)
    with pytest.raises(ValueError, match="CUDA"):
        sp.sparge_forward(q, q[:, :1], q[:, :1], 0.9, 0.5, -5.0)
    with pytest.raises(ValueError, match="bf16 or fp16"):
        sp._validate(q.float(), q, q, None, None, False)
    with pytest.raises(ValueError, match="q's dtype"):
        sp._validate(q, q.half(), q, None, None, False)
    with pytest.raises(ValueError, match="Hkv"):
        sp._validate(q, q[:, :1, :128], q[:, :1, :128], None, None, False)
    q4 = torch.zeros(1, 4, 256, 64, dtype=torch.bfloat16)
    with pytest.raises(ValueError, match="multiple of Hkv"):
        sp._validate(q4, q4[:, :3], q4[:, :3], None, None, False)
    with pytest.raises(ValueError, match="out"):
        sp._validate(q4, q4[:, :2], q4[:, :2], q4[:, :1], None, False)


def test_predict_rejects_rows_longer_than_max_tn(sp):
    """T_n = ceil(N / 64) above SPARGE_MAX_TN = 16384 (N > 2^20) is rejected
    before any launch (one compressed-map row per warp in shared memory)."""
    fake = ctypes.c_void_p(1 << 20)                       # 256-B aligned, never touched
    for N, ok in ((1 << 20, True), ((1 << 20) + 1, False)):
        shape = sp.make_shape(1, 1, 1, N, 128)
        ws = sp._lib.sparge_predict_workspace(ctypes.byref(shape))
        assert ws > 0
        if ok:
            continue                                      # a valid call would launch
        rc = sp._lib.sparge_predict_mask(ctypes.byref(shape), fake, fake, fake, fake, 0.9, 0.5,
                                         None, fake, fake, fake, ws, None)
        assert rc == sp.SPARGE_EINVAL


@pytest.mark.parametrize("Hq,Hkv,chunks", [(32, 8, 8), (32, 8, 1), (24, 24, 8), (30, 30, 6),
                                           (8, 4, 2), (4, 4, 4), (2, 1, 1), (1, 1, 1), (12, 4, 3)])
def test_pipeline_plan_partitions_heads(sp, Hq, Hkv, chunks):
    """HostPipeline's chunk plan (host logic only): the chunks partition the
    q-heads in order; each chunk is whole kv-groups or lies inside one group
    and is paired with exactly its kv-heads (GQA h -> h // group); every
    kv-head is copied once, by the first chunk that reads it; with the tail
    split the last chunk is one q-head."""
    group = Hq // Hkv
    for tail in (False, True):
        plan = sp.pipeline_plan(Hq, Hkv, chunks, tail)
        assert plan[0][0] == 0 and plan[-1][1] == Hq
        copied = set()
        for (q0, q1, k0, k1, copy_kv), nxt in zip(plan, plan[1:] + [None]):
            assert q0 < q1 and (nxt is None or nxt[0] == q1)
            assert k0 == q0 // group and k1 == (q1 - 1) // group + 1
            whole = q0 % group == 0 and q1 % group == 0
            assert whole or k1 - k0 == 1
            if copy_kv:
                assert not (set(range(k0, k1)) & copied)
                copied |= set(range(k0, k1))
            else:
                assert set(range(k0, k1)) <= copied
        assert copied == set(range(Hkv))
        if tail:
            assert plan[-1][1] - plan[-1][0] == 1
