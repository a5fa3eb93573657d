"""The host-parallel oracle (bench.py's cpu_baseline / reference arm) runs the
serial oracle's arithmetic call for call: identical O, mask and counters."""

import numpy as np

import oracle as O
from oracle.parallel import spargeattn_head_parallel
from paper_2502_18137_b200 import inputs


def test_parallel_equals_serial():
    q, k, v = inputs.llm_local(3, 1000, d=64, Hq=1, Hkv=1, gamma=1.5)
    q, k, v = (a[0, 0].astype(np.float64) for a in (q, k, v))
    for causal in (False, True):
        o1, m1, n1, c1, _ = O.spargeattn_head(q, k, v, 0.9, 0.5, -5.0, causal=causal)
        o2, m2, n2, c2, _, w = spargeattn_head_parallel(q, k, v, 0.9, 0.5, -5.0, causal=causal,
                                                        workers=3)
        assert w == 3
        assert np.array_equal(o1, o2) and np.array_equal(m1, m2) and np.array_equal(n1, n2)
        assert c1 == c2
    # sampled q-blocks: the other rows stay NaN, as in the serial oracle
    o3, _, _, c3, _, _ = spargeattn_head_parallel(q, k, v, 0.9, 0.5, -5.0, qblocks=[0, 5, 7],
                                                  workers=2)
    o4, _, _, c4, _ = O.spargeattn_head(q, k, v, 0.9, 0.5, -5.0, qblocks=[0, 5, 7])
    assert np.array_equal(np.isnan(o3), np.isnan(o4))
    assert np.array_equal(o3[~np.isnan(o3)], o4[~np.isnan(o4)]) and c3 == c4
