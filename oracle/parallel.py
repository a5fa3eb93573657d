"""The fp64 oracle fanned out over host cores (TEST INFRASTRUCTURE ONLY; see
oracle/__init__).

SURVEY §8(d) asks for the oracle "with std::thread = nproc" over
(head, q-block).  Algorithm 1's stage 2 is independent per query block
(every (head, i) runs its own online-softmax loop), so the
q-blocks are split across worker processes (fork: the inputs are shared
copy-on-write), each running the unchanged serial `sparse_attention` on its
share with single-threaded BLAS.  Stage 1 runs once in the
parent.  The arithmetic is the serial oracle's, call for call: the result is
bit-identical to `spargeattn_head` (tests/test_oracle_parallel.py).
"""

import multiprocessing as mp
import os

import numpy as np

from . import sparge_oracle as so

_SHARED = {}


def cores():
    """Host cores this process may run on."""
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def _work(args):
    blocks = args
    s = _SHARED
    try:
        from threadpoolctl import threadpool_limits
        ctx = threadpool_limits(1)
    except Exception:          # pragma: no cover - threadpoolctl is installed here
        ctx = None
    O, cnt = so.sparse_attention(s["q"], s["k"], s["v"], s["M"], s["lam"], s["bq"], s["bk"],
                                 s["cw"], s["causal"], s["quant"], s["pv_round"], blocks,
                                 s["v_fp8"])
    if ctx is not None:
        ctx.unregister()
    rows = np.concatenate([np.arange(i * s["bq"], min((i + 1) * s["bq"], s["n"]))
                           for i in blocks]) if blocks else np.zeros(0, int)
    return rows, O[rows], cnt


def spargeattn_head_parallel(q, k, v, tau, theta, lam, bq=128, bk=64, cw=4, causal=False,
                             sim_mode="cosine", quantize=True, pv_round="bf16", qblocks=None,
                             workers=None):
    """`spargeattn_head` with stage 2 split over `workers` processes (default:
    every core).  Returns (O, M, near, counters, quant, workers_used)."""
    q = np.asarray(q, dtype=np.float64)
    k = np.asarray(k, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    n = q.shape[0]
    M, near = so.predict_mask(q, k, tau, theta, bq, bk, causal, sim_mode)
    quant = None
    if quantize:
        quant = so.quantize_blocks(q, bq) + so.quantize_blocks(k, bk)
    v_fp8 = so.fp8_v_quant(v) if pv_round == "fp8" else None
    blocks = list(range(so.block_count(n, bq))) if qblocks is None else list(qblocks)
    workers = max(1, min(workers or cores(), len(blocks)))
    # round-robin shares: causal rows differ in cost, interleaving balances them
    shares = [blocks[w::workers] for w in range(workers)]
    _SHARED.update(q=q, k=k, v=v, M=M, lam=lam, bq=bq, bk=bk, cw=cw, causal=causal, quant=quant,
                   pv_round=pv_round, v_fp8=v_fp8, n=n)
    O = np.full(v.shape, np.nan)
    cnt = dict(qk=0, pv_slices=0)
    try:
        if workers == 1:
            results = [_work(shares[0])]
        else:
            with mp.get_context("fork").Pool(workers) as pool:
                results = pool.map(_work, shares)
    finally:
        _SHARED.clear()
    for rows, o_rows, c in results:
        O[rows] = o_rows
        cnt["qk"] += c["qk"]
        cnt["pv_slices"] += c["pv_slices"]
    return O, M, near, cnt, quant, workers
