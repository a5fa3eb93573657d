"""Multi-rank host logic on CPU (gloo, world_size 2): shard arithmetic and the
property that sharded execution gathered back equals the single-process
result bit for bit (the shards are independent; any difference is a bug).
The per-head compute here is the oracle (the GPU kernels need a B200)."""

import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2502_18137_b200.shard import shard_batch, shard_heads, static_efficiency


def test_shard_heads_cover_and_keep_groups():
    for Hq, Hkv in [(32, 8), (30, 30), (24, 24), (32, 32), (8, 2)]:
        for world in (1, 2, 4, 8):
            seen = []
            for r in range(world):
                q0, q1, kv0, kv1 = shard_heads(Hq, Hkv, world, r)
                assert q1 - q0 == (kv1 - kv0) * (Hq // Hkv)
                seen.extend(range(q0, q1))
                for h in range(q0, q1):
                    assert kv0 <= h // (Hq // Hkv) < kv1
            assert seen == list(range(Hq))


def test_static_efficiency_matches_survey():
    """C3's 30 heads -> 8/8/7/7 at 4 ranks (93.75 %)."""
    assert [shard_heads(30, 30, 4, r)[1] - shard_heads(30, 30, 4, r)[0] for r in range(4)] == \
        [8, 8, 7, 7]
    assert static_efficiency(30, 4) == pytest.approx(30 / 4 / 8)
    assert static_efficiency(8, 8) == 1.0


def test_shard_batch():
    for B in (1, 2, 7, 8):
        for world in (1, 2, 4):
            got = [shard_batch(B, world, r) for r in range(world)]
            assert got[0][0] == 0 and got[-1][1] == B
            assert all(a[1] == b[0] for a, b in zip(got, got[1:]))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q, k, v, out_path):
    """One rank of the head-sharded run, through the product's plumbing
    (paper_2502_18137_b200.multigpu): its heads, its compute (here the
    oracle: the kernels need a B200), the all-gather of O and the
    max-over-ranks timing reduction."""
    import oracle as O
    from paper_2502_18137_b200 import multigpu
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    Hq, Hkv = q.shape[0], k.shape[0]
    hq, hkv = multigpu.local_heads(Hq, Hkv)
    group = Hq // Hkv
    assert all(h // group in hkv for h in hq)
    mine = np.stack([O.spargeattn_head(q[h], k[h // group], v[h // group], 0.9, 0.5, -5.0,
                                       causal=True)[0] for h in hq]) if hq else \
        np.zeros((0,) + q.shape[1:])
    full = multigpu.gather_heads(torch.from_numpy(mine)[None], Hq, Hkv)[0]
    tm = multigpu.max_over_ranks(float(rank + 1))
    assert tm == world
    if rank == 0:
        np.save(out_path, full.numpy())
    dist.destroy_process_group()


@pytest.mark.parametrize("Hq,Hkv", [(4, 2), (6, 3), (2, 2)])
def test_head_sharded_gather_equals_single_process(tmp_path, Hq, Hkv):
    """Uneven shards too: 3 kv-groups over 2 ranks -> 2 + 1."""
    g = np.random.default_rng(0)
    N, d = 300, 32
    q = g.standard_normal((Hq, N, d))
    k = g.standard_normal((Hkv, N, d))
    v = g.standard_normal((Hkv, N, d))
    out = str(tmp_path / "o.npy")
    mp.spawn(_worker, args=(2, _free_port(), q, k, v, out), nprocs=2, join=True)
    got = np.load(out)
    import oracle as O
    grp = Hq // Hkv
    ref = np.stack([O.spargeattn_head(q[h], k[h // grp], v[h // grp], 0.9, 0.5, -5.0,
                                      causal=True)[0] for h in range(Hq)])
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("kind", ["llm_rope", "llm_local", "video"])
def test_head_shard_inputs_equal_slices_of_full(kind):
    """Each rank generates only its heads from per-global-head seeds
    (nothing is sent); the shard must equal the same slice of
    the single-GPU input, so gathered O can equal the single-GPU O bit for
    bit."""
    import bench
    from paper_2502_18137_b200 import multigpu
    if kind == "video":
        cfg = dict(kind="video", T=2, H=4, W=6, text_prefix=5, d=64, Hq=6, Hkv=6)
        cfg["N"] = 5 + 2 * 4 * 6
    else:
        cfg = dict(kind=kind, N=300, d=64, Hq=8, Hkv=2)
    q, k, v = bench.gen_inputs(cfg, 1000)
    for world in (2, 4):
        for rank in range(world):
            hq, hkv = multigpu.local_heads(cfg["Hq"], cfg["Hkv"], world, rank)
            if not hq:
                continue
            qs, ks, vs = bench.gen_inputs(cfg, 1000, heads=hq)
            assert np.array_equal(qs, q[:, hq]) and np.array_equal(ks, k[:, hkv])
            assert np.array_equal(vs, v[:, hkv])
