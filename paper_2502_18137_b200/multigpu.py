"""Multi-GPU plumbing of the hot path.

Every (batch, head) problem of SpargeAttn is independent -- stage 1 and
stage 2 never mix heads -- so one sequence's heads are
split across ranks by contiguous kv-groups (`shard.shard_heads`) and each
rank runs the C-ABI path on its own shard with no data-path collective.
The only collective is `gather_heads`: an all-gather of the per-rank O
shards (NCCL over NVLink on GPUs, gloo on CPU) used OUTSIDE the timed region
to check the sharded result against a single-GPU run.  Timing is reduced as
the max over ranks (`max_over_ranks`).
"""

import torch
import torch.distributed as dist

from .shard import shard_heads


def world_rank():
    if dist.is_available() and dist.is_initialized():
        return dist.get_world_size(), dist.get_rank()
    return 1, 0


def local_heads(Hq, Hkv, world=None, rank=None):
    """This rank's (q-heads, kv-heads) as lists of global indices."""
    if world is None:
        world, rank = world_rank()
    q0, q1, kv0, kv1 = shard_heads(Hq, Hkv, world, rank)
    return list(range(q0, q1)), list(range(kv0, kv1))


def gather_heads(o_local, Hq, Hkv):
    """All-gather per-rank O shards [B, Hq_r, N, d] along the head axis into
    the full [B, Hq, N, d] on every rank (shards may differ in size: they are
    padded to the largest, as all_gather needs equal shapes)."""
    world, _ = world_rank()
    if world == 1:
        return o_local
    sizes = [shard_heads(Hq, Hkv, world, r)[1] - shard_heads(Hq, Hkv, world, r)[0]
             for r in range(world)]
    mx = max(sizes)
    B, hr, N, d = o_local.shape
    dev = o_local.device
    # gloo gathers host tensors (the CPU tests; NCCL gathers device memory)
    host = dist.get_backend() == "gloo"
    src = o_local.cpu() if host else o_local
    pad = src.new_zeros((B, mx, N, d))
    pad[:, :hr] = src
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad.contiguous())
    return torch.cat([p[:, :s] for p, s in zip(parts, sizes)], dim=1).to(dev)


def max_over_ranks(x, device=None):
    """Max of a host float over all ranks (the bench's step-time reduction)."""
    world, _ = world_rank()
    if world == 1:
        return x
    if dist.get_backend() == "gloo":
        device = "cpu"
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
