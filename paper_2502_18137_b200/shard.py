"""Work partitioning across ranks.

The hot path has no exchange step: every (batch, head) is independent
(S:L246), so ranks never talk on the data path.  Two partitions:

  batch  every rank runs whole sequences (weak scaling; bench default)
  heads  one sequence's heads split by contiguous kv-groups, so a GQA group
         (q-heads h with h // (Hq/Hkv) == g) never straddles two ranks
         (strong scaling); balanced to within one kv-group.
"""


def shard_heads(Hq, Hkv, world, rank):
    """(q0, q1, kv0, kv1): this rank's q-head range [q0, q1) and kv-head range
    [kv0, kv1).  Ranks beyond the kv-head count get an empty range."""
    if Hq % Hkv:
        raise ValueError("Hq must be a multiple of Hkv")
    group = Hq // Hkv
    base, extra = divmod(Hkv, world)
    kv0 = rank * base + min(rank, extra)
    kv1 = kv0 + base + (1 if rank < extra else 0)
    return kv0 * group, kv1 * group, kv0, kv1


def shard_batch(B, world, rank):
    """Batch range [b0, b1) of this rank (balanced to within one)."""
    base, extra = divmod(B, world)
    b0 = rank * base + min(rank, extra)
    return b0, b0 + base + (1 if rank < extra else 0)


def static_efficiency(Hkv, world):
    """Ideal strong-scaling efficiency of head sharding: mean / max shard."""
    sizes = [shard_heads(Hkv, Hkv, world, r)[3] - shard_heads(Hkv, Hkv, world, r)[2]
             for r in range(world)]
    return (Hkv / world) / max(sizes) if max(sizes) else 0.0
