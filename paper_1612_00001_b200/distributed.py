"""Multi-GPU host logic: target sharding and result gathering.

Inverse blocks are independent units (reference `invert_full(jobs>1)`,
engine.py:331-350; "embarrassingly parallel").  Ranks take
contiguous row-major chunks of the target list — targets of one block row
share their column map, which maximizes DAG sharing inside a rank — and run
their own deduplicated DAG.  The only collective is the final gather of
result blocks to rank 0 (NCCL over NVLink on GPUs; gloo in the CPU tests).
A single target cannot be split this way: every rank then runs a replica.
"""

from __future__ import annotations

__all__ = ["shard_targets", "gather_blocks"]


def shard_targets(targets, rank: int, world: int):
    """(my targets, scaling) — contiguous chunks; a lone target is replicated ("weak")."""
    targets = list(targets)
    if world <= 1:
        return targets, "strong" if len(targets) > 1 else "weak"
    if len(targets) == 1:
        return targets, "weak"
    per = (len(targets) + world - 1) // world
    return targets[rank * per:(rank + 1) * per], "strong"


def gather_blocks(blocks, targets, rank: int, world: int, b: int, group=None):
    """Gather every rank's result blocks to rank 0 -> {target: tensor} on rank 0, None elsewhere.

    blocks: list of (b, b) float64 tensors for this rank's shard (same device
    as the process group's backend expects).  Shards are padded to the
    largest shard so one `gather` of equal-sized tensors suffices.
    """
    import torch
    import torch.distributed as dist

    per = (len(targets) + world - 1) // world if len(targets) > 1 else 1
    dev = blocks[0].device if blocks else torch.device("cpu")
    pad = torch.zeros((per, b, b), dtype=torch.float64, device=dev)
    for i, blk in enumerate(blocks):
        pad[i].copy_(blk)
    bucket = [torch.empty_like(pad) for _ in range(world)] if rank == 0 else None
    dist.gather(pad, bucket, dst=0, group=group)
    if rank != 0:
        return None
    out = {}
    for r in range(world):
        mine, _ = shard_targets(targets, r, world)
        for i, t in enumerate(mine):
            out[tuple(t)] = bucket[r][i]
    return out
