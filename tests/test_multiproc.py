"""Multi-rank host logic on CPU (gloo, world_size 2): target sharding + gather to rank 0.

The per-rank compute is the CPU oracle standing in for the device run; what is
under test is the partition and the collective protocol bench.py uses on GPUs.
"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import ROOT, shifted


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, m, k, q):
    import sys

    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    from oracle import bri_oracle as orc
    from paper_1612_00001_b200.distributed import gather_blocks, shard_targets

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    a = shifted(m, 5)
    targets = [(x, y) for x in range(1, k + 1) for y in range(1, k + 1)]
    mine, scaling = shard_targets(targets, rank, world)
    blocks = [torch.from_numpy(orc.invert_block(a, k, *t, memo=True)) for t in mine]
    got = gather_blocks(blocks, targets, rank, world, m // k)
    if rank == 0:
        full = orc.assemble({t: v.numpy() for t, v in got.items()}, k, m // k)
        q.put((scaling, sorted(got), float(np.abs(full @ a - np.eye(m)).max())))
    dist.destroy_process_group()


@pytest.mark.parametrize("m,k", [(12, 3), (20, 5)])
def test_sharded_full_inverse_gathers_on_rank0(m, k):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, m, k, q)) for r in range(2)]
    for p in procs:
        p.start()
    scaling, keys, resid = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert scaling == "strong"
    assert keys == [(x, y) for x in range(1, k + 1) for y in range(1, k + 1)]
    assert resid <= 1e-10  # BRI accuracy at k=5, not the gather


def test_shard_partition_covers_targets_once():
    from paper_1612_00001_b200.distributed import shard_targets

    tg = [(a, b) for a in range(1, 9) for b in range(1, 9)]
    for world in (1, 2, 3, 4, 8):
        seen = []
        for r in range(world):
            mine, scaling = shard_targets(tg, r, world)
            seen += mine
        assert seen == tg
    assert shard_targets([(1, 1)], 1, 4) == ([(1, 1)], "weak")
