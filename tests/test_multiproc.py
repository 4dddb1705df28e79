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


class _OracleExecutor:
    """run_sharded executor on the host: the oracle's fold on torch CPU buffers (the device
    executor is engine._ArenaExecutor; what is under test is the partition and the exchange)."""

    device = "cpu"

    def __init__(self, src, b):
        import torch

        self.torch, self.src, self.b = torch, src, b
        self.bufs, self.next, self.st, self.peak = {}, 0, {}, 0

    def alloc(self):
        h = self.next
        self.next += 1
        self.bufs[h] = self.torch.empty((self.b, self.b), dtype=self.torch.float64)
        self.peak = max(self.peak, len(self.bufs))
        return h

    def tensor(self, h):
        return self.bufs[h]

    def release(self, h):
        del self.bufs[h]

    def load(self, refs):
        out = {}
        for i, j in refs:
            out[(i, j)] = h = self.alloc()
            self.bufs[h].copy_(self.torch.from_numpy(self.src.block(i, j)))
        return out

    def schur(self, items, nids):
        from oracle import bri_oracle as orc

        for (p, rt, l_, r, o), nid in zip(items, nids):
            pv, rtv, lv, rv = (self.bufs[h].numpy() for h in (p, rt, l_, r))
            try:
                self.bufs[o].copy_(self.torch.from_numpy(rv - lv @ (orc.invert_dense(pv) @ rtv)))
            except orc.OracleSingular as e:
                self.st[nid] = e.pivot_index
                self.bufs[o].fill_(float("nan"))

    def invert(self, h):
        from oracle import bri_oracle as orc

        try:
            return self.torch.from_numpy(orc.invert_dense(self.bufs[h].numpy())), 0
        except orc.OracleSingular as e:
            return self.torch.full((self.b, self.b), float("nan"), dtype=self.torch.float64), e.pivot_index

    def status(self, nids):
        return {nid: self.st.get(nid, 0) for nid in nids}

    def empty_result(self):
        return self.torch.empty((self.b, self.b), dtype=self.torch.float64)


def _node_worker(rank, world, port, m, k, targets, q, singular):
    import sys

    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    from oracle import bri_oracle as orc
    from paper_1612_00001_b200 import dag
    from paper_1612_00001_b200.distributed import assign_owners, rank_peak_blocks, run_sharded

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    a = np.load(singular) if singular else shifted(m, 9)
    sched = dag.build_schedule(k, targets)
    ex = _OracleExecutor(orc.BlockSource(a, k), m // k)
    res, pst, rst = run_sharded(sched, rank, world, ex)
    err = None
    try:
        sched.first_failure(pst, rst, m // k)
    except Exception as e:  # every rank must raise the reference's error
        err = (type(e).__name__, [q_.name for q_ in e.path] if hasattr(e, "path") else None)
    mine = sum(1 for v in assign_owners(sched, world).values() if v == rank)
    peak_ok = ex.peak <= rank_peak_blocks(sched, assign_owners(sched, world), rank, scratch=0)
    if rank == 0:
        q.put(("res", {t: v.numpy() for t, v in res.items()}, err, mine, peak_ok))
    else:
        q.put(("rank", None, err, mine, peak_ok))
    dist.destroy_process_group()


@pytest.mark.parametrize("m,k,targets,world", [
    (16, 8, [(1, 1)], 2),                       # config-5 shape: one deep target, 270 nodes
    (24, 6, [(1, b) for b in range(1, 7)], 3),  # config-4 shape: a block row
    (20, 5, "all", 2),                          # config-3 shape: every block
])
def test_node_sharded_dag_matches_reference(m, k, targets, world):
    """One DAG over all targets, each level's nodes dealt to ranks, one operand exchange per
    level (gloo here, NCCL P2P on GPUs): rank 0 gets every block bit-identical to the
    reference recursion, every node runs on exactly one rank, and the per-rank footprint
    stays within rank_peak_blocks."""
    from oracle import bri_oracle as orc
    from paper_1612_00001_b200 import dag

    tg = [(x, y) for x in range(1, k + 1) for y in range(1, k + 1)] if targets == "all" else targets
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_node_worker, args=(r, world, port, m, k, tg, q, None)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res = next(g[1] for g in got if g[0] == "res")
    assert all(g[2] is None and g[4] for g in got)
    assert sum(g[3] for g in got) == len(dag.build_schedule(k, tg).nodes)
    a = shifted(m, 9)
    for t, (al, be) in enumerate(tg):
        np.testing.assert_array_equal(res[t], orc.invert_block(a, k, al, be, memo=True))


def test_node_sharded_singular_path(golden, tmp_path):
    """A failing pivot on one rank is reported on every rank as the reference's
    SingularPivotError path (statuses are all-reduced, then replayed)."""
    data, meta = golden
    f = tmp_path / "sing.npy"
    np.save(f, data["singular_matrix"])
    m = data["singular_matrix"].shape[0]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_node_worker, args=(r, 2, port, m, 3, [(1, 1)], q, str(f))) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for g in got:
        assert g[2] == ("SingularPivotError", meta["singular"]["path"])


def test_owner_assignment_balances_levels():
    from paper_1612_00001_b200 import dag
    from paper_1612_00001_b200.distributed import assign_owners, level_transfers

    sched = dag.build_schedule(8, [(1, 1)])
    for world in (1, 2, 4, 8):
        own = assign_owners(sched, world)
        for n, ids in sched.levels().items():
            counts = [sum(1 for nid in ids if own[nid] == r) for r in range(world)]
            assert max(counts) <= -(-len(ids) // world)
        moved = sum(len(level_transfers(sched, own, ids)) for ids in sched.levels().values())
        if world == 1:
            assert moved == 0
        # affinity keeps traffic well below "every operand moves"
        assert moved <= 0.75 * sum(4 for nd in sched.nodes if nd.n > 2)


class _OracleSlotExecutor:
    """run_sharded_bounded executor on the host: numbered slots and host buffers of torch CPU
    blocks, the oracle's fold per node (the device executor is engine._BoundedExecutor)."""

    device = "cpu"

    def __init__(self, src, b, nslots):
        import torch

        self.torch, self.src, self.b = torch, src, b
        self.slots = torch.full((nslots, b, b), float("nan"), dtype=torch.float64)
        self.host, self.st, self.rst, self.live, self.peak, self.moves = {}, {}, {}, set(), 0, 0

    def claim(self, s):
        assert s not in self.live, f"slot {s} claimed twice"
        self.live.add(s)
        self.peak = max(self.peak, len(self.live))

    def release(self, s):
        self.live.discard(s)

    def slot(self, s):
        return self.slots[s]

    def load(self, s, ij):
        self.slots[s].copy_(self.torch.from_numpy(self.src.block(*ij)))

    def node(self, nid, sl):
        from oracle import bri_oracle as orc

        pv, rtv, lv, rv = (self.slots[h].numpy() for h in sl[:4])
        try:
            self.slots[sl[4]].copy_(self.torch.from_numpy(rv - lv @ (orc.invert_dense(pv) @ rtv)))
        except orc.OracleSingular as e:
            self.st[nid] = e.pivot_index
            self.slots[sl[4]].fill_(float("nan"))
        self.slots[sl[5]].fill_(float("nan"))   # scratch contents must not matter
        self.slots[sl[6]].fill_(float("nan"))

    def invert(self, t, sl):
        from oracle import bri_oracle as orc

        try:
            return self.torch.from_numpy(orc.invert_dense(self.slots[sl[0]].numpy()))
        except orc.OracleSingular as e:
            self.rst[t] = e.pivot_index
            return self.torch.full((self.b, self.b), float("nan"), dtype=self.torch.float64)

    def output(self, t, s):
        return self.slots[s].clone()

    def spill(self, s, hb):
        self.host[hb] = self.slots[s].clone()
        self.moves += 1

    def reload(self, s, hb):
        self.slots[s].copy_(self.host[hb])
        self.moves += 1

    def statuses(self, nids):
        return {nid: self.st.get(nid, 0) for nid in nids}

    def root_status(self, t):
        return self.rst.get(t, 0)

    def empty_result(self):
        return self.torch.empty((self.b, self.b), dtype=self.torch.float64)


def _bounded_node_worker(rank, world, port, m, k, targets, nslots, q):
    import sys

    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    from oracle import bri_oracle as orc
    from paper_1612_00001_b200 import bounded as bd
    from paper_1612_00001_b200 import dag
    from paper_1612_00001_b200.distributed import assign_owners, run_sharded_bounded

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    a = shifted(m, 9)
    sched = dag.build_schedule(k, targets)
    owner = assign_owners(sched, world)
    p = bd.plan_rank(sched, owner, rank, nslots)
    ex = _OracleSlotExecutor(orc.BlockSource(a, k), m // k, bd.slots_used(p))
    res, pst, rst = run_sharded_bounded(sched, rank, world, ex, p)
    sched.first_failure(pst, rst, m // k)
    info = (ex.peak, bd.slots_used(p), p.spills, p.transfers, sum(1 for v in owner.values() if v == rank))
    q.put((rank, {t: v.numpy() for t, v in res.items()} if res is not None else None, info))
    dist.destroy_process_group()


@pytest.mark.parametrize("m,k,targets,world,nslots", [
    (16, 8, [(1, 1)], 2, 9),                    # config-5 shape, 2 ranks, tight: spills
    (16, 8, [(1, 1)], 4, 8),                    # config-5 shape, 4 ranks
    (24, 6, [(1, b) for b in range(1, 7)], 3, 10),   # config-4 shape, 3 ranks
    (20, 5, "all", 2, 12),                      # config-3 shape
])
def test_node_sharded_bounded_matches_reference(m, k, targets, world, nslots):
    """Node sharding inside a per-rank slot budget (the config-5-on-N-GPUs plan): each rank
    replays bounded.plan_rank (Belady spills of own and received values), transfers in one
    global order; rank 0 gets every block bit-identical to the reference recursion, every node
    runs exactly once, and no rank ever holds more than its budget."""
    from oracle import bri_oracle as orc
    from paper_1612_00001_b200 import dag

    tg = [(x, y) for x in range(1, k + 1) for y in range(1, k + 1)] if targets == "all" else targets
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bounded_node_worker, args=(r, world, port, m, k, tg, nslots, q))
             for r in range(world)]
    for p in procs:
        p.start()
    got = sorted([q.get(timeout=300) for _ in range(world)], key=lambda g: g[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res = got[0][1]
    assert sum(g[2][4] for g in got) == len(dag.build_schedule(k, tg).nodes)
    for _, _, (peak, used, spills, transfers, _) in got:
        assert peak <= used <= nslots
    if world == 2 and nslots == 9:
        assert sum(g[2][2] for g in got) > 0     # the tight budget really spills
    a = shifted(m, 9)
    for t, (al, be) in enumerate(tg):
        np.testing.assert_array_equal(res[t], orc.invert_block(a, k, al, be, memo=True))


def test_config5_sharded_bounded_plans_fit():
    """Config 5 (k=8, b=20480, 3.36 GB blocks) node-sharded over 2 / 4 / 8 GPUs within a
    48-block (161 GB) device budget per rank: host spills only at 2 ranks."""
    from paper_1612_00001_b200 import bounded as bd
    from paper_1612_00001_b200 import dag
    from paper_1612_00001_b200.distributed import assign_owners

    sched = dag.build_schedule(8, [(1, 1)])
    for world in (2, 4, 8):
        owner = assign_owners(sched, world)
        plans = [bd.plan_rank(sched, owner, r, 48) for r in range(world)]
        assert all(bd.slots_used(p) <= 48 for p in plans)
        assert sum(sum(1 for v in owner.values() if v == r) for r in range(world)) == 270
        if world >= 4:
            assert all(p.spills == 0 for p in plans)
        # balanced: no rank runs more than ceil(level / world) nodes of any level
        assert max(sum(1 for v in owner.values() if v == r) for r in range(world)) <= 270 // world + 8
