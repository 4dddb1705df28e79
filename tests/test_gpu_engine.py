"""Engine parity against the reference's golden vectors and the CPU oracle (needs a B200)."""

import os

import numpy as np
import pytest

from conftest import rel_err, rng, shifted

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def bri():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1612_00001_b200 as bri

    return bri


def _rel(x, y):
    return float(np.abs(x - y).max() / max(np.abs(y).max(), 1e-300))


@pytest.mark.parametrize("schedule", ["dag", "tree", "bounded"])
def test_worked_example(bri, golden, schedule):
    data, _ = golden
    prov = bri.make_memory_provider(np.array([[4.0, 2.0], [1.0, 3.0]]), 2)
    ws = bri.Workspace(schedule=schedule)
    for al in (1, 2):
        for be in (1, 2):
            out = bri.invert_block(prov, al, be, ws)
            assert abs(out.data[0, 0] - data[f"worked_{al}{be}"][0, 0]) <= 1e-15
            out.release()
    assert ws.gauge.live_blocks == 0


@pytest.mark.parametrize("schedule", ["dag", "tree", "bounded"])
def test_trace_4x4(bri, golden, schedule):
    data, meta = golden
    seen = {}
    ws = bri.Workspace(schedule=schedule)
    out = bri.invert_block(bri.make_memory_provider(data["trace4_matrix"], 4), 1, 1, ws,
                           trace=lambda p, f, v: seen.__setitem__("/".join(q.name for q in p), v))
    assert list(seen) == meta["trace4_paths"]  # same visiting order as the reference
    for path in meta["trace4_paths"]:
        assert abs(seen[path][0, 0] - data[f"trace4_node_{path}"][0, 0]) <= 1e-12
    assert abs(out.data[0, 0] - data["trace4_out"][0, 0]) <= 1e-12


def test_config1_full_inverse(bri, golden):
    """BASELINE config 1 (k=4, b=64, Uniform[-1,1] + mI, seed 0): all 16 blocks vs the reference."""
    data, meta = golden
    a = rng(0).uniform(-1.0, 1.0, (256, 256)) + 256 * np.eye(256)
    prov = bri.make_memory_provider(a, 4)
    sink = bri.MemorySink(prov.layout)
    summ = bri.invert_full(prov, sink)
    got = sink.finalize()
    ref = data["cfg1_inverse"]
    for al in range(4):
        for be in range(4):
            blk = slice(al * 64, al * 64 + 64), slice(be * 64, be * 64 + 64)
            assert _rel(got[blk], ref[blk]) <= 1e-9  # north-star tolerance, per block
    assert np.abs(a @ got - np.eye(256)).max() <= 1e-12
    c = summ.counters
    assert [c.block_inversions, c.block_multiplications, c.block_subtractions, c.schur_nodes] == meta["cfg1_counters"]
    assert summ.executed.schur_nodes == 116  # distinct DAG nodes


def test_random_cases_vs_reference(bri, golden):
    data, meta = golden
    for m, k, seed in meta["cases"]:
        name = f"rand_m{m}_k{k}_s{seed}"
        prov = bri.make_memory_provider(data[name + "_matrix"], k)
        keys = [key for key in data.files if key.startswith(name + "_t")]
        for key in keys:
            al, be = map(int, key[len(name) + 2:].split("_"))
            out = bri.invert_block(prov, al, be)
            assert _rel(out.data, data[key]) <= 1e-9, key


def test_spd_k2(bri, golden):
    data, _ = golden
    for m in (64, 128):
        out = bri.invert_block(bri.make_memory_provider(data[f"spd_m{m}_matrix"], 2), 1, 1)
        assert _rel(out.data, data[f"spd_m{m}_t1_1"]) <= 1e-12


@pytest.mark.parametrize("schedule", ["dag", "tree", "bounded"])
def test_singular_path(bri, golden, schedule):
    data, meta = golden
    with pytest.raises(bri.SingularPivotError) as exc:
        bri.invert_block(bri.make_memory_provider(data["singular_matrix"], 3), 1, 1,
                         bri.Workspace(schedule=schedule))
    assert [q.name for q in exc.value.path] == meta["singular"]["path"]
    assert list(exc.value.pivot_block) == meta["singular"]["pivot_block"]


def test_dag_equals_tree_bitwise(bri, monkeypatch):
    """Memoization changes the schedule, not the arithmetic (b > 96 path), as long as every
    pivot is solved from the left (W = p^-1 l); with right-side solves chosen where they are
    fewer (C = rt p^-1, the default) the association differs and the runs agree to rounding."""
    from paper_1612_00001_b200 import engine

    a = shifted(128 * 4, 77)
    prov = bri.make_memory_provider(a, 4)
    monkeypatch.setattr(engine, "_SOLVE_SIDE", "l")
    for target in [(1, 1), (2, 3), (4, 1)]:
        x = bri.invert_block(prov, *target, bri.Workspace(schedule="dag")).data
        y = bri.invert_block(prov, *target, bri.Workspace(schedule="tree")).data
        np.testing.assert_array_equal(x, y)
    monkeypatch.setattr(engine, "_SOLVE_SIDE", "auto")
    targets = [(al, be) for al in range(1, 5) for be in range(1, 5)]
    got, _ = bri.invert_blocks(prov, targets)
    for t, x in zip(targets, got):
        y = bri.invert_block(prov, *t, bri.Workspace(schedule="tree")).data
        assert _rel(x.cpu().numpy(), y) <= 1e-12, t


def test_right_side_solves_match_left_side(bri, monkeypatch):
    """The right-side solve path (C = rt p^-1 through the transposed factor, dinv of U^T / L^T,
    transpose + column permutation) against the left-side path on a full inverse where both
    sides are chosen (k = 6, b = 256, plain Gaussian + shift: heavy pivoting inside the factors)."""
    from paper_1612_00001_b200 import engine
    from paper_1612_00001_b200.dag import build_schedule

    k, b = 6, 256
    a = rng(91).standard_normal((k * b, k * b)) + 0.5 * k * b * np.eye(k * b)
    prov = bri.make_memory_provider(a, k)
    targets = [(al, be) for al in range(1, k + 1) for be in range(1, k + 1)]
    sched = build_schedule(k, targets)
    nr = sum(1 for ids in sched.levels().values() for side in engine._solve_sides(sched, ids).values()
             if side == "rt")
    assert nr > 0
    monkeypatch.setattr(engine, "_SOLVE_SIDE", "l")
    left, info_l = bri.invert_blocks(prov, targets)
    monkeypatch.setattr(engine, "_SOLVE_SIDE", "auto")
    right, info_r = bri.invert_blocks(prov, targets)
    assert info_r.solves < info_l.solves
    dense = np.linalg.inv(a)
    for t, x, y in zip(targets, right, left):
        al, be = t
        ref = dense[(al - 1) * b:al * b, (be - 1) * b:be * b]
        ex, ey = _rel(x.cpu().numpy(), ref), _rel(y.cpu().numpy(), ref)
        assert ex <= max(1e-9, 4 * ey), (t, ex, ey)


@pytest.mark.parametrize("k", [2, 3, 4, 5])
def test_counts_and_tree_footprint(bri, k):
    ws = bri.Workspace(schedule="tree")
    prov = bri.make_memory_provider(shifted(k * 4, 82), k)
    with bri.gauge_scope(ws.gauge) as scope:
        out = bri.invert_block(prov, 1, 1, ws)
        out.release()
    want = bri.predicted_counts(k)
    assert ws.counters == want
    assert scope.peak_blocks <= 2 * k + 4


def test_block_row_vs_oracle_floor(bri):
    """Off-diagonal targets at k=6: parity judged against the reference's own 1-ulp floor."""
    from conftest import oracle_with_floor

    a = shifted(6 * 100, 31)
    prov = bri.make_memory_provider(a, 6)
    row = bri.invert_block_row(prov, 2)
    targets = [(2, b) for b in range(1, 7)]
    want, floor = oracle_with_floor(a, 6, targets)
    for b, blk in enumerate(row, start=1):
        assert _rel(blk.data, want[(2, b)]) <= max(1e-9, 8 * floor[(2, b)]), (b, floor[(2, b)])
    # the diagonal-relative residual of the whole row stays tight
    x = np.concatenate([blk.data for blk in row], axis=1)  # rows of M^-1 for block row 2
    resid = np.abs(x @ a - np.eye(600)[100:200]).max()
    assert resid <= 1e-10


def test_config2_full_size(bri):
    """BASELINE config 2 at true size: k=2, b=4096, SPD G G^T/m + I, seed 1, block (1,1)."""
    import torch

    from oracle import bri_oracle as orc
    from paper_1612_00001_b200.workloads import make_matrix

    a = make_matrix(2)
    prov = bri.make_memory_provider(a, 2)
    out = bri.invert_block(prov, 1, 1).data
    want = orc.invert_block(a, 2, 1, 1)
    assert _rel(out, want) <= 1e-9
    # block residual: (M X)[:, block 1] = e_1 block column
    x_col = np.linalg.solve(a, np.eye(8192)[:, :4096])[:4096]  # dense reference column
    assert _rel(out, x_col) <= 1e-9


def test_bounded_arena_groups_targets(monkeypatch):
    """A DAG that does not fit the arena budget is split into target groups
    (engine._run_grouped); results equal the unbounded run bit for bit, the
    device footprint stays under the budget, and a single target that cannot
    fit runs the bounded-footprint schedule instead.  (Bitwise with left-side
    solves: which side a pivot is solved from depends on the nodes that share it,
    so grouping can change it — and with it the rounding.)"""
    from paper_1612_00001_b200 import engine

    monkeypatch.setattr(engine, "_SOLVE_SIDE", "l")
    import torch

    import paper_1612_00001_b200 as bri
    from paper_1612_00001_b200.dag import build_schedule

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    a = shifted(1024, 29)
    prov = bri.make_memory_provider(a, 8)           # b = 128
    targets = [(al, be) for al in range(1, 9) for be in range(1, 9)]
    need = lambda tg: len(build_schedule(8, tg).m_blocks_used()) + build_schedule(8, tg).peak_level_blocks()
    budget = need(targets[:8]) + 40                 # room for a group of 8 targets, not for all 64
    assert need(targets) > budget
    full, _ = bri.invert_blocks(prov, targets)
    block = 128 * 128 * 8
    ws = bri.Workspace(arena_bytes=budget * block)
    part, info = bri.invert_blocks(prov, targets, ws)
    assert ws.gauge.peak_blocks <= budget
    for x, y in zip(full, part):
        assert torch.equal(x, y)
    one, info = bri.invert_blocks(prov, [(1, 1)], bri.Workspace(arena_bytes=(need([(1, 1)]) - 10) * block))
    assert info.schedule == "bounded" and torch.equal(one[0], full[0])


@pytest.mark.parametrize("b,budget", [(128, 9), (128, 24), (64, 8), (200, 12)])
def test_bounded_schedule_spills_bitwise(bri, b, budget):
    """One config-5-shaped target (k=8) whose DAG does not fit: every node runs once within
    `budget` device blocks, values spill to pinned host blocks and come back, and the block is
    bit-identical to the same schedule run without any spill (spilling moves bytes, never
    arithmetic); it matches the level-batched DAG run and the oracle within 1e-9 (batches of more
    than two factorizations take the unfolded LU variant, a different rounding once b spans
    several 128-column blocks)."""
    import torch

    from oracle import bri_oracle as orc

    a = shifted(8 * b, 41 + b)
    prov = bri.make_memory_provider(a, 8)
    ld = (b + 7) // 8 * 8
    roomy = bri.Workspace(schedule="bounded", arena_bytes=400 * b * ld * 8)
    ref, rinfo = bri.invert_blocks(prov, [(1, 1)], roomy)
    assert rinfo.schedule == "bounded" and rinfo.spills == 0
    ws = bri.Workspace(arena_bytes=budget * b * ld * 8)
    got, info = bri.invert_blocks(prov, [(1, 1)], ws)
    assert info.schedule == "bounded" and info.dag_nodes == 270 and info.spills > 0
    assert ws.gauge.peak_blocks <= budget and ws.gauge.live_blocks == 0
    assert ws.executed.schur_nodes == 270
    assert torch.equal(got[0], ref[0])
    want = bri.invert_block(prov, 1, 1).data
    assert rel_err(got[0].cpu().numpy(), want) <= 1e-9
    from conftest import oracle_with_floor

    ref_cpu, floor = oracle_with_floor(a, 8, [(1, 1)])   # k = 8: the reference's own 1-ulp floor
    assert rel_err(want, ref_cpu[(1, 1)]) <= max(1e-9, 8 * floor[(1, 1)])
    with pytest.raises(bri.BadPartitionError):
        bri.invert_blocks(prov, [(1, 1)], bri.Workspace(arena_bytes=budget * b * ld * 8, host_bytes=b * ld * 8))


def test_bounded_schedule_many_targets_and_reduce_frame(bri, monkeypatch):
    """schedule='bounded' over several targets (roots inverted as soon as they exist) and
    through reduce_frame (un-inverted roots) equals the DAG run bit for bit (both with
    left-side solves: the bounded schedule runs one node at a time)."""
    from paper_1612_00001_b200 import engine

    monkeypatch.setattr(engine, "_SOLVE_SIDE", "l")
    import torch

    a = shifted(6 * 104, 43)
    prov = bri.make_memory_provider(a, 6)
    targets = [(1, 1), (3, 2), (6, 6), (2, 5)]
    x, _ = bri.invert_blocks(prov, targets)
    ws = bri.Workspace(schedule="bounded", arena_bytes=10 * 104 * 104 * 8)
    y, info = bri.invert_blocks(prov, targets, ws)
    assert info.schedule == "bounded"
    for u, v in zip(x, y):
        assert torch.equal(u, v)
    fr = bri.frame_at(6, (bri.Quadrant.A, bri.Quadrant.D))
    r1 = bri.reduce_frame(prov, fr).data
    r2 = bri.reduce_frame(prov, fr, bri.Workspace(schedule="bounded", arena_bytes=8 * 104 * 104 * 8)).data
    np.testing.assert_array_equal(r1, r2)


def test_node_sharded_device_executor_world1(bri, golden, monkeypatch):
    """invert_blocks_sharded on the device executor (NCCL process group of one rank: the
    exchange is empty, the arena executor, status replay and root hand-off are exercised);
    blocks equal the single-process DAG run (left-side solves) bit for bit.  The multi-rank
    exchange itself is covered on CPU (tests/test_multiproc.py, gloo)."""
    from paper_1612_00001_b200 import engine

    monkeypatch.setattr(engine, "_SOLVE_SIDE", "l")
    import socket

    import torch
    import torch.distributed as dist

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda:0"))
    try:
        a = shifted(6 * 128, 47)
        prov = bri.make_memory_provider(torch.from_numpy(a).cuda(), 6)
        targets = [(1, b) for b in range(1, 7)]
        want, _ = bri.invert_blocks(prov, targets)
        ws = bri.Workspace()
        got, info = bri.invert_blocks_sharded(prov, targets, ws)
        assert info.schedule == "sharded" and ws.executed.schur_nodes == info.dag_nodes
        for x, y in zip(got, want):
            assert torch.equal(x, y)
        assert ws.gauge.live_blocks == 0
        # the per-rank bounded plan (config 5 on N GPUs): 9 device blocks, spills to pinned host
        wsb = bri.Workspace(schedule="bounded", arena_bytes=9 * 128 * 128 * 8)
        got_b, info_b = bri.invert_blocks_sharded(prov, targets, wsb)
        assert info_b.schedule == "sharded-bounded" and info_b.spills > 0 and info_b.arena_slots <= 9, info_b
        for x, y in zip(got_b, want):
            assert torch.equal(x, y)
        assert wsb.gauge.live_blocks == 0
        data, meta = golden
        with pytest.raises(bri.SingularPivotError) as exc:
            bri.invert_blocks_sharded(bri.make_memory_provider(data["singular_matrix"], 3), [(1, 1)])
        assert [q.name for q in exc.value.path] == meta["singular"]["path"]
    finally:
        dist.destroy_process_group()


def test_run_program_replay_small_order(bri, golden):
    """Small-order DAG runs on an HBM-resident matrix are one bri_dag_small call whose arrays are
    built once (engine._SMALL_PROGRAMS): a repeat returns the same bits, the gauge sees the same
    peak, the counters advance the same way, and a singular pivot is reported again."""
    import torch

    from paper_1612_00001_b200 import engine

    a = torch.from_numpy(rng(0).uniform(-1.0, 1.0, (256, 256)) + 256 * np.eye(256)).cuda()
    prov = bri.make_memory_provider(a, 4)
    targets = [(al, be) for al in range(1, 5) for be in range(1, 5)]
    ws1 = bri.Workspace()
    first, i1 = bri.invert_blocks(prov, targets, ws1)
    n_prog = len(engine._SMALL_PROGRAMS)
    ws2 = bri.Workspace()
    second, i2 = bri.invert_blocks(prov, targets, ws2)
    assert len(engine._SMALL_PROGRAMS) == n_prog and n_prog >= 1
    for x, y in zip(first, second):
        assert torch.equal(x, y)
    assert ws1.gauge.peak_blocks == ws2.gauge.peak_blocks and ws2.gauge.live_blocks == 0
    assert ws1.counters == ws2.counters and ws1.executed == ws2.executed
    assert (i1.dag_nodes, i1.levels) == (i2.dag_nodes, i2.levels)
    data, meta = golden
    sing = bri.make_memory_provider(torch.from_numpy(data["singular_matrix"]).cuda(), 3)
    for _ in range(2):
        with pytest.raises(bri.SingularPivotError) as exc:
            bri.invert_blocks(sing, [(1, 1)])
        assert [q.name for q in exc.value.path] == meta["singular"]["path"]
