"""Multi-GPU host logic: target sharding, and node sharding with one
operand exchange per DAG level.

Node sharding (`run_sharded`, engine.invert_blocks_sharded): one deduplicated
DAG over all targets; each level's nodes are dealt to ranks, preferring the
rank that already holds a node's operands; the operand values that cross ranks
move in one batch of NCCL P2P sends/receives per level, straight into arena
slots; root blocks go to rank 0.  Every node runs exactly once in the job.

Target sharding:

Inverse blocks are independent units (reference `invert_full(jobs>1)`,
engine.py:331-350; "embarrassingly parallel").  Ranks take
contiguous row-major chunks of the target list — targets of one block row
share their column map, which maximizes DAG sharing inside a rank — and run
their own deduplicated DAG.  The only collective is the final gather of
result blocks to rank 0 (NCCL over NVLink on GPUs; gloo in the CPU tests).
A single target cannot be split this way: every rank then runs a replica.
"""

from __future__ import annotations

__all__ = ["shard_targets", "gather_blocks", "assign_owners", "level_transfers", "exchange", "run_sharded",
           "run_sharded_bounded", "rank_peak_blocks"]


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


# --------------------------------------------------------------------------
# Node sharding: one deduplicated DAG over all targets, each level's nodes
# dealt to ranks, one operand exchange per level (SURVEY.md §8(e), config 5
# "one exchange step per level"; config 4 "recursion branches sharded").
# --------------------------------------------------------------------------

def assign_owners(sched, world: int) -> dict:
    """Owner rank of every DAG node: level by level, each node goes to the rank that already
    holds most of its operand values (fewest transfers), among ranks below the level's
    balanced cap ceil(len(level) / world); ties -> least loaded, then lowest rank.
    Leaf-level nodes read only base blocks (every rank can load them) and are dealt by load."""
    owner = {}
    for n, ids in sched.levels().items():
        cap = -(-len(ids) // world)
        load = [0] * world
        for nid in ids:
            aff = [0] * world
            for ref in sched.nodes[nid].operands:
                if ref[0] == "v":
                    aff[owner[ref[1]]] += 1
            best = min((r for r in range(world) if load[r] < cap), key=lambda r: (-aff[r], load[r], r))
            owner[nid] = best
            load[best] += 1
    return owner


def level_transfers(sched, owner: dict, ids) -> list:
    """(src rank, dst rank, node id) for every operand value a node of `ids` reads from another
    rank, deduplicated per destination, in a deterministic order every rank agrees on."""
    out, seen = [], set()
    for nid in ids:
        dst = owner[nid]
        for ref in sched.nodes[nid].operands:
            if ref[0] == "v":
                src = owner[ref[1]]
                if src != dst and (ref[1], dst) not in seen:
                    seen.add((ref[1], dst))
                    out.append((src, dst, ref[1]))
    return out


def exchange(transfers, rank: int, tensor_of, recv_into, group=None) -> None:
    """Post this rank's sends and receives of one level's transfers as one batch of P2P ops
    (NCCL over NVLink on GPUs, gloo on CPU) and wait for them.  tensor_of(nid) is the local
    value to send; recv_into(nid) returns the (contiguous) tensor a received value lands in."""
    import torch.distributed as dist

    ops = []
    for src, dst, nid in transfers:
        if src == rank:
            ops.append(dist.P2POp(dist.isend, tensor_of(nid), dst, group))
        elif dst == rank:
            ops.append(dist.P2POp(dist.irecv, recv_into(nid), src, group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()


def run_sharded(sched, rank: int, world: int, ex, invert_roots: bool = True, group=None):
    """Level-synchronous DAG run over `world` ranks with executor `ex`.

    ex.load(refs) -> {("m", i, j): handle}      base blocks this rank's leaves read
    ex.schur(items, nids)                        items: (p, rt, l, r) handles + out handle per node
    ex.alloc() -> handle; ex.tensor(handle)      a block buffer and its contiguous tensor
    ex.release(handle)
    ex.invert(handle) -> tensor                  final inversion of a root value
    ex.status(nids) -> {nid: int}               pivot statuses of this rank's nodes
    Returns ({target index: result tensor} on rank 0 else None, node statuses of all ranks).
    Roots are inverted by their owners and sent to rank 0.
    """
    import torch
    import torch.distributed as dist

    if world > 1:
        dist.barrier(group=group)  # the communicator exists before the first P2P batch
    owner = assign_owners(sched, world)
    roots = set(sched.roots)
    val = {}          # node id -> handle (own values and received copies)
    for n, ids in sched.levels().items():
        mine = [nid for nid in ids if owner[nid] == rank]
        recv_h = {}

        def recv_into(nid):
            h = ex.alloc()
            recv_h[nid] = h
            return ex.tensor(h)

        exchange(level_transfers(sched, owner, ids), rank, lambda nid: ex.tensor(val[nid]), recv_into, group)
        val.update(recv_h)
        mrefs = sorted({(r[1], r[2]) for nid in mine for r in sched.nodes[nid].operands if r[0] == "m"})
        mh = ex.load(mrefs) if mrefs else {}
        items = []
        for nid in mine:
            ops = [mh[(r[1], r[2])] if r[0] == "m" else val[r[1]] for r in sched.nodes[nid].operands]
            items.append(tuple(ops) + (ex.alloc(),))
        if items:
            ex.schur(items, mine)
        for h in mh.values():
            ex.release(h)
        # values of the previous level (own and received) are dead once this level ran
        for nid in [v for v in val if sched.nodes[v].n == n - 1 and v not in roots]:
            ex.release(val.pop(nid))
        for nid, it in zip(mine, items):
            val[nid] = it[4]
    # roots: owners invert them (or take the value as is); statuses of every node and root,
    # agreed on all ranks; then the results go to rank 0
    results, root_st = {}, {}
    for t, nid in enumerate(sched.roots):
        if owner[nid] == rank:
            if invert_roots:
                x, root_st[t] = ex.invert(val[nid])
            else:
                x = ex.tensor(val[nid])[:, : ex.b].clone()
            results[t] = x.contiguous()
    st = ex.status([nid for nid in owner if owner[nid] == rank])
    nn = len(sched.nodes)
    flat = torch.zeros(nn + len(sched.roots), dtype=torch.int64, device=ex.device)
    for nid, v in st.items():
        flat[nid] = int(v)
    for t, v in root_st.items():
        flat[nn + t] = int(v)
    if world > 1:
        dist.all_reduce(flat, group=group)
    ops = []
    for t, nid in enumerate(sched.roots):
        o = owner[nid]
        if o == rank and rank != 0:
            ops.append(dist.P2POp(dist.isend, results[t], 0, group))
        elif o != rank and rank == 0:
            results[t] = ex.empty_result()
            ops.append(dist.P2POp(dist.irecv, results[t], o, group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    for h in val.values():
        ex.release(h)
    host = flat.cpu().numpy()
    return (results if rank == 0 else None), host[:nn], host[nn:]


def rank_peak_blocks(sched, owner: dict, rank: int, scratch: int = 2) -> int:
    """Peak blocks one rank holds during run_sharded (values, received copies, base blocks,
    `scratch` per node of a level, 2 for a root inversion) — the arena a device executor needs."""
    roots = set(sched.roots)
    prev_own, held_roots, peak = 0, 0, 0
    for n, ids in sched.levels().items():
        mine = [nid for nid in ids if owner[nid] == rank]
        recv = sum(1 for _, dst, _ in level_transfers(sched, owner, ids) if dst == rank)
        mrefs = {(r[1], r[2]) for nid in mine for r in sched.nodes[nid].operands if r[0] == "m"}
        peak = max(peak, held_roots + prev_own + recv + len(mrefs) + (1 + scratch) * len(mine))
        prev_own = sum(1 for nid in mine if nid not in roots)
        held_roots += sum(1 for nid in mine if nid in roots)
    return max(peak, held_roots + 2)


# --------------------------------------------------------------------------
# Node sharding within a per-rank memory bound (config 5 on 2 / 4 / 8 GPUs)
# --------------------------------------------------------------------------

def run_sharded_bounded(sched, rank: int, world: int, ex, plan, invert_roots: bool = True, group=None):
    """Replay one rank's bounded plan (bounded.plan_rank) of a node-sharded run.

    Every node still runs exactly once in the job, on its owner; each rank keeps at most
    plan.nslots device blocks, spilling values (own or received) to pinned host buffers;
    operand values move between ranks by point-to-point transfers posted in the job's one
    global order (no deadlock, see plan_rank).  Executor `ex` (device: engine._BoundedExecutor,
    CPU tests: an oracle executor):

      ex.claim(slot) / ex.release(slot)      slot bookkeeping
      ex.slot(slot) -> tensor                the block buffer (P2P source / destination)
      ex.load(slot, (i, j))                  base block M_ij (1-based) into slot
      ex.node(nid, slots)                    (p, rt, l, r, out, f, w) Schur node
      ex.invert(t, (root, f, out)) -> tensor final inversion of root t (result tensor)
      ex.output(t, slot) -> tensor           root value as the result (invert_roots=False)
      ex.spill(slot, hbuf) / ex.reload(slot, hbuf)
      ex.statuses(nids) -> {nid: int}; ex.root_status(t) -> int
      ex.empty_result() -> tensor            receive buffer for a root result on rank 0
    Returns ({target: tensor} on rank 0 else None, node statuses, root statuses) — the statuses
    all-reduced so that every rank raises the reference's error."""
    import torch
    import torch.distributed as dist

    from . import bounded as bd

    if world > 1:
        dist.barrier(group=group)
    results, mine_roots = {}, []
    for op in plan.ops:
        kind = op[0]
        if kind == bd.NODE:
            for s in op[2][4:]:
                ex.claim(s)
            ex.node(op[1], op[2])
        elif kind == bd.FREE:
            ex.release(op[1])
        elif kind == bd.LOAD:
            ex.claim(op[2])
            ex.load(op[2], op[1])
        elif kind == bd.SPILL:
            ex.spill(op[2], op[3])
        elif kind == bd.RELOAD:
            ex.claim(op[2])
            ex.reload(op[2], op[3])
        elif kind == bd.SEND:
            dist.send(ex.slot(op[2]), op[3], group=group)
        elif kind == bd.RECV:
            ex.claim(op[2])
            dist.recv(ex.slot(op[2]), op[3], group=group)
        elif kind == bd.INVERT:
            t, (r, f, o) = op[1], op[2]
            ex.claim(f)
            ex.claim(o)
            results[t] = ex.invert(t, (r, f, o))
            mine_roots.append(t)
        elif kind == bd.OUTPUT:
            results[op[1]] = ex.output(op[1], op[2])
            mine_roots.append(op[1])
    owner = assign_owners(sched, world)
    st = ex.statuses([nid for nid in owner if owner[nid] == rank])
    nn = len(sched.nodes)
    flat = torch.zeros(nn + len(sched.roots), dtype=torch.int64, device=ex.device)
    for nid, v in st.items():
        flat[nid] = int(v)
    if invert_roots:
        for t in mine_roots:
            flat[nn + t] = int(ex.root_status(t))
    if world > 1:
        dist.all_reduce(flat, group=group)
    # root results to rank 0, in target order (a global order again)
    for t, nid in enumerate(sched.roots):
        o = owner[nid]
        if o == rank and rank != 0:
            dist.send(results[t].contiguous(), 0, group=group)
        elif o != rank and rank == 0:
            results[t] = ex.empty_result()
            dist.recv(results[t], o, group=group)
    host = flat.cpu().numpy()
    return (results if rank == 0 else None), host[:nn], host[nn:]
