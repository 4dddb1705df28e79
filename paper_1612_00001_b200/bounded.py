"""Host scheduler for DAG runs larger than the device: a bounded-footprint plan.

The level-by-level DAG run (engine._run_dag) keeps two adjacent levels of
node values resident; for BASELINE config 5 (k=8, b=20480: 3.36 GB per block)
that is 164 blocks = 550 GB, three times one B200.  The reference's answer to
"M does not fit" is the literal recursion with its <= 2k+4 live blocks
(SPEC.md:286), which re-evaluates shared subtrees: 5,461
nodes instead of the DAG's 270 for one config-5 target.

This module plans a third schedule: every distinct node is still evaluated
exactly once (the DAG's work), but in a topological order chosen to keep few
values alive, with a fixed number of device slots.  When a slot is needed and
none is free, the resident block whose next use is farthest away is evicted
(Belady): a base-matrix block is simply dropped (it is re-loaded from its
source), a node value is copied once to a pinned host buffer (values are
immutable, so a value evicted a second time needs no copy) and copied back
before its next reader.  Config 5 at 45 device slots: 270 nodes, a few dozen
3.36 GB spills, i.e. ~1% of the node arithmetic in PCIe time.

`plan()` is pure Python (tested on CPU); engine._run_bounded replays the op
list on the device, one node per launch.  Spilling moves bytes, never
arithmetic: a run with spills is bit-identical to the same plan without.
"""

from __future__ import annotations

import random
from dataclasses import dataclass, field

from .errors import BadPartitionError

__all__ = ["low_footprint_order", "Plan", "plan", "plan_rank", "best_plan", "peak_live", "slots_used"]

# op kinds of a plan
LOAD = "load"        # ("load", (i, j), slot): base block M_ij from the source
SPILL = "spill"      # ("spill", nid, slot, hbuf): value -> pinned host buffer hbuf
RELOAD = "reload"    # ("reload", nid, slot, hbuf): host buffer -> slot
NODE = "node"        # ("node", nid, (p, rt, l, r, out, f, w))
INVERT = "invert"    # ("invert", t, (root_slot, f, out)): final inversion of root t
OUTPUT = "output"    # ("output", t, slot): root t's (un-inverted) value is the result
FREE = "free"        # ("free", slot): slot returns to the free list (no copy)
HFREE = "hfree"      # ("hfree", hbuf): host buffer no longer needed
SEND = "send"        # ("send", nid, slot, dst rank): node-sharded runs, value -> another rank
RECV = "recv"        # ("recv", nid, slot, src rank): a value from another rank lands in slot


def _consumers(sched):
    kids = {}
    for node in sched.nodes:
        kids[node.nid] = [r[1] for r in node.operands if r[0] == "v"]
    cons = {n.nid: 0 for n in sched.nodes}
    parents = {n.nid: [] for n in sched.nodes}
    for nid, ks in kids.items():
        for c in ks:
            cons[c] += 1
            parents[c].append(nid)
    return kids, cons, parents


def low_footprint_order(sched, seed: int | None = None) -> list:
    """Topological order of every node of `sched` that keeps few values live.

    Greedy list scheduling: among the ready nodes, run the one that retires the
    most operand values (last reader), then the highest order (closer to a
    root), then the smallest node id.  Roots are kept alive until their target
    is inverted, which happens right after the root is produced.
    Config 5 (k=8, one target): 64 live values at peak vs 164 for the
    level-by-level run and 115 for the reference's post-order memoization.
    """
    kids, cons, parents = _consumers(sched)
    rng = random.Random(seed) if seed is not None else None
    rem = dict(cons)
    done = set()
    waiting = {nid: len(set(ks)) for nid, ks in kids.items()}
    ready = sorted(nid for nid, w in waiting.items() if w == 0)
    order = []
    while ready:
        best, best_key = None, None
        for nid in ready:
            ks = kids[nid]
            frees = sum(1 for c in set(ks) if rem[c] == ks.count(c))
            key = (-frees, -sched.nodes[nid].n, rng.random() if rng is not None else nid)
            if best_key is None or key < best_key:
                best, best_key = nid, key
        ready.remove(best)
        order.append(best)
        done.add(best)
        for c in kids[best]:
            rem[c] -= 1
        for p in set(parents[best]):
            waiting[p] -= 1
            if waiting[p] == 0:
                ready.append(p)
    if len(order) != len(sched.nodes):  # pragma: no cover - schedules are DAGs by construction
        raise RuntimeError("schedule is not acyclic")
    return order


def peak_live(sched, order) -> int:
    """Peak number of live node values when evaluating `order` with immediate frees."""
    kids, cons, _ = _consumers(sched)
    rem = dict(cons)
    roots = set(sched.roots)
    live = peak = 0
    for nid in order:
        live += 1
        for c in kids[nid]:
            rem[c] -= 1
            if rem[c] == 0 and c not in roots:
                live -= 1
        peak = max(peak, live)
        if nid in roots and rem[nid] == 0:
            live -= 1          # inverted right away
    return peak


@dataclass
class Plan:
    ops: list
    nslots: int
    host_buffers: int = 0     # peak pinned host buffers in use
    spills: int = 0           # device -> host copies
    reloads: int = 0          # host -> device copies
    loads: int = 0            # base-block loads from the source
    transfers: int = 0        # node-sharded plans: sends + receives
    peak_slots: int = 0
    order: list = field(default_factory=list)


def plan(sched, nslots: int, max_host: int | None = None, invert_roots: bool = True,
         order: list | None = None, keep_host: bool = True) -> Plan:
    """Op list evaluating every node of `sched` once within `nslots` device slots.

    Each node needs its 4 operands plus 3 fresh slots (out, factor scratch,
    solve scratch) resident at once; each root inversion needs the root plus 2.
    Raises BadPartitionError when nslots < 7 or more than `max_host` host
    buffers would be needed.
    """
    # a plan never holds more than every value and base block at once
    if nslots >= 7:
        nslots = min(nslots, len(sched.nodes) + len(sched.m_blocks_used()) + 8)
    if order is None:
        order = low_footprint_order(sched)
    root_of = {}
    for t, nid in enumerate(sched.roots):
        root_of.setdefault(nid, []).append(t)
    # the access sequence: one step per node (its operands), then per root inversion
    steps = []
    for nid in order:
        steps.append(("node", nid, _refs(sched, nid)))
        for t in root_of.get(nid, ()):
            steps.append(("invert" if invert_roots else "output", t, [("v", nid)]))
    return _plan_steps(steps, nslots, max_host, keep_host, order)


def _refs(sched, nid):
    return [("m", r[1], r[2]) if r[0] == "m" else ("v", r[1]) for r in sched.nodes[nid].operands]


def plan_rank(sched, owner: dict, rank: int, nslots: int, max_host: int | None = None,
              invert_roots: bool = True, order: list | None = None) -> Plan:
    """Bounded-footprint plan of ONE rank of a node-sharded run (distributed.run_sharded_bounded).

    The job's step list is level-synchronous and identical on every rank: for each DAG level,
    first the level's operand transfers in `distributed.level_transfers` order (a SEND reads a
    value this rank owns or holds, a RECV lands a value from another rank in a fresh slot),
    then this rank's own nodes of the level (in `order`, default the low-footprint order), each
    root inverted right after it is produced.  The same Belady eviction as `plan` keeps the
    rank within `nslots` device slots, spilling values — own or received — to pinned host
    buffers.  Every rank posts its transfers in one global order, so blocking point-to-point
    transfers cannot deadlock (the earliest unfinished transfer always has both ends posted).
    """
    from .distributed import level_transfers

    if order is None:
        order = low_footprint_order(sched)
    rank_pos = {nid: i for i, nid in enumerate(order)}
    root_of = {}
    for t, nid in enumerate(sched.roots):
        root_of.setdefault(nid, []).append(t)
    steps = []
    for n, ids in sched.levels().items():
        for src, dst, nid in level_transfers(sched, owner, ids):
            if src == rank:
                steps.append(("send", (nid, dst), [("v", nid)]))
            elif dst == rank:
                steps.append(("recv", (nid, src), []))
        for nid in sorted((i for i in ids if owner[i] == rank), key=rank_pos.__getitem__):
            steps.append(("node", nid, _refs(sched, nid)))
            for t in root_of.get(nid, ()):
                steps.append(("invert" if invert_roots else "output", t, [("v", nid)]))
    mine = [nid for nid in order if owner[nid] == rank]
    return _plan_steps(steps, nslots, max_host, True, mine)


def _plan_steps(steps, nslots: int, max_host, keep_host: bool, order) -> Plan:
    """Belady slot assignment over an access sequence (see `plan`)."""
    need = 7
    if nslots < need:
        raise BadPartitionError(f"a bounded DAG run needs at least {need} device blocks, the budget holds {nslots}")
    # next-use positions for Belady, per entity
    uses: dict = {}
    for pos, (_, _, refs) in enumerate(steps):
        for e in refs:
            uses.setdefault(e, []).append(pos)
    ptr = {e: 0 for e in uses}

    def next_use(e, pos):
        lst = uses.get(e, ())
        i = ptr.get(e, 0)
        while i < len(lst) and lst[i] < pos:
            i += 1
        ptr[e] = i
        return lst[i] if i < len(lst) else None

    free = list(range(nslots - 1, -1, -1))
    where: dict = {}          # entity -> slot (resident)
    host: dict = {}           # node id -> host buffer holding a valid copy
    hfree: list = []
    hcount = 0
    out = Plan(ops=[], nslots=nslots, order=list(order))
    ops = out.ops

    def take(pos, pinned):
        nonlocal hcount
        if free:
            return free.pop()
        # evict the resident entity (not needed by this step) used farthest in the future
        victim, far = None, -1
        for e, s in where.items():
            if e in pinned:
                continue
            nu = next_use(e, pos)
            d = float("inf") if nu is None else nu
            if d > far:
                victim, far = e, d
        if victim is None:  # pragma: no cover - nslots >= 7 guarantees a victim
            raise BadPartitionError("bounded plan: no evictable block")
        s = where.pop(victim)
        if victim[0] == "v" and far != float("inf") and victim[1] not in host:
            if hfree:
                hb = hfree.pop()
            else:
                if max_host is not None and hcount >= max_host:
                    raise BadPartitionError(
                        f"bounded DAG run needs more than {max_host} pinned host blocks for spills; "
                        f"raise Workspace(host_bytes=...) or the device budget, or use schedule='tree'")
                hb = hcount
                hcount += 1
            host[victim[1]] = hb
            ops.append((SPILL, victim[1], s, hb))
            out.spills += 1
        elif victim[0] == "v" and far == float("inf") and victim[1] in host:
            hb = host.pop(victim[1])
            ops.append((HFREE, hb))
            hfree.append(hb)
        ops.append((FREE, s))
        return s

    def retire(e, pos):
        """Drop e if it has no use after pos."""
        if next_use(e, pos + 1) is None:
            s = where.pop(e)
            ops.append((FREE, s))
            free.append(s)
            if e[0] == "v" and e[1] in host:
                hb = host.pop(e[1])
                ops.append((HFREE, hb))
                hfree.append(hb)

    for pos, (kind, ident, refs) in enumerate(steps):
        pinned = set(refs)
        slots = []
        for e in refs:
            if e not in where:
                s = take(pos, pinned)
                if e[0] == "m":
                    ops.append((LOAD, (e[1], e[2]), s))
                    out.loads += 1
                else:
                    if e[1] not in host:  # pragma: no cover - values are produced before use
                        raise RuntimeError(f"value {e[1]} read before it was produced")
                    ops.append((RELOAD, e[1], s, host[e[1]]))
                    out.reloads += 1
                    if not keep_host:
                        hb = host.pop(e[1])
                        ops.append((HFREE, hb))
                        hfree.append(hb)
                where[e] = s
            slots.append(where[e])
        produced = None
        if kind == "node":
            fresh = [take(pos, pinned) for _ in range(3)]
            ops.append((NODE, ident, tuple(slots) + tuple(fresh)))
            o, f, w = fresh
            ops.append((FREE, f))
            ops.append((FREE, w))
            free += [w, f]
            produced = ident
            where[("v", ident)] = o
        elif kind == "recv":
            nid, peer = ident
            o = take(pos, pinned)
            ops.append((RECV, nid, o, peer))
            out.transfers += 1
            produced = nid
            where[("v", nid)] = o
        elif kind == "send":
            nid, peer = ident
            ops.append((SEND, nid, slots[0], peer))
            out.transfers += 1
        elif kind == "output":
            ops.append((OUTPUT, ident, slots[0]))
        else:
            fresh = [take(pos, pinned) for _ in range(2)]
            ops.append((INVERT, ident, (slots[0],) + tuple(fresh)))
            ops.append((FREE, fresh[0]))
            ops.append((FREE, fresh[1]))
            free += [fresh[1], fresh[0]]
        for e in set(refs):
            if e in where:
                retire(e, pos)
        if produced is not None:
            e = ("v", produced)
            if next_use(e, pos + 1) is None:
                retire(e, pos)
        out.peak_slots = max(out.peak_slots, nslots - len(free))
    out.host_buffers = hcount
    return out


def best_plan(sched, nslots: int, max_host: int | None = None, invert_roots: bool = True,
              tries: int | None = None) -> Plan:
    """The plan with the fewest pinned host buffers (then spills, then loads) over the
    deterministic greedy order and `tries` randomized tie-breaks of it (default 64 for
    schedules up to 2,000 nodes; config 5 at 45 slots: 58 host blocks -> 29).
    Memoized on the schedule per (nslots, invert_roots)."""
    cache = sched.__dict__.setdefault("_bounded_plans", {})
    key = (nslots, invert_roots)
    best = cache.get(key)
    if best is None:
        if tries is None:
            tries = 64 if len(sched.nodes) <= 2000 else 0
        best_key = None
        for seed in [None] + list(range(tries)):
            p = plan(sched, nslots, None, invert_roots, order=low_footprint_order(sched, seed))
            k = (p.host_buffers, p.spills, p.loads)
            if best_key is None or k < best_key:
                best, best_key = p, k
        cache[key] = best
    if max_host is not None and best.host_buffers > max_host:
        raise BadPartitionError(
            f"bounded DAG run needs {best.host_buffers} pinned host blocks for spilled values but the "
            f"host budget holds {max_host}; raise Workspace(host_bytes=...) or the device budget, "
            f"or use schedule='tree'")
    return best


def slots_used(p: Plan) -> int:
    """Highest device slot index the plan touches, plus one (the arena size it needs)."""
    top = -1
    for op in p.ops:
        kind = op[0]
        if kind in (LOAD, SPILL, RELOAD, SEND, RECV):
            top = max(top, op[2])
        elif kind in (NODE, INVERT):
            top = max(top, *op[2])
        elif kind in (OUTPUT,):
            top = max(top, op[2])
        elif kind == FREE:
            top = max(top, op[1])
    return top + 1
