"""Engine: single-block, block-row and full inversion on the device (reference engine.py).

Public entry points keep the reference's signatures and semantics
(engine.py:183-364): `invert_block`, `invert_full`, `reduce_frame`,
`schur_eliminate`, plus `invert_block_row` (block row alpha of M^-1, the
BASELINE "block row" workload; sugar over the same run).

Execution (the host scheduler):

* "dag" schedule (default): `dag.build_schedule` deduplicates the reduction
  trees of all requested targets; every level of the DAG is ONE batched call
  `bri_schur_batch` (LU with partial pivoting of each node's pivot, the solve,
  and the fused GEMM-subtract), the roots go through `bri_invert_batch`.  The
  matrix is uploaded once and its blocks gathered on the device.  Level n-1
  values are dropped after level n, scratch slots are reused per chunk, and a
  level wider than the arena budget is processed in chunks.
* "tree" schedule: the reference's depth-first recursion (engine.py:196-241)
  one node at a time with the staged fold (factor pivot -> solve -> fused
  update), keeping <= 2 blocks per active level (the footprint contract
  <= 2k + 4).

Both schedules perform the same per-node arithmetic while b fits one
128-column LU block (bit-identical results); for larger b the LU variant
depends on the launch's batch size and results agree within 1e-9.

Errors: per-node pivot statuses come back from the device; the first failing
pivot in the reference's evaluation order is reported as
SingularPivotError(path, anchor) (engine.py:235-238); a singular root
reduction raises SingularBlockError (core.py:252-254).
"""

from __future__ import annotations

import ctypes
import os
import threading
import time
from collections import OrderedDict
from dataclasses import dataclass, field

import numpy as np

from .core import Block, Workspace
from .dag import build_from_specs, build_schedule, target_maps
from . import _native
from .device import SMALL_MAX, Arena, cached_arena, cached_bytes, current_device, free_bytes, padded_ld
from .errors import (BadPartitionError, DimensionMismatchError, IndexOutOfRangeError,
                     SingularBlockError, SingularPivotError)
from .frames import PLAN, Frame, Quadrant, root_frame, split_frame
from .instrumentation import OpCounters
from .providers import BlockProvider

__all__ = ["invert_block", "invert_block_row", "invert_blocks", "invert_blocks_sharded", "invert_full",
           "reduce_frame", "schur_eliminate", "InversionSummary", "RunInfo"]


def _torch():
    import torch

    return torch


# --------------------------------------------------------------------------
# block sources: how base blocks M_ij reach the arena
# --------------------------------------------------------------------------

class _DeviceSource:
    """Whole matrix resident in HBM; blocks gathered by one kernel launch."""

    def __init__(self, matrix, b: int):
        self.matrix, self.b = matrix, b

    def load(self, arena: Arena, items) -> None:
        arena.gather(self.matrix, [(i - 1, j - 1, s) for i, j, s in items])


class _HostSource:
    """Generic and out-of-core providers: blocks read through `_block` into a
    ring of pinned staging buffers by reader threads, then copied host -> device
    asynchronously on the run's stream, so the read (page cache, disk or a
    Python provider) of the next blocks overlaps the H2D copy of this one.
    A buffer is reused only after the copy that drained it has completed."""

    RING = 4

    def __init__(self, provider: BlockProvider):
        self.provider = provider
        self.b = provider.layout.b
        self._bufs = None
        self._events = [None] * self.RING

    def _read(self, idx: int, ij) -> None:
        ev = self._events[idx]
        if ev is not None:
            ev.synchronize()
        np.copyto(self._bufs[idx].numpy(), self.provider._block(*ij), casting="unsafe")

    def load(self, arena: Arena, items) -> None:
        from concurrent.futures import ThreadPoolExecutor

        torch = _torch()
        items = list(items)
        if not items:
            return
        R = self.RING
        if self._bufs is None:
            self._bufs = [torch.empty((self.b, self.b), dtype=torch.float64).pin_memory() for _ in range(R)]
        stream = torch.cuda.current_stream(arena.device)
        with ThreadPoolExecutor(max_workers=R) as pool:
            pending = {n: pool.submit(self._read, n % R, items[n][:2]) for n in range(min(R, len(items)))}
            for n, (_, _, s) in enumerate(items):
                pending.pop(n).result()
                idx = n % R
                arena.view(s).copy_(self._bufs[idx], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(stream)
                self._events[idx] = ev
                if n + R < len(items):
                    pending[n + R] = pool.submit(self._read, idx, items[n + R][:2])


_COPY_STREAMS: dict = {}


class _PinnedSource:
    """Matrix in pinned host memory, not resident on the device: the blocks a
    run needs are copied host -> slot (2-D async copies) on a dedicated copy
    stream, in the order the run first reads them.  `load` makes the caller's
    stream wait for its copies; `load_gated` instead returns events so a DAG
    level can factor its pivots while the other operands are still in flight.
    The events are persistent per device and thread (re-recorded every run), so
    the gated schur graph captured on them replays."""

    def __init__(self, pinned, b: int, device: int):
        torch = _torch()
        self.t, self.b, self.device = pinned, b, device
        key = (device, threading.get_ident())
        if key not in _COPY_STREAMS:
            _COPY_STREAMS[key] = (torch.cuda.Stream(device), [torch.cuda.Event() for _ in range(4)])
        self.copy, self.events = _COPY_STREAMS[key]

    def _issue(self, arena: Arena, items, ev):
        torch = _torch()
        self.copy.wait_stream(torch.cuda.current_stream(self.device))   # slots may have been in use
        arena.load_host(self.t, [(i - 1, j - 1, s) for i, j, s in items], stream=self.copy)
        ev.record(self.copy)
        return ev

    def load(self, arena: Arena, items) -> None:
        items = list(items)
        if items:
            _torch().cuda.current_stream(self.device).wait_event(self._issue(arena, items, self.events[3]))

    def load_gated(self, arena: Arena, groups):
        """groups: item lists in first-use order (at most 3); returns one event per group."""
        return [self._issue(arena, g, self.events[q]) if g else None for q, g in enumerate(groups)]


class _WindowSource:
    """Padded layouts: view blocks gathered element-wise from M on the device."""

    def __init__(self, matrix, m: int, b: int, rmap, cmap, device: int):
        torch = _torch()
        self.matrix, self.m, self.b = matrix, m, b
        self.rmap = torch.as_tensor(np.asarray(rmap, dtype=np.int32), device=f"cuda:{device}")
        self.cmap = torch.as_tensor(np.asarray(cmap, dtype=np.int32), device=f"cuda:{device}")

    def load(self, arena: Arena, items) -> None:
        arena.gather_elements(self.matrix, self.m, self.rmap, self.cmap, [(i - 1, j - 1, s) for i, j, s in items])


class _GenSource:
    """Generated providers (LS-SVM kernel matrix, seeded Gaussian matrix): blocks
    computed straight into their slots on the device; maps select a padded window view."""

    def __init__(self, gen, b: int, rmap, cmap, device: int):
        torch = _torch()
        self.gen, self.b = gen, b
        self.rmap = self.cmap = None
        if rmap is not None:
            self.rmap = torch.as_tensor(np.asarray(rmap, dtype=np.int32), device=f"cuda:{device}")
            self.cmap = torch.as_tensor(np.asarray(cmap, dtype=np.int32), device=f"cuda:{device}")

    def load(self, arena: Arena, items) -> None:
        self.gen.fill(arena, [(i - 1, j - 1, s) for i, j, s in items], self.rmap, self.cmap)


def _source_for(provider: BlockProvider, device: int):
    base, mr, mc = provider._base()
    lay = base.layout
    if hasattr(base, "_generator"):
        return _GenSource(base._generator(), lay.b, None, None, device), base, mr, mc
    if lay.l == 0 and getattr(base, "_pinned", None) is not None and device not in base._dev:
        return _PinnedSource(base._pinned, lay.b, device), base, mr, mc
    dm = base._device_matrix(device)
    if lay.l != 0:
        if dm is None:
            return _HostSource(base), base, mr, mc
        ident = np.arange(lay.n)
        return _WindowSource(dm, lay.m, lay.b, ident, ident, device), base, mr, mc
    src = _DeviceSource(dm, lay.b) if dm is not None else _HostSource(base)
    return src, base, mr, mc


# --------------------------------------------------------------------------
# run bookkeeping
# --------------------------------------------------------------------------

@dataclass
class RunInfo:
    """What one device run did (attached to InversionSummary / returned by helpers)."""

    schedule: str
    targets: int
    dag_nodes: int
    tree_nodes: int
    levels: dict = field(default_factory=dict)
    arena_slots: int = 0
    chunk: int = 0
    peak_blocks: int = 0
    spills: int = 0          # bounded runs: device -> pinned host copies of node values
    reloads: int = 0         # bounded runs: host -> device copies back
    host_blocks: int = 0     # bounded runs: pinned host blocks used for spills
    factorizations: int = 0  # DAG runs: pivot factorizations executed (shared across a level's nodes)
    solves: int = 0          # DAG runs: W = p^-1 l solves executed (shared per distinct (pivot, l))


class _TooBig(Exception):
    """The schedule's resident working set does not fit the arena budget."""


def _budget_slots(ws: Workspace, b: int, device: int) -> int:
    torch = _torch()
    block_bytes = b * padded_ld(b) * 8
    if ws.arena_bytes is not None:
        budget = ws.arena_bytes
    else:
        budget = int((free_bytes(device) + cached_bytes(device, b)) * 0.85)
    return max(1, budget // block_bytes)


def _run_dag(src, sched, ws: Workspace, device: int, trace=None, invert_roots=True):
    """Execute a schedule level by level; returns (list of root result tensors, RunInfo)."""
    torch = _torch()
    b = src.b
    levels = sched.levels()
    used = sorted(sched.m_blocks_used())
    nroots = len(sched.specs)
    keep_all = trace is not None
    width = max(len(v) for v in levels.values())
    live_values = sum(len(v) for v in levels.values()) if keep_all else sched.peak_level_blocks()
    max_slots = _budget_slots(ws, b, device)
    base_need = len(used) + live_values
    if base_need + 3 > max_slots:
        raise _TooBig(f"DAG needs {base_need} resident blocks of order {b} but the arena budget holds "
                      f"{max_slots}; raise Workspace(arena_bytes=...) or use schedule='tree'")
    # scratch per node of a chunk: factor + W (left-side solves), or factor + transposed
    # factor + S + C (right-side solves, b > SMALL_MAX)
    per = 4 if (b > SMALL_MAX and _SOLVE_SIDE != "l") else 2
    chunk = max(1, min(width, (max_slots - base_need) // per, 65535))
    nslots = min(max_slots, base_need + per * chunk + 1)
    info = RunInfo("dag", nroots, len(sched.nodes), sum(sched.tree_nodes(t) for t in range(nroots)),
                   {n: len(v) for n, v in levels.items()}, nslots, chunk)
    # one status tensor (nodes, then roots): one fill, one device -> host read
    nst = max(1, len(sched.nodes))
    # small orders on an HBM-resident matrix: the whole run is one C-ABI call (bri_dag_small)
    # whose arrays are built once per (schedule, matrix, arena) and reused
    if trace is None and b <= SMALL_MAX and isinstance(src, _DeviceSource):
        return _run_dag_small(src, sched, ws, device, invert_roots, info, nslots, chunk, nst)
    st_all = torch.zeros(nst + max(1, nroots), dtype=torch.int32, device=f"cuda:{device}")
    status, root_status = st_all[:nst], st_all[nst:]
    results = []
    arena = cached_arena(b, nslots, device, gauge=ws.gauge)
    try:
        mslot = {}
        for ij in used:
            mslot[ij] = arena.alloc()
        gates = None
        if isinstance(src, _PinnedSource) and len(levels[min(levels)]) <= chunk:
            # copy in first-use order: the level's pivots, then l, then rt and r;
            # the pivots' factorization starts as soon as they have landed
            first = [sched.nodes[nid] for nid in levels[min(levels)]]
            order, seen = [], set()
            for roles in ((0,), (2,), (1, 3)):
                grp = []
                for node in first:
                    for q in roles:
                        r = node.operands[q]
                        if r[0] == "m" and (r[1], r[2]) not in seen:
                            seen.add((r[1], r[2]))
                            grp.append((r[1], r[2], mslot[(r[1], r[2])]))
                order.append(grp)
            rest = [(i, j, s) for (i, j), s in mslot.items() if (i, j) not in seen]
            ev_p, ev_l, ev_rtr = src.load_gated(arena, order)
            if rest:
                src.load(arena, rest)
            if ev_p is not None:
                torch.cuda.current_stream(device).wait_event(ev_p)
            gates = (ev_l, ev_rtr)
        else:
            src.load(arena, [(i, j, s) for (i, j), s in mslot.items()])
        val = {}
        pos = {}      # node id -> position of its pivot status in `status`
        pbase = 0
        prev = None
        for n, ids in levels.items():
            for c0 in range(0, len(ids), chunk):
                part = ids[c0:c0 + chunk]
                slot_of = lambda r: mslot[(r[1], r[2])] if r[0] == "m" else val[r[1]]
                scratch = []
                if b > SMALL_MAX and len(part) > 2:
                    # shared work: one factorization per distinct pivot; per pivot, one solve
                    # per distinct l (W = p^-1 l, out = r - rt W) or — when its nodes share
                    # fewer distinct rt than l — per distinct rt (C = rt p^-1, out = r - C l);
                    # one fused GEMM-subtract per node
                    sides = _solve_sides(sched, part)
                    fidx, sidx, tidx, fitems, sitems, titems, ritems, gitems = {}, {}, {}, [], [], [], [], []
                    for nid in part:
                        refs = sched.nodes[nid].operands
                        if refs[0] not in fidx:
                            f = arena.alloc()
                            fidx[refs[0]] = len(fitems)
                            fitems.append((slot_of(refs[0]), f))
                            scratch.append(f)
                        out = arena.alloc()
                        if sides[refs[0]] == "l":
                            sk = ("l", refs[0], refs[2])
                            if sk not in sidx:
                                w = arena.alloc()
                                sidx[sk] = w
                                sitems.append((fidx[refs[0]], slot_of(refs[2]), w))
                                scratch.append(w)
                            gitems.append((slot_of(refs[1]), sidx[sk], slot_of(refs[3]), out))
                        else:
                            if refs[0] not in tidx:
                                ft = arena.alloc()
                                tidx[refs[0]] = len(titems)
                                titems.append((fidx[refs[0]], ft))
                                scratch.append(ft)
                            sk = ("rt", refs[0], refs[1])
                            if sk not in sidx:
                                s_, c_ = arena.alloc(), arena.alloc()
                                sidx[sk] = c_
                                ritems.append((tidx[refs[0]], slot_of(refs[1]), s_, c_))
                                scratch += (s_, c_)
                            gitems.append((sidx[sk], slot_of(refs[2]), slot_of(refs[3]), out))
                        val[nid] = out
                        pos[nid] = pbase + fidx[refs[0]]
                    lv_gates = gates if gates is not None else (None, None)
                    gates = None    # first level from pinned host: l, rt, r may still be in flight
                    arena.level(fitems, sitems, gitems, status[pbase:pbase + len(fitems)], *lv_gates,
                                titems=titems, ritems=ritems)
                    pbase += len(fitems)
                    info.factorizations += len(fitems)
                    info.solves += len(sitems) + len(ritems)
                else:
                    items = []
                    small = b <= SMALL_MAX   # the one-CTA node kernel keeps its factor in registers
                    for nid in part:
                        ops = [slot_of(r) for r in sched.nodes[nid].operands]
                        out = arena.alloc()
                        if small:
                            f = w = out
                        else:
                            f, w = arena.alloc(), arena.alloc()
                            scratch += (f, w)
                        items.append((ops[0], ops[1], ops[2], ops[3], out, f, w))
                        val[nid] = out
                        pos[nid] = pbase + len(items) - 1
                    if gates is not None:
                        arena.schur_gated(items, status[pbase:pbase + len(part)], *gates)
                        gates = None
                    else:
                        arena.schur(items, status[pbase:pbase + len(part)])
                    pbase += len(part)
                    info.factorizations += len(part)
                    info.solves += len(part)
                for s in scratch:
                    arena.release(s)
            if not keep_all:
                if prev is None:
                    # the leaves were the only readers of the matrix blocks
                    for s_ in mslot.values():
                        arena.release(s_)
                    mslot = {}
                else:
                    for nid in prev:
                        arena.release(val.pop(nid))
            prev = ids
        if invert_roots:
            for t0 in range(0, nroots, chunk):
                part = list(range(t0, min(nroots, t0 + chunk)))
                items, outs = [], []
                for t in part:
                    f, out = arena.alloc(), arena.alloc()
                    items.append((val[sched.roots[t]], f, out))
                    outs.append((f, out))
                arena.invert(items, root_status[t0:t0 + len(part)])
                # one gather for the whole chunk (the blocks are views of one result tensor)
                results += _gather_slots(arena, [out for _, out in outs])
                for f, out in outs:
                    arena.release(f)
                    arena.release(out)
        else:
            results += _gather_slots(arena, [val[sched.roots[t]] for t in range(nroots)])
        st_host = st_all.cpu().numpy()  # synchronizes the stream
        node_status = st_host[: len(sched.nodes)]
        rstat = st_host[nst:nst + nroots] if invert_roots else None
        # map device positions back to node ids
        pstat = np.zeros(len(sched.nodes), dtype=np.int64)
        for nid, p in pos.items():
            pstat[nid] = node_status[p]
        if trace is not None and not pstat.any():
            host = {}

            def on_node(nid, path, frame):
                if nid not in host:
                    host[nid] = arena.view(val[nid]).cpu().numpy().copy()
                trace(path, frame, host[nid].copy())

            for t in range(nroots):
                sched.walk(t, on_node=on_node)
        info.peak_blocks = ws.gauge.peak_blocks
    finally:
        arena.release_all()
    sched.first_failure(pstat, rstat, b)
    return results, info


@dataclass
class _SmallProgram:
    """Arrays of one small-order DAG run (bri_dag_small), built once per schedule, matrix and arena:
    slot of every matrix block / node value / result, node items level by level, the status tensor,
    and the run's peak live blocks (reported to the gauge on every run)."""

    sched: object
    arena: object
    handle: int
    args: tuple           # bri_dag_small arguments after (arena, stream)
    out_slots: list
    st_all: object
    pos_arr: object
    nst: int
    peak: int


_SMALL_PROGRAMS: "OrderedDict" = OrderedDict()


def _build_small(arena, src, sched, invert_roots, nst, device):
    torch = _torch()
    levels = sched.levels()
    used = sorted(sched.m_blocks_used())
    mslot = {ij: arena.alloc() for ij in used}
    gitems = [x for (i, j), s_ in mslot.items() for x in (i - 1, j - 1, s_)]
    val, order, counts, nitems, prev = {}, [], [], [], None
    slot_of = lambda r: mslot[(r[1], r[2])] if r[0] == "m" else val[r[1]]
    for n, ids in levels.items():
        for nid in ids:
            out = arena.alloc()
            nitems += [slot_of(r) for r in sched.nodes[nid].operands] + [out]
            val[nid] = out
            order.append(nid)
        counts.append(len(ids))
        if prev is None:   # the leaves were the only readers of the matrix blocks
            for s_ in mslot.values():
                arena.release(s_)
        else:
            for nid in prev:
                arena.release(val.pop(nid))
        prev = ids
    iitems, out_slots = [], []
    if invert_roots:
        for nid in sched.roots:
            out = arena.alloc()
            iitems += [val[nid], out]
            out_slots.append(out)
    else:
        out_slots = [val[nid] for nid in sched.roots]
    nroots = len(sched.specs)
    st_all = torch.zeros(nst + max(1, nroots), dtype=torch.int32, device=f"cuda:{device}")
    pos_arr = np.zeros(len(sched.nodes), dtype=np.int64)
    for p_, nid in enumerate(order):
        pos_arr[nid] = p_
    ia = lambda v: _native.int_array(v) if v else None
    args = (ctypes.c_void_p(src.matrix.data_ptr()), src.matrix.stride(0), len(used), ia(gitems), len(counts),
            ia(counts), ia(nitems), ctypes.c_void_p(st_all.data_ptr()), len(iitems) // 2, ia(iitems),
            ctypes.c_void_p(st_all[nst:].data_ptr()))
    peak = arena.max_live
    arena.release_all()
    return _SmallProgram(sched, arena, arena.handle.value, args, [out_slots], st_all, pos_arr, nst, peak)


def _run_dag_small(src, sched, ws, device, invert_roots, info, nslots, chunk, nst):
    """_run_dag for b <= SMALL_MAX on an HBM-resident matrix: one bri_dag_small call (gather, one
    one-CTA node launch per level, final inversions: a single CUDA graph); the call's arrays are
    cached per (schedule, matrix, arena), so a repeated run does no host-side item building."""
    key = (id(sched), src.b, device, bool(invert_roots), nslots, src.matrix.data_ptr(), src.matrix.stride(0),
           threading.get_ident())
    arena = cached_arena(src.b, nslots, device, gauge=None)
    prog = _SMALL_PROGRAMS.get(key)
    if prog is None or prog.sched is not sched or prog.arena is not arena or prog.handle != arena.handle.value:
        arena.max_live = 0
        prog = _build_small(arena, src, sched, invert_roots, nst, device)
        _SMALL_PROGRAMS[key] = prog
        if len(_SMALL_PROGRAMS) > 32:
            _SMALL_PROGRAMS.popitem(last=False)
    lib = arena.lib
    _native.check(lib.bri_dag_small(arena.handle, arena.stream, *prog.args), "bri_dag_small")
    if ws.gauge is not None and prog.peak:
        ws.gauge.on_alloc(prog.peak)    # the run held `peak` arena blocks at once
        ws.gauge.on_release(prog.peak)
    results = []
    for slots in prog.out_slots:
        results += _gather_slots(arena, slots)
    st_host = prog.st_all.cpu().numpy()  # synchronizes the stream
    pstat = st_host[: prog.nst][prog.pos_arr].astype(np.int64)
    rstat = st_host[prog.nst:prog.nst + len(sched.specs)] if invert_roots else None
    info.chunk = max(len(v) for v in sched.levels().values())
    info.peak_blocks = ws.gauge.peak_blocks if ws.gauge is not None else prog.peak
    sched.first_failure(pstat, rstat, src.b)
    return results, info


_SOLVE_SIDE = os.environ.get("BRI_SOLVE_SIDE", "auto")   # "auto" | "l" (always W = p^-1 l)


def _solve_sides(sched, part) -> dict:
    """Per distinct pivot of a level chunk: "l" (solve W = p^-1 l per distinct l) or "rt"
    (solve C = rt p^-1 per distinct rt), whichever needs fewer solves (ties: "l").
    Config 3: 3,902 -> 3,204 solves; config 4: 22,224 -> 18,012."""
    ls, rts = {}, {}
    for nid in part:
        refs = sched.nodes[nid].operands
        ls.setdefault(refs[0], set()).add(refs[2])
        rts.setdefault(refs[0], set()).add(refs[1])
    if _SOLVE_SIDE == "l":
        return {p: "l" for p in ls}
    return {p: ("rt" if len(rts[p]) < len(ls[p]) else "l") for p in ls}


def _gather_slots(arena, slots):
    """Copies of the blocks in `slots`, as (b, b) views of one new (len, b, b) tensor:
    one gather launch instead of a clone per block (config 1: 16 roots)."""
    torch = _torch()
    if not slots:
        return []
    idx = torch.as_tensor(slots, dtype=torch.long).to(arena.tensor.device, non_blocking=True)
    out = arena.tensor.index_select(0, idx)
    if out.shape[2] != arena.n:
        out = out[:, :, : arena.n].contiguous()
    return list(out.unbind(0))


def _run_tree(src, sched, ws: Workspace, device: int, trace=None, invert_roots=True):
    """The reference's depth-first recursion, one node at a time (engine.py:196-241)."""
    torch = _torch()
    b = src.b
    k = sched.k
    nslots = 2 * k + 8
    dev = f"cuda:{device}"
    results = []
    info = RunInfo("tree", len(sched.specs), len(sched.nodes),
                   sum(sched.tree_nodes(t) for t in range(len(sched.specs))), {}, nslots, 1)
    st = torch.zeros(1, dtype=torch.int32, device=dev)
    # one permutation buffer per recursion depth: a node's pivot permutation must
    # survive the evaluation of its rt and l subtrees
    perms = [torch.zeros(b, dtype=torch.int32, device=dev) for _ in range(k + 1)]
    arena = cached_arena(b, nslots, device, gauge=ws.gauge)
    try:
        for t, (frame0, mr, mc) in enumerate(sched.specs):

            def fetch(i, j):
                s = arena.alloc()
                src.load(arena, [(mr(i), mc(j), s)])
                return s

            def rec(frame: Frame, path: tuple) -> int:
                if frame.n == 2:
                    (r1, r2), (c1, c2) = frame.rows, frame.cols
                    spot = {Quadrant.A: (r1, c1), Quadrant.B: (r1, c2),
                            Quadrant.C: (r2, c1), Quadrant.D: (r2, c2)}
                    supply = {q: (lambda rc=spot[q]: fetch(*rc)) for q in spot}
                    roles = PLAN[Quadrant.D]
                else:
                    kids = {ch.label: ch for ch in split_frame(frame)}
                    supply = {q: (lambda ch=kids[q]: rec(ch, path + (ch.label,))) for q in kids}
                    roles = PLAN[frame.label.mirror]
                pq, rtq, lq, rq = roles
                perm = perms[len(path) - len(sched.paths0[t])]
                p = supply[pq]()
                arena.getrf([p], perm, st)            # factor the pivot in place
                bad = int(st.item())
                if bad:
                    arena.release_all()
                    raise SingularPivotError(path, frame.anchor)
                rt = supply[rtq]()
                l_ = supply[lq]()
                w = arena.alloc()
                arena.getrs([(p, l_, w)], perm)       # W = P^-1 l (column-major views)
                arena.release(p)
                arena.release(l_)
                r = supply[rq]()
                # r <- r - rt * W   (X-world of r - l @ inv(p) @ rt), fused in place
                arena.gemm([(rt, w, r, r)], b, b, b, alpha=-1.0, beta=1.0)
                arena.release(rt)
                arena.release(w)
                ws.executed.add_nodes(1)
                if trace is not None:
                    trace(path, frame, arena.view(r).cpu().numpy().copy())
                return r

            root = rec(frame0, sched.paths0[t])
            if invert_roots:
                f, out = arena.alloc(), arena.alloc()
                arena.invert([(root, f, out)], st)
                bad = int(st.item())
                if bad:
                    arena.release_all()
                    raise SingularBlockError(bad, b)
                results.append(arena.view(out).clone())
                for s in (root, f, out):
                    arena.release(s)
            else:
                results.append(arena.view(root).clone())
                arena.release(root)
        info.peak_blocks = ws.gauge.peak_blocks
    finally:
        arena.release_all()
    return results, info


_HOST_POOL: dict = {}


def _pool_key(device: int, b: int, ld: int):
    # per device AND per thread, like _COPY_STREAMS: concurrent bounded runs of the same
    # order from several threads (invert_full(jobs>1)) must not share spill buffers
    return (device, threading.get_ident(), b, ld)


def _pinned_pool(device: int, b: int, ld: int, count: int):
    """Pinned host blocks for spilled values, kept across runs (pinning is slow)."""
    torch = _torch()
    pool = _HOST_POOL.setdefault(_pool_key(device, b, ld), [])
    while len(pool) < count:
        pool.append(torch.empty((b, ld), dtype=torch.float64, pin_memory=True))
    return pool


def release_host_pool() -> None:
    """Unpin and free the spill buffers of bounded runs (also from PyTorch's pinned-memory cache,
    which would otherwise keep them out of the host's available memory)."""
    _HOST_POOL.clear()
    torch = _torch()
    empty = getattr(torch._C, "_host_emptyCache", None)
    if empty is not None:
        empty()


def _host_slots(ws: Workspace, b: int, device: int) -> int:
    ld = padded_ld(b)
    blk = b * ld * 8
    if ws.host_bytes is not None:
        return ws.host_bytes // blk
    import psutil

    pooled = len(_HOST_POOL.get(_pool_key(device, b, ld), ())) * blk
    return int((psutil.virtual_memory().available * 0.6 + pooled) // blk)


def _run_bounded(src, sched, ws: Workspace, device: int, trace=None, invert_roots=True):
    """Evaluate every DAG node once within the device budget (bounded.py): nodes run
    one at a time in a low-footprint order; base blocks are loaded when a node needs
    them; values evicted from the arena go to pinned host blocks and come back before
    their next reader.  All copies are on the run's stream, in plan order."""
    from . import bounded as bd

    torch = _torch()
    b = src.b
    nroots = len(sched.specs)
    # more slots than blocks the run ever holds would change nothing (and cost host time)
    cap = len(sched.nodes) + len(sched.m_blocks_used()) + 8
    p = bd.best_plan(sched, min(_budget_slots(ws, b, device), cap), max_host=_host_slots(ws, b, device),
                     invert_roots=invert_roots)
    nslots = bd.slots_used(p)
    info = RunInfo("bounded", nroots, len(sched.nodes), sum(sched.tree_nodes(t) for t in range(nroots)),
                   {n: len(v) for n, v in sched.levels().items()}, nslots, 1,
                   spills=p.spills, reloads=p.reloads, host_blocks=p.host_buffers)
    nst = max(1, len(sched.nodes))
    st_all = torch.zeros(nst + max(1, nroots), dtype=torch.int32, device=f"cuda:{device}")
    status, root_status = st_all[:nst], st_all[nst:]
    results = [None] * nroots
    host_vals = {}
    arena = cached_arena(b, nslots, device, gauge=ws.gauge)
    hbufs = _pinned_pool(device, b, arena.ld, p.host_buffers)
    try:
        for op in p.ops:
            kind = op[0]
            if kind == bd.NODE:
                nid, items = op[1], op[2]
                for s_ in items[4:]:
                    arena.claim(s_)
                arena.schur([items], status[nid:nid + 1])
                if trace is not None:
                    host_vals[nid] = arena.view(items[4]).cpu().numpy().copy()
            elif kind == bd.FREE:
                arena.release(op[1])
            elif kind == bd.LOAD:
                (i, j), s_ = op[1], op[2]
                arena.claim(s_)
                src.load(arena, [(i, j, s_)])
            elif kind == bd.SPILL:
                hbufs[op[3]].copy_(arena.tensor[op[2]], non_blocking=True)
            elif kind == bd.RELOAD:
                arena.claim(op[2])
                arena.tensor[op[2]].copy_(hbufs[op[3]], non_blocking=True)
            elif kind == bd.INVERT:
                t, (r, f, o) = op[1], op[2]
                arena.claim(f)
                arena.claim(o)
                arena.invert([(r, f, o)], root_status[t:t + 1])
                results[t] = arena.view(o).clone()
            elif kind == bd.OUTPUT:
                results[op[1]] = arena.view(op[2]).clone()
        st_host = st_all.cpu().numpy()  # synchronizes the stream
        pstat = st_host[: len(sched.nodes)].astype(np.int64)
        rstat = st_host[nst:nst + nroots] if invert_roots else None
        if trace is not None and not pstat.any():
            for t in range(nroots):
                sched.walk(t, on_node=lambda nid, path, frame: trace(path, frame, host_vals[nid].copy()))
        info.peak_blocks = ws.gauge.peak_blocks
    finally:
        arena.release_all()
    sched.first_failure(pstat, rstat, b)
    return results, info


class _ArenaExecutor:
    """Device executor of distributed.run_sharded: blocks are arena slots; received
    operands land straight in slots (NCCL P2P into arena.tensor[s])."""

    def __init__(self, arena: Arena, src, device: int, nnodes: int):
        torch = _torch()
        self.arena, self.src, self.b = arena, src, src.b
        self.device = f"cuda:{device}"
        self.st = torch.zeros(max(1, nnodes) + 1, dtype=torch.int32, device=self.device)
        self.nodes_run = 0

    def alloc(self):
        return self.arena.alloc()

    def tensor(self, h):
        return self.arena.tensor[h]

    def release(self, h):
        self.arena.release(h)

    def load(self, refs):
        out = {ij: self.arena.alloc() for ij in refs}
        self.src.load(self.arena, [(i, j, s) for (i, j), s in out.items()])
        return out

    def schur(self, items, nids):
        torch = _torch()
        if self.b <= SMALL_MAX or len(items) <= 2:
            scratch = [(self.arena.alloc(), self.arena.alloc()) for _ in items]
            tmp = torch.zeros(len(items), dtype=torch.int32, device=self.device)
            self.arena.schur([it + sc for it, sc in zip(items, scratch)], tmp)
            self.st[torch.as_tensor(nids, device=self.device)] = tmp
            for f, w in scratch:
                self.arena.release(f)
                self.arena.release(w)
            self.nodes_run += len(items)
            return
        # the rank's nodes of a level share work exactly like a one-GPU level (engine._run_dag):
        # one factorization per distinct pivot slot, one solve per distinct partner on the
        # cheaper side, one GEMM-subtract per node (bri_level_batch_ex)
        ls, rts = {}, {}
        for p, rt, l_, r, o in items:
            ls.setdefault(p, set()).add(l_)
            rts.setdefault(p, set()).add(rt)
        side = {p: ("rt" if _SOLVE_SIDE != "l" and len(rts[p]) < len(ls[p]) else "l") for p in ls}
        fidx, sidx, tidx, pos = {}, {}, {}, []
        fitems, sitems, titems, ritems, gitems, scratch = [], [], [], [], [], []
        alloc = self.arena.alloc
        for p, rt, l_, r, o in items:
            if p not in fidx:
                f = alloc()
                fidx[p] = len(fitems)
                fitems.append((p, f))
                scratch.append(f)
            if side[p] == "l":
                key = ("l", p, l_)
                if key not in sidx:
                    w = alloc()
                    sidx[key] = w
                    sitems.append((fidx[p], l_, w))
                    scratch.append(w)
                gitems.append((rt, sidx[key], r, o))
            else:
                if p not in tidx:
                    ft = alloc()
                    tidx[p] = len(titems)
                    titems.append((fidx[p], ft))
                    scratch.append(ft)
                key = ("rt", p, rt)
                if key not in sidx:
                    s_, c_ = alloc(), alloc()
                    sidx[key] = c_
                    ritems.append((tidx[p], rt, s_, c_))
                    scratch += (s_, c_)
                gitems.append((sidx[key], l_, r, o))
            pos.append(fidx[p])
        tmp = torch.zeros(len(fitems), dtype=torch.int32, device=self.device)
        self.arena.level(fitems, sitems, gitems, tmp, titems=titems, ritems=ritems)
        self.st[torch.as_tensor(nids, device=self.device)] = tmp[torch.as_tensor(pos, device=self.device)]
        for sl in scratch:
            self.arena.release(sl)
        self.nodes_run += len(items)

    def invert(self, h):
        f, o = self.arena.alloc(), self.arena.alloc()
        st = self.st[-1:]
        st.zero_()
        self.arena.invert([(h, f, o)], st)
        x = self.arena.view(o).clone()
        self.arena.release(f)
        self.arena.release(o)
        return x, int(st.item())

    def status(self, nids):
        host = self.st.cpu().numpy()
        return {nid: int(host[nid]) for nid in nids}

    def empty_result(self):
        torch = _torch()
        return torch.empty((self.b, self.b), dtype=torch.float64, device=self.device)


class _BoundedExecutor:
    """Device executor of distributed.run_sharded_bounded: a fixed arena (the rank's plan
    slots) plus pinned host buffers for spilled values; every copy and P2P transfer is
    ordered on the run's stream, exactly like the one-GPU bounded run (_run_bounded)."""

    def __init__(self, arena: Arena, src, device: int, nnodes: int, hbufs):
        torch = _torch()
        self.arena, self.src, self.b, self.hbufs = arena, src, src.b, hbufs
        self.device = f"cuda:{device}"
        self.st = torch.zeros(max(1, nnodes), dtype=torch.int32, device=self.device)
        self.rst = {}
        self.nodes_run = 0

    def claim(self, s):
        self.arena.claim(s)

    def release(self, s):
        self.arena.release(s)

    def slot(self, s):
        return self.arena.tensor[s]

    def load(self, s, ij):
        self.src.load(self.arena, [(ij[0], ij[1], s)])

    def node(self, nid, slots):
        self.arena.schur([slots], self.st[nid:nid + 1])
        self.nodes_run += 1

    def invert(self, t, slots):
        torch = _torch()
        st = torch.zeros(1, dtype=torch.int32, device=self.device)
        self.arena.invert([slots], st)
        self.rst[t] = st
        return self.arena.view(slots[2]).clone()

    def output(self, t, s):
        return self.arena.view(s)[:, : self.b].clone()

    def spill(self, s, hb):
        self.hbufs[hb].copy_(self.arena.tensor[s], non_blocking=True)

    def reload(self, s, hb):
        self.arena.tensor[s].copy_(self.hbufs[hb], non_blocking=True)

    def statuses(self, nids):
        host = self.st.cpu().numpy()
        return {nid: int(host[nid]) for nid in nids}

    def root_status(self, t):
        return int(self.rst[t].item())

    def empty_result(self):
        torch = _torch()
        return torch.empty((self.b, self.b), dtype=torch.float64, device=self.device)


def invert_blocks_sharded(provider: BlockProvider, targets, ws: Workspace | None = None, group=None):
    """Blocks `targets` of M^-1 over all ranks of the process group (one per GPU): ONE
    deduplicated DAG over every target, each level's nodes dealt to ranks with operand
    affinity, one NCCL P2P exchange of operand values per level, root blocks sent to rank 0
    (distributed.run_sharded; "one exchange step per level").  Every node
    runs once in the whole job, unlike target sharding, which repeats shared subtrees on
    each rank.  Returns (tensors in target order on rank 0 / None elsewhere, RunInfo of this
    rank); every rank raises the reference's error if a pivot fails."""
    import torch.distributed as dist

    from .distributed import assign_owners, rank_peak_blocks, run_sharded

    if ws is None:
        ws = Workspace()
    device = ws.device if ws.device is not None else current_device()
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    targets = [tuple(t) for t in targets]
    lay = provider._base()[0].layout
    for a_, b_ in targets:
        _check_target(lay, a_, b_)
    if lay.l != 0:
        raise BadPartitionError("node-sharded runs need m % k == 0 (padded layouts run per target)")
    src, base, mr, mc = _source_for(provider, device)
    k = base.layout.k
    specs = _target_specs(k, targets)(mr, mc)
    key = (k, tuple(targets)) if (mr is None and mc is None) else None
    sched = _schedule(key, k, specs, None)
    owner = assign_owners(sched, world)
    # scratch per node: f + w, or (level batch, b > SMALL_MAX) up to f + ft + s + c
    need = rank_peak_blocks(sched, owner, rank, scratch=4 if src.b > SMALL_MAX else 2)
    budget = _budget_slots(ws, src.b, device)
    # every rank decides the same way (the plans must agree on the transfer sequence)
    import torch

    flag = torch.tensor([1 if need > budget or ws.schedule == "bounded" else 0], device=f"cuda:{device}")
    if world > 1:
        dist.all_reduce(flag, group=group)
    if int(flag.item()):
        return _sharded_bounded(src, sched, owner, rank, world, ws, device, budget, targets, group)
    arena = cached_arena(src.b, need, device, gauge=ws.gauge)
    ex = _ArenaExecutor(arena, src, device, len(sched.nodes))
    try:
        res, pstat, rstat = run_sharded(sched, rank, world, ex, group=group)
    finally:
        arena.release_all()
    sched.first_failure(pstat, rstat, src.b)
    for t in range(len(sched.specs)):
        ws.counters.add_nodes(sched.tree_nodes(t), targets=1)
    ws.executed.add_nodes(ex.nodes_run, targets=sum(1 for nid in sched.roots if owner[nid] == rank))
    info = RunInfo("sharded", len(targets), len(sched.nodes), sum(sched.tree_nodes(t) for t in range(len(targets))),
                   {n: len(v) for n, v in sched.levels().items()}, need, 0, ws.gauge.peak_blocks)
    out = [res[t] for t in range(len(targets))] if res is not None else None
    return out, info


def _sharded_bounded(src, sched, owner, rank, world, ws, device, budget, targets, group):
    """invert_blocks_sharded when a rank's level-by-level footprint exceeds its budget (config 5
    on 2 / 4 / 8 GPUs): each rank replays its own bounded plan (bounded.plan_rank) — its nodes of
    each level in a low-footprint order within `budget` slots, spilled values in pinned host
    buffers (the host budget is shared by the ranks of one node), operand values exchanged
    point to point in the job's global order (distributed.run_sharded_bounded)."""
    from . import bounded as bd
    from .distributed import run_sharded_bounded

    local = int(os.environ.get("LOCAL_WORLD_SIZE", world))
    max_host = max(0, _host_slots(ws, src.b, device) // max(1, local))
    p = bd.plan_rank(sched, owner, rank, budget, max_host=max_host)
    nslots = bd.slots_used(p)
    arena = cached_arena(src.b, nslots, device, gauge=ws.gauge)
    hbufs = _pinned_pool(device, src.b, arena.ld, p.host_buffers)
    ex = _BoundedExecutor(arena, src, device, len(sched.nodes), hbufs)
    try:
        res, pstat, rstat = run_sharded_bounded(sched, rank, world, ex, p, group=group)
    finally:
        arena.release_all()
    sched.first_failure(pstat, rstat, src.b)
    for t in range(len(sched.specs)):
        ws.counters.add_nodes(sched.tree_nodes(t), targets=1)
    ws.executed.add_nodes(ex.nodes_run, targets=sum(1 for nid in sched.roots if owner[nid] == rank))
    info = RunInfo("sharded-bounded", len(targets), len(sched.nodes),
                   sum(sched.tree_nodes(t) for t in range(len(targets))),
                   {n: len(v) for n, v in sched.levels().items()}, nslots, 1, ws.gauge.peak_blocks,
                   spills=p.spills, reloads=p.reloads, host_blocks=p.host_buffers)
    out = [res[t] for t in range(len(targets))] if res is not None else None
    return out, info


_SCHED_CACHE: "OrderedDict" = OrderedDict()


def _schedule(key, k, specs, paths0):
    """build_from_specs, memoized for plain target lists (key not None): a
    schedule is immutable once built and depends only on (k, targets)."""
    if key is None:
        return build_from_specs(k, specs, paths0)
    sched = _SCHED_CACHE.get(key)
    if sched is None:
        sched = build_from_specs(k, specs, paths0)
        _SCHED_CACHE[key] = sched
        if len(_SCHED_CACHE) > 64:
            _SCHED_CACHE.popitem(last=False)
    else:
        _SCHED_CACHE.move_to_end(key)
    return sched


def _run_grouped(src, k, specs, paths0, ws, device, trace, invert_roots, key=None):
    """DAG run over all roots; if the union does not fit the arena, split the
    roots into halves (shared nodes are recomputed, memory stays bounded).
    Groups run in root order, so the first error raised is the reference's."""
    sched = _schedule(key, k, specs, paths0)
    try:
        tensors, info = _run_dag(src, sched, ws, device, trace=trace, invert_roots=invert_roots)
        return tensors, info, [sched]
    except _TooBig:
        if len(specs) == 1:
            # one target whose DAG does not fit: same nodes, bounded footprint
            tensors, info = _run_bounded(src, sched, ws, device, trace=trace, invert_roots=invert_roots)
            return tensors, info, [sched]
    h = len(specs) // 2
    p0 = paths0[:h] if paths0 is not None else None
    p1 = paths0[h:] if paths0 is not None else None
    k0 = None if key is None else key + ("lo", h)
    k1 = None if key is None else key + ("hi", h)
    t0, i0, s0 = _run_grouped(src, k, specs[:h], p0, ws, device, trace, invert_roots, k0)
    t1, i1, s1 = _run_grouped(src, k, specs[h:], p1, ws, device, trace, invert_roots, k1)
    i0.dag_nodes += i1.dag_nodes
    i0.tree_nodes += i1.tree_nodes
    i0.targets += i1.targets
    i0.arena_slots = max(i0.arena_slots, i1.arena_slots)
    return t0 + t1, i0, s0 + s1


def _execute_padded(provider: BlockProvider, targets, ws: Workspace, trace=None):
    """Padded layouts (l > 0): each target runs over its own shifted-window view
    (providers.window_maps, reference providers.py:338-402), then the finisher
    places the window into the padded output block."""
    torch = _torch()
    device = ws.device if ws.device is not None else current_device()
    base, _, _ = provider._base()
    lay = base.layout
    gen = base._generator() if hasattr(base, "_generator") else None
    dm = None if gen is not None else base._device_matrix(device)
    out, info = [], None
    for alpha, beta in targets:
        view, finish = base.run_view(alpha, beta)
        if gen is not None:
            src = _GenSource(gen, lay.b, view.rmap, view.cmap, device)
        elif dm is not None:
            src = _WindowSource(dm, lay.m, lay.b, view.rmap, view.cmap, device)
        else:  # M does not fit in HBM: stream the view's blocks from the host
            src = _HostSource(view)
        sched = build_from_specs(lay.k, [(root_frame(lay.k), None, None)])
        run = {"tree": _run_tree, "bounded": _run_bounded}.get(ws.schedule, _run_dag)
        try:
            tensors, info = run(src, sched, ws, device, trace=trace, invert_roots=True)
        except _TooBig:
            tensors, info = _run_bounded(src, sched, ws, device, trace=trace, invert_roots=True)
        ws.counters.add_nodes(sched.tree_nodes(0), targets=1)
        if ws.schedule != "tree":
            ws.executed.add_nodes(len(sched.nodes), targets=1)
        else:
            ws.executed.block_inversions += 1
        done = finish(tensors[0].cpu().numpy())
        out.append(torch.from_numpy(done).to(f"cuda:{device}"))
    return out, info


def _execute(provider: BlockProvider, specs_fn, ws: Workspace, trace=None, invert_roots=True,
             paths0=None, targets=None):
    device = ws.device if ws.device is not None else current_device()
    if targets is not None and provider._base()[0].layout.l != 0:
        return _execute_padded(provider, targets, ws, trace)
    src, base, mr, mc = _source_for(provider, device)
    k = base.layout.k
    specs = specs_fn(mr, mc)
    key = (k, tuple(targets)) if (targets is not None and mr is None and mc is None and paths0 is None) else None
    if ws.schedule in ("tree", "bounded"):
        sched = _schedule(key, k, specs, paths0)
        run = _run_tree if ws.schedule == "tree" else _run_bounded
        tensors, info = run(src, sched, ws, device, trace=trace, invert_roots=invert_roots)
        scheds = [sched]
    else:
        tensors, info, scheds = _run_grouped(src, k, specs, paths0, ws, device, trace, invert_roots, key)
    executed_nodes = sum(len(s.nodes) for s in scheds)
    sched = scheds[0]
    if len(scheds) > 1:
        sched = _schedule(key, k, specs, paths0)
    # reference accounting (tree semantics), per root
    for t in range(len(sched.specs)):
        ws.counters.add_nodes(sched.tree_nodes(t), targets=1 if invert_roots else 0)
    if ws.schedule != "tree":
        ws.executed.add_nodes(executed_nodes, targets=len(sched.specs) if invert_roots else 0)
    elif invert_roots:
        ws.executed.block_inversions += len(sched.specs)
    return tensors, info


def _compose(mr0, mc0, perm_r, perm_c):
    mr = perm_r if mr0 is None else (lambda i: mr0(perm_r(i)))
    mc = perm_c if mc0 is None else (lambda j: mc0(perm_c(j)))
    return mr, mc


def _target_specs(k: int, targets):
    def specs_fn(mr0, mc0):
        out = []
        for alpha, beta in targets:
            pr, pc = target_maps(alpha, beta)
            out.append((root_frame(k),) + _compose(mr0, mc0, pr, pc))
        return out

    return specs_fn


def _check_target(lay, alpha, beta):
    if not (1 <= alpha <= lay.k and 1 <= beta <= lay.k):
        raise IndexOutOfRangeError(f"inverse block ({alpha}, {beta}) outside 1..{lay.k}")


# --------------------------------------------------------------------------
# public API
# --------------------------------------------------------------------------

def invert_block(provider: BlockProvider, alpha: int, beta: int, ws: Workspace | None = None,
                 trace=None) -> Block:
    """Block (alpha, beta), 1-based, of M^-1 (engine.py:244-273)."""
    lay = provider.layout
    _check_target(lay, alpha, beta)
    if ws is None:
        ws = Workspace()
    tensors, _ = _execute(provider, _target_specs(lay.k, [(alpha, beta)]), ws, trace=trace,
                          targets=[(alpha, beta)])
    return Block(tensors[0], ws)


def invert_block_row(provider: BlockProvider, alpha: int, ws: Workspace | None = None) -> list:
    """Block row alpha of M^-1: [N_{alpha,1}, ..., N_{alpha,k}] as Blocks (one shared DAG run)."""
    lay = provider.layout
    _check_target(lay, alpha, 1)
    if ws is None:
        ws = Workspace()
    targets = [(alpha, beta) for beta in range(1, lay.k + 1)]
    tensors, _ = _execute(provider, _target_specs(lay.k, targets), ws, targets=targets)
    return [Block(t, ws) for t in tensors]


def invert_blocks(provider: BlockProvider, targets, ws: Workspace | None = None):
    """Any list of (alpha, beta) targets in one run; returns (tensors, RunInfo)."""
    lay = provider.layout
    for a, b in targets:
        _check_target(lay, a, b)
    if ws is None:
        ws = Workspace()
    return _execute(provider, _target_specs(lay.k, list(targets)), ws, targets=list(targets))


@dataclass
class InversionSummary:
    """Merged accounting of one full-inverse run (engine.py:276-293)."""

    m: int
    k: int
    b: int
    l: int
    wall_ms: float
    counters: OpCounters
    peak_blocks: int
    peak_bytes: int
    jobs: int = 1
    peak_blocks_bound: int = 0
    executed: OpCounters | None = None
    run: RunInfo | None = None

    def __post_init__(self):
        if self.peak_blocks_bound == 0:
            self.peak_blocks_bound = self.peak_blocks


def invert_full(provider: BlockProvider, sink, ws: Workspace | None = None, jobs: int = 1) -> InversionSummary:
    """All k*k inverse blocks streamed to sink.put(alpha, beta, data) (engine.py:296-364).

    All targets share one deduplicated device run; `jobs` is accepted for
    signature compatibility (the device batches every target at once).
    """
    lay = provider.layout
    if ws is None:
        ws = Workspace()
    before, ex_before = ws.counters.copy(), ws.executed.copy()
    ws.gauge.reset_peak()
    t0 = time.perf_counter()
    targets = [(a, b) for a in range(1, lay.k + 1) for b in range(1, lay.k + 1)]
    tensors, info = _execute(provider, _target_specs(lay.k, targets), ws, targets=targets)
    for (a, b), t in zip(targets, tensors):
        sink.put(a, b, t)
    wall_ms = (time.perf_counter() - t0) * 1e3
    merged = OpCounters(ws.counters.block_inversions - before.block_inversions,
                        ws.counters.block_multiplications - before.block_multiplications,
                        ws.counters.block_subtractions - before.block_subtractions,
                        ws.counters.schur_nodes - before.schur_nodes)
    executed = OpCounters(ws.executed.block_inversions - ex_before.block_inversions,
                          ws.executed.block_multiplications - ex_before.block_multiplications,
                          ws.executed.block_subtractions - ex_before.block_subtractions,
                          ws.executed.schur_nodes - ex_before.schur_nodes)
    peak = ws.gauge.peak_blocks
    return InversionSummary(m=lay.m, k=lay.k, b=lay.b, l=lay.l, wall_ms=wall_ms, counters=merged,
                            peak_blocks=peak, peak_bytes=peak * 8 * lay.b * lay.b, jobs=max(1, min(jobs, len(targets))),
                            peak_blocks_bound=peak, executed=executed, run=info)


def reduce_frame(provider: BlockProvider, frame: Frame, ws: Workspace | None = None, trace=None,
                 _path=None) -> Block:
    """Reduce one frame of the provider's (view) index space to a single block (engine.py:196-241).

    Branch paths reported to `trace` and in SingularPivotError start at
    `_path` (default: the frame's own label), as in the reference.
    """
    if ws is None:
        ws = Workspace()
    path0 = (frame.label,) if _path is None else tuple(_path)

    def specs_fn(mr0, mc0):
        return [(frame, mr0, mc0)]

    tensors, _ = _execute(provider, specs_fn, ws, trace=trace, invert_roots=False, paths0=[path0])
    return Block(tensors[0], ws)


def schur_eliminate(g, q: Quadrant) -> Block:
    """Schur complement of quadrant q in the 2x2 block arrangement g (engine.py:183-193).

    g = ((a, b), (c, d)) of Blocks; all four are consumed (released) and the
    result is a new block in the same workspace.  q = D gives a - b d^-1 c.
    """
    (a, b_), (c, d) = g
    blocks = {Quadrant.A: a, Quadrant.B: b_, Quadrant.C: c, Quadrant.D: d}
    n = a.order
    for blk in (b_, c, d):
        if blk.order != n:
            raise DimensionMismatchError(f"operand orders differ: {n} vs {blk.order}")
    ws = blocks[q].workspace
    pq, rtq, lq, rq = PLAN[q]
    torch = _torch()
    dev = a.tensor.device
    st = torch.zeros(1, dtype=torch.int32, device=dev)
    with Arena(n, 7, device=dev.index) as arena:
        for i, role in enumerate((pq, rtq, lq, rq)):
            arena.view(i).copy_(blocks[role].tensor)
        arena.schur([(0, 1, 2, 3, 4, 5, 6)], st)
        bad = int(st.item())
        out = arena.view(4).clone()
    if ws is not None:
        ws.counters.add_nodes(1)
        ws.executed.add_nodes(1)
    for blk in blocks.values():
        blk.release()
    if bad:
        raise SingularBlockError(bad, n)
    return Block(out, ws)
