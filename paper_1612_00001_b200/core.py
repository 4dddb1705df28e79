"""Device-resident blocks and the primitive block operations (reference core.py).

`Block` keeps its b x b float64 buffer in HBM (a torch CUDA tensor with the
reference's row-major layout); `.data` is a host numpy copy made on demand
(and cached until the device buffer changes), `.tensor` is the device view.
Every Block registers with its workspace gauge and must be released exactly
once (core.py:78-128).

The primitive operations keep the reference's names, counters and error
behaviour (core.py:173-263) and run on libbri_b200.so:

* `multiply`      — TMA/DMMA GEMM (gemm.cu)                 core.py:173-181
* `subtract`      — axpby kernel                            core.py:184-197
* `invert_dense`  — blocked LU + pivot test + solves        core.py:238-263
* `lu_factor`     — blocked LU of x itself                  core.py:212-235

They are the drop-in surface for single-block use; the engine's hot path
does not call them (it batches whole DAG levels, engine.py).
"""

from __future__ import annotations

import os

import numpy as np

from .device import Arena, current_device
from .errors import DimensionMismatchError, GaugeUnderflowError, SingularBlockError
from .instrumentation import MemoryGauge, OpCounters

__all__ = ["Block", "LuFactors", "Workspace", "multiply", "subtract", "lu_factor", "invert_dense"]


def _torch():
    import torch

    return torch


class Workspace:
    """Per-run context: tree-semantics counters, executed counters, gauge, schedule.

    schedule: "dag" (default) evaluates each distinct reduction node once,
    level by level, batched on the device; "tree" follows the reference's
    depth-first evaluation one node at a time with its bounded footprint
    (<= 2k + 4 live blocks).  "bounded" evaluates each distinct
    node once in a low-footprint order within the device budget, spilling
    node values to pinned host memory (bounded.py); "dag" switches to it by
    itself when one target's DAG does not fit.  All return the same values.
    The default (schedule=None) is "dag", or the BRI_SCHEDULE environment variable:
    the DAG run trades the reference's <= 2k+4 live-block contract
    for evaluating every distinct node once; "tree" keeps the contract exactly.
    arena_bytes: device-memory budget of one run (default: 85% of free HBM).
    host_bytes: pinned host memory a bounded run may use for spilled values
    (default: 60% of the host's available memory).
    """

    __slots__ = ("counters", "gauge", "executed", "schedule", "arena_bytes", "host_bytes", "device")

    def __init__(self, counters: OpCounters | None = None, gauge: MemoryGauge | None = None, *,
                 schedule: str | None = None, arena_bytes: int | None = None, host_bytes: int | None = None,
                 device: int | None = None):
        if schedule is None:   # process-wide default: BRI_SCHEDULE=tree keeps the reference's <= 2k+4 bound
            schedule = os.environ.get("BRI_SCHEDULE", "dag")
        if schedule not in ("dag", "tree", "bounded"):
            raise ValueError(f"schedule must be 'dag', 'tree' or 'bounded', got {schedule!r}")
        self.counters = counters if counters is not None else OpCounters()
        self.gauge = gauge if gauge is not None else MemoryGauge()
        self.executed = OpCounters()
        self.schedule = schedule
        self.arena_bytes = arena_bytes
        self.host_bytes = host_bytes
        self.device = device

    def adopt(self, buf) -> "Block":
        return Block(buf, self)

    def from_array(self, a, copy: bool = True) -> "Block":
        torch = _torch()
        if isinstance(a, torch.Tensor):   # device or host tensor: copied on the device side
            t = a.to(device=_dev(self), dtype=torch.float64)
            if copy and t.data_ptr() == a.data_ptr():
                t = t.clone(memory_format=torch.contiguous_format)
            return Block(t.contiguous(), self)
        return Block(np.array(a, dtype=np.float64, order="C", copy=True) if copy else a, self)

    def zeros(self, order: int) -> "Block":
        torch = _torch()
        return Block(torch.zeros((order, order), dtype=torch.float64, device=_dev(self)), self)

    def identity(self, order: int) -> "Block":
        torch = _torch()
        return Block(torch.eye(order, dtype=torch.float64, device=_dev(self)), self)


def _dev(ws) -> str:
    d = ws.device if ws is not None and ws.device is not None else current_device()
    return f"cuda:{d}"


def _to_host(t) -> np.ndarray:
    """D2H into pinned memory from PyTorch's caching host allocator (full PCIe rate,
    no page faults); the ndarray shares and keeps alive that buffer."""
    torch = _torch()
    t = t.detach()
    if t.numel() * t.element_size() < (1 << 20):
        return t.cpu().numpy()
    host = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    host.copy_(t)
    return host.numpy()


class Block:
    """One square float64 block resident in device memory."""

    __slots__ = ("_t", "_host", "_ws", "_released")

    def __init__(self, buf, ws: Workspace | None = None):
        torch = _torch()
        if isinstance(buf, torch.Tensor):
            if buf.dim() != 2 or buf.shape[0] != buf.shape[1]:
                raise DimensionMismatchError(f"block buffer must be square, got {tuple(buf.shape)}")
            t = buf
            if not t.is_cuda or t.dtype != torch.float64:
                t = t.to(device=_dev(ws), dtype=torch.float64)
        else:
            a = np.asarray(buf, dtype=np.float64)
            if a.ndim != 2 or a.shape[0] != a.shape[1]:
                raise DimensionMismatchError(f"block buffer must be square, got {a.shape}")
            t = torch.from_numpy(np.ascontiguousarray(a)).to(_dev(ws))
        self._t = t
        self._host = None
        self._ws = ws
        self._released = False
        if ws is not None:
            ws.gauge.on_alloc()

    @property
    def order(self) -> int:
        return self._t.shape[0]

    @property
    def workspace(self) -> Workspace | None:
        return self._ws

    @property
    def tensor(self):
        """Device (order, order) row-major view."""
        return self._t

    @property
    def data(self) -> np.ndarray:
        """Host copy (numpy, C-ordered); refreshed after device-side updates."""
        if self._host is None:
            self._host = _to_host(self._t)
        return self._host

    def _touch(self) -> None:
        self._host = None

    def release(self) -> None:
        if self._released:
            raise GaugeUnderflowError("block released twice")
        self._released = True
        if self._ws is not None:
            self._ws.gauge.on_release()

    def copy(self) -> "Block":
        return Block(self._t.clone(), self._ws)

    def __repr__(self) -> str:  # pragma: no cover
        return f"Block(order={self.order}, {'released' if self._released else 'live'}, device)"


class LuFactors:
    """Packed LU (unit lower + upper, row-major) and 1-based pivots of one block (core.py:131-159)."""

    __slots__ = ("packed_lu", "pivots", "_ws", "_released")

    def __init__(self, packed_lu: np.ndarray, pivots: np.ndarray, ws: Workspace | None):
        self.packed_lu = packed_lu
        self.pivots = pivots
        self._ws = ws
        self._released = False
        if ws is not None:
            ws.gauge.on_alloc()

    @property
    def order(self) -> int:
        return self.packed_lu.shape[0]

    def release(self) -> None:
        if self._released:
            raise GaugeUnderflowError("LU factors released twice")
        self._released = True
        if self._ws is not None:
            self._ws.gauge.on_release()


def _same_order(*blocks) -> int:
    n = blocks[0].order
    for b in blocks[1:]:
        if b.order != n:
            raise DimensionMismatchError(f"operand orders differ: {n} vs {b.order}")
    return n


def _count(ws, field: str) -> None:
    if ws is not None:
        setattr(ws.counters, field, getattr(ws.counters, field) + 1)
        setattr(ws.executed, field, getattr(ws.executed, field) + 1)


class _Scratch:
    """Short-lived arena holding copies of the operands of one primitive op."""

    def __init__(self, blocks, extra: int):
        n = blocks[0].order
        self.arena = Arena(n, len(blocks) + extra, device=blocks[0].tensor.device.index)
        for i, b in enumerate(blocks):
            self.arena.view(i).copy_(b.tensor)

    def __enter__(self):
        return self.arena

    def __exit__(self, *exc):
        self.arena.close()


def multiply(x: Block, y: Block) -> Block:
    """x @ y as one new block; counts one multiplication (core.py:173-181)."""
    n = _same_order(x, y)
    with _Scratch([x, y], 1) as ar:
        # row-major x @ y == column-major (y^ x^): A = y, B = x
        ar.gemm([(1, 0, 2, 2)], n, n, n, alpha=1.0, beta=0.0)
        out = Block(ar.view(2).clone(), x._ws)
    _count(x._ws, "block_multiplications")
    return out


def subtract(x: Block, y: Block, in_place: bool = False) -> Block:
    """x - y; with in_place the result overwrites x and x is returned (core.py:184-197)."""
    _same_order(x, y)
    with _Scratch([x, y], 1) as ar:
        ar.axpby([(0, 1, 2)], 1.0, -1.0)
        if in_place:
            x.tensor.copy_(ar.view(2))
            x._touch()
            out = x
        else:
            out = Block(ar.view(2).clone(), x._ws)
    _count(x._ws, "block_subtractions")
    return out


def _status_tensor(n: int, device):
    torch = _torch()
    return torch.zeros(n, dtype=torch.int32, device=device)


def invert_dense(x: Block) -> Block:
    """X^-1 via LU with partial pivoting + solves against I; counts one inversion.

    Raises SingularBlockError(pivot_index, order) on the growth-scaled test
    |u_ii| <= b*eps*max|A| of core.py:200-209.  The input is left intact (the
    reference leaves it unspecified).
    """
    n = x.order
    with _Scratch([x], 2) as ar:
        st = _status_tensor(1, x.tensor.device)
        ar.invert([(0, 1, 2)], st)
        bad = int(st.item())
        if bad:
            raise SingularBlockError(bad, n)
        out = Block(ar.view(2).clone(), x._ws)
    _count(x._ws, "block_inversions")
    return out


def lu_factor(x: Block) -> LuFactors:
    """P A = L U of x itself (row pivoting, core.py:212-235); no counter bump."""
    torch = _torch()
    n = x.order
    with _Scratch([x], 1) as ar:
        ar.transpose([(0, 1)])          # slot 1, column-major view == x
        st = _status_tensor(1, x.tensor.device)
        perm = torch.zeros(n, dtype=torch.int32, device=x.tensor.device)
        ar.getrf([1], perm, st)
        ar.transpose([(1, 0)])          # back to row-major packed factors
        bad = int(st.item())
        if bad:
            raise SingularBlockError(bad, n)
        packed = ar.view(0).cpu().numpy().copy()
        pivots = perm.cpu().numpy().astype(np.int64) + 1
    return LuFactors(packed, pivots, x._ws)
