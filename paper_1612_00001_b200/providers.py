"""Block providers: the input plugin API of the hot path (reference providers.py).

A provider exposes `.layout` (m, k, l, b), `._block(alpha, beta)` returning a
(b, b) float64 ndarray (deterministic, read-only) and `.run_view(alpha, beta)`
(providers.py:279-301).  Any object honouring that protocol can be handed to
the engine; it will be read block by block and uploaded to the device arena.

The fast route: `make_memory_provider` keeps M on the host *and* uploads it
once to HBM on first use; the engine then gathers the blocks it needs with
one device kernel (bri_gather_blocks) instead of per-fetch host copies
(providers.py:318-336 + core.py:92-98).  A CUDA tensor may be passed as the
matrix to keep M device-resident from the start.

Padded layouts (m not divisible by k, providers.py:203-271) are out of the
round-1 device scope and rejected with BadPartitionError.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .core import Block, Workspace
from .errors import BadPartitionError, DimensionMismatchError, IndexOutOfRangeError

__all__ = ["BlockLayout", "BlockPermutation", "BlockProvider", "fetch_block", "make_memory_provider",
           "permute_provider"]


@dataclass(frozen=True)
class BlockLayout:
    """Order m split into k block rows of width b, with l padding indices (providers.py:63-90)."""

    m: int
    k: int
    l: int
    b: int

    @property
    def n(self) -> int:
        return self.m + self.l

    @classmethod
    def for_order(cls, m: int, k: int) -> "BlockLayout":
        if m < 1:
            raise BadPartitionError(f"matrix order must be >= 1, got {m}")
        if k < 2:
            raise BadPartitionError(f"partition needs k >= 2, got {k}")
        l = (-m) % k
        return cls(m=m, k=k, l=l, b=(m + l) // k)


@dataclass(frozen=True)
class BlockPermutation:
    """Target (alpha, beta) exchange: rows 1<->beta, columns 1<->alpha (providers.py:123-145)."""

    alpha: int
    beta: int

    def map_row(self, i: int) -> int:
        return self.beta if i == 1 else (1 if i == self.beta else i)

    def map_col(self, j: int) -> int:
        return self.alpha if j == 1 else (1 if j == self.alpha else j)


class BlockProvider:
    """Abstract block source over one layout."""

    layout: BlockLayout

    def _block(self, alpha: int, beta: int) -> np.ndarray:
        raise NotImplementedError

    def fetch_block(self, alpha: int, beta: int, ws: Workspace | None = None) -> Block:
        k = self.layout.k
        if not (1 <= alpha <= k and 1 <= beta <= k):
            raise IndexOutOfRangeError(f"block ({alpha}, {beta}) outside 1..{k}")
        return Block(self._block(alpha, beta), ws)

    def run_view(self, alpha: int, beta: int):
        return permute_provider(self, alpha, beta), None

    # engine hooks -----------------------------------------------------
    def _base(self):
        """(base provider, row map, col map) this provider reads through."""
        return self, None, None

    def _device_matrix(self, device: int):
        """Dense device copy of the whole matrix, or None if not available."""
        return None


class _MemoryProvider(BlockProvider):
    """Blocks of an in-memory matrix (l = 0); host copy plus a lazily uploaded device copy."""

    def __init__(self, matrix, k: int):
        import torch

        if isinstance(matrix, torch.Tensor):
            if matrix.dim() != 2 or matrix.shape[0] != matrix.shape[1]:
                raise DimensionMismatchError(f"matrix must be square, got shape {tuple(matrix.shape)}")
            self._dev = {matrix.device.index: matrix.to(torch.float64).contiguous()} if matrix.is_cuda else {}
            self._pinned = (matrix.contiguous() if (not matrix.is_cuda and matrix.is_pinned()
                                                    and matrix.dtype == torch.float64) else None)
            host = None if matrix.is_cuda else matrix.to(torch.float64).numpy()
            m = matrix.shape[0]
        else:
            host = np.array(matrix, dtype=np.float64, order="C", copy=True)
            if host.ndim != 2 or host.shape[0] != host.shape[1]:
                raise DimensionMismatchError(f"matrix must be square, got shape {host.shape}")
            host.setflags(write=False)
            self._dev = {}
            self._pinned = None
            m = host.shape[0]
        self._host = host
        self.layout = BlockLayout.for_order(m, k)
        if self.layout.l != 0:
            raise BadPartitionError(
                f"order {m} is not divisible by k={k}: padded layouts are not supported on the device path yet")

    @property
    def matrix(self) -> np.ndarray:
        if self._host is None:
            t = next(iter(self._dev.values()))
            self._host = t.cpu().numpy()
            self._host.setflags(write=False)
        return self._host

    def _block(self, alpha: int, beta: int) -> np.ndarray:
        b = self.layout.b
        return self.matrix[(alpha - 1) * b: alpha * b, (beta - 1) * b: beta * b]

    def _device_matrix(self, device: int):
        t = self._dev.get(device)
        if t is None:
            import torch

            if self._pinned is not None:  # pinned host tensor: one async H2D copy
                t = self._pinned.to(f"cuda:{device}", non_blocking=True)
            else:
                src = torch.from_numpy(np.array(self.matrix, copy=True))
                t = src.pin_memory().to(f"cuda:{device}", non_blocking=True)
            self._dev[device] = t
        return t


class _PermutedProvider(BlockProvider):
    """Lazy index-mapped view (providers.py:405-414)."""

    def __init__(self, base: BlockProvider, perm: BlockPermutation):
        self.base = base
        self.perm = perm
        self.layout = base.layout

    def _block(self, alpha: int, beta: int) -> np.ndarray:
        return self.base._block(self.perm.map_row(alpha), self.perm.map_col(beta))

    def _base(self):
        base, mr0, mc0 = self.base._base()
        pr, pc = self.perm.map_row, self.perm.map_col
        mr = pr if mr0 is None else (lambda i: mr0(pr(i)))
        mc = pc if mc0 is None else (lambda j: mc0(pc(j)))
        return base, mr, mc


def fetch_block(provider: BlockProvider, alpha: int, beta: int, ws: Workspace | None = None) -> Block:
    return provider.fetch_block(alpha, beta, ws)


def make_memory_provider(matrix, k: int) -> BlockProvider:
    """Provider over an in-memory square matrix (numpy array or torch tensor)."""
    return _MemoryProvider(matrix, k)


def permute_provider(provider: BlockProvider, alpha: int, beta: int) -> BlockProvider:
    k = provider.layout.k
    if not (1 <= alpha <= k and 1 <= beta <= k):
        raise IndexOutOfRangeError(f"target block ({alpha}, {beta}) outside 1..{k}")
    return _PermutedProvider(provider, BlockPermutation(alpha=alpha, beta=beta))
