"""Output sinks (reference formats.py:249-282).

`sink.put(alpha, beta, block)` accepts an ndarray, a torch tensor or an object
with `.data`, in any order and from any thread; `finalize()` returns the
assembled inverse or raises MissingBlocksError.  BRIM files are out of the
round-1 scope.
"""

from __future__ import annotations

import threading

import numpy as np

from .errors import IndexOutOfRangeError, MissingBlocksError

__all__ = ["MemorySink"]


def _as_host(block) -> np.ndarray:
    try:
        import torch

        if isinstance(block, torch.Tensor):
            return block.detach().cpu().numpy()
    except ImportError:  # pragma: no cover
        pass
    return np.asarray(getattr(block, "data", block))


class MemorySink:
    """Collect inverse blocks into a host (m, m) array."""

    def __init__(self, layout):
        self.layout = layout
        self.canvas = np.zeros((layout.m, layout.m))
        self._received: set = set()
        self._lock = threading.Lock()

    def put(self, alpha: int, beta: int, block) -> None:
        lay = self.layout
        if not (1 <= alpha <= lay.k and 1 <= beta <= lay.k):
            raise IndexOutOfRangeError(f"block ({alpha}, {beta}) outside 1..{lay.k}")
        data = _as_host(block)
        r0, c0 = (alpha - 1) * lay.b, (beta - 1) * lay.b
        nr, nc = min(lay.b, lay.m - r0), min(lay.b, lay.m - c0)
        with self._lock:
            if nr > 0 and nc > 0:
                self.canvas[r0:r0 + nr, c0:c0 + nc] = data[:nr, :nc]
            self._received.add((alpha, beta))

    def finalize(self) -> np.ndarray:
        lay = self.layout
        missing = [(a, b) for a in range(1, lay.k + 1) for b in range(1, lay.k + 1)
                   if (a, b) not in self._received]
        if missing:
            raise MissingBlocksError(missing)
        return self.canvas
