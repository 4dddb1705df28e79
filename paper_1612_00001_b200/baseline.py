"""Dense whole-matrix inversion on the device and the verify path (reference baseline.py, cli.py:261-296).

`lu_invert_full` inverts the order-m matrix with one blocked LU factorization
and two triangular sweeps against I on the GPU (the same kernels as a block
inversion, at order m).  `verify` is the `bri verify` check as a library call:
dense-LU inverse as the yardstick, the BRI inverse (computed here, or read
from a BRIM file / passed in) as the candidate, max-norm relative gap.
"""

from __future__ import annotations

import time

import numpy as np

from .core import Workspace, invert_dense
from .errors import (DimensionMismatchError, MaterializeLimitError, SingularBlockError, SingularMatrixError,
                     UsageError)
from .instrumentation import BenchRecord
from .providers import BlockProvider

__all__ = ["lu_invert_full", "bench_lu", "materialize", "verify", "MATERIALIZE_LIMIT"]

MATERIALIZE_LIMIT = 4096


def _as_square(a):
    try:
        import torch

        if isinstance(a, torch.Tensor):
            if a.dim() != 2 or a.shape[0] != a.shape[1]:
                raise DimensionMismatchError(f"matrix must be square, got shape {tuple(a.shape)}")
            return a.to(torch.float64)
    except ImportError:  # pragma: no cover
        pass
    a = np.asarray(a, dtype=np.float64)
    if a.ndim != 2 or a.shape[0] != a.shape[1]:
        raise DimensionMismatchError(f"matrix must be square, got shape {a.shape}")
    return a


def _invert_on_device(a):
    ws = Workspace()
    work = ws.from_array(a)
    try:
        inv = invert_dense(work)
    except SingularBlockError as e:
        raise SingularMatrixError(e.pivot_index, a.shape[0]) from e
    finally:
        work.release()
    return inv


def lu_invert_full(a) -> np.ndarray:
    """Dense inverse via LU with partial pivoting (baseline.py:27-42); input left intact.

    Raises SingularMatrixError(pivot, m) under the same growth-scaled pivot test
    as a block inversion."""
    inv = _invert_on_device(_as_square(a))
    out = inv.data.copy()
    inv.release()
    return out


def bench_lu(a, seed: int):
    """One timed dense inversion with its peak bytes (baseline.py:45-66): input,
    factorization workspace and output, three order-m buffers."""
    a = _as_square(a)
    m = a.shape[0]
    t0 = time.perf_counter()
    inv = lu_invert_full(a)
    wall_ms = (time.perf_counter() - t0) * 1e3
    return inv, BenchRecord(method="lu", m=m, k=1, wall_ms=wall_ms, peak_bytes=3 * 8 * m * m,
                            n_block_inv=1, n_block_mul=0, seed=seed)


def materialize(provider: BlockProvider, trim: bool = True, limit: int = MATERIALIZE_LIMIT) -> np.ndarray:
    """A provider's matrix assembled densely (baseline.py:69-88); with `trim` the
    original m x m, else the padded working matrix with its identity corner."""
    lay = provider.layout
    if lay.n > limit:
        raise MaterializeLimitError(lay.n, limit)
    out = np.empty((lay.n, lay.n))
    b = lay.b
    for alpha in range(1, lay.k + 1):
        for beta in range(1, lay.k + 1):
            out[(alpha - 1) * b:alpha * b, (beta - 1) * b:beta * b] = provider._block(alpha, beta)
    return out[:lay.m, :lay.m] if trim else out


def verify(matrix, k: int | None = None, inverse=None, tol: float = 1e-8) -> dict:
    """`bri verify` as a call (cli.py:261-296).

    matrix / inverse: arrays or BRIM paths.  Without `inverse`, the candidate
    is invert_full over a memory provider with k blocks per side.  Returns the
    reference's report: m, max_rel_error, at, tol, pass.
    """
    from .engine import invert_full
    from .formats import MemorySink, read_matrix
    from .providers import make_memory_provider

    a = read_matrix(matrix) if isinstance(matrix, (str, bytes)) or hasattr(matrix, "__fspath__") else \
        np.asarray(matrix, dtype=np.float64)
    a = _as_square(a)
    ref = lu_invert_full(a)
    if inverse is not None:
        cand = read_matrix(inverse) if isinstance(inverse, (str, bytes)) or hasattr(inverse, "__fspath__") else \
            np.asarray(inverse, dtype=np.float64)
        if cand.shape != a.shape:
            raise UsageError(f"inverse order {cand.shape[0]} does not match input order {a.shape[0]}")
    else:
        if k is None:
            raise UsageError("verify needs k (blocks per side) when no inverse is given")
        prov = make_memory_provider(a, k)
        sink = MemorySink(prov.layout)
        invert_full(prov, sink, Workspace())
        cand = sink.finalize()
    gap = np.abs(cand - ref)
    at = np.unravel_index(int(np.argmax(gap)), gap.shape)
    rel = float(gap[at] / np.abs(ref).max())
    return {"command": "verify", "m": int(a.shape[0]), "max_rel_error": rel, "at": [int(at[0]), int(at[1])],
            "tol": tol, "pass": rel <= tol}
