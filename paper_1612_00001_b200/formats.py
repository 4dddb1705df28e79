"""Sinks and the BRIM matrix file (reference formats.py:49-282).

`sink.put(alpha, beta, block)` accepts an ndarray, a torch tensor or an object
with `.data`, in any order and from any thread; `finalize()` completes the
output or raises MissingBlocksError.

BRIM (the reference's on-disk format, formats.py:1-14): a 24-byte
little-endian header — magic b"BRIM", u32 version, u64 order m, u8 dtype tag
(1 = float64), 7 reserved bytes — followed by m*m row-major float64.  A sink
writes version 0 first and stamps version 1 only in `finalize()`, so a
partial file is detectable; readers reject version 0.  `make_file_provider`
(providers.py) reads BRIM inputs through a memory map.
"""

from __future__ import annotations

import os
import struct
import threading
from dataclasses import dataclass

import numpy as np

from .errors import DimensionMismatchError, FormatError, IndexOutOfRangeError, MissingBlocksError

__all__ = ["MemorySink", "BrimSink", "BrimHeader", "BrimReader", "write_matrix", "read_header", "read_matrix",
           "open_matrix", "MAGIC", "VERSION", "HEADER_BYTES", "CSV_COLUMNS", "write_bench_csv",
           "read_bench_csv"]

MAGIC = b"BRIM"
VERSION = 1
DTYPE_F64 = 1
HEADER_BYTES = 24
_LAYOUT = struct.Struct("<4sIQB7x")


@dataclass(frozen=True)
class BrimHeader:
    m: int
    version: int = VERSION
    dtype_tag: int = DTYPE_F64

    def pack(self) -> bytes:
        return _LAYOUT.pack(MAGIC, self.version, self.m, self.dtype_tag)

    @property
    def total_bytes(self) -> int:
        return HEADER_BYTES + 8 * self.m * self.m


def _parse(raw: bytes, where: str) -> BrimHeader:
    if len(raw) < HEADER_BYTES:
        raise FormatError(f"{where}: truncated header ({len(raw)} of {HEADER_BYTES} bytes)")
    magic, version, m, tag = _LAYOUT.unpack(raw[:HEADER_BYTES])
    if magic != MAGIC:
        raise FormatError(f"{where}: bad magic {magic!r}, expected {MAGIC!r}")
    if version != VERSION:
        hint = " (version 0 marks a partial or aborted write)" if version == 0 else ""
        raise FormatError(f"{where}: unsupported version {version}{hint}")
    if tag != DTYPE_F64:
        raise FormatError(f"{where}: unsupported dtype tag {tag}, expected {DTYPE_F64}")
    return BrimHeader(m=int(m))


def read_header(path) -> BrimHeader:
    path = os.fspath(path)
    with open(path, "rb") as fh:
        head = _parse(fh.read(HEADER_BYTES), path)
        size = fh.seek(0, os.SEEK_END)
    if size != head.total_bytes:
        raise FormatError(f"{path}: expected {head.total_bytes} bytes for order {head.m}, found {size}")
    return head


def write_matrix(path, matrix) -> None:
    a = np.ascontiguousarray(matrix, dtype="<f8")
    if a.ndim != 2 or a.shape[0] != a.shape[1]:
        raise DimensionMismatchError(f"matrix must be square, got shape {a.shape}")
    with open(os.fspath(path), "wb") as fh:
        fh.write(BrimHeader(m=a.shape[0]).pack())
        a.tofile(fh)


def open_matrix(path) -> np.ndarray:
    """Read-only memory map of a BRIM payload as an (m, m) float64 array."""
    head = read_header(path)
    return np.memmap(os.fspath(path), dtype="<f8", mode="r", offset=HEADER_BYTES, shape=(head.m, head.m))


def read_matrix(path) -> np.ndarray:
    return np.array(open_matrix(path), dtype=np.float64)


class BrimReader:
    """Rectangle reads from a BRIM file (reference formats.py:127-176).

    Served from a read-only memory map, so a rectangle costs its own pages and
    concurrent readers need no seek lock; the header is validated on open."""

    def __init__(self, path):
        self.path = os.fspath(path)
        self.header = read_header(self.path)
        self._map = open_matrix(self.path)

    @property
    def m(self) -> int:
        return self.header.m

    def read_rect(self, r0: int, r1: int, c0: int, c1: int) -> np.ndarray:
        m = self.header.m
        if not (0 <= r0 <= r1 <= m and 0 <= c0 <= c1 <= m):
            raise IndexOutOfRangeError(f"rectangle [{r0}:{r1}, {c0}:{c1}] outside order {m}")
        if self._map is None:
            raise FormatError(f"{self.path}: reader is closed")
        return np.array(self._map[r0:r1, c0:c1], dtype=np.float64)

    def close(self) -> None:
        mm, self._map = self._map, None
        if mm is not None and getattr(mm, "_mmap", None) is not None:
            del mm

    def __enter__(self) -> "BrimReader":
        return self

    def __exit__(self, exc_type, exc, tb) -> None:
        self.close()


# bench CSV (reference formats.py:285-318): one BenchRecord per row
CSV_COLUMNS = ("method", "m", "k", "wall_ms", "peak_bytes", "n_block_inv", "n_block_mul", "seed")


def write_bench_csv(path, records) -> None:
    import csv

    with open(os.fspath(path), "w", newline="") as fh:
        out = csv.writer(fh)
        out.writerow(CSV_COLUMNS)
        out.writerows(rec.row() for rec in records)


def read_bench_csv(path) -> list:
    import csv

    from .instrumentation import BenchRecord

    types = (str, int, int, float, int, int, int, int)
    with open(os.fspath(path), newline="") as fh:
        rows = list(csv.reader(fh))
    if not rows or tuple(rows[0]) != CSV_COLUMNS:
        raise FormatError(f"{path}: bad bench CSV header {rows[0] if rows else None}")
    return [BenchRecord(*(t(v) for t, v in zip(types, r))) for r in rows[1:] if r]


def _as_host(block) -> np.ndarray:
    try:
        import torch

        if isinstance(block, torch.Tensor):
            return block.detach().cpu().numpy()
    except ImportError:  # pragma: no cover
        pass
    return np.asarray(getattr(block, "data", block))


class _BlockSink:
    """Shared put/finalize bookkeeping: validates (alpha, beta) and the block
    shape, trims the augmentation padding, and records arrivals; subclasses
    provide the (m, m) row-major `self._canvas` the trimmed block lands in."""

    def __init__(self, layout):
        self.layout = layout
        self._received: set = set()
        self._lock = threading.Lock()

    _pinned = None
    _pending: list = []

    def put(self, alpha: int, beta: int, block) -> None:
        if self._put_device(alpha, beta, block):
            return
        lay = self.layout
        if not (1 <= alpha <= lay.k and 1 <= beta <= lay.k):
            raise IndexOutOfRangeError(f"block ({alpha}, {beta}) outside 1..{lay.k}")
        data = _as_host(block)
        if data.shape != (lay.b, lay.b):
            raise DimensionMismatchError(f"block ({alpha}, {beta}) has shape {data.shape}, "
                                         f"expected ({lay.b}, {lay.b})")
        r0, c0 = (alpha - 1) * lay.b, (beta - 1) * lay.b
        r1, c1 = min(r0 + lay.b, lay.m), min(c0 + lay.b, lay.m)
        with self._lock:
            if r1 > r0 and c1 > c0:
                self._canvas[r0:r1, c0:c1] = data[: r1 - r0, : c1 - c0]
            self._received.add((alpha, beta))

    def _put_device(self, alpha: int, beta: int, block) -> bool:
        """A CUDA-tensor block into a pinned canvas: one async 2-D D2H copy (bri_store_host) on
        the block's current stream, no pageable bounce, no host-side copy; the canvas is
        synchronized before anyone reads it.  False when this sink cannot take that path."""
        if self._pinned is None or not getattr(block, "is_cuda", False):
            return False
        import ctypes

        import torch

        from . import _native

        lay = self.layout
        if not (1 <= alpha <= lay.k and 1 <= beta <= lay.k):
            raise IndexOutOfRangeError(f"block ({alpha}, {beta}) outside 1..{lay.k}")
        if tuple(block.shape) != (lay.b, lay.b) or block.dtype != torch.float64 or block.stride(1) != 1:
            return False
        r0, c0 = (alpha - 1) * lay.b, (beta - 1) * lay.b
        nr, nc = min(lay.b, lay.m - r0), min(lay.b, lay.m - c0)
        stream = torch.cuda.current_stream(block.device)
        with self._lock:
            if nr > 0 and nc > 0:
                host = self._pinned.data_ptr() + 8 * (r0 * lay.m + c0)
                _native.check(_native.load_library().bri_store_host(
                    ctypes.c_void_p(stream.cuda_stream), ctypes.c_void_p(host), lay.m,
                    ctypes.c_void_p(block.data_ptr()), block.stride(0), nr, nc), "bri_store_host")
                ev = torch.cuda.Event()
                ev.record(stream)
                self._pending.append((ev, block))
            self._received.add((alpha, beta))
        return True

    def _sync(self) -> None:
        with self._lock:
            pending, self._pending = self._pending, []
        for ev, _ in pending:
            ev.synchronize()

    def _check_complete(self) -> None:
        k = self.layout.k
        missing = [(a, b) for a in range(1, k + 1) for b in range(1, k + 1) if (a, b) not in self._received]
        if missing:
            raise MissingBlocksError(missing)


class BrimSink(_BlockSink):
    """Stream inverse blocks into a BRIM file (padding trimmed).

    The payload is a writable memory map over the file, so a put is one
    strided copy; the header carries version 0 until `finalize()` has seen
    all k*k blocks, then version 1 is written in place.  Closing without
    finalizing (or leaving the context on an exception) keeps the marker.
    """

    def __init__(self, path, layout):
        super().__init__(layout)
        self.path = os.fspath(path)
        m = layout.m
        with open(self.path, "wb") as fh:
            fh.write(BrimHeader(m=m, version=0).pack())
            fh.truncate(HEADER_BYTES + 8 * m * m)
        self._canvas = np.memmap(self.path, dtype="<f8", mode="r+", offset=HEADER_BYTES, shape=(m, m))
        self._finalized = False

    def finalize(self) -> None:
        self._check_complete()
        with self._lock:
            self._canvas.flush()
            fd = os.open(self.path, os.O_WRONLY)
            try:
                os.pwrite(fd, BrimHeader(m=self.layout.m).pack(), 0)
            finally:
                os.close(fd)
            self._finalized = True

    def close(self) -> None:
        if self._canvas is not None:
            self._canvas.flush()
            self._canvas = None

    def __enter__(self) -> "BrimSink":
        return self

    def __exit__(self, exc_type, exc, tb) -> None:
        try:
            if exc_type is None and not self._finalized:
                self.finalize()
        finally:
            self.close()


class MemorySink(_BlockSink):
    """Collect inverse blocks into a host (m, m) array.

    With a CUDA device present the canvas lives in pinned host memory (PyTorch's caching host
    allocator, so repeated runs reuse it) and device blocks land in it by asynchronous 2-D
    copies straight from HBM; `canvas` / `finalize()` wait for them.  Entries of blocks not
    received read as 0, as with the reference's np.zeros canvas (formats.py:249-282)."""

    def __init__(self, layout):
        super().__init__(layout)
        m = layout.m
        self._pending = []
        self._pinned = None
        try:
            import torch

            if torch.cuda.is_available() and m > 0:
                self._pinned = torch.empty((m, m), dtype=torch.float64, pin_memory=True)
        except Exception:  # pragma: no cover - no usable CUDA runtime: plain host canvas
            self._pinned = None
        self._canvas = self._pinned.numpy() if self._pinned is not None else np.zeros((m, m))
        self._zeroed = self._pinned is None

    def _zero_missing(self) -> None:
        """Pinned canvases start uninitialized: give unreceived blocks the reference's zeros."""
        if self._zeroed:
            return
        lay = self.layout
        with self._lock:
            got = set(self._received)
        for a in range(1, lay.k + 1):
            for b in range(1, lay.k + 1):
                if (a, b) not in got:
                    self._canvas[(a - 1) * lay.b:a * lay.b, (b - 1) * lay.b:b * lay.b] = 0.0
        if len(got) == lay.k * lay.k:
            self._zeroed = True

    @property
    def canvas(self) -> np.ndarray:
        self._sync()
        self._zero_missing()
        return self._canvas

    def finalize(self) -> np.ndarray:
        self._sync()
        self._check_complete()
        self._zeroed = True
        return self._canvas
