"""Device slot arena: the bounded-HBM block store behind every BRI run.

An arena is one torch CUDA tensor of shape (nslots, n, ld) float64 — slot s
holds one b x b block with exactly the bytes of the reference's C-ordered
ndarray (row stride ld, ld a multiple of 8) — wrapped by a `bri_arena` handle
that carries the TMA descriptors the kernels load through.  Slots are handed
out by a free list and every allocation is reported to the workspace gauge,
so `MemoryGauge.peak_blocks` is the run's true device footprint in blocks.

PyTorch supplies the memory and the stream; all arithmetic is in
libbri_b200.so (`_native.py`).
"""

from __future__ import annotations

import ctypes
import threading

from . import _native
from .errors import BadPartitionError, DeviceError


def _torch():
    import torch

    return torch


def current_device() -> int:
    torch = _torch()
    if not torch.cuda.is_available():
        raise DeviceError("CUDA device required: the BRI hot path runs only on the GPU")
    return torch.cuda.current_device()


def stream_handle(device: int):
    return ctypes.c_void_p(_torch().cuda.current_stream(device).cuda_stream)


_FREE0: dict = {}


def free_bytes(device: int) -> int:
    """Device memory available to this process: free + PyTorch's cached-but-unused.

    cudaMemGetInfo costs milliseconds (occasionally ~100 ms) per call, so it is
    queried once per device; afterwards the estimate follows PyTorch's own
    reservations (other processes' later allocations are not seen)."""
    torch = _torch()
    if device not in _FREE0:
        free, _ = torch.cuda.mem_get_info(device)
        _FREE0[device] = (free, _torch_bytes(device)[0])
    free0, res0 = _FREE0[device]
    reserved, allocated = _torch_bytes(device)
    return max(0, free0 - (reserved - res0)) + (reserved - allocated)


def _torch_bytes(device: int):
    """(reserved, allocated) bytes of PyTorch's caching allocator.  Reads the raw
    nested statistics: torch.cuda.memory_reserved() flattens all of them first
    (~0.2 ms per call, on every run's critical host path)."""
    torch = _torch()
    try:
        st = torch._C._cuda_memoryStats(device)
        return int(st["reserved_bytes"]["all"]["current"]), int(st["allocated_bytes"]["all"]["current"])
    except (AttributeError, KeyError, TypeError):
        return torch.cuda.memory_reserved(device), torch.cuda.memory_allocated(device)


# orders up to this run whole Schur nodes in one CTA (small.cu; csrc/bri_internal.h SMALL_MAX)
SMALL_MAX = 96


def padded_ld(n: int) -> int:
    return (n + 7) // 8 * 8


class Arena:
    """nslots device blocks of order n plus a free list and gauge hooks."""

    def __init__(self, n: int, nslots: int, device: int | None = None, gauge=None):
        torch = _torch()
        if n < 1 or nslots < 1:
            raise BadPartitionError(f"arena needs n >= 1 and nslots >= 1, got {n}, {nslots}")
        self.device = current_device() if device is None else device
        self.n = n
        self.ld = padded_ld(n)
        self.nslots = nslots
        self.gauge = gauge
        self.lib = _native.load_library()
        self.ctx = _native.context(self.device)
        try:
            self.tensor = torch.empty((nslots, n, self.ld), dtype=torch.float64, device=f"cuda:{self.device}")
        except torch.cuda.OutOfMemoryError as e:  # pragma: no cover - depends on device
            raise BadPartitionError(
                f"arena of {nslots} blocks of order {n} ({nslots * n * self.ld * 8 / 2**30:.1f} GiB) "
                f"does not fit in device memory") from e
        handle = ctypes.c_void_p()
        _native.check(self.lib.bri_arena_create(self.ctx, ctypes.c_void_p(self.tensor.data_ptr()), n,
                                                self.ld, nslots, ctypes.byref(handle)), "bri_arena_create")
        self.handle = handle
        self._free = list(range(nslots - 1, -1, -1))
        self._live = set()
        self.max_live = 0      # most slots live at once since the last reset (engine._build_small)

    def _call(self, name: str, *args) -> None:
        """Issue one C-ABI entry point."""
        _native.check(getattr(self.lib, name)(*args), name)

    # ------------------------------------------------------------ slots
    def alloc(self) -> int:
        if not self._free:
            raise BadPartitionError(f"arena exhausted ({self.nslots} blocks of order {self.n})")
        s = self._free.pop()
        self._live.add(s)
        if len(self._live) > self.max_live:
            self.max_live = len(self._live)
        if self.gauge is not None:
            self.gauge.on_alloc()
        return s

    def claim(self, s: int) -> None:
        """Take a specific free slot (plans that assign slots themselves, bounded.py)."""
        self._free.remove(s)
        self._live.add(s)
        if self.gauge is not None:
            self.gauge.on_alloc()

    def release(self, s: int) -> None:
        self._live.remove(s)
        self._free.append(s)
        if self.gauge is not None:
            self.gauge.on_release()

    def release_all(self) -> None:
        for s in list(self._live):
            self.release(s)

    def reset(self, gauge=None) -> None:
        """Reuse for a new run: every slot free, accounting to `gauge`."""
        self.release_all()
        self.gauge = gauge
        self._free = list(range(self.nslots - 1, -1, -1))

    @property
    def live(self) -> int:
        return len(self._live)

    def view(self, s: int):
        """Row-major (n, n) view of slot s (the reference block's layout)."""
        return self.tensor[s, :, : self.n]

    @property
    def stream(self):
        return stream_handle(self.device)

    # ------------------------------------------------------------ ops
    def _items(self, flat):
        return _native.int_array(flat)

    def schur(self, items, status) -> None:
        """items: list of (p, rt, l, r, out, f, w) slot tuples; status: int32 device tensor."""
        flat = [s for it in items for s in it]
        self._call("bri_schur_batch", self.handle, self.stream, len(items), self._items(flat),
                   ctypes.c_void_p(status.data_ptr()))

    def level(self, fitems, sitems, gitems, fstatus, ev_l=None, ev_rtr=None, titems=(), ritems=()) -> None:
        """One DAG level with shared work (bri_level_batch_ex): fitems (p, F) factor each distinct
        pivot once, sitems (factor index, l, W) solve each distinct (pivot, l) once, titems
        (factor index, Ft) / ritems (titem index, rt, S, C) solve C = rt p^-1 once per distinct
        (pivot, rt) for pivots solved from the right, gitems (A, B, r, out) one fused
        GEMM-subtract per node ((rt, W, ...) or (C, l, ...)); fstatus: int32 device tensor (nf).
        ev_l / ev_rtr: torch.cuda.Events the solves / GEMMs wait on (operands in flight)."""
        arr = lambda items: self._items([s for it in items for s in it]) if items else None
        h = lambda ev: ctypes.c_void_p(ev.cuda_event) if ev is not None else None
        _native.check(self.lib.bri_level_batch_ex(self.handle, self.stream, len(fitems), arr(fitems), len(sitems),
                                                  arr(sitems), len(titems), arr(titems), len(ritems), arr(ritems),
                                                  len(gitems), arr(gitems), ctypes.c_void_p(fstatus.data_ptr()),
                                                  h(ev_l), h(ev_rtr)),
                      "bri_level_batch")

    def schur_gated(self, items, status, ev_l, ev_rtr) -> None:
        """schur() whose l / (rt, r) operands may still be in flight: the stream waits on
        the torch.cuda.Events ev_l / ev_rtr (or None) before reading them."""
        flat = [s for it in items for s in it]
        h = lambda ev: ctypes.c_void_p(ev.cuda_event) if ev is not None else None
        _native.check(self.lib.bri_schur_batch_gated(self.handle, self.stream, len(items), self._items(flat),
                                                     ctypes.c_void_p(status.data_ptr()), h(ev_l), h(ev_rtr)),
                      "bri_schur_batch_gated")

    def load_host(self, host, items, stream=None) -> None:
        """Copy blocks of a pinned row-major host tensor into slots: items (block row, block col, slot), 0-based."""
        flat = [s for it in items for s in it]
        st = self.stream if stream is None else ctypes.c_void_p(stream.cuda_stream)
        _native.check(self.lib.bri_load_host_blocks(self.handle, st, ctypes.c_void_p(host.data_ptr()), host.stride(0),
                                                    len(items), self._items(flat)), "bri_load_host_blocks")

    def invert(self, items, status) -> None:
        """items: list of (in, f, out)."""
        flat = [s for it in items for s in it]
        self._call("bri_invert_batch", self.handle, self.stream, len(items), self._items(flat),
                   ctypes.c_void_p(status.data_ptr()))

    def getrf(self, slots, perm, status, ipiv=None) -> None:
        _native.check(self.lib.bri_getrf_batch(
            self.handle, self.stream, len(slots), self._items(list(slots)),
            ctypes.c_void_p(ipiv.data_ptr()) if ipiv is not None else None,
            ctypes.c_void_p(perm.data_ptr()), ctypes.c_void_p(status.data_ptr())), "bri_getrf_batch")

    def getrs(self, items, perm) -> None:
        """items: list of (f, src, dst)."""
        flat = [s for it in items for s in it]
        _native.check(self.lib.bri_getrs_batch(self.handle, self.stream, len(items), self._items(flat),
                                               ctypes.c_void_p(perm.data_ptr())), "bri_getrs_batch")

    def gemm(self, items, M, N, K, a0=(0, 0), b0=(0, 0), c0=(0, 0), alpha=1.0, beta=0.0) -> None:
        """Column-major window GEMM on slots; items: list of (A, B, C_in, C_out)."""
        flat = [s for it in items for s in it]
        _native.check(self.lib.bri_gemm(self.handle, self.stream, len(items), self._items(flat), M, N, K,
                                        a0[0], a0[1], b0[0], b0[1], c0[0], c0[1], alpha, beta), "bri_gemm")

    def axpby(self, items, alpha, beta) -> None:
        flat = [s for it in items for s in it]
        _native.check(self.lib.bri_axpby(self.handle, self.stream, len(items), self._items(flat),
                                         alpha, beta), "bri_axpby")

    def transpose(self, items) -> None:
        flat = [s for it in items for s in it]
        _native.check(self.lib.bri_transpose(self.handle, self.stream, len(items), self._items(flat)),
                      "bri_transpose")

    def gather(self, matrix, items) -> None:
        """Copy blocks of a device row-major matrix: items (block row, block col, slot), 0-based."""
        flat = [s for it in items for s in it]
        self._call("bri_gather_blocks", self.handle, self.stream, ctypes.c_void_p(matrix.data_ptr()),
                   matrix.stride(0), len(items), self._items(flat))

    def gather_elements(self, matrix, m, rmap, cmap, items) -> None:
        """Padded-view gather: items (block row, block col, slot); rmap/cmap int32 device tensors."""
        flat = [s for it in items for s in it]
        _native.check(self.lib.bri_gather_elements(
            self.handle, self.stream, ctypes.c_void_p(matrix.data_ptr()), matrix.stride(0), m,
            ctypes.c_void_p(rmap.data_ptr()), ctypes.c_void_p(cmap.data_ptr()), len(items), self._items(flat)),
            "bri_gather_elements")

    def rbf(self, gen, items, rmap=None, cmap=None) -> None:
        """Generate kernel-matrix view blocks into slots (gen: providers.KernelGenerator);
        items (block row, block col, slot), 0-based; rmap/cmap int32 device tensors or None."""
        flat = [s for it in items for s in it]
        x = gen.inputs_on(self.device)
        _native.check(self.lib.bri_rbf_blocks(
            self.handle, self.stream, ctypes.c_void_p(x.data_ptr()), gen.n, gen.d, gen.denom, gen.ridge,
            ctypes.c_void_p(rmap.data_ptr()) if rmap is not None else None,
            ctypes.c_void_p(cmap.data_ptr()) if cmap is not None else None, len(items), self._items(flat)),
            "bri_rbf_blocks")

    def randn(self, spec, items, rmap=None, cmap=None) -> None:
        """Generate view blocks of a providers.GaussianSpec matrix into slots: items
        (block row, block col, slot), 0-based; rmap/cmap int32 device tensors or None."""
        flat = [s for it in items for s in it]
        _native.check(self.lib.bri_randn_blocks(
            self.handle, self.stream, spec.order, spec.seed, float(spec.shift),
            ctypes.c_void_p(rmap.data_ptr()) if rmap is not None else None,
            ctypes.c_void_p(cmap.data_ptr()) if cmap is not None else None, len(items), self._items(flat)),
            "bri_randn_blocks")

    def close(self) -> None:
        if getattr(self, "handle", None) is not None:
            if self.gauge is not None and self._live:
                self.release_all()
            self.lib.bri_arena_destroy(self.handle)
            self.handle = None
            self.tensor = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):  # pragma: no cover - best effort
        try:
            if getattr(self, "handle", None) is not None:
                self.lib.bri_arena_destroy(self.handle)
                self.handle = None
        except Exception:
            pass


_CACHE: dict = {}


def _cache_key(device: int):
    # one arena per (device, thread): concurrent runs from several threads (the
    # reference's invert_full(jobs > 1) pattern) never share slots; each thread
    # also drives its own bri_ctx (_native.context)
    return (device, threading.get_ident())


def cached_arena(n: int, nslots: int, device: int, gauge=None) -> Arena:
    """One reusable arena per device and thread: repeated runs of the same geometry
    keep the same device addresses (so their CUDA graphs replay) and skip reallocation."""
    key = _cache_key(device)
    ar = _CACHE.get(key)
    if ar is not None and ar.handle is not None and ar.n == n and ar.nslots >= nslots:
        ar.reset(gauge)
        return ar
    if ar is not None:
        ar.close()
        _CACHE.pop(key, None)
    ar = Arena(n, nslots, device=device, gauge=gauge)
    _CACHE[key] = ar
    return ar


def cached_bytes(device: int, n: int) -> int:
    """Device bytes held by this thread's cached arena that a run of order n could reuse."""
    ar = _CACHE.get(_cache_key(device))
    if ar is None or ar.handle is None:
        return 0
    return ar.nslots * ar.n * ar.ld * 8


def release_cached_memory() -> None:
    """Free the cached arenas (their memory returns to PyTorch's allocator)."""
    for ar in list(_CACHE.values()):
        ar.close()
    _CACHE.clear()


def fp64_peak_tflops(iters: int = 4096) -> float:
    """Measured DMMA throughput of this GPU (register-only mma.sync loop)."""
    lib = _native.load_library()
    out = ctypes.c_double()
    dev = current_device()
    _native.context(dev)
    _native.check(lib.bri_fp64_peak(stream_handle(dev), iters, ctypes.byref(out)), "bri_fp64_peak")
    return out.value
