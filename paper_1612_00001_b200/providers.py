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

Padded layouts (m not divisible by k, l > 0): the working matrix is
[[M, 0], [0, I]] of order m + l.  As in the reference (providers.py:338-402),
a target's run goes through an element-shifted window view (`window_maps`)
so that padding rows and columns stay paired in every pivot; the device
gathers those view blocks straight from M (bri_gather_elements) and a
finisher places the computed window into the padded output block.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .core import Block, Workspace
from .errors import BadPartitionError, DimensionMismatchError, IndexOutOfRangeError

__all__ = ["BlockLayout", "BlockPermutation", "BlockProvider", "fetch_block", "make_memory_provider",
           "permute_provider", "window_maps", "window_finisher", "make_file_provider", "KernelSpec",
           "make_kernel_provider", "kernel_matrix", "augment_provider", "cache_provider"]


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


def _window_start(lay: BlockLayout, j: int) -> int:
    """First of b consecutive real indices covering block j's real part."""
    return min((j - 1) * lay.b, lay.m - lay.b)


def window_maps(lay: BlockLayout, alpha: int, beta: int):
    """Element row / column maps of the shifted-window view for target (alpha, beta).

    The rows lead with beta's b-wide real window, the columns with alpha's;
    the remaining real indices follow (those outside both windows first, so
    the two maps agree wherever they can); the l padding indices sit at the
    same positions in both maps: up to b of them at the very end (last
    block), any overflow right after the first b - overflow fillers (the
    anchor block).  Same construction as providers.py:245-271, which keeps
    every reduction pivot generically nonsingular.
    """
    b, m, n, l = lay.b, lay.m, lay.n, lay.l
    wa, wb = _window_start(lay, alpha), _window_start(lay, beta)
    idx = np.arange(m)
    in_a = (idx >= wa) & (idx < wa + b)
    in_b = (idx >= wb) & (idx < wb + b)
    shared = idx[~(in_a | in_b)]
    pad = np.arange(m, n)
    spill = max(0, l - b)

    def arrange(lead, others):
        return np.concatenate([lead, others[: b - spill], pad[:spill], others[b - spill:], pad[spill:]])

    rows = arrange(idx[in_b], np.concatenate([shared, idx[in_a & ~in_b]]))
    cols = arrange(idx[in_a], np.concatenate([shared, idx[in_b & ~in_a]]))
    return rows, cols


def window_finisher(lay: BlockLayout, alpha: int, beta: int):
    """Map the window result (inverse rows wa.., cols wb..) to the padded block (alpha, beta)."""
    wa, wb = _window_start(lay, alpha), _window_start(lay, beta)

    def finish(win: np.ndarray) -> np.ndarray:
        out = np.zeros((lay.b, lay.b))
        rg = np.arange((alpha - 1) * lay.b, alpha * lay.b)
        cg = np.arange((beta - 1) * lay.b, beta * lay.b)
        rr, cc = rg < lay.m, cg < lay.m
        if rr.any() and cc.any():
            out[np.ix_(rr, cc)] = win[np.ix_(rg[rr] - wa, cg[cc] - wb)]
        if alpha == beta:
            padded = np.flatnonzero(~rr)
            out[padded, padded] = 1.0
        return out

    return finish


class _WindowView(BlockProvider):
    """Element-permuted view of [[M, 0], [0, I]] for one padded-target run."""

    def __init__(self, base: "BlockProvider", rmap: np.ndarray, cmap: np.ndarray):
        self.base = base
        self.layout = base.layout
        self.rmap, self.cmap = rmap, cmap

    def _block(self, alpha: int, beta: int) -> np.ndarray:
        lay = self.layout
        rows = self.rmap[(alpha - 1) * lay.b: alpha * lay.b]
        cols = self.cmap[(beta - 1) * lay.b: beta * lay.b]
        return self.base._elements(rows, cols)


class _MatrixElements:
    """Element access to [[M, 0], [0, I]] for window views of a stored M."""

    def _elements(self, rows: np.ndarray, cols: np.ndarray) -> np.ndarray:
        lay = self.layout
        a = self.matrix
        out = np.zeros((rows.size, cols.size))
        rr, cc = rows < lay.m, cols < lay.m
        out[np.ix_(rr, cc)] = a[np.ix_(rows[rr], cols[cc])]
        for i in np.flatnonzero(~rr):
            hit = np.flatnonzero(cols == rows[i])
            if hit.size:
                out[i, hit[0]] = 1.0
        return out


def _augmented_run_view(prov, alpha: int, beta: int):
    """run_view of an augmented provider (providers.py:338-402): the permuted
    provider when l == 0, else the shifted-window view plus its finisher."""
    lay = prov.layout
    if lay.l == 0:
        return permute_provider(prov, alpha, beta), None
    if lay.k >= 5 and lay.l > 2 * lay.b:
        raise BadPartitionError(
            f"order {lay.m} with k={lay.k} needs {lay.l} padding indices, more than two blocks' worth "
            f"({2 * lay.b}); use a partition with k <= 4 or one that divides the order more evenly")
    rmap, cmap = window_maps(lay, alpha, beta)
    return _WindowView(prov, rmap, cmap), window_finisher(lay, alpha, beta)


RESIDENT_FRACTION = 0.5


def upload_rows(host: np.ndarray, device: int, chunk_bytes: int = 64 << 20):
    """Host (m, n) array -> CUDA float64 tensor through two pinned staging
    chunks: the host-side copy of chunk c+1 (a memory map reads the file here)
    overlaps the H2D copy of chunk c, and nothing the size of M is pinned."""
    import torch

    m, n = host.shape
    dst = torch.empty((m, n), dtype=torch.float64, device=f"cuda:{device}")
    rows = max(1, min(m, chunk_bytes // (8 * max(n, 1))))
    bufs = [torch.empty((rows, n), dtype=torch.float64).pin_memory() for _ in range(2)]
    done = [None, None]
    stream = torch.cuda.current_stream(device)
    for c, r0 in enumerate(range(0, m, rows)):
        idx, r1 = c % 2, min(m, r0 + rows)
        if done[idx] is not None:
            done[idx].synchronize()
        np.copyto(bufs[idx][: r1 - r0].numpy(), host[r0:r1], casting="unsafe")
        dst[r0:r1].copy_(bufs[idx][: r1 - r0], non_blocking=True)
        done[idx] = torch.cuda.Event()
        done[idx].record(stream)
    return dst


class _MemoryProvider(_MatrixElements, BlockProvider):
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

    @property
    def matrix(self) -> np.ndarray:
        if self._host is None:
            t = next(iter(self._dev.values()))
            self._host = t.cpu().numpy()
            self._host.setflags(write=False)
        return self._host

    def _block(self, alpha: int, beta: int) -> np.ndarray:
        lay = self.layout
        b, m = lay.b, lay.m
        r0, c0 = (alpha - 1) * b, (beta - 1) * b
        if lay.l == 0 or (r0 + b <= m and c0 + b <= m):
            return self.matrix[r0:r0 + b, c0:c0 + b]
        out = np.zeros((b, b))  # block of [[M, 0], [0, I]]
        nr, nc = max(0, min(b, m - r0)), max(0, min(b, m - c0))
        if nr and nc:
            out[:nr, :nc] = self.matrix[r0:r0 + nr, c0:c0 + nc]
        for g in range(max(r0, c0, m), min(r0 + b, c0 + b)):
            out[g - r0, g - c0] = 1.0
        return out

    def run_view(self, alpha: int, beta: int):
        return _augmented_run_view(self, alpha, beta)

    def _device_matrix(self, device: int):
        """M resident in HBM (uploaded once), or None when it would take more
        than RESIDENT_FRACTION of the free device memory: the engine then
        streams blocks from the host instead (out-of-core)."""
        t = self._dev.get(device)
        if t is None:
            import torch

            from .device import free_bytes

            m = self.layout.m
            if 8 * m * m > RESIDENT_FRACTION * free_bytes(device):
                return None
            if self._pinned is not None:  # pinned host tensor: one async H2D copy
                t = self._pinned.to(f"cuda:{device}", non_blocking=True)
            else:
                t = upload_rows(self.matrix, device)
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


class _SourceProvider(BlockProvider):
    """Blocks of [[M, 0], [0, I]] from a user element source exposing `.m` and
    `.rect(r0, r1, c0, c1)` (reference providers.py:318-336).  The engine reads it
    block by block through its pinned host ring (no device copy of M exists)."""

    def __init__(self, source, layout: BlockLayout):
        if int(source.m) != layout.m:
            raise DimensionMismatchError(f"source order {source.m} does not match layout order {layout.m}")
        self.source = source
        self.layout = layout

    def _elements(self, rows: np.ndarray, cols: np.ndarray) -> np.ndarray:
        m = self.layout.m
        out = np.zeros((rows.size, cols.size))
        rr, cc = rows < m, cols < m
        if rr.any() and cc.any():
            r_in, c_in = rows[rr], cols[cc]
            r0, r1, c0, c1 = int(r_in.min()), int(r_in.max()) + 1, int(c_in.min()), int(c_in.max()) + 1
            rect = np.asarray(self.source.rect(r0, r1, c0, c1), dtype=np.float64)
            out[np.ix_(rr, cc)] = rect[np.ix_(r_in - r0, c_in - c0)]
        for i in np.flatnonzero(~rr):   # padding rows: the identity part of the augmentation
            hit = np.flatnonzero(cols == rows[i])
            if hit.size:
                out[i, hit[0]] = 1.0
        return out

    def _block(self, alpha: int, beta: int) -> np.ndarray:
        b = self.layout.b
        idx_r = np.arange((alpha - 1) * b, alpha * b)
        idx_c = np.arange((beta - 1) * b, beta * b)
        return self._elements(idx_r, idx_c)

    def run_view(self, alpha: int, beta: int):
        return _augmented_run_view(self, alpha, beta)


def augment_provider(source, layout: BlockLayout) -> BlockProvider:
    """Padded block provider over an element source (reference providers.py:453-464)."""
    return _SourceProvider(source, layout)


class _CachedProvider(BlockProvider):
    """Bounded LRU block cache in front of any provider (reference providers.py:417-450).

    On this engine the device arena already keeps every block a run needs resident
    (each base block is gathered once per run), so the cache only saves repeated host
    reads across runs of a slow provider; fetches still return fresh buffers."""

    def __init__(self, base: BlockProvider, capacity: int):
        import threading
        from collections import OrderedDict

        if capacity < 1:
            raise BadPartitionError(f"cache capacity must be >= 1, got {capacity}")
        self.base = base
        self.layout = base.layout
        self.capacity = int(capacity)
        self._lru: "OrderedDict[tuple, np.ndarray]" = OrderedDict()
        self._lock = threading.Lock()

    def _block(self, alpha: int, beta: int) -> np.ndarray:
        key = (alpha, beta)
        with self._lock:
            got = self._lru.get(key)
            if got is not None:
                self._lru.move_to_end(key)
                return got.copy()
        data = np.array(self.base._block(alpha, beta), dtype=np.float64)
        with self._lock:
            self._lru[key] = data
            self._lru.move_to_end(key)
            while len(self._lru) > self.capacity:
                self._lru.popitem(last=False)
        return data.copy()

    def _elements(self, rows: np.ndarray, cols: np.ndarray) -> np.ndarray:
        return self.base._elements(rows, cols)

    def run_view(self, alpha: int, beta: int):
        view, finish = self.base.run_view(alpha, beta)
        if finish is None:
            return permute_provider(self, alpha, beta), None
        return view, finish   # element windows bypass the block cache (as in the reference)


def cache_provider(provider: BlockProvider, capacity: int) -> BlockProvider:
    """Optional bounded LRU cache around any provider (reference providers.py:503-505)."""
    return _CachedProvider(provider, capacity)


class _FileProvider(_MemoryProvider):
    """BRIM file input (providers.py:166-172, 473-476) over a read-only memory map.

    When M fits the device it is streamed once into HBM through pinned staging
    chunks (`upload_rows`); otherwise the engine's host source reads only the
    blocks a run needs, through its pinned ring, straight from the map."""

    def __init__(self, path, k: int):
        from .formats import open_matrix

        mm = open_matrix(path)
        self._host = mm
        self._dev = {}
        self._pinned = None
        self.path = path
        self.layout = BlockLayout.for_order(mm.shape[0], k)


def make_file_provider(path, k: int) -> BlockProvider:
    """Provider over a BRIM file."""
    return _FileProvider(path, k)


# --------------------------------------------------------------------------
# LS-SVM kernel system matrix, generated on the device
# --------------------------------------------------------------------------

@dataclass(frozen=True)
class KernelSpec:
    """Gaussian-kernel system matrix of order n + 1 for n training inputs (providers.py:93-120).

    Entry (1,1) is 0, the rest of the first row and column are 1, interior
    (i, j) is exp(-||x_{i-1} - x_{j-1}||^2 / (2 sigma^2)) + delta_ij / gamma.
    """

    inputs: np.ndarray
    gamma: float = 1.0
    sigma: float = 1.0

    def __post_init__(self):
        x = np.ascontiguousarray(self.inputs, dtype=np.float64)
        if x.ndim == 1:
            x = x[:, None]
        if x.ndim != 2 or x.shape[0] < 1 or x.shape[1] < 1:
            raise DimensionMismatchError(f"kernel inputs must be (n, d), got {np.shape(self.inputs)}")
        if not (self.gamma > 0) or not (self.sigma > 0):
            raise BadPartitionError("kernel gamma and sigma must be positive")
        x.setflags(write=False)
        object.__setattr__(self, "inputs", x)

    @property
    def order(self) -> int:
        return self.inputs.shape[0] + 1


class KernelGenerator:
    """Device-side state of a KernelSpec: the inputs (uploaded once per device)
    and the two scalars exactly as the reference computes them
    (`sq / (-2.0 * sigma**2)`, `+ 1.0 / gamma`, providers.py:192-198)."""

    def __init__(self, spec: KernelSpec):
        self.spec = spec
        self.n, self.d = spec.inputs.shape
        self.denom = -2.0 * spec.sigma ** 2
        self.ridge = 1.0 / spec.gamma
        self._dev = {}

    def inputs_on(self, device: int):
        t = self._dev.get(device)
        if t is None:
            import torch

            t = torch.from_numpy(np.array(self.spec.inputs)).to(f"cuda:{device}")
            self._dev[device] = t
        return t

    def fill(self, arena, items, rmap=None, cmap=None) -> None:
        """Generate view blocks into arena slots: items (block row, block col, slot), 0-based."""
        arena.rbf(self, items, rmap, cmap)


def _generate_host(gen: KernelGenerator, rows: np.ndarray, cols: np.ndarray) -> np.ndarray:
    """Elements (rows x cols) of [[A, 0], [0, I]] computed on the device, returned to the host."""
    import torch

    from .device import Arena, current_device

    dev = current_device()
    nr, nc = rows.size, cols.size
    n = max(nr, nc)
    r = np.full(n, 2**31 - 1, dtype=np.int32)
    c = np.full(n, 2**31 - 2, dtype=np.int32)
    r[:nr], c[:nc] = rows, cols
    rmap = torch.from_numpy(r).to(f"cuda:{dev}")
    cmap = torch.from_numpy(c).to(f"cuda:{dev}")
    with Arena(n, 1, device=dev) as ar:
        gen.fill(ar, [(0, 0, 0)], rmap, cmap)
        return ar.view(0)[:nr, :nc].cpu().numpy()


class _KernelProvider(BlockProvider):
    """LS-SVM system matrix provider (providers.py:175-200, 479-482).

    Nothing of order m is ever stored: every block the engine loads is
    generated straight into its arena slot by `bri_rbf_blocks`, from the n x d
    inputs held on the device.  Host fetches (`fetch_block`) go through the
    same kernel.
    """

    def __init__(self, spec: KernelSpec, k: int):
        self.spec = spec
        self._gen = KernelGenerator(spec)
        self.layout = BlockLayout.for_order(spec.order, k)

    def _generator(self) -> KernelGenerator:
        return self._gen

    def _block(self, alpha: int, beta: int) -> np.ndarray:
        b = self.layout.b
        return _generate_host(self._gen, np.arange((alpha - 1) * b, alpha * b), np.arange((beta - 1) * b, beta * b))

    def _elements(self, rows: np.ndarray, cols: np.ndarray) -> np.ndarray:
        return _generate_host(self._gen, rows, cols)

    def run_view(self, alpha: int, beta: int):
        return _augmented_run_view(self, alpha, beta)


def make_kernel_provider(spec: KernelSpec, k: int) -> BlockProvider:
    """Provider over a kernel system matrix, blocks generated on the device."""
    return _KernelProvider(spec, k)


def kernel_matrix(spec: KernelSpec) -> np.ndarray:
    """The whole order-(n+1) kernel system matrix, generated on the device (providers.py:485-487)."""
    import ctypes

    import torch

    from . import _native
    from .device import current_device, stream_handle

    dev = current_device()
    gen = KernelGenerator(spec)
    m = spec.order
    out = torch.empty((m, m), dtype=torch.float64, device=f"cuda:{dev}")
    lib = _native.load_library()
    _native.context(dev)
    x = gen.inputs_on(dev)
    _native.check(lib.bri_rbf_dense(stream_handle(dev), ctypes.c_void_p(x.data_ptr()), gen.n, gen.d, gen.denom,
                                    gen.ridge, ctypes.c_void_p(out.data_ptr()), m), "bri_rbf_dense")
    return out.cpu().numpy()


# --------------------------------------------------------------------------
# Seeded Gaussian matrices generated blockwise on the device (BASELINE config 5)
# --------------------------------------------------------------------------

@dataclass(frozen=True)
class GaussianSpec:
    """M = G + shift * I of order m, G i.i.d. N(0, 1) from a counter-based stream.

    BASELINE config 5 asks for M = G + m I "generated blockwise from seed 4";
    the reference's generator (`bri gen --kind randn`, cli.py:122-130) draws
    the whole matrix from one PCG64 stream and has no blockwise form, so this
    scheme is new and documented in include/bri_b200.h (bri_randn_blocks):
    Philox4x64-10 keyed by the seed at counter (r*m + c) / 4, Box-Muller on
    the counter's output pairs.  Any block is generated independently, and
    the matrix does not depend on the partition.
    """

    order: int
    seed: int
    shift: float = 0.0

    def __post_init__(self):
        if self.order < 1:
            raise DimensionMismatchError(f"order must be positive, got {self.order}")
        if not (0 <= self.seed < 2 ** 64):
            raise BadPartitionError("seed must fit in 64 bits")


class GaussianGenerator:
    def __init__(self, spec: GaussianSpec):
        self.spec = spec

    def fill(self, arena, items, rmap=None, cmap=None) -> None:
        arena.randn(self.spec, items, rmap, cmap)


class _GaussianProvider(BlockProvider):
    """Seeded Gaussian provider: every block the engine loads is generated
    straight into its arena slot (`bri_randn_blocks`); M (215 GB at config 5)
    is never stored.  Host fetches go through the same kernel."""

    def __init__(self, spec: GaussianSpec, k: int):
        self.spec = spec
        self._gen = GaussianGenerator(spec)
        self.layout = BlockLayout.for_order(spec.order, k)

    def _generator(self) -> GaussianGenerator:
        return self._gen

    def _block(self, alpha: int, beta: int) -> np.ndarray:
        b = self.layout.b
        return _generate_host(self._gen, np.arange((alpha - 1) * b, alpha * b), np.arange((beta - 1) * b, beta * b))

    def _elements(self, rows: np.ndarray, cols: np.ndarray) -> np.ndarray:
        return _generate_host(self._gen, rows, cols)

    def run_view(self, alpha: int, beta: int):
        return _augmented_run_view(self, alpha, beta)


def make_gaussian_provider(spec: GaussianSpec, k: int) -> BlockProvider:
    """Provider over a seeded Gaussian matrix (BASELINE config 5), blocks generated on the device."""
    return _GaussianProvider(spec, k)


def gaussian_window(spec: GaussianSpec, row0: int, col0: int, rows: int, cols: int, out=None):
    """Window of M on the current device as a (rows, cols) float64 tensor (or into `out`,
    a row-major CUDA tensor with unit column stride)."""
    import ctypes

    import torch

    from . import _native
    from .device import current_device, stream_handle

    dev = current_device()
    if out is None:
        out = torch.empty((rows, cols), dtype=torch.float64, device=f"cuda:{dev}")
    lib = _native.load_library()
    _native.context(dev)
    _native.check(lib.bri_randn_window(stream_handle(dev), spec.order, spec.seed, float(spec.shift), row0, col0,
                                       rows, cols, ctypes.c_void_p(out.data_ptr()), out.stride(0)),
                  "bri_randn_window")
    return out


def permute_provider(provider: BlockProvider, alpha: int, beta: int) -> BlockProvider:
    k = provider.layout.k
    if not (1 <= alpha <= k and 1 <= beta <= k):
        raise IndexOutOfRangeError(f"target block ({alpha}, {beta}) outside 1..{k}")
    return _PermutedProvider(provider, BlockPermutation(alpha=alpha, beta=beta))
