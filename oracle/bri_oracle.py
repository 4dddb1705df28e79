"""CPU oracle for the BRI hot path — TEST INFRASTRUCTURE ONLY.

This module is a numpy/scipy restatement of the reference package's hot path
(`/root/reference/pkg/src/bri`), used as the checker for the CUDA path and as
the CPU baseline leg of `bench.py`.  Only `tests/`, `__graft_entry__.smoke()`
and `bench.py` (cpu_baseline / `--impl reference`) may import it; the product
package `paper_1612_00001_b200` never does.

Parity pin: the arithmetic lives in third-party BLAS/LAPACK that is not part
of `/root/reference` (pins `numpy>=1.24`, `scipy>=1.10`, `pkg/pyproject.toml:11-14`;
in this image numpy 2.3.5 + OpenBLAS 0.3.30, scipy 1.18.1).  The restatement
issues the *same* LAPACK/BLAS calls in the same order as the reference:

* `multiply`      -> `x @ y`                                  (core.py:173-181)
* `subtract`      -> `np.subtract(x, y, out=x)`               (core.py:184-197)
* `invert_dense`  -> `dgetrf` in place on the F-view `x.T`,
                     growth-scaled pivot test, `dgetrs` vs I  (core.py:200-209, 238-263)
* `_fold`         -> `r - l @ (inv(p) @ rt)` with `_PLAN`     (engine.py:146-180)
* `reduce_frame`  -> leaf eliminates D, node eliminates mirror (engine.py:196-241)
* `invert_block`  -> permuted view + root inversion           (engine.py:244-273,
                                                               providers.py:123-145)

so on the same machine it is bit-identical to the reference; that is checked
against golden vectors produced by the reference itself
(`tests/golden/make_golden.py`) in `tests/test_oracle.py`.

`memo=True` evaluates each distinct (base rows, base cols, label|None) frame
once.  The reference documents that node values depend only on that key
(engine.py:214-236); memoization is bit-identical to the literal tree walk
 and is what makes configs 3-5 CPU-feasible.
"""

from __future__ import annotations

import numpy as np
from scipy.linalg import lapack

EPS = float(np.finfo(np.float64).eps)

# Quadrant labels as plain strings; mirror A<->D, B<->C (engine.py:65-83).
MIRROR = {"A": "D", "D": "A", "B": "C", "C": "B"}
# result = r - l @ (inv(pivot) @ rt); roles (pivot, rt, l, r) (engine.py:149-154).
PLAN = {
    "D": ("D", "C", "B", "A"),
    "C": ("C", "D", "A", "B"),
    "B": ("B", "A", "D", "C"),
    "A": ("A", "B", "C", "D"),
}


class OracleSingular(Exception):
    """Singular pivot (pivot_index 1-based) — mirrors SingularBlockError (errors.py:26-39)."""

    def __init__(self, pivot_index, order):
        self.pivot_index = int(pivot_index)
        self.order = int(order)
        super().__init__(f"singular block: pivot {pivot_index} (order {order})")


class OracleSingularPivot(Exception):
    """Singular pivot inside the tree — mirrors SingularPivotError (errors.py:53-69)."""

    def __init__(self, path, pivot_block):
        self.path = tuple(path)
        self.pivot_block = tuple(pivot_block)
        super().__init__(f"singular pivot at {'/'.join(self.path)} block {self.pivot_block}")


# --------------------------------------------------------------------------
# block arithmetic (core.py)
# --------------------------------------------------------------------------

def singular_index(diag: np.ndarray, order: int, scale: float) -> int:
    """First 1-based index with |u_ii| <= order*eps*scale, NaN-flagged (core.py:200-209)."""
    tol = order * EPS * scale
    ok = np.abs(diag) > tol
    if ok.all():
        return 0
    return int(np.flatnonzero(~ok)[0]) + 1


def invert_dense(x: np.ndarray) -> np.ndarray:
    """X^-1 exactly as core.py:238-263: dgetrf on the transposed (F) view, in place."""
    x = np.array(x, dtype=np.float64, order="C", copy=True)
    order = x.shape[0]
    scale = float(np.abs(x).max()) if order else 0.0
    lu, piv, info = lapack.dgetrf(x.T, overwrite_a=1)
    if info < 0:
        raise ValueError(f"illegal LAPACK argument {-info}")
    bad = singular_index(lu.diagonal(), order, scale)
    if bad:
        raise OracleSingular(bad, order)
    res = np.zeros((order, order))
    np.fill_diagonal(res, 1.0)
    _, info = lapack.dgetrs(lu, piv, res.T, trans=0, overwrite_b=1)
    if info != 0:
        raise OracleSingular(abs(info), order)
    return res


def lu_factor(x: np.ndarray):
    """(packed_lu, pivots 1-based) as core.py:212-235 (row-pivoted LU of x itself)."""
    x = np.asarray(x, dtype=np.float64)
    order = x.shape[0]
    scale = float(np.abs(x).max()) if order else 0.0
    lu, piv, info = lapack.dgetrf(x)
    bad = singular_index(lu.diagonal(), order, scale)
    if bad:
        raise OracleSingular(bad, order)
    perm = np.arange(order)
    for i, p in enumerate(piv):
        if p != i:
            perm[i], perm[p] = perm[p], perm[i]
    return np.ascontiguousarray(lu), perm + 1


def fold(pivot, rt, l, r):
    """One Schur node: r - l @ (inv(pivot) @ rt) (engine.py:157-180)."""
    inv = invert_dense(pivot)
    t = inv @ rt
    u = l @ t
    r = np.array(r, dtype=np.float64, order="C", copy=True)
    np.subtract(r, u, out=r)
    return r


# --------------------------------------------------------------------------
# frames (engine.py:88-143) and views (providers.py:123-145)
# --------------------------------------------------------------------------

def split_frame(rows, cols):
    """Children (A, B, C, D) of a frame, order n-1 (engine.py:119-132)."""
    rx = (rows[2], rows[1]) + tuple(rows[3:])
    cx = (cols[2], cols[1]) + tuple(cols[3:])
    return (
        (tuple(rows[:-1]), tuple(cols[:-1]), "A"),
        (tuple(rows[:-1]), cx, "B"),
        (rx, tuple(cols[:-1]), "C"),
        (rx, cx, "D"),
    )


def view_maps(alpha: int, beta: int):
    """Block permutation for target (alpha, beta): rows 1<->beta, cols 1<->alpha."""

    def map_row(i):
        return beta if i == 1 else (1 if i == beta else i)

    def map_col(j):
        return alpha if j == 1 else (1 if j == alpha else j)

    return map_row, map_col


class BlockSource:
    """k x k blocks of a dense row-major matrix (l = 0 layouts only)."""

    def __init__(self, matrix: np.ndarray, k: int):
        a = np.ascontiguousarray(matrix, dtype=np.float64)
        m = a.shape[0]
        if m % k:
            raise ValueError("oracle supports l = 0 layouts (m divisible by k)")
        self.a, self.k, self.b, self.m = a, k, m // k, m

    def block(self, i: int, j: int) -> np.ndarray:
        b = self.b
        return np.array(self.a[(i - 1) * b : i * b, (j - 1) * b : j * b], order="C", copy=True)


# --------------------------------------------------------------------------
# recursion (engine.py:196-273)
# --------------------------------------------------------------------------

class Reducer:
    """reduce_frame over one target's view; optional memo keyed on base indices."""

    def __init__(self, src: BlockSource, alpha: int, beta: int, memo=None, trace=None,
                 counters=None):
        self.src = src
        self.map_row, self.map_col = view_maps(alpha, beta)
        self.memo = memo
        self.trace = trace
        self.counters = counters if counters is not None else {"nodes": 0, "executed": 0}

    def fetch(self, i, j):
        return self.src.block(self.map_row(i), self.map_col(j))

    def key(self, rows, cols, label):
        n = len(rows)
        return (
            tuple(self.map_row(r) for r in rows),
            tuple(self.map_col(c) for c in cols),
            label if n > 2 else None,
        )

    def reduce(self, rows, cols, label, path):
        n = len(rows)
        self.counters["nodes"] += 1
        key = self.key(rows, cols, label) if self.memo is not None else None
        if key is not None and key in self.memo:
            hit = self.memo[key]
            if isinstance(hit, OracleSingularPivot):
                raise OracleSingularPivot(path, (rows[1], cols[1]))
            out = hit.copy()
            if self.trace is not None:
                self._replay_trace(rows, cols, label, path, out)
            return out
        if n == 2:
            (r1, r2), (c1, c2) = rows, cols
            spots = {"A": (r1, c1), "B": (r1, c2), "C": (r2, c1), "D": (r2, c2)}
            supply = {q: (lambda rc=rc: self.fetch(*rc)) for q, rc in spots.items()}
            q = "D"
        else:
            supply = {}
            for ch_rows, ch_cols, ch_label in split_frame(rows, cols):
                supply[ch_label] = (
                    lambda cr=ch_rows, cc=ch_cols, cl=ch_label: self.reduce(cr, cc, cl, path + (cl,))
                )
            q = MIRROR[label]
        pq, rtq, lq, rq = PLAN[q]
        p = supply[pq]()
        try:
            inv = invert_dense(p)
        except OracleSingular as e:
            raise OracleSingularPivot(path, (rows[1], cols[1])) from e
        rt = supply[rtq]()
        t = inv @ rt
        l_ = supply[lq]()
        u = l_ @ t
        r = supply[rq]()
        np.subtract(r, u, out=r)
        self.counters["executed"] += 1
        if key is not None:
            self.memo[key] = r.copy()
        if self.trace is not None:
            self.trace(path, (rows, cols, label), r.copy())
        return r

    def _replay_trace(self, rows, cols, label, path, value):
        # A memo hit stands for a whole subtree: replay its node values in the
        # reference's visiting order (children first, root of subtree last).
        if len(rows) > 2:
            for ch_rows, ch_cols, ch_label in split_frame(rows, cols):
                k = self.key(ch_rows, ch_cols, ch_label)
                self._replay_trace(ch_rows, ch_cols, ch_label, path + (ch_label,), self.memo[k])
        self.trace(path, (rows, cols, label), value.copy())


def invert_block(matrix_or_src, k, alpha, beta, memo=False, trace=None, counters=None):
    """Block (alpha, beta), 1-based, of M^-1 via BRI (engine.py:244-273)."""
    src = matrix_or_src if isinstance(matrix_or_src, BlockSource) else BlockSource(matrix_or_src, k)
    if not (1 <= alpha <= src.k and 1 <= beta <= src.k):
        raise IndexError(f"inverse block ({alpha}, {beta}) outside 1..{src.k}")
    memo_dict = memo if isinstance(memo, dict) else ({} if memo else None)
    red = Reducer(src, alpha, beta, memo_dict, trace, counters)
    idx = tuple(range(1, src.k + 1))
    root = red.reduce(idx, idx, "A", ("A",))
    return invert_dense(root)


def invert_full(matrix, k, memo=False, targets=None):
    """All (or the listed) inverse blocks, row-major order (engine.py:296-330)."""
    src = BlockSource(matrix, k)
    out = {}
    pairs = targets or [(a, b) for a in range(1, k + 1) for b in range(1, k + 1)]
    for alpha, beta in pairs:
        out[(alpha, beta)] = invert_block(src, k, alpha, beta, memo=memo)
    return out


def assemble(blocks: dict, k: int, b: int) -> np.ndarray:
    m = k * b
    full = np.zeros((m, m))
    for (a, c), blk in blocks.items():
        full[(a - 1) * b : a * b, (c - 1) * b : c * b] = blk
    return full


def lu_invert_full(a: np.ndarray) -> np.ndarray:
    """Dense LU inverse (baseline.py:27-42): invert_dense at order m."""
    return invert_dense(a)


def kernel_matrix(inputs: np.ndarray, gamma: float = 1.0, sigma: float = 1.0) -> np.ndarray:
    """LS-SVM system matrix of order n + 1 (providers.py:93-120 element rule,
    evaluated like _KernelSource.rect providers.py:182-200): 0 at (1,1), ones on
    the rest of the first row/column, Gaussian Gram + ridge 1/gamma inside."""
    x = np.ascontiguousarray(inputs, dtype=np.float64)
    if x.ndim == 1:
        x = x[:, None]
    m = x.shape[0] + 1
    out = np.ones((m, m))
    out[0, 0] = 0.0
    sq = ((x[:, None, :] - x[None, :, :]) ** 2).sum(axis=2)
    gram = np.exp(sq / (-2.0 * sigma ** 2))
    gram[np.diag_indices(m - 1)] += 1.0 / gamma
    out[1:, 1:] = gram
    return out


def predicted_nodes(k: int) -> int:
    """(4^(k-1) - 1) / 3 Schur nodes per target (instrumentation.py:124-139)."""
    return (4 ** (k - 1) - 1) // 3


# --------------------------------------------------------------------------
# Config-5 input: seeded Gaussian matrix generated blockwise (no reference
# counterpart: the reference draws M from one PCG64 stream, cli.py:122-130,
# which cannot produce a block without the blocks before it).  Restated here
# from Random123's Philox4x64-10 — the algorithm behind numpy's
# np.random.Philox, against which tests/test_oracle.py pins it — plus the
# Box-Muller map documented in include/bri_b200.h (bri_randn_blocks).
# --------------------------------------------------------------------------

_PH_M = (0xD2E7470EE14C6C93, 0xCA5A826395121157)
_PH_W = (0x9E3779B97F4A7C15, 0xBB67AE8584CAA73B)
_MASK32 = np.uint64(0xFFFFFFFF)


def _mul_hilo(a: int, x: np.ndarray):
    """(hi, lo) 64-bit halves of the 128-bit products a * x (x uint64 array)."""
    a_lo, a_hi = np.uint64(a & 0xFFFFFFFF), np.uint64(a >> 32)
    x_lo, x_hi = x & _MASK32, x >> np.uint64(32)
    ll, lh = a_lo * x_lo, a_lo * x_hi
    hl, hh = a_hi * x_lo, a_hi * x_hi
    mid = (ll >> np.uint64(32)) + (lh & _MASK32) + (hl & _MASK32)
    hi = hh + (lh >> np.uint64(32)) + (hl >> np.uint64(32)) + (mid >> np.uint64(32))
    lo = (mid << np.uint64(32)) | (ll & _MASK32)
    return hi, lo


def philox4x64_10(counter0: np.ndarray, key0: int, key1: int = 0) -> np.ndarray:
    """Philox4x64-10 outputs (n, 4) uint64 for counters (counter0[i], 0, 0, 0)."""
    c = [np.asarray(counter0, dtype=np.uint64).copy()] + [np.zeros(np.shape(counter0), np.uint64)] * 3
    k0, k1 = key0 & 0xFFFFFFFFFFFFFFFF, key1 & 0xFFFFFFFFFFFFFFFF
    with np.errstate(over="ignore"):
        for _ in range(10):
            hi0, lo0 = _mul_hilo(_PH_M[0], c[0])
            hi1, lo1 = _mul_hilo(_PH_M[1], c[2])
            c = [hi1 ^ c[1] ^ np.uint64(k0), lo1, hi0 ^ c[3] ^ np.uint64(k1), lo0]
            k0 = (k0 + _PH_W[0]) & 0xFFFFFFFFFFFFFFFF
            k1 = (k1 + _PH_W[1]) & 0xFFFFFFFFFFFFFFFF
    return np.stack(c, axis=-1)


def gaussian_window(m: int, seed: int, shift: float, row0: int, col0: int, rows: int, cols: int) -> np.ndarray:
    """Window [row0:row0+rows, col0:col0+cols] of M = G + shift*I (order m, identity padding beyond)."""
    r = np.arange(row0, row0 + rows, dtype=np.uint64)[:, None]
    c = np.arange(col0, col0 + cols, dtype=np.uint64)[None, :]
    inside = (r < np.uint64(m)) & (c < np.uint64(m))
    e = (r * np.uint64(m) + c).ravel()
    o = philox4x64_10(e >> np.uint64(2), seed)
    q = ((e & np.uint64(3)) >> np.uint64(1)).astype(np.int64)
    a = o[np.arange(e.size), 2 * q]
    bb = o[np.arange(e.size), 2 * q + 1]
    u1 = ((a >> np.uint64(11)) + np.uint64(1)).astype(np.float64) * 2.0 ** -53
    u2 = (bb >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    rho = np.sqrt(-2.0 * np.log(u1))
    theta = 6.283185307179586 * u2
    g = rho * np.where((e & np.uint64(1)) == 1, np.sin(theta), np.cos(theta))
    g = g.reshape(rows, cols)
    diag = r == c
    g = np.where(diag, g + shift, g)
    return np.where(inside, g, np.where(diag, 1.0, 0.0))
