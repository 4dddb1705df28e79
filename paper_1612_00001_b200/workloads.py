"""Synthetic inputs for the BASELINE.json configurations.

No dataset is involved: every matrix is generated from PCG64 seeds, the
reference's convention (`np.random.Generator(np.random.PCG64(seed))`,
cli.py:122, tests/conftest.py:9-10).  The same bytes feed the device path
and the CPU oracle.

  cfg 1: k=4,  b=64,    Uniform[-1,1] + m I,       seed 0, all 16 blocks
  cfg 2: k=2,  b=4096,  G G^T / m + I (SPD),       seed 1, block (1,1)
  cfg 3: k=8,  b=1024,  G + m I,                   seed 2, all 64 blocks
  cfg 4: k=16, b=2048,  G G^T / m + I (SPD),       seed 3, block row 1
  cfg 5: k=8,  b=20480, G + m I blockwise,         seed 4, block (1,1)

cfg 5 (215 GB) needs a blockwise generator the reference does not have: the
counter-based Philox4x64-10 + Box-Muller scheme of `GaussianSpec` /
bri_randn_blocks (include/bri_b200.h), so a proxy at smaller b (e.g. b=2048)
and the true-size run on the device draw from the SAME input family — element
(r, c) depends only on (seed, m, r, c).  `_gaussian_rows` is the host form
used for proxies; tests pin it against the device kernel and the oracle.
"""

from __future__ import annotations

import numpy as np

CONFIGS = {
    1: dict(k=4, b=64, kind="uniform_shift", seed=0, targets="all"),
    2: dict(k=2, b=4096, kind="spd", seed=1, targets=[(1, 1)]),
    3: dict(k=8, b=1024, kind="randn_shift", seed=2, targets="all"),
    4: dict(k=16, b=2048, kind="spd", seed=3, targets="row1"),
    5: dict(k=8, b=20480, kind="randn_shift_blockwise", seed=4, targets=[(1, 1)]),
}


def rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def config(cfg: int, b: int | None = None) -> dict:
    c = dict(CONFIGS[cfg])
    if b is not None:
        c["b"] = b
    c["m"] = c["k"] * c["b"]
    k = c["k"]
    if c["targets"] == "all":
        c["targets"] = [(a, bb) for a in range(1, k + 1) for bb in range(1, k + 1)]
    elif c["targets"] == "row1":
        c["targets"] = [(1, bb) for bb in range(1, k + 1)]
    return c


def _spd(g: np.ndarray) -> np.ndarray:
    """G G^T / m + I, row-blocked (a one-shot 32768^2 product segfaulted in OpenBLAS)."""
    m = g.shape[0]
    out = np.empty((m, m))
    step = 4096
    for r0 in range(0, m, step):
        out[r0:r0 + step] = g[r0:r0 + step] @ g.T
    out /= m
    out[np.diag_indices(m)] += 1.0
    return out


def make_matrix(cfg: int, b: int | None = None) -> np.ndarray:
    """Dense row-major float64 M for a BASELINE config (optionally at a smaller b)."""
    c = config(cfg, b)
    m, seed, kind = c["m"], c["seed"], c["kind"]
    if kind == "uniform_shift":
        a = rng(seed).uniform(-1.0, 1.0, (m, m))
        a[np.diag_indices(m)] += m
        return a
    if kind == "randn_shift":
        a = rng(seed).standard_normal((m, m))
        a[np.diag_indices(m)] += m
        return a
    if kind == "spd":
        return _spd(rng(seed).standard_normal((m, m)))
    if kind == "randn_shift_blockwise":
        a = np.empty((m, m))
        step = max(1, (1 << 22) // m)
        for r0 in range(0, m, step):
            a[r0:r0 + step] = _gaussian_rows(m, seed, float(m), r0, min(step, m - r0))
        return a
    raise ValueError(kind)


_PH_M = (0xD2E7470EE14C6C93, 0xCA5A826395121157)
_PH_W = (0x9E3779B97F4A7C15, 0xBB67AE8584CAA73B)


def _mulhilo(a: int, x: np.ndarray):
    lo32 = np.uint64(0xFFFFFFFF)
    s32 = np.uint64(32)
    al, ah = np.uint64(a & 0xFFFFFFFF), np.uint64(a >> 32)
    xl, xh = x & lo32, x >> s32
    p0, p1, p2, p3 = al * xl, al * xh, ah * xl, ah * xh
    mid = (p0 >> s32) + (p1 & lo32) + (p2 & lo32)
    return p3 + (p1 >> s32) + (p2 >> s32) + (mid >> s32), (mid << s32) | (p0 & lo32)


def _gaussian_rows(m: int, seed: int, shift: float, r0: int, rows: int) -> np.ndarray:
    """Rows [r0, r0+rows) of M = G + shift*I, G(r, c) = Box-Muller of Philox4x64-10 (key = seed)
    at counter (r*m + c) >> 2: words 2q, 2q+1 (q = bit 1 of r*m + c) give u1 = ((w>>11)+1)/2^53,
    u2 = (w>>11)/2^53, then sqrt(-2 ln u1) * (sin if bit 0 else cos)(2 pi u2)."""
    e = (np.arange(r0, r0 + rows, dtype=np.uint64)[:, None] * np.uint64(m)
         + np.arange(m, dtype=np.uint64)[None, :]).ravel()
    ctr = [e >> np.uint64(2), np.zeros_like(e), np.zeros_like(e), np.zeros_like(e)]
    k0, k1 = seed & 0xFFFFFFFFFFFFFFFF, 0
    with np.errstate(over="ignore"):
        for _ in range(10):
            h0, l0 = _mulhilo(_PH_M[0], ctr[0])
            h1, l1 = _mulhilo(_PH_M[1], ctr[2])
            ctr = [h1 ^ ctr[1] ^ np.uint64(k0), l1, h0 ^ ctr[3] ^ np.uint64(k1), l0]
            k0 = (k0 + _PH_W[0]) & 0xFFFFFFFFFFFFFFFF
            k1 = (k1 + _PH_W[1]) & 0xFFFFFFFFFFFFFFFF
    hiq = ((e >> np.uint64(1)) & np.uint64(1)).astype(bool)
    wa = np.where(hiq, ctr[2], ctr[0])
    wb = np.where(hiq, ctr[3], ctr[1])
    u1 = ((wa >> np.uint64(11)) + np.uint64(1)).astype(np.float64) * 2.0 ** -53
    u2 = (wb >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    rho, th = np.sqrt(-2.0 * np.log(u1)), 6.283185307179586 * u2
    g = (rho * np.where((e & np.uint64(1)) == 1, np.sin(th), np.cos(th))).reshape(rows, m)
    idx = np.arange(rows)
    g[idx, r0 + idx] += shift
    return g


def node_flops(b: int) -> float:
    """Algorithmic FLOPs per Schur node: inverse 2b^3 + two GEMMs 4b^3 + subtract b^2."""
    return 6.0 * b ** 3 + b ** 2


def run_flops(b: int, nodes: int, targets: int) -> float:
    """Algorithmic FLOPs of a run: nodes * F_node + targets * 2b^3 (final inversions)."""
    return nodes * node_flops(b) + targets * 2.0 * b ** 3
