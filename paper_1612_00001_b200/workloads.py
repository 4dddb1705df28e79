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

cfg 5 (215 GB) needs a blockwise generator the reference does not have:
block (i, j) is drawn from its own stream `SeedSequence(4).spawn` indexed
row-major, plus m on the diagonal blocks' diagonals.  `scale` shrinks b for
the proxies the survey used (e.g. cfg 5 at b=2048).
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
        k, bb = c["k"], c["b"]
        a = np.empty((m, m))
        streams = np.random.SeedSequence(seed).spawn(k * k)
        for i in range(k):
            for j in range(k):
                g = np.random.Generator(np.random.PCG64(streams[i * k + j]))
                a[i * bb:(i + 1) * bb, j * bb:(j + 1) * bb] = g.standard_normal((bb, bb))
        a[np.diag_indices(m)] += m
        return a
    raise ValueError(kind)


def node_flops(b: int) -> float:
    """Algorithmic FLOPs per Schur node: inverse 2b^3 + two GEMMs 4b^3 + subtract b^2."""
    return 6.0 * b ** 3 + b ** 2


def run_flops(b: int, nodes: int, targets: int) -> float:
    """Algorithmic FLOPs of a run: nodes * F_node + targets * 2b^3 (final inversions)."""
    return nodes * node_flops(b) + targets * 2.0 * b ** 3
