"""Golden fixtures for BASELINE config 3 at TRUE size, made by the UNMODIFIED reference.

Run once in the build container (the reference is importable there; it does not exist on
the GPU box).  Takes ~10 minutes on 8 cores:

    python tests/golden/make_config_golden.py

Config 3 (k=8, b=1024, M = G + m I from PCG64 seed 2): block row 1 of M^-1, the 8
targets (1, beta), through the reference's own public API `bri.invert_block`.  The reference
walks the literal tree (5,461 nodes per target); the harness memoizes `bri.engine.reduce_frame`
on the node's BASE block indices — bit-identical to the tree walk — so the 8
targets cost 1,256 distinct nodes.  The same run is repeated on M perturbed by one ulp
(M * (1 + eps N(0,1)), seed 123) to record the reference's own 1-ulp sensitivity
per block, the floor the off-diagonal targets are judged against.

Blocks are 8 MiB each, too large to commit, so the fixture keeps, per target:
  * 4096 entries at fixed pseudo-random positions (same positions for every target),
  * the block's first row and column and its diagonal,
  * max |block|, the 1-ulp floor, the block's relative distance from the dense-LU inverse
    (numpy.linalg.inv of the same M), and the block-row residual  max |(X M)[:, rows] - I|
    of the reference's whole block row (X = [N_11 .. N_18]).
Writes tests/golden/config3_row1.npz.
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import bri  # noqa: E402  (the reference)
import bri.engine as bengine  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "config3_row1.npz")
K, B, SEED = 8, 1024, 2
M = K * B
NPOS = 4096


def config3_matrix() -> np.ndarray:
    a = np.random.Generator(np.random.PCG64(SEED)).standard_normal((M, M))
    a[np.diag_indices(M)] += M
    return a


class Memo:
    """Memoize bri.engine.reduce_frame on (base rows, base cols, label if n > 2)."""

    def __init__(self):
        self.cache = {}
        self.orig = bengine.reduce_frame
        self.executed = 0

    def __enter__(self):
        orig, cache = self.orig, self.cache

        def memo_reduce(provider, frame, ws=None, trace=None, _path=None):
            perm = getattr(provider, "perm", None)
            mr = perm.map_row if perm is not None else (lambda i: i)
            mc = perm.map_col if perm is not None else (lambda j: j)
            key = (tuple(mr(r) for r in frame.rows), tuple(mc(c) for c in frame.cols),
                   frame.label if frame.n > 2 else None)
            hit = cache.get(key)
            if hit is not None:
                return bri.Block(hit.copy(), ws) if ws is not None else bri.Block(hit.copy())
            out = orig(provider, frame, ws, trace, _path)
            cache[key] = out.data.copy()
            self.executed += 1
            return out

        bengine.reduce_frame = memo_reduce
        return self

    def __exit__(self, *exc):
        bengine.reduce_frame = self.orig


def block_row(a):
    prov = bri.make_memory_provider(a, K)
    out = []
    with Memo() as memo:
        for beta in range(1, K + 1):
            blk = bri.invert_block(prov, 1, beta)
            out.append(blk.data.copy())
            blk.release()
    return out, memo.executed


def main():
    t0 = time.time()
    a = config3_matrix()
    row, executed = block_row(a)
    t1 = time.time()
    pert = a * (1.0 + 2.220446049250313e-16 * np.random.Generator(np.random.PCG64(123)).standard_normal(a.shape))
    row_p, _ = block_row(pert)
    t2 = time.time()
    x = np.concatenate(row, axis=1)                       # block row 1 of M^-1: (b, m)
    resid = float(np.abs(x @ a - np.eye(M)[:B]).max())
    dense = np.linalg.inv(a)[:B]                          # block row 1 of the dense-LU inverse
    pos = np.random.Generator(np.random.PCG64(77)).integers(0, B, size=(NPOS, 2))
    arrays = {"positions": pos}
    meta = {"k": K, "b": B, "seed": SEED, "targets": [[1, be] for be in range(1, K + 1)],
            "reference_nodes_executed": executed, "row_residual": resid,
            "seconds": {"row": t1 - t0, "perturbed_row": t2 - t1}, "per_target": {}}
    for be, (blk, blk_p) in enumerate(zip(row, row_p), start=1):
        arrays[f"t1_{be}_samples"] = blk[pos[:, 0], pos[:, 1]]
        arrays[f"t1_{be}_row0"] = blk[0].copy()
        arrays[f"t1_{be}_col0"] = blk[:, 0].copy()
        arrays[f"t1_{be}_diag"] = np.diagonal(blk).copy()
        meta["per_target"][str(be)] = {
            "maxabs": float(np.abs(blk).max()),
            "floor_1ulp": float(np.abs(blk_p - blk).max() / np.abs(blk).max()),
            "dense_rel": float(np.abs(blk - dense[:, (be - 1) * B:be * B]).max()
                               / np.abs(dense[:, (be - 1) * B:be * B]).max()),
        }
    np.savez_compressed(OUT, meta=np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8), **arrays)
    print(json.dumps(meta, indent=1))


if __name__ == "__main__":
    main()
