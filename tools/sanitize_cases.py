"""Small cases for compute-sanitizer (racecheck / synccheck / memcheck), one process:

  * config-3 shape: k=4, b=128 full inverse of G + m I (level batches: shared factorizations,
    solves, the TMA/DMMA GEMM and TRSM, lu_panel cluster kernels, row panels, laswp)
  * config-1 shape: k=4, b=64 full inverse (the one-CTA small-node kernel, both modes)
  * tall panels with heavy pivoting: n = 1536 plain Gaussian dense inverse with
    BRI_TALL_ROWS=256 (set by the caller), i.e. lu_panel_tall_kernel on 16-CTA clusters
  * a bounded run with spills (k=4, b=128)

usage: BRI_TALL_ROWS=256 compute-sanitizer --tool racecheck python tools/sanitize_cases.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1612_00001_b200 as bri
from paper_1612_00001_b200 import baseline


def main():
    g = np.random.Generator(np.random.PCG64(3))
    a = g.standard_normal((512, 512)) + 512 * np.eye(512)
    prov = bri.make_memory_provider(a, 4)
    sink = bri.MemorySink(prov.layout)
    bri.invert_full(prov, sink)
    x = sink.finalize()
    print("cfg3-shape resid", float(np.abs(a @ x - np.eye(512)).max()), flush=True)
    a1 = g.uniform(-1, 1, (256, 256)) + 256 * np.eye(256)
    p1 = bri.make_memory_provider(a1, 4)
    s1 = bri.MemorySink(p1.layout)
    bri.invert_full(p1, s1)
    print("cfg1-shape resid", float(np.abs(a1 @ s1.finalize() - np.eye(256)).max()), flush=True)
    t = g.standard_normal((1536, 1536))
    xt = baseline.lu_invert_full(t)
    print("tall resid", float(np.abs(t @ xt - np.eye(1536)).max()), "BRI_TALL_ROWS",
          os.environ.get("BRI_TALL_ROWS"), flush=True)
    ws = bri.Workspace(schedule="bounded", arena_bytes=9 * 128 * 128 * 8)
    xb = bri.invert_block(prov, 2, 3, ws).data
    print("bounded err", float(np.abs(xb - x[128:256, 256:384]).max() / np.abs(x[128:256, 256:384]).max()),
          flush=True)
    torch.cuda.synchronize()
    print("sanitize cases done")


if __name__ == "__main__":
    main()
