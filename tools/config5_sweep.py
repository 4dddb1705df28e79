"""Accuracy of the config-5 workload (k=8, M = G + m I, GaussianSpec seed 4, target (1,1)) as the
block order grows, on the GPU, to tell kernel error from BRI's own numerical behaviour:

  gpu_vs_neumann : max|X - Y11| / max|Y11|, Y11 from the Neumann series (tools/run_config5.py)
  floor          : the same BRI run on M with its diagonal moved by ONE ulp (shift = nextafter(m)):
                   max|X - X'| / max|X| — what BRI itself does with a 1-ulp change of its input
  cpu_vs_neumann : the CPU oracle (= the reference's LAPACK calls, memoized) on the same bytes,
                   for orders where it runs in about a minute
  gpu_vs_cpu     : GPU block against that CPU block

usage: python tools/config5_sweep.py [--bs 512,1024,2048,4096,8192] [--cpu-max 2048] [--out FILE]
"""

from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--bs", default="512,1024,2048,4096,8192")
    ap.add_argument("--k", type=int, default=8)
    ap.add_argument("--seed", type=int, default=4)
    ap.add_argument("--cpu-max", type=int, default=2048)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()

    import numpy as np
    import torch

    import paper_1612_00001_b200 as bri
    from paper_1612_00001_b200 import engine
    from paper_1612_00001_b200.device import release_cached_memory
    from run_config5 import neumann_y11

    torch.cuda.set_device(0)
    k = args.k
    rows = []
    for b in [int(x) for x in args.bs.split(",")]:
        m = k * b
        rel = lambda x, y: float((x - y).abs().max() / y.abs().max())
        t0 = time.perf_counter()
        x = bri.invert_blocks(bri.make_gaussian_provider(bri.GaussianSpec(m, args.seed, float(m)), k), [(1, 1)])[0][0]
        t_run = time.perf_counter() - t0
        xp = bri.invert_blocks(bri.make_gaussian_provider(
            bri.GaussianSpec(m, args.seed, float(np.nextafter(float(m), math.inf))), k), [(1, 1)])[0][0]
        release_cached_memory()
        engine.release_host_pool()
        ratio = 2.0 / math.sqrt(m)
        terms = max(4, math.ceil(math.log(1e-19) / math.log(ratio)))
        y11, last = neumann_y11(m, k, b, args.seed, terms)
        row = {"k": k, "b": b, "m": m, "seed": args.seed, "run_s": t_run, "neumann_terms": terms,
               "neumann_last_term_rel": last, "gpu_vs_neumann": rel(x, y11), "floor_1ulp": rel(xp, x)}
        if b <= args.cpu_max:
            from oracle import bri_oracle as orc

            a = bri.gaussian_window(bri.GaussianSpec(m, args.seed, float(m)), 0, 0, m, m).cpu().numpy()
            t1 = time.perf_counter()
            c = torch.from_numpy(orc.invert_block(a, k, 1, 1, memo=True)).cuda()
            row["cpu_s"] = time.perf_counter() - t1
            row["cpu_vs_neumann"] = rel(c, y11)
            row["gpu_vs_cpu"] = rel(x, c)
            del a
        print(json.dumps(row), flush=True)
        rows.append(row)
        del x, xp, y11
        torch.cuda.empty_cache()
    if args.out:
        with open(args.out, "w") as f:
            json.dump({"workload": "config5 shape (k=8, M = G + mI, GaussianSpec seed 4, target (1,1))",
                       "rows": rows}, f, indent=1)
            f.write("\n")


if __name__ == "__main__":
    main()
