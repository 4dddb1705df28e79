"""Time one Schur node + final inversion at a large block order on the device-generated
config-5 matrix (k=2: invert_block(1,1) = 1 node + 1 inversion), for sweeping the LU's
concurrency caps (BRI_TRAIL_CAP, BRI_FOLD_CAP, BRI_CAP_ROWS) per process.

    python tools/node_time.py --b 20480 [--reps 3]   -> one JSON line (median ms, TFLOP/s)
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1612_00001_b200 as bri
from paper_1612_00001_b200 import workloads

ap = argparse.ArgumentParser()
ap.add_argument("--b", type=int, default=20480)
ap.add_argument("--k", type=int, default=2)
ap.add_argument("--reps", type=int, default=3)
args = ap.parse_args()
m = args.k * args.b
prov = bri.make_gaussian_provider(bri.GaussianSpec(m, 4, float(m)), args.k)
bri.invert_blocks(prov, [(1, 1)])
ms = []
for _ in range(args.reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    x, info = bri.invert_blocks(prov, [(1, 1)])
    e1.record()
    torch.cuda.synchronize()
    ms.append(e0.elapsed_time(e1))
med = statistics.median(ms)
flops = workloads.run_flops(args.b, info.dag_nodes, 1)
env = {k: os.environ[k] for k in ("BRI_TRAIL_CAP", "BRI_FOLD_CAP", "BRI_CAP_ROWS") if k in os.environ}
print(json.dumps({"b": args.b, "k": args.k, "nodes": info.dag_nodes, "ms": ms, "median_ms": med,
                  "tflops": flops / med / 1e9, "env": env}), flush=True)
