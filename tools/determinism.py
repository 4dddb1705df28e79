"""Run-to-run determinism and accuracy of one large node + inversion (k=2, config-5 matrix):
the same block computed --reps times must be bit-identical (sha256 of the bytes); each run is
also compared with the Neumann-series block (tools/run_config5.neumann_y11).  Run once per
LU concurrency setting (BRI_CAP_ROWS etc.) to check the multi-stream schedule for races.

    python tools/determinism.py --b 20480 [--reps 3]
"""
import argparse
import hashlib
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

ap = argparse.ArgumentParser()
ap.add_argument("--b", type=int, default=20480)
ap.add_argument("--k", type=int, default=2)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--target", default="1,1", help="alpha,beta (the Neumann check needs 1,1)")
ap.add_argument("--ballast-gb", type=float, default=0.0,
                help="hold this much device memory first (mimics config 5's nearly full HBM)")
args = ap.parse_args()
target = tuple(int(v) for v in args.target.split(","))

import torch

import paper_1612_00001_b200 as bri
from paper_1612_00001_b200.device import release_cached_memory
from run_config5 import neumann_y11

m = args.k * args.b
ballast = torch.empty(int(args.ballast_gb * 2**30) // 8, dtype=torch.float64, device="cuda:0") if args.ballast_gb else None
prov = bri.make_gaussian_provider(bri.GaussianSpec(m, 4, float(m)), args.k)
hashes, xs, infos = [], [], []
for _ in range(args.reps):
    x, info = bri.invert_blocks(prov, [target])
    x = x[0]
    infos.append([info.schedule, info.arena_slots, info.spills])
    hashes.append(hashlib.sha256(x.cpu().numpy().tobytes()).hexdigest()[:16])
    xs.append(x)
release_cached_memory()
del ballast
torch.cuda.empty_cache()
rel = None
if target == (1, 1):
    terms = max(4, math.ceil(math.log(1e-19) / math.log(2.0 / math.sqrt(m))))
    y, _ = neumann_y11(m, args.k, args.b, 4, terms)
    rel = [float((x - y).abs().max() / y.abs().max()) for x in xs]
env = {k: v for k, v in os.environ.items() if k.startswith("BRI_")}
print(json.dumps({"b": args.b, "k": args.k, "target": list(target), "env": env, "hashes": hashes, "deterministic": len(set(hashes)) == 1, "runs": infos,
                  "rel_vs_neumann": rel}), flush=True)
