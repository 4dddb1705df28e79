"""Bounded-schedule determinism: one config-5-shaped target (k=8, M = G + mI generated on the
device) under a device budget that forces spills, run --reps times in this process; each block's
sha256 is printed with the tree schedule's (same one-node-per-launch kernels: must be equal).

    PYTHONHASHSEED=<s> python tools/bounded_determinism.py --b 2048 --slots 40 [--reps 3]
"""
import argparse
import hashlib
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
ap = argparse.ArgumentParser()
ap.add_argument("--b", type=int, default=2048)
ap.add_argument("--k", type=int, default=8)
ap.add_argument("--slots", type=int, default=40)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--tree", action="store_true")
args = ap.parse_args()

import torch

import paper_1612_00001_b200 as bri

m = args.k * args.b
prov = bri.make_gaussian_provider(bri.GaussianSpec(m, 4, float(m)), args.k)
h = lambda x: hashlib.sha256(x.cpu().numpy().tobytes()).hexdigest()[:16]
out = {"b": args.b, "slots": args.slots, "hashseed": os.environ.get("PYTHONHASHSEED"), "bounded": [], "info": None}
for _ in range(args.reps):
    ws = bri.Workspace(arena_bytes=args.slots * args.b * args.b * 8)
    x, info = bri.invert_blocks(prov, [(1, 1)], ws)
    out["bounded"].append(h(x[0]))
    out["info"] = [info.schedule, info.arena_slots, info.spills, info.host_blocks]
if args.tree:
    out["tree"] = h(bri.invert_block(prov, 1, 1, bri.Workspace(schedule="tree")).tensor)
out["dag"] = h(bri.invert_blocks(prov, [(1, 1)])[0][0])
print(json.dumps(out), flush=True)
