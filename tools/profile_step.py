"""Run W warm-up steps and then S profiled steps of a BASELINE config (for ncu launch lists)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1612_00001_b200 as bri
from paper_1612_00001_b200 import workloads

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--b", type=int, default=None)
ap.add_argument("--warmup", type=int, default=1)
ap.add_argument("--steps", type=int, default=1)
ap.add_argument("--targets", type=int, default=None)
args = ap.parse_args()
cfg = workloads.config(args.config, args.b)
a = torch.from_numpy(workloads.make_matrix(args.config, args.b)).cuda()
prov = bri.make_memory_provider(a, cfg["k"])
targets = cfg["targets"][: args.targets] if args.targets else cfg["targets"]
for _ in range(args.warmup):
    bri.invert_blocks(prov, targets)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
for _ in range(args.steps):
    bri.invert_blocks(prov, targets)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("done")
