"""sha256 of every result block of a BASELINE config (bit-identity checks across builds of the
library: BRI_LIB=<other .so> python tools/hash_config.py --config 3).

Prints one JSON line: the hash over all blocks in target order, plus the first block's own.
"""
import argparse
import hashlib
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1612_00001_b200 as bri
from paper_1612_00001_b200 import workloads

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, required=True)
ap.add_argument("--b", type=int, default=None)
args = ap.parse_args()

cfg = workloads.config(args.config, args.b)
a = workloads.make_matrix(args.config, args.b)
prov = bri.make_memory_provider(torch.from_numpy(a).cuda(), cfg["k"])
tensors, info = bri.invert_blocks(prov, cfg["targets"], bri.Workspace())
torch.cuda.synchronize()
h = hashlib.sha256()
first = None
for x in tensors:
    raw = x.cpu().numpy().tobytes()
    if first is None:
        first = hashlib.sha256(raw).hexdigest()[:16]
    h.update(raw)
print(json.dumps({"config": args.config, "b": cfg["b"], "k": cfg["k"], "targets": len(cfg["targets"]),
                  "lib": os.environ.get("BRI_LIB", "default"), "sha256_all": h.hexdigest()[:16],
                  "sha256_first": first}), flush=True)
