"""Tall-panel heavy-pivoting regression probe (lu_panel_tall_kernel, panels > 8192 rows).

Inverts a plain Gaussian matrix (no diagonal shift: partial pivoting interchanges rows in
almost every column) REPEATS times, half of them with a concurrent FP64 GEMM on a side
stream so the panel cluster's CTAs run skewed, and prints one JSON line with the sha256 of
every result and the residual max|A·X − I|.  Run it with BRI_CAP_ROWS=1000000 to force the
LU's capped persistent GEMMs next to the panel chain (the round-1 failure condition).

    python tools/tall_pivot_check.py --n 12288 --repeats 4 [--node]

--node runs one Schur node + final inversion of order n (k=2, b=n) instead of a dense
inverse; the residual is then max|S·X − I| with S = A − B·D⁻¹·C formed by cuSOLVER (checker only).
"""
import argparse
import hashlib
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1612_00001_b200 as bri
from paper_1612_00001_b200 import baseline

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=12288)
ap.add_argument("--repeats", type=int, default=4)
ap.add_argument("--seed", type=int, default=7)
ap.add_argument("--node", action="store_true", help="k=2 Schur node of order n (b = n) instead")
args = ap.parse_args()

n = args.n
g = np.random.Generator(np.random.PCG64(args.seed))
m = 2 * n if args.node else n
a = g.standard_normal((m, m))
a_dev = torch.from_numpy(a).cuda()
side = torch.cuda.Stream()
noise = torch.randn(6144, 6144, dtype=torch.float64, device="cuda")

hashes, resid = [], []
for r in range(args.repeats):
    busy = r % 2 == 1
    if busy:   # long FP64 GEMMs occupying SMs while the panel chain runs
        with torch.cuda.stream(side):
            for _ in range(6):
                noise = (noise @ noise) * (1.0 / 6144 ** 0.5)
    if args.node:
        x = bri.invert_block(bri.make_memory_provider(a_dev, 2), 1, 1).data
        if r == 0:   # checker only (cuSOLVER): S = A - B D^-1 C, the node's Schur complement
            s_ = a_dev[:n, :n] - a_dev[:n, n:] @ torch.linalg.solve(a_dev[n:, n:], a_dev[n:, :n])
        xt = torch.from_numpy(x).cuda()
        resid.append(float((s_ @ xt - torch.eye(n, dtype=torch.float64, device="cuda")).abs().max().item()))
    else:
        x = baseline.lu_invert_full(a)
        xt = torch.from_numpy(x).cuda()
        resid.append(float((a_dev @ xt - torch.eye(n, dtype=torch.float64, device="cuda")).abs().max().item()))
    torch.cuda.synchronize()
    hashes.append(hashlib.sha256(np.ascontiguousarray(x).tobytes()).hexdigest()[:16])

print(json.dumps({"n": n, "node": args.node, "seed": args.seed, "cap_rows": os.environ.get("BRI_CAP_ROWS"),
                  "hashes": hashes, "identical": len(set(hashes)) == 1, "resid": resid}))
