"""One DAG level's Schur GEMM batch in isolation (the launch bench.py's roofline names): COUNT
items of out = r - rt*W at order B, CUDA-event timed; run under ncu --set full for DRAM traffic.

    python tools/gemm_level_probe.py --b 1024 --count 148
    ncu --set full --import-source on --clock-control none -k regex:gemm_kernel -s 2 -c 1 \\
        python tools/gemm_level_probe.py --b 1024 --count 148
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1612_00001_b200.device import Arena

ap = argparse.ArgumentParser()
ap.add_argument("--b", type=int, default=1024)
ap.add_argument("--count", type=int, default=148)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--shape", default=None, help="M,N,K window inside the order-B slots (default B,B,B)")
args = ap.parse_args()
b, cnt = args.b, args.count
M, N, K = (int(v) for v in args.shape.split(",")) if args.shape else (b, b, b)
with Arena(b, 3 * cnt) as ar:
    ar.tensor.normal_()
    items = [(3 * i, 3 * i + 1, 3 * i + 2, 3 * i + 2) for i in range(cnt)]
    for _ in range(2):
        ar.gemm(items, M, N, K, alpha=-1.0, beta=1.0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(args.reps):
        ar.gemm(items, M, N, K, alpha=-1.0, beta=1.0)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.reps
flops = cnt * (2.0 * M * N * K + M * N)
# algorithmic bytes: read rt, W, r and write out once per item
print(json.dumps({"b": b, "shape": [M, N, K], "count": cnt, "ms": ms, "tflops": flops / ms / 1e9,
                  "algorithmic_bytes_per_launch": cnt * 4 * b * b * 8}))
