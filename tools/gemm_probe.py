"""Time the DMMA GEMM kernel on representative shapes (CUDA events)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1612_00001_b200.device import Arena, fp64_peak_tflops
shapes = [(4096, 4096, 4096), (2048, 4096, 2048), (1024, 4096, 1024), (512, 4096, 512), (3968, 3968, 128),
          (2048, 2048, 128), (4064, 96, 32), (1024, 1024, 1024)]
n = 4096
out = {"peak": fp64_peak_tflops()}
with Arena(n, 4) as ar:
    for s in range(4):
        ar.view(s).normal_()
    for (M, N, K) in shapes:
        for _ in range(2):
            ar.gemm([(0, 1, 2, 3)], M, N, K, alpha=-1.0, beta=1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 10
        e0.record()
        for _ in range(reps):
            ar.gemm([(0, 1, 2, 3)], M, N, K, alpha=-1.0, beta=1.0)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        out[f"{M}x{N}x{K}"] = {"us": round(ms * 1000, 1), "tflops": round(2 * M * N * K / ms / 1e9, 2)}
# a batched DAG level: 64 independent b=1024 Schur updates in one launch
with Arena(1024, 4 * 64) as ar:
    ar.tensor.normal_()
    items = [(4 * i, 4 * i + 1, 4 * i + 2, 4 * i + 3) for i in range(64)]
    for _ in range(2):
        ar.gemm(items, 1024, 1024, 1024, alpha=-1.0, beta=1.0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        ar.gemm(items, 1024, 1024, 1024, alpha=-1.0, beta=1.0)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    out["64x1024^3"] = {"us": round(ms * 1000, 1), "tflops": round(64 * 2 * 1024**3 / ms / 1e9, 2)}
print(json.dumps(out))
