"""Run a BASELINE config through the device engine; time it and check parity against the oracle.

  python tools/run_config.py --config 3 [--oracle-targets 2] [--b B]
Prints one JSON line: time, algorithmic TFLOP/s, DAG stats, per-target errors vs the CPU
oracle (and the oracle's own 1-ulp floor when --floor), residual checks.
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1612_00001_b200 as bri
from paper_1612_00001_b200 import workloads
from paper_1612_00001_b200.dag import build_schedule

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, required=True)
ap.add_argument("--b", type=int, default=None)
ap.add_argument("--oracle-targets", type=int, default=1)
ap.add_argument("--floor", action="store_true")
ap.add_argument("--reps", type=int, default=1)
args = ap.parse_args()

cfg = workloads.config(args.config, args.b)
k, b = cfg["k"], cfg["b"]
t0 = time.time()
a = workloads.make_matrix(args.config, args.b)
gen_s = time.time() - t0
targets = cfg["targets"]
sched = build_schedule(k, targets)
flops = workloads.run_flops(b, len(sched.nodes), len(targets))
prov = bri.make_memory_provider(torch.from_numpy(a).cuda(), k)
out = {"config": args.config, "k": k, "b": b, "targets": len(targets), "dag_nodes": len(sched.nodes),
       "tree_nodes": len(targets) * ((4 ** (k - 1) - 1) // 3), "gen_s": gen_s}
try:
    ws = bri.Workspace()
    bri.invert_blocks(prov, targets, ws)  # warm-up (also builds kernels' attributes)
    torch.cuda.synchronize()
    times = []
    for _ in range(args.reps):
        t1 = time.perf_counter()
        tensors, info = bri.invert_blocks(prov, targets, bri.Workspace())
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t1)
    sec = min(times)
    out.update({"seconds": sec, "tflops": flops / sec / 1e12, "sec_per_block": sec / len(targets),
                "arena_slots": info.arena_slots, "chunk": info.chunk, "levels": info.levels})
    got = {t: x.cpu().numpy() for t, x in zip(targets, tensors)}
    # residual of block rows / columns we computed (cheap on host for one block row)
    errs = {}
    if args.oracle_targets:
        from oracle import bri_oracle as orc

        pick = targets[: args.oracle_targets] if args.oracle_targets < len(targets) else targets
        if len(targets) > 1 and args.oracle_targets >= 2:
            pick = [targets[0], targets[len(targets) // 2 + 1]][: args.oracle_targets]
        t2 = time.time()
        src = orc.BlockSource(a, k)
        memo = {}
        for t in pick:
            want = orc.invert_block(src, k, *t, memo=memo)
            rel = float(np.abs(got[t] - want).max() / np.abs(want).max())
            errs[str(t)] = {"rel_vs_oracle": rel}
        out["oracle_s"] = time.time() - t2
        if args.floor:
            pert = a * (1.0 + 2.220446049250313e-16 * np.random.Generator(np.random.PCG64(123)).standard_normal(a.shape))
            srcp = orc.BlockSource(pert, k)
            memo = {}
            for t in pick:
                want = orc.invert_block(src, k, *t, memo={})
                moved = orc.invert_block(srcp, k, *t, memo=memo)
                errs[str(t)]["oracle_1ulp_floor"] = float(np.abs(moved - want).max() / np.abs(want).max())
    out["parity"] = errs
except bri.BriError as e:
    out["error"] = f"{type(e).__name__}: {e}"
print(json.dumps(out))
