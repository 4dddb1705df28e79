"""Kernel timeline of one step (CUPTI via torch.profiler): start/end of every kernel, stream
concurrency, idle gaps between kernels — what ncu's serialised launch list cannot show.

    python tools/timeline.py --config 2 [--out gpurun_out/timeline.json]
"""
import argparse
import json
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1612_00001_b200 as bri
from paper_1612_00001_b200 import workloads

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--b", type=int, default=None)
ap.add_argument("--warmup", type=int, default=3)
ap.add_argument("--out", default="gpurun_out/timeline.json")
ap.add_argument("--top", type=int, default=25)
ap.add_argument("--gauss", action="store_true",
                help="M = G + mI generated on the device (GaussianSpec seed 4, the config-5 input) instead "
                     "of the config's host-generated matrix: large --b without a host GEMM")
args = ap.parse_args()

cfg = workloads.config(args.config, args.b)
if args.gauss:
    m = cfg["k"] * cfg["b"]
    prov = bri.make_gaussian_provider(bri.GaussianSpec(m, 4, float(m)), cfg["k"])
else:
    a = torch.from_numpy(workloads.make_matrix(args.config, args.b)).cuda()
    prov = bri.make_memory_provider(a, cfg["k"])
targets = cfg["targets"]
for _ in range(args.warmup):
    bri.invert_blocks(prov, targets)
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    bri.invert_blocks(prov, targets)
    torch.cuda.synchronize()
path = "/tmp/bri_trace.json"
prof.export_chrome_trace(path)
ev = [e for e in json.load(open(path))["traceEvents"] if e.get("cat") in ("kernel", "gpu_memcpy")]
ev.sort(key=lambda e: e["ts"])


def short(n):
    n = n.replace("(anonymous namespace)::", "").replace("bri::", "").replace("void ", "")
    return n.split("(")[0].split("<")[0]


t0 = ev[0]["ts"]
t1 = max(e["ts"] + e["dur"] for e in ev)
wall = t1 - t0
# union of busy intervals and the idle gaps
busy, cur_s, cur_e, gaps = 0.0, None, None, []
for e in ev:
    s, f = e["ts"], e["ts"] + e["dur"]
    if cur_e is None or s > cur_e:
        if cur_e is not None:
            busy += cur_e - cur_s
            gaps.append(s - cur_e)
        cur_s, cur_e = s, f
    else:
        cur_e = max(cur_e, f)
busy += cur_e - cur_s
per = defaultdict(lambda: [0, 0.0])
for e in ev:
    per[short(e["name"])][0] += 1
    per[short(e["name"])][1] += e["dur"]
streams = defaultdict(float)
for e in ev:
    streams[e["args"].get("stream", "?")] += e["dur"]
out = {"kernels": len(ev), "wall_us": wall, "busy_us": busy, "idle_us": wall - busy, "gaps": len(gaps),
       "gap_us_mean": (sum(gaps) / len(gaps)) if gaps else 0.0,
       "per_kernel_us": {k: {"n": v[0], "us": round(v[1], 1)} for k, v in sorted(per.items(), key=lambda x: -x[1][1])},
       "per_stream_us": {str(k): round(v, 1) for k, v in streams.items()}}
os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
json.dump({"summary": out, "events": [(short(e["name"]), e["args"].get("stream"), e["ts"] - t0, e["dur"],
                                       e["args"].get("grid")) for e in ev]}, open(args.out, "w"))
print(json.dumps({k: v for k, v in out.items() if k != "per_kernel_us"}, indent=1))
for k, v in list(out["per_kernel_us"].items())[: args.top]:
    print(f"{k:28s} {v['n']:6d} {v['us']:10.1f} us")
