"""Where the end-to-end step of a config goes: provider from pinned host memory, the device run,
the sink puts (D2H + canvas), finalize — host wall clock with a synchronize at each boundary,
plus the CUPTI memcpy list of one step.

usage: python tools/e2e_breakdown.py [--config 3] [--steps 3]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--steps", type=int, default=3)
    args = ap.parse_args()
    import torch

    import paper_1612_00001_b200 as bri
    from paper_1612_00001_b200 import engine, workloads

    cfg = workloads.config(args.config)
    k = cfg["k"]
    a = workloads.make_matrix(args.config)
    a_pin = torch.from_numpy(a).pin_memory()
    ws = bri.Workspace()
    targets = cfg["targets"]

    def step(rec):
        sync = torch.cuda.synchronize
        sync()
        t0 = time.perf_counter()
        p = bri.make_memory_provider(a_pin, k)
        sink = bri.MemorySink(p.layout)
        t1 = time.perf_counter()
        tensors, info = engine._execute(p, engine._target_specs(k, targets), ws, targets=targets)
        sync()
        t2 = time.perf_counter()
        for (al, be), t in zip(targets, tensors):
            sink.put(al, be, t)
        t3 = time.perf_counter()
        out = sink.finalize()
        sync()
        t4 = time.perf_counter()
        rec.append({"provider_sink_ms": (t1 - t0) * 1e3, "execute_ms": (t2 - t1) * 1e3,
                    "puts_ms": (t3 - t2) * 1e3, "finalize_ms": (t4 - t3) * 1e3, "total_ms": (t4 - t0) * 1e3})
        return out

    warm = []
    for _ in range(2):
        step(warm)
    recs = []
    for _ in range(args.steps):
        step(recs)
    for r in recs:
        print(json.dumps({k_: round(v, 2) for k_, v in r.items()}))
    # the public call, timed the way bench.py's e2e does
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        p = bri.make_memory_provider(a_pin, k)
        sink = bri.MemorySink(p.layout)
        bri.invert_full(p, sink, ws)
        sink.finalize()
    torch.cuda.synchronize()
    print(json.dumps({"invert_full_ms": (time.perf_counter() - t0) * 1e3 / args.steps}))
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        p = bri.make_memory_provider(a_pin, k)
        sink = bri.MemorySink(p.layout)
        bri.invert_full(p, sink, ws)
        sink.finalize()
        torch.cuda.synchronize()
    mem = {}
    for e in prof.events():
        if "Memcpy" in e.name or "memcpy" in e.name.lower():
            d = mem.setdefault(e.name, [0, 0.0])
            d[0] += 1
            d[1] += (e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total) / 1e3
    print(json.dumps({"memcpy": {n: {"count": c, "ms": round(ms, 2)} for n, (c, ms) in mem.items()}}))


if __name__ == "__main__":
    main()
