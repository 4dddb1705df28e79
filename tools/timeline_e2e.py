"""CUPTI timeline of one e2e step (pinned host input -> result on the host), with memcpys."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1612_00001_b200 as bri
from paper_1612_00001_b200 import workloads

a = workloads.make_matrix(2)
a_pin = torch.from_numpy(a).pin_memory()
def step():
    p = bri.make_memory_provider(a_pin, 2)
    blk = bri.invert_block(p, 1, 1)
    h = blk.data
    blk.release()
    return h
for _ in range(3):
    step()
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA, torch.profiler.ProfilerActivity.CPU]) as prof:
    step()
    torch.cuda.synchronize()
prof.export_chrome_trace("/tmp/e2e.json")
ev = json.load(open("/tmp/e2e.json"))["traceEvents"]
gpu = sorted([e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")], key=lambda e: e["ts"])
t0 = gpu[0]["ts"]
print("gpu span ms", (max(e["ts"] + e["dur"] for e in gpu) - t0) / 1e3)
for e in gpu:
    if e.get("cat") == "gpu_memcpy" or e["dur"] > 3000:
        print(f'{e["cat"]:12s} {e["name"][:40]:40s} t={(e["ts"]-t0)/1e3:8.2f} dur={e["dur"]/1e3:7.2f} ms')
last = t0; gaps = []
for e in gpu:
    if e["ts"] - last > 100: gaps.append(((e["ts"] - last) / 1e3, (e["ts"] - t0) / 1e3, e["name"][:30]))
    last = max(last, e["ts"] + e["dur"])
print("gaps > 0.1 ms:", [(round(g, 2), round(t, 2), n) for g, t, n in gaps])
