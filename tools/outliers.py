"""Profile N steps of a config with CUPTI (torch.profiler) and explain slow steps:
per step wall, busy, idle gaps and the kernels that grew vs the median step."""
import json, os, sys, collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1612_00001_b200 as bri
from paper_1612_00001_b200 import workloads

cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 2
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 30
cfg = workloads.config(cfg_id)
a = torch.from_numpy(workloads.make_matrix(cfg_id)).cuda()
prov = bri.make_memory_provider(a, cfg["k"])
for _ in range(3):
    bri.invert_blocks(prov, cfg["targets"])
torch.cuda.synchronize()
marks = []
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    for i in range(steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); bri.invert_blocks(prov, cfg["targets"]); e1.record()
        marks.append((e0, e1))
    torch.cuda.synchronize()
ms = [e0.elapsed_time(e1) for e0, e1 in marks]
prof.export_chrome_trace("/tmp/outl.json")
ev = sorted([e for e in json.load(open("/tmp/outl.json"))["traceEvents"] if e.get("cat") == "kernel"], key=lambda e: e["ts"])
# split into steps by the gather kernel that starts every step
starts = [i for i, e in enumerate(ev) if e["name"].find("gather_kernel") >= 0]
starts.append(len(ev))
rows = []
for s in range(len(starts) - 1):
    seg = ev[starts[s]:starts[s + 1]]
    t0, t1 = seg[0]["ts"], max(e["ts"] + e["dur"] for e in seg)
    per = collections.Counter()
    gaps = []
    end = seg[0]["ts"]
    for k, e in enumerate(seg):
        nm = e["name"].replace("(anonymous namespace)::", "").replace("bri::", "").replace("void ", "")
        nm = nm.split("(")[0].split("<")[0]
        per[nm] += e["dur"]
        if e["ts"] > end + 50:
            gaps.append((round((e["ts"] - end) / 1e3, 2), k, nm, round((e["ts"] - t0) / 1e3, 2)))
        end = max(end, e["ts"] + e["dur"])
    rows.append({"wall": round((t1 - t0) / 1e3, 2), "n": len(seg), "per": per, "gaps": sorted(gaps, reverse=True)[:4]})
med = sorted(r["wall"] for r in rows)[len(rows) // 2]
mp = rows[[r["wall"] for r in rows].index(med)]["per"]
print(json.dumps({"event_ms": [round(x, 2) for x in ms], "kernel_walls": [r["wall"] for r in rows]}))
for i, r in enumerate(rows):
    if r["wall"] > 1.1 * med:
        grew = sorted(((k, round((v - mp.get(k, 0)) / 1e3, 2)) for k, v in r["per"].items()), key=lambda x: -x[1])[:5]
        print("step", i, "wall", r["wall"], "kernels", r["n"], "grew(ms):", grew[:3], "gaps(ms, idx, next kernel, at):", r["gaps"])
