"""Per-step device times of a config (distribution, not just the mean)."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1612_00001_b200 as bri
from paper_1612_00001_b200 import workloads
cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 2
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 12
cfg = workloads.config(cfg_id)
a = torch.from_numpy(workloads.make_matrix(cfg_id)).cuda()
prov = bri.make_memory_provider(a, cfg["k"])
import gc, time as _t
gc.disable()
ts = []; hs = []
for i in range(steps):
    h0 = _t.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); bri.invert_blocks(prov, cfg["targets"]); e1.record(); torch.cuda.synchronize()
    ts.append(round(e0.elapsed_time(e1), 2)); hs.append(round((_t.perf_counter() - h0) * 1e3, 2))
print(json.dumps({"config": cfg_id, "ms": ts, "host_ms": hs, "lookahead": os.environ.get("BRI_LOOKAHEAD", "1"),
                  "graphs": os.environ.get("BRI_GRAPHS", "1")}))
