"""Host latency from invert_blocks() entry to its first device work (GPU idle at step start)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1612_00001_b200 as bri
from paper_1612_00001_b200 import _native, workloads
cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 2
cfg = workloads.config(cfg_id)
a = torch.from_numpy(workloads.make_matrix(cfg_id)).cuda()
prov = bri.make_memory_provider(a, cfg["k"])
lib = _native.load_library()
marks = []
for name in ("bri_gather_blocks", "bri_gather_elements", "bri_schur_batch", "bri_schur_batch_gated",
             "bri_invert_batch", "bri_load_host_blocks"):
    if hasattr(lib, name):
        f = getattr(lib, name)
        def wrap(*args, _f=f, _n=name):
            marks.append((_n, time.perf_counter()))
            r = _f(*args)
            marks.append((_n + ":ret", time.perf_counter()))
            return r
        setattr(lib, name, wrap)
for _ in range(4):
    bri.invert_blocks(prov, cfg["targets"])
torch.cuda.synchronize()
for _ in range(3):
    marks.clear()
    t0 = time.perf_counter()
    bri.invert_blocks(prov, cfg["targets"])
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print([(n, round((t - t0) * 1e3, 3)) for n, t in marks], "call", round((t1 - t0) * 1e3, 3), "sync", round((t2 - t0) * 1e3, 3))
