"""cProfile of N steps of a config: where host time goes (outlier hunting)."""
import cProfile, os, pstats, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1612_00001_b200 as bri
from paper_1612_00001_b200 import workloads
cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 2
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 40
cfg = workloads.config(cfg_id)
a = torch.from_numpy(workloads.make_matrix(cfg_id)).cuda()
prov = bri.make_memory_provider(a, cfg["k"])
for _ in range(3):
    bri.invert_blocks(prov, cfg["targets"])
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(steps):
    bri.invert_blocks(prov, cfg["targets"])
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(18)
