"""Launch every hot-path kernel family a few times for `ncu --set full` captures (one kernel per
capture with -k regex:NAME -s SKIP -c 1):

  small_node_kernel   config 1 (k=4, b=64) full inverse, 116 nodes in 3 launches
  randn_kernel        8 config-5-style blocks of order 4096 generated into slots (HBM writes)
  lu_panel_kernel, rowpanel_kernel, trsm_kernel, gemm_kernel, skinny_kernel, laswp_kernel
                      one config-2-shaped node (k=2, b=4096) + final inversion
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1612_00001_b200 as bri
from paper_1612_00001_b200.device import Arena

torch.cuda.set_device(0)
a = np.random.Generator(np.random.PCG64(0)).uniform(-1.0, 1.0, (256, 256)) + 256 * np.eye(256)
prov = bri.make_memory_provider(a, 4)
for _ in range(3):
    bri.invert_full(prov, bri.MemorySink(prov.layout))
with Arena(4096, 8, device=0) as ar:
    spec = bri.GaussianSpec(8 * 4096, 4, float(8 * 4096))
    for _ in range(3):
        ar.randn(spec, [(i, 0, i) for i in range(8)])
    torch.cuda.synchronize()
g = bri.make_gaussian_provider(bri.GaussianSpec(8192, 4, 8192.0), 2)
for _ in range(3):
    bri.invert_block(g, 1, 1)
torch.cuda.synchronize()
print("probe done")
