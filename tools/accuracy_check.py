"""Accuracy of one target vs the dense inverse: GPU BRI, CPU BRI (oracle) and the oracle's
1-ulp sensitivity, all on the same matrix.  python tools/accuracy_check.py --config 5 --b 2048"""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import scipy.linalg as sla
import torch
import paper_1612_00001_b200 as bri
from paper_1612_00001_b200 import workloads
from oracle import bri_oracle as orc

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=5)
ap.add_argument("--b", type=int, default=2048)
ap.add_argument("--target", default="1,1")
args = ap.parse_args()
cfg = workloads.config(args.config, args.b)
k, b = cfg["k"], cfg["b"]
al, be = (int(x) for x in args.target.split(","))
a = workloads.make_matrix(args.config, args.b)
gpu = bri.invert_blocks(bri.make_memory_provider(torch.from_numpy(a).cuda(), k), [(al, be)])[0][0].cpu().numpy()
t0 = time.time()
cpu = orc.invert_full(a, k, memo=True, targets=[(al, be)])[(al, be)]
t_cpu = time.time() - t0
pert = a * (1.0 + 2.220446049250313e-16 * np.random.Generator(np.random.PCG64(123)).standard_normal(a.shape))
cpu_p = orc.invert_full(pert, k, memo=True, targets=[(al, be)])[(al, be)]
lu, piv = sla.lu_factor(a)
e = np.zeros((a.shape[0], b)); e[(be - 1) * b + np.arange(b), np.arange(b)] = 1.0   # columns of block column beta
col = sla.lu_solve((lu, piv), e)                                                    # M^-1[:, block col beta]
dense = col[(al - 1) * b: al * b, :]
rel = lambda x, y: float(np.abs(x - y).max() / np.abs(y).max())
print(json.dumps({"config": args.config, "b": b, "k": k, "target": [al, be],
                  "gpu_vs_dense": rel(gpu, dense), "cpu_bri_vs_dense": rel(cpu, dense),
                  "gpu_vs_cpu_bri": rel(gpu, cpu), "cpu_1ulp_floor": rel(cpu_p, cpu), "oracle_s": t_cpu}))
