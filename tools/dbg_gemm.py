import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_1612_00001_b200.device import Arena
n = int(sys.argv[1]); a0 = (int(sys.argv[2]), int(sys.argv[3])); K = int(sys.argv[4]); beta = float(sys.argv[5])
rng = np.random.default_rng(0)
ar = Arena(n, 4)
host = rng.standard_normal((4, n, n))
for s in range(4): ar.view(s).copy_(torch.from_numpy(host[s]))
X = [h.T for h in host]
M, N = n // 2, n // 2
ar.gemm([(0, 1, 2, 3)], M, N, K, a0=a0, b0=(0, 0), c0=(0, 0), alpha=1.0, beta=beta)
torch.cuda.synchronize()
got = ar.view(3).cpu().numpy().T[:M, :N]
want = X[0][a0[0]:a0[0]+M, a0[1]:a0[1]+K] @ X[1][:K, :N] + beta * X[2][:M, :N]
print(sys.argv[1:], "err", np.abs(got - want).max())
