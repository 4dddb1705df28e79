import sys, numpy as np, torch
sys.path.insert(0, '.')
from scipy.linalg import lapack
from paper_1612_00001_b200.device import Arena
for n in [1, 2, 3, 5, 64, 100, 200, 600]:
    rng = np.random.default_rng(n)
    a = rng.standard_normal((n, n)) + n * np.eye(n)
    bm = rng.standard_normal((n, n))
    ar = Arena(n, 3)
    ar.view(0).copy_(torch.from_numpy(a)); ar.view(1).copy_(torch.from_numpy(bm))
    perm = torch.zeros(n, dtype=torch.int32, device='cuda'); st = torch.zeros(1, dtype=torch.int32, device='cuda')
    ar.getrf([0], perm, st)
    lu_got = ar.view(0).cpu().numpy().T
    lu, piv, info = lapack.dgetrf(a.T)
    e1 = np.abs(lu_got - lu).max()
    ar.getrs([(0, 1, 2)], perm)
    x = ar.view(2).cpu().numpy().T     # X-world solution of A^T x = B^T
    want = np.linalg.solve(a.T, bm.T)
    e2 = np.abs(x - want).max() / np.abs(want).max()
    # gemm n: C = C - A*B
    ar.view(0).copy_(torch.from_numpy(a)); ar.view(1).copy_(torch.from_numpy(bm)); ar.view(2).copy_(torch.from_numpy(bm))
    ar.gemm([(0, 1, 2, 2)], n, n, n, alpha=-1.0, beta=1.0)
    c = ar.view(2).cpu().numpy().T
    e3 = np.abs(c - (bm.T - a.T @ bm.T)).max()
    print(n, 'getrf', e1, 'getrs', e2, 'gemm', e3, 'status', int(st.item()), flush=True)
