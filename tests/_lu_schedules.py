"""Helper for test_lu_schedules_agree (run in a subprocess: the LU schedule
switches BRI_LOOKAHEAD / BRI_LU_EXTEND are read once per process).  Writes each
result and its max-abs error against numpy's LAPACK inverse."""
import sys

import numpy as np
import torch

import paper_1612_00001_b200 as bri
from paper_1612_00001_b200 import baseline

out = sys.argv[1]
g = np.random.Generator(np.random.PCG64(77))
dense = g.standard_normal((1000, 1000))               # one factorization, 8 outer blocks
inv = baseline.lu_invert_full(dense)
# k = 8: batches of order-384..2688 factorizations; a weak diagonal shift keeps
# partial pivoting busy (and the pivot blocks poorly conditioned)
a = g.standard_normal((3072, 3072)) + 8.0 * np.eye(3072)
targets = [(1, 1), (3, 5), (8, 8)]
blocks = bri.invert_blocks(bri.make_memory_provider(torch.from_numpy(a).cuda(), 8), targets)[0]
res = {"dense": inv}
err = {"dense": np.abs(inv - np.linalg.inv(dense)).max() / np.abs(inv).max()}
ainv = np.linalg.inv(a)
for (i, j), x in zip(targets, blocks):
    x = x.cpu().numpy()
    want = ainv[(i - 1) * 384:i * 384, (j - 1) * 384:j * 384]
    res[f"b{i}{j}"] = x
    err[f"b{i}{j}"] = np.abs(x - want).max() / np.abs(want).max()
np.savez(out, **res, **{"err_" + k: v for k, v in err.items()})
