"""BASELINE config 5's stated check: the block residual ||(M X)[:, 1] - e_1|| (BASELINE's
"(M·X)[:,0] - e0", 0-based) for k=8, b=20480 (M = G + m I, 214.7 GB, generated on the device).

The first block column of X = M^-1 is computed by BRI target by target — (1,1), (2,1), ...,
(k,1), each through the public API (invert_blocks on make_gaussian_provider; each run is the
bounded-footprint schedule with spills to pinned host memory) — and kept in pinned host memory
(k blocks, 27 GB).  Then for every block row r the device forms
  R_r = sum_j M_rj X_j1 - delta_r1 I
with M_rj generated again into arena slots and the library's own batched DMMA GEMM, and reports
max|R_r| and ||R_r||_F, plus max|X_11 - Neumann Y_11| for the (1,1) block.

usage: python tools/run_config5_column.py [--b 20480] [--k 8] [--out profiles/r02_config5_column.json]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--b", type=int, default=20480)
    ap.add_argument("--k", type=int, default=8)
    ap.add_argument("--seed", type=int, default=4)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    import torch

    import paper_1612_00001_b200 as bri
    from paper_1612_00001_b200 import engine
    from paper_1612_00001_b200.device import Arena, release_cached_memory

    torch.cuda.set_device(0)
    k, b = args.k, args.b
    m = k * b
    spec = bri.GaussianSpec(m, args.seed, float(m))
    prov = bri.make_gaussian_provider(spec, k)
    rec = {"workload": "config5-column", "k": k, "b": b, "m": m, "seed": args.seed, "targets": [],
           "input": "GaussianSpec(m, seed, shift m): Philox4x64-10 + Box-Muller, generated into arena slots"}
    col = []
    t_all = time.perf_counter()
    for i in range(1, k + 1):
        t0 = time.perf_counter()
        x, info = bri.invert_blocks(prov, [(i, 1)], bri.Workspace())
        torch.cuda.synchronize()
        host = torch.empty((b, b), dtype=torch.float64, pin_memory=True)
        host.copy_(x[0])
        col.append(host)
        rec["targets"].append({"target": [i, 1], "seconds": time.perf_counter() - t0, "schedule": info.schedule,
                               "dag_nodes": info.dag_nodes, "spills": info.spills, "host_blocks": info.host_blocks})
        print(json.dumps(rec["targets"][-1]), flush=True)
        del x
        release_cached_memory()
    rec["bri_seconds"] = time.perf_counter() - t_all
    engine.release_host_pool()
    torch.cuda.empty_cache()

    # residual, block row by block row: acc = sum_j M_rj X_j1 (row-major), minus I for r = 1
    t1 = time.perf_counter()
    ar = Arena(b, 3, device=0)
    XS, MS, ACC = 0, 1, 2
    rows = []
    worst = 0.0
    for r in range(k):
        for j in range(k):
            ar.tensor[XS, :, :b].copy_(col[j], non_blocking=True)
            ar.randn(spec, [(r, j, MS)])
            # row-major ACC = beta ACC + M_rj @ X_j1
            ar.gemm([(XS, MS, ACC, ACC)], b, b, b, alpha=1.0, beta=0.0 if j == 0 else 1.0)
        res = ar.view(ACC)
        if r == 0:
            res.diagonal().sub_(1.0)
        mx = float(res.abs().max())
        fro = float(torch.linalg.norm(res))
        rows.append({"block_row": r + 1, "max_abs": mx, "fro": fro})
        worst = max(worst, mx)
        print(json.dumps(rows[-1]), flush=True)
    ar.close()
    rec.update({"residual_rows": rows, "residual_max_abs": worst,
                "residual_fro": sum(x["fro"] ** 2 for x in rows) ** 0.5, "residual_s": time.perf_counter() - t1,
                "check": "||(M X)[:, block 1] - E_1||: X's first block column by BRI, M regenerated, DMMA GEMMs"})
    line = json.dumps(rec)
    print(line, flush=True)
    if args.out:
        with open(args.out, "w") as f:
            f.write(json.dumps(rec, indent=1) + "\n")


if __name__ == "__main__":
    main()
