"""Generate golden vectors by running the UNMODIFIED reference package.

Run once in the build container (the reference is importable there, it does
not exist on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes tests/golden/golden.npz.  Every array comes out of the reference's own
public API (`bri.invert_block`, `bri.invert_full`, `bri.invert_dense`,
`bri.lu_factor`, `bri.reduce_frame` trace hook, `bri.predicted_counts`) on
seeded PCG64 inputs (the reference's convention, pkg/tests/conftest.py:9-15).
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import bri  # noqa: E402  (the reference)

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")


def rng(seed):
    return np.random.Generator(np.random.PCG64(seed))


def shifted(m, seed):
    return rng(seed).standard_normal((m, m)) + m * np.eye(m)


def main():
    arrays = {}
    meta = {"cases": []}

    # 1. worked 2x2 example (pkg/tests/test_engine.py:149-157)
    a = np.array([[4.0, 2.0], [1.0, 3.0]])
    prov = bri.make_memory_provider(a, 2)
    for al in (1, 2):
        for be in (1, 2):
            blk = bri.invert_block(prov, al, be)
            arrays[f"worked_{al}{be}"] = blk.data.copy()
            blk.release()

    # 2. scalar 4x4 trace (pkg/tests/test_engine.py:228-255)
    a = shifted(4, 7)
    arrays["trace4_matrix"] = a
    seen = {}
    out = bri.invert_block(bri.make_memory_provider(a, 4), 1, 1, bri.Workspace(),
                           trace=lambda p, f, v: seen.__setitem__("/".join(q.name for q in p), v.copy()))
    for path, v in seen.items():
        arrays[f"trace4_node_{path}"] = v
    arrays["trace4_out"] = out.data.copy()
    meta["trace4_paths"] = list(seen.keys())

    # 3. BASELINE config 1 (k=4, b=64, Uniform[-1,1] + m I, seed 0), all 16 blocks
    m = 256
    a = rng(0).uniform(-1.0, 1.0, (m, m)) + m * np.eye(m)
    prov = bri.make_memory_provider(a, 4)
    sink = bri.MemorySink(prov.layout)
    ws = bri.Workspace()
    summ = bri.invert_full(prov, sink, ws)
    arrays["cfg1_inverse"] = sink.finalize().copy()
    meta["cfg1_counters"] = [summ.counters.block_inversions, summ.counters.block_multiplications,
                             summ.counters.block_subtractions, summ.counters.schur_nodes]

    # 4. small random cases over k, b and targets (row-major block outputs)
    cases = [(6, 3, 11), (8, 4, 12), (12, 3, 13), (12, 4, 14), (16, 4, 15), (20, 5, 16),
             (24, 6, 17), (32, 4, 18), (48, 6, 19), (64, 4, 20), (96, 3, 21), (128, 4, 22)]
    for m, k, seed in cases:
        a = shifted(m, seed)
        name = f"rand_m{m}_k{k}_s{seed}"
        arrays[name + "_matrix"] = a
        prov = bri.make_memory_provider(a, k)
        for al, be in {(1, 1), (1, k), (k, 1), (2, min(3, k)), (k, k)}:
            blk = bri.invert_block(prov, al, be)
            arrays[f"{name}_t{al}_{be}"] = blk.data.copy()
            blk.release()
        meta["cases"].append([m, k, seed])

    # 5. SPD class (G G^T / m + I) at k=2 (config-2 class, small)
    for m, seed in ((64, 1), (128, 1)):
        g = rng(seed).standard_normal((m, m))
        a = g @ g.T / m + np.eye(m)
        arrays[f"spd_m{m}_matrix"] = a
        blk = bri.invert_block(bri.make_memory_provider(a, 2), 1, 1)
        arrays[f"spd_m{m}_t1_1"] = blk.data.copy()
        blk.release()

    # 6. singular anchor (pkg/tests/test_engine.py:209-225)
    a = shifted(6, 85)
    a[2:4, 2:4] = 0.0
    try:
        bri.invert_block(bri.make_memory_provider(a, 3), 1, 1)
        meta["singular"] = None
    except bri.SingularPivotError as e:
        meta["singular"] = {"path": [q.name for q in e.path], "pivot_block": list(e.pivot_block)}
    arrays["singular_matrix"] = a

    # 7. dense kernels: invert_dense / lu_factor known answers
    arrays["hilbert4_inv"] = bri.lu_invert_full(1.0 / (np.arange(4)[:, None] + np.arange(4)[None, :] + 1.0))
    r = rng(5).standard_normal((6, 6))
    fac = bri.lu_factor(bri.Workspace().from_array(r))
    arrays["lu6_matrix"] = r
    arrays["lu6_packed"] = fac.packed_lu.copy()
    arrays["lu6_pivots"] = fac.pivots.copy()
    for n in (1, 5, 12, 33, 64, 100):
        x = shifted(n, 500 + n)
        arrays[f"inv{n}_matrix"] = x
        arrays[f"inv{n}_out"] = bri.invert_dense(bri.Workspace().from_array(x)).data.copy()

    # 8. padded layouts (m % k != 0): shifted-window runs (providers.py:338-402)
    meta["padded"] = []
    for m, k, seed in ((10, 4, 88), (13, 4, 13), (30, 8, 30), (50, 6, 51)):
        a = shifted(m, seed)
        prov = bri.make_memory_provider(a, k)
        sink = bri.MemorySink(prov.layout)
        bri.invert_full(prov, sink)
        arrays[f"pad_m{m}_k{k}_matrix"] = a
        arrays[f"pad_m{m}_k{k}_inverse"] = sink.finalize().copy()
        meta["padded"].append([m, k, seed])

    # 9. LS-SVM kernel system (providers.py:93-120,175-200; pkg/tests/test_providers.py:100-136,
    #    test_acceptance.py:195-205): full matrices, a padded layout and full inverses
    meta["kernel"] = []
    for name, n, d, gamma, sigma, seed, k in (("k63", 63, 3, 1.0, 1.0, 63, 4), ("k5", 5, 3, 1.5, 0.8, 32, 2),
                                              ("k40", 40, 9, 2.0, 1.3, 7, 4), ("k150", 150, 200, 0.5, 9.0, 8, 3)):
        x = rng(seed).standard_normal((n, d))
        spec = bri.KernelSpec(inputs=x, gamma=gamma, sigma=sigma)
        arrays[f"kern_{name}_inputs"] = x
        arrays[f"kern_{name}_matrix"] = bri.kernel_matrix(spec)
        prov = bri.make_kernel_provider(spec, k)
        sink = bri.MemorySink(prov.layout)
        bri.invert_full(prov, sink)
        arrays[f"kern_{name}_inverse"] = sink.finalize().copy()
        meta["kernel"].append([name, n, d, gamma, sigma, k])

    # 10. exact operation counts k=2..7 (pkg/tests/test_instrumentation.py:42-50)
    meta["counts"] = {str(k): [c.block_inversions, c.block_multiplications, c.block_subtractions,
                               c.schur_nodes] for k in range(2, 8) for c in [bri.predicted_counts(k)]}

    np.savez_compressed(OUT, meta=np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8), **arrays)
    print(f"wrote {OUT}: {len(arrays)} arrays")


if __name__ == "__main__":
    main()
