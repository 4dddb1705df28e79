"""Helper for test_small_node_schedules_bitwise (run in a subprocess: BRI_SMALL_BLOCKED is read
once per process).  Full inverses through the small-node kernel (b <= 96) on heavily pivoting,
diagonally dominant and singular inputs, every result written for a bitwise comparison."""
import sys

import numpy as np

import paper_1612_00001_b200 as bri

out = sys.argv[1]
g = np.random.Generator(np.random.PCG64(2024))
res = {}
for k, b in [(2, 1), (3, 2), (2, 7), (4, 16), (3, 31), (2, 32), (4, 33), (2, 50), (4, 64), (2, 65), (3, 80), (2, 96)]:
    m = k * b
    for kind in ("pivoting", "dominant"):
        a = g.standard_normal((m, m))
        if kind == "dominant":
            a += m * np.eye(m)
        prov = bri.make_memory_provider(a, k)
        sink = bri.MemorySink(prov.layout)
        try:
            bri.invert_full(prov, sink)
            res[f"{kind}_{k}_{b}"] = sink.finalize()
        except bri.BriError as exc:   # a singular pivot block is part of the comparison too
            res[f"{kind}_{k}_{b}"] = np.frombuffer(repr(exc).encode(), dtype=np.uint8)
# a singular pivot: the reported branch and anchor must not depend on the schedule
a = g.standard_normal((96, 96))
a[32:64, 32:64] = 0.0
try:
    bri.invert_block(bri.make_memory_provider(a, 3), 1, 1)
    res["singular"] = np.zeros(1)
except bri.BriError as exc:
    res["singular"] = np.frombuffer(repr(exc).encode(), dtype=np.uint8)
np.savez(out, **res)
