"""Pivot-chain analysis of a config-2 kernel timeline (tools/timeline.py --config 2 --out X.json):
per factorization, the spacing between the ends of consecutive LU panel kernels, grouped by outer
block (4 inner panels each) — a stall shows up as spacing well above panel + ~10 us — plus the
time between / after the two factorizations.

    python tools/chain_gaps.py gpurun_out/timeline.json
"""
import json
import sys

import numpy as np

d = json.load(open(sys.argv[1]))
ev = d["events"]
panels = [e for e in ev if e[0] == "lu_panel_kernel"]
ends = [e[2] + e[3] for e in panels]
starts = [e[2] for e in panels]
half = len(panels) // 2
print(f"wall {d['summary']['wall_us']:.0f} us, {len(panels)} panel launches ({half} per factorization)")
for name, lo, hi in (("LU of p (Schur node, folded W)", 0, half), ("LU of S (inverse, folded L^-1)", half, len(panels))):
    sp = np.diff(ends[lo:hi])
    dur = ends[hi - 1] - starts[lo]
    floor = float(np.sum(np.minimum(sp, np.percentile(sp, 25) * 1.5)))
    print(f"\n{name}: first panel start -> last panel end {dur:.0f} us; spacing sum {sp.sum():.0f} us, "
          f"median {np.median(sp):.1f}, p90 {np.percentile(sp, 90):.1f}, max {sp.max():.0f}")
    print("spacing of consecutive panel ends per outer block (us):")
    line = []
    for blk in range((hi - lo) // 4):
        seg = sp[blk * 4: blk * 4 + 4]
        line.append(f"{blk:2d} {[int(round(x)) for x in seg]}")
        if len(line) == 4:
            print("  " + " | ".join(line))
            line = []
    if line:
        print("  " + " | ".join(line))
print(f"\nbetween the factorizations (U sweep of W, node GEMM, copy, max|S|): {starts[half] - ends[half - 1]:.0f} us")
print(f"after the last panel (U sweep of the inverse, column scatter): {d['summary']['wall_us'] - ends[-1]:.0f} us")
print(f"before the first panel (gather, copy, max|p|; host time under the profiler): {starts[0]:.0f} us")
agg = {}
for e in ev:
    a = agg.setdefault(e[0], [0, 0.0])
    a[0] += 1
    a[1] += e[3]
print("\nkernel time (sum of durations; early-resident chain kernels include their wait):")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:12]:
    print(f"  {k:28s} n={v[0]:5d} {v[1]:10.1f} us")
