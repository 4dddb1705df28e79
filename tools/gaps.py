"""Idle gaps of a tools/timeline.py trace (no kernel on any stream): the largest ones with the
kernels that end before and start after them, and a histogram.

    python tools/gaps.py gpurun_out/timeline.json [--top 20]
"""
import json
import sys

path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/timeline.json"
top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 20
ev = sorted(json.load(open(path))["events"], key=lambda e: e[2])   # (name, stream, ts, dur, ...)
gaps, end, last = [], None, None
for name, stream, t, dur, *_ in ev:
    if end is not None and t > end:
        gaps.append((t - end, end - ev[0][2], last, (name, stream)))
    if end is None or t + dur > end:
        end, last = t + dur, (name, stream)
gaps.sort(reverse=True)
tot = sum(g[0] for g in gaps)
print(f"{len(gaps)} gaps, {tot:.0f} us idle")
for lo, hi in ((0, 5), (5, 10), (10, 20), (20, 50), (50, 100), (100, 1e9)):
    sel = [g[0] for g in gaps if lo <= g[0] < hi]
    print(f"  [{lo:>4}, {hi:>6}) us: {len(sel):4d} gaps, {sum(sel):8.0f} us")
for g, at, before, after in gaps[:top]:
    print(f"{g:8.1f} us at {at:9.0f}: {before[0]}@{before[1]} -> {after[0]}@{after[1]}")
