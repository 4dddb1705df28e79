"""Phase split of a timeline.json (tools/timeline.py): LU runs = maximal runs of lu_panel_kernel
launches separated by < 300 us; everything between them is reported as the gap phase."""
import json, sys
d = json.load(open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/timeline.json"))
ev = d["events"]
t_end = max(t + dur for _, _, t, dur, _ in ev)
pan = sorted((t, t + dur) for name, _, t, dur, _ in ev if name.startswith("lu_panel"))
runs = []
for s, e in pan:
    if runs and s - runs[-1][1] < 300:
        runs[-1][1] = e
    else:
        runs.append([s, e])
prev = ev[0][2]
for i, (s, e) in enumerate(runs):
    print(f"pre-LU{i+1} {s - prev:9.0f} us   LU{i+1} panels {e - s:9.0f} us  ({s:.0f}..{e:.0f})")
    prev = e
print(f"tail     {t_end - prev:9.0f} us   total {t_end - ev[0][2]:.0f} us")
