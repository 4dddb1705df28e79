"""Summarise `ncu --set full` reports (one kernel each) into JSON: duration, DRAM traffic and
GB/s, FP64 tensor (DMMA) pipe utilisation, SM / memory throughput, occupancy, registers.

    python tools/ncu_summary.py gpurun_out/ncu_*.ncu-rep > profiles/r01_kernels_ncu.json
"""
import csv
import io
import json
import subprocess
import sys

WANT = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active": "dmma_pipe_pct_active",
    "sm__ops_path_tensor_src_fp64.avg.pct_of_peak_sustained_elapsed": "fp64_tensor_pct_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "memory_throughput_pct",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "launch__cluster_size": "cluster",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active": "fp64_alu_pipe_pct_active",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
}
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
              "s": 1, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1}


def summarise(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units, vals = rows[0], rows[1], rows[2]
    out = {"report": path.split("/")[-1], "kernel": vals[head.index("Kernel Name")].split("(")[0]}
    for name, key in WANT.items():
        if name in head:
            i = head.index(name)
            v = vals[i].replace(",", "")
            try:
                x = float(v) * UNIT_SCALE.get(units[i], 1)
            except ValueError:
                x = v
            out[key] = x
    if "duration" in out and "dram_read" in out:
        out["dram_bytes"] = out["dram_read"] + out["dram_write"]
        out["dram_GBps"] = out["dram_bytes"] / out["duration"] / 1e9
        out["duration_us"] = out.pop("duration") * 1e6
    return out


if __name__ == "__main__":
    print(json.dumps([summarise(p) for p in sys.argv[1:]], indent=1))
