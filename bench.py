"""Benchmark: FP64 TFLOP/s and seconds per inverse block of the BRI hot path on B200.

Default workload = BASELINE.json configs[1] ("config 2"): k=2, b=4096 (m=8192),
SPD M = G G^T/m + I from PCG64 seed 1, inverse block (1,1) — one Schur node
(1 factorization + 1 solve + 1 fused GEMM-subtract) plus the final b x b
inversion.  A "step" is one complete inversion of the requested target(s).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C]

value      : algorithmic FP64 TFLOP/s (SURVEY §8(d) convention: 6b^3+b^2 per Schur node
             executed + 2b^3 per target), M resident in HBM, device-timed (CUDA events).
e2e        : same metric through the public API from pinned HOST memory: H2D of M and
             D2H of the result block inside the timed region.
roofline   : dominant kernel = the fused Schur GEMM (gemm_kernel, C = R - RT*W, b^3 DMMA
             tile work), timed live with CUDA events; peak = FP64 DMMA throughput measured
             in this run by bri_fp64_peak (MEASURED_PEAKS.json has no FP64 entry).
cpu_baseline: the oracle port (numpy/scipy = the reference's own LAPACK/BLAS calls) on this
             host's cores, one target per sample.
Multi-GPU: multi-target configs run one DAG with each level's nodes dealt to ranks and one NCCL
P2P operand exchange per level (--shard nodes, default; strong scaling), or each rank its own
chunk of targets gathered to rank 0 at the end (--shard targets); a single-target config runs
one replica per rank (weak).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "FP64 TFLOP/s (% of FP64 tensor peak) and sec per inverse block vs CPU ref"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--b", type=int, default=None, help="override block order (proxy runs)")
    ap.add_argument("--schedule", default="dag", choices=["dag", "tree"])
    ap.add_argument("--shard", default="nodes", choices=["nodes", "targets"],
                    help="multi-GPU, multi-target configs: one DAG with its levels dealt to ranks "
                         "(nodes) or each rank its own chunk of targets (targets)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run_nvml(self):
        """In-process NVML queries: no nvidia-smi process spawned next to the timed region."""
        import pynvml as nv

        nv.nvmlInit()
        h = nv.nvmlDeviceGetHandleByIndex(self.index)
        bits = (nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap)
        while not self._stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.rows.append([str(sm), str(mx), "", ""] + ["Active" if r & b else "Not Active" for b in bits])
            except Exception:
                pass
            self._stop.wait(0.1)

    def _run(self):
        try:
            import pynvml  # noqa: F401

            return self._run_nvml()
        except Exception:
            pass
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=6)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 4 + i and "Active" in r[4 + i]
                          and "Not" not in r[4 + i]})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ------------------------------------------------------------------ helpers
def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def cpu_oracle_step(a, k, targets):
    from oracle import bri_oracle as orc

    memo = {}
    src = orc.BlockSource(a, k)
    out = []
    for al, be in targets:
        out.append(orc.invert_block(src, k, al, be, memo=memo))
    return out


def ncu_traffic():
    """dram bytes per launch of the Schur GEMM from the committed ncu --set full summary, if any."""
    path = os.path.join(ROOT, "profiles", "gemm_ncu_summary.json")
    try:
        with open(path) as fh:
            return json.load(fh).get("dram_bytes_per_launch")
    except Exception:
        return None


# ------------------------------------------------------------------ reference arm
def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from paper_1612_00001_b200 import workloads

    cfg = workloads.config(args.config, args.b)
    k, b = cfg["k"], cfg["b"]
    a = workloads.make_matrix(args.config, args.b)
    targets = cfg["targets"][:1]  # bounded sample: one target per step
    from paper_1612_00001_b200.dag import build_schedule

    nodes = len(build_schedule(k, targets).nodes)
    flops = workloads.run_flops(b, nodes, len(targets))
    for _ in range(args.warmup):
        cpu_oracle_step(a, k, targets)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        cpu_oracle_step(a, k, targets)
        times.append(time.perf_counter() - t0)
    sec = sum(times) / len(times)
    tf = flops / sec / 1e12
    cores = os.cpu_count()
    line = {
        "impl": "reference", "metric": METRIC, "value": tf, "unit": "TFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (PCG64, BASELINE configs)",
        "config": {"workload": f"config{args.config}", "k": k, "b": b, "m": k * b, "targets": [list(t) for t in targets],
                   "memoized": True},
        "sec_per_block": sec / len(targets),
        "cpu_baseline": {"value": tf, "unit": "TFLOP/s", "cores": cores, "kind": "port",
                         "sample": f"{len(targets)} target(s) of config {args.config} per step, memoized oracle "
                                   "(numpy/scipy LAPACK, the reference's own calls)"},
        "e2e": {"value": tf, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


# ------------------------------------------------------------------ our arm
def run_ours(args):
    import torch

    rank, world, local = dist_env()
    if not torch.cuda.is_available():
        print(json.dumps({"metric": METRIC, "error": "no CUDA device"}))
        sys.exit(1)
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))

    import paper_1612_00001_b200 as bri
    from paper_1612_00001_b200 import _native, workloads
    from paper_1612_00001_b200.dag import build_schedule
    from paper_1612_00001_b200.device import fp64_peak_tflops

    cfg = workloads.config(args.config, args.b)
    k, b = cfg["k"], cfg["b"]
    a = workloads.make_matrix(args.config, args.b)
    from paper_1612_00001_b200.distributed import gather_blocks, shard_targets

    my_targets, scaling = shard_targets(cfg["targets"], rank, world)
    node_shard = world > 1 and len(cfg["targets"]) > 1 and args.shard == "nodes"
    if node_shard:  # one DAG for the job: every rank walks all targets, nodes dealt per level
        my_targets = list(cfg["targets"])
    sched = build_schedule(k, my_targets)
    flops_rank = workloads.run_flops(b, len(sched.nodes), len(my_targets))
    if node_shard:
        flops_rank /= world   # summed over ranks below: the job's algorithmic FLOPs once

    a_dev = torch.from_numpy(a).to(f"cuda:{local}")
    prov = bri.make_memory_provider(a_dev, k)
    stream = torch.cuda.current_stream()
    ws = bri.Workspace(schedule=args.schedule)

    def step():
        if node_shard:
            tensors, _ = bri.invert_blocks_sharded(prov, my_targets, ws)
            return tensors
        tensors, _ = bri.invert_blocks(prov, my_targets, ws)
        return tensors

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- device-resident timing (value)
    for _ in range(args.warmup):
        step()
    barrier()
    lib = _native.load_library()
    l0 = lib.bri_launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            out = step()
        e1.record(stream)
        barrier()
    launches = (lib.bri_launch_count() - l0) // args.steps
    ms = e0.elapsed_time(e1) / args.steps
    ms_all = ms
    if dist is not None:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_all = float(t.item())
        tot = torch.tensor([flops_rank], device="cuda", dtype=torch.float64)
        dist.all_reduce(tot)
        flops_total = float(tot.item())
    else:
        flops_total = flops_rank
    value = flops_total / (ms_all * 1e-3) / 1e12

    # ---- gather results to rank 0 (strong scaling: the full inverse lands on rank 0)
    if dist is not None and scaling == "strong" and not node_shard:
        gather_blocks(out, cfg["targets"], rank, world, b)

    # ---- end-to-end through the public API from pinned host memory
    a_pin = torch.from_numpy(a).pin_memory()

    def e2e_step():
        p = bri.make_memory_provider(a_pin, k)
        if node_shard:
            res = bri.invert_blocks_sharded(p, my_targets, ws)[0] or []
            blocks = [bri.Block(x, ws) for x in res]
        else:
            blocks = [bri.invert_block(p, *t, ws) for t in my_targets] if len(my_targets) == 1 else \
                [bri.Block(x, ws) for x in bri.invert_blocks(p, my_targets, ws)[0]]
        host = [blk.data for blk in blocks]
        for blk in blocks:
            blk.release()
        return host

    for _ in range(max(1, args.warmup)):
        e2e_step()
    barrier()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    for _ in range(args.steps):
        e2e_step()
    f1.record(stream)
    barrier()
    e2e_ms = f0.elapsed_time(f1) / args.steps
    if dist is not None:
        t = torch.tensor([e2e_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e_value = flops_total / (e2e_ms * 1e-3) / 1e12
    h2d = a.nbytes
    d2h = len(my_targets) * b * b * 8

    # ---- roofline of the dominant kernel: the fused Schur GEMM (b x b x b)
    peak = fp64_peak_tflops()
    from paper_1612_00001_b200.device import Arena

    reps = 5
    with Arena(b, 4, device=local) as ar:
        for s in range(4):
            ar.view(s).normal_()
        ar.gemm([(0, 1, 2, 3)], b, b, b, alpha=-1.0, beta=1.0)
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        g0.record(stream)
        for _ in range(reps):
            ar.gemm([(0, 1, 2, 3)], b, b, b, alpha=-1.0, beta=1.0)
        g1.record(stream)
        torch.cuda.synchronize()
        gemm_ms = g0.elapsed_time(g1) / reps
    gemm_flops = 2.0 * b ** 3 + b ** 2
    achieved = gemm_flops / (gemm_ms * 1e-3) / 1e12
    traffic = ncu_traffic()

    # ---- CPU baseline (rank 0, N = 1 only): one target of the same workload on host cores
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        sample = cfg["targets"][:1]
        nodes_s = len(build_schedule(k, sample).nodes)
        t0 = time.perf_counter()
        cpu_oracle_step(a, k, sample)
        dt = time.perf_counter() - t0
        cpu = {"value": workloads.run_flops(b, nodes_s, 1) / dt / 1e12, "unit": "TFLOP/s",
               "cores": os.cpu_count(), "kind": "port", "sec_per_block": dt,
               "sample": f"target {sample[0]} of config {args.config} (k={k}, b={b}), memoized oracle = "
                         "numpy/scipy LAPACK calls of the reference, all host cores"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_all, "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (PCG64 seeds of BASELINE.json configs)",
            "config": {"workload": f"config{args.config}", "k": k, "b": b, "m": k * b,
                       "targets": len(cfg["targets"]), "schedule": args.schedule,
                       "dag_nodes_per_rank": len(sched.nodes) if not node_shard else None,
                       "dag_nodes": len(sched.nodes),
                       "shard": (args.shard if node_shard else "targets") if world > 1 else None,
                       "l2": "inputs larger than L2 (M = %.0f MiB > 126 MB)" % (a.nbytes / 2**20)},
            "pct_fp64_peak": 100.0 * value / (peak * world),
            "sec_per_block": (ms_all * 1e-3) / max(1, len(my_targets)) if scaling == "weak" else
            (ms_all * 1e-3) / len(cfg["targets"]),
            "fp64_peak_tflops": peak,
            "roofline": {"bound": "tensor", "kernel": "gemm_kernel (fused Schur update R - RT*W)",
                         "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                         "traffic": traffic, "per_launch_flops": gemm_flops, "launch_ms": gemm_ms,
                         "peak_source": "bri_fp64_peak DMMA microbenchmark measured in this run "
                                        "(MEASURED_PEAKS.json has no FP64 figure)"},
            "e2e": {"value": e2e_value, "unit": "TFLOP/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "ms_per_step": e2e_ms},
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
        }
        if cpu is not None:
            line["cpu_baseline"] = cpu
            line["speedup_vs_cpu_e2e"] = e2e_value / cpu["value"]
        print(json.dumps(line))
    if dist is not None:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
