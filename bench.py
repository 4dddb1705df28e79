"""Benchmark: FP64 TFLOP/s and seconds per inverse block of the BRI hot path on B200.

Default workload = BASELINE.json config 3 (the largest single-GPU config and the reference's
main entry point, invert_full, engine.py:296-364): k=8, b=1024 (m=8192), M = G + m I from PCG64
seed 2, ALL 64 inverse blocks.  A "step" is one complete full inverse: the deduplicated DAG of
the 64 targets (6,499 Schur nodes) plus 64 final inversions.  --config 2 (one
b=4096 node + inversion) and --config 1 (k=4, b=64, 16 blocks) stay available.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C]

value      : algorithmic FP64 TFLOP/s (SURVEY §8(d) convention: 6b^3+b^2 per DAG node + 2b^3 per
             target), M resident in HBM, device-timed (CUDA events).  The device shares a level's
             pivot factorizations and solves between nodes (bri_level_batch), so it EXECUTES fewer
             FLOPs than the convention counts: `executed` reports those and their % of peak.
e2e        : same metric through the public API (invert_full into a MemorySink; invert_block for
             a single target) from pinned HOST memory: H2D of M and D2H of every block timed.
roofline   : the dominant kernel by in-step time share (CUPTI timestamps of one extra, untimed
             step) with its executed FLOPs from the library's ledger (bri_flop_count) divided by
             its in-step kernel time; `isolated` = the same kernel alone on one level-sized
             batch, CUDA-event timed.  peak = FP64 DMMA throughput measured in this run by
             bri_fp64_peak (MEASURED_PEAKS.json has no FP64 entry).
cpu_baseline / --impl reference: the reference's own LAPACK/BLAS calls (oracle port, memoized DAG,
             all host cores).  Configs 1-2 run the whole workload per step; larger configs time a
             bounded sample of the SAME DAG (real leaf nodes of M + real final inversions) and
             report the whole-job time N_exec*t_node + T*t_inv — same metric, same config dict.
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
    ap.add_argument("--config", type=int, default=3)
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


FULL_CPU_CONFIGS = (1, 2)     # the whole workload per CPU step; larger configs are sampled


def config_dict(cfg_id, cfg, nodes):
    """The workload description both arms print (identical dicts)."""
    return {"workload": f"config{cfg_id}", "k": cfg["k"], "b": cfg["b"], "m": cfg["m"],
            "targets": len(cfg["targets"]), "schedule": "dag", "dag_nodes": nodes,
            "l2": ("inputs larger than L2 (M = %.0f MiB > 126 MB)" % (cfg["m"] ** 2 * 8 / 2 ** 20)
                   if cfg["m"] ** 2 * 8 > 126e6 else
                   "M (%.1f MiB) fits in L2 and is NOT flushed between steps" % (cfg["m"] ** 2 * 8 / 2 ** 20))}


def cpu_step(a, cfg, sched, cfg_id, sample_nodes=6, sample_inv=1):
    """One CPU step of the reference's own LAPACK/BLAS calls (oracle port, memoized DAG).

    Returns (estimated whole-job seconds, description, measured seconds).  For configs 1-2 the
    whole workload runs; otherwise `sample_nodes` real leaf nodes of the SAME DAG (operands are
    blocks of M) and `sample_inv` real block inversions are timed and the job time is
    N_exec * t_node + T * t_inv (a node's LAPACK/BLAS cost does not depend on its values)."""
    from oracle import bri_oracle as orc

    k, b = cfg["k"], cfg["b"]
    targets = cfg["targets"]
    if cfg_id in FULL_CPU_CONFIGS:
        t0 = time.perf_counter()
        memo, src = {}, orc.BlockSource(a, k)
        for al, be in targets:
            orc.invert_block(src, k, al, be, memo=memo)
        dt = time.perf_counter() - t0
        return dt, f"all {len(targets)} target(s) of config {cfg_id} (memoized DAG, {len(sched.nodes)} nodes)", dt
    src = orc.BlockSource(a, k)
    leaves = [nd for nd in sched.nodes if nd.n == 2][:sample_nodes]
    t0 = time.perf_counter()
    for nd in leaves:
        orc.fold(*[src.block(r[1], r[2]) for r in nd.operands])
    t1 = time.perf_counter()
    for i in range(sample_inv):
        orc.invert_dense(src.block(1 + i % k, 1 + i % k))
    t2 = time.perf_counter()
    t_node, t_inv = (t1 - t0) / len(leaves), (t2 - t1) / sample_inv
    est = len(sched.nodes) * t_node + len(targets) * t_inv
    desc = (f"{len(leaves)} leaf nodes of config {cfg_id}'s DAG ({t_node * 1e3:.0f} ms/node) + {sample_inv} "
            f"block inversion(s) ({t_inv * 1e3:.0f} ms) per step -> whole job {len(sched.nodes)} nodes + "
            f"{len(targets)} inversions")
    return est, desc, t2 - t0


def blas_threads():
    try:
        from threadpoolctl import threadpool_info

        n = [d.get("num_threads") for d in threadpool_info() if d.get("user_api") == "blas"]
        return max(n) if n else os.cpu_count()
    except Exception:
        return os.cpu_count()


def ncu_traffic(b):
    """DRAM bytes per launch of the level-batch Schur GEMM from the committed ncu --set full summary."""
    path = os.path.join(ROOT, "profiles", "gemm_ncu_summary.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        ent = d.get("by_order", {}).get(str(b))
        return ent if ent else None
    except Exception:
        return None


def short_name(n):
    n = n.replace("(anonymous namespace)::", "").replace("bri::", "").replace("void ", "")
    return n.split("(")[0].split("<")[0].strip()


FAMILY = {"gemm_kernel": "gemm", "gemm_persistent_kernel": "gemm", "skinny_kernel": "gemm",
          "trsm_kernel": "trsm"}


def instep_profile(step, stream):
    """Per-kernel in-step device time (CUPTI timestamps via torch.profiler) of one untimed step,
    plus the library's executed-FLOP ledger delta per kernel family over the same step."""
    import torch

    from paper_1612_00001_b200 import _native

    lib = _native.load_library()
    f0 = [lib.bri_flop_count(q) for q in (0, 1)]
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        step()
        torch.cuda.synchronize()
    f1 = [lib.bri_flop_count(q) for q in (0, 1)]
    per, total = {}, 0.0
    for e in prof.events():
        if e.device_type != torch.autograd.DeviceType.CUDA:
            continue
        dt = e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
        name = short_name(e.name)
        per[name] = per.get(name, 0.0) + dt
        total += dt
    fam = {"gemm": 0.0, "trsm": 0.0}
    for name, us in per.items():
        if name in FAMILY:
            fam[FAMILY[name]] += us
    flops = {"gemm": float(f1[0] - f0[0]), "trsm": float(f1[1] - f0[1])}
    return per, total, fam, flops


# ------------------------------------------------------------------ reference arm
def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from paper_1612_00001_b200 import workloads
    from paper_1612_00001_b200.dag import build_schedule

    cfg = workloads.config(args.config, args.b)
    k, b = cfg["k"], cfg["b"]
    a = workloads.make_matrix(args.config, args.b)
    targets = cfg["targets"]
    sched = build_schedule(k, targets)
    flops = workloads.run_flops(b, len(sched.nodes), len(targets))
    for _ in range(args.warmup):
        cpu_step(a, cfg, sched, args.config)
    est, meas = [], []
    for _ in range(args.steps):
        e, desc, m = cpu_step(a, cfg, sched, args.config)
        est.append(e)
        meas.append(m)
    sec = sum(est) / len(est)
    tf = flops / sec / 1e12
    cores = blas_threads()
    line = {
        "impl": "reference", "metric": METRIC, "value": tf, "unit": "TFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True,
        "scaling": "strong" if len(targets) > 1 else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (PCG64 seeds of BASELINE.json configs)",
        "config": config_dict(args.config, cfg, len(sched.nodes)),
        "sec_per_block": sec / len(targets),
        "cpu_baseline": {"value": tf, "unit": "TFLOP/s", "cores": cores, "kind": "port",
                         "sample": desc + f"; oracle = numpy/scipy LAPACK/BLAS calls of the reference "
                                          f"(core.py:173-263), measured {sum(meas) / len(meas):.2f} s/step"},
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
    full_sched = build_schedule(k, cfg["targets"])
    flops_rank = workloads.run_flops(b, len(sched.nodes), len(my_targets))
    if node_shard:
        flops_rank /= world   # summed over ranks below: the job's algorithmic FLOPs once

    a_dev = torch.from_numpy(a).to(f"cuda:{local}")
    prov = bri.make_memory_provider(a_dev, k)
    stream = torch.cuda.current_stream()
    ws = bri.Workspace(schedule=args.schedule)
    last_info = {}

    def step():
        if node_shard:
            tensors, _ = bri.invert_blocks_sharded(prov, my_targets, ws)
            return tensors
        tensors, info = bri.invert_blocks(prov, my_targets, ws)
        last_info["info"] = info
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
            host = [x.cpu().numpy() for x in res]
        elif len(my_targets) == 1:
            blk = bri.invert_block(p, *my_targets[0], ws)
            host = [blk.data]
            blk.release()
        elif world == 1 and len(my_targets) == k * k:
            sink = bri.MemorySink(p.layout)   # the reference's main entry point (engine.py:296-364)
            bri.invert_full(p, sink, ws)
            host = [sink.finalize()]
        else:
            blocks = [bri.Block(x, ws) for x in bri.invert_blocks(p, my_targets, ws)[0]]
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

    # ---- executed FLOPs (shared factorizations / solves counted once)
    peak = fp64_peak_tflops()
    info = last_info.get("info")
    executed = None
    if info is not None and not node_shard:
        nf = info.factorizations or info.dag_nodes
        ns = info.solves or info.dag_nodes
        ex_flops = (nf * (2.0 / 3.0) * b ** 3 + ns * 2.0 * b ** 3 + info.dag_nodes * (2.0 * b ** 3 + b ** 2)
                    + len(my_targets) * 2.0 * b ** 3)
        ex_tf = ex_flops / (ms * 1e-3) / 1e12
        executed = {"tflops": ex_tf, "pct_fp64_peak": 100.0 * ex_tf / peak, "factorizations": nf, "solves": ns,
                    "schur_gemms": info.dag_nodes, "final_inversions": len(my_targets),
                    "convention": "LU 2/3 b^3 per factorization, 2b^3 per solve (two sweeps), 2b^3+b^2 per "
                                  "node GEMM-subtract, 2b^3 per final inversion"}

    # ---- roofline: dominant kernel by in-step share, its ledger FLOPs over its in-step time
    per, total_us, fam, fam_flops = instep_profile(step, stream)
    dom = max(per.items(), key=lambda kv: kv[1])[0] if per else "?"
    dom_fam = FAMILY.get(dom, None)
    shares = {kn: round(us / total_us, 4) for kn, us in sorted(per.items(), key=lambda kv: -kv[1])[:8]}
    bound, r_unit, r_peak, r_src = "tensor", "TFLOP/s", None, None
    if dom_fam is not None and fam[dom_fam] > 0:
        achieved = fam_flops[dom_fam] / (fam[dom_fam] * 1e-6) / 1e12
    elif dom == "small_node_kernel" and per.get(dom):
        # small b (config 1): SURVEY §8(d) asks for HBM GB/s — algorithmic bytes 40 b^2 per node
        # (4 operand blocks read, 1 written) + 16 b^2 per final inversion, over the kernel's in-step time
        nodes = len(full_sched.nodes) if not node_shard else len(sched.nodes)
        algo = (40.0 * nodes + 16.0 * len(cfg["targets"])) * b * b
        achieved = algo / (per[dom] * 1e-6) / 1e9
        bound, r_unit = "hbm", "GB/s"
        try:
            with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
                r_peak = float(json.load(fh)["hbm_gbs"])
            r_src = "MEASURED_PEAKS.json hbm_gbs (driver-measured copy bandwidth)"
        except Exception:
            r_peak, r_src = 7700.0, "B200 nominal HBM3e (MEASURED_PEAKS.json unreadable)"
    else:
        achieved = None

    # isolated: the Schur GEMM batch of one level (148 items of b x b x b), CUDA-event timed
    from paper_1612_00001_b200.device import Arena

    reps = 3
    cnt = 148 if b <= 2048 else 2
    iso = None
    try:
        with Arena(b, 3 * cnt, device=local) as ar:
            ar.tensor.normal_()
            items = [(3 * i, 3 * i + 1, 3 * i + 2, 3 * i + 2) for i in range(cnt)]
            ar.gemm(items, b, b, b, alpha=-1.0, beta=1.0)
            g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            g0.record(stream)
            for _ in range(reps):
                ar.gemm(items, b, b, b, alpha=-1.0, beta=1.0)
            g1.record(stream)
            torch.cuda.synchronize()
            gemm_ms = g0.elapsed_time(g1) / reps
        gf = (2.0 * b ** 3 + b ** 2) * cnt
        iso = {"kernel": "gemm_kernel", "items": cnt, "per_launch_flops": gf, "launch_ms": gemm_ms,
               "achieved": gf / (gemm_ms * 1e-3) / 1e12, "frac": gf / (gemm_ms * 1e-3) / 1e12 / peak}
    except Exception as exc:  # pragma: no cover - memory-limited boxes
        iso = {"error": str(exc)[:200]}
    traffic = ncu_traffic(b)

    # ---- CPU baseline (rank 0, N = 1 only): the reference's calls on the host cores
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        est, desc, meas = cpu_step(a, cfg, full_sched, args.config, sample_nodes=3)
        cpu = {"value": flops_total / est / 1e12 if len(my_targets) == len(cfg["targets"]) else None,
               "unit": "TFLOP/s", "cores": blas_threads(), "kind": "port", "sec_per_block": est / len(cfg["targets"]),
               "sample": desc + f"; oracle = numpy/scipy LAPACK/BLAS calls of the reference, measured {meas:.2f} s"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_all, "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (PCG64 seeds of BASELINE.json configs)",
            "config": config_dict(args.config, cfg, len(full_sched.nodes)),
            "pct_fp64_peak_convention": 100.0 * value / (peak * world),
            "executed": executed,
            "sec_per_block": (ms_all * 1e-3) / max(1, len(my_targets)) if scaling == "weak" else
            (ms_all * 1e-3) / len(cfg["targets"]),
            "fp64_peak_tflops": peak,
            "roofline": {"bound": bound, "kernel": dom, "family": dom_fam, "achieved": achieved,
                         "peak": r_peak if bound == "hbm" else peak, "unit": r_unit,
                         "frac": (achieved / (r_peak if bound == "hbm" else peak)) if achieved else None,
                         "step_share": round(per.get(dom, 0.0) / total_us, 4) if total_us else None,
                         "family_share": round(fam.get(dom_fam, 0.0) / total_us, 4) if dom_fam else None,
                         "traffic": traffic.get("dram_bytes_per_launch") if traffic else None,
                         "traffic_algorithmic_bytes": traffic.get("algorithmic_bytes_per_launch") if traffic else None,
                         "kernel_shares": shares,
                         "method": "one extra untimed step under CUPTI (torch.profiler): family kernel time; "
                                   "executed FLOPs from bri_flop_count over the same step",
                         "isolated": iso,
                         "peak_source": r_src if bound == "hbm" else
                                        ("bri_fp64_peak DMMA microbenchmark measured in this run "
                                         "(MEASURED_PEAKS.json has no FP64 figure)")},
            "e2e": {"value": e2e_value, "unit": "TFLOP/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "ms_per_step": e2e_ms},
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
        }
        if cpu is not None:
            line["cpu_baseline"] = cpu
            if cpu["value"]:
                line["speedup_vs_cpu_e2e"] = e2e_value / cpu["value"]
        if node_shard:
            line["config"]["shard"] = args.shard
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
