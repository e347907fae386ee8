#!/usr/bin/env python
"""Benchmark: DOF*stage updates/s of the NDG RHS + RK step on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c3|c2|c4|c5] [--arith exact|fast]

Default workload (BASELINE.json metric, configs[2] = C3): 2D isothermal Euler,
order-8 NDG, RK4, 768^2 cells (6144^2 nodes, 1.13e8 DOF), init_euler_subsonic
initial condition (synthetic), cfl 0.4, periodic unit box.

* value: device-resident throughput -- K fixed CFL steps (alpha scan, dt,
  4 fused stage kernels per step), CUDA events on the solver's stream, after
  W warm-up steps; max over ranks.  Every state array (906 MB) is larger
  than L2 (126 MB), so no explicit flush is needed.
* e2e: the same metric through the reference-facing call with host buffers:
  upload (pinned host AoS -> device) + advance(K steps) + download, wall clock.
* roofline: the fused stage kernel vs measured HBM bandwidth
  (MEASURED_PEAKS.json), algorithmic bytes per DOF*stage from SURVEY.md §8d.
* cpu_baseline: the reference itself (oracle/_ref, run_partitioned over the
  host's cores) on a bounded sample of the same workload.
* --impl reference: the reference CPU arm alone (same metric/config).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (dim, cells, order, equation, rk, description)
    "c2": (2, (388, 388), 8, 0, 1, "C2: 2D linear advection, order 8, RK4, 388^2 cells (3104^2 nodes)"),
    "c3": (2, (768, 768), 8, 1, 1, "C3: 2D isothermal Euler, order 8, RK4, 768^2 cells (6144^2 nodes)"),
    "c4": (3, (128, 128, 128), 4, 1, 2, "C4: 3D isothermal Euler, order 4, RK6, 128^3 cells per GPU"),
    "c5": (2, (2048, 2048), 8, 1, 1, "C5: 2D isothermal Euler, order 8, RK4, 2048^2 cells (16384^2 nodes)"),
}
STAGES = {0: 3, 1: 4, 2: 7}
RK_NAME = {0: "rk3", 1: "rk4", 2: "rk6"}
# algorithmic HBM bytes per DOF*stage of the minimum K-storage schedule
BYTES_PER_DOF_STAGE = {0: 24.0, 1: 26.0, 2: 40.0}
METRIC = "DOF·stage updates/s (2D isothermal Euler, order 8, RK4) at 1/2/4/8 B200"
UNIT = "DOF*stage/s"


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """Samples SM clock and throttle reasons via NVML during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, device: int, period_s: float = 0.02):
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._period = period_s
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:  # pragma: no cover
            self._nv = None
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self._nv.nvmlDeviceGetClockInfo(self._h, self._nv.NVML_CLOCK_SM))
                r = self._nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self._period)

    def __enter__(self):
        if self._nv:
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._nv:
            self._t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "samples": len(self.samples),
                "reasons": sorted(self.reasons)}


def reference_lib():
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_lib  # the checker / CPU baseline only
    kind = "reference" if os.path.exists(oracle_lib.REF_SO) else "port"
    return oracle_lib, oracle_lib.Oracle(kind), kind


def physical_cores() -> int:
    try:
        import psutil
        n = psutil.cpu_count(logical=False)
        if n:
            return int(n)
    except Exception:
        pass
    return os.cpu_count() or 1


def run_cpu_reference(cfg_name: str, max_steps: int, warmup: int, budget_s: float = 30.0):
    """The reference's thread-parallel path (run_partitioned, partition.cpp:186-333)
    over the host's physical cores on the benchmark workload.  Steps are capped so
    the sample stays within `budget_s` of CPU time."""
    dim, cells, order, eq, rk, desc = CONFIGS[cfg_name]
    ol, orc, kind = reference_lib()
    p = ol.Problem(dim, cells, order, ol.EULER if eq else ol.ADVECTION, rk)
    u0 = orc.initial(p)
    cores = physical_cores()
    workers = cores
    if kind == "reference":
        # largest feasible worker count <= cores
        while workers > 1:
            try:
                orc.decompose(p, workers)
                break
            except ol.CheckerError:
                workers -= 1
        probe, st = orc.run_partitioned(p, u0, workers, 1, False)
        per_step = st.wall_seconds
        steps = int(max(1, min(max_steps, budget_s // max(per_step, 1e-9))))
        if warmup:
            steps_w = max(0, min(warmup, 1))
        else:
            steps_w = 0
        _, st = orc.run_partitioned(p, u0, workers, steps, bool(steps_w))
    else:
        workers = 1
        _, st = orc.advance(p, u0, 1, False)
        steps = 1
    dof = p.size
    value = dof * STAGES[rk] * st.steps / st.wall_seconds
    sample = (f"{desc}; {st.steps} timed step(s) of the full workload after "
              f"{'one untimed warm-up step' if kind == 'reference' else 'none'}; "
              f"{'run_partitioned' if workers > 1 else 'advance'} with {workers} worker thread(s)")
    return {"value": value, "unit": UNIT, "cores": workers, "kind": kind, "sample": sample,
            "seconds": st.wall_seconds, "steps": st.steps}


def bench_reference_arm(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    r = run_cpu_reference(args.config, max_steps=min(args.steps, 10), warmup=args.warmup)
    dim, cells, order, eq, rk, desc = CONFIGS[args.config]
    line = {
        "metric": METRIC, "value": r["value"], "unit": UNIT, "n_gpus": args.gpus, "steps": r["steps"],
        "warmup": min(args.warmup, 1), "ms_per_step": r["seconds"] / r["steps"] * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (init_euler_subsonic / init_multisine, the reference's own ICs)",
        "impl": "reference",
        "config": {"workload": desc, "cells": list(cells), "order": order, "rk": RK_NAME[rk],
                   "dof": int(np.prod(cells)) * order ** dim * ((dim + 1) if eq else 1),
                   "parallelism": f"run_partitioned x{r['cores']} host threads"},
        "cpu_baseline": {k: r[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "e2e": {"value": r["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def bench_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2510_05254_b200 as ndgx

    rank, world, local = dist_env()
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = local
    dim, cells, order, eq, rk, desc = CONFIGS[args.config]
    arith = ndgx.ARITH_FAST if args.arith == "fast" else ndgx.ARITH_EXACT
    # weak scaling: every GPU owns the configuration's mesh; N GPUs stack N
    # copies along the last axis (decompose() then gives slabs, one per rank)
    gcells = list(cells)
    if not args.strong:
        gcells[dim - 1] *= world
    mesh = ndgx.Mesh(dim, tuple(gcells), order)
    model = ndgx.EquationModel.isothermal_euler(dim, 1.0) if eq else ndgx.EquationModel.advection(dim, (1, 0, 0))
    cfg = ndgx.SolverConfig(mesh, model, rk, 0.4, 1.0)
    stages = STAGES[rk]

    ranked = world > 1 or args.force_exchange
    if ranked:
        # NCCL bootstrap over torch.distributed, then one ndgx rank per GPU
        # (--force-exchange: the same path at world size 1, every axis through NCCL)
        obj = [ndgx.nccl_unique_id() if rank == 0 else None]
        if world > 1:
            dist.broadcast_object_list(obj, src=0)
        s = ndgx.Solver.for_rank(cfg, world, rank, obj[0], device=dev, arith=arith,
                                 force_exchange=args.force_exchange)
        lo, hi = tuple(s.plan.lo), tuple(s.plan.hi)
    else:
        s = ndgx.Solver(cfg, device=dev, arith=arith)
        lo, hi = (0, 0, 0), tuple(mesh.cells)
    dof = s.dof  # this rank's block
    dof_total = mesh.dof(model)  # all ranks (weak: world * dof; strong: the configuration's mesh)

    # pinned host state (the reference AoS layout), synthetic IC of this block
    host = torch.empty(dof, dtype=torch.float64, pin_memory=True)
    u0 = host.numpy()
    if ranked:
        ndgx.init_block(cfg, lo, hi, out=u0)
    elif eq:
        ndgx.init_euler_subsonic(mesh, model, out=u0)
    else:
        ndgx.init_multisine(mesh, model, n_modes=40, seed=42, out=u0)

    def barrier():
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()

    s.upload_ptr(host.data_ptr())
    # warm-up: W untimed steps (graph capture, clocks)
    s.launch_steps(max(args.warmup, 3) if args.warmup >= 3 else 3)
    s.sync()
    s.upload_ptr(host.data_ptr())

    # ---- device-resident timed region (CUDA events on the solver stream) ----
    barrier()
    with ClockSampler(dev) as clk:
        s.launch_steps(args.steps)
        st = s.sync()
    barrier()
    t_dev = st.wall_seconds
    if world > 1:
        t = torch.tensor([t_dev], dtype=torch.float64, device=f"cuda:{dev}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_dev = float(t.item())
    value = dof_total * stages * args.steps / t_dev

    # ---- kernel-level timing for the roofline (events around each stage) ----
    stage_ms = []
    ctl_ms = []
    for _ in range(5):
        ms, c = s.profile_step()
        stage_ms.append(ms)
        ctl_ms.append(c)
    stage_ms = np.array(stage_ms[1:]).mean(axis=0)  # drop the first
    avg_stage_ms = float(stage_ms.mean())
    bytes_per_launch = BYTES_PER_DOF_STAGE[rk] * dof
    peak, peak_src = measured_peaks()
    achieved = bytes_per_launch / (avg_stage_ms * 1e-3) / 1e9
    traffic = None
    prof_path = os.path.join(ROOT, "profiles", "ncu_stage_traffic.json")
    if os.path.exists(prof_path):
        with open(prof_path) as f:
            tr = json.load(f).get(args.config, {}).get(args.arith)
        if tr:
            traffic = tr.get("dram_bytes_per_launch")

    # ---- end-to-end through the reference-facing call (host buffers) ----
    barrier()
    t0 = time.perf_counter()
    s.upload_ptr(host.data_ptr())
    st_e = s.advance(ndgx.StepPlan(args.steps, False))
    s.download_ptr(host.data_ptr())
    barrier()
    t_e2e = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([t_e2e], dtype=torch.float64, device=f"cuda:{dev}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_e2e = float(t.item())
    e2e = dof_total * stages * st_e.steps / t_e2e
    s.close()

    # ---- the bit-identical (reference operation order) mode, same workload ----
    exact = None
    if args.arith == "fast" and not args.no_exact_arm:
        if ranked:
            obj = [ndgx.nccl_unique_id() if rank == 0 else None]
            if world > 1:
                dist.broadcast_object_list(obj, src=0)
            sx = ndgx.Solver.for_rank(cfg, world, rank, obj[0], device=dev, arith=ndgx.ARITH_EXACT,
                                      force_exchange=args.force_exchange)
        else:
            sx = ndgx.Solver(cfg, device=dev, arith=ndgx.ARITH_EXACT)
        sx.upload_ptr(host.data_ptr())
        sx.launch_steps(3)
        sx.sync()
        sx.upload_ptr(host.data_ptr())
        barrier()
        sx.launch_steps(args.steps)
        stx = sx.sync()
        barrier()
        tx = stx.wall_seconds
        if world > 1:
            t = torch.tensor([tx], dtype=torch.float64, device=f"cuda:{dev}")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            tx = float(t.item())
        exact = {"value": dof_total * stages * args.steps / tx, "unit": UNIT,
                 "ms_per_step": tx / args.steps * 1e3,
                 "note": "arith=exact: the reference's IEEE operation order, states bit-identical to the CPU reference"}
        sx.close()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            r = run_cpu_reference(args.config, max_steps=3, warmup=1, budget_s=20.0)
            cpu = {k: r[k] for k in ("value", "unit", "cores", "kind", "sample")}
        except Exception as e:  # noqa: BLE001
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference", "sample": f"failed: {e}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_dev / args.steps * 1e3, "higher_is_better": True,
            "scaling": "strong" if args.strong else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (init_euler_subsonic IC of the reference, generated on the host)",
            "config": {"workload": desc, "cells": list(cells), "global_cells": gcells, "order": order,
                       "rk": RK_NAME[rk], "dof": dof, "dof_total": dof_total, "arith": args.arith,
                       "arith_note": ("fast = FP64 with FMA contraction and FP64 tensor-core (DMMA) volume "
                                      "quadrature, <= 1e-12 relative L2 vs the reference (tests/test_gpu_parity.py); "
                                      "exact = bit-identical") ,
                       "parallelism": ("1 GPU" if not ranked else
                                       f"{world} rank(s), decompose() blocks {list(s.plan.grid)}, NCCL face-halo "
                                       f"exchange per RK stage" + (" (forced on every axis)" if args.force_exchange
                                                                   else "")),
                       "l2": "no flush needed: each state array (8*dof bytes) exceeds the 126 MB L2"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": "ndgx::stage_kernel (fused NDG RHS + RK stage)",
                         "bytes_per_dof_stage": BYTES_PER_DOF_STAGE[rk],
                         "avg_launch_ms": avg_stage_ms, "stage_ms": stage_ms.tolist(),
                         "peak_source": peak_src,
                         "step_frac": value / world * BYTES_PER_DOF_STAGE[rk] / 1e9 / peak},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": 8 * dof / args.steps,
                    "d2h_bytes_per_step": 8 * dof / args.steps,
                    "note": "one advance(StepPlan{K}) call: pinned host AoS upload, K steps, download"},
            "exact_mode": exact,
            "gpu_launches": args.steps * (1 + stages) + (1 if eq else 0),
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
        if args.csv:
            write_csv_row(args, cfg, st, t_dev, world, torch.cuda.get_device_name(dev))
    if world > 1:
        dist.destroy_process_group()


def write_csv_row(args, cfg, st, wall, world, device):
    """--csv: the device-timed run as one row of the reference's report
    (report_to_csv, src/report.cpp:180-198; row = base_row + fill_stats,
    src/experiments.cpp:50-75), wall_seconds = max over ranks."""
    import paper_2510_05254_b200 as ndgx
    from paper_2510_05254_b200 import report as rp
    stats = ndgx.StepStats(st.steps, st.dt_min, st.dt_max, wall)
    row = rp.timing_row(cfg, stats, world, f"{device} (ndgx {args.arith})", experiment="timing",
                        note=f"bench.py --config {args.config}")
    meta = rp.ReportMeta("ndgx-" + ndgx.version().split()[1], "", time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()))
    with open(args.csv, "w") as f:
        f.write(rp.report_to_csv(rp.BenchReport(meta, [row])))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--arith", default="fast", choices=["exact", "fast"])
    ap.add_argument("--no-exact-arm", action="store_true", help="skip the bit-exact side measurement")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--strong", action="store_true",
                    help="strong scaling: the configuration's mesh is split across the N GPUs (C5) "
                         "instead of stacking N copies (weak scaling, the default)")
    ap.add_argument("--force-exchange", action="store_true",
                    help="run the multi-GPU rank path even at one rank (every axis through NCCL)")
    ap.add_argument("--csv", default=None, help="also write the run as a reference-schema report CSV")
    args = ap.parse_args()
    if args.impl == "reference":
        bench_reference_arm(args)
    else:
        bench_ours(args)


if __name__ == "__main__":
    main()
