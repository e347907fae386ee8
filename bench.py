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
* N > 1 (torchrun): weak scaling by default (N copies of the mesh stacked
  along the last axis, one decompose() block per rank, NCCL halos under the
  interior elements); the line adds the sharded roofline (HBM time vs the
  halo time at the measured NCCL/NVLink bandwidth) and run_scale rows
  (src/experiments.cpp:306-399) against a 1-GPU run of the same mode.
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


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


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
            "seconds": st.wall_seconds, "steps": st.steps, "cpu_model": cpu_model(),
            "logical_cpus": os.cpu_count()}


def run_cpu_serial(cfg_name: str, cells_per_axis: int = 96, steps: int = 2):
    """The reference's serial advance (P = 1, src/solver.cpp:372-440) on a reduced
    mesh of the same configuration (BASELINE.md §2 asks for the serial figure)."""
    dim, cells, order, eq, rk, desc = CONFIGS[cfg_name]
    ol, orc, kind = reference_lib()
    small = tuple(min(c, cells_per_axis) for c in cells)
    p = ol.Problem(dim, small, order, ol.EULER if eq else ol.ADVECTION, rk)
    u0 = orc.initial(p)
    _, st = orc.advance(p, u0, steps, True)
    return {"value": p.size * STAGES[rk] * st.steps / st.wall_seconds, "unit": UNIT, "cores": 1, "kind": kind,
            "sample": f"serial advance, {steps} steps after one warm-up, {'x'.join(map(str, small))} cells "
                      f"({p.size} DOF) of the same equation/order/RK"}


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


L2_NOTE = {
    "c2": "no flush: one RK4 step streams u and the K_j (5 arrays of 77 MB = 385 MB) through the 126 MB L2",
    "c3": "no flush needed: each state array (906 MB) exceeds the 126 MB L2",
    "c4": "no flush needed: each state array (4.3 GB) exceeds the 126 MB L2",
    "c5": "no flush needed: each state array (6.4 GB / N GPUs) exceeds the 126 MB L2",
}


def link_probe(plan, dev, iters: int = 20):
    """NCCL point-to-point over NVLink between this rank and its neighbours
    along the first split axis, through torch.distributed (the same transport
    ndgx's halo exchange uses): the time of one exchange of the real halo
    plane (send up, receive from below) and the per-direction bandwidth of a
    256 MB message.  Every rank calls it (matched collectives)."""
    import torch
    import torch.distributed as dist
    axes = [a for a in range(3) if plan.split[a]]
    a = axes[0]
    up, down = plan.nbr[a][1], plan.nbr[a][0]

    def run(n):
        snd = torch.ones(n, dtype=torch.float64, device=f"cuda:{dev}")
        rcv = torch.empty_like(snd)

        def once():
            for w in dist.batch_isend_irecv([dist.P2POp(dist.isend, snd, up), dist.P2POp(dist.irecv, rcv, down)]):
                w.wait()
        for _ in range(3):
            once()
        torch.cuda.synchronize(dev)
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(iters):
            once()
        e1.record()
        torch.cuda.synchronize(dev)
        return e0.elapsed_time(e1) / iters * 1e-3  # seconds per exchange

    plane = int(plan.plane[a])
    t_plane = run(plane)
    big = 32 * 1024 * 1024  # 256 MB
    t_big = run(big)
    return {"axis": a, "plane_bytes": 8 * plane, "plane_exchange_ms": t_plane * 1e3,
            "link_gbs": 8 * big / t_big / 1e9,
            "how": "torch.distributed NCCL batch_isend_irecv to the split-axis neighbours, CUDA events, "
                   f"mean of {iters}; link_gbs from a 256 MB message (per direction)"}


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
    # copies along the last axis (decompose() then gives slabs, one per rank;
    # run_scale's lowest-interface weak mesh, src/experiments.cpp:353-380)
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
    plan = s.plan
    dof = s.dof  # this rank's block
    dof_total = mesh.dof(model)  # all ranks (weak: world * dof; strong: the configuration's mesh)
    exchanging = any(plan.split[a] for a in range(3))

    # pinned host state (the reference AoS layout), synthetic IC of this block
    host = torch.empty(dof, dtype=torch.float64, pin_memory=True)
    u0 = host.numpy()
    t0 = time.perf_counter()
    if ranked:
        ndgx.init_block(cfg, lo, hi, out=u0)
    elif eq:
        ndgx.init_euler_subsonic(mesh, model, out=u0)
    else:
        ndgx.init_multisine(mesh, model, n_modes=40, seed=42, out=u0)
    t_host_init = time.perf_counter() - t0
    # the same IC generated in HBM (f4: ndgx_init_device), timed for the setup
    # comparison; the uploads below overwrite it with the host field
    ic_amps = None if eq else ndgx.multisine_amplitudes(40, 42)
    s.init_device(ndgx.IC_EULER_SUBSONIC if eq else ndgx.IC_MULTISINE, ic_amps)  # first call: module load
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    s.init_device(ndgx.IC_EULER_SUBSONIC if eq else ndgx.IC_MULTISINE, ic_amps)
    torch.cuda.synchronize(dev)
    t_dev_init = time.perf_counter() - t0
    t0 = time.perf_counter()
    s.upload_ptr(host.data_ptr())
    torch.cuda.synchronize(dev)
    t_upload = time.perf_counter() - t0

    def barrier():
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=f"cuda:{dev}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    s.upload_ptr(host.data_ptr())
    # warm-up: W untimed steps (graph capture, clocks)
    s.launch_steps(max(args.warmup, 3))
    s.sync()
    s.upload_ptr(host.data_ptr())

    # ---- device-resident timed region (CUDA events on the solver stream) ----
    barrier()
    with ClockSampler(dev) as clk:
        s.launch_steps(args.steps)
        st = s.sync()
    barrier()
    t_dev = max_over_ranks(st.wall_seconds)
    value = dof_total * stages * args.steps / t_dev

    # ---- per-stage timing inside the replayed step graph (globaltimer stamps) ----
    # (median over 5 replays: a single replay varies by a few percent between runs)
    profs = [s.profile_step() for _ in range(5)]
    stamp_ms = np.median(np.array([pr[0] for pr in profs]), axis=0)
    ctl_ms = float(np.median([pr[1] for pr in profs]))
    # the stamps add one 1-thread launch per stage: they give each stage's
    # SHARE; the absolute times are those shares of the graph-timed step
    step_ms = t_dev / args.steps * 1e3
    stage_ms = stamp_ms * max(step_ms - ctl_ms, 1e-9) / float(stamp_ms.sum())
    avg_stage_ms = float(stage_ms.mean())
    bytes_per_launch = BYTES_PER_DOF_STAGE[rk] * dof
    peak, peak_src = measured_peaks()
    achieved = bytes_per_launch / (avg_stage_ms * 1e-3) / 1e9
    traffic, traffic_src = None, ""
    prof_path = os.path.join(ROOT, "profiles", "ncu_stage_traffic.json")
    if os.path.exists(prof_path):
        with open(prof_path) as f:
            prof = json.load(f)
        tr = prof.get(args.config, {}).get(args.arith)
        if tr:
            traffic = tr.get("dram_bytes_per_launch")
            traffic_src = tr.get("source", "")

    # ---- sharded roofline (N > 1): HBM time vs halo time over NVLink ----
    sharded = None
    if world > 1 and exchanging:
        lp = link_probe(plan, dev)
        halo_bytes = sum(2 * 8 * int(plan.plane[a]) for a in range(3) if plan.split[a])
        t_hbm = bytes_per_launch / (peak * 1e9)
        t_halo = halo_bytes / (lp["link_gbs"] * 1e9)
        lp_max = {k: max_over_ranks(v) if isinstance(v, float) else v for k, v in lp.items()}
        sharded = {"halo_bytes_per_stage_per_gpu": halo_bytes, "hbm_bytes_per_stage_per_gpu": bytes_per_launch,
                   "t_hbm_ms": t_hbm * 1e3, "t_halo_bw_ms": t_halo * 1e3,
                   "t_halo_exchange_measured_ms": lp_max["plane_exchange_ms"],
                   "link_gbs_measured": lp["link_gbs"], "bound": "hbm" if t_hbm >= t_halo else "nvlink",
                   "stage_roofline_ms": max(t_hbm, t_halo) * 1e3, "probe": lp_max["how"],
                   "note": "the halo exchange runs on the comm stream under the interior elements"}

    # ---- end-to-end through the reference-facing call (host buffers) ----
    barrier()
    t0 = time.perf_counter()
    s.upload_ptr(host.data_ptr())
    st_e = s.advance(ndgx.StepPlan(args.steps, False))
    s.download_ptr(host.data_ptr())
    barrier()
    t_e2e = max_over_ranks(time.perf_counter() - t0)
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
        tx = max_over_ranks(stx.wall_seconds)
        exact = {"value": dof_total * stages * args.steps / tx, "unit": UNIT,
                 "ms_per_step": tx / args.steps * 1e3,
                 "note": "arith=exact: the reference's IEEE operation order, states bit-identical to the CPU reference"}
        sx.close()

    # ---- run_scale rows (N > 1): the 1-GPU baseline of the same mode, on rank 0 ----
    scale_rows = None
    if world > 1 and not args.no_scale_baseline:
        from paper_2510_05254_b200 import report as rp
        base = None
        if rank == 0:
            # weak: one GPU with the per-GPU mesh; strong: one GPU with the whole mesh
            bmesh = ndgx.Mesh(dim, tuple(cells), order)
            bcfg = ndgx.SolverConfig(bmesh, model, rk, 0.4, 1.0)
            hb = ndgx.init_euler_subsonic(bmesh, model) if eq else \
                ndgx.init_multisine(bmesh, model, n_modes=40, seed=42)
            with ndgx.Solver(bcfg, device=dev, arith=arith) as sb:
                sb.upload(hb)
                sb.launch_steps(3)
                sb.sync()
                sb.upload(hb)
                sb.launch_steps(args.steps)
                base = (bcfg, sb.sync())
        barrier()
        if rank == 0:
            devname = torch.cuda.get_device_name(dev)
            mode = "strong" if args.strong else "weak"
            bcfg, bst = base
            r1 = rp.scale_row(bcfg, bst, 1, devname, mode, note=f"ndgx {args.arith}, 1 GPU")
            stats_n = ndgx.StepStats(st.steps, st.dt_min, st.dt_max, t_dev)
            rn = rp.scale_row(cfg, stats_n, world, devname, mode,
                              baseline_wall=bst.wall_seconds if args.strong else 0.0,
                              baseline_tpd=0.0 if args.strong else r1.time_per_dof,
                              note=f"ndgx {args.arith}, {world} GPUs, blocks {list(plan.grid)}")
            scale_rows = [{c: rp._cell(r, c) for c in rp.COLUMNS} for r in (r1, rn)]

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            r = run_cpu_reference(args.config, max_steps=3, warmup=1, budget_s=20.0)
            cpu = {k: r[k] for k in ("value", "unit", "cores", "kind", "sample", "cpu_model", "logical_cpus")}
            cpu["serial_p1"] = run_cpu_serial(args.config)
        except Exception as e:  # noqa: BLE001
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference", "sample": f"failed: {e}"}

    if rank == 0:
        # our kernels in the timed region: the first step's wavespeed scan (Euler),
        # per step the step control and per stage one fused stage kernel (an
        # exchanging block: pack + interior + boundary shell)
        per_stage = 3 if exchanging else 1
        launches = args.steps * (1 + stages * per_stage) + (1 if eq else 0)
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
                                       f"{world} rank(s), decompose() blocks {list(plan.grid)}, NCCL face-halo "
                                       f"exchange per RK stage on a comm stream under the interior elements" +
                                       (" (forced on every axis)" if args.force_exchange else "")),
                       "l2": L2_NOTE[args.config]},
            "roofline": {"bound": sharded["bound"] if sharded else "hbm", "achieved": achieved, "peak": peak,
                         "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                         "traffic_source": "profiles/ncu_stage_traffic.json: ncu dram__bytes_read.sum + "
                                           "dram__bytes_write.sum averaged over the stage launches of one step, "
                                           "measured on the same kernel build, not in this run (" + traffic_src + ")",
                         "kernel": "ndgx::stage_kernel (fused NDG RHS + RK stage)",
                         "bytes_per_dof_stage": BYTES_PER_DOF_STAGE[rk],
                         "avg_launch_ms": avg_stage_ms, "stage_ms": stage_ms.tolist(), "step_control_ms": ctl_ms,
                         "stage_timing": "per-stage shares from globaltimer stamps between the stages of the replayed "
                                         "two-step graph (median of 5 replays), applied to the graph-timed step "
                                         "minus step control; the raw stamps (one extra 1-thread launch per "
                                         "stage) are stage_ms_stamps",
                         "stage_ms_stamps": stamp_ms.tolist(),
                         "peak_source": peak_src,
                         "step_frac": value / world * BYTES_PER_DOF_STAGE[rk] / 1e9 / peak,
                         "sharded": sharded},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": 8 * dof / args.steps,
                    "d2h_bytes_per_step": 8 * dof / args.steps,
                    "note": "one advance(StepPlan{K}) call: pinned host AoS upload, K steps, download"},
            "setup": {"host_init_s": t_host_init, "upload_s": t_upload, "device_init_s": t_dev_init,
                      "note": "initial condition of this rank's block: host init_* + pinned H2D upload "
                              "vs ndgx_init_device (generated in HBM, no host field)"},
            "exact_mode": exact,
            "scale_rows": scale_rows,
            "gpu_launches": launches,
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
    ap.add_argument("--no-scale-baseline", action="store_true",
                    help="N > 1: skip the 1-GPU baseline run behind the run_scale rows")
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
