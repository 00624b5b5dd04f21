"""Benchmark of the B200 HEVI 1D-IMEX ARK2 step (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg5]
    python bench.py --impl reference ...     # the reference CPU path (oracle port)

One "step" is one ARK2 HEVI time step (3 explicit evaluations, 2 Schur
column solves) of the whole grid.  ``value`` = unique DOF-updates/s with the
state resident in HBM (5 fields x unique lattice points / step time, whole
job, max over ranks); ``e2e`` = the same metric through the reference-facing
call ``imexcore.ark_imex_step`` on host (pinned) E-vector buffers, H2D + D2H
inside the timed region.  Default workload: SURVEY 8(d) config 5 (the
largest single-GPU configuration), C = 15.  For N > 1 (torchrun) the same
grid is split into px x py column blocks with NCCL halo exchange (strong
scaling).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "DOF-updates/s (fp64) per 1D-IMEX step at C=15, 1/2/4/8 B200; % HBM roofline"
UNIT = "DOF-updates/s"

# SURVEY 8(d) configurations (3D box, 40:1 elements, neutral 300 K background)
CONFIGS = {
    "cfg5": dict(nx=176, ny=176, nz=10, N=4, Lx=704_000.0, Ly=704_000.0, Lz=1000.0,
                 centre=(352_000.0, 352_000.0, 350.0), radii=(10_000.0, 10_000.0, 250.0),
                 courant=15.0,
                 desc="cfg5: 3D rising thermal bubble, 176x176x10 elements N=4 "
                      "(704x704x1 km, 4 km x 100 m elements), HEVI ARK2 Schur direct, C=15"),
    # config 2 at C_V = 150 keeps C_H = 0.375 with 10x wider elements
    "cfg5w": dict(nx=176, ny=176, nz=10, N=4, Lx=7_040_000.0, Ly=7_040_000.0, Lz=1000.0,
                  centre=(3_520_000.0, 3_520_000.0, 350.0), radii=(100_000.0, 100_000.0, 250.0),
                  courant=150.0,
                  desc="cfg5w: config-5 grid with 40 km x 100 m elements (7040x7040x1 km), "
                       "C_V=150 (C_H=0.375)"),
    "cfg1": dict(nx=10, ny=10, nz=10, N=4, Lx=40_000.0, Ly=40_000.0, Lz=1000.0,
                 centre=(20_000.0, 20_000.0, 350.0), radii=(250.0, 250.0, 250.0),
                 courant=15.0,
                 desc="cfg1: 3D rising thermal bubble, 10x10x10 elements N=4 (40x40x1 km), C=15"),
}

# algorithmic HBM bytes per unique point, per launch: each field
# read / written once; 8 B per fp64 value.  P' of each stage input is one
# plane (stage 0: k_pp_plane; stages 1, 2: written by the column solves) that
# the explicit kernels read instead of forming it for every staged
# (halo-overlapped) point.
KERNEL_BYTES_PER_POINT = {
    # stage 0 = k_pp_plane (reads rho', theta', writes P'(Q)) + the explicit kernel
    "explicit_stage0": 8 * (2 + 1) + 8 * (5 + 1 + 15),
    "solve_stage0": 8 * (3 + 3 + 1),
    "explicit_stage1": 8 * (15 + 1 + 10),
    "solve_stage1": 8 * (3 + 3 + 1),
    "explicit_stage2": 8 * (10 + 1 + 5),
}
STEP_BYTES_PER_POINT = sum(KERNEL_BYTES_PER_POINT.values())   # 640 B
SURVEY_BYTES_PER_POINT = 640                                   # SURVEY 8(d) 16 state passes


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.sw_power_cap,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown")

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        time.sleep(0.15)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.1)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["sw_power_cap", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        sm.sort()
        med = sm[len(sm) // 2] if sm else None
        return {"sm_mhz": med, "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def count_launches(fn):
    """Kernel launches of one call of ``fn`` seen by the CUDA activity
    profiler (untimed): (ours, total) where ``ours`` are the library's
    kernels (k_* / k3_*), or None when the profiler is unavailable."""
    import re
    import torch
    try:
        from torch.profiler import profile, ProfilerActivity
        from torch.autograd import DeviceType
        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            fn()
            torch.cuda.synchronize()
        names = [e.name for e in prof.events() if e.device_type == DeviceType.CUDA
                 and not e.name.startswith(("Memcpy", "Memset"))]
    except Exception:
        return None
    ours = [n for n in names if re.search(r"(^|::|\s)k3?_\w+", n)]
    return len(ours), len(names)


def ncu_traffic():
    """Per-launch DRAM bytes of the dominant kernel from the committed ncu
    summary (profiles/), or None."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as f:
            return json.load(f)
    except Exception:
        return None


# ---------------------------------------------------------------------------
# reference arm / CPU baseline: the oracle port of the reference algorithm
# ---------------------------------------------------------------------------

def reference_sample(steps, warmup, budget_s=150.0, cfg_name="cfg5"):
    """Time the CPU port on a bounded sample of the workload: an n x n x nz
    sub-box with the same elements (4 km x 4 km x 100 m, N=4) and bubble
    shape, n sized so (steps + warmup) steps fit the time budget."""
    import numpy as np
    from oracle.hevi_oracle import BoxOracle
    cfg = CONFIGS[cfg_name]
    ex = cfg["Lx"] / cfg["nx"]
    ez = cfg["Lz"] / cfg["nz"]
    n = int(20 * math.sqrt(budget_s / (1.7 * max(1, steps + warmup))))
    n = max(4, min(20, n, cfg["nx"]))
    o = BoxOracle(n, n, cfg["nz"], n * ex, n * ex, cfg["nz"] * ez, cfg["N"])
    q = o.bubble(0.5, (0.5 * n * ex, 0.5 * n * ex, cfg["centre"][2]), cfg["radii"])
    dt = o.dt_for_courant(q, cfg["courant"])
    for _ in range(max(1, warmup)):
        q = o.step(q, dt)          # first step also probes + factors the columns
    times = []
    for _ in range(max(1, steps)):
        t0 = time.perf_counter()
        q = o.step(q, dt)
        times.append(time.perf_counter() - t0)
    med = float(np.median(times))
    n_unique = o.X * o.Y * o.Z
    return {"value": 5 * n_unique / med, "ms_per_step": 1e3 * med, "n": n,
            "sample": f"{n}x{n}x{cfg['nz']} elements N={cfg['N']} sub-box of {cfg_name} "
                      f"({n_unique} unique points), median of {len(times)} oracle steps "
                      f"after {max(1, warmup)} warm-up (factor) step(s)",
            "storage_dof_per_s": 5 * o.nel * (o.N + 1) ** 3 / med}


def cpu_threads():
    return os.cpu_count() or 1


def cpu_model():
    """lscpu model name of the host."""
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    os.environ.setdefault("OPENBLAS_NUM_THREADS", str(cpu_threads()))
    os.environ.setdefault("OMP_NUM_THREADS", str(cpu_threads()))
    r = reference_sample(args.steps, args.warmup, cfg_name=args.config)
    # the same sample with one BLAS/OpenMP thread
    try:
        from threadpoolctl import threadpool_limits
        with threadpool_limits(limits=1):
            r1 = reference_sample(args.steps, args.warmup, cfg_name=args.config)
    except Exception:
        r1 = None
    threads_all = r
    if r1 is not None and r1["value"] > r["value"]:
        r = r1          # the reference's best CPU configuration is the baseline
    cfg = CONFIGS[args.config]
    out = {"impl": "reference", "metric": METRIC, "value": r["value"], "unit": UNIT,
           "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": r["ms_per_step"], "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": cfg["desc"], "sample": r["sample"],
                      "parallelism": "single host process (numpy)"},
           "cpu_baseline": {"value": r["value"], "unit": UNIT, "cores": 1,
                            "kind": "port", "sample": r["sample"], "cpu_model": cpu_model(),
                            "host_threads_allowed": cpu_threads(),
                            "value_threads_all": threads_all["value"],
                            "value_threads_1": r1["value"] if r1 else None,
                            "value_is": "the faster of the two thread settings",
                            "note": "oracle/hevi_oracle.py (numpy restatement of dycore): a "
                                    "single-threaded numpy program; OpenBLAS may use every host "
                                    "thread but the 5x5 dgemms do not thread (SURVEY 6), so the "
                                    "work runs on one core"},
           "e2e": {"value": r["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------

def run_gpu(args):
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_1702_04316_b200 import specgrid, euler, imexcore, cases
    from paper_1702_04316_b200.plan import tableau_array

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = CONFIGS[args.config]
    mesh = specgrid.build_box_mesh_3d(cfg["nx"], cfg["ny"], cfg["nz"], cfg["Lx"], cfg["Ly"],
                                      cfg["Lz"], cfg["N"])
    ref = euler.hydrostatic_reference(mesh, 300.0)
    disc = euler.build_discretization(mesh)
    sn = args.set
    q0 = cases.bubble_lattice(mesh, ref, 0.5, cfg["centre"], cfg["radii"], set_name=sn)
    courant = args.courant if args.courant else cfg["courant"]
    dt = cases.dt_for_courant(mesh, ref, q0, courant, sn)
    tab = imexcore.ark2_tableau()
    lam = tab.diag * dt
    n_unique = mesh.n_unique
    dof = 5 * n_unique

    if world == 1:
        plan = disc.plan_for(ref, sn)
        torch.cuda.synchronize()
        tf = time.perf_counter()
        plan.factor(lam)      # columnsolve.get_factors: probe + banded LU (once per lam)
        torch.cuda.synchronize()
        factor_ms = 1e3 * (time.perf_counter() - tf)
        Q = plan.zeros()
        Q[..., :mesh.X].copy_(q0)
        work = plan.workspace()
        plan.pp_refresh(Q, work)
        exch = None
        px, py = 1, 1
    else:
        from paper_1702_04316_b200.distributed import DistributedStepper, grid_for
        px, py = grid_for(world)
        torch.cuda.synchronize()
        tf = time.perf_counter()
        ds = DistributedStepper(mesh, ref, disc, dt, px, py, rank, set_name=sn)   # factors in __init__
        torch.cuda.synchronize()
        factor_ms = 1e3 * (time.perf_counter() - tf)
        ds.load_global(q0)
        plan, Q, work = ds.plan, ds.Q, ds.work

        def exch(s):
            """halo refresh of everything stage s reads (state [+ P' plane])"""
            for t in ds.stage_inputs(s):
                ds.exchange(t)
    del q0
    tarr = tableau_array(tab)
    stream = torch.cuda.current_stream()
    names = list(KERNEL_BYTES_PER_POINT)

    chain = plan.chains_pp
    # algorithmic bytes: with the chained P' plane stage 0 reads it from the
    # previous stage 2 (which writes it) instead of a separate k_pp_plane pass
    kb = dict(KERNEL_BYTES_PER_POINT)
    if args.set == "set2c":
        # flux form: no P' planes (the explicit kernels form EOS per point)
        kb = {"explicit_stage0": 8 * (5 + 15), "solve_stage0": 8 * (3 + 3),
              "explicit_stage1": 8 * (15 + 10), "solve_stage1": 8 * (3 + 3),
              "explicit_stage2": 8 * (10 + 5)}
    elif chain:
        kb["explicit_stage0"] = 8 * (5 + 1 + 15)
        kb["explicit_stage2"] = 8 * (10 + 1 + 5 + 1)
    step_bytes = sum(kb.values())
    rk = args.integrator == "rk35"
    if rk and world > 1:
        raise SystemExit("--integrator rk35 runs on one GPU")

    # N > 1: the halo exchange of each stage runs on a side stream while the
    # interior tiles (no neighbour-provided halo point) run; the boundary tiles
    # wait for it (HEVI_STAGE_INTERIOR / _BOUNDARY)
    side = torch.cuda.Stream() if (exch is not None and not args.no_overlap) else None

    def explicit(s, e0, e1):
        pp = chain if s == 0 else False   # P'(Q) chained from the previous step's stage 2
        if side is None:
            if exch is not None:
                exch(s)
            if e0 is not None:
                e0.record(stream)
            plan.stage(s, dt, tarr, Q, work, pp_valid=pp)
        else:
            ready = torch.cuda.Event()
            ready.record(stream)
            with torch.cuda.stream(side):
                side.wait_event(ready)
                exch(s)
                done = torch.cuda.Event()
                done.record(side)
            if e0 is not None:
                e0.record(stream)
            plan.stage(s, dt, tarr, Q, work, pp_valid=pp, part="interior")
            stream.wait_event(done)
            plan.stage(s, dt, tarr, Q, work, pp_valid=pp, part="boundary")
        if e1 is not None:
            e1.record(stream)

    def one_step(ev=None):
        if rk:
            plan.rk35(dt, Q, work)
            return
        E = ev if ev is not None else [None] * 8
        explicit(0, E[0], E[1])
        plan.stage_solve(0, lam, work)
        if ev is not None:
            ev[2].record(stream)
        explicit(1, E[6], E[3])
        plan.stage_solve(1, lam, work)
        if ev is not None:
            ev[4].record(stream)
        explicit(2, E[7], E[5])

    for _ in range(max(3, args.warmup)):
        one_step()
    plan.check_flags()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()

    sampler = ClockSampler(local) if rank == 0 else None
    if sampler:
        sampler.start()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    halo0 = ds.exchange.launches if world > 1 else 0
    # the timed steps: nothing recorded between the launches
    t_start.record(stream)
    for k in range(args.steps):
        one_step()
    t_end.record(stream)
    torch.cuda.synchronize()
    halo_launches = (ds.exchange.launches - halo0) if world > 1 else 0
    if world > 1:
        dist.barrier()
    clocks = sampler.stop() if sampler else None
    elapsed = t_start.elapsed_time(t_end)    # ms
    # per-launch times: the same steps again with CUDA events around every
    # launch on the launching stream (their shares scale the timed total)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(8)] for _ in range(args.steps)]
    i_start = torch.cuda.Event(enable_timing=True)
    i_end = torch.cuda.Event(enable_timing=True)
    i_start.record(stream)
    for k in range(args.steps):
        one_step(evs[k])
    i_end.record(stream)
    torch.cuda.synchronize()
    instr_elapsed = i_start.elapsed_time(i_end)
    ktimes = {n: 0.0 for n in names}
    for ev in ([] if rk else evs):
        ktimes["explicit_stage0"] += ev[0].elapsed_time(ev[1])
        ktimes["solve_stage0"] += ev[1].elapsed_time(ev[2])
        ktimes["explicit_stage1"] += ev[6].elapsed_time(ev[3])
        ktimes["solve_stage1"] += ev[3].elapsed_time(ev[4])
        ktimes["explicit_stage2"] += ev[7].elapsed_time(ev[5])
    plan.check_flags()
    if world > 1:
        t = torch.tensor([elapsed], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed = float(t.item())
        kt = torch.tensor([ktimes[n] for n in names], device="cuda", dtype=torch.float64)
        dist.all_reduce(kt, op=dist.ReduceOp.MAX)
        ktimes = {n: float(v) for n, v in zip(names, kt.tolist())}
    ms_step = elapsed / args.steps
    value = dof / (ms_step * 1e-3)

    # roofline of the dominant kernel (per rank: points this rank owns)
    pts_rank = n_unique / world
    peak, peak_src = peaks()
    kern = {}
    for n in names:
        avg = ktimes[n] / args.steps
        if avg <= 0.0:
            continue
        gbs = kb[n] * pts_rank / (avg * 1e-3) / 1e9
        kern[n] = {"ms": round(avg, 4), "alg_bytes_per_point": kb[n],
                   "alg_GBps": round(gbs, 1), "share": round(ktimes[n] / instr_elapsed, 4)}
    if rk:   # whole RK35 step: 5 fused R + Shu-Osher launches (13 reads + 5 writes per point)
        kern = {"rk35_step": {"ms": round(ms_step, 4), "alg_bytes_per_point": 8 * 5 * 18,
                              "alg_GBps": round(8 * 5 * 18 * pts_rank / (ms_step * 1e-3) / 1e9, 1),
                              "share": 1.0}}
        kb["rk35_step"] = 8 * 5 * 18
        ktimes = {"rk35_step": elapsed}
        names = ["rk35_step"]
    # launches per step: counted by the CUDA activity profiler on one extra
    # (untimed) step; the static schedule count if the profiler is unavailable
    counted = count_launches(one_step)
    plan.check_flags()
    if counted is not None:
        launches_per_step = counted[0]
        halo_launches = 0     # the halo kernels run inside one_step and are counted
    elif rk:
        launches_per_step = 5
    else:
        launches_per_step = 8 if chain or args.set != "set2nc" else 9
    dom = max(names, key=lambda n: ktimes[n])
    traffic = None
    summ = ncu_traffic()
    skey = args.config if args.set == "set2nc" else args.config + ":" + args.set
    if summ and skey in summ and dom in summ[skey]:
        traffic = summ[skey][dom].get("dram_bytes_per_launch")
    achieved = kern[dom]["alg_GBps"]
    roof = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": round(achieved / peak, 4), "traffic": traffic,
            "alg_bytes_per_launch": kb[dom] * pts_rank,
            "peak_source": peak_src}
    step_gbs = step_bytes * pts_rank / (ms_step * 1e-3) / 1e9
    step_roof = {"alg_bytes_per_point": step_bytes, "achieved_GBps": round(step_gbs, 1),
                 "frac": round(step_gbs / peak, 4),
                 "survey_640B_frac": round(SURVEY_BYTES_PER_POINT * pts_rank / (ms_step * 1e-3)
                                           / 1e9 / peak, 4)}

    # e2e through the reference-facing call with host buffers (rank 0 drives
    # the single-GPU drop-in; N > 1 ranks do window H2D / owned D2H)
    e2e = None
    if not args.no_e2e and not rk:
        e2e = run_e2e(args, mesh, ref, disc, dt, tab, plan, Q, work, exch, world, rank, dof)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and not rk:
        r = reference_sample(args.cpu_steps, 1, budget_s=args.cpu_budget, cfg_name=args.config)
        cpu = {"value": r["value"], "unit": UNIT, "cores": 1, "kind": "port",
               "sample": r["sample"], "ms_per_step": r["ms_per_step"], "cpu_model": cpu_model(),
               "note": "single-threaded numpy oracle port of dycore (the reference path)"}

    if rank == 0:
        out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
               "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
               "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
               "dtype": "f64", "data": "synthetic",
               "config": {"workload": cfg["desc"], "unique_points": n_unique,
                          "unique_dof": dof, "storage_dof": 5 * mesh.n_nodes,
                          "columns": mesh.n_col, "levels": mesh.n_lev, "dt_s": dt,
                          "parallelism": f"columns {px}x{py}" + (
                              ", halo exchange on a side stream beside the interior tiles"
                              if side is not None else ""),
                          "integrator": args.integrator, "courant_v": courant,
                          "equation_set": sn,
                          "sim_seconds_per_wall_second": dt / (ms_step * 1e-3),
                          "l2": "inputs larger than L2 (state %.0f MB vs 126 MB L2)"
                                % (8 * dof / 1e6)},
               "storage_dof_per_s": 5 * mesh.n_nodes / (ms_step * 1e-3),
               "roofline": roof, "step_roofline": step_roof, "kernels": kern,
               "kernels_pass_ms_per_step": round(instr_elapsed / args.steps, 4),
               "clocks": clocks, "e2e": e2e, "cpu_baseline": cpu,
               "setup": {"factor_ms": round(factor_ms, 3),
                         "what": "columnsolve.get_factors on the device (k_lamtab + k_probe + "
                                 "k_lu_dense: probe of lhs_schur, banded LU), once per lam; "
                                 "outside the timed steps, as the reference builds it in its "
                                 "first step (columnsolve.py:184-188)"},
               # fused HEVI step: 3 explicit stages (explicit_col: main + domain-end
               # kernel each) + 2 column solves [+ the P' plane of Q when not chained];
               # at N > 1 plus the halo pack/unpack kernels
               "gpu_launches": launches_per_step * args.steps + halo_launches,
               "launches_per_step": {"ours": launches_per_step,
                                     "all_kernels": counted[1] if counted else None,
                                     "source": "torch.profiler CUDA activity, one untimed step"
                                     if counted else "static schedule count"}}
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_e2e(args, mesh, ref, disc, dt, tab, plan, Q, work, exch, world, rank, dof):
    import torch
    from paper_1702_04316_b200 import imexcore, euler
    from paper_1702_04316_b200.plan import tableau_array
    if world == 1:
        prob = imexcore.ImplicitProblem(disc=disc, ref=ref, set_name=args.set, dim="1d",
                                        solver=imexcore.SolverSpec(method="direct"))
        rhs = euler.make_rhs(ref, disc, args.set)
        host = torch.empty((5,) + tuple(mesh.nshape), dtype=torch.float64, pin_memory=True)
        host.copy_(plan.l2e(Q))
        torch.cuda.synchronize()
        q = imexcore.ark_imex_step(host, dt, tab, prob, rhs)      # warm (pinned pools)
        times = []
        for _ in range(args.e2e_steps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            q = imexcore.ark_imex_step(q, dt, tab, prob, rhs)
            torch.cuda.synchronize()
            times.append(time.perf_counter() - t0)
        ms = 1e3 * sorted(times)[len(times) // 2]
        nbytes = host.numel() * 8
        return {"value": dof / (ms * 1e-3), "unit": UNIT, "h2d_bytes_per_step": nbytes,
                "d2h_bytes_per_step": nbytes, "ms_per_step": ms,
                "path": "imexcore.ark_imex_step(pinned host E-vector) -> H2D, E->lattice, "
                        "fused step, lattice->E, D2H"}
    # multi-GPU: the rank's window in, its owned block out, per step
    import torch.distributed as dist
    tarr = tableau_array(tab)
    lam = tab.diag * dt
    hin = torch.empty_like(Q, device="cpu").pin_memory()
    hout = torch.empty_like(Q, device="cpu").pin_memory()
    hin.copy_(Q)
    times = []
    for _ in range(args.e2e_steps):
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        Q.copy_(hin, non_blocking=True)
        exch(0)
        plan.stage(0, dt, tarr, Q, work)
        plan.stage_solve(0, lam, work)
        exch(1)
        plan.stage(1, dt, tarr, Q, work)
        plan.stage_solve(1, lam, work)
        exch(2)
        plan.stage(2, dt, tarr, Q, work)
        hout.copy_(Q, non_blocking=True)
        torch.cuda.synchronize()
        plan.check_flags()
        t = torch.tensor([time.perf_counter() - t0], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        times.append(float(t.item()))
    ms = 1e3 * sorted(times)[len(times) // 2]
    nbytes = Q.numel() * 8
    return {"value": dof / (ms * 1e-3), "unit": UNIT, "h2d_bytes_per_step": nbytes * world,
            "d2h_bytes_per_step": nbytes * world, "ms_per_step": ms,
            "path": "per-rank pinned window H2D, partitioned fused step, D2H"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg5", choices=sorted(CONFIGS))
    ap.add_argument("--integrator", default="ark2", choices=["ark2", "rk35"],
                    help="ark2: HEVI 1D-IMEX (the metric); rk35: explicit reference (config 2)")
    ap.add_argument("--set", default="set2nc", choices=["set2nc", "set2c"],
                    help="equation set (set2nc: the reference's default)")
    ap.add_argument("--courant", type=float, default=0.0, help="override the config's C_V")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-overlap", action="store_true",
                    help="N > 1: exchange before the whole stage instead of beside its interior tiles")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-steps", type=int, default=4)
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        raise SystemExit(self_launch(args))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


def self_launch(args) -> int:
    """``python bench.py --gpus N`` without torchrun: launch N ranks (one
    process per GPU) the way the driver does, and pass rank 0's line through."""
    import socket
    if args.impl != "reference":
        import torch
        if torch.cuda.device_count() < args.gpus:
            print(json.dumps({"metric": METRIC, "error": f"--gpus {args.gpus} but "
                              f"{torch.cuda.device_count()} CUDA device(s) visible"}), flush=True)
            return 1
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1", "--master-port",
           str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


if __name__ == "__main__":
    main()
