"""Simulation driver on the device path (drop-in for ``dycore.cli`` run mode
and the ``dycore.bench`` diagnostics).

Same configuration format (``key = value`` lines, ``--key=value``
overrides), validation rules, exit codes, time-series CSV
(``time,mass,max_rho_p,max_theta_p,probe_*``, bench.py:158-168) and
snapshot format (``x y z rho_p u v w theta_p``, cli.py:157-170) as the
reference.  The state stays on the unique lattice in HBM for the whole run:
ARK2 steps are the fused five-kernel schedule, RK35 steps the five fused
Shu-Osher launches, BDF2 steps the reference stage loop over the device
operators; diagnostics are one device reduction per record
(``hevi_diagnostics``); the E-vector is materialised only for the final
snapshot.  Supported: box meshes (``case = bubble | rest-state``), cG,
``set2nc``/``set2c``, ``integrator = rk35``, and ARK2 / BDF2 with the Schur
form: ``imex = 1d, solver = direct`` (fused column solve) or the Krylov
solvers on either form (``imex = 1d | 3d``); the cubed-sphere acoustic case
(``case = acoustic``: the general-mesh plan of ``sphere``, E-vector state,
ARK2 / BDF2 with ``imex = 1d, solver = direct`` and per-column factors, or
RK35).  dG and the standard (5-variable) form raise ``NotImplementedError``.

    python -m paper_1702_04316_b200.driver run <config> [--key=value ...]
"""
from __future__ import annotations

import ctypes
import os
import sys
import time
from dataclasses import dataclass, field, fields

import numpy as np

from . import _native as nv
from . import cases, euler, imexcore
from . import specgrid as sg


@dataclass
class RunConfig:
    """cli.py:25-50 (same keys and defaults)."""
    case: str = "bubble"            # acoustic | bubble | rest-state
    equation_set: str = "set2nc"    # set2nc | set2c
    disc: str = "cg"                # cg | dg
    integrator: str = "rk35"        # rk35 | ark2 | bdf2
    imex: str = "none"              # none | 3d | 1d
    form: str = "schur"             # standard | schur
    solver: str = "gmres"           # gmres | bicgstab | richardson | direct
    precon_order: int = 1
    tolerance: float = 1e-6
    dt: float = 0.0                 # 0 -> auto from courant
    courant: float = 0.5
    end_time: float = 100.0
    nx: int = 10
    nz: int = 10
    ne_panel: int = 4
    ne_vert: int = 3
    order: int = 4
    theta0: float = 300.0
    output_dir: str = "out"
    snapshot_interval: float = 0.0
    diag_interval: float = 0.0
    threads: int = 1


_CHOICES = {
    "case": {"acoustic", "bubble", "rest-state"},
    "equation_set": {"set2nc", "set2c"},
    "disc": {"cg", "dg"},
    "integrator": {"rk35", "ark2", "bdf2"},
    "imex": {"none", "3d", "1d"},
    "form": {"standard", "schur"},
    "solver": {"gmres", "bicgstab", "richardson", "direct"},
}


class ConfigError(ValueError):
    pass


def parse_config(path=None, overrides=()) -> RunConfig:
    """``key = value`` lines plus ``--key=value`` overrides, validated as
    cli.parse_config (cli.py:70-118)."""
    kv = {}
    if path is not None:
        with open(path) as f:
            for ln, line in enumerate(f, 1):
                line = line.split("#", 1)[0].strip()
                if not line:
                    continue
                if "=" not in line:
                    raise ConfigError(f"{path}:{ln}: expected key = value")
                k, v = line.split("=", 1)
                kv[k.strip()] = v.strip()
    for ov in overrides:
        if not ov.startswith("--") or "=" not in ov:
            raise ConfigError(f"bad override {ov!r}; expected --key=value")
        k, v = ov[2:].split("=", 1)
        kv[k.strip()] = v.strip()
    cfg = RunConfig()
    names = {f.name for f in fields(RunConfig)}
    for k, v in kv.items():
        if k not in names:
            raise ConfigError(f"unknown config key {k!r}")
        t = type(getattr(cfg, k))
        try:
            setattr(cfg, k, t(v))
        except ValueError as exc:
            raise ConfigError(f"bad value for {k!r}: {v!r}") from exc
    for k, allowed in _CHOICES.items():
        if getattr(cfg, k) not in allowed:
            raise ConfigError(f"{k} must be one of {sorted(allowed)}")
    if cfg.solver == "direct" and cfg.imex != "1d":
        raise ConfigError("the direct column solver requires imex=1d")
    if cfg.disc == "dg" and cfg.form == "schur" and cfg.imex != "none":
        raise ConfigError("the pressure-reduced form is unsupported with dG "
                          "(the flux construction does not converge)")
    if cfg.disc == "dg" and cfg.equation_set != "set2c":
        raise ConfigError("dG requires the conservative set (set2c)")
    if cfg.integrator in ("ark2", "bdf2") and cfg.imex == "none":
        cfg.imex = "3d"
    return cfg


def _check_supported(cfg: RunConfig):
    if cfg.disc != "cg":
        raise NotImplementedError("dG is outside the HEVI direct path")
    if cfg.integrator in ("ark2", "bdf2") and cfg.form != "schur":
        raise NotImplementedError("the device path implements the Schur (pressure) form")


# ---------------------------------------------------------------------------
# diagnostics (bench.py:131-168)
# ---------------------------------------------------------------------------

@dataclass
class Diagnostics:
    times: list = field(default_factory=list)
    mass: list = field(default_factory=list)
    max_rho_p: list = field(default_factory=list)
    max_theta_p: list = field(default_factory=list)
    probes: list = field(default_factory=list)

    def record_values(self, t, mass, max_rho_p, max_theta_p, probe_values=()):
        """bench.Diagnostics.record with the reductions already done."""
        if self.times and t <= self.times[-1]:
            raise ValueError("diagnostic timestamps must increase")
        self.times.append(t)
        self.mass.append(float(mass))
        self.max_rho_p.append(float(max_rho_p))
        self.max_theta_p.append(float(max_theta_p))
        self.probes.append(tuple(probe_values))

    def write_csv(self, path):
        nprobe = len(self.probes[0]) if self.probes else 0
        header = "time,mass,max_rho_p,max_theta_p" + "".join(
            f",probe_{i+1}" for i in range(nprobe))
        with open(path, "w") as f:
            f.write(header + "\n")
            for i, t in enumerate(self.times):
                row = [f"{t:.10g}", f"{self.mass[i]:.14g}",
                       f"{self.max_rho_p[i]:.10g}", f"{self.max_theta_p[i]:.10g}"]
                row += [f"{v:.10g}" for v in self.probes[i]]
                f.write(",".join(row) + "\n")


def axis_mass_weights(mesh: sg.BoxMesh):
    """Per-axis unique-point quadrature weights: W_a[g] = sum over the element
    copies of lattice index g of w_i * h_k / 2, so that the reference's
    sum(wJ * f) over E-vector nodes (bench.py:131-133) equals
    sum_g W_x W_y W_z f on the lattice for continuous f."""
    xe, ye, ze = mesh.edges()
    out = []
    for axis, (e, q, n, ne) in enumerate(((xe, mesh.quad_r, mesh.N, mesh.nx),
                                          (ye, mesh.quad_s, mesh.Ny, mesh.ny),
                                          (ze, mesh.quad_t, mesh.N, mesh.nz))):
        if axis == 1 and mesh.slab:
            out.append(np.asarray(q.weights) * 0.5 * mesh.Ly)
            continue
        W = np.zeros(ne * n + 1)
        for k in range(ne):
            W[k * n:k * n + n + 1] += np.asarray(q.weights) * 0.5 * (e[k + 1] - e[k])
        out.append(W)
    return out


class DeviceDiagnostics:
    """Mass and max |rho'|, |theta'| of a lattice state in one device reduction
    (fixed reduction order: bitwise reproducible)."""

    def __init__(self, plan, mesh):
        import torch
        self.plan = plan
        self.w = [torch.as_tensor(a, dtype=torch.float64, device=plan.device)
                  for a in axis_mass_weights(mesh)]

    def __call__(self, Q):
        out = np.zeros(3)
        nv.check(self.plan.lib.hevi_diagnostics(
            self.plan.h, nv.ptr(Q), nv.ptr(self.w[0]), nv.ptr(self.w[1]), nv.ptr(self.w[2]),
            out.ctypes.data_as(ctypes.c_void_p), nv.stream_ptr()))
        return out


def nearest_lattice_point(mesh: sg.BoxMesh, point):
    """bench.nearest_node (bench.py:171-174) on the lattice: the flat E-vector
    node nearest to the point, returned as its lattice (gz, gy, gx)."""
    c = mesh.coords.reshape(-1, 3)
    i = int(np.argmin(np.linalg.norm(c - np.asarray(point), axis=1)))
    x, y, z = mesh.lattice_coords()
    px, py, pz = c[i]
    return (int(np.argmin(np.abs(z - pz))), int(np.argmin(np.abs(y - py))),
            int(np.argmin(np.abs(x - px))))


def write_snapshot(path, t, q, mesh, ref, set_name):
    """cli.write_snapshot (cli.py:157-170): x y z rho_p u v w theta_p per node."""
    q = q.cpu().numpy() if hasattr(q, "cpu") else np.asarray(q)
    nel, nt, ns, nr = mesh.nshape
    lev = ((np.arange(nel) // (mesh.nx * mesh.ny))[:, None] * mesh.N
           + np.arange(nt)[None, :])[:, :, None, None]
    vel = np.moveaxis(q[1:4], 0, -1)
    if set_name == "set2c":
        rho = ref.rho0[lev] + q[0]
        vel = vel / rho[..., None]
        th_p = (ref.Theta0[lev] + q[4]) / rho - ref.theta0[lev]
    else:
        th_p = q[4]
    xyz = mesh.coords.reshape(-1, 3)
    data = np.column_stack([xyz, q[0].reshape(-1), vel.reshape(-1, 3),
                            np.broadcast_to(th_p, q[4].shape).reshape(-1)])
    np.savetxt(path, data, fmt="%.10g", header=f"time={t:.10g} fields=x y z rho_p u v w theta_p")


# ---------------------------------------------------------------------------
# run (cli.py:173-263)
# ---------------------------------------------------------------------------

@dataclass
class RunResult:
    steps: int
    wall_time: float
    dt: float
    courant_h: float
    courant_v: float
    stats: imexcore.SolveStats
    diagnostics: Diagnostics
    final_q: object
    exit_code: int = 0
    message: str = ""


def _bubble_centre(mesh):
    # bench.RisingBubbleConfig: Lx = Lz = 1000 m, r_b = 250 m, centre (500, 350)
    return (500.0, 0.5 * mesh.Ly, 350.0), (250.0, 250.0, 250.0)


def _build_case(cfg: RunConfig):
    const = euler.GasConstants()
    mesh = sg.build_box_mesh(cfg.nx, cfg.nz, 1000.0, 1000.0, cfg.order)
    ref = euler.hydrostatic_reference(mesh, cfg.theta0, const)
    if cfg.case == "bubble":
        centre, radii = _bubble_centre(mesh)
        Q = cases.bubble_lattice(mesh, ref, 0.5, centre, radii, set_name=cfg.equation_set)
        probe = (500.0, 0.0, 350.0)
    else:
        import torch
        Q = torch.zeros((5, mesh.Z, mesh.Y, mesh.X), dtype=torch.float64, device="cuda")
        probe = (500.0, 0.0, 350.0)
    disc = euler.build_discretization(mesh)
    return mesh, ref, disc, Q, probe


def _courants(mesh, ref, Q, dt, set_name):
    """euler.courant_numbers (euler.py:564-580) of a lattice state."""
    cmax_dt = cases.dt_for_courant(mesh, ref, Q, 1.0, set_name)   # dx_v / cmax
    dx_h, dx_v = mesh.min_node_spacing()
    cmax = dx_v / cmax_dt
    return cmax * dt / dx_h, cmax * dt / dx_v


def run_simulation(cfg: RunConfig, quiet=False) -> RunResult:
    import torch
    from .plan import tableau_array
    _check_supported(cfg)
    os.makedirs(cfg.output_dir, exist_ok=True)
    if cfg.case == "acoustic":
        return _run_sphere(cfg, quiet)
    mesh, ref, disc, Q0, probe_xyz = _build_case(cfg)
    set_name = cfg.equation_set
    rho = torch.as_tensor(ref.rho0, device=Q0.device)[:, None, None] + Q0[0]
    if bool((rho <= 0).any()):
        raise FloatingPointError("total density lost positivity")
    plan = disc.plan_for(ref, set_name)
    Q = plan.zeros()
    Q[..., :mesh.X].copy_(Q0)
    work = plan.workspace()

    dx_h, dx_v = mesh.min_node_spacing()
    dt = cfg.dt if cfg.dt > 0 else cases.dt_for_courant(mesh, ref, Q0, cfg.courant, set_name)
    ch, cv = _courants(mesh, ref, Q0, dt, set_name)

    problem = None
    if cfg.integrator in ("ark2", "bdf2"):
        problem = imexcore.ImplicitProblem(
            disc=disc, ref=ref, set_name=set_name, discretization=cfg.disc, form=cfg.form,
            dim="1d" if cfg.imex == "1d" else "3d",
            solver=imexcore.SolverSpec(method=cfg.solver, tol=cfg.tolerance,
                                       precon_order=cfg.precon_order))
    fused = problem is not None and problem.fused
    ark = imexcore.ark2_tableau()
    tarr = tableau_array(ark)
    bdf = imexcore.bdf2_coefficients()
    diag = DeviceDiagnostics(plan, mesh)
    diags = Diagnostics()
    pz, py, px = nearest_lattice_point(mesh, probe_xyz)
    if set_name == "set2nc":
        pc = (float(ref.G0_nc[pz]), float(ref.H0_nc[pz]))
    else:
        pc = (0.0, float(ref.F0_c[pz]))

    def record(t):
        m, mr, mt = diag(Q)
        v = Q[[0, 4], pz, py, px].cpu().numpy()
        diags.record_values(t, m, mr, mt, (pc[0] * v[0] + pc[1] * v[1],))

    t, steps = 0.0, 0
    record(t)
    next_diag = cfg.diag_interval
    rhs = euler.make_rhs(ref, disc, set_name)
    q_prev = None                       # bdf2 history (device E-vector)
    # the fused and RK35 steps overwrite Q in place and report failures only
    # afterwards: keep the last good state so an aborted run writes it, as
    # the reference does (cli.py:224-250 keeps q at the last good step)
    Qgood = plan.empty() if (cfg.integrator == "rk35" or fused) else None
    inplace = False
    t0 = time.perf_counter()
    exit_code, message = 0, ""
    try:
        while t < cfg.end_time - 1e-12:
            step_dt = min(dt, cfg.end_time - t)
            if Qgood is not None:
                Qgood.copy_(Q)
            if cfg.integrator == "rk35":
                inplace = True
                plan.rk35(step_dt, Q, work)
                plan.check_flags()
                inplace = False
            elif not fused and (cfg.integrator == "ark2" or q_prev is None or step_dt != dt):
                # Krylov solves: the reference stage loop over the device operators
                qn = plan.l2e(Q)
                qn1 = imexcore.ark_imex_step(qn, step_dt, ark, problem, rhs)
                if cfg.integrator == "bdf2":
                    q_prev = qn
                plan.e2l(qn1, out=Q)
            elif cfg.integrator == "ark2" or q_prev is None or step_dt != dt:
                if cfg.integrator == "bdf2":
                    q_prev = plan.l2e(Q)
                lam = ark.diag * step_dt
                plan.factor(lam)
                problem.lam = lam
                inplace = True
                plan.step(step_dt, tarr, Q, work)
                plan.check_flags()
                inplace = False
                problem.stats.solves += 2
            else:
                qn = plan.l2e(Q)
                qn1 = imexcore.bdf2_imex_step(qn, q_prev, step_dt, bdf, problem, rhs)
                q_prev = qn
                plan.e2l(qn1, out=Q)
            t += step_dt
            steps += 1
            if cfg.diag_interval <= 0 or t >= next_diag - 1e-12:
                record(t)
                next_diag += cfg.diag_interval
    except imexcore.SolverFailure as exc:
        exit_code, message = 3, str(exc)
    except FloatingPointError as exc:
        exit_code, message = 4, str(exc)
    finally:
        if inplace and Qgood is not None:
            Q.copy_(Qgood)              # the failed in-place step never happened
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0

    diags.write_csv(os.path.join(cfg.output_dir, "timeseries.csv"))
    q = plan.l2e(Q)
    snap = os.path.join(cfg.output_dir, f"snapshot_{t:012.3f}.txt")
    write_snapshot(snap, t, q, mesh, ref, set_name)
    stats = problem.stats if problem is not None else imexcore.SolveStats()
    if not quiet:
        mean_it = stats.iterations / max(stats.solves, 1)
        print(f"steps={steps} wall={wall:.3f}s dt={dt:.6g} C_H={ch:.3g} C_V={cv:.3g} "
              f"solves={stats.solves} mean_iters={mean_it:.2f} matvecs={stats.matvecs}")
        if message:
            print(f"aborted: {message} (last snapshot: {snap})")
    return RunResult(steps=steps, wall_time=wall, dt=dt, courant_h=ch, courant_v=cv,
                     stats=stats, diagnostics=diags, final_q=q, exit_code=exit_code,
                     message=message)


def write_snapshot_nodes(path, t, q, mesh, ref, set_name):
    """cli.write_snapshot (cli.py:157-170) with a per-node background (general meshes)."""
    q = q.cpu().numpy() if hasattr(q, "cpu") else np.asarray(q)
    vel = np.moveaxis(q[1:4], 0, -1)
    if set_name == "set2c":
        rho = ref.rho0 + q[0]
        vel = vel / rho[..., None]
        th_p = (ref.Theta0 + q[4]) / rho - ref.theta0
    else:
        th_p = q[4]
    xyz = mesh.coords.reshape(-1, 3)
    data = np.column_stack([xyz, q[0].reshape(-1), vel.reshape(-1, 3), th_p.reshape(-1)])
    np.savetxt(path, data, fmt="%.10g", header=f"time={t:.10g} fields=x y z rho_p u v w theta_p")


def _run_sphere(cfg: RunConfig, quiet=False) -> RunResult:
    """The acoustic case on the cubed-sphere shell (cli.py:131-141, 173-263):
    E-vector state on the device, the general-mesh plan (sphere.GPlan):
    ARK2 1D-IMEX direct with per-column factors, or RK35."""
    import torch
    from .plan import tableau_array
    acfg = cases.AcousticWaveConfig(theta0=cfg.theta0)
    mesh = sg.build_cubed_sphere_mesh(cfg.ne_panel, cfg.ne_vert, acfg.r_e, acfg.r_T, cfg.order)
    const = euler.GasConstants()
    # constant-temperature background: uniform sound speed (cli.py:136-138)
    ref = euler.isothermal_reference(mesh, cfg.theta0, const)
    set_name = cfg.equation_set
    q0 = cases.init_acoustic_wave(acfg, mesh, ref, set_name)
    if np.any(ref.rho0 + q0[0] <= 0):
        raise FloatingPointError("total density lost positivity")
    disc = euler.build_discretization(mesh)
    plan = disc.plan_for(ref, set_name)
    Q = plan.dss(torch.as_tensor(q0, device=plan.device))   # coincident copies consistent (cli.py:180)
    work = plan.workspace()
    dx_h, dx_v = euler.min_node_spacing(mesh)
    _, cv0 = euler.courant_numbers(Q, ref, disc, 1.0, set_name)
    dt = cfg.dt if cfg.dt > 0 else cfg.courant * dx_v / (cv0 * dx_v)
    ch, cv = euler.courant_numbers(Q, ref, disc, dt, set_name)
    problem = None
    if cfg.integrator in ("ark2", "bdf2"):
        problem = imexcore.ImplicitProblem(
            disc=disc, ref=ref, set_name=set_name, discretization=cfg.disc, form=cfg.form,
            dim="1d" if cfg.imex == "1d" else "3d",
            solver=imexcore.SolverSpec(method=cfg.solver, tol=cfg.tolerance, precon_order=cfg.precon_order))
    ark = imexcore.ark2_tableau()
    tarr = tableau_array(ark)
    bdf = imexcore.bdf2_coefficients()
    rhs = euler.make_rhs(ref, disc, set_name)
    wJ = torch.as_tensor(disc.metrics.wJ, device=plan.device)
    rho0 = torch.as_tensor(ref.rho0, device=plan.device)
    pid = cases.nearest_node(mesh, cases.probe_point_on_sphere(acfg, np.pi / 2, 0.0))
    if set_name == "set2nc":
        pc = (float(ref.G0_nc.ravel()[pid]), float(ref.H0_nc.ravel()[pid]))
    else:
        pc = (0.0, float(ref.F0_c.ravel()[pid]))
    diags = Diagnostics()

    def record(t):
        mass = float((wJ * (rho0 + Q[0])).sum())
        v = Q[[0, 4]].reshape(2, -1)[:, pid].cpu().numpy()
        diags.record_values(t, mass, float(Q[0].abs().max()), float(Q[4].abs().max()),
                            (pc[0] * v[0] + pc[1] * v[1],))

    t, steps = 0.0, 0
    record(t)
    next_diag = cfg.diag_interval
    q_prev = None
    Qgood = torch.empty_like(Q)
    inplace = False
    t0 = time.perf_counter()
    exit_code, message = 0, ""
    try:
        while t < cfg.end_time - 1e-12:
            step_dt = min(dt, cfg.end_time - t)
            Qgood.copy_(Q)
            if cfg.integrator == "rk35":
                inplace = True
                plan.rk35(step_dt, Q, work)
                plan.check_flags()
                inplace = False
            elif cfg.integrator == "ark2" or q_prev is None or step_dt != dt:
                if cfg.integrator == "bdf2":
                    q_prev = Q.clone()
                if problem.fused:       # 1D-IMEX direct: the device step
                    problem.lam = ark.diag * step_dt
                    inplace = True
                    plan.step(step_dt, tarr, Q, work)
                    plan.check_flags()
                    inplace = False
                    problem.stats.solves += 2
                else:                   # Krylov solves: the reference stage loop on the device operators
                    Q.copy_(imexcore.ark_imex_step(Q.clone(), step_dt, ark, problem, rhs))
            else:
                qn = Q.clone()
                Q.copy_(imexcore.bdf2_imex_step(qn, q_prev, step_dt, bdf, problem, rhs))
                q_prev = qn
            t += step_dt
            steps += 1
            if cfg.diag_interval <= 0 or t >= next_diag - 1e-12:
                record(t)
                next_diag += cfg.diag_interval
    except imexcore.SolverFailure as exc:
        exit_code, message = 3, str(exc)
    except FloatingPointError as exc:
        exit_code, message = 4, str(exc)
    finally:
        if inplace:
            Q.copy_(Qgood)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    diags.write_csv(os.path.join(cfg.output_dir, "timeseries.csv"))
    snap = os.path.join(cfg.output_dir, f"snapshot_{t:012.3f}.txt")
    write_snapshot_nodes(snap, t, Q, mesh, ref, set_name)
    stats = problem.stats if problem is not None else imexcore.SolveStats()
    if not quiet:
        mean_it = stats.iterations / max(stats.solves, 1)
        print(f"steps={steps} wall={wall:.3f}s dt={dt:.6g} C_H={ch:.3g} C_V={cv:.3g} "
              f"solves={stats.solves} mean_iters={mean_it:.2f} matvecs={stats.matvecs}")
        if message:
            print(f"aborted: {message} (last snapshot: {snap})")
    return RunResult(steps=steps, wall_time=wall, dt=dt, courant_h=ch, courant_v=cv, stats=stats,
                     diagnostics=diags, final_q=Q.cpu().numpy(), exit_code=exit_code, message=message)


def main(argv=None) -> int:
    """``run <config> [--key=value ...]`` with the reference's exit codes
    (0 ok, 2 config error, 3 solver failure, 4 non-finite state)."""
    argv = list(sys.argv[1:] if argv is None else argv)
    if len(argv) < 2 or argv[0] != "run":
        print(__doc__.strip().splitlines()[-1].strip(), file=sys.stderr)
        return 2
    try:
        cfg = parse_config(argv[1], argv[2:])
    except (ConfigError, OSError) as exc:
        print(f"config error: {exc}", file=sys.stderr)
        return 2
    res = run_simulation(cfg)
    return res.exit_code


if __name__ == "__main__":
    raise SystemExit(main())
