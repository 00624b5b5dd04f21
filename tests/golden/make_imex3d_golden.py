"""Golden fixtures of the reference's 3D-IMEX path (ImplicitProblem with
dim="3d", form="schur", Krylov solvers + PBNO; SURVEY 8(d) config 4 /
8(f) rank 1), made by the UNMODIFIED reference:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_imex3d_golden.py [--1d | --standard | --direct-standard]

Per case (isotropic 3D box, 3x3x3 elements, N=4, both equation sets):
full linear operator L(q), Schur rhs, lhs_schur(P), Krylov solves
(GMRES no preconditioner, GMRES + PBNO(1), BiCGstab + PBNO(3), Richardson +
PBNO(1)) with their iteration counts, and 3 ARK2 3D-IMEX steps."""
from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from make_golden import (HERE, box3d_mesh, bubble_state, continuous_random_state, dt_for,  # noqa: E402
                         euler, imx, lattice_index, to_lattice)

SOLVES = {
    "gmres0": dict(method="gmres", tol=1e-11, precon_order=0),
    "gmres1": dict(method="gmres", tol=1e-11, precon_order=1),
    "bicg3": dict(method="bicgstab", tol=1e-11, precon_order=3),
    "rich1": dict(method="richardson", tol=1e-9, precon_order=1),
}


def run(name, set_name, lam=0.4, C=4.0, nsteps=3):
    mesh = box3d_mesh(3, 3, 3, 1200.0, 1200.0, 1200.0, 4)
    ref = euler.hydrostatic_reference(mesh, 300.0)
    disc = euler.build_discretization(mesh)
    rep, dims, _ = lattice_index(mesh, 4)
    L = lambda f: to_lattice(f, rep, dims)  # noqa: E731
    out = {}
    qr = continuous_random_state(disc, ref, 21, slab=False)
    out["ops_q"] = L(qr)
    out["ops_L3"] = L(euler.linear_operator(qr, ref, disc, set_name))
    prob = imx.ImplicitProblem(disc=disc, ref=ref, set_name=set_name, form="schur", dim="3d")
    prob.lam = lam
    out["ops_lam"] = np.array(lam)
    rhsP, ua = prob.rhs_schur_build(qr)
    out["ops_schur_rhs"] = L(rhsP)
    out["ops_ua"] = L(np.moveaxis(ua, -1, 0))
    P = euler.linearized_pressure(qr, ref, set_name)
    out["ops_P"] = L(P)
    out["ops_lhs"] = L(prob.lhs_schur(P))
    for tag, spec in SOLVES.items():
        p = imx.ImplicitProblem(disc=disc, ref=ref, set_name=set_name, form="schur", dim="3d",
                                solver=imx.SolverSpec(**spec))
        p.lam = lam
        out[f"solve_{tag}"] = L(p.solve(qr))
        out[f"iters_{tag}"] = np.array(p.stats.iterations)
        out[f"matvecs_{tag}"] = np.array(p.stats.matvecs)
    q = bubble_state(mesh, ref, disc, 0.5, (600.0, 600.0, 350.0), (250.0, 250.0, 250.0),
                     slab=False, set_name=set_name)
    dt = dt_for(mesh, ref, disc, q, C, set_name)
    out["step_q0"] = L(q)
    out["step_dt"] = np.array(dt)
    prob = imx.ImplicitProblem(disc=disc, ref=ref, set_name=set_name, form="schur", dim="3d",
                               solver=imx.SolverSpec(method="gmres", tol=1e-11, precon_order=1))
    rhs = lambda s: euler.nonlinear_rhs(s, ref, disc, set_name)  # noqa: E731
    tab = imx.ark2_tableau()
    for k in range(1, nsteps + 1):
        q = imx.ark_imex_step(q, dt, tab, prob, rhs)
        out[f"step_q{k}"] = L(q)
    out["step_iters"] = np.array(prob.stats.iterations)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(name, "dt", dt, {k: int(v) for k, v in out.items() if k.startswith(("iters", "step_it"))})


if __name__ == "__main__" and not set(sys.argv) & {"--1d", "--standard", "--direct-standard"}:
    run("imex3d_box", "set2nc")
    run("imex3d_box_c", "set2c")


def run_1d(name="krylov1d_slab"):
    """Krylov solves of the 1D form (dim='1d', grad_vc/div_vc) on the slab_aniso
    case (test_columnsolve.py:240-252: direct == GMRES to 1e-8 at lam = 0.8)."""
    from make_golden import sg
    mesh = sg.build_box_mesh(5, 4, 20_000.0, 1000.0, 4)
    mesh.meta["ny"] = 1
    ref = euler.hydrostatic_reference(mesh, 300.0)
    disc = euler.build_discretization(mesh)
    rep, dims, _ = lattice_index(mesh, 1)
    L = lambda f: to_lattice(f, rep, dims)  # noqa: E731
    qr = continuous_random_state(disc, ref, 32, slab=True)
    out = {"ops_q": L(qr), "ops_lam": np.array(0.8)}
    for tag, spec in {"gmres0": dict(method="gmres", tol=1e-12, precon_order=0),
                      "gmres1": dict(method="gmres", tol=1e-12, precon_order=1),
                      "bicg3": dict(method="bicgstab", tol=1e-12, precon_order=3)}.items():
        p = imx.ImplicitProblem(disc=disc, ref=ref, set_name="set2nc", form="schur", dim="1d",
                                solver=imx.SolverSpec(**spec))
        p.lam = 0.8
        out[f"solve_{tag}"] = L(p.solve(qr))
        out[f"iters_{tag}"] = np.array(p.stats.iterations)
    p = imx.ImplicitProblem(disc=disc, ref=ref, set_name="set2nc", form="schur", dim="1d",
                            solver=imx.SolverSpec(method="direct"))
    p.lam = 0.8
    out["solve_direct"] = L(p.solve(qr))
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(name, {k: int(v) for k, v in out.items() if k.startswith("iters")})


if __name__ == "__main__" and "--1d" in sys.argv:
    run_1d()


def run_standard(name="krylov_standard"):
    """Standard (5-variable) form Krylov solves (imexcore.py:330-355) on the 3D
    box (dim='3d') and on the anisotropic slab (dim='1d')."""
    from make_golden import sg
    out = {}
    mesh = box3d_mesh(3, 3, 3, 1200.0, 1200.0, 1200.0, 4)
    ref = euler.hydrostatic_reference(mesh, 300.0)
    disc = euler.build_discretization(mesh)
    rep, dims, _ = lattice_index(mesh, 4)
    qr = continuous_random_state(disc, ref, 21, slab=False)
    out["box_q"] = to_lattice(qr, rep, dims)
    for sn in ("set2nc", "set2c"):
        p = imx.ImplicitProblem(disc=disc, ref=ref, set_name=sn, form="standard", dim="3d",
                                solver=imx.SolverSpec(method="gmres", tol=1e-11, precon_order=1))
        p.lam = 0.4
        out[f"box_{sn}"] = to_lattice(p.solve(qr), rep, dims)
        out[f"box_{sn}_iters"] = np.array(p.stats.iterations)
    mesh = sg.build_box_mesh(5, 4, 20_000.0, 1000.0, 4)
    mesh.meta["ny"] = 1
    ref = euler.hydrostatic_reference(mesh, 300.0)
    disc = euler.build_discretization(mesh)
    rep, dims, _ = lattice_index(mesh, 1)
    qr = continuous_random_state(disc, ref, 32, slab=True)
    out["slab_q"] = to_lattice(qr, rep, dims)
    p = imx.ImplicitProblem(disc=disc, ref=ref, set_name="set2nc", form="standard", dim="1d",
                            solver=imx.SolverSpec(method="bicgstab", tol=1e-11, precon_order=3))
    p.lam = 0.8
    out["slab_bicg"] = to_lattice(p.solve(qr), rep, dims)
    out["slab_bicg_iters"] = np.array(p.stats.iterations)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(name, {k: int(v) for k, v in out.items() if k.endswith("iters")})


if __name__ == "__main__" and "--standard" in sys.argv:
    run_standard()


def run_standard_direct(name="direct_standard"):
    """Direct (column LU) solves of the standard 5-variable form (dim='1d',
    columnsolve.py:196-204) and the probed column matrix."""
    from make_golden import sg, cs
    out = {}
    mesh = sg.build_box_mesh(5, 4, 20_000.0, 1000.0, 4)
    mesh.meta["ny"] = 1
    ref = euler.hydrostatic_reference(mesh, 300.0)
    disc = euler.build_discretization(mesh)
    rep, dims, _ = lattice_index(mesh, 1)
    qr = continuous_random_state(disc, ref, 32, slab=True)
    out["slab_q"] = to_lattice(qr, rep, dims)
    p = imx.ImplicitProblem(disc=disc, ref=ref, set_name="set2nc", form="standard", dim="1d",
                            solver=imx.SolverSpec(method="direct"))
    p.lam = 0.8
    out["slab_solve"] = to_lattice(p.solve(qr), rep, dims)
    cj = cs.build_column_jacobian(p)
    out["slab_A0"] = cj.matrices[0]
    out["slab_nb"] = np.array(cj.bandwidth)
    mesh = box3d_mesh(3, 3, 3, 12_000.0, 12_000.0, 300.0, 4)
    ref = euler.hydrostatic_reference(mesh, 300.0)
    disc = euler.build_discretization(mesh)
    rep, dims, _ = lattice_index(mesh, 4)
    qr = continuous_random_state(disc, ref, 22, slab=False)
    out["box_q"] = to_lattice(qr, rep, dims)
    for sn in ("set2nc", "set2c"):
        p = imx.ImplicitProblem(disc=disc, ref=ref, set_name=sn, form="standard", dim="1d",
                                solver=imx.SolverSpec(method="direct"))
        p.lam = 0.3
        out[f"box_{sn}"] = to_lattice(p.solve(qr), rep, dims)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(name, "nb", int(out["slab_nb"]))


if __name__ == "__main__" and "--direct-standard" in sys.argv:
    run_standard_direct()
