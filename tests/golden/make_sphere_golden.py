"""Golden fixtures on the cubed-sphere shell from the UNMODIFIED reference
(cubed-sphere meshes, per-column factors, the acoustic
case).  Run in the build container, where /root/reference exists:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_sphere_golden.py

Cases ``sphere_n3``, ``sphere_n4`` (ne_panel = ne_vert = 2) and ``sphere_n8``
(ne_panel = ne_vert = 1, the largest element the device kernels take):
build_cubed_sphere_mesh(ne_panel, ne_vert, r_e, r_T = the AcousticWaveConfig shell, N), the isothermal 300 K
background the reference driver uses for the acoustic case (cli.py:131-141),
the balanced acoustic pulse (bench.init_acoustic_wave) plus a DSS-projected
random velocity, and through the reference's public API:

  R    nonlinear_rhs, set2nc and set2c (set2c input: the linearised Theta')
  LV   vertical_restriction
  A    the probed per-column Schur matrices of columns 0, 7, n_col-1
       (build_column_jacobian, lam = 0.5 dt)
  X    ImplicitProblem.solve (direct) of the state, lam = 0.5 dt
  Q1,Q3  one and three ARK2 1D-IMEX direct steps at C_V = 5
  X3g, X3b   the 3D-IMEX Schur solve (dim 3d) by GMRES and by BiCGstab +
       PBNO (order 3), tol 1e-10, with their iteration counts; L3 the full
       3D linear operator
  K1   one RK35 step at C_V = 0.5
for each equation set; the mesh coordinates and DSS groups are stored so the
tests can check the device path's mesh set-up first.  E-vector layout, fp64.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import make_golden as mg  # noqa: E402  (imports the reference read-only)

sg, euler, imx, cs, bench = mg.sg, mg.euler, mg.imx, mg.cs, mg.bench


def run_case(N, ne_panel=2, ne_vert=2, seed=7):
    acfg = bench.AcousticWaveConfig(theta0=300.0)
    mesh = sg.build_cubed_sphere_mesh(ne_panel, ne_vert, acfg.r_e, acfg.r_T, N)
    ref = euler.isothermal_reference(mesh, 300.0)
    disc = euler.build_discretization(mesh)
    out = {"coords": mesh.coords, "gid": disc.dss.gid.reshape(mesh.nshape),
           "col_id": mesh.col_id, "lev_id": mesh.lev_id}
    rng = np.random.default_rng(seed)
    dx_h, dx_v = euler.min_node_spacing(mesh)
    for sn in ("set2nc", "set2c"):
        q = bench.init_acoustic_wave(acfg, mesh, ref, sn).q
        q[1:4] = 0.5 * rng.standard_normal(q[1:4].shape)
        q = sg.apply_dss_many(q, disc.dss)
        mom = np.moveaxis(q[1:4], 0, -1).copy()
        euler.zero_normal_velocity(mom, disc.bidx, disc.bproj)
        q[1:4] = np.moveaxis(mom, -1, 0)
        _, cv = euler.courant_numbers(q, ref, disc, 1.0, sn)
        dt = 5.0 / cv
        out[f"{sn}_q0"] = q.copy()
        out[f"{sn}_dt"] = np.array(dt)
        out[f"{sn}_R"] = euler.nonlinear_rhs(q, ref, disc, sn)
        out[f"{sn}_LV"] = euler.vertical_restriction(q, ref, disc, sn)
        prob = imx.ImplicitProblem(disc=disc, ref=ref, set_name=sn, form="schur", dim="1d",
                                   solver=imx.SolverSpec(method="direct"))
        prob.lam = 0.5 * dt
        cj = cs.build_column_jacobian(prob)
        cols = [0, 7, cj.space.n_col - 1]
        out[f"{sn}_A"] = cj.matrices[cols].copy()
        out[f"{sn}_Acols"] = np.array(cols)
        out[f"{sn}_X"] = prob.solve(q)
        tab = imx.ark2_tableau()
        rhs = (lambda s, sn=sn: euler.nonlinear_rhs(s, ref, disc, sn))
        qs = q.copy()
        for k in range(3):
            qs = imx.ark_imex_step(qs, dt, tab, prob, rhs)
            if k in (0, 2):
                out[f"{sn}_Q{k + 1}"] = qs.copy()
        # 3D-IMEX: the Schur pressure equation by GMRES and by BiCGstab + PBNO
        for tag, spec in (("g", imx.SolverSpec(method="gmres", tol=1e-10)),
                          ("b", imx.SolverSpec(method="bicgstab", tol=1e-10, precon_order=3))):
            p3 = imx.ImplicitProblem(disc=disc, ref=ref, set_name=sn, form="schur", dim="3d", solver=spec)
            p3.lam = 0.5 * dt
            out[f"{sn}_X3{tag}"] = p3.solve(q)
            out[f"{sn}_X3{tag}_it"] = np.array(p3.stats.iterations)
        out[f"{sn}_L3"] = euler.linear_operator(q, ref, disc, sn)
        dte = 0.5 / cv
        out[f"{sn}_dte"] = np.array(dte)
        out[f"{sn}_K1"] = imx.rk35_step(q.copy(), dte, rhs)
    return out


def main():
    for N, ne_p, ne_v in ((3, 2, 2), (4, 2, 2), (8, 1, 1)):
        out = run_case(N, ne_p, ne_v)
        path = os.path.join(HERE, f"sphere_n{N}.npz")
        np.savez_compressed(path, **out)
        print(path, os.path.getsize(path))


if __name__ == "__main__":
    main()
