"""Generate golden fixtures by running the UNMODIFIED reference ``dycore``.

Run in the build container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports the reference read-only from /root/reference/pkg/src, builds the
cases below through the reference's public helpers (plus the SURVEY.md 8(c)
harness 3D box, assembled only from reference helpers), runs the reference
operators / stepper on them and stores inputs and outputs as compact
unique-lattice arrays ``(5, Z, Y, X)`` (first-occurrence copy per DSS group;
the reference cG state is continuous, so nothing is lost) in
``tests/golden/<case>.npz``.  The host CPU / numpy build is recorded in
``tests/golden/HOST.json`` because numpy's SIMD ``pow`` makes velocity
fields host-dependent at the 1e-10 level.

The GPU box never runs this script; tests there read the .npz files only.
"""
from __future__ import annotations

import json
import os
import platform
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
sys.dont_write_bytecode = True

from dycore import specgrid as sg  # noqa: E402
from dycore import euler  # noqa: E402
from dycore import imexcore as imx  # noqa: E402
from dycore import columnsolve as cs  # noqa: E402
from dycore import bench  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def box3d_mesh(nx, ny, nz, Lx, Ly, Lz, N):
    """SURVEY 8(c) harness 3D box built from reference helpers only."""
    q = sg.lgl_nodes_weights(N)
    nq = N + 1
    nel = nx * ny * nz
    coords = np.empty((nel, nq, nq, nq, 3))
    xe = np.linspace(0.0, Lx, nx + 1)
    ye = np.linspace(0.0, Ly, ny + 1)
    ze = np.linspace(0.0, Lz, nz + 1)
    bfaces = []
    for kz in range(nz):
        zs = ze[kz] + (q.nodes + 1.0) * 0.5 * (ze[kz + 1] - ze[kz])
        for ky in range(ny):
            ys = ye[ky] + (q.nodes + 1.0) * 0.5 * (ye[ky + 1] - ye[ky])
            for kx in range(nx):
                e = (kz * ny + ky) * nx + kx
                xs = xe[kx] + (q.nodes + 1.0) * 0.5 * (xe[kx + 1] - xe[kx])
                coords[e, ..., 0] = xs[None, None, :]
                coords[e, ..., 1] = ys[None, :, None]
                coords[e, ..., 2] = zs[:, None, None]
                if kz == 0:
                    bfaces.append((e, 2, 0, "bottom"))
                if kz == nz - 1:
                    bfaces.append((e, 2, 1, "top"))
                if kx == 0:
                    bfaces.append((e, 0, 0, "lateral"))
                if kx == nx - 1:
                    bfaces.append((e, 0, 1, "lateral"))
                if ky == 0:
                    bfaces.append((e, 1, 0, "lateral"))
                if ky == ny - 1:
                    bfaces.append((e, 1, 1, "lateral"))
    vert = np.zeros_like(coords)
    vert[..., 2] = 1.0
    height = coords[..., 2].copy()
    tol = 1e-8 * max(Lx, Ly, Lz)
    col = sg._group_points(coords[..., :2].reshape(-1, 2), tol)
    lev = sg._group_points(height.reshape(-1, 1), tol)
    col_id, lev_id, n_col, n_lev = sg._order_columns_levels(col, lev, height.ravel())
    shape = (nel, nq, nq, nq)
    return sg.ElementMesh(kind="box", N=N, quad_r=q, quad_s=q, quad_t=q,
                          coords=coords, vert=vert, height=height,
                          col_id=col_id.reshape(shape), lev_id=lev_id.reshape(shape),
                          n_col=n_col, n_lev=n_lev, boundary_faces=bfaces,
                          meta={"nx": nx, "ny": ny, "nz": nz})


def lattice_index(mesh, N_s):
    """Flat first-occurrence node of every (gz, gy, gx) lattice point."""
    c = mesh.coords
    N = mesh.N
    nel = mesh.nel
    # recover element indices from the element order used by both builders
    meta = mesh.meta
    nx, nz = meta["nx"], meta["nz"]
    ny = meta.get("ny", 1)
    X, Y, Z = nx * N + 1, ny * N_s + 1, nz * N + 1
    gid = np.empty(mesh.nshape, dtype=np.int64)
    nt, ns, nr = mesh.nshape[1:]
    for e in range(nel):
        kx = e % nx
        ky = (e // nx) % ny
        kz = e // (nx * ny)
        gx = kx * N + np.arange(nr)
        gy = ky * N_s + np.arange(ns)
        gz = kz * N + np.arange(nt)
        gid[e] = (gz[:, None, None] * Y + gy[None, :, None]) * X + gx[None, None, :]
    _, rep = np.unique(gid.ravel(), return_index=True)
    return rep, (Z, Y, X), c


def to_lattice(f, rep, dims):
    lead = f.shape[:-4] if f.ndim > 4 else ()
    flat = f.reshape(lead + (-1,))
    return flat[..., rep].reshape(lead + dims)


def continuous_random_state(disc, ref, seed, amp=1e-3, slab=True):
    """Restates conftest.continuous_random_state (tests/conftest.py:52-67)."""
    rng = np.random.default_rng(seed)
    mesh = disc.mesh
    q = rng.standard_normal((5,) + mesh.nshape)
    if slab:
        q[...] = q[..., :1, :]
        q[2] = 0.0
    q = sg.apply_dss_many(q, disc.dss)
    vel = np.moveaxis(q[1:4], 0, -1).copy()
    euler.zero_normal_velocity(vel, disc.bidx, disc.bproj)
    q[1:4] = np.moveaxis(vel, -1, 0)
    scale = np.array([ref.rho0.mean(), 1.0, 1.0, 1.0, ref.theta0.mean()])
    return amp * scale[:, None, None, None, None] * q


def bubble_state(mesh, ref, disc, theta_c, centre, radii, slab, set_name="set2nc"):
    c = mesh.coords
    if slab:
        r = np.sqrt(((c[..., 0] - centre[0]) / radii[0]) ** 2
                    + ((c[..., 2] - centre[2]) / radii[2]) ** 2)
    else:
        r = np.sqrt(((c[..., 0] - centre[0]) / radii[0]) ** 2
                    + ((c[..., 1] - centre[1]) / radii[1]) ** 2
                    + ((c[..., 2] - centre[2]) / radii[2]) ** 2)
    th = np.where(r <= 1.0, 0.5 * theta_c * (1.0 + np.cos(np.pi * r)), 0.0)
    q = np.zeros((5,) + mesh.nshape)
    q[0] = ref.rho0 * (ref.theta0 / (ref.theta0 + th) - 1.0)
    q[4] = 0.0 if set_name == "set2c" else th     # bench.py:118-123
    return sg.apply_dss_many(q, disc.dss)


def dt_for(mesh, ref, disc, q, C, set_name="set2nc"):
    """cli.run_simulation dt rule (cli.py:187-194)."""
    dx_h, dx_v = euler.min_node_spacing(mesh)
    ch0, cv0 = euler.courant_numbers(q, ref, disc, 1.0, set_name)
    return C * dx_v / (cv0 * dx_v)


def run_case(name, mesh, N_s, slab, ops_seed, lam, bubble, C, nsteps, keep,
             background="hydrostatic", set_name="set2nc"):
    if background == "hydrostatic":
        ref = euler.hydrostatic_reference(mesh, 300.0)
    else:
        ref = euler.isothermal_reference(mesh, 300.0)
    disc = euler.build_discretization(mesh)
    rep, dims, _ = lattice_index(mesh, N_s)
    L = lambda f: to_lattice(f, rep, dims)  # noqa: E731
    out = {}
    # operator level on a continuous random state
    qr = continuous_random_state(disc, ref, ops_seed, slab=slab)
    out["ops_q"] = L(qr)
    out["ops_R"] = L(euler.nonlinear_rhs(qr, ref, disc, set_name))
    out["ops_L"] = L(euler.vertical_restriction(qr, ref, disc, set_name))
    prob = imx.ImplicitProblem(disc=disc, ref=ref, set_name=set_name, form="schur",
                               dim="1d", solver=imx.SolverSpec(method="direct"))
    prob.lam = lam
    out["ops_lam"] = np.array(lam)
    rhsP, ua = prob.rhs_schur_build(qr)
    out["ops_schur_rhs"] = L(rhsP)
    out["ops_solve"] = L(prob.solve(qr))
    cj = cs.get_factors(prob)
    A = cs.build_column_jacobian(prob).matrices
    out["col_A0"] = A[0]
    out["col_LU0"] = cj.matrices[0]
    out["col_nb"] = np.array(cj.bandwidth)
    out["col_spread"] = np.array(np.abs(A - A[0:1]).max())
    # ARK2 HEVI steps from the bubble IC
    q = bubble_state(mesh, ref, disc, *bubble, slab=slab, set_name=set_name)
    dt = dt_for(mesh, ref, disc, q, C, set_name)
    out["step_q0"] = L(q)
    out["step_dt"] = np.array(dt)
    prob = imx.ImplicitProblem(disc=disc, ref=ref, set_name=set_name, form="schur",
                               dim="1d", solver=imx.SolverSpec(method="direct"))
    rhs = lambda s: euler.nonlinear_rhs(s, ref, disc, set_name)  # noqa: E731
    tab = imx.ark2_tableau()
    for k in range(1, nsteps + 1):
        q = imx.ark_imex_step(q, dt, tab, prob, rhs)
        if k in keep:
            out[f"step_q{k}"] = L(q)
    out["solves"] = np.array(prob.stats.solves)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(name, {k: v.shape for k, v in out.items()}, "dt", dt)


def run_rk35_case(name, mesh, N_s, slab, bubble, C, nsteps, keep):
    """Explicit SSP RK(5,3) reference trajectory (imexcore.rk35_step)."""
    ref = euler.hydrostatic_reference(mesh, 300.0)
    disc = euler.build_discretization(mesh)
    rep, dims, _ = lattice_index(mesh, N_s)
    L = lambda f: to_lattice(f, rep, dims)  # noqa: E731
    q = bubble_state(mesh, ref, disc, *bubble, slab=slab)
    dt = dt_for(mesh, ref, disc, q, C)
    out = {"step_q0": L(q), "step_dt": np.array(dt)}
    rhs = lambda s: euler.nonlinear_rhs(s, ref, disc, "set2nc")  # noqa: E731
    for k in range(1, nsteps + 1):
        q = imx.rk35_step(q, dt, rhs)
        if k in keep:
            out[f"step_q{k}"] = L(q)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(name, "dt", dt)


def main():
    host = {"numpy": np.__version__, "python": platform.python_version(),
            "machine": platform.machine(), "processor": platform.processor()}
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    host["cpu"] = line.split(":", 1)[1].strip()
                if line.startswith("flags"):
                    host["avx512f"] = " avx512f " in line
                    break
    except OSError:
        pass
    # 1. reference 2D slab, anisotropic (tests/conftest.py:39-43 grid)
    mesh = sg.build_box_mesh(5, 4, 20_000.0, 1000.0, 4)
    mesh.meta["ny"] = 1
    run_case("slab_aniso", mesh, 1, True, ops_seed=32, lam=0.8,
             bubble=(0.5, (10_000.0, 0.0, 350.0), (2000.0, 1.0, 250.0)),
             C=15.0, nsteps=10, keep=(1, 10))
    # 2. harness 3D box, 40:1 elements (SURVEY 8(c)/(d) config 1 geometry, reduced)
    mesh = box3d_mesh(4, 4, 4, 16_000.0, 16_000.0, 400.0, 4)
    run_case("box3d_n4", mesh, 4, False, ops_seed=7, lam=0.3,
             bubble=(0.5, (8_000.0, 8_000.0, 200.0), (4000.0, 4000.0, 100.0)),
             C=15.0, nsteps=10, keep=(1, 10))
    # 3. harness 3D box on an isothermal (stratified) background: exercises
    #    the Sherman-Morrison inverse and the theta0 gradient terms
    mesh = box3d_mesh(3, 2, 3, 12_000.0, 8_000.0, 300.0, 3)
    run_case("box3d_n3_iso", mesh, 3, False, ops_seed=11, lam=0.25,
             bubble=(0.5, (6_000.0, 4_000.0, 150.0), (3000.0, 3000.0, 80.0)),
             C=15.0, nsteps=3, keep=(1, 3), background="isothermal")
    # 4. inviscid Straka density current, reference slab, N=7 (config 3)
    mesh = sg.build_box_mesh(32, 4, 51_200.0, 6_400.0, 7)
    mesh.meta["ny"] = 1
    run_case("straka_n7", mesh, 1, True, ops_seed=3, lam=0.5,
             bubble=(-15.0, (25_600.0, 0.0, 3_000.0), (4_000.0, 1.0, 2_000.0)),
             C=0.7, nsteps=5, keep=(1, 5))
    # 5. explicit SSP RK(5,3) at C=1 on the 3D box (BASELINE config 2's explicit run)
    mesh = box3d_mesh(4, 4, 4, 16_000.0, 16_000.0, 400.0, 4)
    run_rk35_case("rk35_box3d_n4", mesh, 4, False,
                  bubble=(0.5, (8_000.0, 8_000.0, 200.0), (4000.0, 4000.0, 100.0)),
                  C=1.0, nsteps=10, keep=(1, 10))
    # 6. conservative set (set2c, flux form) on the slab and the 3D box
    mesh = sg.build_box_mesh(5, 4, 20_000.0, 1000.0, 4)
    mesh.meta["ny"] = 1
    run_case("slab_aniso_c", mesh, 1, True, ops_seed=33, lam=0.8,
             bubble=(0.5, (10_000.0, 0.0, 350.0), (2000.0, 1.0, 250.0)),
             C=15.0, nsteps=10, keep=(1, 10), set_name="set2c")
    mesh = box3d_mesh(4, 4, 4, 16_000.0, 16_000.0, 400.0, 4)
    run_case("box3d_n4_c", mesh, 4, False, ops_seed=8, lam=0.3,
             bubble=(0.5, (8_000.0, 8_000.0, 200.0), (4000.0, 4000.0, 100.0)),
             C=15.0, nsteps=10, keep=(1, 10), set_name="set2c")
    with open(os.path.join(HERE, "HOST.json"), "w") as f:
        json.dump(host, f, indent=1)


def extra():
    """Further polynomial orders and stratifications for the parity gates."""
    mesh = box3d_mesh(3, 3, 3, 15_000.0, 15_000.0, 600.0, 5)
    run_case("box3d_n5", mesh, 5, False, ops_seed=41, lam=0.3,
             bubble=(0.5, (7_500.0, 7_500.0, 300.0), (3000.0, 3000.0, 150.0)),
             C=15.0, nsteps=5, keep=(1, 5))
    mesh = box3d_mesh(3, 2, 2, 12_000.0, 8_000.0, 400.0, 6)
    run_case("box3d_n6_c", mesh, 6, False, ops_seed=42, lam=0.3,
             bubble=(0.5, (6_000.0, 4_000.0, 200.0), (3000.0, 3000.0, 100.0)),
             C=15.0, nsteps=5, keep=(1, 5), set_name="set2c")
    mesh = sg.build_box_mesh(8, 6, 16_000.0, 600.0, 2)
    mesh.meta["ny"] = 1
    run_case("slab_n2", mesh, 1, True, ops_seed=43, lam=0.5,
             bubble=(0.5, (8_000.0, 0.0, 300.0), (2000.0, 1.0, 150.0)),
             C=15.0, nsteps=10, keep=(1, 10))
    mesh = box3d_mesh(4, 4, 5, 8_000.0, 8_000.0, 500.0, 2)
    run_case("box3d_n2_iso", mesh, 2, False, ops_seed=44, lam=0.25,
             bubble=(0.5, (4_000.0, 4_000.0, 250.0), (2000.0, 2000.0, 120.0)),
             C=15.0, nsteps=5, keep=(1, 5), background="isothermal")


if __name__ == "__main__":
    extra() if "--extra" in sys.argv else main()
