"""The cubed-sphere shell on the device against goldens
from the unmodified reference (tests/golden/make_sphere_golden.py): R(q),
L_V(q), the per-column probed Schur matrices, the direct solve, ARK2 1D-IMEX
steps through the drop-in ``ark_imex_step`` and an RK35 step, set2nc and
set2c, N = 3 and 4.

Tolerances (relative L2 per field against the reference): the reference
forms P' = P0 (rho R theta / P0)^gamma - P0f with a cancellation of |P| eps
~ 1e-11 Pa; the device uses the cancellation-free series (as the box path).
The operators agree to 1e-11; steps to 1e-9 (the box path's tiers)."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def _case(N):
    from paper_1702_04316_b200 import specgrid as sg, euler
    d = np.load(os.path.join(HERE, "golden", f"sphere_n{N}.npz"))
    ne = (1, 1) if N == 8 else (2, 2)
    mesh = sg.build_cubed_sphere_mesh(*ne, 6_371_000.0, 10_000.0, N)
    ref = euler.isothermal_reference(mesh, 300.0)
    disc = euler.build_discretization(mesh)
    return d, mesh, ref, disc


def rel(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    out = []
    for f in range(a.shape[0]):
        n = np.linalg.norm(b[f])
        out.append(np.linalg.norm(a[f] - b[f]) / (n if n > 0 else 1.0))
    return np.array(out)


@pytest.mark.parametrize("N", [3, 4, 8])
@pytest.mark.parametrize("sn", ["set2nc", "set2c"])
def test_sphere_operators(N, sn):
    from paper_1702_04316_b200 import euler
    d, mesh, ref, disc = _case(N)
    q = d[f"{sn}_q0"]
    R = euler.nonlinear_rhs(q, ref, disc, sn)
    e = rel(R, d[f"{sn}_R"])
    print(sn, N, "R", e)
    assert e.max() < 1e-10, e
    L = euler.vertical_restriction(q, ref, disc, sn)
    e = rel(L, d[f"{sn}_LV"])
    print(sn, N, "LV", e)
    # the balanced pulse's vertical momentum L_V is a near-cancellation of the
    # pressure gradient and the buoyancy q0 g / rho0: measure its error
    # against the size of the cancelling terms (at N = 8 the small result
    # itself differs by ~1e-9 relative)
    G = d[f"{sn}_LV"]
    buoy = np.abs(q[0] / ref.rho0).max() * ref.const.g
    for f in range(5):
        scale = np.abs(G[f]).max() + (buoy if f in (1, 2, 3) else 0.0)
        assert np.abs(np.asarray(L[f]) - G[f]).max() <= 1e-11 * scale, (f, e)


@pytest.mark.parametrize("N", [3, 4, 8])
@pytest.mark.parametrize("sn", ["set2nc", "set2c"])
def test_sphere_columns_and_solve(N, sn):
    from paper_1702_04316_b200 import imexcore as imx
    d, mesh, ref, disc = _case(N)
    q = d[f"{sn}_q0"]
    dt = float(d[f"{sn}_dt"])
    prob = imx.ImplicitProblem(disc=disc, ref=ref, set_name=sn, form="schur", dim="1d",
                               solver=imx.SolverSpec(method="direct"))
    prob.lam = 0.5 * dt
    plan = disc.plan_for(ref, sn)
    for i, c in enumerate(d[f"{sn}_Acols"]):
        A = plan.column_matrix(prob.lam, int(c))
        G = d[f"{sn}_A"][i]
        err = np.abs(A - G).max() / np.abs(G).max()
        assert err < 1e-13, (c, err)
    X = prob.solve(q)
    e = rel(X, d[f"{sn}_X"])
    print(sn, N, "X", e)
    assert e.max() < 1e-11, e


@pytest.mark.parametrize("N", [3, 4, 8])
@pytest.mark.parametrize("sn", ["set2nc", "set2c"])
def test_sphere_ark2_and_rk35(N, sn):
    from paper_1702_04316_b200 import euler, imexcore as imx
    d, mesh, ref, disc = _case(N)
    q = d[f"{sn}_q0"]
    dt = float(d[f"{sn}_dt"])
    prob = imx.ImplicitProblem(disc=disc, ref=ref, set_name=sn, form="schur", dim="1d",
                               solver=imx.SolverSpec(method="direct"))
    rhs = euler.make_rhs(ref, disc, sn)
    tab = imx.ark2_tableau()
    qs = q.copy()
    for k in range(3):
        qs = imx.ark_imex_step(qs, dt, tab, prob, rhs)
        if k in (0, 2):
            e = rel(qs, d[f"{sn}_Q{k + 1}"])
            print(sn, N, f"Q{k + 1}", e)
            assert e.max() < 1e-9, e
    # the reference's generic stage loop on a plain lambda gives the same
    q1 = imx.ark_imex_step(q.copy(), dt, tab, prob, lambda s: euler.nonlinear_rhs(s, ref, disc, sn))
    assert rel(q1, d[f"{sn}_Q1"]).max() < 1e-9
    K = imx.rk35_step(q.copy(), float(d[f"{sn}_dte"]), rhs)
    e = rel(K, d[f"{sn}_K1"])
    print(sn, N, "K1", e)
    assert e.max() < 1e-10, e


def test_sphere_dss_and_derivatives():
    """apply_dss and the Discretization derivatives on the shell: DSS is a
    projection (idempotent), and the vertical gradient of the height is the
    radial unit vector (the height is linear along t)."""
    import torch
    from paper_1702_04316_b200 import specgrid as sg
    d, mesh, ref, disc = _case(4)
    rng = np.random.default_rng(3)
    f = rng.standard_normal(mesh.nshape)
    g1 = sg.apply_dss(f, disc.dss)
    g2 = sg.apply_dss(g1, disc.dss)
    assert np.abs(g2 - g1).max() < 1e-14 * np.abs(g1).max()
    gh = disc.grad_vc(mesh.height)
    assert np.abs(gh - mesh.vert).max() < 1e-9
    # full gradient: height depends on t only, so gradc = DSS(ft a^t); a^t is
    # not exactly radial on the gnomonic elements (a few 1e-4)
    gg = disc.gradc(mesh.height)
    assert np.abs(gg - mesh.vert).max() < 1e-3
    dv = disc.div_vc(mesh.vert * 1.0)
    assert np.isfinite(dv).all()
    del torch


@pytest.mark.parametrize("N", [3, 4])
@pytest.mark.parametrize("sn", ["set2nc", "set2c"])
def test_sphere_imex3d(N, sn):
    """3D-IMEX on the shell: the full linear operator, and the Schur pressure
    equation by GMRES and by BiCGstab + PBNO (order 3), against the
    reference's solutions and iteration counts."""
    from paper_1702_04316_b200 import euler, imexcore as imx
    d, mesh, ref, disc = _case(N)
    q = d[f"{sn}_q0"]
    dt = float(d[f"{sn}_dt"])
    L3 = euler.linear_operator(q, ref, disc, sn)
    G = d[f"{sn}_L3"]
    buoy = np.abs(q[0] / ref.rho0).max() * ref.const.g
    for f in range(5):
        scale = np.abs(G[f]).max() + (buoy if f in (1, 2, 3) else 0.0)
        assert np.abs(np.asarray(L3[f]) - G[f]).max() <= 1e-11 * scale, f
    for tag, spec in (("g", imx.SolverSpec(method="gmres", tol=1e-10)),
                      ("b", imx.SolverSpec(method="bicgstab", tol=1e-10, precon_order=3))):
        p3 = imx.ImplicitProblem(disc=disc, ref=ref, set_name=sn, form="schur", dim="3d", solver=spec)
        p3.lam = 0.5 * dt
        X = p3.solve(q)
        e = rel(X, d[f"{sn}_X3{tag}"])
        print(sn, N, "X3" + tag, p3.stats.iterations, int(d[f"{sn}_X3{tag}_it"]), e)
        assert abs(p3.stats.iterations - int(d[f"{sn}_X3{tag}_it"])) <= 1
        assert e.max() < 1e-8, e


def test_sphere_hydrostatic_rest_state_stays_at_rest():
    """The constant-theta hydrostatic background on the shell (grad theta0 = 0:
    A^-1 is the identity, imexcore.py:203-206): the rest state is a discrete
    equilibrium to round-off through R, L_V and ARK2 steps."""
    from paper_1702_04316_b200 import specgrid as sg, euler, imexcore as imx
    mesh = sg.build_cubed_sphere_mesh(2, 2, 6_371_000.0, 10_000.0, 4)
    ref = euler.hydrostatic_reference(mesh, 300.0)
    disc = euler.build_discretization(mesh)
    q = np.zeros((5,) + mesh.nshape)
    R = euler.nonlinear_rhs(q, ref, disc, "set2nc")
    L = euler.vertical_restriction(q, ref, disc, "set2nc")
    assert np.abs(R).max() < 1e-9 and np.abs(L).max() < 1e-12
    prob = imx.ImplicitProblem(disc=disc, ref=ref, set_name="set2nc", form="schur", dim="1d",
                               solver=imx.SolverSpec(method="direct"))
    rhs = euler.make_rhs(ref, disc, "set2nc")
    qs = q
    for _ in range(5):
        qs = imx.ark_imex_step(qs, 30.0, imx.ark2_tableau(), prob, rhs)
    assert np.abs(qs[1:4]).max() < 1e-7 and np.abs(qs[0]).max() < 1e-10
