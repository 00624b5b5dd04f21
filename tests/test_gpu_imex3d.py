"""3D-IMEX on the device: full linear operator, Schur
pressure operators, Krylov solves with the PBNO preconditioner and ARK2
3D-IMEX steps against the unmodified reference
(tests/golden/make_imex3d_golden.py)."""
import os

import numpy as np
import pytest

from conftest import rel_fields

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_1702_04316_b200 import euler, imexcore, specgrid  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
CASES = {"imex3d_box": "set2nc", "imex3d_box_c": "set2c"}


@pytest.fixture(scope="module", params=sorted(CASES))
def case(request):
    from oracle.hevi_oracle import BoxOracle
    name = request.param
    sn = CASES[name]
    g = np.load(os.path.join(HERE, "golden", f"{name}.npz"))
    mesh = specgrid.build_box_mesh_3d(3, 3, 3, 1200.0, 1200.0, 1200.0, 4)
    ref = euler.hydrostatic_reference(mesh, 300.0)
    disc = euler.build_discretization(mesh)
    o = BoxOracle(3, 3, 3, 1200.0, 1200.0, 1200.0, 4, set_name=sn)
    return name, sn, mesh, ref, disc, o, g


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def test_full_linear_operator_matches_reference(case):
    name, sn, mesh, ref, disc, o, g = case
    q = o.from_lattice(g["ops_q"])
    L = euler.linear_operator(q, ref, disc, sn)
    errs = rel_fields(o.to_lattice(L), g["ops_L3"])
    assert max(errs) < 1e-13, errs


def test_schur_operators_match_reference(case):
    name, sn, mesh, ref, disc, o, g = case
    plan = disc.plan_for(ref, sn)
    lam = float(g["ops_lam"])
    Qe = plan.padded(torch.as_tensor(g["ops_q"], device="cuda"))
    ua, Pe = plan.zeros(3), plan.zeros(1)[0]
    plan.schur3_ua(lam, Qe, ua, Pe)
    rhs = plan.schur3_flux(lam, Pe, ua, plan.zeros(1)[0])
    X = mesh.X
    assert rel(ua[..., :X].cpu().numpy(), g["ops_ua"]) < 1e-13
    assert rel(rhs[..., :X].cpu().numpy(), g["ops_schur_rhs"]) < 1e-13
    P = plan.padded(torch.as_tensor(g["ops_P"][None], device="cuda"))[0]
    up = plan.schur3_up(lam, P, plan.zeros(3))
    lhs = plan.schur3_flux(lam, P, up, plan.zeros(1)[0])
    assert rel(lhs[..., :X].cpu().numpy(), g["ops_lhs"]) < 1e-13


SOLVES = {
    "gmres0": dict(method="gmres", tol=1e-11, precon_order=0),
    "gmres1": dict(method="gmres", tol=1e-11, precon_order=1),
    "bicg3": dict(method="bicgstab", tol=1e-11, precon_order=3),
    "rich1": dict(method="richardson", tol=1e-9, precon_order=1),
}


@pytest.mark.parametrize("tag", sorted(SOLVES))
def test_krylov_solve_matches_reference(case, tag):
    name, sn, mesh, ref, disc, o, g = case
    prob = imexcore.ImplicitProblem(disc=disc, ref=ref, set_name=sn, form="schur", dim="3d",
                                    solver=imexcore.SolverSpec(**SOLVES[tag]))
    prob.lam = float(g["ops_lam"])
    q = o.from_lattice(g["ops_q"])
    out = prob.solve(q)
    errs = rel_fields(o.to_lattice(out), g[f"solve_{tag}"])
    tol = 1e-7 if tag == "rich1" else 1e-9
    assert max(errs) < tol, (tag, errs)
    want = int(g[f"iters_{tag}"])
    got = prob.stats.iterations
    print(name, tag, "iterations", got, "reference", want, "errs", errs)
    # same Krylov iterates as the reference's E-vector iteration (measured: equal
    # counts for every solver; PBNO's Ritz start vector differs, so allow one)
    assert abs(got - want) <= 1, (got, want)
    assert prob.stats.solves == 1 and prob.stats.failures == 0


def test_imex3d_steps_match_reference(case):
    name, sn, mesh, ref, disc, o, g = case
    prob = imexcore.ImplicitProblem(disc=disc, ref=ref, set_name=sn, form="schur", dim="3d",
                                    solver=imexcore.SolverSpec(method="gmres", tol=1e-11,
                                                               precon_order=1))
    rhs = euler.make_rhs(ref, disc, sn)
    q = torch.as_tensor(o.from_lattice(g["step_q0"]), device="cuda")
    dt = float(g["step_dt"])
    tab = imexcore.ark2_tableau()
    for k in range(1, 4):
        q = imexcore.ark_imex_step(q, dt, tab, prob, rhs)
        errs = rel_fields(o.to_lattice(q.cpu().numpy()), g[f"step_q{k}"])
        print(name, "step", k, errs)
        assert errs[0] < 1e-8 and errs[2] < 1e-8 and errs[1] < 1e-7, (k, errs)
    assert prob.stats.solves == 6


def test_solver_failure_raises(case):
    name, sn, mesh, ref, disc, o, g = case
    prob = imexcore.ImplicitProblem(disc=disc, ref=ref, set_name=sn, form="schur", dim="3d",
                                    solver=imexcore.SolverSpec(method="gmres", tol=1e-14,
                                                               max_iter=3, precon_order=0))
    prob.lam = float(g["ops_lam"])
    with pytest.raises(imexcore.SolverFailure):
        prob.solve(o.from_lattice(g["ops_q"]))
    assert prob.stats.failures == 1


@pytest.mark.parametrize("tag", ["gmres0", "gmres1", "bicg3"])
def test_krylov_1d_form_matches_reference_and_direct(tag):
    """Krylov solves of the 1D form (grad_vc/div_vc) on the anisotropic slab:
    reference iteration counts, and direct == GMRES to 1e-8 at lam = 0.8
    (test_columnsolve.py:240-252)."""
    from oracle.hevi_oracle import BoxOracle
    g = np.load(os.path.join(HERE, "golden", "krylov1d_slab.npz"))
    mesh = specgrid.build_box_mesh(5, 4, 20_000.0, 1000.0, 4)
    ref = euler.hydrostatic_reference(mesh, 300.0)
    disc = euler.build_discretization(mesh)
    o = BoxOracle(5, 1, 4, 20_000.0, None, 1000.0, 4, slab=True)
    spec = {"gmres0": dict(method="gmres", tol=1e-12, precon_order=0),
            "gmres1": dict(method="gmres", tol=1e-12, precon_order=1),
            "bicg3": dict(method="bicgstab", tol=1e-12, precon_order=3)}[tag]
    prob = imexcore.ImplicitProblem(disc=disc, ref=ref, set_name="set2nc", form="schur", dim="1d",
                                    solver=imexcore.SolverSpec(**spec))
    prob.lam = 0.8
    q = o.from_lattice(g["ops_q"])
    out = o.to_lattice(prob.solve(q))
    assert max(rel_fields(out, g[f"solve_{tag}"])) < 1e-9
    assert max(rel_fields(out, g["solve_direct"])) < 1e-8
    assert abs(prob.stats.iterations - int(g[f"iters_{tag}"])) <= 1
    direct = imexcore.ImplicitProblem(disc=disc, ref=ref, set_name="set2nc", form="schur", dim="1d",
                                      solver=imexcore.SolverSpec(method="direct"))
    direct.lam = 0.8
    assert max(rel_fields(out, o.to_lattice(direct.solve(q)))) < 1e-8


@pytest.mark.parametrize("which", ["box_set2nc", "box_set2c", "slab_bicg"])
def test_standard_form_krylov_matches_reference(which):
    """5-variable form with the reference's diagonal scaling (imexcore.py:330-355)."""
    from oracle.hevi_oracle import BoxOracle
    g = np.load(os.path.join(HERE, "golden", "krylov_standard.npz"))
    if which.startswith("box"):
        sn = which[4:]
        mesh = specgrid.build_box_mesh_3d(3, 3, 3, 1200.0, 1200.0, 1200.0, 4)
        o = BoxOracle(3, 3, 3, 1200.0, 1200.0, 1200.0, 4, set_name=sn)
        spec, dim, lam, q = dict(method="gmres", tol=1e-11, precon_order=1), "3d", 0.4, g["box_q"]
    else:
        sn = "set2nc"
        mesh = specgrid.build_box_mesh(5, 4, 20_000.0, 1000.0, 4)
        o = BoxOracle(5, 1, 4, 20_000.0, None, 1000.0, 4, slab=True)
        spec, dim, lam, q = dict(method="bicgstab", tol=1e-11, precon_order=3), "1d", 0.8, g["slab_q"]
    ref = euler.hydrostatic_reference(mesh, 300.0)
    disc = euler.build_discretization(mesh)
    prob = imexcore.ImplicitProblem(disc=disc, ref=ref, set_name=sn, form="standard", dim=dim,
                                    solver=imexcore.SolverSpec(**spec))
    prob.lam = lam
    out = o.to_lattice(prob.solve(o.from_lattice(q)))
    errs = rel_fields(out, g[which])
    print(which, prob.stats.iterations, int(g[f"{which}_iters"]), errs)
    if which.startswith("box"):
        assert max(errs) < 1e-8, errs
    else:
        # the 1D standard form is ill-conditioned (cond ~5e5): a
        # 1e-11 residual leaves ~1e-7 solution error in either implementation,
        # so both are measured against the exact (direct Schur) solution
        exact = np.load(os.path.join(HERE, "golden", "krylov1d_slab.npz"))["solve_direct"]
        e_ref = max(rel_fields(g[which], exact))
        e_mine = max(rel_fields(out, exact))
        print("vs exact: reference", e_ref, "device", e_mine)
        assert e_mine < max(10 * e_ref, 1e-9), (e_mine, e_ref)
    # PBNO is fitted on Ritz values from a different random start vector; on the
    # ill-conditioned 1D standard form BiCGstab's count moves with it (95 vs 105)
    want = int(g[f"{which}_iters"])
    assert abs(prob.stats.iterations - want) <= max(2, want // (10 if which.startswith("box") else 4))
