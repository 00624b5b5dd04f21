"""Reference-behaviour tests of the device path (error types, column API,
conversions), mirroring pkg/tests/test_columnsolve.py and test_imexcore.py."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_1702_04316_b200 import specgrid, euler, imexcore, columnsolve as cs  # noqa: E402


@pytest.fixture(scope="module")
def aniso():
    mesh = specgrid.build_box_mesh(5, 4, 20_000.0, 1000.0, 4)
    ref = euler.hydrostatic_reference(mesh, 300.0)
    return mesh, ref, euler.build_discretization(mesh)


@pytest.fixture(scope="module")
def box3():
    mesh = specgrid.build_box_mesh_3d(3, 2, 3, 12_000.0, 8_000.0, 300.0, 4)
    ref = euler.hydrostatic_reference(mesh, 300.0)
    return mesh, ref, euler.build_discretization(mesh)


def problem(fix, lam=0.5):
    mesh, ref, disc = fix
    return imexcore.ImplicitProblem(disc=disc, ref=ref, set_name="set2nc", dim="1d", lam=lam,
                                    solver=imexcore.SolverSpec(method="direct"))


def random_continuous(fix, seed=0):
    mesh, ref, disc = fix
    rng = np.random.default_rng(seed)
    plan = disc.plan_for(ref)
    L = torch.as_tensor(rng.standard_normal((5, mesh.Z, mesh.Y, mesh.X)), device="cuda")
    scale = torch.tensor([ref.rho0.mean(), 1, 1, 1, 300.0], device="cuda")[:, None, None, None]
    return plan.l2e((1e-3 * L * scale).contiguous())


def test_evec_lattice_roundtrip_exact(box3):
    mesh, ref, disc = box3
    plan = disc.plan_for(ref)
    E = random_continuous(box3, 1)
    assert torch.equal(plan.l2e(plan.e2l(E)), E)


def test_rest_state_is_well_balanced(box3):
    mesh, ref, disc = box3
    R = euler.nonlinear_rhs(np.zeros((5,) + mesh.nshape), ref, disc, "set2nc")
    assert np.abs(R).max() < 1e-9          # test_euler.py:252-256


def test_nonfinite_input_raises(box3):
    mesh, ref, disc = box3
    q = np.zeros((5,) + mesh.nshape)
    q[1, 3, 1, 1, 1] = np.nan
    with pytest.raises(FloatingPointError):
        euler.nonlinear_rhs(q, ref, disc, "set2nc")


def test_nonpositive_density_raises_value_error(box3):
    mesh, ref, disc = box3
    q = np.zeros((5,) + mesh.nshape)
    q[0] = -2.0 * ref.rho0.max()
    with pytest.raises(ValueError):
        euler.nonlinear_rhs(q, ref, disc, "set2nc")
    # the flag is consumed: a valid call afterwards succeeds
    euler.nonlinear_rhs(np.zeros((5,) + mesh.nshape), ref, disc, "set2nc")


def test_step_nan_detection(box3):
    mesh, ref, disc = box3
    q = np.zeros((5,) + mesh.nshape)
    q[4, 0, 0, 0, 0] = np.inf
    prob = problem(box3)
    with pytest.raises(FloatingPointError):
        imexcore.ark_imex_step(q, 0.5, imexcore.ark2_tableau(), prob,
                               euler.make_rhs(ref, disc, "set2nc"))


def test_solve_requires_positive_lam(box3):
    prob = problem(box3, lam=0.0)
    with pytest.raises(ValueError):
        prob.solve(np.zeros((5,) + box3[0].nshape))


def test_solve_zero_rhs_is_zero(aniso):
    prob = problem(aniso, lam=0.5)
    out = prob.solve(np.zeros((5,) + aniso[0].nshape))
    assert np.abs(out).max() == 0.0


def test_identity_at_lam_zero(aniso):
    prob = problem(aniso, lam=0.0)
    cj = cs.build_column_jacobian(prob)
    eye = torch.eye(cj.M, device="cuda").expand_as(cj.matrices)
    assert (cj.matrices - eye).abs().max() < 1e-13


def test_matrix_sizes(aniso):
    mesh = aniso[0]
    cj = cs.build_column_jacobian(problem(aniso, lam=0.4))
    assert cj.M == mesh.n_lev
    assert tuple(cj.matrices.shape) == (mesh.n_col, cj.M, cj.M)


def test_factor_solve_roundtrip(aniso):
    cj = cs.build_column_jacobian(problem(aniso, lam=0.5))
    A = cj.matrices.clone()
    cs.lu_factor_banded(cj)
    assert cj.factored and not cj.pivoted_fallback
    rng = np.random.default_rng(31)
    x = rng.standard_normal((A.shape[0], cj.M))
    b = torch.einsum("cij,cj->ci", A, torch.as_tensor(x, device="cuda")).cpu().numpy()
    got = cs.solve_columns_direct(cj, b)
    assert np.abs(got - x).max() < 1e-9 * max(1.0, np.abs(x).max())


def test_lu_reconstructs_probed_matrix(aniso):
    cj = cs.build_column_jacobian(problem(aniso, lam=0.4))
    A = cj.matrices.clone().cpu().numpy()
    cs.lu_factor_banded(cj)
    F = cj.matrices.cpu().numpy()
    for c in (0, A.shape[0] // 2):
        L = np.tril(F[c], -1) + np.eye(cj.M)
        U = np.triu(F[c])
        assert np.abs(L @ U - A[c]).max() < 1e-11 * max(1.0, np.abs(A[c]).max())


def test_lu_tridiagonal_oracle(aniso):
    A = torch.tensor([[[2.0, 1.0, 0.0], [1.0, 2.0, 1.0], [0.0, 1.0, 2.0]]], device="cuda")
    cj = cs.ColumnJacobian(matrices=A.clone(), bandwidth=2, n_dof=1,
                           space=cs.unique_space(aniso[0]), pivoted_fallback=[], piv={})
    cs.lu_factor_banded(cj)
    F = cj.matrices[0].cpu().numpy()
    L = np.tril(F, -1) + np.eye(3)
    U = np.triu(F)
    assert np.abs(L @ U - A[0].cpu().numpy()).max() < 1e-12


def test_lu_reports_degenerate_diagonal(aniso):
    A = torch.tensor([[[0.0, 1.0], [1.0, 0.0]]], device="cuda")
    cj = cs.ColumnJacobian(matrices=A, bandwidth=2, n_dof=1,
                           space=cs.unique_space(aniso[0]), pivoted_fallback=[], piv={})
    with pytest.raises(RuntimeError):
        cs.lu_factor_banded(cj)


def test_solve_requires_factorization(aniso):
    cj = cs.build_column_jacobian(problem(aniso, lam=0.5))
    with pytest.raises(ValueError):
        cs.solve_columns_direct(cj, np.zeros((cj.matrices.shape[0], cj.M)))


def test_factors_cached_per_lam(aniso):
    prob = problem(aniso, lam=0.5)
    c1 = cs.get_factors(prob)
    assert cs.get_factors(prob) is c1
    prob.lam = 0.25
    assert cs.get_factors(prob) is not c1


def test_column_solve_matches_batched_banded_api(box3):
    """solve_direct's fused column kernel == rhs gathered by hand through the
    generic per-column banded API (columnsolve.py:191-210 spelled out)."""
    from oracle.hevi_oracle import BoxOracle
    mesh, ref, disc = box3
    o = BoxOracle(3, 2, 3, 12_000.0, 8_000.0, 300.0, 4)
    lam = 0.6
    q = random_continuous(box3, 5).cpu().numpy()
    rhsP, _ = o.schur_rhs(q, lam)
    prob = problem(box3, lam=lam)
    cj = cs.get_factors(prob)
    rhs = rhsP.ravel()[o.rep].reshape(o.n_col, o.n_lev)
    P = cs.solve_columns_direct(cj, rhs)
    LU, nb = o.factors(lam)
    want = o.band_solve(LU, nb, rhs)
    assert np.abs(P - want).max() <= 1e-13 * np.abs(want).max()


def test_direct_solve_cost_flat_in_courant(box3):
    """test_acceptance.py:442-468 analogue: the per-solve work does not depend
    on lam once the factor is cached (same kernels, same band)."""
    mesh, ref, disc = box3
    plan = disc.plan_for(ref)
    nbs = {plan.factor(lam) for lam in (0.05, 0.5, 5.0)}
    assert len(nbs) == 1


def test_direct_solve_time_flat_in_courant():
    """test_acceptance.py:442-468: the time of a direct solve is flat in the
    Courant number (lam spans 100x): the spread of the median solve times
    stays within 20 % (CUDA events, a 64x64x10-element box)."""
    from paper_1702_04316_b200 import specgrid
    mesh = specgrid.build_box_mesh_3d(64, 64, 10, 256_000.0, 256_000.0, 1000.0, 4)
    ref = euler.hydrostatic_reference(mesh, 300.0)
    disc = euler.build_discretization(mesh)
    plan = disc.plan_for(ref)
    g = torch.Generator(device="cuda").manual_seed(2)
    qe = plan.padded(0.01 * torch.rand((5, mesh.Z, mesh.Y, mesh.X), generator=g, device="cuda",
                                       dtype=torch.float64))
    out = plan.zeros()
    med = []
    for lam in (0.5, 5.0, 50.0):
        plan.factor(lam)
        for _ in range(3):
            plan.solve(lam, qe, out)
        ts = []
        for _ in range(15):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            plan.solve(lam, qe, out)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        med.append(sorted(ts)[len(ts) // 2])
    plan.check_flags()
    assert max(med) <= 1.2 * min(med), med


@pytest.mark.parametrize("integrator", ["ark2", "rk35"])
def test_host_and_device_inputs_give_bitwise_equal_steps(box3, integrator):
    """Pinned host, device and numpy E-vectors through the fused entry points
    give the same bits, returned in the caller's array type."""
    mesh, ref, disc = box3
    qd = random_continuous(box3, seed=3)
    qh = torch.empty(qd.shape, dtype=torch.float64, pin_memory=True)
    qh.copy_(qd)
    qn = qd.cpu().numpy()
    rhs = euler.make_rhs(ref, disc, "set2nc")
    tab = imexcore.ark2_tableau()
    outs = []
    for q in (qd, qh, qn):
        if integrator == "ark2":
            prob = problem(box3)
            r = imexcore.ark_imex_step(q, 0.5, tab, prob, rhs)
        else:
            r = imexcore.rk35_step(q, 0.05, rhs)
        outs.append(r.cpu().numpy() if isinstance(r, torch.Tensor) else r)
    assert isinstance(imexcore.rk35_step(qh, 0.05, rhs), torch.Tensor)
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])


def test_discontinuous_evector_rejected_when_checking():
    """Opt-in DSS-continuity check of the drop-in entry (plan.lattice_in)."""
    from paper_1702_04316_b200 import specgrid, euler, cases
    mesh = specgrid.build_box_mesh_3d(3, 2, 2, 12_000.0, 8_000.0, 200.0, 4)
    ref = euler.hydrostatic_reference(mesh, 300.0)
    disc = euler.build_discretization(mesh)
    plan = disc.plan_for(ref)
    q0 = cases.bubble_lattice(mesh, ref, 0.5, (6_000.0, 4_000.0, 100.0), (3000.0, 3000.0, 80.0))
    E = plan.l2e(plan.padded(q0))
    plan.check_continuity = True
    try:
        plan.lattice_in(E)                      # continuous: accepted
        E2 = E.clone()
        E2[0, 1, 0, 0, 0] += 1.0                # element 1's copy of a shared face node
        with pytest.raises(ValueError):
            plan.lattice_in(E2)
    finally:
        plan.check_continuity = False
