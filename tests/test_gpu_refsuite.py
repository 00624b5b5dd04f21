"""The reference's own hot-path tests, ported to the drop-in (SURVEY.md §4
"tests that pin the hot path"), calling the repo through the reference
signatures:

  test_columnsolve.py:111-262   column Jacobian / banded LU / direct solve
  test_imexcore.py:190-324,368  ImplicitProblem operator pieces and solves
  test_euler.py:141-345         linearised pressure, linear operator, L_V,
                                well balance, boundary projection, Courant

Ported as written except where the drop-in documents a deviation:
ReferenceState keeps per-level tables (``ref.node(a)`` gives the reference's
per-node arrays; its gradient fields are per node), only the Schur form is
a device column solve (the standard-form probes are not ported), and there
are no dG or cubed-sphere cases.  The scalar-problem stepper tests run on
CPU in test_host.py.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_1702_04316_b200 import specgrid as sg, euler, imexcore as imx, columnsolve as cs  # noqa: E402


def build_setup(nx=4, nz=4, Lx=1000.0, Lz=1000.0, N=4, theta0=300.0):
    mesh = sg.build_box_mesh(nx, nz, Lx, Lz, N)
    disc = euler.build_discretization(mesh)
    ref = euler.hydrostatic_reference(mesh, theta0)
    return mesh, disc, ref


@pytest.fixture(scope="module")
def box44():
    """tests/conftest.py:27-30: 4x4-element N=4 box over 1 km x 1 km."""
    return build_setup(4, 4, N=4)


@pytest.fixture(scope="module")
def aniso_box():
    """tests/conftest.py:39-43: 5x4 N=4, 20 km x 1 km."""
    return build_setup(5, 4, Lx=20_000.0, Lz=1000.0, N=4)


def continuous_random_state(disc, ref, set_name="set2nc", seed=0, amp=1e-3):
    """tests/conftest.py:52-67 with the drop-in's apply_dss_many /
    zero_normal_velocity (device) and per-node reference means."""
    rng = np.random.default_rng(seed)
    mesh = disc.mesh
    q = rng.standard_normal((5,) + mesh.nshape)
    q[...] = q[..., :1, :]
    q[2] = 0.0
    q = sg.apply_dss_many(q, disc.dss)
    vel = np.moveaxis(q[1:4], 0, -1).copy()
    euler.zero_normal_velocity(vel, disc.bidx, disc.bproj)
    q[1:4] = np.moveaxis(vel, -1, 0)
    scale = np.array([ref.node(ref.rho0).mean(), 1.0, 1.0, 1.0, ref.node(ref.theta0).mean()])
    return amp * scale[:, None, None, None, None] * q


def make_problem(disc, ref, set_name="set2nc", form="schur", dim="3d", lam=1.0, **solver_kw):
    spec = imx.SolverSpec(**solver_kw) if solver_kw else imx.SolverSpec()
    p = imx.ImplicitProblem(disc=disc, ref=ref, set_name=set_name, form=form, dim=dim, solver=spec)
    p.lam = lam
    return p


def column_problem(fix, set_name="set2nc", form="schur", lam=0.5):
    mesh, disc, ref = fix
    return make_problem(disc, ref, set_name, form=form, dim="1d", lam=lam, method="direct")


def host(a):
    return a.cpu().numpy() if isinstance(a, torch.Tensor) else np.asarray(a)


# ---------------------------------------------------------------------------
# test_columnsolve.py
# ---------------------------------------------------------------------------
def test_unique_space_roundtrip(box44):
    mesh, _, _ = box44
    space = cs.unique_space(mesh)
    assert space.n_col == mesh.n_col and space.n_lev == mesh.n_lev
    assert np.array_equal(space.uid[space.rep], np.arange(space.n_col * space.n_lev))


def test_identity_at_lam_zero(box44):
    cj = cs.build_column_jacobian(column_problem(box44, lam=0.0))
    eye = np.broadcast_to(np.eye(cj.M), cj.matrices.shape)
    assert np.abs(host(cj.matrices) - eye).max() < 1e-13


def test_matrix_sizes(box44):
    mesh, _, _ = box44
    cj = cs.build_column_jacobian(column_problem(box44, lam=0.4))
    assert cj.M == mesh.n_lev
    assert tuple(cj.matrices.shape) == (mesh.n_col, cj.M, cj.M)


def test_matrix_equals_matrix_free_apply(box44):
    prob = column_problem(box44, lam=0.3)
    cj = cs.build_column_jacobian(prob)
    space = cj.space
    rng = np.random.default_rng(30)
    U = rng.standard_normal((space.n_col, space.n_lev, 1))
    free = np.asarray(cs._unique_apply(prob, space, 1)(U)).reshape(space.n_col, cj.M)
    mat = np.einsum("cij,cj->ci", host(cj.matrices), U.reshape(space.n_col, cj.M))
    assert np.abs(free - mat).max() < 1e-12 * max(1.0, np.abs(free).max())


def test_requires_one_d_problem(box44):
    mesh, disc, ref = box44
    with pytest.raises(ValueError):
        cs.build_column_jacobian(make_problem(disc, ref, dim="3d", lam=0.3))


def _jac_from_matrices(mats, bandwidth, n_dof, space):
    return cs.ColumnJacobian(matrices=mats, bandwidth=bandwidth, n_dof=n_dof, space=space,
                             pivoted_fallback=[], piv={})


def test_lu_identity(box44):
    cj = cs.build_column_jacobian(column_problem(box44, lam=0.0))
    cs.lu_factor_banded(cj)
    eye = np.broadcast_to(np.eye(cj.M), cj.matrices.shape)
    assert np.abs(host(cj.matrices) - eye).max() < 1e-13


def test_lu_tridiagonal_oracle(box44):
    mesh, _, _ = box44
    A = np.array([[[2.0, 1.0, 0.0], [1.0, 2.0, 1.0], [0.0, 1.0, 2.0]]])
    cj = _jac_from_matrices(A.copy(), 2, 1, cs.unique_space(mesh))
    cs.lu_factor_banded(cj)
    LU = host(cj.matrices)[0]
    L = np.tril(LU, -1) + np.eye(3)
    U = np.triu(LU)
    assert np.abs(L @ U - A[0]).max() < 1e-12


def test_lu_reports_degenerate_diagonal(box44):
    mesh, _, _ = box44
    A = np.zeros((1, 2, 2))
    A[0] = [[0.0, 1.0], [1.0, 0.0]]
    cj = _jac_from_matrices(A, 2, 1, cs.unique_space(mesh))
    with pytest.raises(RuntimeError):
        cs.lu_factor_banded(cj)


def test_factor_solve_roundtrip(box44):
    cj = cs.build_column_jacobian(column_problem(box44, lam=0.5))
    A = host(cj.matrices).copy()
    cs.lu_factor_banded(cj)
    assert cj.factored
    assert not cj.pivoted_fallback
    rng = np.random.default_rng(31)
    x = rng.standard_normal((A.shape[0], cj.M))
    b = np.einsum("cij,cj->ci", A, x)
    got = host(cs.solve_columns_direct(cj, b))
    assert np.abs(got - x).max() < 1e-9 * max(1.0, np.abs(x).max())


def test_solve_zero_rhs(box44):
    cj = cs.factor_with_fallback(column_problem(box44, lam=0.5))
    out = host(cs.solve_columns_direct(cj, np.zeros((cj.matrices.shape[0], cj.M))))
    assert np.abs(out).max() == 0.0


def test_solve_requires_factorization(box44):
    cj = cs.build_column_jacobian(column_problem(box44, lam=0.5))
    with pytest.raises(ValueError):
        cs.solve_columns_direct(cj, np.zeros((cj.matrices.shape[0], cj.M)))


def test_lu_reconstructs_probed_matrix(box44):
    cj = cs.build_column_jacobian(column_problem(box44, lam=0.4))
    A = host(cj.matrices).copy()
    cs.lu_factor_banded(cj)
    LU = host(cj.matrices)
    for c in (0, A.shape[0] // 2):
        L = np.tril(LU[c], -1) + np.eye(cj.M)
        U = np.triu(LU[c])
        assert np.abs(L @ U - A[c]).max() < 1e-11 * max(1.0, np.abs(A[c]).max())


def test_direct_matches_gmres(aniso_box):
    mesh, disc, ref = aniso_box
    q_e = continuous_random_state(disc, ref, "set2nc", seed=32)
    lam = 0.8
    p_dir = make_problem(disc, ref, "set2nc", form="schur", dim="1d", lam=lam, method="direct")
    p_it = make_problem(disc, ref, "set2nc", form="schur", dim="1d", lam=lam, method="gmres",
                        tol=1e-12, restart=300, max_iter=5000)
    q_dir = host(p_dir.solve(q_e))
    q_it = host(p_it.solve(q_e))
    assert np.abs(q_dir - q_it).max() < 1e-8 * max(1.0, np.abs(q_dir).max())


def test_factors_cached_per_lam(box44):
    prob = column_problem(box44, lam=0.5)
    c1 = cs.get_factors(prob)
    c2 = cs.get_factors(prob)
    assert c1 is c2
    prob.lam = 0.25
    assert cs.get_factors(prob) is not c1


# ---------------------------------------------------------------------------
# test_imexcore.py (operator structure and solves)
# ---------------------------------------------------------------------------
def test_lhs_standard_identity_at_lam_zero(box44):
    mesh, disc, ref = box44
    prob = make_problem(disc, ref, "set2nc", lam=0.0)
    q = continuous_random_state(disc, ref, seed=20)
    assert np.array_equal(prob.lhs_standard(q), q)


def test_lhs_schur_identity_at_lam_zero(box44):
    mesh, disc, ref = box44
    prob = make_problem(disc, ref, "set2nc", lam=0.0)
    P = np.sin(mesh.coords[..., 0] / 300.0)
    assert np.abs(prob.lhs_schur(P) - P).max() < 1e-14


def test_pressure_only_state_couples_momentum_rows(box44):
    mesh, disc, ref = box44
    prob = make_problem(disc, ref, "set2c", lam=1.0)
    q = np.zeros((5,) + mesh.nshape)
    q[4] = 1.0
    out = prob.lhs_standard(q)
    assert np.abs(out[1:4]).max() > 0.0
    assert np.abs(out[0] - q[0]).max() == 0.0


def test_rhs_schur_zero_estimate(box44):
    mesh, disc, ref = box44
    prob = make_problem(disc, ref, "set2c", lam=0.5)
    rhs, ua = prob.rhs_schur_build(np.zeros((5,) + mesh.nshape))
    assert np.abs(rhs).max() == 0.0
    assert np.abs(ua).max() == 0.0


def test_rank_one_inverse_trivial_for_constant_background(box44):
    mesh, disc, ref = box44
    prob = make_problem(disc, ref, "set2c", lam=0.7)
    q_e = continuous_random_state(disc, ref, "set2c", seed=21)
    vel_e = np.moveaxis(q_e[1:4], 0, -1)
    want = vel_e - (0.7 * (q_e[0] - q_e[4] / ref.node(ref.G0_c)))[..., None] * ref.gvec
    euler.zero_normal_velocity(want, disc.bidx, disc.bproj)
    _, ua = prob.rhs_schur_build(q_e)
    assert np.abs(ua - want).max() < 1e-13 * max(1.0, np.abs(want).max())


def test_schur_quadratic_form_positive(box44):
    mesh, disc, ref = box44
    prob = make_problem(disc, ref, "set2nc", lam=0.05)
    rng = np.random.default_rng(22)
    for _ in range(3):
        P = sg.apply_dss(rng.standard_normal(mesh.nshape), disc.dss)
        assert np.sum(disc.metrics.wJ * P * prob.lhs_schur(P)) > 0.0


def test_extract_zero_pressure_zero_estimates(box44):
    mesh, disc, ref = box44
    prob = make_problem(disc, ref, "set2c", lam=0.5)
    q = prob.extract_from_pressure(np.zeros(mesh.nshape), np.zeros(mesh.nshape + (3,)),
                                   np.zeros((5,) + mesh.nshape))
    assert np.abs(q).max() == 0.0


@pytest.mark.parametrize("set_name", ["set2nc", "set2c"])
def test_solve_schur_residual_and_pressure_identity(box44, set_name):
    mesh, disc, ref = box44
    prob = make_problem(disc, ref, set_name, form="schur", lam=0.2, method="gmres", tol=1e-12,
                        restart=200, max_iter=3000)
    q_e = continuous_random_state(disc, ref, set_name, seed=24)
    q = prob.solve(q_e)
    resid = prob.lhs_standard(q) - q_e
    assert np.abs(resid).max() < 1e-7 * np.abs(q_e).max()
    if set_name == "set2c":
        P = euler.linearized_pressure(q, ref, "set2c")
        want = (euler.linearized_pressure(q_e, ref, "set2c")
                - prob._helmholtz_flux(prob.rhs_schur_build(q_e)[1]))
        assert np.abs(prob.lhs_schur(P) - want).max() < 1e-6 * max(1.0, np.abs(P).max())


def test_schur_pieces_compose_to_the_direct_solve(box44):
    """rhs_schur_build -> column solve of lhs_schur -> extract_from_pressure
    (imexcore.py:229-298, columnsolve.py:191-210) equals the fused solve."""
    mesh, disc, ref = box44
    prob = make_problem(disc, ref, "set2nc", form="schur", dim="1d", lam=0.4, method="direct")
    q_e = continuous_random_state(disc, ref, seed=41)
    rhs, ua = prob.rhs_schur_build(q_e)
    cj = cs.get_factors(prob)
    space = cj.space
    col_rhs = np.asarray(rhs).reshape(-1)[space.rep].reshape(space.n_col, space.n_lev)
    P = host(cs.solve_columns_direct(cj, col_rhs)).reshape(-1)[space.uid].reshape(mesh.nshape)
    q = prob.extract_from_pressure(P, ua, q_e)
    want = host(prob.solve(q_e))
    assert np.abs(q - want).max() < 1e-12 * max(1.0, np.abs(want).max())
    assert np.abs(prob.lhs_schur(P) - rhs).max() < 1e-10 * max(1.0, np.abs(rhs).max())


def test_solve_requires_positive_lam(box44):
    mesh, disc, ref = box44
    with pytest.raises(ValueError):
        make_problem(disc, ref, lam=0.0).solve(np.zeros((5,) + mesh.nshape))


def test_solver_failure_surfaces_report(box44):
    mesh, disc, ref = box44
    prob = make_problem(disc, ref, "set2nc", form="schur", lam=5.0, method="gmres", tol=1e-14,
                        max_iter=2, restart=2)
    with pytest.raises(imx.SolverFailure) as exc:
        prob.solve(continuous_random_state(disc, ref, seed=25))
    assert exc.value.report.iterations >= 2


def test_one_d_matches_three_d_on_uniform_columns(box44):
    mesh, disc, ref = box44
    q = np.zeros((5,) + mesh.nshape)
    z = mesh.height
    q[0] = 1e-4 * np.sin(np.pi * z / 1000.0) * ref.node(ref.rho0)
    q[3] = 0.1 * np.sin(np.pi * z / 1000.0)
    a3 = make_problem(disc, ref, "set2nc", dim="3d", lam=0.3).lhs_standard(q)
    a1 = make_problem(disc, ref, "set2nc", dim="1d", lam=0.3).lhs_standard(q)
    assert np.abs(a3 - a1).max() < 1e-10 * max(1.0, np.abs(a3).max())


# ---------------------------------------------------------------------------
# test_euler.py
# ---------------------------------------------------------------------------
def test_linearized_pressure_zero_state(box44):
    mesh, _, ref = box44
    q = np.zeros((5,) + mesh.nshape)
    assert np.abs(euler.linearized_pressure(q, ref, "set2nc")).max() == 0.0
    assert np.abs(euler.linearized_pressure(q, ref, "set2c")).max() == 0.0


def test_linearized_pressure_set2c_identity(box44):
    mesh, _, ref = box44
    q = np.zeros((5,) + mesh.nshape)
    q[4] = ref.node(ref.Theta0) / ref.const.gamma
    P = euler.linearized_pressure(q, ref, "set2c")
    assert np.abs(P - ref.node(ref.P0f)).max() < 1e-10 * ref.P0f.max()


def test_linearized_pressure_matches_eos_derivative(box44):
    mesh, _, ref = box44
    c = ref.const
    rng = np.random.default_rng(7)
    rho0, th0 = ref.node(ref.rho0), ref.node(ref.theta0)
    drho = 1e-7 * rho0 * rng.standard_normal(mesh.nshape)
    dth = 1e-7 * th0 * rng.standard_normal(mesh.nshape)
    q = np.zeros((5,) + mesh.nshape)
    q[0], q[4] = drho, dth
    lin = euler.linearized_pressure(q, ref, "set2nc")
    full = euler.equation_of_state(rho0 + drho, th0 + dth, c) - ref.node(ref.P0f)
    assert np.abs(lin - full).max() < 1e-6 * np.abs(full).max()


def test_unknown_set_rejected(box44):
    mesh, _, ref = box44
    with pytest.raises(ValueError):
        euler.linearized_pressure(np.zeros((5,) + mesh.nshape), ref, "set3")


@pytest.mark.parametrize("set_name", ["set2nc", "set2c"])
def test_linear_operator_zero(box44, set_name):
    mesh, disc, ref = box44
    assert np.abs(euler.linear_operator(np.zeros((5,) + mesh.nshape), ref, disc, set_name)).max() == 0.0


@pytest.mark.parametrize("set_name", ["set2nc", "set2c"])
def test_linear_operator_superposition(box44, set_name):
    mesh, disc, ref = box44
    q1 = continuous_random_state(disc, ref, set_name, seed=1)
    q2 = continuous_random_state(disc, ref, set_name, seed=2)
    a, b = 2.0, -3.0
    lhs = euler.linear_operator(a * q1 + b * q2, ref, disc, set_name)
    rhs = a * euler.linear_operator(q1, ref, disc, set_name) + b * euler.linear_operator(q2, ref, disc, set_name)
    assert np.abs(lhs - rhs).max() < 1e-12 * max(1.0, np.abs(lhs).max())


def test_theta_tendency_vanishes_constant_background(box44):
    mesh, disc, ref = box44
    L = euler.linear_operator(continuous_random_state(disc, ref, "set2nc", seed=3), ref, disc, "set2nc")
    assert np.abs(L[4]).max() == 0.0


@pytest.mark.parametrize("set_name", ["set2nc", "set2c"])
def test_vertical_restriction_on_uniform_columns(box44, set_name):
    mesh, disc, ref = box44
    q = np.zeros((5,) + mesh.nshape)
    z = mesh.height
    q[0] = 1e-4 * np.sin(np.pi * z / 1000.0) * ref.node(ref.rho0)
    q[3] = 0.1 * np.sin(np.pi * z / 1000.0)
    q[4] = 1e-4 * np.cos(np.pi * z / 1000.0) * ref.node(ref.theta0)
    full = euler.linear_operator(q, ref, disc, set_name)
    vert = euler.vertical_restriction(q, ref, disc, set_name)
    assert np.abs(full - vert).max() < 1e-12 * max(1.0, np.abs(full).max())


def test_vertical_restriction_ignores_horizontal_velocity(box44):
    mesh, disc, ref = box44
    q = np.zeros((5,) + mesh.nshape)
    q[1] = 1.0
    assert np.abs(euler.vertical_restriction(q, ref, disc, "set2nc")).max() < 1e-14


@pytest.mark.parametrize("set_name", ["set2nc", "set2c"])
def test_well_balanced_rest_state(box44, set_name):
    mesh, disc, ref = box44
    assert np.abs(euler.nonlinear_rhs(np.zeros((5,) + mesh.nshape), ref, disc, set_name)).max() < 1e-9


def test_rhs_minus_linear_zero_state(box44):
    mesh, disc, ref = box44
    q = np.zeros((5,) + mesh.nshape)
    diff = euler.nonlinear_rhs(q, ref, disc, "set2nc") - euler.linear_operator(q, ref, disc, "set2nc")
    assert np.abs(diff).max() < 1e-9


def test_set2c_mass_tendency_zero(box44):
    mesh, disc, ref = box44
    q = continuous_random_state(disc, ref, "set2c", seed=8)
    R = euler.nonlinear_rhs(q, ref, disc, "set2c")
    wJ = disc.metrics.wJ
    assert abs(np.sum(wJ * R[0])) < 1e-12 * abs(np.sum(wJ * (ref.node(ref.rho0) + q[0])))


def test_rhs_rejects_unknown_set(box44):
    mesh, disc, ref = box44
    with pytest.raises(ValueError):
        euler.nonlinear_rhs(np.zeros((5,) + mesh.nshape), ref, disc, "bogus")


def test_zero_normal_velocity_on_all_faces(box44):
    mesh, disc, ref = box44
    rng = np.random.default_rng(9)
    vel = rng.standard_normal(mesh.nshape + (3,))
    euler.zero_normal_velocity(vel, disc.bidx, disc.bproj)
    flat = vel.reshape(-1, 3)[disc.bidx]
    # box faces have axis normals: every removed component is exactly zero
    normal = np.stack([np.diagonal(disc.bproj, axis1=1, axis2=2)[:, a] == 0.0 for a in range(3)], -1)
    assert np.abs(flat[normal]).max() < 1e-12
    assert normal.any(axis=1).all()


def test_boundary_projection_idempotent(box44):
    mesh, disc, _ = box44
    vel = np.random.default_rng(10).standard_normal(mesh.nshape + (3,))
    euler.zero_normal_velocity(vel, disc.bidx, disc.bproj)
    v2 = vel.copy()
    euler.zero_normal_velocity(v2, disc.bidx, disc.bproj)
    assert np.abs(v2 - vel).max() < 1e-13


def test_courant_scales_with_dt(box44):
    mesh, disc, ref = box44
    q = np.zeros((5,) + mesh.nshape)
    ch1, cv1 = euler.courant_numbers(q, ref, disc, 1.0, "set2nc")
    ch2, cv2 = euler.courant_numbers(q, ref, disc, 2.0, "set2nc")
    assert ch2 == pytest.approx(2 * ch1, rel=1e-13)
    assert cv2 == pytest.approx(2 * cv1, rel=1e-13)


def test_rest_state_sound_speed(box44):
    mesh, disc, ref = box44
    q = np.zeros((5,) + mesh.nshape)
    dxh, dxv = euler.min_node_spacing(mesh)
    ch, _ = euler.courant_numbers(q, ref, disc, 1.0, "set2nc")
    assert abs(ch * dxh - 347.32) / 347.32 < 5e-3


def test_courant_rejects_bad_dt(box44):
    mesh, disc, ref = box44
    with pytest.raises(ValueError):
        euler.courant_numbers(np.zeros((5,) + mesh.nshape), ref, disc, 0.0, "set2nc")


# ---------------------------------------------------------------------------
# apply_dss / DSS-projected derivatives (specgrid.py:535-548, euler.py:281-300)
# ---------------------------------------------------------------------------
def test_apply_dss_projection_and_mass(box44):
    """DSS is a projection (idempotent) that conserves sum(wJ f)."""
    mesh, disc, _ = box44
    f = np.random.default_rng(11).standard_normal(mesh.nshape)
    g = sg.apply_dss(f, disc.dss)
    wJ = disc.metrics.wJ
    assert np.abs(sg.apply_dss(g, disc.dss) - g).max() < 1e-14
    assert abs(np.sum(wJ * g) - np.sum(wJ * f)) < 1e-12 * np.sum(wJ * np.abs(f))


def test_dss_derivatives_of_linear_fields(box44):
    mesh, disc, _ = box44
    c = mesh.coords
    f = 3.0 * c[..., 0] - 2.0 * c[..., 2]
    g = disc.gradc(f)
    assert np.abs(g[..., 0] - 3.0).max() < 1e-11 and np.abs(g[..., 2] + 2.0).max() < 1e-11
    gv = disc.grad_vc(f)
    assert np.abs(gv[..., :2]).max() == 0.0 and np.abs(gv[..., 2] + 2.0).max() < 1e-11
    vec = np.stack([c[..., 0], 0.0 * c[..., 0], 2.0 * c[..., 2]], -1)
    assert np.abs(disc.divc(vec) - 3.0).max() < 1e-11
    assert np.abs(disc.div_vc(vec) - 2.0).max() < 1e-11
