"""Pivoted fallback of the column factorisation (columnsolve.py:141-167):
batched partial-pivoting LU against scipy.linalg.lu_factor/lu_solve, the
reference's degenerate-pivot RuntimeError, and the fused step running on a
forced pivoted factor (same trajectory as the banded factor)."""
import numpy as np
import pytest

from conftest import load_golden, oracle_for, rel_fields, set_of

torch = pytest.importorskip("torch")
scipy_linalg = pytest.importorskip("scipy.linalg")
pytestmark = pytest.mark.gpu

from paper_1702_04316_b200 import columnsolve, euler, imexcore  # noqa: E402
from test_gpu_parity import build, dev  # noqa: E402


def _cj(mats, nb):
    space = columnsolve.UniqueSpace(mesh=None, n_col=mats.shape[0], n_lev=mats.shape[1],
                                    shape=(mats.shape[0], mats.shape[1]))
    return columnsolve.ColumnJacobian(matrices=torch.as_tensor(mats, device="cuda"),
                                      bandwidth=nb, n_dof=1, space=space,
                                      pivoted_fallback=[], piv={})


def test_pivoted_lu_matches_scipy():
    rng = np.random.default_rng(5)
    n_col, M = 7, 23
    mats = rng.standard_normal((n_col, M, M))
    mats[:, np.arange(M), np.arange(M)] = 0.0          # forces row interchanges
    cj = columnsolve.lu_factor_pivoted(_cj(mats, M))
    for c in range(n_col):
        lu, piv = scipy_linalg.lu_factor(mats[c])
        assert np.array_equal(cj.lu_piv[c].cpu().numpy(), piv)
        np.testing.assert_allclose(cj.lu[c].cpu().numpy(), lu, rtol=0, atol=1e-12 * np.abs(lu).max())
    rhs = rng.standard_normal((n_col, M))
    x = columnsolve.solve_columns_direct(cj, rhs)
    for c in range(n_col):
        want = scipy_linalg.lu_solve(scipy_linalg.lu_factor(mats[c]), rhs[c])
        np.testing.assert_allclose(x[c], want, rtol=1e-11, atol=1e-11 * np.abs(want).max())


def test_degenerate_pivot_raises_then_falls_back():
    """test_columnsolve.py:186-192 (zero pivot -> RuntimeError), then the
    fallback of factor_with_fallback on the same matrices."""
    A = np.array([[[0.0, 1.0, 0.0], [1.0, 2.0, 1.0], [0.0, 1.0, 2.0]]])
    cj = _cj(A.copy(), 2)
    with pytest.raises(RuntimeError):
        columnsolve.lu_factor_banded(cj)
    cj = columnsolve.lu_factor_pivoted(_cj(A.copy(), 2))
    assert cj.factored and cj.pivoted_fallback == [0]
    b = np.array([[1.0, 2.0, 3.0]])
    x = columnsolve.solve_columns_direct(cj, b)
    np.testing.assert_allclose(A[0] @ x[0], b[0], rtol=0, atol=1e-14)


def test_singular_column_reports_info():
    A = np.zeros((1, 4, 4))
    A[0, :2, :2] = [[1.0, 2.0], [2.0, 4.0]]
    cj = columnsolve.lu_factor_pivoted(_cj(A, 4))
    assert cj.lu_info[0] == 2          # getrf: first exactly-zero pivot at k = 1


@pytest.mark.parametrize("name", ["box3d_n4", "box3d_n4_c", "slab_aniso"])
def test_fused_step_on_forced_pivoted_factor(name):
    mesh, ref, disc = build(name)
    o, g = oracle_for(name), load_golden(name)
    sn = set_of(name)
    plan = disc.plan_for(ref, sn)
    plan.force_pivoted(True)
    q0 = o.from_lattice(g["step_q0"])
    dt = float(g["step_dt"])
    prob = imexcore.ImplicitProblem(disc=disc, ref=ref, set_name=sn, dim="1d",
                                    solver=imexcore.SolverSpec(method="direct"))
    rhs = euler.make_rhs(ref, disc, sn)
    tab = imexcore.ark2_tableau()
    q = dev(q0)
    for _ in range(10):
        q = imexcore.ark_imex_step(q, dt, tab, prob, rhs)
    assert plan.factor_pivoted(tab.diag * dt)
    # the same trajectory on the banded factor (fresh discretisation)
    mesh2, ref2, disc2 = build(name)
    prob2 = imexcore.ImplicitProblem(disc=disc2, ref=ref2, set_name=sn, dim="1d",
                                     solver=imexcore.SolverSpec(method="direct"))
    rhs2 = euler.make_rhs(ref2, disc2, sn)
    q2 = dev(q0)
    for _ in range(10):
        q2 = imexcore.ark_imex_step(q2, dt, tab, prob2, rhs2)
    assert not disc2.plan_for(ref2, sn).factor_pivoted(tab.diag * dt)
    errs = rel_fields(o.to_lattice(q.cpu().numpy()), o.to_lattice(q2.cpu().numpy()))
    assert max(errs) < 1e-12, errs
    errs = rel_fields(o.to_lattice(q.cpu().numpy()), g["step_q10"])
    assert errs[0] < 1e-10 and errs[1] < 5e-9 and errs[2] < 5e-9, errs
