"""Direct (column LU) solve of the standard 5-variable form (dim='1d',
columnsolve.py:75-108, 196-204) against the unmodified reference
(tests/golden/make_imex3d_golden.py --direct-standard)."""
import os

import numpy as np
import pytest

from conftest import rel_fields

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_1702_04316_b200 import columnsolve, euler, imexcore, specgrid  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def g():
    return np.load(os.path.join(HERE, "golden", "direct_standard.npz"))


def test_standard_column_matrix_and_solve_slab(g):
    from oracle.hevi_oracle import BoxOracle
    mesh = specgrid.build_box_mesh(5, 4, 20_000.0, 1000.0, 4)
    ref = euler.hydrostatic_reference(mesh, 300.0)
    disc = euler.build_discretization(mesh)
    o = BoxOracle(5, 1, 4, 20_000.0, None, 1000.0, 4, slab=True)
    prob = imexcore.ImplicitProblem(disc=disc, ref=ref, set_name="set2nc", form="standard", dim="1d",
                                    solver=imexcore.SolverSpec(method="direct"))
    prob.lam = 0.8
    out = o.to_lattice(prob.solve(o.from_lattice(g["slab_q"])))
    A, _, nb = columnsolve.standard_column_factor(prob)
    assert nb == int(g["slab_nb"])
    assert np.abs(A - g["slab_A0"]).max() <= 1e-13 * np.abs(g["slab_A0"]).max()
    # cond ~5e5: substitution rounding is amplified accordingly
    assert max(rel_fields(out, g["slab_solve"])) < 1e-9
    assert prob.stats.solves == 1


@pytest.mark.parametrize("sn", ["set2nc", "set2c"])
def test_standard_direct_solve_box(g, sn):
    from oracle.hevi_oracle import BoxOracle
    mesh = specgrid.build_box_mesh_3d(3, 3, 3, 12_000.0, 12_000.0, 300.0, 4)
    ref = euler.hydrostatic_reference(mesh, 300.0)
    disc = euler.build_discretization(mesh)
    o = BoxOracle(3, 3, 3, 12_000.0, 12_000.0, 300.0, 4, set_name=sn)
    prob = imexcore.ImplicitProblem(disc=disc, ref=ref, set_name=sn, form="standard", dim="1d",
                                    solver=imexcore.SolverSpec(method="direct"))
    prob.lam = 0.3
    out = o.to_lattice(prob.solve(o.from_lattice(g["box_q"])))
    assert max(rel_fields(out, g[f"box_{sn}"])) < 1e-9


def test_standard_direct_step_equals_schur_direct_step():
    """ARK2 with the standard-form direct solve reproduces the Schur-form step
    (same implicit problem, different elimination) to the conditioning floor."""
    from oracle.hevi_oracle import BoxOracle
    mesh = specgrid.build_box_mesh_3d(3, 3, 3, 12_000.0, 12_000.0, 300.0, 4)
    ref = euler.hydrostatic_reference(mesh, 300.0)
    disc = euler.build_discretization(mesh)
    o = BoxOracle(3, 3, 3, 12_000.0, 12_000.0, 300.0, 4)
    q0 = o.bubble(0.5, (6000.0, 6000.0, 150.0), (3000.0, 3000.0, 80.0))
    dt = o.dt_for_courant(q0, 15.0)
    rhs = euler.make_rhs(ref, disc, "set2nc")
    tab = imexcore.ark2_tableau()
    outs = []
    for form in ("standard", "schur"):
        prob = imexcore.ImplicitProblem(disc=disc, ref=ref, set_name="set2nc", form=form, dim="1d",
                                        solver=imexcore.SolverSpec(method="direct"))
        q = torch.as_tensor(q0, device="cuda")
        for _ in range(3):
            q = imexcore.ark_imex_step(q, dt, tab, prob, rhs)
        outs.append(o.to_lattice(q.cpu().numpy()))
    assert max(rel_fields(outs[0], outs[1])) < 1e-8
