"""The production column-sweep kernels (explicit_col / explicit_colc) against
the round-1 kernels (explicit_v2 / explicit_c, pinned to the reference by
test_gpu_parity.py) on states the bubble cases do not reach: random,
DSS-continuous, non-zero on every wall, multi-tile grids with partial tiles
and the domain-end planes.  Each fused stage's outputs and three full steps
must agree to round-off, for both equation sets."""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_1702_04316_b200 import specgrid, euler, imexcore  # noqa: E402
from paper_1702_04316_b200.plan import tableau_array  # noqa: E402

TOL = 1e-12


def _plan(disc, ref, sn, kernels):
    old = os.environ.get("HEVI_KERNELS")
    if kernels:
        os.environ["HEVI_KERNELS"] = kernels
    else:
        os.environ.pop("HEVI_KERNELS", None)
    try:
        disc._plans = {}
        return disc.plan_for(ref, sn)
    finally:
        if old is None:
            os.environ.pop("HEVI_KERNELS", None)
        else:
            os.environ["HEVI_KERNELS"] = old


def _run(p, q, dt, lam, sn):
    tab = tableau_array(imexcore.ark2_tableau())
    p.factor(lam)
    Q = p.padded(q.clone())
    W = p.workspace()
    outs = []
    p.stage(0, dt, tab, Q, W)
    outs += [W[1].clone(), W[2].clone(), W[3][[0, 3, 4]].clone()]
    p.stage_solve(0, lam, W)
    p.stage(1, dt, tab, Q, W)
    outs += [W[1].clone(), W[2].clone(), W[3][[0, 3, 4]].clone()]
    p.stage_solve(1, lam, W)
    p.stage(2, dt, tab, Q, W)
    outs.append(Q.clone())
    for _ in range(2):
        p.step(dt, tab, Q, W)
    outs.append(Q.clone())
    R = p.zeros()
    p.rhs(p.padded(q.clone()), R)
    outs.append(R)
    p.check_flags()
    return outs


@pytest.mark.parametrize("sn", ["set2nc", "set2c"])
@pytest.mark.parametrize("dims", [(5, 6, 3), (9, 7, 2)])
def test_column_sweep_matches_round1_kernels_on_wall_data(sn, dims):
    nx, ny, nz = dims
    mesh = specgrid.build_box_mesh_3d(nx, ny, nz, 4000.0 * nx, 4000.0 * ny, 100.0 * nz, 4)
    ref = euler.hydrostatic_reference(mesh, 300.0)
    disc = euler.build_discretization(mesh)
    rng = np.random.default_rng(11 + nx)
    scale = np.array([1e-3, 0.5, 0.5, 0.5, 0.3])[:, None, None, None]
    q = torch.as_tensor(scale * rng.standard_normal((5, mesh.Z, mesh.Y, mesh.X)), device="cuda")
    # no-flux walls as the reference state has them (euler.zero_normal_velocity)
    q[1, :, :, 0] = q[1, :, :, -1] = 0.0
    q[2, :, 0, :] = q[2, :, -1, :] = 0.0
    q[3, 0] = q[3, -1] = 0.0
    dt, lam = 0.05, 0.05 * imexcore.ark2_tableau().diag
    new = _run(_plan(disc, ref, sn, None), q, dt, lam, sn)
    old = _run(_plan(disc, ref, sn, "v2"), q, dt, lam, sn)
    X = mesh.X
    for i, (a, b) in enumerate(zip(new, old)):
        a, b = a[..., :X], b[..., :X]
        for f in range(a.shape[0]):
            n = float(b[f].norm())
            err = float((a[f] - b[f]).norm()) / n if n > 0 else float(a[f].norm())
            assert err < TOL, (sn, dims, i, f, err)
