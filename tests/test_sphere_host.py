"""Host set-up of the cubed-sphere path (no GPU): the mesh, the coincidence
groups, the column/level numbering and the boundary projectors against the
unmodified reference's (tests/golden/sphere_n*.npz), and the geometry
invariants the device kernels rely on."""
import os

import numpy as np
import pytest

from paper_1702_04316_b200 import sphere

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.parametrize("N", [3, 4, 8])
def test_mesh_matches_reference(N):
    d = np.load(os.path.join(HERE, "golden", f"sphere_n{N}.npz"))
    ne = (1, 1) if N == 8 else (2, 2)
    mesh = sphere.build_cubed_sphere_mesh(*ne, 6_371_000.0, 10_000.0, N)
    assert mesh.coords.shape == d["coords"].shape
    assert np.abs(mesh.coords - d["coords"]).max() <= 1e-9          # metres on a 6371 km shell
    assert np.array_equal(mesh.col_id, d["col_id"])
    assert np.array_equal(mesh.lev_id, d["lev_id"])
    metrics = sphere.compute_metrics(mesh)
    dss = sphere.build_dss_map(mesh, metrics)
    assert np.array_equal(dss.gid.reshape(mesh.nshape), d["gid"])


def test_geometry_invariants():
    mesh = sphere.build_cubed_sphere_mesh(2, 2, 6_371_000.0, 10_000.0, 4)
    m = sphere.compute_metrics(mesh)
    assert (m.J > 0).all()
    # n_col radial columns of n_lev levels cover the unique points exactly
    uid = mesh.col_id.astype(np.int64) * mesh.n_lev + mesh.lev_id
    assert len(np.unique(uid)) == mesh.n_col * mesh.n_lev
    assert mesh.n_lev == 2 * 4 + 1
    assert mesh.n_col == 6 * (2 * 4) ** 2 + 2          # 6 N^2 ne^2 + 2 points on the sphere
    dss = sphere.build_dss_map(mesh, m)
    # groups: members in flat order, CSR consistent with gid
    assert dss.ptr[-1] == mesh.n_nodes
    assert np.all(np.diff(dss.gid[dss.idx]) >= 0)
    # the total mass weight of the shell is its volume 4/3 pi (R^3 - r^3) to quadrature accuracy
    r0, r1 = 6_371_000.0, 6_381_000.0
    vol = 4.0 / 3.0 * np.pi * (r1 ** 3 - r0 ** 3)
    assert abs(m.wJ.sum() / vol - 1.0) < 1e-4
    # every bottom/top node group has one symmetric projector I - sum b b^T
    # over its orthonormalised face normals a^t / |a^t|; a^t is not exactly
    # radial on the gnomonic elements, so where elements meet the copies'
    # normals differ by ~3e-4 and the reference keeps more than one of them
    bidx, bproj, slot, projs = sphere.boundary_projectors(mesh, m, dss)
    assert np.abs(np.einsum("nab,nbc->nac", projs, projs) - projs).max() < 1e-10
    assert np.abs(projs - np.swapaxes(projs, 1, 2)).max() == 0.0
    v = mesh.vert.reshape(-1, 3)[bidx]
    assert np.abs(np.einsum("nab,nb->na", bproj, v)).max() < 1e-3
    assert len(projs) == 2 * mesh.n_col


def test_reference_state_per_node():
    from paper_1702_04316_b200 import euler
    mesh = sphere.build_cubed_sphere_mesh(2, 1, 6_371_000.0, 10_000.0, 3)
    ref = euler.isothermal_reference(mesh, 300.0)
    assert ref.rho0.shape == mesh.nshape
    c = euler.GasConstants()
    np.testing.assert_allclose(ref.gvec, c.g * mesh.vert)
    h = euler.hydrostatic_reference(mesh, 300.0)
    assert not h.grad_theta0.any()
    np.testing.assert_allclose(h.theta0, 300.0)
