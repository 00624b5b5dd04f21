"""CPU-only tests: the C ABI library, host-side set-up and the stepper logic.

No compute call reaches the GPU here.  Tests marked ``needs_reference``
compare host tables against the unmodified reference and are skipped where
/root/reference is absent (the GPU box)."""
import ctypes
import math
import os
import re

import numpy as np
import pytest

from conftest import ROOT

from paper_1702_04316_b200 import _native, specgrid, euler, imexcore, columnsolve
from paper_1702_04316_b200 import distributed as dd

REF = "/root/reference/pkg/src"
needs_reference = pytest.mark.skipif(not os.path.isdir(REF), reason="reference not mounted")


# ---------------------------------------------------------------------------
# the C ABI
# ---------------------------------------------------------------------------

def header_symbols():
    txt = open(os.path.join(ROOT, "include", "hevi.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return set(re.findall(r"\b(hevi_[a-z0-9_]+)\s*\(", txt))


def test_header_declares_exactly_the_bound_symbols():
    assert header_symbols() == set(_native.SIGNATURES)


def test_library_loads_and_exports_every_header_symbol():
    lib = _native.load()
    for name in header_symbols():
        assert hasattr(lib, name), name
    # pure host entry points are callable without a GPU
    assert lib.hevi_state_size(None) == 0
    assert lib.hevi_plan_destroy(None) == 0


def test_library_rejects_bad_plan_arguments_without_gpu():
    lib = _native.load()
    gd = _native.GridDesc(nex=2, ney=2, nez=2, N=9, Ny=9, slab=0, x0=0, y0=0, lX=19, lY=19,
                          px=20, ex_b=0, ex_e=2, ey_b=0, ey_e=2)
    arrs = [np.zeros(64) for _ in range(18)]
    rd = _native.RefDesc(*[a.ctypes.data_as(ctypes.POINTER(ctypes.c_double)) for a in arrs],
                         9.8, 287.0, 1e5, 1.4, 0)
    h = ctypes.c_void_p()
    rc = lib.hevi_plan_create(ctypes.byref(h), ctypes.byref(gd), ctypes.byref(rd))
    assert rc == -1 and b"order" in lib.hevi_last_error()


def test_compute_entry_points_require_cuda():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    mesh = specgrid.build_box_mesh_3d(2, 2, 2, 8000.0, 8000.0, 200.0, 4)
    ref = euler.hydrostatic_reference(mesh, 300.0)
    disc = euler.build_discretization(mesh)
    with pytest.raises(RuntimeError, match="CUDA"):
        euler.nonlinear_rhs(np.zeros((5,) + mesh.nshape), ref, disc, "set2nc")


def test_unsupported_paths_raise_not_implemented():
    mesh = specgrid.build_box_mesh_3d(2, 2, 2, 8000.0, 8000.0, 200.0, 4)
    ref = euler.hydrostatic_reference(mesh, 300.0)
    disc = euler.build_discretization(mesh)
    q = np.zeros((5,) + mesh.nshape)
    with pytest.raises(NotImplementedError):
        euler.nonlinear_rhs(q, ref, disc, "set2c", dg=True)
    with pytest.raises(ValueError):
        euler.nonlinear_rhs(q, ref, disc, "set3")
    prob = imexcore.ImplicitProblem(disc=disc, ref=ref, set_name="set2nc", dim="3d", lam=0.3,
                                    form="bogus")
    with pytest.raises(ValueError):
        prob.solve(q)
    prob = imexcore.ImplicitProblem(disc=disc, ref=ref, set_name="set2nc", dim="3d", lam=0.3,
                                    solver=imexcore.SolverSpec(method="direct"))
    with pytest.raises(ValueError):
        prob.solve(q)
    with pytest.raises(ValueError):
        imexcore.ImplicitProblem(disc=disc, ref=ref, set_name="set2nc", discretization="dg",
                                 form="schur")


# ---------------------------------------------------------------------------
# integrator logic (ports of pkg/tests/test_imexcore.py:16-158, 368-374)
# ---------------------------------------------------------------------------

def test_ark2_tableau_consistency():
    t = imexcore.ark2_tableau()
    assert np.allclose(t.a.sum(axis=1), t.c, atol=1e-14)
    assert np.allclose(t.at.sum(axis=1), t.ct, atol=1e-14)
    assert abs(t.b.sum() - 1.0) < 1e-14
    assert t.diag == pytest.approx(1.0 - 1.0 / np.sqrt(2.0))
    assert abs(t.b @ t.c - 0.5) < 1e-14
    assert abs(t.b @ t.ct - 0.5) < 1e-14
    assert np.allclose(t.at[-1], t.b, atol=1e-14)


class ScalarProblem:
    """test_imexcore.py:93-106: q' = k q treated implicitly."""

    def __init__(self, k):
        self.k, self.lam = k, 0.0

    def linear(self, q):
        return np.zeros_like(q) if self.k == 0.0 else self.k * q

    def solve(self, q_e):
        return q_e / (1.0 - self.lam * self.k)


def explicit_rk(q, dt, a, b, rhs):
    k = []
    for i in range(len(b)):
        qi = q.copy()
        for j in range(i):
            qi = qi + dt * a[i, j] * k[j]
        k.append(rhs(qi))
    out = q.copy()
    for i in range(len(b)):
        out = out + dt * b[i] * k[i]
    return out


def test_ark2_reduces_to_explicit_rk_when_linear_zero():
    t = imexcore.ark2_tableau()
    rhs = lambda q: np.sin(q) - 0.3 * q  # noqa: E731
    q = np.array([0.7])
    got = imexcore.ark_imex_step(q, 0.2, t, ScalarProblem(0.0), rhs)
    assert np.array_equal(got, explicit_rk(q, 0.2, t.a, t.b, rhs))


def test_ark2_stable_and_second_order_on_split_scalar():
    t = imexcore.ark2_tableau()
    prob = ScalarProblem(-1000.0)
    q = np.array([1.0])
    for _ in range(50):
        q = imexcore.ark_imex_step(q, 1.0, t, prob, prob.linear)
        assert abs(q[0]) <= 1.0
    assert abs(q[0]) < 1e-3

    def err(dt):
        p = ScalarProblem(-0.7)
        q, s = np.array([1.0]), 0.0
        while s < 1.0 - 1e-12:
            q = imexcore.ark_imex_step(q, dt, t, p, lambda x: -x)
            s += dt
        return abs(q[0] - np.exp(-1.0))
    assert 1.8 < math.log2(err(0.1) / err(0.05)) < 2.2


def test_imex_step_nan_detection_generic():
    with pytest.raises(FloatingPointError):
        imexcore.ark_imex_step(np.array([1.0]), 0.1, imexcore.ark2_tableau(), ScalarProblem(0.0),
                               lambda q: np.full_like(q, np.inf))


# ---------------------------------------------------------------------------
# host tables against the reference (build container only)
# ---------------------------------------------------------------------------

@pytest.fixture(scope="module")
def dyc():
    import sys
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import dycore
    return dycore


@needs_reference
def test_slab_coords_and_level_tables_match_reference_bitwise(dyc):
    rmesh = dyc.specgrid.build_box_mesh(5, 4, 20_000.0, 1000.0, 4)
    rref = dyc.euler.hydrostatic_reference(rmesh, 300.0)
    mesh = specgrid.build_box_mesh(5, 4, 20_000.0, 1000.0, 4)
    ref = euler.hydrostatic_reference(mesh, 300.0)
    assert np.array_equal(mesh.coords, rmesh.coords)
    sp = dyc.columnsolve.unique_space(rmesh)
    us = columnsolve.unique_space(mesh)
    assert np.array_equal(us.uid, sp.uid) and np.array_equal(us.rep, sp.rep)
    lev = rmesh.lev_id.ravel()
    _, first = np.unique(lev, return_index=True)
    for name, mine in (("rho0", ref.rho0), ("theta0", ref.theta0), ("P0f", ref.P0f),
                       ("G0_nc", ref.G0_nc), ("H0_nc", ref.H0_nc)):
        theirs = getattr(rref, name).ravel()[first]
        assert np.array_equal(mine, theirs), name
    theirs = rref.grad_rho0[..., 2].ravel()[first]
    assert np.array_equal(ref.drho0, theirs)


@needs_reference
def test_isothermal_tables_match_reference_bitwise(dyc):
    rmesh = dyc.specgrid.build_box_mesh(3, 3, 9_000.0, 3000.0, 3)
    rref = dyc.euler.isothermal_reference(rmesh, 280.0)
    ref = euler.isothermal_reference(specgrid.build_box_mesh(3, 3, 9_000.0, 3000.0, 3), 280.0)
    _, first = np.unique(rmesh.lev_id.ravel(), return_index=True)
    assert np.array_equal(ref.theta0, rref.theta0.ravel()[first])
    assert np.array_equal(ref.dtheta0, rref.grad_theta0[..., 2].ravel()[first])
    assert np.array_equal(ref.F0z_nc, rref.F0vec_nc[..., 2].ravel()[first])


@needs_reference
def test_axis_factors_match_reference_metrics(dyc):
    """c[g] equals the DSS average of the per-copy metric factor a_r_x =
    1/(dx/dr) weighted by wJ (specgrid.py:404-430, 523-540)."""
    rmesh = dyc.specgrid.build_box_mesh(5, 4, 20_000.0, 1000.0, 4)
    disc = dyc.euler.build_discretization(rmesh)
    mesh = specgrid.build_box_mesh(5, 4, 20_000.0, 1000.0, 4)
    mine = euler.build_discretization(mesh)
    m = disc.metrics
    # DSS of (wJ a) / DSS of wJ == c with the lattice convention
    num = np.bincount(disc.dss.gid, weights=(m.wJ * m.a_r[..., 0]).ravel())
    den = np.bincount(disc.dss.gid, weights=m.wJ.ravel())
    c_ref = (num / den)[disc.dss.gid].reshape(rmesh.nshape)
    # the derivative sum at a face carries each copy's raw d/dr, so the
    # folded coefficient is half the mass-weighted average on faces
    x = mesh.lattice_coords()[0]
    gx = np.searchsorted(x, rmesh.coords[..., 0].ravel()).reshape(rmesh.nshape)
    face = (gx % 4 == 0) & (gx > 0) & (gx < mesh.X - 1)
    want = np.where(face, 0.5 * c_ref, c_ref)
    assert np.allclose(mine.cx[gx], want, rtol=1e-14, atol=0)


def test_lattice_coordinates_are_first_occurrence_copies():
    from oracle.hevi_oracle import BoxOracle
    mesh = specgrid.build_box_mesh_3d(3, 2, 3, 12_000.0, 8_000.0, 300.0, 3)
    o = BoxOracle(3, 2, 3, 12_000.0, 8_000.0, 300.0, 3)
    x, y, z = mesh.lattice_coords()
    c = o.coords.reshape(-1, 3)[o.grep]
    X, Y, Z = mesh.X, mesh.Y, mesh.Z
    c = c.reshape(Z, Y, X, 3)
    assert np.array_equal(c[0, 0, :, 0], x)
    assert np.array_equal(c[0, :, 0, 1], y)
    assert np.array_equal(c[:, 0, 0, 2], z)
    assert np.array_equal(mesh.coords, o.coords)


def test_min_node_spacing_matches_oracle():
    from oracle.hevi_oracle import BoxOracle
    mesh = specgrid.build_box_mesh_3d(3, 2, 3, 12_000.0, 8_000.0, 300.0, 4)
    o = BoxOracle(3, 2, 3, 12_000.0, 8_000.0, 300.0, 4)
    assert mesh.min_node_spacing() == pytest.approx(o.min_node_spacing(), rel=1e-15)


# ---------------------------------------------------------------------------
# partition geometry
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_partition_covers_the_lattice_once(world):
    mesh = specgrid.build_box_mesh_3d(8, 6, 2, 32_000.0, 24_000.0, 200.0, 4)
    px, py = dd.grid_for(world)
    owned = np.zeros((mesh.Y, mesh.X), dtype=int)
    for r in range(world):
        st = dd.make_block(mesh, px, py, r)
        x0 = st.ex[0] * mesh.N
        x1 = st.ex[1] * mesh.N + (1 if st.ex[1] == mesh.nx else 0)
        y0 = st.ey[0] * mesh.Ny
        y1 = st.ey[1] * mesh.Ny + (1 if st.ey[1] == mesh.ny else 0)
        owned[y0:y1, x0:x1] += 1
        w = st.window
        assert w["x0"] <= max(0, x0 - mesh.N) and w["x0"] + w["lX"] >= min(mesh.X, x1 + 1)
    assert (owned == 1).all()


@pytest.mark.parametrize("world", [2, 4, 8])
def test_halo_plan_is_symmetric(world):
    mesh = specgrid.build_box_mesh_3d(8, 6, 2, 32_000.0, 24_000.0, 200.0, 4)
    px, py = dd.grid_for(world)
    plans = [dd.halo_plan(mesh, px, py, r)[1] for r in range(world)]
    for r in range(world):
        for ph, phase in enumerate(plans[r]):
            for peer, sreg, rreg in phase:
                back = [t for t in plans[peer][ph] if t[0] == r]
                assert len(back) == 1
                assert back[0][1] == rreg and back[0][2] == sreg


def test_rk35_butcher_order_conditions():
    """test_imexcore.py:43-50."""
    a, b, c = imexcore.rk35_butcher()
    assert abs(b.sum() - 1.0) < 1e-13
    assert abs(b @ c - 0.5) < 1e-13
    assert abs(b @ c ** 2 - 1.0 / 3.0) < 1e-13
    assert abs(b @ (a @ c) - 1.0 / 6.0) < 1e-13


def test_rk35_generic_third_order_and_nan():
    def err(dt):
        q, t = np.array([1.0]), 0.0
        while t < 1.0 - 1e-12:
            q = imexcore.rk35_step(q, dt, lambda x: -x)
            t += dt
        return abs(q[0] - np.exp(-1.0))
    assert 2.7 < math.log2(err(0.1) / err(0.05)) < 3.3
    with pytest.raises(FloatingPointError):
        imexcore.rk35_step(np.array([1.0]), 1.0, lambda x: x * np.nan)


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "straka100"])
def test_baseline_inputs_match_reference(name):
    """The bench's synthetic inputs at the BASELINE configs are the
    reference's: bubble IC (bench.py:108-124, harness 3D extension) and the
    Courant dt rule (cli.py:187-194), against tests/golden/<name>.npz."""
    import torch
    from test_gpu_baseline_parity import BASE, build
    from paper_1702_04316_b200 import cases
    from conftest import load_golden
    mesh, ref, disc = build(name)
    g = load_golden(name)
    b = BASE[name]
    q0 = cases.bubble_lattice(mesh, ref, *b["bubble"], device="cpu")
    want = g["step_q0"]
    assert np.abs(q0.numpy() - want).max() <= 1e-14 * max(np.abs(want).max(), 1.0)
    dt = cases.dt_for_courant(mesh, ref, q0, b["C"])
    assert dt == pytest.approx(float(g["step_dt"]), rel=1e-12)
    assert torch.isfinite(q0).all()


def test_rounding_floor_file_covers_the_baseline_goldens():
    """tests/golden/floor.json (make_baseline_golden.py) holds the reference's
    same-host rounding floor for every kept step of every baseline golden."""
    import json
    from conftest import GOLDEN, load_golden
    fl = json.load(open(os.path.join(GOLDEN, "floor.json")))
    for name in ("cfg1", "cfg2", "straka100"):
        g = load_golden(name)
        keep = sorted(int(k[6:]) for k in g.files if k.startswith("step_q") and k != "step_q0")
        for k in keep:
            f = fl[name][str(k)]
            assert 0.0 < f["vel"] < 1e-6 and f["rho"] < 1e-9 and f["theta"] < 1e-12, (name, k, f)


# --- reference test_imexcore.py:93-158, 368-374: the stepper's duck-typed
# problem protocol (a scalar problem solved exactly, no device operators) ---
class ScalarProblem:
    """q' = k q treated implicitly; exact scalar solve (test_imexcore.py:93-106)."""

    def __init__(self, k_lin):
        self.k = k_lin
        self.lam = 0.0

    def linear(self, q):
        return np.zeros_like(q) if self.k == 0.0 else self.k * q

    def solve(self, q_e):
        return q_e / (1.0 - self.lam * self.k)


def _explicit_rk(q, dt, a, b, rhs):
    k = []
    for i in range(len(b)):
        qi = q.copy()
        for j in range(i):
            qi = qi + dt * a[i, j] * k[j]
        k.append(rhs(qi))
    out = q.copy()
    for i in range(len(b)):
        out = out + dt * b[i] * k[i]
    return out


def test_ark2_reduces_to_explicit_rk_when_linear_zero():
    t = imexcore.ark2_tableau()
    rhs = lambda q: np.sin(q) - 0.3 * q  # noqa: E731
    q = np.array([0.7])
    got = imexcore.ark_imex_step(q, 0.2, t, ScalarProblem(0.0), rhs)
    assert np.array_equal(got, _explicit_rk(q, 0.2, np.asarray(t.a), np.asarray(t.b), rhs))


def test_ark2_stable_on_stiff_linear_problem():
    t = imexcore.ark2_tableau()
    prob = ScalarProblem(-1000.0)
    q = np.array([1.0])
    for _ in range(50):
        q = imexcore.ark_imex_step(q, 1.0, t, prob, lambda x: prob.linear(x))
        assert np.all(np.isfinite(q)) and abs(q[0]) <= 1.0
    assert abs(q[0]) < 1e-3


def test_ark2_second_order_on_split_scalar():
    t = imexcore.ark2_tableau()

    def err(dt):
        prob = ScalarProblem(-0.7)
        q = np.array([1.0])
        s = 0.0
        while s < 1.0 - 1e-12:
            q = imexcore.ark_imex_step(q, dt, t, prob, lambda x: -x)
            s += dt
        return abs(q[0] - np.exp(-1.0))
    assert 1.8 < np.log2(err(0.1) / err(0.05)) < 2.2


def test_imex_step_nan_detection():
    with pytest.raises(FloatingPointError):
        imexcore.ark_imex_step(np.array([1.0]), 0.1, imexcore.ark2_tableau(), ScalarProblem(0.0),
                               lambda q: np.full_like(q, np.inf))


def test_box_boundary_projectors_match_reference_semantics():
    """euler.boundary_projectors (euler.py:218-258) on the slab: x faces, the
    dummy y layer and the bottom/top lose their normal components; a corner
    node loses all of them; interior nodes are not listed."""
    mesh = specgrid.build_box_mesh(3, 2, 1000.0, 500.0, 2)
    bidx, bproj = euler.boundary_projectors(mesh)
    assert bproj.shape == (bidx.size, 3, 3)
    d = np.diagonal(bproj, axis1=1, axis2=2)
    assert np.all(d[:, 1] == 0.0)            # the slab's y faces bound every node
    assert bidx.size == mesh.n_nodes          # so every node is a boundary node
    m3 = specgrid.build_box_mesh_3d(2, 2, 2, 1.0, 1.0, 1.0, 2)
    bidx3, bproj3 = euler.boundary_projectors(m3)
    nel, nt, ns, nr = m3.nshape
    interior = (np.arange(m3.n_nodes).reshape(m3.nshape)[0, 1, 1, 1])
    assert interior not in set(bidx3.tolist())
