"""Parity at the BASELINE.json configurations as stated (SURVEY 8(c) gate B,
8(d) configs 1-3), against trajectories of the unmodified reference
(tests/golden/make_baseline_golden.py):

  cfg1       3D 10x10x10 N=4, 40 x 40 x 1 km, C = 15, 10 ARK2 steps
  cfg2       same grid at 400 km, C = 150, 10 steps
  straka100  inviscid Straka density current (slab 32x4 N=7), C = 0.7, 100 steps

Gate, per kept step, relative L2: rho', theta' <= 1e-10; velocity (as a
vector) <= 10x the reference's own rounding floor on the golden host
(tests/golden/floor.json: the reference re-run with EOS pow as exp(g log x)
and reverse-order DSS sums).
The resident stepper (CUDA graph, chained P' plane) and the drop-in
``imexcore.ark_imex_step`` (E-vector, reference call signature) are both
checked; cfg1 is also compared with the cancellation-free oracle.
"""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, load_golden, rel_fields

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_1702_04316_b200 import specgrid, euler, imexcore, cases  # noqa: E402
from paper_1702_04316_b200.stepper import HeviStepper  # noqa: E402

SCALAR_TOL = 1e-10
FLOOR_FACTOR = 10.0
BASE = {
    "cfg1": dict(box=(10, 10, 10, 40_000.0, 40_000.0, 1_000.0, 4), C=15.0,
                 bubble=(0.5, (20_000.0, 20_000.0, 350.0), (250.0, 250.0, 250.0))),
    "cfg2": dict(box=(10, 10, 10, 400_000.0, 400_000.0, 1_000.0, 4), C=150.0,
                 bubble=(0.5, (200_000.0, 200_000.0, 350.0), (2_500.0, 2_500.0, 250.0))),
    "straka100": dict(slab=(32, 4, 51_200.0, 6_400.0, 7), C=0.7,
                      bubble=(-15.0, (25_600.0, 0.0, 3_000.0), (4_000.0, 1.0, 2_000.0))),
}


def floors():
    with open(os.path.join(GOLDEN, "floor.json")) as f:
        return json.load(f)


def build(name):
    b = BASE[name]
    if "box" in b:
        mesh = specgrid.build_box_mesh_3d(*b["box"])
    else:
        mesh = specgrid.build_box_mesh(*b["slab"])
    ref = euler.hydrostatic_reference(mesh, 300.0)
    return mesh, ref, euler.build_discretization(mesh)


def gate(name, k, got, want):
    e_rho, e_vel, e_th = rel_fields(got, want)
    vtol = FLOOR_FACTOR * floors()[name][str(k)]["vel"]
    assert e_rho <= SCALAR_TOL and e_th <= SCALAR_TOL, (name, k, e_rho, e_th)
    assert e_vel <= vtol, (name, k, e_vel, vtol)
    return e_rho, e_vel, e_th


@pytest.mark.parametrize("name", sorted(BASE))
def test_resident_stepper_matches_reference(name):
    mesh, ref, disc = build(name)
    g = load_golden(name)
    dt = float(g["step_dt"])
    st = HeviStepper(disc, ref, dt)
    st.set_state(torch.as_tensor(g["step_q0"], device="cuda"), lattice=True)
    keep = sorted(int(k[6:]) for k in g.files if k.startswith("step_q") and k != "step_q0")
    st.capture()     # one (counted) warm step, then graph replays
    done = 1
    report = []
    if 1 in keep:
        report.append((1, gate(name, 1, st.state(lattice=True).cpu().numpy(), g["step_q1"])))
    for k in keep:
        if k <= done:
            continue
        st.step(k - done)
        done = k
        report.append((k, gate(name, k, st.state(lattice=True).cpu().numpy(), g[f"step_q{k}"])))
    print("baseline parity", name, report)


@pytest.mark.parametrize("name", ["cfg1", "cfg2"])
def test_drop_in_step_matches_reference(name):
    """imexcore.ark_imex_step on the reference E-vector layout, first step."""
    mesh, ref, disc = build(name)
    g = load_golden(name)
    dt = float(g["step_dt"])
    plan = disc.plan_for(ref)
    E = plan.l2e(plan.padded(torch.as_tensor(g["step_q0"], device="cuda")))
    prob = imexcore.ImplicitProblem(disc=disc, ref=ref, set_name="set2nc", dim="1d",
                                    solver=imexcore.SolverSpec(method="direct"))
    out = imexcore.ark_imex_step(E, dt, imexcore.ark2_tableau(), prob,
                                 euler.make_rhs(ref, disc, "set2nc"))
    got = plan.e2l(out)[..., :mesh.X].cpu().numpy()
    gate(name, 1, got, g["step_q1"])
    assert prob.stats.solves == 2


def test_cfg1_against_cancellation_free_oracle():
    """Kernel arithmetic at full config-1 size: 10 steps against the oracle
    whose P' carries no cancellation (the reference's EOS floor removed)."""
    from oracle.hevi_oracle import BoxOracle
    mesh, ref, disc = build("cfg1")
    g = load_golden("cfg1")
    dt = float(g["step_dt"])
    o = BoxOracle(10, 10, 10, 40_000.0, 40_000.0, 1_000.0, 4, pprime="exact")
    st = HeviStepper(disc, ref, dt)
    st.set_state(torch.as_tensor(g["step_q0"], device="cuda"), lattice=True)
    qx = o.from_lattice(g["step_q0"])
    errs = []
    for k in range(1, 11):
        st.step(1)
        qx = o.step(qx, dt)
        if k in (1, 10):
            errs.append(rel_fields(st.state(lattice=True).cpu().numpy(), o.to_lattice(qx)))
    print("cfg1 exact-oracle", errs)
    for e in errs:
        assert max(e) < 2e-12, errs
