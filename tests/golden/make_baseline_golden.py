"""Golden fixtures at the BASELINE.json configurations as stated, from the
UNMODIFIED reference, plus the same-host rounding-emulation floor that sets
the velocity parity gate (SURVEY.md 8(c) gate B).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_baseline_golden.py

Cases:
  cfg1       3D 10x10x10 elements N=4, 40 x 40 x 1 km, bubble theta_c = 0.5 K,
             r = 250 m, centre (20 km, 20 km, 350 m), HEVI ARK2 Schur direct,
             C = 15, 10 steps (steps 1, 5, 10 kept);
  cfg2       same grid, 400 x 400 x 1 km (C_H = 0.375 at C_V = 150), centre
             and horizontal radius scaled by 10, C = 150, 10 steps;
  straka100  inviscid Straka density current, reference slab 32 x 4 N=7,
             51.2 x 6.4 km, C = 0.7, 100 steps (1, 10, 50, 100 kept).

The floor: each case is run a second time with the reference's two
rounding-sensitive operations replaced by mathematically identical ones a GPU
implementation may use -- EOS pow evaluated as exp(gamma log x)
(euler.py:185) and the DSS scatter-add summed in reverse node order
(specgrid.py:535-540).  The per-field relative L2 distance between the two
reference runs is the reference's own rounding floor on this host; the GPU
velocity gate is 10x that floor (tests/test_gpu_baseline_parity.py).
Results: tests/golden/<case>.npz and tests/golden/floor.json.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import make_golden as mg  # noqa: E402  (imports the reference read-only)

sg, euler, imx = mg.sg, mg.euler, mg.imx

CASES = {
    "cfg1": dict(mesh=("box3d", 10, 10, 10, 40_000.0, 40_000.0, 1_000.0, 4), slab=False, N_s=4,
                 bubble=(0.5, (20_000.0, 20_000.0, 350.0), (250.0, 250.0, 250.0)),
                 C=15.0, nsteps=10, keep=(1, 5, 10)),
    "cfg2": dict(mesh=("box3d", 10, 10, 10, 400_000.0, 400_000.0, 1_000.0, 4), slab=False, N_s=4,
                 bubble=(0.5, (200_000.0, 200_000.0, 350.0), (2_500.0, 2_500.0, 250.0)),
                 C=150.0, nsteps=10, keep=(1, 5, 10)),
    "straka100": dict(mesh=("slab", 32, 4, 51_200.0, 6_400.0, 7), slab=True, N_s=1,
                      bubble=(-15.0, (25_600.0, 0.0, 3_000.0), (4_000.0, 1.0, 2_000.0)),
                      C=0.7, nsteps=100, keep=(1, 10, 50, 100)),
}


def build_mesh(spec):
    if spec[0] == "box3d":
        return mg.box3d_mesh(*spec[1:])
    mesh = sg.build_box_mesh(*spec[1:])
    mesh.meta["ny"] = 1
    return mesh


def trajectory(mesh, N_s, slab, bubble, C, nsteps, keep):
    ref = euler.hydrostatic_reference(mesh, 300.0)
    disc = euler.build_discretization(mesh)
    rep, dims, _ = mg.lattice_index(mesh, N_s)
    q = mg.bubble_state(mesh, ref, disc, *bubble, slab=slab)
    dt = mg.dt_for(mesh, ref, disc, q, C)
    out = {"step_q0": mg.to_lattice(q, rep, dims), "step_dt": np.array(dt)}
    prob = imx.ImplicitProblem(disc=disc, ref=ref, set_name="set2nc", form="schur", dim="1d",
                               solver=imx.SolverSpec(method="direct"))
    rhs = lambda s: euler.nonlinear_rhs(s, ref, disc, "set2nc")  # noqa: E731
    tab = imx.ark2_tableau()
    for k in range(1, nsteps + 1):
        q = imx.ark_imex_step(q, dt, tab, prob, rhs)
        if k in keep:
            out[f"step_q{k}"] = mg.to_lattice(q, rep, dims)
    out["solves"] = np.array(prob.stats.solves)
    return out


class Emulation:
    """EOS pow as exp(gamma log x) and reverse-order DSS sums, patched into
    the reference modules for the duration of a run."""

    def __enter__(self):
        self.eos, self.dss = euler.equation_of_state, sg.apply_dss

        def eos(rho, theta, const):
            if np.any(rho <= 0) or np.any(theta <= 0):
                raise ValueError("EOS requires positive density and temperature")
            return const.P0 * np.exp(const.gamma * np.log(rho * const.R * theta / const.P0))

        def apply_dss(f, dss):
            if f.shape != dss.shape:
                raise ValueError("field/DSS map shape mismatch")
            num = np.bincount(dss.gid[::-1], weights=(dss.w * f.ravel())[::-1], minlength=dss.n_groups)
            return (num / dss.wsum)[dss.gid].reshape(dss.shape)

        euler.equation_of_state, sg.apply_dss = eos, apply_dss
        return self

    def __exit__(self, *exc):
        euler.equation_of_state, sg.apply_dss = self.eos, self.dss


def rel_fields(a, b):
    """rho', |(u, v, w)| (vector), theta' relative L2 distances."""
    n = lambda x: float(np.linalg.norm(x))  # noqa: E731
    return {"rho": n(a[0] - b[0]) / max(n(b[0]), 1e-300),
            "vel": n(a[1:4] - b[1:4]) / max(n(b[1:4]), 1e-300),
            "theta": n(a[4] - b[4]) / max(n(b[4]), 1e-300)}


def main(names):
    floor_path = os.path.join(HERE, "floor.json")
    floors = json.load(open(floor_path)) if os.path.exists(floor_path) else {}
    for name in names:
        c = CASES[name]
        mesh = build_mesh(c["mesh"])
        args = (mesh, c["N_s"], c["slab"], c["bubble"], c["C"], c["nsteps"], c["keep"])
        plain = trajectory(*args)
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **plain)
        with Emulation():
            emu = trajectory(*args)
        floors[name] = {str(k): rel_fields(emu[f"step_q{k}"], plain[f"step_q{k}"]) for k in c["keep"]}
        print(name, "dt", float(plain["step_dt"]), "floor", json.dumps(floors[name]))
        with open(floor_path, "w") as f:
            json.dump(floors, f, indent=1)


if __name__ == "__main__":
    main([a for a in sys.argv[1:] if a in CASES] or list(CASES))
