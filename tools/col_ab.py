"""A/B of the explicit_col kernels against the v2 kernels (same plan inputs):
each explicit stage and the full step, relative L2 per field.  GPU only.

    python tools/col_ab.py [nx ny nz] [set2nc|set2c]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1702_04316_b200 import specgrid, euler, imexcore, cases  # noqa: E402
from paper_1702_04316_b200.plan import tableau_array  # noqa: E402


def plan_with(kernels, disc, ref, set_name):
    if kernels:
        os.environ["HEVI_KERNELS"] = kernels
    else:
        os.environ.pop("HEVI_KERNELS", None)
    disc._plans = {}
    p = disc.plan_for(ref, set_name)
    os.environ.pop("HEVI_KERNELS", None)
    return p


def rel(a, b):
    out = []
    for f in range(5):
        n = float(torch.linalg.norm(b[f]))
        out.append(float(torch.linalg.norm(a[f] - b[f])) / max(n, 1e-300))
    return out


def main():
    nx, ny, nz = [int(v) for v in sys.argv[1:4]] if len(sys.argv) > 3 else (9, 7, 3)
    sn = sys.argv[4] if len(sys.argv) > 4 else "set2nc"
    N = 4
    mesh = specgrid.build_box_mesh_3d(nx, ny, nz, 4000.0 * nx, 4000.0 * ny, 100.0 * nz, N)
    ref = euler.hydrostatic_reference(mesh, 300.0)
    disc = euler.build_discretization(mesh)
    q0 = cases.bubble_lattice(mesh, ref, 0.5, (2000.0 * nx, 2000.0 * ny, 35.0 * nz),
                              (1200.0 * nx, 1500.0 * ny, 25.0 * nz), set_name=sn)
    if sn == "set2c":
        q0[4] += 0.2 * q0[0] * 300.0    # a Theta' perturbation as well
    g = torch.Generator(device="cuda").manual_seed(1)
    q0[1:4] += 0.3 * torch.rand(q0[1:4].shape, generator=g, device="cuda", dtype=torch.float64)
    q0[1, :, :, 0] = 0
    q0[1, :, :, -1] = 0
    q0[2, :, 0, :] = 0
    q0[2, :, -1, :] = 0
    q0[3, 0] = 0
    q0[3, -1] = 0
    dt = cases.dt_for_courant(mesh, ref, q0, 15.0, sn)
    tab = tableau_array(imexcore.ark2_tableau())
    res = {}
    for name, kern in (("v2", "v2"), ("col", None)):
        p = plan_with(kern, disc, ref, sn)
        lam = imexcore.ark2_tableau().diag * dt
        p.factor(lam)
        Q = p.padded(q0.clone())
        W = p.workspace()
        outs = []
        p.stage(0, dt, tab, Q, W)
        outs.append([W[k].clone() for k in range(4)])
        p.stage_solve(0, lam, W)
        p.stage(1, dt, tab, Q, W)
        outs.append([W[k].clone() for k in range(4)])
        p.stage_solve(1, lam, W)
        p.stage(2, dt, tab, Q, W)
        outs.append([Q.clone()])
        p.check_flags()
        Q2 = p.padded(q0.clone())
        for _ in range(3):
            p.step(dt, tab, Q2, W)
        p.check_flags()
        outs.append([Q2.clone()])
        R = p.zeros()
        p.rhs(p.padded(q0.clone()), R)
        outs.append([R.clone()])
        torch.cuda.synchronize()
        res[name] = outs
    X = mesh.X
    labels = ["stage0 [Q1 A F P]", "stage1 [Q1 A F P]", "stage2 Q", "3 steps Q", "rhs"]
    worst = 0.0
    for i, lab in enumerate(labels):
        for j, (a, b) in enumerate(zip(res["col"][i], res["v2"][i])):
            r = rel(a[..., :X], b[..., :X])
            worst = max(worst, max(r))
            print(f"{lab} buf{j}: " + " ".join(f"{v:.2e}" for v in r))
    print("worst", worst)


if __name__ == "__main__":
    main()
