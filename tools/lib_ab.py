"""Bitwise A/B of two builds of the library (GPU only): run a fixed sequence
of stages, solves, steps and R evaluations with the library named by
HEVI_LIB and save every output; compare two such files.

    HEVI_LIB=... python tools/lib_ab.py run out_a.npz
    HEVI_LIB=... python tools/lib_ab.py run out_b.npz
    python tools/lib_ab.py cmp out_a.npz out_b.npz
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def run(path):
    import torch
    from paper_1702_04316_b200 import specgrid, euler, imexcore, cases
    from paper_1702_04316_b200.plan import tableau_array
    out = {}
    shapes = [("box", (9, 7, 3)), ("box2", (5, 4, 2))]
    for sn in ("set2nc", "set2c"):
        for tag, (nx, ny, nz) in shapes:
            N = 4
            mesh = specgrid.build_box_mesh_3d(nx, ny, nz, 4000.0 * nx, 4000.0 * ny, 100.0 * nz, N)
            ref = euler.hydrostatic_reference(mesh, 300.0)
            disc = euler.build_discretization(mesh)
            p = disc.plan_for(ref, sn)
            q0 = cases.bubble_lattice(mesh, ref, 0.5, (2000.0 * nx, 2000.0 * ny, 35.0 * nz),
                                      (1200.0 * nx, 1500.0 * ny, 25.0 * nz), set_name=sn)
            g = torch.Generator(device="cuda").manual_seed(1)
            q0[1:4] += 0.3 * torch.rand(q0[1:4].shape, generator=g, device="cuda", dtype=torch.float64)
            dt = cases.dt_for_courant(mesh, ref, q0, 15.0, sn)
            tab = tableau_array(imexcore.ark2_tableau())
            lam = imexcore.ark2_tableau().diag * dt
            p.factor(lam)
            Q = p.padded(q0.clone())
            W = p.workspace()
            key = f"{sn}_{tag}"
            X = mesh.X   # pad columns beyond the lattice are not compared
            p.stage(0, dt, tab, Q, W)
            p.stage_solve(0, lam, W)
            out[key + "_s0"] = W[..., :X].detach().cpu().numpy().copy()
            p.stage(1, dt, tab, Q, W)
            p.stage_solve(1, lam, W)
            out[key + "_s1"] = W[..., :X].detach().cpu().numpy().copy()
            p.stage(2, dt, tab, Q, W)
            out[key + "_q"] = Q[..., :X].detach().cpu().numpy().copy()
            for _ in range(3):
                p.step(dt, tab, Q, W)
            p.check_flags()
            out[key + "_q3"] = Q[..., :X].detach().cpu().numpy().copy()
            R = p.zeros()
            p.rhs(p.padded(q0.clone()), R)
            out[key + "_rhs"] = R[..., :X].detach().cpu().numpy().copy()
    np.savez(path, **out)
    print("saved", path, len(out))


def cmp(a, b):
    A, B = np.load(a), np.load(b)
    worst = 0
    for k in A.files:
        x, y = A[k], B[k]
        fin = np.isfinite(x) & np.isfinite(y)
        same = np.array_equal(x[fin], y[fin]) and np.array_equal(np.isfinite(x), np.isfinite(y))
        d = float(np.max(np.abs(x[fin] - y[fin]))) if fin.any() else 0.0
        worst = max(worst, d)
        where = ""
        if not same:
            dd = np.where(fin, np.abs(x - y), np.inf)
            idx = np.argwhere(dd != 0)
            where = f" n={len(idx)} first={tuple(idx[0])} last={tuple(idx[-1])} shape={x.shape}"
        print(f"{k:24s} {'bitwise' if same else 'DIFF'} max|d| {d:.3e}{where}")
    print("worst", worst)


if __name__ == "__main__":
    if sys.argv[1] == "run":
        run(sys.argv[2])
    else:
        cmp(sys.argv[2], sys.argv[3])
