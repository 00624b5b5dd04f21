"""R of the column-sweep kernels vs the round-1 kernels on a random
DSS-continuous state with non-zero values on every wall (GPU)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1702_04316_b200 import specgrid, euler, imexcore  # noqa: E402
from paper_1702_04316_b200.plan import tableau_array  # noqa: E402


def plan_with(kernels, disc, ref, sn):
    if kernels:
        os.environ["HEVI_KERNELS"] = kernels
    else:
        os.environ.pop("HEVI_KERNELS", None)
    disc._plans = {}
    p = disc.plan_for(ref, sn)
    os.environ.pop("HEVI_KERNELS", None)
    return p


mesh = specgrid.build_box_mesh_3d(5, 6, 3, 20_000.0, 24_000.0, 300.0, 4)
ref = euler.hydrostatic_reference(mesh, 300.0)
disc = euler.build_discretization(mesh)
rng = np.random.default_rng(5)
for sn in ("set2nc", "set2c"):
    q = 1e-3 * rng.standard_normal((5, mesh.Z, mesh.Y, mesh.X)) * np.array(
        [1.0, 1, 1, 1, 300.0])[:, None, None, None]
    q = torch.as_tensor(q, device="cuda")
    tab = tableau_array(imexcore.ark2_tableau())
    outs = {}
    for name, k in (("v2", "v2"), ("col", None)):
        p = plan_with(k, disc, ref, sn)
        Q = p.padded(q.clone())
        W = p.workspace()
        p.factor(0.1)
        p.stage(0, 0.1, tab, Q, W)          # F = q + dt b0 R
        F = W[2][..., :mesh.X].clone()
        R = p.zeros()
        p.rhs(p.padded(q.clone()), R)
        torch.cuda.synchronize()
        outs[name] = ((F - q) / (0.1 * imexcore.ark2_tableau().b[0]), R[..., :mesh.X].clone())
    for i, lab in enumerate(("stage0 R", "rhs R")):
        a, b = outs["col"][i], outs["v2"][i]
        err = [float((a[f] - b[f]).norm() / b[f].norm()) for f in range(5)]
        d = (a - b).abs().amax(dim=(0, 1))
        bad = torch.nonzero(d > 1e-9 * float(b.abs().max()))
        print(sn, lab, " ".join(f"{e:.1e}" for e in err), "bad (y,x):", bad[:6].tolist())
