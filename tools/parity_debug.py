import sys, numpy as np, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from conftest import rel_fields
from paper_1702_04316_b200 import specgrid, euler
from oracle.hevi_oracle import BoxOracle
import subprocess
N = int(sys.argv[1]); slab = sys.argv[2] == "slab"; bg = sys.argv[3]
if slab:
    mesh = specgrid.build_box_mesh(6, 3, 6000.0*6, 300.0*3, N); o = BoxOracle(6, 1, 3, 36000.0, None, 900.0, N, slab=True, background=bg)
else:
    mesh = specgrid.build_box_mesh_3d(3, 2, 3, 12000., 8000., 300., N); o = BoxOracle(3, 2, 3, 12000., 8000., 300., N, background=bg)
ref = euler.hydrostatic_reference(mesh, 300.0) if bg == "hydrostatic" else euler.isothermal_reference(mesh, 300.0)
disc = euler.build_discretization(mesh)
q = o.bubble(0.5, (mesh.Lx/2, mesh.Ly/2, 150.0), (3000., 3000., 80.))
rng = np.random.default_rng(0); q = q + 1e-3*o.dss_many(rng.standard_normal(q.shape))
try:
    R = euler.nonlinear_rhs(torch.as_tensor(q, device='cuda'), ref, disc, "set2nc").cpu().numpy()
    print(N, slab, bg, "R", ["%.1e" % e for e in rel_fields(o.to_lattice(R), o.to_lattice(o.rhs(q)))], flush=True)
except Exception as e:
    print(N, slab, bg, "FAILED", str(e)[:80], flush=True)
