"""Per-phase cycle breakdown of the explicit kernel (debug build with
-DHEVI_PHASE_TIMING, loaded via HEVI_LIB).  Usage on the GPU box:
    HEVI_LIB=$PWD/paper_1702_04316_b200/_lib/libhevi_pt.so python tools/phase_timing.py"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1702_04316_b200 import specgrid, euler, imexcore, cases, _native
from paper_1702_04316_b200.plan import tableau_array

mesh = specgrid.build_box_mesh_3d(176, 176, 10, 704_000.0, 704_000.0, 1000.0, 4)
ref = euler.hydrostatic_reference(mesh, 300.0)
disc = euler.build_discretization(mesh)
q0 = cases.bubble_lattice(mesh, ref, 0.5, (352_000.0, 352_000.0, 350.0), (10_000.0, 10_000.0, 250.0))
dt = cases.dt_for_courant(mesh, ref, q0, 15.0)
plan = disc.plan_for(ref)
tab = imexcore.ark2_tableau()
lam = tab.diag * dt
plan.factor(lam)
Q = plan.zeros()
Q[..., :mesh.X].copy_(q0)
W = plan.workspace()
tarr = tableau_array(tab)
lib = _native.load()
fn = lib.hevi_debug_phase
fn.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_ulonglong)]
buf = (ctypes.c_ulonglong * 8)()
names = ["tma wait", "convert", "bar1", "xface", "bar2", "points", "bar3"]
for s in range(3):
    plan.stage(0, dt, tarr, Q, W); plan.stage_solve(0, lam, W)
    plan.stage(1, dt, tarr, Q, W); plan.stage_solve(1, lam, W)
    plan.stage(2, dt, tarr, Q, W)
torch.cuda.synchronize()
fn(plan.h, buf)
for st in range(3):
    if st == 0:
        plan.stage(0, dt, tarr, Q, W)
    elif st == 1:
        plan.stage_solve(0, lam, W); plan.stage(1, dt, tarr, Q, W)
    else:
        plan.stage_solve(1, lam, W); plan.stage(2, dt, tarr, Q, W)
    torch.cuda.synchronize()
    fn(plan.h, buf)
    v = [buf[i] for i in range(8)]
    thr = v[7]
    tot = sum(v[:7])
    print(f"stage {st}: cycles/thread/layer " + ", ".join(
        f"{n} {v[i] / thr / mesh.nz:.0f} ({100 * v[i] / tot:.1f}%)" for i, n in enumerate(names)))
