"""Throughput of the cubed-sphere (general-mesh) path: the acoustic case of
the reference driver (cli.py:131-141) at a larger shell, ARK2 1D-IMEX direct
with per-column factors, device-resident E-vector state, CUDA-event timing.
Not the headline bench (BASELINE's configs are boxes); evidence that the
general path runs at scale.  GPU only.

    python tools/sphere_bench.py [ne_panel ne_vert N] [--steps K] [--set set2nc|set2c]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np
    import torch
    from paper_1702_04316_b200 import specgrid as sg, euler, imexcore, cases
    from paper_1702_04316_b200.plan import tableau_array
    ap = argparse.ArgumentParser()
    ap.add_argument("shape", nargs="*", type=int, default=[32, 8, 4])
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--set", default="set2nc")
    ap.add_argument("--courant", type=float, default=5.0)
    a = ap.parse_args()
    ne_p, ne_v, N = a.shape
    acfg = cases.AcousticWaveConfig()
    t0 = time.perf_counter()
    mesh = sg.build_cubed_sphere_mesh(ne_p, ne_v, acfg.r_e, acfg.r_T, N)
    ref = euler.isothermal_reference(mesh, 300.0)
    disc = euler.build_discretization(mesh)
    q0 = cases.init_acoustic_wave(acfg, mesh, ref, a.set)
    plan = disc.plan_for(ref, a.set)
    setup_s = time.perf_counter() - t0
    Q = plan.dss(torch.as_tensor(q0, device="cuda"))
    work = plan.workspace()
    dx_h, dx_v = euler.min_node_spacing(mesh)
    _, cv0 = euler.courant_numbers(Q, ref, disc, 1.0, a.set)
    dt = a.courant / cv0
    tab = imexcore.ark2_tableau()
    tarr = tableau_array(tab)
    torch.cuda.synchronize()
    tf = time.perf_counter()
    nb, piv = plan.factor(tab.diag * dt)
    torch.cuda.synchronize()
    factor_ms = 1e3 * (time.perf_counter() - tf)
    for _ in range(a.warmup):
        plan.step(dt, tarr, Q, work)
    plan.check_flags()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(a.steps):
        plan.step(dt, tarr, Q, work)
    e1.record()
    torch.cuda.synchronize()
    plan.check_flags()
    ms = e0.elapsed_time(e1) / a.steps
    n_unique = mesh.n_col * mesh.n_lev
    out = {"metric": "unique DOF-updates/s (fp64) per 1D-IMEX ARK2 step, cubed-sphere shell",
           "value": 5 * n_unique / (ms * 1e-3), "unit": "DOF-updates/s", "ms_per_step": ms,
           "steps": a.steps, "warmup": a.warmup, "dtype": "f64", "data": "synthetic (acoustic pulse)",
           "config": {"ne_panel": ne_p, "ne_vert": ne_v, "N": N, "elements": mesh.nel,
                      "nodes": mesh.n_nodes, "columns": mesh.n_col, "levels": mesh.n_lev,
                      "unique_points": n_unique, "equation_set": a.set, "courant_v": a.courant,
                      "dt_s": dt, "bandwidth": nb, "pivoted": piv},
           "setup": {"host_mesh_metrics_s": round(setup_s, 2), "factor_ms": round(factor_ms, 2)},
           "node_dof_per_s": 5 * mesh.n_nodes / (ms * 1e-3)}
    print(json.dumps(out), flush=True)
    del np


if __name__ == "__main__":
    main()
