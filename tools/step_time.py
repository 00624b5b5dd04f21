"""Whole-step time of the fused ARK2 step (hevi_ark2_step_ex, no events between
the launches) at config 5 for the library named by HEVI_LIB.  GPU only.

    HEVI_LIB=... python tools/step_time.py [steps]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_1702_04316_b200 import specgrid, euler, imexcore, cases
    from paper_1702_04316_b200.plan import tableau_array
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 30
    graph = "graph" in sys.argv[2:]
    mesh = specgrid.build_box_mesh_3d(176, 176, 10, 704_000.0, 704_000.0, 1000.0, 4)
    ref = euler.hydrostatic_reference(mesh, 300.0)
    disc = euler.build_discretization(mesh)
    q0 = cases.bubble_lattice(mesh, ref, 0.5, (352_000.0, 352_000.0, 350.0), (10_000.0, 10_000.0, 250.0))
    dt = cases.dt_for_courant(mesh, ref, q0, 15.0)
    p = disc.plan_for(ref, "set2nc")
    tab = imexcore.ark2_tableau()
    tarr = tableau_array(tab)
    p.factor(tab.diag * dt)
    Q = p.padded(q0)
    W = p.workspace()
    p.pp_refresh(Q, W)
    for _ in range(5):
        p.step(dt, tarr, Q, W, pp_valid=True)
    p.check_flags()
    g = None
    if graph:   # one step captured as a CUDA graph, replayed
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            p.step(dt, tarr, Q, W, pp_valid=True)
    out = []
    for rep in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(steps):
            if g is not None:
                g.replay()
            else:
                p.step(dt, tarr, Q, W, pp_valid=True)
        e1.record()
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1) / steps)
    p.check_flags()
    print(os.environ.get("HEVI_LIB", "libhevi.so"), "graph" if graph else "eager", " ".join(f"{v:.4f}" for v in out), "ms/step")


if __name__ == "__main__":
    main()
