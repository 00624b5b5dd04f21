"""Per-rank compute time of the column-partitioned step at config 5, one rank
at a time on one B200 (the halo exchange replaced by nothing: the kernels'
share of an N-GPU step).  With the exchange hidden beside the interior tiles,
N x (single-GPU step) / (slowest rank) bounds the strong-scaling efficiency
the partitioned kernels allow.  GPU only.

    python tools/rank_time.py [world ...]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_1702_04316_b200 import specgrid, euler, cases
    from paper_1702_04316_b200 import distributed as dd
    worlds = [int(w) for w in sys.argv[1:]] or [1, 2, 4, 8]
    mesh = specgrid.build_box_mesh_3d(176, 176, 10, 704_000.0, 704_000.0, 1000.0, 4)
    ref = euler.hydrostatic_reference(mesh, 300.0)
    disc = euler.build_discretization(mesh)
    q0 = cases.bubble_lattice(mesh, ref, 0.5, (352_000.0, 352_000.0, 350.0), (10_000.0, 10_000.0, 250.0))
    dt = cases.dt_for_courant(mesh, ref, q0, 15.0)
    out = {}
    for world in worlds:
        px, py = dd.grid_for(world)
        times = []
        for rank in range(world):
            s = dd.DistributedStepper(mesh, ref, disc, dt, px, py, rank, exchange=lambda t: None)
            s.load_global(q0)
            for _ in range(3):
                s.step()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10):
                s.step()
            e1.record()
            torch.cuda.synchronize()
            s.plan.check_flags()
            times.append(e0.elapsed_time(e1) / 10)
            del s
            torch.cuda.empty_cache()
        out[world] = {"grid": f"{px}x{py}", "rank_ms": [round(t, 4) for t in times],
                      "max_ms": round(max(times), 4)}
        print(world, json.dumps(out[world]), flush=True)
    t1 = out.get(1, {}).get("max_ms")
    if t1:
        for w, o in out.items():
            print(f"world {w}: kernel-limited efficiency {t1 / (w * o['max_ms']):.3f}")


if __name__ == "__main__":
    main()
