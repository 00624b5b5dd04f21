"""Wave tail of one explicit stage at config 5 (a rank window of an N-GPU
decomposition, timed alone on one B200): when the tiles before the last
partial wave end vs the last tile, from %globaltimer.  GPU only; needs a
timing build:

    bash tools/dev_build.sh tt -DHEVI_EDGE_TIMING
    HEVI_LIB=paper_1702_04316_b200/_lib/libhevi_tt.so python tools/tail_timing.py [world] [rank]
"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_1702_04316_b200 import specgrid, euler, cases, _native
    from paper_1702_04316_b200 import distributed as dd
    world = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    rank = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    mesh = specgrid.build_box_mesh_3d(176, 176, 10, 704_000.0, 704_000.0, 1000.0, 4)
    ref = euler.hydrostatic_reference(mesh, 300.0)
    disc = euler.build_discretization(mesh)
    q0 = cases.bubble_lattice(mesh, ref, 0.5, (352_000.0, 352_000.0, 350.0), (10_000.0, 10_000.0, 250.0))
    dt = cases.dt_for_courant(mesh, ref, q0, 15.0)
    px, py = dd.grid_for(world)
    s = dd.DistributedStepper(mesh, ref, disc, dt, px, py, rank, exchange=lambda t: None)
    s.load_global(q0)
    for _ in range(3):
        s.step()
    torch.cuda.synchronize()
    lib = _native.load()
    f = lib.hevi_debug_phase
    f.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_ulonglong)]
    buf = (ctypes.c_ulonglong * 8)()
    for st in range(3):
        s.step()
        torch.cuda.synchronize()
        f(s.plan.h, buf)
        s.plan.stage(st, s.dt, s.tab, s.Q, s.work, pp_valid=(getattr(s, 'chain', False) if st == 0 else False))
        torch.cuda.synchronize()
        f(s.plan.h, buf)
        t0 = (2**64 - 1) - buf[0]
        print(f"world {world} rank {rank} stage {st}: last tile start {(buf[1]-t0)/1e3:.1f} us, "
              f"full waves end {(buf[5]-t0)/1e3:.1f} us, sweep end {(buf[2]-t0)/1e3:.1f} us")


if __name__ == "__main__":
    main()
