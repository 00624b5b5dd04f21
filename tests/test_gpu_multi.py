"""The partitioned step across real processes over NCCL: two
ranks, one GPU each, HaloExchange with the library's pack/unpack kernels
and NCCL send/recv, the chained P' plane exchanged with the state.  Each
rank's owned block after two steps must be bitwise the single-GPU result.
Needs >= 2 GPUs (skipped otherwise; the CPU gloo test covers the exchange
logic, tests/test_distributed.py)."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_1702_04316_b200 import specgrid, euler, cases  # noqa: E402

NEED = 2


def _setup():
    mesh = specgrid.build_box_mesh_3d(8, 6, 3, 32_000.0, 24_000.0, 300.0, 4)
    ref = euler.hydrostatic_reference(mesh, 300.0)
    disc = euler.build_discretization(mesh)
    return mesh, ref, disc


def _rank(rank, world, port, outdir):
    import torch.distributed as dist
    from paper_1702_04316_b200 import distributed as dd
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world,
                            device_id=torch.device("cuda", rank))
    mesh, ref, disc = _setup()
    q0 = cases.bubble_lattice(mesh, ref, 0.5, (16_000.0, 12_000.0, 150.0), (6000.0, 6000.0, 100.0))
    dt = cases.dt_for_courant(mesh, ref, q0, 15.0)
    px, py = dd.grid_for(world)
    ds = dd.DistributedStepper(mesh, ref, disc, dt, px, py, rank)
    ds.load_global(q0)
    side = torch.cuda.Stream()
    ds.step()
    ds.step(side_stream=side)     # exchange beside the interior tiles
    torch.cuda.synchronize()
    ds.plan.check_flags()
    x0, x1, y0, y1 = ds.owned_region()
    np.save(os.path.join(outdir, f"rank{rank}.npy"), ds.owned()[..., :x1 - x0].cpu().numpy())
    np.save(os.path.join(outdir, f"region{rank}.npy"), np.array([x0, x1, y0, y1]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < NEED,
                    reason=f"needs >= {NEED} GPUs")
def test_nccl_partitioned_step_is_bitwise_single_gpu(tmp_path):
    import torch.multiprocessing as mp
    from paper_1702_04316_b200.stepper import HeviStepper
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    mp.spawn(_rank, args=(NEED, port, str(tmp_path)), nprocs=NEED, join=True)
    mesh, ref, disc = _setup()
    q0 = cases.bubble_lattice(mesh, ref, 0.5, (16_000.0, 12_000.0, 150.0), (6000.0, 6000.0, 100.0))
    st = HeviStepper(disc, ref, cases.dt_for_courant(mesh, ref, q0, 15.0))
    st.set_state(q0, lattice=True)
    st.step(2)
    want = st.state(lattice=True).cpu().numpy()
    for r in range(NEED):
        x0, x1, y0, y1 = np.load(tmp_path / f"region{r}.npy")
        got = np.load(tmp_path / f"rank{r}.npy")
        assert np.array_equal(got, want[:, :, y0:y1, x0:x1]), r
