"""Multi-rank halo exchange of the partitioned step, on CPU with ``gloo``
(world sizes 2 and 4; the NCCL path runs the same code on GPU tensors)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1702_04316_b200 import specgrid
from paper_1702_04316_b200 import distributed as dd


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _field(mesh):
    Z, Y, X = mesh.Z, mesh.Y, mesh.X
    gz, gy, gx = np.meshgrid(np.arange(Z), np.arange(Y), np.arange(X), indexing="ij")
    base = (gz * 1e6 + gy * 1e3 + gx).astype(np.float64)
    return np.stack([base + 0.1 * f for f in range(5)])


def _worker(rank, world, port, shape_args, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mesh = specgrid.build_box_mesh_3d(*shape_args)
        px, py = dd.grid_for(world)
        ex = dd.HaloExchange(mesh, px, py, rank)
        w = ex.block.window
        glob = torch.as_tensor(_field(mesh))
        pitch = (w["lX"] + 3) // 4 * 4
        local = torch.full((5, mesh.Z, w["lY"], pitch), float("nan"), dtype=torch.float64)
        # only owned points are valid before the exchange
        ox0, ox1 = ex.block.ex[0] * mesh.N, ex.block.ex[1] * mesh.N + (ex.block.ex[1] == mesh.nx)
        oy0, oy1 = ex.block.ey[0] * mesh.Ny, ex.block.ey[1] * mesh.Ny + (ex.block.ey[1] == mesh.ny)
        local[:, :, oy0 - w["y0"]:oy1 - w["y0"], ox0 - w["x0"]:ox1 - w["x0"]] = \
            glob[:, :, oy0:oy1, ox0:ox1]
        ex(local)
        want = glob[:, :, w["y0"]:w["y0"] + w["lY"], w["x0"]:w["x0"] + w["lX"]]
        got = local[..., :w["lX"]]
        # every point an owned point's element lines reach must be filled
        need = torch.zeros_like(got[0, 0], dtype=torch.bool)
        need[oy0 - w["y0"]:oy1 - w["y0"], :] = True      # x halos on owned rows
        need[:, ox0 - w["x0"]:ox1 - w["x0"]] = True      # y halos on owned columns
        ok = bool(torch.equal(got[:, :, need], want[:, :, need]))
        results[rank] = ok
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_gloo_halo_exchange_fills_every_needed_halo(world):
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    results = mgr.dict()
    port = _free_port()
    shape = (6, 4, 2, 24_000.0, 16_000.0, 200.0, 4)
    procs = [ctx.Process(target=_worker, args=(r, world, port, shape, results)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert all(results[r] for r in range(world)), dict(results)
