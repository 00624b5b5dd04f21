"""Synthetic benchmark inputs on the unique lattice (host/device set-up).

Rising thermal bubble (bench.py:108-124; the reference's 2D radius extended
to the ellipsoid SURVEY 8(d) uses for the 3D configs) and the inviscid
Straka density current, both with P' = 0, plus the
Courant-number time-step rule of cli.run_simulation (cli.py:187-194).
"""
from __future__ import annotations

import math



def bubble_lattice(mesh, ref, theta_c=0.5, centre=None, radii=(250.0, 250.0, 250.0),
                   device="cuda", set_name="set2nc"):
    """(5, Z, Y, X) fp64 tensor: cosine theta' bump, rho' for zero P'.
    set2c: Theta' = 0 (rho theta unchanged, so P' = 0), as bench.py:118-123."""
    import torch
    if centre is None:
        centre = (0.5 * mesh.Lx, 0.5 * mesh.Ly, 350.0)
    x, y, z = [torch.as_tensor(a, dtype=torch.float64, device=device) for a in mesh.lattice_coords()]
    rr = ((x[None, None, :] - centre[0]) / radii[0]) ** 2 + ((z[:, None, None] - centre[2]) / radii[2]) ** 2
    if not mesh.slab:
        rr = rr + ((y[None, :, None] - centre[1]) / radii[1]) ** 2
    r = torch.sqrt(rr).expand(mesh.Z, mesh.Y, mesh.X)
    th = torch.where(r <= 1.0, 0.5 * theta_c * (1.0 + torch.cos(math.pi * r)), torch.zeros_like(r))
    rho0 = torch.as_tensor(ref.rho0, device=device)[:, None, None]
    theta0 = torch.as_tensor(ref.theta0, device=device)[:, None, None]
    q = torch.zeros((5, mesh.Z, mesh.Y, mesh.X), dtype=torch.float64, device=device)
    q[0] = rho0 * (theta0 / (theta0 + th) - 1.0)
    if set_name != "set2c":
        q[4] = th
    return q


def straka_lattice(mesh, ref, device="cuda"):
    """Inviscid Straka cold bubble: theta_c = -15 K, radii 4 km x 2 km,
    centre (Lx/2, 3 km)."""
    return bubble_lattice(mesh, ref, theta_c=-15.0, centre=(0.5 * mesh.Lx, 0.5 * mesh.Ly, 3000.0),
                          radii=(4000.0, 4000.0, 2000.0), device=device)


def dt_for_courant(mesh, ref, q, courant, set_name="set2nc"):
    """dt = C dx_v / max(|u| + c_s) (cli.py:187-194, euler.py:564-580)."""
    import torch
    c = ref.const
    rho0 = torch.as_tensor(ref.rho0, device=q.device)[:, None, None]
    theta0 = torch.as_tensor(ref.theta0, device=q.device)[:, None, None]
    rho = rho0 + q[0]
    if set_name == "set2c":     # momentum and Theta' (euler.py:572-574)
        vel = q[1:4] / rho
        theta = (torch.as_tensor(ref.Theta0, device=q.device)[:, None, None] + q[4]) / rho
    else:
        vel = q[1:4]
        theta = theta0 + q[4]
    P = c.P0 * (rho * c.R * theta / c.P0) ** c.gamma
    speed = torch.sqrt(vel[0] ** 2 + vel[1] ** 2 + vel[2] ** 2) + torch.sqrt(c.gamma * P / rho)
    cmax = float(speed.max())
    _, dx_v = mesh.min_node_spacing()
    return courant * dx_v / cmax
