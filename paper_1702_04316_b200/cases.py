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


# ---------------------------------------------------------------------------
# acoustic wave on the cubed-sphere shell (bench.py:23-105, cli.py:131-141)
# ---------------------------------------------------------------------------

class AcousticWaveConfig:
    """bench.AcousticWaveConfig (bench.py:23-45): a cosine-bell pressure pulse
    of amplitude dP with n_v vertical half-waves, centred at (lon0, lat0),
    radius r_c on a shell [r_e, r_e + r_T]."""

    def __init__(self, dP=100.0, n_v=1, r_e=6_371_000.0, r_T=10_000.0, r_c=None, lon0=0.0, lat0=0.0,
                 theta0=300.0):
        self.dP, self.n_v, self.r_e, self.r_T = dP, n_v, r_e, r_T
        self.r_c = r_e / 3.0 if r_c is None else r_c
        self.lon0, self.lat0, self.theta0 = lon0, lat0, theta0
        if self.r_c > math.pi * self.r_e:
            raise ValueError("perturbation radius exceeds the antipode")
        if self.r_T <= 0:
            raise ValueError("shell thickness must be positive")


def init_acoustic_wave(cfg: AcousticWaveConfig, mesh, ref, set_name="set2nc", balance=True):
    """bench.init_acoustic_wave (bench.py:78-120): P' = f(lon, lat) g(h), the
    pulse put in hydrostatic balance (rho' = -(dP'/dh)/g, theta' from the
    linearised EOS) or, with balance=False, pure density.  E-vector (numpy)."""
    import numpy as np
    from . import euler
    c = mesh.coords
    rad = np.linalg.norm(c, axis=-1)
    lon = np.arctan2(c[..., 1], c[..., 0])
    lat = np.arcsin(np.clip(c[..., 2] / rad, -1, 1))
    cosang = math.sin(cfg.lat0) * np.sin(lat) + math.cos(cfg.lat0) * np.cos(lat) * np.cos(lon - cfg.lon0)
    dist = cfg.r_e * np.arccos(np.clip(cosang, -1.0, 1.0))
    f = np.where(dist <= cfg.r_c, 0.5 * cfg.dP * (1.0 + np.cos(np.pi * dist / cfg.r_c)), 0.0)
    m = cfg.n_v * np.pi / cfg.r_T
    Pp = f * np.sin(m * mesh.height)
    q = np.zeros((5,) + tuple(mesh.nshape))
    if balance:
        rho_p = -f * m * np.cos(m * mesh.height) / euler.GasConstants().g
        th_p = (Pp - ref.G0_nc * rho_p) / ref.H0_nc
    else:
        rho_p = Pp / ref.G0_nc
        th_p = np.zeros_like(rho_p)
    q[0] = rho_p
    q[4] = ref.theta0 * rho_p + ref.rho0 * th_p if set_name == "set2c" else th_p
    return q


def probe_point_on_sphere(cfg: AcousticWaveConfig, angle_rad: float, height: float):
    """bench.probe_point_on_sphere (bench.py:177-185): great-circle angle east
    of the source at a height above r_e."""
    lon = cfg.lon0 + angle_rad
    r = cfg.r_e + height
    return (r * math.cos(cfg.lat0) * math.cos(lon), r * math.cos(cfg.lat0) * math.sin(lon),
            r * math.sin(cfg.lat0))


def nearest_node(mesh, point) -> int:
    """bench.nearest_node (bench.py:171-174): flat node index nearest a point."""
    import numpy as np
    d = np.linalg.norm(mesh.coords.reshape(-1, 3) - np.asarray(point), axis=1)
    return int(np.argmin(d))
