"""Structured spectral-element box meshes (host-side setup).

Mirrors the parts of the reference ``dycore.specgrid`` that the HEVI path
needs, for the two box geometries the path runs on:

* ``build_box_mesh(nx, nz, Lx, Lz, N, Ly=None)`` -- same signature and node
  placement as the reference 2D slab (specgrid.py:173-231): x-z elements of
  degree N, one dummy y layer of degree 1, columns keyed by x only;
* ``build_box_mesh_3d(nx, ny, nz, Lx, Ly, Lz, N)`` -- the SURVEY.md 8(c)
  harness 3D box (degree N on all axes, element e = (kz*ny + ky)*nx + kx).

Field arrays handed to the public API use the reference E-vector layout
``(5, nel, nqt, nqs, nqr)``.  Internally the state lives on the
unique-point lattice ``(5, Z, Y, X)``; ``lattice_coords``
gives the coordinates of the lattice points, taken from the
first-occurrence element copy exactly as the reference computes them.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
from numpy.polynomial import legendre as npleg


@dataclass
class Quadrature1D:
    N: int
    nodes: np.ndarray
    weights: np.ndarray
    D: np.ndarray


def lgl_nodes_weights(N: int) -> Quadrature1D:
    """Degree-N LGL nodes/weights/derivative matrix (specgrid.py:39-77)."""
    if N < 1:
        raise ValueError("polynomial degree must be >= 1")
    basis = np.zeros(N + 1)
    basis[N] = 1.0
    if N == 1:
        x = np.array([-1.0, 1.0])
    else:
        dP = npleg.legder(basis)
        ddP = npleg.legder(dP)
        guess = np.cos(np.pi * np.arange(N - 1, 0, -1) / N)
        for _ in range(100):
            delta = npleg.legval(guess, dP) / npleg.legval(guess, ddP)
            guess = guess - delta
            if np.max(np.abs(delta)) < 1e-15:
                break
        x = np.concatenate(([-1.0], np.sort(guess), [1.0]))
    w = 2.0 / (N * (N + 1) * npleg.legval(x, basis) ** 2)
    diff = x[:, None] - x[None, :]
    np.fill_diagonal(diff, 1.0)
    bw = 1.0 / diff.prod(axis=1)
    D = (bw[None, :] / bw[:, None]) / diff
    np.fill_diagonal(D, 0.0)
    np.fill_diagonal(D, -D.sum(axis=1))
    return Quadrature1D(N=N, nodes=x, weights=w, D=D)


def _rep(g, N, ne):
    """(element, local index) of the first-occurrence copy of lattice index g."""
    g = np.asarray(g)
    face = (g > 0) & (g % N == 0)
    k = np.where(face, g // N - 1, np.minimum(g // N, ne - 1))
    return k, g - k * N


@dataclass
class BoxMesh:
    """Structured box of nx x ny x nz elements (ny = 1, Ny = 1 for the slab)."""
    kind: str
    N: int
    Ny: int
    nx: int
    ny: int
    nz: int
    Lx: float
    Ly: float
    Lz: float
    slab: bool
    quad_r: Quadrature1D
    quad_s: Quadrature1D
    quad_t: Quadrature1D
    meta: dict = field(default_factory=dict)

    # ---- sizes ---------------------------------------------------------
    @property
    def nel(self) -> int:
        return self.nx * self.ny * self.nz

    @property
    def nshape(self):
        return (self.nel, self.N + 1, self.Ny + 1, self.N + 1)

    @property
    def n_nodes(self) -> int:
        return int(np.prod(self.nshape))

    @property
    def X(self) -> int:
        return self.nx * self.N + 1

    @property
    def Y(self) -> int:
        return self.ny * self.Ny + 1

    @property
    def Z(self) -> int:
        return self.nz * self.N + 1

    @property
    def n_lev(self) -> int:
        return self.Z

    @property
    def n_col(self) -> int:
        return self.X if self.slab else self.X * self.Y

    @property
    def n_unique(self) -> int:
        return self.X * self.Y * self.Z

    # ---- element edges and node coordinates ------------------------------
    def edges(self):
        return (np.linspace(0.0, self.Lx, self.nx + 1),
                np.linspace(0.0, self.Ly, self.ny + 1),
                np.linspace(0.0, self.Lz, self.nz + 1))

    def _axis_coords(self, axis):
        """Coordinates of lattice indices along one axis, first-occurrence copy."""
        xe, ye, ze = self.edges()
        e, q, n, ne = {0: (xe, self.quad_r, self.N, self.nx),
                       1: (ye, self.quad_s, self.Ny, self.ny),
                       2: (ze, self.quad_t, self.N, self.nz)}[axis]
        G = ne * n + 1
        k, i = _rep(np.arange(G), n, ne)
        if axis == 1 and self.slab:
            return np.array([0.0, self.Ly])[i]
        out = np.empty(G)
        for kk in range(ne):
            sel = k == kk
            nodes_x = e[kk] + (q.nodes + 1.0) * 0.5 * (e[kk + 1] - e[kk])
            out[sel] = nodes_x[i[sel]]
        return out

    def lattice_coords(self):
        """(x[X], y[Y], z[Z]) coordinates of the unique lattice points."""
        return self._axis_coords(0), self._axis_coords(1), self._axis_coords(2)

    @property
    def coords(self) -> np.ndarray:
        """E-vector node coordinates (nel, nqt, nqs, nqr, 3), as the reference."""
        xe, ye, ze = self.edges()
        c = np.empty(self.nshape + (3,))
        for kz in range(self.nz):
            zs = ze[kz] + (self.quad_t.nodes + 1.0) * 0.5 * (ze[kz + 1] - ze[kz])
            for ky in range(self.ny):
                if self.slab:
                    ys = np.array([0.0, self.Ly])
                else:
                    ys = ye[ky] + (self.quad_s.nodes + 1.0) * 0.5 * (ye[ky + 1] - ye[ky])
                for kx in range(self.nx):
                    e = (kz * self.ny + ky) * self.nx + kx
                    xs = xe[kx] + (self.quad_r.nodes + 1.0) * 0.5 * (xe[kx + 1] - xe[kx])
                    c[e, ..., 0] = xs[None, None, :]
                    c[e, ..., 1] = ys[None, :, None]
                    c[e, ..., 2] = zs[:, None, None]
        return c

    @property
    def height(self) -> np.ndarray:
        return self.coords[..., 2].copy()

    # ---- DSS-averaged metric factors ("folded DSS") -------
    def axis_factor(self, axis):
        """c[g]: 1/(dx/dr) inside an element, 1/(dx/dr|left + dx/dr|right)
        on an element face -- the weight the mass-weighted DSS average
        (specgrid.py:535-540, wJ = w J) puts on the raw local derivative of
        each copy once the per-copy metric a = 1/(dx/dr) is applied."""
        xe, ye, ze = self.edges()
        e, n, ne, L = {0: (xe, self.N, self.nx, self.Lx), 1: (ye, self.Ny, self.ny, self.Ly),
                       2: (ze, self.N, self.nz, self.Lz)}[axis]
        if axis == 1 and self.slab:
            h = np.array([self.Ly])
        else:
            h = np.diff(e)
        half = 0.5 * h
        G = ne * n + 1
        g = np.arange(G)
        own = np.minimum(g // n, ne - 1)
        c = 1.0 / half[own]
        face = (g > 0) & (g % n == 0) & (g < G - 1)
        c[face] = 1.0 / (half[g[face] // n - 1] + half[g[face] // n])
        return c

    def min_node_spacing(self):
        """euler.min_node_spacing (euler.py:583-593) for the box."""
        xe, ye, ze = self.edges()

        def spacing(e, q):
            d = np.inf
            for k in range(len(e) - 1):
                xs = e[k] + (q.nodes + 1.0) * 0.5 * (e[k + 1] - e[k])
                d = min(d, float(np.abs(np.diff(xs)).min()))
            return d

        d_r = spacing(xe, self.quad_r)
        d_t = spacing(ze, self.quad_t)
        if self.slab:
            return d_r, d_t
        return min(d_r, spacing(ye, self.quad_s)), d_t


def build_box_mesh(nx: int, nz: int, Lx: float, Lz: float, N: int,
                   Ly: float | None = None) -> BoxMesh:
    """Reference 2D slab (specgrid.build_box_mesh, specgrid.py:173-231)."""
    if nx < 1 or nz < 1:
        raise ValueError("element counts must be >= 1")
    if Lx <= 0 or Lz <= 0:
        raise ValueError("extents must be positive")
    if Ly is None:
        Ly = Lx / nx
    return BoxMesh(kind="box", N=N, Ny=1, nx=nx, ny=1, nz=nz, Lx=Lx, Ly=Ly, Lz=Lz,
                   slab=True, quad_r=lgl_nodes_weights(N), quad_s=lgl_nodes_weights(1),
                   quad_t=lgl_nodes_weights(N),
                   meta={"nx": nx, "nz": nz, "Lx": Lx, "Lz": Lz, "Ly": Ly})


def build_box_mesh_3d(nx: int, ny: int, nz: int, Lx: float, Ly: float, Lz: float,
                      N: int) -> BoxMesh:
    """SURVEY 8(c) harness 3D box: degree N on all axes."""
    if min(nx, ny, nz) < 1:
        raise ValueError("element counts must be >= 1")
    if min(Lx, Ly, Lz) <= 0:
        raise ValueError("extents must be positive")
    q = lgl_nodes_weights(N)
    return BoxMesh(kind="box", N=N, Ny=N, nx=nx, ny=ny, nz=nz, Lx=Lx, Ly=Ly, Lz=Lz,
                   slab=False, quad_r=q, quad_s=q, quad_t=q,
                   meta={"nx": nx, "ny": ny, "nz": nz, "Lx": Lx, "Ly": Ly, "Lz": Lz})


# ---------------------------------------------------------------------------
# Direct stiffness summation on E-vectors (specgrid.py:512-548)
# ---------------------------------------------------------------------------
@dataclass
class BoxDss:
    """The DssMap of a box mesh (specgrid.py:512-532): the per-node mass
    weight wJ = w_r w_s w_t J factors into one table per axis (GLL weight x
    half element width), so the map is three short tables instead of an
    E-vector sized group index.  ``plan`` returns a whole-domain device plan
    of the mesh (the kernel only needs its geometry)."""
    mesh: BoxMesh
    wx: np.ndarray
    wy: np.ndarray
    wz: np.ndarray
    plan: object = None
    _dev: dict = field(default_factory=dict)

    @property
    def shape(self):
        return tuple(self.mesh.nshape)

    @property
    def n_groups(self) -> int:
        return self.mesh.n_unique

    def device_tables(self, device):
        key = str(device)
        if key not in self._dev:
            import torch
            self._dev[key] = tuple(torch.as_tensor(w, dtype=torch.float64, device=device)
                                   for w in (self.wx, self.wy, self.wz))
        return self._dev[key]


def build_dss_map(mesh: BoxMesh, plan_getter=None) -> BoxDss:
    xe, ye, ze = mesh.edges()

    def table(e, q, ne):
        h = np.diff(e) if len(e) == ne + 1 else np.full(ne, e[-1] - e[0])
        return (q.weights[None, :] * (0.5 * h)[:, None]).ravel()
    if mesh.slab:
        wy = mesh.quad_s.weights * (0.5 * mesh.Ly)
    else:
        wy = table(ye, mesh.quad_s, mesh.ny)
    return BoxDss(mesh=mesh, wx=table(xe, mesh.quad_r, mesh.nx), wy=wy,
                  wz=table(ze, mesh.quad_t, mesh.nz), plan=plan_getter)


def apply_dss_many(fields, dss: BoxDss):
    """DSS along the leading axis of stacked E-vector fields (specgrid.py:543-548):
    every coincident copy takes the mass-weighted average of all copies, on
    the device (``hevi_dss``; general meshes: ``hevi_g_dss``).  numpy in ->
    numpy out, torch in -> torch out."""
    from . import _native as nv
    from .plan import to_device
    import torch
    E, back = to_device(fields)
    if tuple(E.shape[1:]) != tuple(dss.shape):
        raise ValueError("field/DSS map shape mismatch")
    if not isinstance(dss, BoxDss):      # sphere.GroupMap
        return back(dss.disc.geometry_plan().dss(E))
    plan = dss.plan()
    out = torch.empty_like(E)
    wx, wy, wz = dss.device_tables(E.device)
    nv.check(plan.lib.hevi_dss(plan.h, nv.ptr(E), nv.ptr(out), E.shape[0], nv.ptr(wx), nv.ptr(wy),
                               nv.ptr(wz), nv.stream_ptr()))
    return back(out)


def apply_dss(f, dss: BoxDss):
    """Replace coincident-node values by their mass-weighted average (specgrid.py:535-540)."""
    if tuple(f.shape) != tuple(dss.shape):
        raise ValueError("field/DSS map shape mismatch")
    return apply_dss_many(f[None], dss)[0]


def build_cubed_sphere_mesh(ne_panel: int, ne_vert: int, r_e: float, r_T: float, N: int):
    """Equiangular gnomonic cubed-sphere shell (specgrid.py:257-306); the
    general-mesh path of ``sphere``."""
    from .sphere import build_cubed_sphere_mesh as build
    return build(ne_panel, ne_vert, r_e, r_T, N)
