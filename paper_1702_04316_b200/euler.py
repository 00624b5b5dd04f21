"""Compressible Euler operators of the HEVI path (drop-in for ``dycore.euler``).

Same entry points and argument meaning as the reference
(/root/reference/pkg/src/dycore/euler.py): ``GasConstants``,
``hydrostatic_reference``, ``isothermal_reference``, ``build_discretization``,
``nonlinear_rhs``, ``vertical_restriction``, ``linear_operator`` (vertical
or full 3D), ``linearized_pressure``, ``equation_of_state``.
Arrays in and out are E-vectors ``(5, nel, nqt, nqs, nqr)`` (numpy or torch);
the arithmetic runs in libhevi.so on the GPU.  Supported: cG, ``set2nc``
(primary) and ``set2c`` (conservative flux form).  dG is outside the device
path and raises ``NotImplementedError``.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import specgrid as sg


@dataclass(frozen=True)
class GasConstants:
    """euler.py:23-36."""
    c_p: float = 1004.5
    c_v: float = 717.5
    P0: float = 1.0e5
    g: float = 9.80616

    @property
    def R(self) -> float:
        return self.c_p - self.c_v

    @property
    def gamma(self) -> float:
        return self.c_p / self.c_v


@dataclass
class ReferenceState:
    """Hydrostatic background sampled per level (box meshes: functions of
    height only).  Arrays have length n_lev and hold exactly the values the
    reference computes at the first-occurrence node of each level
    (euler.py:70-122)."""
    const: GasConstants
    kind: str
    height: np.ndarray
    rho0: np.ndarray
    theta0: np.ndarray
    P0f: np.ndarray
    drho0: np.ndarray      # d rho0 / dh  (grad_rho0 = drho0 * vert)
    dtheta0: np.ndarray    # d theta0 / dh
    mesh: object = None    # the box the levels belong to (per-node views below)
    _cache: dict = field(default_factory=dict)

    # --- per-node views in the reference's E-vector layout (euler.py:70-122) ---
    def node(self, a):
        """Per-level table -> per-node array (nel, nqt, nqs, nqr) of self.mesh."""
        if self.mesh is None:
            raise ValueError("this ReferenceState carries no mesh")
        lev = _node_levels(self.mesh)
        return np.ascontiguousarray(np.asarray(a)[lev])

    def _vert(self, a):
        if a not in self._cache:
            v = np.zeros(tuple(self.mesh.nshape) + (3,))
            v[..., 2] = self.node(getattr(self, a[1:]) if a != "_g" else
                                  np.full(self.mesh.Z, self.const.g))
            self._cache[a] = v
        return self._cache[a]

    @property
    def grad_rho0(self):
        """(nel, nqt, nqs, nqr, 3): analytic, purely vertical (euler.py:130-150)."""
        return self._vert("_drho0")

    @property
    def grad_theta0(self):
        return self._vert("_dtheta0")

    @property
    def gvec(self):
        """g * vertical unit vector per node (euler.py:150)."""
        return self._vert("_g")

    @property
    def F0vec_nc(self):
        """G0 grad rho0 + H0 grad theta0 per node (euler.py:95-100)."""
        if "F0vec" not in self._cache:
            v = np.zeros(tuple(self.mesh.nshape) + (3,))
            v[..., 2] = self.node(self.F0z_nc)
            self._cache["F0vec"] = v
        return self._cache["F0vec"]

    @property
    def grad_G0_c(self):
        """grad(Theta0 / rho0) = grad theta0 (euler.py:119-122)."""
        return self.grad_theta0

    @property
    def G0_nc(self):
        if "G0" not in self._cache:
            self._cache["G0"] = self.const.gamma * self.P0f / self.rho0
        return self._cache["G0"]

    @property
    def H0_nc(self):
        if "H0" not in self._cache:
            self._cache["H0"] = self.const.gamma * self.P0f / self.theta0
        return self._cache["H0"]

    @property
    def F0z_nc(self):
        """z component of F0vec = G0 grad rho0 + H0 grad theta0 (euler.py:95-100)."""
        if "F0z" not in self._cache:
            self._cache["F0z"] = self.G0_nc * self.drho0 + self.H0_nc * self.dtheta0
        return self._cache["F0z"]

    # --- set2c coefficients (euler.py:102-122) ---
    @property
    def Theta0(self):
        if "Theta0" not in self._cache:
            self._cache["Theta0"] = self.rho0 * self.theta0
        return self._cache["Theta0"]

    @property
    def F0_c(self):
        if "F0_c" not in self._cache:
            self._cache["F0_c"] = self.const.gamma * self.P0f / self.Theta0
        return self._cache["F0_c"]

    @property
    def G0_c(self):
        return self.theta0

    @property
    def rho0G0(self):
        """rho0 * G0, the factor of the vertical divergence (imexcore.py:265)."""
        if "rG" not in self._cache:
            self._cache["rG"] = self.rho0 * self.G0_nc
        return self._cache["rG"]


def _level_heights(mesh: sg.BoxMesh) -> np.ndarray:
    return mesh.lattice_coords()[2]


def hydrostatic_reference(mesh: sg.BoxMesh, theta_bg: float,
                          const: GasConstants = GasConstants()) -> ReferenceState:
    """Constant-theta hydrostatic background (euler.py:125-150)."""
    if _general(mesh):
        from . import sphere
        return sphere.hydrostatic_reference(mesh, theta_bg, const)
    if theta_bg <= 0:
        raise ValueError("background potential temperature must be positive")
    c = const
    h = _level_heights(mesh)
    pi = 1.0 - c.g * h / (c.c_p * theta_bg)
    if np.any(pi <= 0):
        raise ValueError("domain too tall for this background temperature")
    P0f = c.P0 * pi ** (c.c_p / c.R)
    rho0 = P0f / (c.R * theta_bg * pi)
    theta0 = np.full_like(h, theta_bg)
    dpi = -c.g / (c.c_p * theta_bg)
    drho0 = rho0 * (c.c_p / c.R - 1.0) * dpi / pi
    return ReferenceState(const=c, kind="hydrostatic", height=h, rho0=rho0, theta0=theta0,
                          P0f=P0f, drho0=drho0, dtheta0=np.zeros_like(h), mesh=mesh)


def isothermal_reference(mesh: sg.BoxMesh, T_bg: float,
                         const: GasConstants = GasConstants()) -> ReferenceState:
    """Constant-temperature hydrostatic background (euler.py:153-177)."""
    if _general(mesh):
        from . import sphere
        return sphere.isothermal_reference(mesh, T_bg, const)
    if T_bg <= 0:
        raise ValueError("background temperature must be positive")
    c = const
    h = _level_heights(mesh)
    pi = np.exp(-c.g * h / (c.c_p * T_bg))
    P0f = c.P0 * pi ** (c.c_p / c.R)
    rho0 = P0f / (c.R * T_bg)
    theta0 = T_bg / pi
    drho0 = -rho0 * c.g / (c.R * T_bg)
    dth0 = (c.g / c.c_p) / pi
    return ReferenceState(const=c, kind="isothermal", height=h, rho0=rho0, theta0=theta0,
                          P0f=P0f, drho0=drho0, dtheta0=dth0, mesh=mesh)


def _general(mesh) -> bool:
    """A general curvilinear mesh (the cubed-sphere shell), not the box."""
    return getattr(mesh, "kind", "box") == "sphere"


def _node_levels(mesh):
    """Level index of every E-vector node."""
    nel, nt, ns, nr = mesh.nshape
    kz = np.arange(nel) // (mesh.nx * mesh.ny)
    lev = kz[:, None] * mesh.N + np.arange(nt)[None, :]
    return np.broadcast_to(lev[:, :, None, None], mesh.nshape)


def linearized_pressure(q, ref: ReferenceState, set_name: str, mesh: sg.BoxMesh = None):
    """Perturbation pressure of the linearised EOS (euler.py:188-194): G0 rho' +
    H0 theta' (set2nc) or F0 Theta' (set2c).  Same call as the reference,
    ``linearized_pressure(q, ref, set_name)`` on an E-vector (numpy or torch);
    the node levels come from the mesh the ReferenceState was built on
    (host/diagnostic helper: the kernels form it inline)."""
    if set_name not in ("set2nc", "set2c"):
        raise ValueError(f"unknown equation set {set_name!r}")
    if not isinstance(ref, ReferenceState):     # per-node background (general mesh)
        import torch
        from .plan import to_device
        E, back = to_device(q)

        def node(a):
            return torch.as_tensor(np.asarray(a), device=E.device)
        if set_name == "set2nc":
            return back(node(ref.G0_nc) * E[0] + node(ref.H0_nc) * E[4])
        return back(node(ref.F0_c) * E[4])
    mesh = mesh if mesh is not None else ref.mesh
    if mesh is None:
        raise ValueError("linearized_pressure needs the mesh the ReferenceState was built on")
    import torch
    from .plan import to_device
    E, back = to_device(q)
    lev = torch.as_tensor(np.ascontiguousarray(_node_levels(mesh)), device=E.device)

    def per_node(a):
        return torch.as_tensor(np.asarray(a), device=E.device)[lev]
    if set_name == "set2nc":
        return back(per_node(ref.G0_nc) * E[0] + per_node(ref.H0_nc) * E[4])
    return back(per_node(ref.F0_c) * E[4])


def equation_of_state(rho, theta, const: GasConstants):
    """Full nonlinear pressure P = P0 (rho R theta / P0)^gamma (euler.py:180-185).
    Host helper for diagnostics; the step evaluates it inside the kernels."""
    if (rho <= 0).any() or (theta <= 0).any():
        raise ValueError("EOS requires positive density and temperature")
    return const.P0 * (rho * const.R * theta / const.P0) ** const.gamma


@dataclass
class Discretization:
    """Grid objects shared by all operator evaluations (euler.py:271-300).
    Holds the host-side axis tables; the device plan is created per
    ReferenceState on first use (``plan_for``).  ``dss``, ``bidx``/``bproj``
    and the DSS-projected derivative methods mirror the reference object
    (their arithmetic runs on the device)."""
    mesh: sg.BoxMesh
    cx: np.ndarray
    cy: np.ndarray
    cz: np.ndarray
    _plans: dict = field(default_factory=dict)
    _bnd: tuple = None
    dss: object = None

    def plan_for(self, ref: ReferenceState, set_name: str = "set2nc"):
        from .plan import HeviPlan
        key = (id(ref), set_name)
        ent = self._plans.get(key)
        if ent is None or ent[0] is not ref:
            ent = (ref, HeviPlan(self.mesh, ref, self, set_name=set_name))
            self._plans[key] = ent
        return ent[1]

    @property
    def metrics(self):
        """The part of MetricTerms (specgrid.py:404-455) callers use: wJ, the
        per-node mass weight (quadrature weight x Jacobian) of the box."""
        if self.dss is None:
            raise ValueError("discretization has no DSS map")
        return _BoxMetrics(self.dss)

    def geometry_plan(self):
        """A whole-domain plan for the geometry-only kernels (DSS, derivatives)."""
        for ref, plan in self._plans.values():
            if plan.window["lX"] == self.mesh.X and plan.window["lY"] == self.mesh.Y:
                return plan
        return self.plan_for(hydrostatic_reference(self.mesh, 300.0))

    # --- boundary projectors (euler.py:218-258) ---------------------------------
    @property
    def bidx(self):
        if self._bnd is None:
            self._bnd = boundary_projectors(self.mesh)
        return self._bnd[0]

    @property
    def bproj(self):
        if self._bnd is None:
            self._bnd = boundary_projectors(self.mesh)
        return self._bnd[1]

    # --- DSS-projected derivatives (euler.py:281-300), on the device ------------
    def _deriv(self, f, kind, vertical_only):
        from . import _native as nv
        from .plan import to_device
        plan = self.geometry_plan()
        if kind == "grad":
            E, back = to_device(f)
            L = plan.e2l(E[None])
            out = plan.zeros(3)
            nv.check(plan.lib.hevi_grad(plan.h, int(vertical_only), nv.ptr(L), nv.ptr(out),
                                        nv.stream_ptr()))
            return back(plan.l2e(out).movedim(0, -1).contiguous())
        E, back = to_device(f)
        L = plan.e2l(E.movedim(-1, 0).contiguous())
        out = plan.zeros(1)
        nv.check(plan.lib.hevi_div(plan.h, int(vertical_only), nv.ptr(L), nv.ptr(out), nv.stream_ptr()))
        return back(plan.l2e(out)[0])

    def gradc(self, f):
        """DSS-projected gradient of a continuous scalar field, (..., 3)."""
        return self._deriv(f, "grad", False)

    def divc(self, vec):
        """DSS-projected divergence of a continuous (..., 3) field."""
        return self._deriv(vec, "div", False)

    def grad_vc(self, f):
        """DSS-projected vertical derivative times the vertical unit vector."""
        return self._deriv(f, "grad", True)

    def div_vc(self, vec):
        """DSS-projected vertical part of the divergence."""
        return self._deriv(vec, "div", True)


class _BoxMetrics:
    def __init__(self, dss):
        self._dss = dss

    @property
    def wJ(self):
        m = self._dss.mesh
        nel, nt, ns, nr = m.nshape
        e = np.arange(nel)
        kx, ky, kz = e % m.nx, (e // m.nx) % m.ny, e // (m.nx * m.ny)
        wx = self._dss.wx.reshape(m.nx, nr)[kx][:, None, None, :]
        wy = (self._dss.wy.reshape(-1, ns)[np.minimum(ky, self._dss.wy.size // ns - 1)])[:, None, :, None]
        wz = self._dss.wz.reshape(m.nz, nt)[kz][:, :, None, None]
        return (wx * wy) * wz


def build_discretization(mesh: sg.BoxMesh) -> Discretization:
    """Metric/DSS set-up (euler.py:303-310): the structured box, or a general
    curvilinear mesh (the cubed-sphere shell, ``sphere``)."""
    if _general(mesh):
        from . import sphere
        return sphere.build_discretization(mesh)
    if not isinstance(mesh, sg.BoxMesh):
        raise TypeError("the B200 HEVI path supports structured box meshes "
                        "(specgrid.build_box_mesh / build_box_mesh_3d)")
    disc = Discretization(mesh=mesh, cx=mesh.axis_factor(0), cy=mesh.axis_factor(1),
                          cz=mesh.axis_factor(2))
    disc.dss = sg.build_dss_map(mesh, plan_getter=disc.geometry_plan)
    return disc


def boundary_projectors(mesh: sg.BoxMesh, metrics=None, dss=None):
    """(bidx, bproj) of euler.boundary_projectors (euler.py:218-258) for the
    box: every E-vector node on a domain face with the tangential projector
    I - sum n n^T over the (orthonormal, axis-aligned) normals meeting there.
    Lateral x faces, the slab's y faces (its dummy layer), lateral y faces
    (3D) and the bottom/top faces.  General meshes: the face normals
    gathered through the coincidence groups (``sphere.boundary_projectors``)."""
    if _general(mesh):
        from . import sphere
        return sphere.boundary_projectors(mesh, metrics, dss)[:2]
    nel, nt, ns, nr = mesh.nshape
    e = np.arange(nel)
    kx = e % mesh.nx
    ky = (e // mesh.nx) % mesh.ny
    kz = e // (mesh.nx * mesh.ny)
    gx = kx[:, None, None, None] * mesh.N + np.arange(nr)[None, None, None, :]
    gy = ky[:, None, None, None] * mesh.Ny + np.arange(ns)[None, None, :, None]
    gz = kz[:, None, None, None] * mesh.N + np.arange(nt)[None, :, None, None]
    bx = np.broadcast_to((gx == 0) | (gx == mesh.X - 1), mesh.nshape)
    by = np.broadcast_to(np.full(gy.shape, mesh.slab) | (gy == 0) | (gy == mesh.Y - 1), mesh.nshape)
    bz = np.broadcast_to((gz == 0) | (gz == mesh.Z - 1), mesh.nshape)
    on = (bx | by | bz).ravel()
    bidx = np.flatnonzero(on).astype(np.int64)
    proj = np.zeros((bidx.size, 3, 3))
    proj[:, 0, 0] = ~bx.ravel()[bidx]
    proj[:, 1, 1] = ~by.ravel()[bidx]
    proj[:, 2, 2] = ~bz.ravel()[bidx]
    return bidx, proj


def zero_normal_velocity(vel, bidx, bproj):
    """In place: remove all boundary-normal components of a (..., 3) field
    (euler.py:261-264); the projection runs on the device."""
    import torch
    from .plan import to_device
    T, _ = to_device(vel)
    flat = T.reshape(-1, 3)
    idx = torch.as_tensor(np.asarray(bidx), device=T.device)
    P = torch.as_tensor(np.asarray(bproj), dtype=T.dtype, device=T.device)
    flat[idx] = torch.einsum("nab,nb->na", P, flat[idx])
    if isinstance(vel, np.ndarray):
        vel[...] = T.cpu().numpy()
    elif T.data_ptr() != vel.data_ptr():
        vel.copy_(T)
    return vel


def min_node_spacing(mesh: sg.BoxMesh):
    """Minimal horizontal / vertical internodal distances (euler.py:583-593)."""
    if _general(mesh):
        from . import sphere
        return sphere.min_node_spacing(mesh)
    return mesh.min_node_spacing()


def courant_numbers(q, ref: ReferenceState, disc: Discretization, dt: float, set_name: str):
    """(C_H, C_V) from |u| + sound speed and the minimal node spacings
    (euler.py:564-580), evaluated on the device."""
    import torch
    from .plan import to_device
    if dt <= 0:
        raise ValueError("dt must be positive")
    _check_set(set_name)
    E, _ = to_device(q)
    mesh = disc.mesh
    dev = E.device
    rho = torch.as_tensor(ref.node(ref.rho0), device=dev) + E[0]
    vel = E[1:4]
    if set_name == "set2c":
        vel = vel / rho
        theta = (torch.as_tensor(ref.node(ref.Theta0), device=dev) + E[4]) / rho
    else:
        theta = torch.as_tensor(ref.node(ref.theta0), device=dev) + E[4]
    c = ref.const
    P = equation_of_state(rho, theta, c)
    cmax = float((torch.sqrt((vel * vel).sum(0)) + torch.sqrt(c.gamma * P / rho)).max())
    dx_h, dx_v = min_node_spacing(mesh)
    return cmax * dt / dx_h, cmax * dt / dx_v


def _check_set(set_name: str, dg: bool = False):
    if set_name not in ("set2nc", "set2c"):
        raise ValueError(f"unknown equation set {set_name!r}")
    if dg:
        raise NotImplementedError("dG is outside the HEVI direct path (SURVEY 2.4)")


def nonlinear_rhs(q, ref: ReferenceState, disc: Discretization, set_name: str,
                  dg: bool = False):
    """R(q), cG set2nc (advective) or set2c (flux form), with DSS and no-flux
    projection (euler.py:438-497)."""
    _check_set(set_name, dg)
    return disc.plan_for(ref, set_name).apply_evec("rhs", q)


def linear_operator(q, ref: ReferenceState, disc: Discretization, set_name: str,
                    vertical_only: bool = False, dg: bool = False):
    """L(q) with DSS-projected derivatives (euler.py:313-365): the vertical
    restriction (HEVI, ``hevi_linear_v``) or the full 3D operator (3D-IMEX,
    ``hevi_linear3``)."""
    _check_set(set_name, dg)
    return disc.plan_for(ref, set_name).apply_evec("linear" if vertical_only else "linear3", q)


def vertical_restriction(q, ref: ReferenceState, disc: Discretization, set_name: str):
    """L_V(q) (euler.py:368-371)."""
    return linear_operator(q, ref, disc, set_name, vertical_only=True)


class RHS:
    """``rhs`` callable for ``ark_imex_step``: same call protocol as the
    reference's ``lambda s: euler.nonlinear_rhs(s, ref, disc, set_name)``
    (cli.py:184-185); passing this object lets the stepper fuse the step."""

    def __init__(self, ref: ReferenceState, disc: Discretization, set_name: str = "set2nc"):
        _check_set(set_name)
        self.ref, self.disc, self.set_name = ref, disc, set_name

    def __call__(self, q):
        return nonlinear_rhs(q, self.ref, self.disc, self.set_name)


def make_rhs(ref, disc, set_name="set2nc") -> RHS:
    return RHS(ref, disc, set_name)
