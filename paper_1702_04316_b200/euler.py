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
    _cache: dict = field(default_factory=dict)

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
                          P0f=P0f, drho0=drho0, dtheta0=np.zeros_like(h))


def isothermal_reference(mesh: sg.BoxMesh, T_bg: float,
                         const: GasConstants = GasConstants()) -> ReferenceState:
    """Constant-temperature hydrostatic background (euler.py:153-177)."""
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
                          P0f=P0f, drho0=drho0, dtheta0=dth0)


def linearized_pressure(q, ref: ReferenceState, set_name: str, mesh: sg.BoxMesh = None):
    """Perturbation pressure of the linearised EOS (euler.py:188-194): G0 rho' +
    H0 theta' (set2nc) or F0 Theta' (set2c).  ``q`` is an E-vector (numpy or
    torch) of ``mesh`` (host/diagnostic helper; the kernels form it inline)."""
    if set_name not in ("set2nc", "set2c"):
        raise ValueError(f"unknown equation set {set_name!r}")
    if mesh is None:
        raise ValueError("linearized_pressure needs the mesh to map nodes to levels")
    nel, nt, ns, nr = mesh.nshape
    kz = np.arange(nel) // (mesh.nx * mesh.ny)
    lev = (kz[:, None] * mesh.N + np.arange(nt)[None, :])[:, :, None, None]

    def per_node(a):
        t = np.broadcast_to(a[lev], (nel, nt, ns, nr))
        if isinstance(q, np.ndarray):
            return t
        import torch
        return torch.as_tensor(np.ascontiguousarray(t), device=q.device)
    if set_name == "set2nc":
        return per_node(ref.G0_nc) * q[0] + per_node(ref.H0_nc) * q[4]
    return per_node(ref.F0_c) * q[4]


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
    ReferenceState on first use (``plan_for``)."""
    mesh: sg.BoxMesh
    cx: np.ndarray
    cy: np.ndarray
    cz: np.ndarray
    _plans: dict = field(default_factory=dict)

    def plan_for(self, ref: ReferenceState, set_name: str = "set2nc"):
        from .plan import HeviPlan
        key = (id(ref), set_name)
        ent = self._plans.get(key)
        if ent is None or ent[0] is not ref:
            ent = (ref, HeviPlan(self.mesh, ref, self, set_name=set_name))
            self._plans[key] = ent
        return ent[1]


def build_discretization(mesh: sg.BoxMesh) -> Discretization:
    """Metric/DSS set-up (euler.py:303-310) for the structured box."""
    if not isinstance(mesh, sg.BoxMesh):
        raise TypeError("the B200 HEVI path supports structured box meshes "
                        "(specgrid.build_box_mesh / build_box_mesh_3d)")
    return Discretization(mesh=mesh, cx=mesh.axis_factor(0), cy=mesh.axis_factor(1),
                          cz=mesh.axis_factor(2))


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
