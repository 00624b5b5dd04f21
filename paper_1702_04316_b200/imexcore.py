"""ARK2 IMEX stepper and the vertically-implicit problem (drop-in for
``dycore.imexcore`` along the HEVI path).

``ark_imex_step(q, dt, tableau, problem, rhs)`` keeps the reference
signature and semantics (imexcore.py:385-414): three explicit evaluations,
two implicit solves with ``problem.lam = tableau.diag * dt``, the combine
with the shared weights, a fresh output array, FloatingPointError on a
non-finite result.  When ``problem`` is this module's ``ImplicitProblem``
(cG, set2nc, Schur form, dim='1d', method='direct') and ``rhs`` is an
``euler.RHS`` on the same discretization, the whole step runs as the fused
five-kernel device schedule; any other duck-typed problem/rhs
pair runs the reference's generic stage loop on the caller's callables.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import euler


@dataclass(frozen=True)
class ButcherPair:
    """Double Butcher tableau (imexcore.py:26-41)."""
    a: np.ndarray
    at: np.ndarray
    b: np.ndarray
    c: np.ndarray
    ct: np.ndarray

    @property
    def stages(self) -> int:
        return len(self.b)

    @property
    def diag(self) -> float:
        return float(self.at[1, 1])


def ark2_tableau() -> ButcherPair:
    """L-stable ARK2 pair with the reference's sign-corrected weights
    (imexcore.py:44-63; the paper's printed row fails sum b = 1)."""
    s2 = math.sqrt(2.0)
    gam = 1.0 - 1.0 / s2
    d = 1.0 / (2.0 * s2)
    a32 = (3.0 + 2.0 * s2) / 6.0
    a = np.array([[0.0, 0.0, 0.0], [2.0 - s2, 0.0, 0.0], [1.0 - a32, a32, 0.0]])
    at = np.array([[0.0, 0.0, 0.0], [gam, gam, 0.0], [d, d, gam]])
    b = np.array([d, d, gam])
    return ButcherPair(a=a, at=at, b=b, c=a.sum(axis=1), ct=at.sum(axis=1))


# Shu-Osher representation of SSP RK(5,3) (imexcore.py:79-94)
_RK35_ALPHA = {
    (1, 0): 1.0,
    (2, 1): 1.0,
    (3, 0): 0.355909775063327, (3, 2): 0.644090224936674,
    (4, 0): 0.367933791638137, (4, 3): 0.632066208361863,
    (5, 2): 0.237593836598569, (5, 4): 0.762406163401431,
}
_RK35_BETA = {
    (1, 0): 0.377268915331368,
    (2, 1): 0.377268915331368,
    (3, 2): 0.242995220537396,
    (4, 3): 0.238458932846290,
    (5, 4): 0.287632146308408,
}


def rk35_butcher():
    """Butcher (A, b, c) of the SSP RK(5,3) scheme (imexcore.py:97-108)."""
    rows = [np.zeros(5)]
    for i in range(1, 6):
        row = np.zeros(5)
        for j in range(i):
            row += _RK35_ALPHA.get((i, j), 0.0) * rows[j]
            row[j] += _RK35_BETA.get((i, j), 0.0)
        rows.append(row)
    A = np.vstack(rows[:5])
    return A, rows[5], A.sum(axis=1)


def rk35_step(q, dt: float, rhs):
    """One SSP RK(5,3) step (imexcore.py:111-126).  With ``rhs`` an
    ``euler.RHS`` the five stages run as fused device launches."""
    if isinstance(rhs, euler.RHS):
        plan = rhs.disc.plan_for(rhs.ref, rhs.set_name)
        Q, back = plan.lattice_in(q, reuse=True)
        work = plan.cached_workspace()
        plan.rk35(dt, Q, work)
        plan.check_flags()
        return back(Q)
    u = [q]
    for i in range(1, 6):
        acc = q * 0.0
        for j in range(i):
            al = _RK35_ALPHA.get((i, j), 0.0)
            be = _RK35_BETA.get((i, j), 0.0)
            if al != 0.0:
                acc += al * u[j]
            if be != 0.0:
                acc += (be * dt) * rhs(u[j])
        u.append(acc)
    out = u[5]
    finite = np.isfinite(out).all() if isinstance(out, np.ndarray) else bool(out.isfinite().all())
    if not finite:
        raise FloatingPointError("non-finite state in explicit stage")
    return out


@dataclass
class SolverSpec:
    """imexcore.py:133-140: 'direct' (1D, fused column solve) or the Krylov
    solvers 'gmres' | 'bicgstab' | 'richardson' (3D Schur form)."""
    method: str = "gmres"
    tol: float = 1e-6
    max_iter: int = 2000
    restart: int = 50
    precon_order: int = 1
    check_every: int = 4


@dataclass
class SolveStats:
    """imexcore.py:143-155; the direct path increments only ``solves``."""
    solves: int = 0
    iterations: int = 0
    matvecs: int = 0
    failures: int = 0

    def add(self, rep):
        self.solves += 1
        self.iterations += rep.iterations
        self.matvecs += rep.matvecs
        if not rep.converged:
            self.failures += 1


class SolverFailure(RuntimeError):
    """imexcore.py:158-162 (raised by iterative solvers only)."""

    def __init__(self, report):
        super().__init__(f"implicit solve failed: iterations={report.iterations} "
                         f"residual={report.residual:.3e} {report.note}")
        self.report = report


@dataclass
class ImplicitProblem:
    """(I - lam L_V) q = q_e on the device (imexcore.py:165-322)."""
    disc: euler.Discretization
    ref: euler.ReferenceState
    set_name: str
    discretization: str = "cg"
    form: str = "schur"
    dim: str = "3d"
    lam: float = 0.0
    solver: SolverSpec = field(default_factory=SolverSpec)
    stats: SolveStats = field(default_factory=SolveStats)
    _column_cache: dict = field(default_factory=dict)
    _pbno_cache: dict = field(default_factory=dict)

    def __post_init__(self):
        if self.discretization == "dg":
            if self.form == "schur":
                raise ValueError("the pressure-reduced form is not supported with dG fluxes")
            if self.set_name != "set2c":
                raise ValueError("dG requires the conservative set")

    # -- what the device path implements --------------------------------------
    def _check_path(self):
        if self.discretization != "cg":
            raise NotImplementedError("dG is outside the HEVI direct path")
        if self.solver.method != "direct":
            raise NotImplementedError("iterative (3D-IMEX) solvers are SURVEY 8(f) 'next'; "
                                      "use SolverSpec(method='direct') with dim='1d'")
        if self.dim != "1d":
            raise ValueError("the direct column solver requires the 1D form")
        if self.form not in ("schur", "standard"):
            raise ValueError(f"unknown form {self.form!r}")
        euler._check_set(self.set_name)

    @property
    def fused(self) -> bool:
        try:
            self._check_path()
        except (NotImplementedError, ValueError):
            return False
        return self.form == "schur"

    def linear(self, q):
        """imexcore.py:190-194."""
        if self.dim == "1d":
            return euler.vertical_restriction(q, self.ref, self.disc, self.set_name)
        return euler.linear_operator(q, self.ref, self.disc, self.set_name)

    def solve(self, q_e):
        """imexcore.py:312-356: the direct column solve (dim='1d') or a Krylov
        solve of the 3D pressure equation (dim='3d', form='schur')."""
        if self.lam <= 0:
            raise ValueError("implicit solve requires positive lam")
        if self.solver.method != "direct":
            return self._solve_krylov(q_e)
        self._check_path()
        from . import columnsolve
        out = columnsolve.solve_direct(self, q_e)
        self.stats.solves += 1
        return out


    # -- operator pieces of the reference object (imexcore.py:190-298) ----------
    # E-vectors in and out (numpy or torch); the arithmetic runs in the
    # library's lattice kernels (hevi_schur3_*, hevi_linear_v / hevi_linear3,
    # hevi_grad / hevi_div), with the vertical-only derivatives when dim="1d".
    def _plan(self):
        euler._check_set(self.set_name, self.discretization == "dg")
        return self.disc.plan_for(self.ref, self.set_name)

    @staticmethod
    def _vec_in(plan, v):
        """(..., 3) E-vector -> (3, Z, lY, px) lattice tensor, and the way back."""
        from .plan import to_device
        E, back = to_device(v)
        return plan.e2l(E.movedim(-1, 0).contiguous()), (lambda L: back(plan.l2e(L).movedim(0, -1).contiguous()))

    @staticmethod
    def _scalar_in(plan, f):
        from .plan import to_device
        E, back = to_device(f)
        return plan.e2l(E[None].contiguous()), (lambda L: back(plan.l2e(L)[0]))

    def lhs_standard(self, q):
        """(I - lam L) q in the 5-variable standard form (imexcore.py:196-198)."""
        plan = self._plan()
        Q, back = plan.lattice_in(q)
        L = plan.linear(Q, plan.zeros()) if self.dim == "1d" else plan.linear3(Q, plan.zeros())
        plan.check_flags()
        plan.axpby(-float(self.lam), L, 1.0, Q)
        return back(Q)

    def _ainv(self, v):
        """Rank-one (Sherman-Morrison) inverse of A = I + lam^2 u w^T
        (imexcore.py:200-217); u, w are vertical on a box, so only the z
        component changes."""
        import torch
        from .plan import to_device
        ref = self.ref
        w = ref.dtheta0      # grad theta0 (set2nc) = grad G0_c (set2c), vertical
        if not np.any(w):
            return v
        E, back = to_device(v)
        dev = E.device
        node = lambda a: torch.as_tensor(ref.node(a), device=dev)  # noqa: E731
        u = (self.lam ** 2 / node(ref.theta0)) * ref.const.g
        den = 1.0 + node(w) * u
        if bool((den.abs() < 1e-12).any()):
            raise FloatingPointError("rank-one inverse denominator underflow")
        out = E.clone()
        out[..., 2] = E[..., 2] - u * ((node(w) * E[..., 2]) / den)
        return back(out)

    def _gradP(self, P):
        return self.disc.grad_vc(P) if self.dim == "1d" else self.disc.gradc(P)

    def _div(self, vec):
        return self.disc.div_vc(vec) if self.dim == "1d" else self.disc.divc(vec)

    def rhs_schur_build(self, q_e):
        """Pressure right-hand side and the stored velocity-like estimate
        (imexcore.py:229-243): (rhs, ua) with ua of shape (..., 3)."""
        plan = self._plan()
        lam = float(self.lam)
        Qe, _ = plan.lattice_in(q_e)
        ua = plan.zeros(3)
        Pe = plan.zeros(1)[0]
        plan.schur3_ua(lam, Qe, ua, Pe)
        rhs = plan.schur3_flux(lam, Pe, ua, plan.zeros(1)[0], self.dim == "1d")
        plan.check_flags()
        E = plan.l2e(rhs[None])[0]
        U = plan.l2e(ua).movedim(0, -1).contiguous()
        return _back_like(q_e, E), _back_like(q_e, U)

    def _up(self, P):
        """Pressure-driven velocity-like variable (imexcore.py:245-257), (..., 3)."""
        plan = self._plan()
        L, _ = self._scalar_in(plan, P)
        up = plan.schur3_up(float(self.lam), L[0], plan.zeros(3), self.dim == "1d")
        plan.check_flags()
        return _back_like(P, plan.l2e(up).movedim(0, -1).contiguous())

    def _helmholtz_flux(self, vel):
        """lam-scaled pressure-equation flux of a velocity-like field (imexcore.py:259-268)."""
        plan = self._plan()
        V, _ = self._vec_in(plan, vel)
        neg = plan.schur3_flux(float(self.lam), plan.zeros(1)[0], V, plan.zeros(1)[0], self.dim == "1d")
        return _back_like(vel, -plan.l2e(neg[None])[0])

    def lhs_schur(self, P):
        """P - helmholtz_flux(up(P)) (imexcore.py:270-271)."""
        plan = self._plan()
        L, _ = self._scalar_in(plan, P)
        lam, vo = float(self.lam), self.dim == "1d"
        up = plan.schur3_up(lam, L[0], plan.zeros(3), vo)
        out = plan.schur3_flux(lam, L[0], up, plan.zeros(1)[0], vo)
        plan.check_flags()
        return _back_like(P, plan.l2e(out[None])[0])

    def extract_from_pressure(self, P, ua, q_e):
        """q from the solved pressure, the estimate ua and q_e (imexcore.py:273-298)."""
        plan = self._plan()
        lam, vo = float(self.lam), self.dim == "1d"
        L, _ = self._scalar_in(plan, P)
        U, _ = self._vec_in(plan, ua)
        Qe, back = plan.lattice_in(q_e)
        up = plan.schur3_up(lam, L[0], plan.zeros(3), vo)
        q = plan.schur3_extract(lam, L[0], U, up, Qe, plan.zeros())
        plan.check_flags()
        return back(q)

    # -- 3D-IMEX Schur form (imexcore.py:229-298, 324-373) ----------------------
    def _krylov_path(self):
        if self.discretization != "cg":
            raise NotImplementedError("dG is outside the device path")
        if self.solver.method not in ("gmres", "bicgstab", "richardson"):
            raise ValueError(f"unknown solver {self.solver.method!r}")
        if self.dim not in ("1d", "3d"):
            raise ValueError(f"unknown dim {self.dim!r}")
        if self.form not in ("schur", "standard"):
            raise ValueError(f"unknown form {self.form!r}")
        euler._check_set(self.set_name)

    def _solve_krylov(self, q_e):
        from . import krylov
        from .plan import to_device
        self._krylov_path()
        plan = self.disc.plan_for(self.ref, self.set_name)
        lam = float(self.lam)
        E, back = to_device(q_e)
        if E.shape != (5,) + tuple(self.disc.mesh.nshape):
            raise ValueError("field/mesh shape mismatch")
        Qe = plan.e2l(E)
        if self.form == "standard":
            return back(plan.l2e(self._solve_standard(plan, Qe, lam)))
        vo = self.dim == "1d"          # grad_vc / div_vc instead of gradc / divc
        ua = plan.zeros(3)
        Pe = plan.zeros(1)[0]
        plan.schur3_ua(lam, Qe, ua, Pe)
        rhs = plan.schur3_flux(lam, Pe, ua, plan.zeros(1)[0], vo)
        up = plan.zeros(3)

        def lhs_schur(v):
            plan.schur3_up(lam, v, up, vo)
            return plan.schur3_flux(lam, v, up, plan.zeros(1)[0], vo)

        amap = krylov.LinearMap(int(np.prod(self.disc.mesh.nshape)), lhs_schur,
                                space=krylov.space_for(plan))
        x, rep = self._run_krylov(amap, rhs, Pe)
        self.stats.add(rep)
        if not rep.converged:
            raise SolverFailure(rep)
        plan.schur3_up(lam, x, up, vo)
        q = plan.schur3_extract(lam, x, ua, up, Qe, plan.zeros(), vertical_only=vo)
        return back(plan.l2e(q))

    def _solve_standard(self, plan, Qe, lam):
        """5-variable form with the reference's per-field diagonal scaling
        q = D x, D = diag(rho/c, 1, 1, 1, theta/c) (imexcore.py:330-355)."""
        from . import krylov
        mesh = self.disc.mesh
        lev = _node_levels(mesh)
        cbar = float(np.sqrt(self.ref.G0_nc[lev].mean()))
        D = np.ones(5)
        D[0] = float(self.ref.rho0[lev].mean()) / cbar
        D[4] = float(self.ref.theta0[lev].mean()) / cbar
        op = plan.linear if self.dim == "1d" else plan.linear3

        def scaled(src, s, dst):
            for f in range(5):
                plan.axpby(float(s[f]), src[f], 0.0, dst[f])
            return dst

        Dinv = 1.0 / D

        def lhs(v):
            t = scaled(v, D, plan.zeros())
            Lt = op(t, plan.zeros())
            plan.axpby(-lam, Lt, 1.0, t)          # q - lam L(q)
            return scaled(t, Dinv, t)

        amap = krylov.LinearMap(5 * int(np.prod(mesh.nshape)), lhs,
                                space=krylov.LatticeSpace(plan, nf=5))
        b = scaled(Qe, Dinv, plan.zeros())
        x, rep = self._run_krylov(amap, b, b.clone())
        plan.check_flags()
        self.stats.add(rep)
        if not rep.converged:
            raise SolverFailure(rep)
        return scaled(x, D, plan.zeros())

    def _get_pbno(self, amap, order, like):
        from . import krylov
        key = (round(self.lam, 12), self.form, self.dim, order, amap.n)
        if key not in self._pbno_cache:
            try:
                self._pbno_cache[key] = krylov.build_pbno(amap, order, like=like)
            except ValueError:
                self._pbno_cache[key] = None     # indefinite estimate: unpreconditioned
        return self._pbno_cache[key]

    def _run_krylov(self, amap, b, x0):
        """imexcore.py:358-373."""
        from . import krylov
        spec = self.solver
        pre = None
        if spec.precon_order >= 0 and spec.method in ("bicgstab", "richardson"):
            pre = self._get_pbno(amap, spec.precon_order, b)
        elif spec.precon_order > 0:
            pre = self._get_pbno(amap, spec.precon_order, b)
        if spec.method == "gmres":
            return krylov.gmres(amap, b, tol=spec.tol, max_iter=spec.max_iter,
                                restart=spec.restart, precon=pre, x0=x0)
        if spec.method == "bicgstab":
            return krylov.bicgstab_pbno(amap, b, tol=spec.tol, max_iter=spec.max_iter,
                                        precon=pre, x0=x0)
        return krylov.richardson_pbno(amap, b, tol=spec.tol, max_iter=spec.max_iter,
                                      precon=pre, x0=x0, check_every=spec.check_every)


def _back_like(like, t):
    """A device result in the array type of ``like`` (numpy -> numpy)."""
    if isinstance(like, np.ndarray):
        return t.cpu().numpy()
    return t.to(like.device) if hasattr(like, "device") else t


def _node_levels(mesh):
    """Level index of every E-vector node (per-node means of level tables)."""
    nel, nt, ns, nr = mesh.nshape
    kz = np.arange(nel) // (mesh.nx * mesh.ny)
    lev = kz[:, None] * mesh.N + np.arange(nt)[None, :]
    return np.broadcast_to(lev[:, :, None, None], mesh.nshape)


def _is_fused(problem, rhs) -> bool:
    return (isinstance(problem, ImplicitProblem) and isinstance(rhs, euler.RHS)
            and problem.fused and rhs.disc is problem.disc and rhs.ref is problem.ref
            and rhs.set_name == problem.set_name)


def ark_imex_step(q, dt: float, tableau: ButcherPair, problem, rhs):
    """One additive Runge-Kutta IMEX step (imexcore.py:385-414)."""
    if _is_fused(problem, rhs) and tableau.stages == 3:
        from .plan import tableau_array
        plan = problem.disc.plan_for(problem.ref, problem.set_name)
        problem.lam = tableau.diag * dt
        Q, back = plan.lattice_in(q, reuse=True)
        work = plan.cached_workspace()
        plan.step(dt, tableau_array(tableau), Q, work)
        plan.check_flags()
        problem.stats.solves += 2
        return back(Q)
    return _generic_step(q, dt, tableau, problem, rhs)


def _generic_step(q, dt, tableau, problem, rhs):
    """The reference stage loop on duck-typed callables (imexcore.py:393-414)."""
    s = tableau.stages
    R = [rhs(q)]
    L = [problem.linear(q)]
    problem.lam = tableau.diag * dt
    for i in range(1, s):
        pred = q.copy() if hasattr(q, "copy") else q.clone()
        for j in range(i):
            pred += dt * (tableau.a[i, j] * (R[j] - L[j]) + tableau.at[i, j] * L[j])
        qi = problem.solve(pred)
        R.append(rhs(qi))
        if i < s - 1:
            L.append(problem.linear(qi))
    out = q.copy() if hasattr(q, "copy") else q.clone()
    for i in range(s):
        out += dt * tableau.b[i] * R[i]
    finite = np.isfinite(out).all() if isinstance(out, np.ndarray) else bool(out.isfinite().all())
    if not finite:
        raise FloatingPointError("non-finite state after IMEX step")
    return out


@dataclass
class BdfCoefficients:
    """imexcore.py:66-70."""
    alpha: np.ndarray
    beta: np.ndarray
    chi: float


def bdf2_coefficients() -> BdfCoefficients:
    """imexcore.py:73-76."""
    return BdfCoefficients(alpha=np.array([4.0 / 3.0, -1.0 / 3.0]),
                           beta=np.array([2.0, -1.0]), chi=2.0 / 3.0)


def bdf2_imex_step(qn, qnm1, dt: float, coeffs: BdfCoefficients, problem, rhs):
    """Two-step BDF2 IMEX step (imexcore.py:417-430): two R evaluations and one
    implicit solve with lam = chi dt, all on the device; the combinations are
    elementwise on the device E-vectors."""
    al, be, chi = coeffs.alpha, coeffs.beta, coeffs.chi
    problem.lam = chi * dt
    qe = (al[0] * qn + al[1] * qnm1
          + chi * dt * (be[0] * rhs(qn) + be[1] * rhs(qnm1)))
    shift = be[0] * qn + be[1] * qnm1
    qtt = problem.solve(qe - shift)
    out = qtt + shift
    finite = np.isfinite(out).all() if isinstance(out, np.ndarray) else bool(out.isfinite().all())
    if not finite:
        raise FloatingPointError("non-finite state after IMEX step")
    return out
