"""Device plan: owns the libhevi plan handle and the lattice <-> E-vector glue.

A plan is built from a mesh (+ Discretization tables) and a ReferenceState.
Its state arrays are lattice tensors ``(5, Z, lY, px)`` (fp64, CUDA) owned by
the PyTorch caching allocator and passed to the C ABI as raw pointers.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _native as nv


def _dp(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def raise_for_flags(flags: int):
    """Map sticky device flags to the reference's exception types, in the
    order the reference would have raised them."""
    for s in (0, 1, 2):
        if flags & nv.F_NONFINITE_IN(s):
            raise FloatingPointError("non-finite state passed to RHS evaluation")
        if flags & nv.F_EOS(s):
            raise ValueError("EOS requires positive density and temperature")
    if flags & nv.F_AINV:
        raise FloatingPointError("rank-one inverse denominator underflow")
    if flags & nv.F_PIVOT:
        raise RuntimeError("no-pivot LU hit a degenerate diagonal")
    if flags & nv.F_NONFINITE_OUT:
        raise FloatingPointError("non-finite state after IMEX step")


class HeviPlan:
    def __init__(self, mesh, ref, disc, window=None, set_name="set2nc"):
        import torch
        nv.require_cuda()
        self.lib = nv.load()
        self.mesh, self.ref, self.disc = mesh, ref, disc
        X, Y, Z = mesh.X, mesh.Y, mesh.Z
        if window is None:
            window = dict(x0=0, y0=0, lX=X, lY=Y, ex_b=0, ex_e=mesh.nx, ey_b=0, ey_e=mesh.ny)
        self.window = window
        # even pitch (TMA strides are 16-byte multiples), rows 32-byte aligned
        px = window.get("px", (window["lX"] + 3) // 4 * 4)
        gd = nv.GridDesc(nex=mesh.nx, ney=mesh.ny, nez=mesh.nz, N=mesh.N, Ny=mesh.Ny,
                         slab=int(mesh.slab), x0=window["x0"], y0=window["y0"],
                         lX=window["lX"], lY=window["lY"], px=px,
                         ex_b=window["ex_b"], ex_e=window["ex_e"],
                         ey_b=window["ey_b"], ey_e=window["ey_e"])
        c = ref.const
        # EOS of the background per level, evaluated exactly as
        # euler.equation_of_state (euler.py:185): the reference point of P'
        Pb = c.P0 * (ref.rho0 * c.R * ref.theta0 / c.P0) ** c.gamma
        self._keep = [np.ascontiguousarray(a, dtype=np.float64) for a in (
            ref.rho0, ref.theta0, ref.P0f, ref.drho0, ref.dtheta0, ref.G0_nc, ref.H0_nc,
            ref.F0z_nc, ref.rho0G0, Pb, disc.cx, disc.cy, disc.cz,
            mesh.quad_r.D, mesh.quad_s.D, mesh.quad_t.D, ref.Theta0, ref.F0_c)]
        if set_name not in ("set2nc", "set2c"):
            raise ValueError(f"unknown equation set {set_name!r}")
        self.set_name = set_name
        rd = nv.RefDesc(*[_dp(a) for a in self._keep], c.g, c.R, c.P0, c.gamma,
                        1 if set_name == "set2c" else 0)
        h = ctypes.c_void_p()
        nv.check(self.lib.hevi_plan_create(ctypes.byref(h), ctypes.byref(gd), ctypes.byref(rd)))
        self.h = h
        self.Z, self.lY, self.lX, self.px = Z, window["lY"], window["lX"], px
        self.shape = (5, Z, self.lY, px)
        self.fs = Z * self.lY * px
        self.device = torch.device("cuda", torch.cuda.current_device())

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and h.value:
            try:
                self.lib.hevi_plan_destroy(h)
            except Exception:
                pass
            self.h = None

    # -- buffers -------------------------------------------------------------
    def empty(self, nf=5):
        import torch
        return torch.empty((nf,) + self.shape[1:], dtype=torch.float64, device=self.device)

    def zeros(self, nf=5):
        import torch
        return torch.zeros((nf,) + self.shape[1:], dtype=torch.float64, device=self.device)

    def workspace(self):
        """[Q1 | A | F | P] of the fused step (a new zero-filled buffer)."""
        import torch
        return torch.zeros((4,) + self.shape, dtype=torch.float64, device=self.device)

    def cached_workspace(self):
        """The plan's persistent workspace for one-shot drop-in calls
        (``imexcore.ark_imex_step``): allocated and zeroed once, then reused
        -- every point a step reads is written earlier in the same step."""
        if getattr(self, "_ws", None) is None:
            self._ws = self.workspace()
        return self._ws

    # -- conversions -----------------------------------------------------------
    def padded(self, L):
        """(nf, Z, lY, lX) -> plan layout (nf, Z, lY, px)."""
        if L.shape[-1] == self.px:
            return L.contiguous()
        out = self.zeros(L.shape[0])
        out[..., :L.shape[-1]].copy_(L)
        return out

    def e2l(self, E, out=None, nf=None):
        nf = E.shape[0] if nf is None else nf
        out = self.zeros(nf) if out is None else out
        nv.check(self.lib.hevi_evec_to_lattice(self.h, nv.ptr(E), nv.ptr(out), nf, nv.stream_ptr()))
        return out

    def l2e(self, L, out=None):
        import torch
        L = self.padded(L)
        nf = L.shape[0]
        if out is None:
            out = torch.empty((nf,) + tuple(self.mesh.nshape), dtype=torch.float64, device=self.device)
        nv.check(self.lib.hevi_lattice_to_evec(self.h, nv.ptr(L), nv.ptr(out), nf, nv.stream_ptr()))
        return out

    # -- operators on lattice tensors -------------------------------------------
    def rhs(self, q, out):
        nv.check(self.lib.hevi_rhs(self.h, nv.ptr(q), nv.ptr(out), nv.stream_ptr()))
        return out

    def linear(self, q, out):
        nv.check(self.lib.hevi_linear_v(self.h, nv.ptr(q), nv.ptr(out), nv.stream_ptr()))
        return out

    def factor(self, lam) -> int:
        nb = ctypes.c_int(0)
        nv.check(self.lib.hevi_factor(self.h, float(lam), ctypes.byref(nb), nv.stream_ptr()))
        return nb.value

    def force_pivoted(self, on=True):
        """Keep the pivoted dense column factor for lam values factored from
        now on (HEVI_OPT_FORCE_PIVOTED: exercises factor_with_fallback)."""
        nv.check(self.lib.hevi_plan_set_option(self.h, 1, int(bool(on))))

    def factor_pivoted(self, lam) -> bool:
        """Whether the factor of lam took the pivoted fallback."""
        p = ctypes.c_int(0)
        nv.check(self.lib.hevi_factor_pivoted(self.h, float(lam), ctypes.byref(p)))
        return bool(p.value)

    def column_matrix(self, lam):
        M = self.Z
        self.factor(lam)
        A = np.empty((M, M))
        LU = np.empty((M, M))
        nv.check(self.lib.hevi_column_matrix(self.h, float(lam), A.ctypes.data_as(ctypes.c_void_p),
                                             LU.ctypes.data_as(ctypes.c_void_p), nv.stream_ptr()))
        return A, LU

    def solve(self, lam, qe, out):
        nv.check(self.lib.hevi_solve(self.h, float(lam), nv.ptr(qe), nv.ptr(out), nv.stream_ptr()))
        return out

    @property
    def chains_pp(self) -> bool:
        """Whether a fused step writes P'(Q^{n+1}) for the next step's stage 0
        (the explicit_col path), so steady stepping may pass pp_valid."""
        return bool(self.lib.hevi_step_chains_pp(self.h))

    def pp_refresh(self, Q, work):
        """P'(Q) into work's Q1 field 0 (the plane a chained stage 0 reads)."""
        nv.check(self.lib.hevi_pp_refresh(self.h, nv.ptr(Q), nv.ptr(work), nv.stream_ptr()))

    def step(self, dt, tab: np.ndarray, Q, work, pp_valid=False):
        """One fused ARK2 step; ``pp_valid``: work's Q1 field 0 already holds
        P'(Q) (written by the previous chained step or pp_refresh)."""
        nv.check(self.lib.hevi_ark2_step_ex(self.h, float(dt), _dp(tab), nv.ptr(Q), nv.ptr(work),
                                            nv.STEP_PP_VALID if pp_valid else 0, nv.stream_ptr()))

    def rk35(self, dt, Q, work):
        nv.check(self.lib.hevi_rk35_step(self.h, float(dt), nv.ptr(Q), nv.ptr(work), nv.stream_ptr()))

    def stage(self, s, dt, tab: np.ndarray, Q, work, pp_valid=False, part=None):
        """One explicit stage; ``part`` = "interior" | "boundary" evaluates the
        tiles that read no neighbour-provided halo point (before the halo
        exchange) or the rest (after it); None: the whole stage."""
        flags = nv.STEP_PP_VALID if pp_valid else 0
        if part == "interior":
            flags |= nv.STAGE_INTERIOR
        elif part == "boundary":
            flags |= nv.STAGE_BOUNDARY
        elif part is not None:
            raise ValueError(f"unknown stage part {part!r}")
        nv.check(self.lib.hevi_stage_ex(self.h, s, float(dt), _dp(tab), nv.ptr(Q), nv.ptr(work),
                                        flags, nv.stream_ptr()))

    def stage_tiles(self):
        """(interior, boundary) tile counts of the column-sweep stage kernels."""
        a, b = ctypes.c_int(), ctypes.c_int()
        nv.check(self.lib.hevi_stage_tiles(self.h, ctypes.byref(a), ctypes.byref(b)))
        return a.value, b.value

    def stage_solve(self, s, lam, work):
        nv.check(self.lib.hevi_stage_solve(self.h, s, float(lam), nv.ptr(work), nv.stream_ptr()))

    # -- 3D-IMEX operators (imex3d.cuh) ------------------------------------------
    def linear3(self, q, out):
        nv.check(self.lib.hevi_linear3(self.h, nv.ptr(q), nv.ptr(out), nv.stream_ptr()))
        return out

    def schur3_up(self, lam, P, up, vertical_only=False):
        nv.check(self.lib.hevi_schur3_up(self.h, float(lam), int(vertical_only), nv.ptr(P), nv.ptr(up),
                                         nv.stream_ptr()))
        return up

    def schur3_flux(self, lam, P, vel, out, vertical_only=False):
        nv.check(self.lib.hevi_schur3_flux(self.h, float(lam), int(vertical_only), nv.ptr(P),
                                           nv.ptr(vel), nv.ptr(out), nv.stream_ptr()))
        return out

    def schur3_ua(self, lam, qe, ua, Pe):
        nv.check(self.lib.hevi_schur3_ua(self.h, float(lam), nv.ptr(qe), nv.ptr(ua), nv.ptr(Pe),
                                         nv.stream_ptr()))

    def schur3_extract(self, lam, P, ua, up, qe, q, vertical_only=False):
        # the box's grad theta0 is vertical: advecting by the vertical part of
        # the velocity or by all of it is the same product (imexcore.py:280-297)
        nv.check(self.lib.hevi_schur3_extract(self.h, float(lam), nv.ptr(P), nv.ptr(ua), nv.ptr(up),
                                              nv.ptr(qe), nv.ptr(q), nv.stream_ptr()))
        return q

    def wdot(self, x, y, nf=1) -> float:
        out = np.zeros(1)
        nv.check(self.lib.hevi_wdot(self.h, nv.ptr(x), nv.ptr(y), int(nf),
                                    out.ctypes.data_as(ctypes.c_void_p), nv.stream_ptr()))
        return float(out[0])

    def axpby(self, alpha, x, beta, y):
        """y <- alpha x + beta y (whole padded arrays)."""
        nv.check(self.lib.hevi_axpby(y.numel(), float(alpha), nv.ptr(x), float(beta), nv.ptr(y),
                                     nv.stream_ptr()))
        return y

    def flags(self, reset=True) -> int:
        f = ctypes.c_uint(0)
        nv.check(self.lib.hevi_flags(self.h, ctypes.byref(f), int(reset), nv.stream_ptr()))
        return f.value

    def check_flags(self):
        raise_for_flags(self.flags(reset=True))

    # -- reference-facing entry: E-vector in, E-vector out ------------------------
    #: opt-in check that drop-in inputs are DSS-continuous (every copy of a
    #: lattice point bitwise equal): the lattice keeps the first-occurrence
    #: copy (columnsolve.unique_space rep), so a discontinuous E-vector would
    #: silently give a different answer from the reference
    check_continuity = False

    def lattice_in(self, q, reuse=False):
        """E-vector (numpy / torch, host or device) -> (lattice tensor, back),
        ``back`` returning the result in the caller's array type.  With
        ``reuse`` the lattice is the plan's persistent buffer (overwritten by
        the next call).  (Gathering the unique copies straight from pinned
        host memory was measured no faster than the DMA copy: PCIe sectors
        make the strided gather read as many bytes, profiles/README.md.)"""
        E, back0 = to_device(q)
        if E.shape != (5,) + tuple(self.mesh.nshape):
            raise ValueError("field/mesh shape mismatch")
        if reuse:
            if getattr(self, "_lat", None) is None:
                self._lat = self.zeros()
            L = self.e2l(E, out=self._lat)
        else:
            L = self.e2l(E)
        if self.check_continuity:
            back_e = self.l2e(L)
            if not bool((back_e == E).all()):
                raise ValueError("E-vector input is not DSS-continuous: coincident node copies "
                                 "differ (the reference would average them; apply specgrid.apply_dss first)")
        return L, (lambda L_: back0(self.l2e(L_)))

    # -- E-vector entry used by the drop-in operators ---------------------------
    def apply_evec(self, op, q, lam=None):
        E, back = to_device(q)
        if E.shape != (5,) + tuple(self.mesh.nshape):
            raise ValueError("field/mesh shape mismatch")
        L = self.e2l(E)
        out = self.zeros()
        if op == "rhs":
            self.rhs(L, out)
        elif op == "linear":
            self.linear(L, out)
        elif op == "linear3":
            self.linear3(L, out)
        elif op == "solve":
            self.solve(lam, L, out)
        else:
            raise ValueError(op)
        self.check_flags()
        return back(self.l2e(out))


def to_device(q):
    """E-vector (numpy or torch) -> contiguous fp64 CUDA tensor, plus a
    function returning results in the caller's array type."""
    import torch
    if isinstance(q, torch.Tensor):
        dev = q.device
        t = q.to(device="cuda", dtype=torch.float64).contiguous()
        if dev.type == "cuda":
            return t, (lambda r: r)

        def back(r):
            # host results land in (cached) pinned memory: full-bandwidth D2H
            out = torch.empty(r.shape, dtype=r.dtype, pin_memory=True)
            out.copy_(r)
            return out
        return t, back
    arr = np.ascontiguousarray(q, dtype=np.float64)
    t = torch.from_numpy(arr).to("cuda")
    return t, (lambda r: r.cpu().numpy())


def tableau_array(tab) -> np.ndarray:
    """{a, at, b} of a ButcherPair packed as the C ABI expects."""
    a = np.asarray(tab.a, dtype=np.float64)
    at = np.asarray(tab.at, dtype=np.float64)
    b = np.asarray(tab.b, dtype=np.float64)
    if a.shape != (3, 3) or at.shape != (3, 3) or b.shape != (3,):
        raise ValueError("the fused HEVI step needs a 3-stage ARK pair")
    return np.ascontiguousarray(np.concatenate([a.ravel(), at.ravel(), b]))
