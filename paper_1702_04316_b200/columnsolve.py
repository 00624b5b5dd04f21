"""Direct solution of the vertically-implicit problem (drop-in for
``dycore.columnsolve``, columnsolve.py:1-210).

Two device paths sit behind the reference API:

* ``solve_direct(problem, q_e)`` -- the production path: the Schur column
  operator is probed and LU-factored once per ``round(lam, 12)`` on the
  device (one factor shared by all columns: on box meshes every column
  carries the same matrix, SURVEY finding 5, asserted in the tests), and
  the fused column kernel builds the Schur RHS, substitutes and extracts.
* ``build_column_jacobian`` / ``lu_factor_banded`` /
  ``solve_columns_direct`` -- the reference's batched per-column API on
  arbitrary ``(n_col, M, M)`` matrices, run by the generic banded kernels
  (column-interleaved band storage, one thread per column).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native as nv


@dataclass
class UniqueSpace:
    """columnsolve.py:18-25 (uid/rep materialised lazily: they are E-vector
    sized index maps, only needed by callers that gather by hand)."""
    mesh: object
    n_col: int
    n_lev: int
    shape: tuple

    def _maps(self):
        m = self.mesh
        nel, nt, ns, nr = m.nshape
        e = np.arange(nel)
        kx = e % m.nx
        ky = (e // m.nx) % m.ny
        kz = e // (m.nx * m.ny)
        gx = kx[:, None, None, None] * m.N + np.arange(nr)[None, None, None, :]
        gy = ky[:, None, None, None] * m.Ny + np.arange(ns)[None, None, :, None]
        gz = kz[:, None, None, None] * m.N + np.arange(nt)[None, :, None, None]
        col = gx if m.slab else gy * m.X + gx
        uid = (np.broadcast_to(col, self.shape).astype(np.int64) * self.n_lev
               + np.broadcast_to(gz, self.shape)).ravel()
        vals, rep = np.unique(uid, return_index=True)
        return uid, rep

    @property
    def uid(self):
        return self._maps()[0]

    @property
    def rep(self):
        return self._maps()[1]


def unique_space(mesh) -> UniqueSpace:
    return UniqueSpace(mesh=mesh, n_col=mesh.n_col, n_lev=mesh.n_lev, shape=tuple(mesh.nshape))


@dataclass
class ColumnJacobian:
    """columnsolve.py:37-49.  ``matrices`` is a CUDA tensor (n_col, M, M),
    overwritten by the LU factors like the reference."""
    matrices: object
    bandwidth: int
    n_dof: int
    space: UniqueSpace
    factored: bool = False
    pivoted_fallback: list = None
    piv: dict = None
    band: object = None          # device band storage after factoring
    lu: object = None            # pivoted fallback: (n_col, M, M) LU factors
    lu_piv: object = None        # pivoted fallback: (n_col, M) int32 interchanges
    lu_info: object = None       # pivoted fallback: getrf-style info per column

    @property
    def M(self) -> int:
        return self.matrices.shape[1]


def _unique_apply(problem, space: UniqueSpace, n_dof: int):
    """Vertical LHS as an operator on (n_col, n_lev, n_dof) unique values
    (columnsolve.py:52-72), Schur form: the values are laid on the lattice
    (unique (column, level) points), lhs_schur runs on the device
    (hevi_schur3_up + hevi_schur3_flux, vertical-only derivatives)."""
    import torch
    if n_dof != 1:
        raise NotImplementedError("the device path implements the Schur (pressure) form")
    mesh = problem.disc.mesh
    plan = problem.disc.plan_for(problem.ref, problem.set_name)
    Z, Y, X = mesh.Z, mesh.Y, mesh.X

    def apply_u(U):
        Ut = torch.as_tensor(np.asarray(U) if not isinstance(U, torch.Tensor) else U,
                             dtype=torch.float64, device=plan.device).reshape(space.n_col, space.n_lev)
        if mesh.slab:
            P = Ut.t()[:, None, :].expand(Z, Y, X)
        else:
            P = Ut.t().reshape(Z, Y, X)
        L = plan.padded(P[None].contiguous())
        lam = float(problem.lam)
        up = plan.schur3_up(lam, L[0], plan.zeros(3), True)
        out = plan.schur3_flux(lam, L[0], up, plan.zeros(1)[0], True)
        O = out[:, :, :X]
        O = O[:, 0, :] if mesh.slab else O.reshape(Z, Y * X)
        res = O.t().reshape(space.n_col, space.n_lev, 1)
        return res if isinstance(U, torch.Tensor) else res.cpu().numpy()
    return apply_u


def _leakage_check(problem, space):
    """Probing one column must not touch any other (columnsolve.py:94-101)."""
    import torch
    apply_u = _unique_apply(problem, space, 1)
    U = torch.zeros((space.n_col, space.n_lev, 1), dtype=torch.float64, device="cuda")
    U[0, space.n_lev // 2, 0] = 1.0
    out = apply_u(U)
    if float(out[1:].abs().max()) > 1e-13 * max(1.0, float(out[0].abs().max())):
        raise RuntimeError("cross-column leakage detected in the vertical operator; "
                           "columns are not independent")


def build_column_jacobian(problem) -> ColumnJacobian:
    """Probe the Schur column operator (columnsolve.py:75-108) on the device.

    The probe runs on one column; box meshes have identical columns, so the
    matrix is broadcast to all n_col columns."""
    import torch
    if problem.dim != "1d":
        raise ValueError("column Jacobians require the 1D implicit form")
    if problem.form != "schur":
        raise NotImplementedError("the device path implements the Schur (pressure) form")
    plan = problem.disc.plan_for(problem.ref, problem.set_name)
    lam = float(problem.lam)
    space = unique_space(problem.disc.mesh)
    if getattr(problem.disc.mesh, "kind", "box") == "sphere":
        # general mesh: every column probed on the device (leakage check included)
        if lam == 0.0:
            mats = torch.eye(space.n_lev, dtype=torch.float64, device=plan.device).expand(
                space.n_col, -1, -1).contiguous()
            return ColumnJacobian(matrices=mats, bandwidth=1, n_dof=1, space=space, pivoted_fallback=[], piv={})
        nb, _ = plan.factor(lam)
        mats = torch.as_tensor(plan.column_matrix(lam, -1), device=plan.device)
        return ColumnJacobian(matrices=mats, bandwidth=nb, n_dof=1, space=space, pivoted_fallback=[], piv={})
    if lam == 0.0:
        A = np.eye(space.n_lev)
        nb = 1
    else:
        A, _ = plan.column_matrix(lam)
        nb = plan.factor(lam)
        _leakage_check(problem, space)
    mats = torch.as_tensor(A, device=plan.device).expand(space.n_col, -1, -1).contiguous()
    return ColumnJacobian(matrices=mats, bandwidth=nb, n_dof=1, space=space,
                          pivoted_fallback=[], piv={})


def lu_factor_banded(cj: ColumnJacobian):
    """In-place no-pivot banded LU, batched over columns (columnsolve.py:111-138)."""
    import torch
    if cj.factored:
        raise ValueError("already factored")
    lib = nv.load()
    A = cj.matrices
    if not isinstance(A, torch.Tensor) or not A.is_cuda:
        A = torch.as_tensor(np.asarray(A, dtype=np.float64), device="cuda")
    A = A.to(torch.float64).contiguous()
    n_col, M, _ = A.shape
    nb = int(cj.bandwidth)
    s = nv.stream_ptr()
    norm = np.zeros(1)
    nv.check(lib.hevi_absmax(nv.ptr(A), A.numel(), norm.ctypes.data_as(
        ctypes.POINTER(ctypes.c_double)), s))
    band = torch.empty((2 * nb - 1, M, n_col), dtype=torch.float64, device=A.device)
    nv.check(lib.hevi_band_pack(nv.ptr(A), nv.ptr(band), n_col, M, nb, s))
    bad = ctypes.c_int(-1)
    nv.check(lib.hevi_band_lu(nv.ptr(band), n_col, M, nb, float(norm[0]),
                              ctypes.byref(bad), s))
    if bad.value >= 0:
        raise RuntimeError(f"no-pivot LU hit a degenerate diagonal in column(s) [{bad.value}]")
    # factors back into the dense matrices, in place (entries outside the band
    # are untouched by the reference's banded elimination)
    dense = torch.empty_like(A)
    nv.check(lib.hevi_band_unpack(nv.ptr(band), nv.ptr(dense), n_col, M, nb, s))
    inband = _band_mask(M, nb, A.device)
    A.copy_(torch.where(inband, dense, A))
    cj.matrices = A
    cj.band = band
    cj.factored = True


def _band_mask(M, nb, device):
    import torch
    i = torch.arange(M, device=device)
    return ((i[:, None] - i[None, :]).abs() < nb)[None]


def lu_factor_pivoted(cj: ColumnJacobian):
    """The pivoted dense fallback of factor_with_fallback (columnsolve.py:148-152):
    partial-pivoting LU of every column on the device (scipy.linalg.lu_factor
    semantics); ``cj.piv[c] = (lu, piv)`` per column like the reference."""
    import torch
    lib = nv.load()
    A = cj.matrices
    if not isinstance(A, torch.Tensor) or not A.is_cuda:
        A = torch.as_tensor(np.asarray(A, dtype=np.float64), device="cuda")
    lu = A.to(torch.float64).contiguous().clone()
    n_col, M, _ = lu.shape
    piv = torch.empty((n_col, M), dtype=torch.int32, device=lu.device)
    info = np.zeros(n_col, dtype=np.int32)
    nv.check(lib.hevi_lu_pivot(nv.ptr(lu), nv.ptr(piv), n_col, M,
                               info.ctypes.data_as(ctypes.c_void_p), nv.stream_ptr()))
    cj.lu, cj.lu_piv, cj.lu_info = lu, piv, info
    cj.piv = {c: (lu[c], piv[c]) for c in range(n_col)}
    cj.pivoted_fallback = list(range(n_col))
    cj.factored = True
    return cj


def factor_with_fallback(problem) -> ColumnJacobian:
    """columnsolve.py:141-153: build and factor, keeping a pivoted dense LU of
    every column if the no-pivot banded LU hits a degenerate diagonal.  The
    fused step's shared factor takes the same fallback inside hevi_factor."""
    cj = build_column_jacobian(problem)
    backup = cj.matrices.clone()
    try:
        lu_factor_banded(cj)
    except RuntimeError:
        cj.matrices = backup
        lu_factor_pivoted(cj)
    return cj


def solve_columns_direct(cj: ColumnJacobian, rhs):
    """Banded forward/backward substitution, batched over columns
    (columnsolve.py:156-181); rhs (n_col, M) numpy or torch."""
    import torch
    if not cj.factored:
        raise ValueError("factor before solving")
    lib = nv.load()
    was_np = not isinstance(rhs, torch.Tensor)
    t = torch.as_tensor(np.asarray(rhs, dtype=np.float64) if was_np else rhs)
    dev = t.device
    x = t.to(device="cuda", dtype=torch.float64).contiguous().clone()
    n_col, M = x.shape
    if cj.pivoted_fallback:    # columnsolve.py:163-167
        nv.check(lib.hevi_lu_pivot_solve(nv.ptr(cj.lu), nv.ptr(cj.lu_piv), nv.ptr(x), n_col, M,
                                         nv.stream_ptr()))
        return x.cpu().numpy() if was_np else x.to(dev)
    nv.check(lib.hevi_band_solve(nv.ptr(cj.band), nv.ptr(x), n_col, M, int(cj.bandwidth),
                                 nv.stream_ptr()))
    if was_np:
        return x.cpu().numpy()
    return x.to(dev)


def get_factors(problem) -> ColumnJacobian:
    """Factor cache keyed by (round(lam, 12), form) (columnsolve.py:184-188)."""
    key = (round(problem.lam, 12), problem.form)
    if key not in problem._column_cache:
        problem._column_cache[key] = factor_with_fallback(problem)
    return problem._column_cache[key]


def standard_column_factor(problem):
    """Shared band LU of the standard-form column operator I - lam L_V
    (M = 5 n_lev unknowns, unknown lev*5 + field; half band 5N+3, SURVEY
    8(a) a17), cached per (round(lam, 12), "standard") like get_factors.
    Probed as the reference does (columnsolve.py:75-108): one device
    application of L_V per unknown with the unit vector in every column (box
    columns are identical), the response of one interior column assembled."""
    import torch
    key = (round(problem.lam, 12), "standard")
    if key in problem._column_cache:
        return problem._column_cache[key]
    plan = problem.disc.plan_for(problem.ref, problem.set_name)
    mesh = problem.disc.mesh
    lam = float(problem.lam)
    Z, X = mesh.Z, mesh.X
    M = 5 * Z
    gx, gy = X // 2, (0 if mesh.slab else mesh.Y // 2)
    U, out = plan.zeros(), plan.zeros()
    A = np.zeros((M, M))
    for lev in range(Z):
        for d in range(5):
            U.zero_()
            U[d, lev, :, :X] = 1.0
            plan.linear(U, out)
            plan.axpby(1.0, U, -lam, out)                 # U - lam L_V(U)
            A[:, lev * 5 + d] = out[:, :, gy, gx].T.reshape(-1).cpu().numpy()
    plan.check_flags()
    scale = np.abs(A).max()
    rows, cols = np.nonzero(np.abs(A) > 1e-14 * scale)
    nb = int(np.abs(rows - cols).max()) + 1 if len(rows) else 1
    lib = nv.load()
    At = torch.as_tensor(A[None], device=plan.device).contiguous()
    band = torch.empty((2 * nb - 1, M, 1), dtype=torch.float64, device=plan.device)
    s = nv.stream_ptr()
    nv.check(lib.hevi_band_pack(nv.ptr(At), nv.ptr(band), 1, M, nb, s))
    bad = ctypes.c_int(-1)
    nv.check(lib.hevi_band_lu(nv.ptr(band), 1, M, nb, float(scale), ctypes.byref(bad), s))
    if bad.value >= 0:
        raise RuntimeError("no-pivot LU of the standard-form column hit a degenerate diagonal")
    ent = (A, band, nb)
    problem._column_cache[key] = ent
    return ent


def solve_direct(problem, q_e):
    """One direct implicit solve (columnsolve.py:191-210): the fused device
    column kernel with the shared per-lam factor (Schur form), or the
    standard-form column substitution on the lattice."""
    plan = problem.disc.plan_for(problem.ref, problem.set_name)
    if problem.form == "standard":
        from .plan import to_device
        _, band, nb = standard_column_factor(problem)
        E, back = to_device(q_e)
        Qe = plan.e2l(E)
        q = plan.zeros()
        nv.check(plan.lib.hevi_std_solve(plan.h, nv.ptr(band), 5 * plan.Z, nb, nv.ptr(Qe), nv.ptr(q),
                                         nv.stream_ptr()))
        return back(plan.l2e(q))
    return plan.apply_evec("solve", q_e, lam=float(problem.lam))
