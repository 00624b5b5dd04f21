"""CPU oracle for the HEVI 1D-IMEX ARK2 step -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference`` arm) may import this module.
The shipped package ``paper_1702_04316_b200`` never imports it; the product
path fails loudly when its CUDA library is missing instead of falling back
to anything here.

What it is: a numpy restatement, on element-local ("E-vector") arrays of
shape ``(5, nel, nqt, nqs, nqr)``, of the reference package ``dycore``
(``/root/reference/pkg/src/dycore``) along the path BASELINE.json names:
cG, equation set ``set2nc``, Schur (pressure) form, vertically-implicit
(``dim='1d'``) direct column solve, ARK2 stepper.  Every routine cites the
reference lines it follows.  Meshes are the structured boxes the path is
benchmarked on: the reference's own 2D slab (``specgrid.build_box_mesh``,
degree-1 dummy y layer) and the SURVEY.md section 8(c) harness 3D box.

Parity of this restatement is pinned against fixtures produced by running
the unmodified reference (``tests/golden/make_golden.py``); see
``tests/test_oracle_golden.py``.

Differences in *mechanism* (not in arithmetic) from the reference:
  * coincidence groups are found from the structured (gx, gy, gz) lattice
    index instead of a KD-tree (``specgrid._group_points``); the DSS sums
    still run in flat-node order through ``np.bincount`` exactly like
    ``specgrid.apply_dss`` (specgrid.py:535-540);
  * the no-flux projection zeroes the axis-normal velocity components,
    which is what the orthonormalised projectors of
    ``euler.boundary_projectors`` (euler.py:218-258) reduce to on an
    axis-aligned box (up to ~1e-16 off-diagonal round-off in the
    reference's metric-derived normals).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
from numpy.polynomial import legendre as npleg

# euler.py:23-36 (GasConstants)
C_P = 1004.5
C_V = 717.5
P_REF = 1.0e5
GRAV = 9.80616
R_GAS = C_P - C_V
GAMMA = C_P / C_V


# ---------------------------------------------------------------------------
# quadrature (specgrid.py:39-77)
# ---------------------------------------------------------------------------

def lgl(N: int):
    """Degree-N Legendre-Gauss-Lobatto nodes, weights, derivative matrix.

    specgrid.lgl_nodes_weights (specgrid.py:39-65): interior nodes are the
    Newton-refined roots of P_N' seeded with Chebyshev points; weights
    2/(N(N+1)P_N^2); derivative matrix from barycentric weights
    (specgrid.py:68-77).
    """
    if N < 1:
        raise ValueError("polynomial degree must be >= 1")
    basis = np.zeros(N + 1)
    basis[N] = 1.0
    if N == 1:
        nodes = np.array([-1.0, 1.0])
    else:
        d1 = npleg.legder(basis)
        d2 = npleg.legder(d1)
        xi = np.cos(np.pi * np.arange(N - 1, 0, -1) / N)
        for _ in range(100):
            step = npleg.legval(xi, d1) / npleg.legval(xi, d2)
            xi = xi - step
            if np.max(np.abs(step)) < 1e-15:
                break
        nodes = np.concatenate(([-1.0], np.sort(xi), [1.0]))
    weights = 2.0 / (N * (N + 1) * npleg.legval(nodes, basis) ** 2)
    gap = nodes[:, None] - nodes[None, :]
    np.fill_diagonal(gap, 1.0)
    bary = 1.0 / gap.prod(axis=1)
    D = (bary[None, :] / bary[:, None]) / gap
    np.fill_diagonal(D, 0.0)
    np.fill_diagonal(D, -D.sum(axis=1))
    return nodes, weights, D


# ---------------------------------------------------------------------------
# ARK2 tableau (imexcore.py:44-63)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class Tableau:
    a: np.ndarray
    at: np.ndarray
    b: np.ndarray

    @property
    def diag(self) -> float:
        return float(self.at[1, 1])


def ark2() -> Tableau:
    """Sign-corrected ARK2 pair used by the reference (imexcore.py:44-63)."""
    s2 = math.sqrt(2.0)
    gam = 1.0 - 1.0 / s2
    d = 1.0 / (2.0 * s2)
    a32 = (3.0 + 2.0 * s2) / 6.0
    a = np.array([[0.0, 0.0, 0.0], [2.0 - s2, 0.0, 0.0], [1.0 - a32, a32, 0.0]])
    at = np.array([[0.0, 0.0, 0.0], [gam, gam, 0.0], [d, d, gam]])
    return Tableau(a=a, at=at, b=np.array([d, d, gam]))


# ---------------------------------------------------------------------------
# structured box mesh on E-vectors
# ---------------------------------------------------------------------------

class BoxOracle:
    """Structured box: mesh, metrics, DSS, reference state and operators.

    ``slab=True`` reproduces ``specgrid.build_box_mesh`` (specgrid.py:173-231):
    nx-by-nz elements in x-z, one dummy y layer of degree 1 spanning
    [0, Ly] (Ly = Lx/nx by default), columns keyed by x only.
    ``slab=False`` is the SURVEY section 8(c) harness 3D box: degree N on
    all three axes, element e = (kz*ny + ky)*nx + kx, columns keyed by (x, y).
    """

    def __init__(self, nx, ny, nz, Lx, Ly, Lz, N, slab=False,
                 background="hydrostatic", theta_bg=300.0, set_name="set2nc",
                 pprime="reference"):
        if set_name not in ("set2nc", "set2c"):
            raise ValueError(set_name)
        if pprime not in ("reference", "exact"):
            raise ValueError(pprime)
        self.set_name = set_name
        # "reference": P' = eos(rho, theta) - P0f exactly as euler.py:456-457 /
        # 479-480 (cancellation leaves ~eps*P0 ~ 1e-11 Pa of noise in P').
        # "exact": the same P' evaluated without cancellation,
        # Pb*expm1(gamma*log1p(delta)) + (Pb - P0f) with Pb = eos(rho0, theta0)
        # and delta the relative perturbation of rho*theta -- the quantity the
        # device series computes; a tighter checker for the kernels.
        self.pprime = pprime
        if slab:
            ny = 1
            if Ly is None:
                Ly = Lx / nx
        self.nx, self.ny, self.nz, self.N, self.slab = nx, ny, nz, N, slab
        self.Lx, self.Ly, self.Lz = Lx, Ly, Lz
        self.Nr, self.Ns, self.Nt = N, (1 if slab else N), N
        self.nr, self.nq_s, self.nt = self.Nr + 1, self.Ns + 1, self.Nt + 1
        self.qr = lgl(self.Nr)
        self.qs = lgl(self.Ns)
        self.qt = lgl(self.Nt)
        self.nel = nx * ny * nz
        self.nshape = (self.nel, self.nt, self.nq_s, self.nr)
        self._build_coords()
        self._build_metrics()
        self._build_dss()
        self._build_reference(background, theta_bg)
        self._column_cache = {}

    # -- geometry ----------------------------------------------------------
    def _build_coords(self):
        """Node coordinates (specgrid.py:185-201 for the slab)."""
        xe = np.linspace(0.0, self.Lx, self.nx + 1)
        ye = np.linspace(0.0, self.Ly, self.ny + 1)
        ze = np.linspace(0.0, self.Lz, self.nz + 1)
        nr_, ns_, nt_ = self.qr[0], self.qs[0], self.qt[0]
        coords = np.empty(self.nshape + (3,))
        gidx = np.empty(self.nshape + (3,), dtype=np.int64)
        for kz in range(self.nz):
            zs = ze[kz] + (nt_ + 1.0) * 0.5 * (ze[kz + 1] - ze[kz])
            for ky in range(self.ny):
                if self.slab:
                    ys = np.array([0.0, self.Ly])
                else:
                    ys = ye[ky] + (ns_ + 1.0) * 0.5 * (ye[ky + 1] - ye[ky])
                for kx in range(self.nx):
                    e = (kz * self.ny + ky) * self.nx + kx
                    xs = xe[kx] + (nr_ + 1.0) * 0.5 * (xe[kx + 1] - xe[kx])
                    coords[e, ..., 0] = xs[None, None, :]
                    coords[e, ..., 1] = ys[None, :, None]
                    coords[e, ..., 2] = zs[:, None, None]
                    gidx[e, ..., 0] = (kx * self.Nr + np.arange(self.nr))[None, None, :]
                    gidx[e, ..., 1] = (ky * self.Ns + np.arange(self.nq_s))[None, :, None]
                    gidx[e, ..., 2] = (kz * self.Nt + np.arange(self.nt))[:, None, None]
        self.coords = coords
        self.X = self.nx * self.Nr + 1
        self.Y = self.ny * self.Ns + 1
        self.Z = self.nz * self.Nt + 1
        gx, gy, gz = gidx[..., 0], gidx[..., 1], gidx[..., 2]
        self.gx, self.gy, self.gz = gx, gy, gz
        # coincidence groups (specgrid.build_dss_map) on the lattice
        self.gid = ((gz * self.Y + gy) * self.X + gx).ravel()
        self.n_lev = self.Z
        # columns: slab keyed by x only (specgrid.py:203-204), 3D by (x, y)
        col = gx if self.slab else gy * self.X + gx
        self.n_col = self.X if self.slab else self.X * self.Y
        # unique (column, level) space (columnsolve.py:28-34)
        self.uid = (col.astype(np.int64) * self.n_lev + gz).ravel()
        _, self.rep = np.unique(self.uid, return_index=True)
        _, self.grep = np.unique(self.gid, return_index=True)
        self.height = coords[..., 2].copy()

    def _d(self, f, axis):
        """Tensor-product derivative along local axis (specgrid.py:391-401)."""
        if axis == 0:
            return f @ self.qr[2].T
        if axis == 1:
            return np.swapaxes(np.swapaxes(f, -2, -1) @ self.qs[2].T, -2, -1)
        ne, nt, ns, nr = f.shape
        return (self.qt[2] @ f.reshape(ne, nt, ns * nr)).reshape(f.shape)

    def _build_metrics(self):
        """Per-node inverse coordinate Jacobian (specgrid.py:404-430)."""
        c = self.coords
        xr = np.stack([self._d(c[..., m], 0) for m in range(3)], axis=-1)
        xs = np.stack([self._d(c[..., m], 1) for m in range(3)], axis=-1)
        xt = np.stack([self._d(c[..., m], 2) for m in range(3)], axis=-1)
        Jm = np.stack([xr, xs, xt], axis=-1)
        J = np.linalg.det(Jm)
        if np.any(J <= 0):
            raise ValueError("degenerate or inverted element")
        Ji = np.linalg.inv(Jm)
        self.a = [np.ascontiguousarray(Ji[..., d, m]) for d in range(3) for m in range(3)]
        self.a_t = Ji[..., 2, :]
        wr, ws, wt = self.qr[1], self.qs[1], self.qt[1]
        w3 = wt[:, None, None] * ws[None, :, None] * wr[None, None, :]
        self.wJ = w3[None, ...] * J
        self.vert = np.zeros(self.nshape + (3,))
        self.vert[..., 2] = 1.0
        self.Jtv = np.einsum("ekjic,ekjic->ekji", self.a_t, self.vert)

    def metric(self, d, m):
        """a_<d>[..., m] (MetricTerms.comp, specgrid.py:343-351)."""
        return self.a[3 * d + m]

    def _build_dss(self):
        """DSS weights (specgrid.py:523-532)."""
        self.w = self.wJ.ravel()
        self.ng = self.X * self.Y * self.Z
        self.wsum = np.bincount(self.gid, weights=self.w, minlength=self.ng)
        bx = (self.gx == 0) | (self.gx == self.X - 1)
        by = (self.gy == 0) | (self.gy == self.Y - 1)
        bz = (self.gz == 0) | (self.gz == self.Z - 1)
        if self.slab:
            by = np.ones_like(by)      # every y face of the slab is lateral
        self.bmask = [bx, by, bz]

    def dss(self, f):
        """Mass-weighted average of coincident nodes (specgrid.py:535-540)."""
        num = np.bincount(self.gid, weights=self.w * f.ravel(), minlength=self.ng)
        return (num / self.wsum)[self.gid].reshape(self.nshape)

    def dss_many(self, q):
        return np.stack([self.dss(q[i]) for i in range(q.shape[0])])

    def no_flux(self, vel):
        """Zero normal velocity on boundary nodes (euler.py:261-264)."""
        out = vel.copy()
        for m in range(3):
            out[m][self.bmask[m]] = 0.0
        return out

    # -- reference state (euler.py:125-177) ---------------------------------
    def _build_reference(self, background, theta_bg):
        h = self.height
        g = GRAV
        if background == "hydrostatic":
            if theta_bg <= 0:
                raise ValueError("background potential temperature must be positive")
            pi = 1.0 - g * h / (C_P * theta_bg)
            if np.any(pi <= 0):
                raise ValueError("domain too tall for this background temperature")
            P0f = P_REF * pi ** (C_P / R_GAS)
            rho0 = P0f / (R_GAS * theta_bg * pi)
            theta0 = np.full_like(h, theta_bg)
            dpi = -g / (C_P * theta_bg)
            drho0 = rho0 * (C_P / R_GAS - 1.0) * dpi / pi
            dth0 = np.zeros_like(h)
        elif background == "isothermal":
            T = theta_bg
            pi = np.exp(-g * h / (C_P * T))
            P0f = P_REF * pi ** (C_P / R_GAS)
            rho0 = P0f / (R_GAS * T)
            theta0 = T / pi
            drho0 = -rho0 * g / (R_GAS * T)
            dth0 = (g / C_P) / pi
        else:
            raise ValueError(background)
        self.background = background
        self.rho0, self.theta0, self.P0f = rho0, theta0, P0f
        self.grad_rho0 = drho0[..., None] * self.vert
        self.grad_theta0 = dth0[..., None] * self.vert
        self.gvec = g * self.vert
        # set2nc coefficients (euler.py:82-100)
        self.G0 = GAMMA * P0f / rho0
        self.H0 = GAMMA * P0f / theta0
        self.F0vec = self.G0[..., None] * self.grad_rho0 + self.H0[..., None] * self.grad_theta0
        # set2c coefficients (euler.py:102-122)
        self.Theta0 = rho0 * theta0
        self.F0c = GAMMA * P0f / self.Theta0

    # -- pointwise pieces -----------------------------------------------------
    @staticmethod
    def eos(rho, theta):
        """euler.equation_of_state (euler.py:180-185)."""
        if np.any(rho <= 0) or np.any(theta <= 0):
            raise ValueError("EOS requires positive density and temperature")
        return P_REF * (rho * R_GAS * theta / P_REF) ** GAMMA

    def pprime_of(self, q):
        """Perturbation pressure P' of the state q for the chosen set."""
        rho = self.rho0 + q[0]
        if self.set_name == "set2c":
            theta = (self.Theta0 + q[4]) / rho
        else:
            theta = self.theta0 + q[4]
        if self.pprime == "reference":
            return self.eos(rho, theta) - self.P0f
        self.eos(rho, theta)          # same positivity checks
        rt0 = self.rho0 * self.theta0
        if self.set_name == "set2c":
            delta = q[4] / self.Theta0
        else:
            delta = (q[0] * self.theta0 + self.rho0 * q[4] + q[0] * q[4]) / rt0
        Pb = self.eos(self.rho0, self.theta0)
        return Pb * np.expm1(GAMMA * np.log1p(delta)) + (Pb - self.P0f)

    def grad(self, f):
        """specgrid.grad (specgrid.py:600-611)."""
        fr, fs, ft = self._d(f, 0), self._d(f, 1), self._d(f, 2)
        out = np.empty(f.shape + (3,))
        for m in range(3):
            gm = fr * self.metric(0, m)
            gm += fs * self.metric(1, m)
            gm += ft * self.metric(2, m)
            out[..., m] = gm
        return out

    def div(self, vec):
        """specgrid.div (specgrid.py:614-622); vec has a trailing axis 3."""
        out = np.zeros(vec.shape[:-1])
        for m in range(3):
            vm = np.ascontiguousarray(vec[..., m])
            out += self._d(vm, 0) * self.metric(0, m)
            out += self._d(vm, 1) * self.metric(1, m)
            out += self._d(vm, 2) * self.metric(2, m)
        return out

    def dvert(self, f):
        """DSS'd vertical derivative (euler.py:292-300, specgrid.py:625-627)."""
        return self.dss(self.Jtv * self._d(f, 2))

    # -- R(q): euler.nonlinear_rhs, cG set2nc (euler.py:438-473, 492-497) ----
    def rhs(self, q):
        if np.any(~np.isfinite(q)):
            raise FloatingPointError("non-finite state passed to RHS evaluation")
        if self.set_name == "set2c":
            return self._rhs_c(q)
        u = np.moveaxis(q[1:4], 0, -1)
        rho = self.rho0 + q[0]
        Pp = self.pprime_of(q)
        divu = self.div(u)

        def advect(f, g0=None):
            a = np.einsum("...a,...a->...", u, self.grad(f))
            if g0 is not None:
                a = a + np.einsum("...a,...a->...", u, g0)
            return a

        out = np.empty_like(q)
        out[0] = -(advect(q[0], self.grad_rho0) + rho * divu)
        gPp = self.grad(Pp)
        mom = -(np.stack([advect(q[m]) for m in (1, 2, 3)], axis=-1)
                + gPp / rho[..., None] + (q[0] / rho)[..., None] * self.gvec)
        out[1:4] = np.moveaxis(mom, -1, 0)
        out[4] = -advect(q[4], self.grad_theta0)
        out = self.dss_many(out)
        out[1:4] = self.no_flux(out[1:4])
        return out

    def _rhs_c(self, q):
        """euler.nonlinear_rhs set2c flux form (euler.py:474-487, 492-497)."""
        U = np.moveaxis(q[1:4], 0, -1)
        rho = self.rho0 + q[0]
        Theta = self.Theta0 + q[4]
        theta = Theta / rho
        Pp = self.pprime_of(q)
        out = np.empty_like(q)
        out[0] = -self.div(U)
        for m in range(3):
            Fm = U[..., m][..., None] * U / rho[..., None]
            Fm[..., m] += Pp
            out[1 + m] = -self.div(Fm)
        out[1:4] -= np.moveaxis(q[0][..., None] * self.gvec, -1, 0)
        out[4] = -self.div(theta[..., None] * U)
        out = self.dss_many(out)
        out[1:4] = self.no_flux(out[1:4])
        return out

    # -- L_V(q): linear_operator(vertical_only=True) (euler.py:313-371)
    def linear(self, q):
        if self.set_name == "set2c":
            return self._linear_c(q)
        vel = np.moveaxis(q[1:4], 0, -1)
        P = self.G0 * q[0] + self.H0 * q[4]
        gradP = self.dvert(P)[..., None] * self.vert
        vv = np.einsum("...a,...a->...", vel, self.vert)
        divU = self.dvert(vv)
        adv = vv[..., None] * self.vert
        out = np.zeros_like(q)
        out[0] = -(np.einsum("...a,...a->...", adv, self.grad_rho0) + self.rho0 * divU)
        mom = -(gradP / self.rho0[..., None] + (q[0] / self.rho0)[..., None] * self.gvec)
        out[4] = -np.einsum("...a,...a->...", adv, self.grad_theta0)
        mom = np.einsum("...a,...a->...", mom, self.vert)[..., None] * self.vert
        out[1:4] = self.no_flux(np.moveaxis(mom, -1, 0))
        return out

    def _linear_c(self, q):
        """set2c branch of linear_operator, vertical only (euler.py:350-361)."""
        vel = np.moveaxis(q[1:4], 0, -1)
        P = self.F0c * q[4]
        gradP = self.dvert(P)[..., None] * self.vert
        vv = np.einsum("...a,...a->...", vel, self.vert)
        divU = self.dvert(vv)
        adv = vv[..., None] * self.vert
        out = np.zeros_like(q)
        out[0] = -divU
        mom = -(gradP + q[0][..., None] * self.gvec)
        out[4] = -(self.theta0 * divU + np.einsum("...a,...a->...", adv, self.grad_theta0))
        mom = np.einsum("...a,...a->...", mom, self.vert)[..., None] * self.vert
        out[1:4] = self.no_flux(np.moveaxis(mom, -1, 0))
        return out

    # -- Schur pieces (imexcore.py:200-298), dim='1d' -------------------------
    def ainv(self, v, lam):
        """Sherman-Morrison inverse of I + lam^2 u w^T (imexcore.py:200-217)."""
        w = self.grad_theta0
        if not np.any(w):
            return v
        u = (lam ** 2 / self.theta0)[..., None] * self.gvec
        den = 1.0 + np.einsum("...a,...a->...", w, u)
        if np.any(np.abs(den) < 1e-12):
            raise FloatingPointError("rank-one inverse denominator underflow")
        wv = np.einsum("...a,...a->...", w, v)
        return v - u * (wv / den)[..., None]

    def _nf(self, vec):
        return np.moveaxis(self.no_flux(np.moveaxis(vec, -1, 0)), 0, -1)

    def helm(self, vel, lam):
        """imexcore._helmholtz_flux (imexcore.py:259-268)."""
        vv = np.einsum("...a,...a->...", vel, self.vert)
        if self.set_name == "set2c":
            return self.F0c * lam * (self.theta0 * self.dvert(vv)
                                     + np.einsum("...a,...a->...", self.grad_theta0, vel))
        return lam * (np.einsum("...a,...a->...", self.F0vec, vel)
                      + self.rho0 * self.G0 * self.dvert(vv))

    def up(self, P, lam):
        """imexcore._up set2nc (imexcore.py:245-257)."""
        gP = self.dvert(P)[..., None] * self.vert
        if self.set_name == "set2c":
            v = self.ainv(lam * (gP + (P / (self.F0c * self.theta0))[..., None] * self.gvec), lam)
        else:
            v = self.ainv(lam * (gP / self.rho0[..., None]
                                 + (P / (self.G0 * self.rho0))[..., None] * self.gvec), lam)
        return self._nf(v)

    def schur_rhs(self, qe, lam):
        """imexcore.rhs_schur_build set2nc (imexcore.py:229-243)."""
        vel = np.moveaxis(qe[1:4], 0, -1)
        if self.set_name == "set2c":
            Pe = self.F0c * qe[4]
            ua = self._nf(self.ainv(vel - (lam * (qe[0] - qe[4] / self.theta0))[..., None]
                                    * self.gvec, lam))
            return Pe - self.helm(ua, lam), ua
        Pe = self.G0 * qe[0] + self.H0 * qe[4]
        coef = lam * self.H0 / (self.G0 * self.rho0)
        ua = self._nf(self.ainv(vel + (coef * qe[4])[..., None] * self.gvec, lam))
        return Pe - self.helm(ua, lam), ua

    def lhs_schur(self, P, lam):
        """imexcore.lhs_schur (imexcore.py:270-271)."""
        return P - self.helm(self.up(P, lam), lam)

    # -- 3D-IMEX pieces, dim='3d' (euler.py:281-290, 313-365; imexcore.py:229-271)
    def gradc(self, f):
        """Discretization.gradc: DSS of every gradient component (euler.py:281-286)."""
        g = self.grad(f)
        return np.stack([self.dss(np.ascontiguousarray(g[..., m])) for m in range(3)], axis=-1)

    def divc(self, vec):
        """Discretization.divc (euler.py:288-290)."""
        return self.dss(self.div(vec))

    def linear3(self, q):
        """euler.linear_operator, vertical_only=False, cG (euler.py:313-365)."""
        vel = np.moveaxis(q[1:4], 0, -1)
        if self.set_name == "set2c":
            P = self.F0c * q[4]
        else:
            P = self.G0 * q[0] + self.H0 * q[4]
        gradP = self.gradc(P)
        divU = self.divc(vel)
        out = np.zeros_like(q)
        if self.set_name == "set2c":
            out[0] = -divU
            mom = -(gradP + q[0][..., None] * self.gvec)
            out[4] = -(self.theta0 * divU + np.einsum("...a,...a->...", vel, self.grad_theta0))
        else:
            out[0] = -(np.einsum("...a,...a->...", vel, self.grad_rho0) + self.rho0 * divU)
            mom = -(gradP / self.rho0[..., None] + (q[0] / self.rho0)[..., None] * self.gvec)
            out[4] = -np.einsum("...a,...a->...", vel, self.grad_theta0)
        out[1:4] = self.no_flux(np.moveaxis(mom, -1, 0))
        return out

    def helm3(self, vel, lam):
        """imexcore._helmholtz_flux with divc (imexcore.py:259-268)."""
        if self.set_name == "set2c":
            return self.F0c * lam * (self.theta0 * self.divc(vel)
                                     + np.einsum("...a,...a->...", self.grad_theta0, vel))
        return lam * (np.einsum("...a,...a->...", self.F0vec, vel)
                      + self.rho0 * self.G0 * self.divc(vel))

    def up3(self, P, lam):
        """imexcore._up with gradc (imexcore.py:245-257)."""
        gP = self.gradc(P)
        if self.set_name == "set2c":
            v = self.ainv(lam * (gP + (P / (self.F0c * self.theta0))[..., None] * self.gvec), lam)
        else:
            v = self.ainv(lam * (gP / self.rho0[..., None]
                                 + (P / (self.G0 * self.rho0))[..., None] * self.gvec), lam)
        return self._nf(v)

    def schur_rhs3(self, qe, lam):
        """rhs_schur_build, dim='3d' (imexcore.py:229-243)."""
        vel = np.moveaxis(qe[1:4], 0, -1)
        if self.set_name == "set2c":
            Pe = self.F0c * qe[4]
            ua = self._nf(self.ainv(vel - (lam * (qe[0] - qe[4] / self.theta0))[..., None]
                                    * self.gvec, lam))
        else:
            Pe = self.G0 * qe[0] + self.H0 * qe[4]
            coef = lam * self.H0 / (self.G0 * self.rho0)
            ua = self._nf(self.ainv(vel + (coef * qe[4])[..., None] * self.gvec, lam))
        return Pe - self.helm3(ua, lam), ua

    def lhs_schur3(self, P, lam):
        """lhs_schur, dim='3d' (imexcore.py:270-271)."""
        return P - self.helm3(self.up3(P, lam), lam)

    def extract(self, P, ua, qe, lam):
        """imexcore.extract_from_pressure set2nc, 1d (imexcore.py:273-287)."""
        vel = ua - self.up(P, lam)
        q = np.empty_like(qe)
        q[1:4] = np.moveaxis(vel, -1, 0)
        uv = np.einsum("...a,...a->...", vel, self.vert)
        adv = uv[..., None] * self.vert
        if self.set_name == "set2c":   # imexcore.py:288-297
            q[4] = P / self.F0c
            q[0] = (P / (self.F0c * self.theta0)
                    + lam / self.theta0 * np.einsum("...a,...a->...", adv, self.grad_theta0)
                    - qe[4] / self.theta0 + qe[0])
            return q
        q[4] = qe[4] - lam * np.einsum("...a,...a->...", adv, self.grad_theta0)
        q[0] = (P - self.H0 * q[4]) / self.G0
        return q

    # -- column direct solver (columnsolve.py) -------------------------------
    def column_matrices(self, lam):
        """Probe the Schur column operator (columnsolve.py:52-108)."""
        nc, nl = self.n_col, self.n_lev
        A = np.zeros((nc, nl, nl))
        for lev in range(nl):
            U = np.zeros((nc, nl))
            U[:, lev] = 1.0
            P = U.reshape(-1)[self.uid].reshape(self.nshape)
            A[:, :, lev] = self.lhs_schur(P, lam).ravel()[self.rep].reshape(nc, nl)
        scale = np.abs(A).max()
        rows, cols = np.nonzero((np.abs(A) > 1e-14 * scale).any(axis=0))
        nb = int(np.abs(rows - cols).max()) + 1 if len(rows) else 1
        return A, nb

    @staticmethod
    def band_lu(A, nb):
        """In-place no-pivot banded Doolittle LU (columnsolve.py:111-138)."""
        M = A.shape[1]
        norm = np.abs(A).max()
        bad = set()
        for k in range(M):
            piv = A[:, k, k]
            small = np.abs(piv) < 1e-12 * norm
            if np.any(small):
                bad.update(np.nonzero(small)[0].tolist())
                piv = np.where(small, 1.0, piv)
            E = min(k + nb, M)
            if E > k + 1:
                A[:, k + 1:E, k] /= piv[:, None]
                A[:, k + 1:E, k + 1:E] -= A[:, k + 1:E, k:k + 1] * A[:, k:k + 1, k + 1:E]
        if bad:
            raise RuntimeError(f"no-pivot LU hit a degenerate diagonal in column(s) {sorted(bad)}")
        return A

    @staticmethod
    def band_solve(LU, nb, rhs):
        """Batched banded substitution (columnsolve.py:156-181)."""
        M = LU.shape[1]
        y = rhs.copy()
        for i in range(1, M):
            j0 = max(0, i - nb + 1)
            y[:, i] -= np.einsum("cj,cj->c", LU[:, i, j0:i], y[:, j0:i])
        for i in range(M - 1, -1, -1):
            j1 = min(i + nb, M)
            if j1 > i + 1:
                y[:, i] -= np.einsum("cj,cj->c", LU[:, i, i + 1:j1], y[:, i + 1:j1])
            y[:, i] /= LU[:, i, i]
        return y

    @staticmethod
    def pivoted_factors(A):
        """factor_with_fallback's pivoted dense path (columnsolve.py:148-152):
        scipy.linalg.lu_factor per column."""
        import scipy.linalg
        return [scipy.linalg.lu_factor(A[c]) for c in range(A.shape[0])]

    @staticmethod
    def pivoted_solve(F, rhs):
        """solve_columns_direct's pivoted branch (columnsolve.py:163-167)."""
        import scipy.linalg
        return np.stack([scipy.linalg.lu_solve(F[c], rhs[c]) for c in range(rhs.shape[0])])

    def factors(self, lam, force_pivoted=False):
        """columnsolve.get_factors cache keyed by round(lam, 12) (:184-188),
        factor_with_fallback (:141-153): (LU, nb) or ("pivoted", factors)."""
        key = (round(lam, 12), force_pivoted)
        if key not in self._column_cache:
            A, nb = self.column_matrices(lam)
            backup = A.copy()
            try:
                if force_pivoted:
                    raise RuntimeError("forced")
                self._column_cache[key] = (self.band_lu(A, nb), nb)
            except RuntimeError:
                self._column_cache[key] = ("pivoted", self.pivoted_factors(backup))
        return self._column_cache[key]

    def solve(self, qe, lam):
        """ImplicitProblem.solve direct branch (imexcore.py:312-322) ->
        columnsolve.solve_direct (columnsolve.py:191-210)."""
        if lam <= 0:
            raise ValueError("implicit solve requires positive lam")
        LU, nb = self.factors(lam, getattr(self, "force_pivoted", False))
        rhsP, ua = self.schur_rhs(qe, lam)
        rhs = rhsP.ravel()[self.rep].reshape(self.n_col, self.n_lev)
        if isinstance(LU, str):
            sol = self.pivoted_solve(nb, rhs)
        else:
            sol = self.band_solve(LU, nb, rhs)
        P = sol.reshape(-1)[self.uid].reshape(self.nshape)
        return self.extract(P, ua, qe, lam)

    # -- ARK2 step (imexcore.py:385-414) -------------------------------------
    def step(self, q, dt, tab=None):
        tab = tab or ark2()
        R = [self.rhs(q)]
        L = [self.linear(q)]
        lam = tab.diag * dt
        for i in (1, 2):
            pred = q.copy()
            for j in range(i):
                pred += dt * (tab.a[i, j] * (R[j] - L[j]) + tab.at[i, j] * L[j])
            qi = self.solve(pred, lam)
            R.append(self.rhs(qi))
            if i < 2:
                L.append(self.linear(qi))
        out = q.copy()
        for i in range(3):
            out += dt * tab.b[i] * R[i]
        if np.any(~np.isfinite(out)):
            raise FloatingPointError("non-finite state after IMEX step")
        return out

    # -- SSP RK(5,3) explicit step (imexcore.py:79-126) -----------------------
    _RK_A = {(1, 0): 1.0, (2, 1): 1.0, (3, 0): 0.355909775063327, (3, 2): 0.644090224936674,
             (4, 0): 0.367933791638137, (4, 3): 0.632066208361863,
             (5, 2): 0.237593836598569, (5, 4): 0.762406163401431}
    _RK_B = {(1, 0): 0.377268915331368, (2, 1): 0.377268915331368, (3, 2): 0.242995220537396,
             (4, 3): 0.238458932846290, (5, 4): 0.287632146308408}

    def rk35(self, q, dt):
        u = [q]
        for i in range(1, 6):
            acc = np.zeros_like(q)
            for j in range(i):
                al = self._RK_A.get((i, j), 0.0)
                be = self._RK_B.get((i, j), 0.0)
                if al != 0.0:
                    acc += al * u[j]
                if be != 0.0:
                    acc += (be * dt) * self.rhs(u[j])
            u.append(acc)
        if np.any(~np.isfinite(u[5])):
            raise FloatingPointError("non-finite state in explicit stage")
        return u[5]

    # -- helpers -------------------------------------------------------------
    def min_node_spacing(self):
        """euler.min_node_spacing (euler.py:583-593)."""
        c = self.coords
        d_r = np.linalg.norm(np.diff(c, axis=3), axis=-1).min()
        d_t = np.linalg.norm(np.diff(c, axis=1), axis=-1).min()
        if self.slab:
            return float(d_r), float(d_t)
        d_s = np.linalg.norm(np.diff(c, axis=2), axis=-1).min()
        return float(min(d_r, d_s)), float(d_t)

    def dt_for_courant(self, q, courant):
        """cli.run_simulation dt rule (cli.py:187-194, euler.py:564-580)."""
        rho = self.rho0 + q[0]
        vel = np.moveaxis(q[1:4], 0, -1)
        if self.set_name == "set2c":     # euler.py:572-574
            vel = vel / rho[..., None]
            theta = (self.Theta0 + q[4]) / rho
        else:
            theta = self.theta0 + q[4]
        P = self.eos(rho, theta)
        cmax = float(np.max(np.linalg.norm(vel, axis=-1) + np.sqrt(GAMMA * P / rho)))
        _, dx_v = self.min_node_spacing()
        return courant * dx_v / cmax

    def bubble(self, theta_c=0.5, centre=(500.0, 0.0, 350.0), radii=(250.0, 250.0, 250.0)):
        """Cosine theta' bump with P' = 0 (bench.py:108-124, extended to an
        ellipsoid in 3D as SURVEY 8(c)/(d) describes), DSS'd like cli.py:180."""
        c = self.coords
        if self.slab:
            r = np.sqrt(((c[..., 0] - centre[0]) / radii[0]) ** 2
                        + ((c[..., 2] - centre[2]) / radii[2]) ** 2)
        else:
            r = np.sqrt(((c[..., 0] - centre[0]) / radii[0]) ** 2
                        + ((c[..., 1] - centre[1]) / radii[1]) ** 2
                        + ((c[..., 2] - centre[2]) / radii[2]) ** 2)
        th = np.where(r <= 1.0, 0.5 * theta_c * (1.0 + np.cos(np.pi * r)), 0.0)
        q = np.zeros((5,) + self.nshape)
        q[0] = self.rho0 * (self.theta0 / (self.theta0 + th) - 1.0)
        q[4] = th
        return self.dss_many(q)

    # -- E <-> unique lattice ------------------------------------------------
    def to_lattice(self, q):
        """(5, nel, ...) -> (5, Z, Y, X) taking the first-occurrence copy."""
        flat = q.reshape(q.shape[0], -1)
        return flat[:, self.grep].reshape(q.shape[0], self.Z, self.Y, self.X)

    def from_lattice(self, ql):
        flat = ql.reshape(ql.shape[0], -1)
        return flat[:, self.gid].reshape((ql.shape[0],) + self.nshape)
