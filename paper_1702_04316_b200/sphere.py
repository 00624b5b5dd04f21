"""General curvilinear element meshes: the cubed-sphere shell (SURVEY 8(f)
rank 4) on the device.

The structured box path folds the DSS into a unique-point lattice; a
cubed-sphere shell has no global lattice (its six panels meet at edges and
corners), so this module keeps the reference's E-vector layout
``(nf, nel, nqt, nqs, nqr)`` and hands the device plan (``hevi_gplan``,
csrc/general.cuh) exactly the per-node data the reference's operators read:

* ``build_cubed_sphere_mesh`` -- the equiangular gnomonic shell of
  specgrid.py:257-306 (same node coordinates), with the reference's
  coincidence groups for the DSS, radial columns and height levels;
* ``compute_metrics`` -- specgrid.compute_metrics (:404-455): contravariant
  vectors by inverting the per-node coordinate Jacobian, wJ, Jtv, the
  boundary-face normals;
* ``boundary_projectors`` -- euler.boundary_projectors (:218-258);
* ``NodeReferenceState`` -- euler.hydrostatic_reference / isothermal_reference
  (:125-177) per node;
* ``SphereDiscretization`` / ``GPlan`` -- the device operators: R(q), L_V(q),
  the per-column probed Schur factors, the direct solve, ARK2 and RK35 steps.

Set-up (geometry, grouping, ordering) is host NumPy, as in the reference;
every operator evaluation runs in libhevi.so.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import specgrid as sg


# ---------------------------------------------------------------------------
# mesh
# ---------------------------------------------------------------------------

@dataclass
class ElementMesh:
    """A general element mesh (specgrid.ElementMesh, kind "sphere")."""
    kind: str
    N: int
    quad_r: sg.Quadrature1D
    quad_s: sg.Quadrature1D
    quad_t: sg.Quadrature1D
    coords: np.ndarray        # (nel, nqt, nqs, nqr, 3)
    vert: np.ndarray          # radial unit vector per node
    height: np.ndarray        # |x| - r_e
    col_id: np.ndarray
    lev_id: np.ndarray
    n_col: int
    n_lev: int
    boundary_faces: list
    meta: dict = field(default_factory=dict)

    @property
    def nel(self) -> int:
        return self.coords.shape[0]

    @property
    def nshape(self):
        return self.coords.shape[:4]

    @property
    def n_nodes(self) -> int:
        return int(np.prod(self.nshape))


# face directions of the six cube panels for tan(alpha) = X, tan(beta) = Y:
# four equatorial panels, then the +z and -z caps (specgrid.py:247-254)
def _panel_direction(p, X, Y):
    one = np.ones_like(X)
    return [(one, X, Y), (-X, one, Y), (-one, -X, Y), (X, -one, Y), (-Y, X, one), (Y, X, -one)][p]


def _group_points(points: np.ndarray, tol: float) -> np.ndarray:
    """Group ids of coincident points (within tol), numbered by first
    occurrence.  1D values: split the sorted values at gaps > tol; 3D points:
    connected components of the pairs within tol (k-d tree)."""
    n = points.shape[0]
    if points.shape[1] == 1:
        v = points[:, 0]
        order = np.argsort(v, kind="stable")
        brk = np.concatenate([[True], np.diff(v[order]) > tol])
        comp = np.empty(n, dtype=np.int64)
        comp[order] = np.cumsum(brk) - 1
    else:
        from scipy.spatial import cKDTree
        from scipy.sparse import coo_matrix
        from scipy.sparse.csgraph import connected_components
        pairs = cKDTree(points).query_pairs(r=tol, output_type="ndarray")
        if len(pairs) == 0:
            comp = np.arange(n)
        else:
            adj = coo_matrix((np.ones(len(pairs)), (pairs[:, 0], pairs[:, 1])), shape=(n, n))
            comp = connected_components(adj, directed=False)[1]
    # renumber by first occurrence
    _, first = np.unique(comp, return_index=True)
    label = np.empty(len(first), dtype=np.int64)
    label[np.argsort(first)] = np.arange(len(first))
    return label[comp]


def _columns_levels(col, lev, height):
    """Levels renumbered bottom to top by their mean height."""
    n_col = int(col.max()) + 1
    n_lev = int(lev.max()) + 1
    mean = np.bincount(lev, weights=height, minlength=n_lev) / np.bincount(lev, minlength=n_lev)
    rank = np.empty(n_lev, dtype=np.int64)
    rank[np.argsort(mean)] = np.arange(n_lev)
    return col.astype(np.int64), rank[lev], n_col, n_lev


def build_cubed_sphere_mesh(ne_panel: int, ne_vert: int, r_e: float, r_T: float, N: int) -> ElementMesh:
    """Equiangular gnomonic cubed-sphere shell over [r_e, r_e + r_T]
    (specgrid.py:257-306).  Element order: panel, beta row, alpha column,
    then the ne_vert radial layers (radial index fastest)."""
    if ne_panel < 1 or ne_vert < 1:
        raise ValueError("element counts must be >= 1")
    q = sg.lgl_nodes_weights(N)
    nq = N + 1
    nel = 6 * ne_panel * ne_panel * ne_vert
    coords = np.empty((nel, nq, nq, nq, 3))
    edges = np.linspace(-np.pi / 4, np.pi / 4, ne_panel + 1)
    shells = np.linspace(r_e, r_e + r_T, ne_vert + 1)
    t01 = (q.nodes + 1.0) * 0.5
    e = 0
    for p in range(6):
        for kb in range(ne_panel):
            b = edges[kb] + t01 * (edges[kb + 1] - edges[kb])
            for ka in range(ne_panel):
                a = edges[ka] + t01 * (edges[ka + 1] - edges[ka])
                A, B = np.meshgrid(a, b, indexing="xy")   # rows: s (beta), columns: r (alpha)
                dx, dy, dz = _panel_direction(p, np.tan(A), np.tan(B))
                nrm = np.sqrt(dx * dx + dy * dy + dz * dz)
                d = np.stack([dx / nrm, dy / nrm, dz / nrm], axis=-1)
                for kr in range(ne_vert):
                    r = shells[kr] + t01 * (shells[kr + 1] - shells[kr])
                    coords[e + kr] = r[:, None, None, None] * d[None, :, :, :]
                e += ne_vert
    rad = np.linalg.norm(coords, axis=-1)
    vert = coords / rad[..., None]
    height = rad - r_e
    col = _group_points(vert.reshape(-1, 3), 1e-9)
    lev = _group_points(height.reshape(-1, 1), 1e-8 * (r_e + r_T))
    col_id, lev_id, n_col, n_lev = _columns_levels(col, lev, height.ravel())
    shape = (nel, nq, nq, nq)
    bfaces = []
    for el in range(nel):
        kr = el % ne_vert
        if kr == 0:
            bfaces.append((el, 2, 0, "bottom"))
        if kr == ne_vert - 1:
            bfaces.append((el, 2, 1, "top"))
    return ElementMesh(kind="sphere", N=N, quad_r=q, quad_s=q, quad_t=q, coords=coords, vert=vert,
                       height=height, col_id=col_id.reshape(shape), lev_id=lev_id.reshape(shape),
                       n_col=n_col, n_lev=n_lev, boundary_faces=bfaces,
                       meta={"ne_panel": ne_panel, "ne_vert": ne_vert, "r_e": r_e, "r_T": r_T})


# ---------------------------------------------------------------------------
# metric terms, DSS groups, projectors
# ---------------------------------------------------------------------------

def _d_r(f, D):
    return f @ D.T


def _d_s(f, D):
    return np.swapaxes(np.swapaxes(f, -2, -1) @ D.T, -2, -1)


def _d_t(f, D):
    ne, nt, ns, nr = f.shape
    return (D @ f.reshape(ne, nt, ns * nr)).reshape(f.shape)


@dataclass
class FaceNormals:
    elem: int
    axis: int
    side: int
    tag: str
    normal: np.ndarray   # (na, nb, 3) outward unit normal


@dataclass
class GeneralMetrics:
    """specgrid.MetricTerms (:331-385) for a general mesh."""
    J: np.ndarray
    a_r: np.ndarray
    a_s: np.ndarray
    a_t: np.ndarray
    wJ: np.ndarray
    Jtv: np.ndarray
    bfaces: list


def _face_sel(mesh, axis, side):
    nq = mesh.N + 1
    idx = nq - 1 if side == 1 else 0
    return {0: (slice(None), slice(None), idx), 1: (slice(None), idx, slice(None)),
            2: (idx, slice(None), slice(None))}[axis]


def compute_metrics(mesh: ElementMesh) -> GeneralMetrics:
    """Contravariant vectors from the inverse of the per-node coordinate
    Jacobian (specgrid.compute_metrics, :404-455)."""
    D = mesh.quad_r.D
    c = mesh.coords
    cols = [np.stack([op(c[..., m], D) for m in range(3)], axis=-1) for op in (_d_r, _d_s, _d_t)]
    Jm = np.stack(cols, axis=-1)                   # [..., component, direction]
    J = np.linalg.det(Jm)
    if np.any(J <= 0):
        bad = np.argwhere(J.reshape(mesh.nel, -1).min(axis=1) <= 0).ravel()
        raise ValueError(f"degenerate or inverted element(s): {bad.tolist()}")
    Ji = np.linalg.inv(Jm)
    a_r, a_s, a_t = Ji[..., 0, :], Ji[..., 1, :], Ji[..., 2, :]
    w = mesh.quad_r.weights
    wJ = (w[:, None, None] * w[None, :, None] * w[None, None, :])[None] * J
    Jtv = np.einsum("ekjic,ekjic->ekji", a_t, mesh.vert)
    faces = []
    for (el, axis, side, tag) in mesh.boundary_faces:
        av = {0: a_r, 1: a_s, 2: a_t}[axis][el][_face_sel(mesh, axis, side)]
        mag = np.linalg.norm(av, axis=-1)
        faces.append(FaceNormals(el, axis, side, tag, (1.0 if side == 1 else -1.0) * av / mag[..., None]))
    return GeneralMetrics(J=J, a_r=a_r, a_s=a_s, a_t=a_t, wJ=wJ, Jtv=Jtv, bfaces=faces)


@dataclass
class GroupMap:
    """specgrid.DssMap (:510-532): coincidence groups and mass weights, plus
    the CSR the device DSS kernel walks (members in flat-node order)."""
    gid: np.ndarray
    w: np.ndarray
    wsum: np.ndarray
    n_groups: int
    shape: tuple
    rep: np.ndarray
    mult: np.ndarray
    ptr: np.ndarray = None
    idx: np.ndarray = None
    disc: object = None        # the discretization (its plan runs apply_dss)


def build_dss_map(mesh: ElementMesh, metrics: GeneralMetrics) -> GroupMap:
    scale = max(np.abs(mesh.coords).max(), 1.0)
    gid = _group_points(mesh.coords.reshape(-1, 3), 1e-8 * scale)
    w = metrics.wJ.ravel()
    ng = int(gid.max()) + 1
    wsum = np.bincount(gid, weights=w, minlength=ng)
    _, rep = np.unique(gid, return_index=True)
    mult = np.bincount(gid, minlength=ng)
    order = np.argsort(gid, kind="stable")            # members of each group in flat order
    ptr = np.concatenate([[0], np.cumsum(mult)]).astype(np.int32)
    return GroupMap(gid=gid, w=w, wsum=wsum, n_groups=ng, shape=mesh.nshape, rep=rep, mult=mult,
                    ptr=ptr, idx=order.astype(np.int32))


def boundary_projectors(mesh: ElementMesh, metrics: GeneralMetrics, dss: GroupMap):
    """(bidx, bproj) and the per-group projector slots (euler.py:218-258): the
    normals of every boundary face meeting at a physical point, gathered
    through its group and orthonormalised; P = I - sum b b^T."""
    nq = mesh.N + 1
    per = nq ** 3
    base = np.arange(per).reshape(nq, nq, nq)
    idx_l, nrm_l = [], []
    for fg in metrics.bfaces:
        idx_l.append(fg.elem * per + base[_face_sel(mesh, fg.axis, fg.side)].ravel())
        nrm_l.append(fg.normal.reshape(-1, 3))
    slot = np.full(dss.n_groups, -1, dtype=np.int32)
    if not idx_l:
        return np.zeros(0, dtype=np.int64), np.zeros((0, 3, 3)), slot, np.zeros((0, 3, 3))
    bidx = np.concatenate(idx_l)
    bnrm = np.concatenate(nrm_l)
    groups = dss.gid[bidx]
    order = np.argsort(groups, kind="stable")
    gs = groups[order]
    starts = np.flatnonzero(np.concatenate([[True], gs[1:] != gs[:-1]]))
    ends = np.concatenate([starts[1:], [len(gs)]])
    projs = np.empty((len(starts), 3, 3))
    for s, (a, b) in enumerate(zip(starts, ends)):
        basis = []
        for nv in bnrm[order[a:b]]:
            v = nv.copy()
            for bv in basis:
                v -= np.dot(v, bv) * bv
            nv_ = np.linalg.norm(v)
            if nv_ > 1e-8:
                basis.append(v / nv_)
        P = np.eye(3)
        for bv in basis:
            P -= np.outer(bv, bv)
        projs[s] = P
        slot[gs[a]] = s
    members = np.flatnonzero(slot[dss.gid] >= 0)
    return members.astype(np.int64), projs[slot[dss.gid[members]]], slot, projs


# ---------------------------------------------------------------------------
# per-node background state
# ---------------------------------------------------------------------------

@dataclass
class NodeReferenceState:
    """euler.ReferenceState (euler.py:70-122) with per-node arrays."""
    const: object
    kind: str
    rho0: np.ndarray
    theta0: np.ndarray
    P0f: np.ndarray
    grad_rho0: np.ndarray
    grad_theta0: np.ndarray
    gvec: np.ndarray
    mesh: object = None
    _cache: dict = field(default_factory=dict)

    def _c(self, k, fn):
        if k not in self._cache:
            self._cache[k] = fn()
        return self._cache[k]

    @property
    def G0_nc(self):
        return self._c("G0", lambda: self.const.gamma * self.P0f / self.rho0)

    @property
    def H0_nc(self):
        return self._c("H0", lambda: self.const.gamma * self.P0f / self.theta0)

    @property
    def F0vec_nc(self):
        return self._c("F0v", lambda: self.G0_nc[..., None] * self.grad_rho0
                       + self.H0_nc[..., None] * self.grad_theta0)

    @property
    def Theta0(self):
        return self._c("Th0", lambda: self.rho0 * self.theta0)

    @property
    def F0_c(self):
        return self._c("F0c", lambda: self.const.gamma * self.P0f / self.Theta0)

    @property
    def G0_c(self):
        return self.theta0

    @property
    def grad_G0_c(self):
        return self.grad_theta0

    def node(self, a):
        return np.asarray(a)


def hydrostatic_reference(mesh: ElementMesh, theta_bg: float, const) -> NodeReferenceState:
    """euler.py:125-150 on every node."""
    if theta_bg <= 0:
        raise ValueError("background potential temperature must be positive")
    c = const
    h = mesh.height
    pi = 1.0 - c.g * h / (c.c_p * theta_bg)
    if np.any(pi <= 0):
        raise ValueError("domain too tall for this background temperature")
    P0f = c.P0 * pi ** (c.c_p / c.R)
    rho0 = P0f / (c.R * theta_bg * pi)
    dpi = -c.g / (c.c_p * theta_bg)
    drho = rho0 * (c.c_p / c.R - 1.0) * dpi / pi
    return NodeReferenceState(const=c, kind="hydrostatic", rho0=rho0, theta0=np.full_like(h, theta_bg),
                              P0f=P0f, grad_rho0=drho[..., None] * mesh.vert,
                              grad_theta0=np.zeros(mesh.nshape + (3,)), gvec=c.g * mesh.vert, mesh=mesh)


def isothermal_reference(mesh: ElementMesh, T_bg: float, const) -> NodeReferenceState:
    """euler.py:153-177 on every node."""
    if T_bg <= 0:
        raise ValueError("background temperature must be positive")
    c = const
    h = mesh.height
    pi = np.exp(-c.g * h / (c.c_p * T_bg))
    P0f = c.P0 * pi ** (c.c_p / c.R)
    rho0 = P0f / (c.R * T_bg)
    drho = -rho0 * c.g / (c.R * T_bg)
    dth = (c.g / c.c_p) / pi
    return NodeReferenceState(const=c, kind="isothermal", rho0=rho0, theta0=T_bg / pi, P0f=P0f,
                              grad_rho0=drho[..., None] * mesh.vert, grad_theta0=dth[..., None] * mesh.vert,
                              gvec=c.g * mesh.vert, mesh=mesh)


# ---------------------------------------------------------------------------
# discretization and the device plan
# ---------------------------------------------------------------------------

def _cm(a):
    """(..., 3) per-node vectors -> component-major [3][nn] (C order)."""
    return np.ascontiguousarray(np.moveaxis(np.asarray(a, dtype=np.float64).reshape(-1, 3), -1, 0))


@dataclass
class SphereDiscretization:
    """euler.Discretization (:271-310) for a general mesh; the derivative
    methods run on the device."""
    mesh: ElementMesh
    metrics: GeneralMetrics
    dss: GroupMap
    bidx: np.ndarray
    bproj: np.ndarray
    gslot: np.ndarray
    projs: np.ndarray
    uid: np.ndarray
    urep: np.ndarray
    _plans: dict = field(default_factory=dict)

    def plan_for(self, ref: NodeReferenceState, set_name: str = "set2nc"):
        key = (id(ref), set_name)
        ent = self._plans.get(key)
        if ent is None or ent[0] is not ref:
            ent = (ref, GPlan(self, ref, set_name))
            self._plans[key] = ent
        return ent[1]

    def geometry_plan(self):
        for ref, plan in self._plans.values():
            return plan
        from . import euler
        return self.plan_for(isothermal_reference(self.mesh, 300.0, euler.GasConstants()))

    def _op(self, kind, f, vertical_only):
        from .plan import to_device
        plan = self.geometry_plan()
        T, back = to_device(f)
        return back(plan.grad(T, vertical_only) if kind == "grad" else plan.div(T, vertical_only))

    def gradc(self, f):
        return self._op("grad", f, False)

    def divc(self, vec):
        return self._op("div", vec, False)

    def grad_vc(self, f):
        return self._op("grad", f, True)

    def div_vc(self, vec):
        return self._op("div", vec, True)


def build_discretization(mesh: ElementMesh) -> SphereDiscretization:
    metrics = compute_metrics(mesh)
    dss = build_dss_map(mesh, metrics)
    bidx, bproj, gslot, projs = boundary_projectors(mesh, metrics, dss)
    uid = (mesh.col_id.astype(np.int64) * mesh.n_lev + mesh.lev_id).ravel()
    vals, urep = np.unique(uid, return_index=True)
    if len(vals) != mesh.n_col * mesh.n_lev:
        raise ValueError("column/level layout has holes")
    disc = SphereDiscretization(mesh=mesh, metrics=metrics, dss=dss, bidx=bidx, bproj=bproj, gslot=gslot,
                                projs=projs, uid=uid, urep=urep)
    dss.disc = disc
    return disc


def min_node_spacing(mesh: ElementMesh):
    """Minimal internodal distances (euler.py:583-593): horizontal over the r
    and s axes, vertical over t."""
    c = mesh.coords
    d_r = np.linalg.norm(np.diff(c, axis=3), axis=-1).min()
    d_s = np.linalg.norm(np.diff(c, axis=2), axis=-1).min()
    d_t = np.linalg.norm(np.diff(c, axis=1), axis=-1).min()
    return float(min(d_r, d_s)), float(d_t)


class GPlan:
    """Device plan of a general mesh + background + equation set
    (``hevi_gplan``); E-vectors in and out, fp64 CUDA tensors."""

    def __init__(self, disc: SphereDiscretization, ref: NodeReferenceState, set_name: str = "set2nc"):
        import torch
        from . import _native as nv
        if set_name not in ("set2nc", "set2c"):
            raise ValueError(f"unknown equation set {set_name!r}")
        nv.require_cuda()
        self.lib = nv.load()
        self.disc, self.ref, self.set_name = disc, ref, set_name
        self.mesh = disc.mesh
        self.shape = (5,) + tuple(self.mesh.nshape)
        self.nn = self.mesh.n_nodes
        self.device = torch.device("cuda")
        m, mt, ds = disc.mesh, disc.metrics, disc.dss
        c = ref.const
        keep = []

        def dp(a):
            a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
            keep.append(a)
            return a.ctypes.data_as(nv._DP)

        def ip(a):
            a = np.ascontiguousarray(np.asarray(a, dtype=np.int32))
            keep.append(a)
            return a.ctypes.data_as(nv._IP)

        md = nv.GMeshDesc()
        md.nel, md.N = m.nel, m.N
        md.D = dp(m.quad_r.D)
        md.ar, md.as_, md.at = dp(_cm(mt.a_r)), dp(_cm(mt.a_s)), dp(_cm(mt.a_t))
        md.vert, md.Jtv, md.w = dp(_cm(m.vert)), dp(mt.Jtv.ravel()), dp(ds.w)
        md.n_groups = ds.n_groups
        md.grp_ptr, md.grp_idx, md.grp_wsum = ip(ds.ptr), ip(ds.idx), dp(ds.wsum)
        md.n_proj = len(disc.projs)
        md.grp_slot = ip(disc.gslot)
        md.proj = dp(disc.projs.reshape(-1) if len(disc.projs) else np.zeros(9))
        md.n_col, md.n_lev = m.n_col, m.n_lev
        md.uid, md.rep = ip(disc.uid), ip(disc.urep)
        rd = nv.GRefDesc()
        rd.rho0, rd.theta0, rd.P0f = dp(ref.rho0.ravel()), dp(ref.theta0.ravel()), dp(ref.P0f.ravel())
        rd.grad_rho0, rd.grad_theta0, rd.gvec = dp(_cm(ref.grad_rho0)), dp(_cm(ref.grad_theta0)), dp(_cm(ref.gvec))
        rd.G0, rd.H0, rd.F0vec = dp(ref.G0_nc.ravel()), dp(ref.H0_nc.ravel()), dp(_cm(ref.F0vec_nc))
        rd.Theta0, rd.F0c = dp(ref.Theta0.ravel()), dp(ref.F0_c.ravel())
        # EOS of the background, the reference point of the P' series (euler.py:180-185)
        Pb = c.P0 * (ref.rho0 * c.R * ref.theta0 / c.P0) ** c.gamma
        rd.Pb = dp(Pb.ravel())
        rd.g, rd.R, rd.P0, rd.gamma = c.g, c.R, c.P0, c.gamma
        rd.eqset = 1 if set_name == "set2c" else 0
        h = ctypes.c_void_p()
        nv.check(self.lib.hevi_gplan_create(ctypes.byref(h), ctypes.byref(md), ctypes.byref(rd)))
        self.h = h
        self._ws = None

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self.lib.hevi_gplan_destroy(self.h)
                self.h = None
        except Exception:
            pass

    # -- buffers -----------------------------------------------------------------
    def zeros(self, nf=5):
        import torch
        return torch.zeros((nf,) + tuple(self.mesh.nshape), dtype=torch.float64, device=self.device)

    def workspace(self):
        import torch
        k = self.lib.hevi_g_work_fields(self.h)
        return torch.zeros((k,) + self.shape, dtype=torch.float64, device=self.device)

    def cached_workspace(self):
        if self._ws is None:
            self._ws = self.workspace()
        return self._ws

    def lattice_in(self, q, reuse=False):
        """The E-vector on the device (this path has no lattice) and the way back."""
        from .plan import to_device
        E, back = to_device(q)
        if tuple(E.shape) != self.shape:
            raise ValueError("field/mesh shape mismatch")
        return E.contiguous().clone(), back

    # -- operators ---------------------------------------------------------------
    def _s(self):
        from . import _native as nv
        return nv.stream_ptr()

    def rhs(self, q, out):
        from . import _native as nv
        nv.check(self.lib.hevi_g_rhs(self.h, nv.ptr(q), nv.ptr(out), self._s()))
        return out

    def linear(self, q, out):
        from . import _native as nv
        nv.check(self.lib.hevi_g_linear_v(self.h, nv.ptr(q), nv.ptr(out), self._s()))
        return out

    def factor(self, lam):
        from . import _native as nv
        nb, piv = ctypes.c_int(), ctypes.c_int()
        nv.check(self.lib.hevi_g_factor(self.h, float(lam), ctypes.byref(nb), ctypes.byref(piv), self._s()))
        return nb.value, bool(piv.value)

    def column_matrix(self, lam, col):
        """The probed (unfactored) Schur matrix of column ``col`` (all columns,
        (n_col, M, M), for col < 0)."""
        from . import _native as nv
        self.factor(lam)
        M = self.mesh.n_lev
        A = np.empty((M, M)) if col >= 0 else np.empty((self.mesh.n_col, M, M))
        nv.check(self.lib.hevi_g_column_matrix(self.h, float(lam), int(col), A.ctypes.data_as(ctypes.c_void_p),
                                               self._s()))
        return A

    def solve(self, lam, qe, out):
        from . import _native as nv
        self.factor(lam)
        nv.check(self.lib.hevi_g_solve(self.h, float(lam), nv.ptr(qe), nv.ptr(out), self._s()))
        return out

    def step(self, dt, tab, Q, work, pp_valid=False):
        from . import _native as nv
        tab = np.ascontiguousarray(tab, dtype=np.float64)
        nv.check(self.lib.hevi_g_ark2_step(self.h, float(dt), tab.ctypes.data_as(ctypes.c_void_p), nv.ptr(Q),
                                           nv.ptr(work), self._s()))

    def rk35(self, dt, Q, work):
        from . import _native as nv
        nv.check(self.lib.hevi_g_rk35_step(self.h, float(dt), nv.ptr(Q), nv.ptr(work), self._s()))

    def dss(self, f, out=None):
        from . import _native as nv
        f = f.contiguous()
        out = f.clone() if out is None else out
        nf = f.numel() // self.nn
        nv.check(self.lib.hevi_g_dss(self.h, nv.ptr(f), nv.ptr(out), nf, self._s()))
        return out

    def grad(self, f, vertical_only=False):
        """(..., ) scalar E-vector -> (..., 3) DSS-projected gradient."""
        from . import _native as nv
        f = f.contiguous()
        out = self.zeros(3)
        fn = self.lib.hevi_g_grad
        nv.check(fn(self.h, int(bool(vertical_only)), nv.ptr(f), nv.ptr(out), self._s()))
        return out.movedim(0, -1).contiguous()

    def div(self, vec, vertical_only=False):
        from . import _native as nv
        v = vec.movedim(-1, 0).contiguous()
        out = self.zeros(1)[0]
        nv.check(self.lib.hevi_g_div(self.h, int(bool(vertical_only)), nv.ptr(v), nv.ptr(out), self._s()))
        return out

    # -- the Krylov (3D-IMEX) path: the box plan's names, on E-vectors -----------
    def e2l(self, E, out=None, nf=None):
        """This path keeps E-vectors: identity (the box plan converts to its lattice)."""
        if out is None:
            return E.contiguous()
        out.copy_(E)
        return out

    def l2e(self, L, out=None):
        if out is None:
            return L
        out.copy_(L)
        return out

    def krylov_space(self, nf=1):
        from . import krylov
        return krylov.EvecSpace(self)

    def schur3_ua(self, lam, qe, ua, Pe):
        from . import _native as nv
        nv.check(self.lib.hevi_g_schur3_ua(self.h, float(lam), nv.ptr(qe), nv.ptr(ua), nv.ptr(Pe), self._s()))

    def schur3_up(self, lam, P, up, vertical_only=False):
        from . import _native as nv
        nv.check(self.lib.hevi_g_schur3_up(self.h, float(lam), int(vertical_only), nv.ptr(P), nv.ptr(up),
                                           self._s()))
        return up

    def schur3_flux(self, lam, P, vel, out, vertical_only=False):
        from . import _native as nv
        nv.check(self.lib.hevi_g_schur3_flux(self.h, float(lam), int(vertical_only), nv.ptr(P), nv.ptr(vel),
                                             nv.ptr(out), self._s()))
        return out

    def schur3_extract(self, lam, P, ua, up, qe, q, vertical_only=False):
        from . import _native as nv
        nv.check(self.lib.hevi_g_schur3_extract(self.h, float(lam), int(vertical_only), nv.ptr(P), nv.ptr(ua),
                                                nv.ptr(up), nv.ptr(qe), nv.ptr(q), self._s()))
        return q

    def linear3(self, q, out):
        from . import _native as nv
        nv.check(self.lib.hevi_g_linear3(self.h, nv.ptr(q), nv.ptr(out), self._s()))
        return out

    def wdot(self, x, y, nf=1) -> float:
        from . import _native as nv
        out = ctypes.c_double()
        nv.check(self.lib.hevi_g_dot(self.h, nv.ptr(x), nv.ptr(y), x.numel(), ctypes.byref(out), self._s()))
        return out.value

    def axpby(self, alpha, x, beta, y):
        from . import _native as nv
        nv.check(self.lib.hevi_axpby(y.numel(), float(alpha), nv.ptr(x), float(beta), nv.ptr(y), self._s()))
        return y

    def flags(self, reset=True) -> int:
        from . import _native as nv
        f = ctypes.c_uint()
        nv.check(self.lib.hevi_g_flags(self.h, ctypes.byref(f), int(reset), self._s()))
        return f.value

    def check_flags(self):
        from .plan import raise_for_flags
        raise_for_flags(self.flags())

    def apply_evec(self, op, q, lam=None):
        from .plan import to_device
        E, back = to_device(q)
        if tuple(E.shape) != self.shape:
            raise ValueError("field/mesh shape mismatch")
        E = E.contiguous()
        out = self.zeros()
        if op == "rhs":
            self.rhs(E, out)
        elif op == "linear":
            self.linear(E, out)
        elif op == "linear3":
            self.linear3(E, out)
        elif op == "solve":
            self.solve(lam, E, out)
        else:
            raise ValueError(f"unknown operator {op!r}")
        self.check_flags()
        return back(out)
