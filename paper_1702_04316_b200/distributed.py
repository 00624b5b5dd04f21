"""Horizontal column partitioning and halo exchange.

The lattice is cut along element boundaries into px x py blocks of whole
columns (vertical columns never split).  A rank owns the lattice points of
its elements (plus the domain's last point on the high side) and keeps a
window with a halo of N points on the low side and 1 point on the high side:
exactly what the explicit kernel's element lines reach.  Before each of the
three explicit stages the stage input (Q, Q1, A) is refreshed in the halos
with one grouped send/recv per neighbour (NCCL over NVLink when the backend
is ``nccl``).  The column solve needs no communication.  Every owned point is
computed by the same code from the same bits as on one GPU, so the
partitioned step is bitwise identical to the single-GPU step.
"""
from __future__ import annotations

from dataclasses import dataclass

from . import imexcore
from .plan import HeviPlan, tableau_array


def split(n: int, parts: int):
    """Element ranges of `parts` nearly equal blocks of n elements."""
    base, extra = divmod(n, parts)
    out, s = [], 0
    for p in range(parts):
        e = s + base + (1 if p < extra else 0)
        out.append((s, e))
        s = e
    return out


def grid_for(world: int):
    """px x py factorisation used for 1/2/4/8 ranks."""
    table = {1: (1, 1), 2: (2, 1), 4: (2, 2), 8: (4, 2), 16: (4, 4)}
    if world in table:
        return table[world]
    return world, 1


@dataclass
class Block:
    rank: int
    ix: int
    iy: int
    ex: tuple
    ey: tuple
    window: dict


def make_block(mesh, px: int, py: int, rank: int) -> Block:
    if mesh.slab and py != 1:
        raise ValueError("the slab has a single element across y: partition along x only")
    ix, iy = rank % px, rank // px
    ex = split(mesh.nx, px)[ix]
    ey = split(mesh.ny, py)[iy]
    if ex[0] == ex[1] or ey[0] == ey[1]:
        raise ValueError("more ranks than elements along an axis")
    N, Ny = mesh.N, mesh.Ny
    x0 = ex[0] * N - (N if ex[0] > 0 else 0)
    x1 = ex[1] * N + 1
    y0 = ey[0] * Ny - (Ny if ey[0] > 0 else 0)
    y1 = ey[1] * Ny + 1
    win = dict(x0=x0, y0=y0, lX=x1 - x0, lY=y1 - y0, ex_b=ex[0], ex_e=ex[1],
               ey_b=ey[0], ey_e=ey[1])
    return Block(rank=rank, ix=ix, iy=iy, ex=ex, ey=ey, window=win)


def halo_plan(mesh, px, py, rank):
    """List of transfers (peer, send_region, recv_region) for one rank, as
    phases.  Regions are (xlo, xhi, ylo, yhi) in GLOBAL lattice indices.

    One phase: the x halos over the owned rows and the y halos over the owned
    columns.  The explicit kernels never read a corner halo point (their x-lines
    and x-face partials lie on owned rows, their y-lines and y-face partials on
    owned columns), so no second phase is needed to fill corners; the
    partitioned-equals-single-GPU tests would catch any corner read (stale
    corners are never refreshed)."""
    me = make_block(mesh, px, py, rank)
    N, Ny = mesh.N, mesh.Ny
    oy0, oy1 = me.ey[0] * Ny, me.ey[1] * Ny + (1 if me.ey[1] == mesh.ny else 0)
    ox0, ox1 = me.ex[0] * N, me.ex[1] * N + (1 if me.ex[1] == mesh.nx else 0)
    phase = []
    if me.ix > 0:       # left neighbour owns [ex0*N - N, ex0*N); I own ex0*N (its high halo)
        L = rank - 1
        phase.append((L, (ox0, ox0 + 1, oy0, oy1), (ox0 - N, ox0, oy0, oy1)))
    if me.ix < px - 1:  # right neighbour owns ex1*N (my high halo); it needs my last N columns
        R = rank + 1
        x1 = me.ex[1] * N
        phase.append((R, (x1 - N, x1, oy0, oy1), (x1, x1 + 1, oy0, oy1)))
    if me.iy > 0:
        D = rank - px
        phase.append((D, (ox0, ox1, oy0, oy0 + 1), (ox0, ox1, oy0 - Ny, oy0)))
    if me.iy < py - 1:
        U = rank + px
        y1 = me.ey[1] * Ny
        phase.append((U, (ox0, ox1, y1 - Ny, y1), (ox0, ox1, y1, y1 + 1)))
    return me, [phase]


def _view(t, region, w):
    """Slice of a local (F, Z, lY, px) tensor for a global region."""
    xlo, xhi, ylo, yhi = region
    return t[:, :, ylo - w["y0"]:yhi - w["y0"], xlo - w["x0"]:xhi - w["x0"]]


def pack(plan, t, region, buf=None):
    """Region (global lattice indices) of a CUDA lattice tensor -> contiguous
    (nf, Z, ny, nx) buffer by the ``hevi_halo_pack`` kernel."""
    import torch
    from . import _native as nv
    xlo, xhi, ylo, yhi = region
    nf = t.shape[0]
    if buf is None:
        buf = torch.empty((nf, t.shape[1], yhi - ylo, xhi - xlo), dtype=t.dtype, device=t.device)
    nv.check(plan.lib.hevi_halo_pack(plan.h, nv.ptr(t), nf, xlo, xhi, ylo, yhi, nv.ptr(buf),
                                     nv.stream_ptr()))
    return buf


def unpack(plan, t, region, buf):
    """Contiguous buffer -> region of a CUDA lattice tensor (``hevi_halo_unpack``)."""
    from . import _native as nv
    xlo, xhi, ylo, yhi = region
    nv.check(plan.lib.hevi_halo_unpack(plan.h, nv.ptr(t), t.shape[0], xlo, xhi, ylo, yhi,
                                       nv.ptr(buf), nv.stream_ptr()))


class HaloExchange:
    """Grouped point-to-point halo refresh over torch.distributed.  With a
    plan and CUDA tensors the regions are packed / unpacked by the library's
    halo kernels into reused contiguous buffers (one NCCL send and receive per
    neighbour and phase); CPU tensors (gloo tests) use strided copies."""

    def __init__(self, mesh, px, py, rank, group=None, plan=None):
        self.block, self.phases = halo_plan(mesh, px, py, rank)
        self.group = group
        self.plan = plan
        self._bufs = {}
        self.launches = 0   # halo pack/unpack kernels launched so far

    def _buf(self, key, shape, like):
        """Reused buffer per (direction, phase, peer, shape): the stage state
        (5 fields) and the P' plane (1 field) alternate without reallocating."""
        import torch
        key = key + (tuple(shape),)
        b = self._bufs.get(key)
        if b is None:
            b = torch.empty(shape, dtype=like.dtype, device=like.device)
            self._bufs[key] = b
        return b

    def __call__(self, t):
        import torch
        import torch.distributed as dist
        w = self.block.window
        native = self.plan is not None and t.is_cuda
        for ip, phase in enumerate(self.phases):
            if not phase:
                continue
            ops, recvs = [], []
            for peer, sreg, rreg in phase:
                if native:
                    shp = lambda r: (t.shape[0], t.shape[1], r[3] - r[2], r[1] - r[0])  # noqa: E731
                    sbuf = pack(self.plan, t, sreg, self._buf(("s", ip, peer), shp(sreg), t))
                    self.launches += 1
                    rbuf = self._buf(("r", ip, peer), shp(rreg), t)
                else:
                    sbuf = _view(t, sreg, w).contiguous()
                    rbuf = torch.empty_like(_view(t, rreg, w))
                ops.append(dist.P2POp(dist.isend, sbuf, peer, group=self.group))
                ops.append(dist.P2POp(dist.irecv, rbuf, peer, group=self.group))
                recvs.append((rreg, rbuf))
            for req in dist.batch_isend_irecv(ops):
                req.wait()
            for rreg, rbuf in recvs:
                if native:
                    unpack(self.plan, t, rreg, rbuf)
                    self.launches += 1
                else:
                    _view(t, rreg, w).copy_(rbuf)


class DistributedStepper:
    """One rank of the partitioned fused ARK2 step."""

    def __init__(self, mesh, ref, disc, dt, px, py, rank, exchange=None, tableau=None,
                 set_name="set2nc"):
        self.block = make_block(mesh, px, py, rank)
        self.plan = HeviPlan(mesh, ref, disc, window=self.block.window, set_name=set_name)
        self.exchange = (exchange if exchange is not None
                         else HaloExchange(mesh, px, py, rank, plan=self.plan))
        self.tableau = tableau or imexcore.ark2_tableau()
        self.tab = tableau_array(self.tableau)
        self.dt = float(dt)
        self.lam = self.tableau.diag * self.dt
        self.plan.factor(self.lam)
        self.Q = self.plan.zeros()
        self.work = self.plan.workspace()
        # P'(Q) chained from stage 2 into the next step's stage 0; its halo is
        # then exchanged with the state (stage_inputs(0))
        self.chain = self.plan.chains_pp

    def load_global(self, q_lattice):
        """Copy this rank's window out of a global (5, Z, Y, X) lattice tensor."""
        w = self.block.window
        self.Q[:, :, :, :w["lX"]].copy_(
            q_lattice[:, :, w["y0"]:w["y0"] + w["lY"], w["x0"]:w["x0"] + w["lX"]])
        self.plan.pp_refresh(self.Q, self.work)   # whole window, halos included

    def owned_region(self):
        m = self.plan.mesh
        ex, ey = self.block.ex, self.block.ey
        x0, x1 = ex[0] * m.N, ex[1] * m.N + (1 if ex[1] == m.nx else 0)
        y0, y1 = ey[0] * m.Ny, ey[1] * m.Ny + (1 if ey[1] == m.ny else 0)
        return x0, x1, y0, y1

    def owned(self, t=None):
        t = self.Q if t is None else t
        return _view(t, self.owned_region(), self.block.window)

    def stage_inputs(self, s):
        """Arrays whose halos stage s reads: the stage state, plus (set2nc) the
        P' plane the preceding column solve wrote into field s of the P
        buffer (hevi_stage_solve), so the explicit kernel need not form it."""
        W = self.work
        if s == 0:
            return [self.Q, W[0][0:1]] if self.chain else [self.Q]
        state = W[0] if s == 1 else W[1]
        if self.plan.set_name == "set2c":
            return [state]
        return [state, W[3][s:s + 1]]

    def step_stages(self, overlap=False):
        """Generator over the ordered sub-steps (per stage: [the interior
        tiles,] the halo exchange of the stage inputs, the stage [boundary
        tiles], the solve) so a single-process driver can interleave ranks.
        With ``overlap`` the interior tiles, which read no halo point a
        neighbour provides, are evaluated before the exchange ("pre" marks
        the point where they start)."""
        p, Q, W = self.plan, self.Q, self.work
        for s in range(3):
            pp = self.chain if s == 0 else False
            if overlap:
                yield ("pre", s)
                p.stage(s, self.dt, self.tab, Q, W, pp_valid=pp, part="interior")
            yield ("exchange", self.stage_inputs(s))
            p.stage(s, self.dt, self.tab, Q, W, pp_valid=pp, part="boundary" if overlap else None)
            if s < 2:
                p.stage_solve(s, self.lam, W)
        yield ("done", None)

    def step(self, side_stream=None):
        """One step.  With a side CUDA stream the halo exchange of every stage
        runs on it while the interior tiles run on the current stream; the
        boundary tiles wait for the exchange (event), so the exchange latency
        hides behind the interior sweep."""
        if side_stream is None:
            for kind, ts in self.step_stages():
                if kind == "exchange":
                    for t in ts:
                        self.exchange(t)
            return
        import torch
        main = torch.cuda.current_stream()
        p, Q, W = self.plan, self.Q, self.work
        for s in range(3):
            pp = self.chain if s == 0 else False
            ready = torch.cuda.Event()
            ready.record(main)                    # the previous solve wrote the inputs
            with torch.cuda.stream(side_stream):
                side_stream.wait_event(ready)
                for t in self.stage_inputs(s):
                    self.exchange(t)
                done = torch.cuda.Event()
                done.record(side_stream)
            p.stage(s, self.dt, self.tab, Q, W, pp_valid=pp, part="interior")
            main.wait_event(done)
            p.stage(s, self.dt, self.tab, Q, W, pp_valid=pp, part="boundary")
            if s < 2:
                p.stage_solve(s, self.lam, W)


class LocalExchange:
    """Single-process stand-in for HaloExchange: copies halo regions between
    the windows of several DistributedSteppers living on one device (used to
    check that the partitioned step is bitwise the single-GPU step without
    running ranks that wait on one another)."""

    def __init__(self, mesh, px, py, plans=None):
        self.mesh, self.px, self.py = mesh, px, py
        self.plans = plans

    def fill(self, rank, t_by_rank, phases=(0,)):
        """The given phases for one rank, as HaloExchange: the sender's halo
        kernel packs the region out of its window, the receiver's unpacks it
        into its own."""
        me, plan = halo_plan(self.mesh, self.px, self.py, rank)
        w = me.window
        for ip in phases:
            for peer, sreg, rreg in plan[ip]:
                if self.plans is not None and t_by_rank[rank].is_cuda:
                    buf = pack(self.plans[peer], t_by_rank[peer], rreg)
                    unpack(self.plans[rank], t_by_rank[rank], rreg, buf)
                else:
                    pw = make_block(self.mesh, self.px, self.py, peer).window
                    _view(t_by_rank[rank], rreg, w).copy_(_view(t_by_rank[peer], rreg, pw))

    def fill_all(self, t_by_rank):
        """Every phase on every rank before the next phase, the order the real
        exchange has (one phase: x halos on owned rows, y halos on owned columns)."""
        nph = len(halo_plan(self.mesh, self.px, self.py, 0)[1])
        for ip in range(nph):
            for r in range(len(t_by_rank)):
                self.fill(r, t_by_rank, phases=(ip,))


def run_local_partitioned(steppers, exchange: LocalExchange, nsteps=1, overlap=False, pre=None):
    """Advance all emulated ranks in lock-step on one device.  ``overlap``:
    interior tiles before the exchange; ``pre(stepper, stage)`` runs on every
    rank just before its interior tiles (tests poison the halos there)."""
    if exchange.plans is None:
        exchange.plans = [s.plan for s in steppers]
    for _ in range(nsteps):
        gens = [s.step_stages(overlap=overlap) for s in steppers]
        while True:
            items = [next(g) for g in gens]
            kind = items[0][0]
            if kind == "done":
                break
            if kind == "pre":
                if pre is not None:
                    for s, it in zip(steppers, items):
                        pre(s, it[1])
                continue
            lists = [it[1] for it in items]
            for j in range(len(lists[0])):
                exchange.fill_all([lst[j] for lst in lists])
