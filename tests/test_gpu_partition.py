"""The column-partitioned step is bitwise the single-GPU step (SURVEY 8(c)
gate C).  Ranks are emulated on one device in lock-step (LocalExchange)
rather than as processes that wait on one another on one GPU."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_1702_04316_b200 import specgrid, euler, imexcore, cases  # noqa: E402
from paper_1702_04316_b200 import distributed as dd  # noqa: E402
from paper_1702_04316_b200.stepper import HeviStepper  # noqa: E402


@pytest.fixture(scope="module")
def setup():
    mesh = specgrid.build_box_mesh_3d(8, 6, 3, 32_000.0, 24_000.0, 300.0, 4)
    ref = euler.hydrostatic_reference(mesh, 300.0)
    disc = euler.build_discretization(mesh)
    q0 = cases.bubble_lattice(mesh, ref, 0.5, (16_000.0, 12_000.0, 150.0), (6000.0, 6000.0, 100.0))
    dt = cases.dt_for_courant(mesh, ref, q0, 15.0)
    return mesh, ref, disc, q0, dt


def single(setup, nsteps):
    mesh, ref, disc, q0, dt = setup
    st = HeviStepper(disc, ref, dt)
    st.set_state(q0, lattice=True)
    st.step(nsteps)
    return st.state(lattice=True).clone()


def _poison_corners(s):
    """NaN into the window points no exchange refreshes (halo corners): the
    single-phase exchange is only right if no kernel ever reads them."""
    w = s.block.window
    x0, x1, y0, y1 = s.owned_region()
    xs = [i for i in range(w["lX"]) if not x0 <= w["x0"] + i < x1]
    ys = [j for j in range(w["lY"]) if not y0 <= w["y0"] + j < y1]
    for j in ys:
        for i in xs:
            s.Q[:, :, j, i] = float("nan")


@pytest.mark.parametrize("world", [2, 4, 8])
def test_partitioned_step_is_bitwise_single_gpu(setup, world):
    mesh, ref, disc, q0, dt = setup
    want = single(setup, 2)
    px, py = dd.grid_for(world)
    ex = dd.LocalExchange(mesh, px, py)
    steppers = [dd.DistributedStepper(mesh, ref, disc, dt, px, py, r, exchange=ex)
                for r in range(world)]
    for s in steppers:
        s.work.fill_(float("nan"))       # nothing a stage reads may be left unwritten
        s.load_global(q0)
        _poison_corners(s)
    dd.run_local_partitioned(steppers, ex, nsteps=2)
    torch.cuda.synchronize()
    for s in steppers:
        s.plan.check_flags()
        x0, x1, y0, y1 = s.owned_region()
        got = s.owned()[..., :x1 - x0]
        assert torch.equal(got, want[:, :, y0:y1, x0:x1]), (world, s.block.rank)


def _poison_halos(s, stage):
    """NaN into every window point the rank does not own, in every array stage
    `stage` reads: the interior tiles run before the exchange refills them."""
    w = s.block.window
    x0, x1, y0, y1 = s.owned_region()
    ox = [i for i in range(w["lX"]) if not x0 <= w["x0"] + i < x1]
    oy = [j for j in range(w["lY"]) if not y0 <= w["y0"] + j < y1]
    for t in s.stage_inputs(stage):
        for i in ox:
            t[:, :, :, i] = float("nan")
        for j in oy:
            t[:, :, j, :] = float("nan")


@pytest.mark.parametrize("world,sn", [(4, "set2nc"), (2, "set2nc"), (4, "set2c")])
def test_overlapped_exchange_is_bitwise_single_gpu(world, sn):
    """Interior tiles before the halo exchange, boundary tiles after it
    (hevi_stage_ex HEVI_STAGE_INTERIOR / _BOUNDARY): with every halo poisoned
    before the interior tiles run, the step is still bitwise the single-GPU
    step, so the interior subset reads no neighbour-provided point."""
    mesh = specgrid.build_box_mesh_3d(24, 24, 2, 96_000.0, 96_000.0, 200.0, 4)
    ref = euler.hydrostatic_reference(mesh, 300.0)
    disc = euler.build_discretization(mesh)
    q0 = cases.bubble_lattice(mesh, ref, 0.5, (40_000.0, 52_000.0, 90.0), (20_000.0, 20_000.0, 60.0),
                              set_name=sn)
    g = torch.Generator(device="cuda").manual_seed(5)
    q0[1:4] += 0.2 * torch.rand(q0[1:4].shape, generator=g, device="cuda", dtype=torch.float64)
    q0[1, :, :, 0] = q0[1, :, :, -1] = 0
    q0[2, :, 0, :] = q0[2, :, -1, :] = 0
    q0[3, 0] = q0[3, -1] = 0
    dt = cases.dt_for_courant(mesh, ref, q0, 15.0, sn)
    st = HeviStepper(disc, ref, dt, set_name=sn)
    st.set_state(q0, lattice=True)
    st.step(2)
    want = st.state(lattice=True).clone()
    px, py = dd.grid_for(world)
    ex = dd.LocalExchange(mesh, px, py)
    steppers = [dd.DistributedStepper(mesh, ref, disc, dt, px, py, r, exchange=ex, set_name=sn)
                for r in range(world)]
    assert any(s.plan.stage_tiles()[0] > 0 for s in steppers)
    for s in steppers:
        s.work.fill_(float("nan"))
        s.load_global(q0)
    dd.run_local_partitioned(steppers, ex, nsteps=2, overlap=True, pre=_poison_halos)
    torch.cuda.synchronize()
    for s in steppers:
        s.plan.check_flags()
        x0, x1, y0, y1 = s.owned_region()
        assert torch.equal(s.owned(), want[:, :, y0:y1, x0:x1]), s.block.rank


def test_side_stream_step_matches_plain_step(setup):
    """DistributedStepper.step(side_stream): the exchange on a side stream,
    interior tiles on the main stream, boundary tiles after the exchange's
    event -- the same bits as the plain step (one rank: the exchange is a
    stream-ordered copy of nothing, the event logic still runs)."""
    mesh, ref, disc, q0, dt = setup
    calls = []
    res = []
    for side in (None, torch.cuda.Stream()):
        s = dd.DistributedStepper(mesh, ref, disc, dt, 1, 1, 0,
                                  exchange=lambda t: calls.append(torch.cuda.current_stream()))
        s.load_global(q0)
        for _ in range(2):
            s.step(side_stream=side)
        torch.cuda.synchronize()
        s.plan.check_flags()
        res.append(s.Q.clone())
    assert torch.equal(res[0], res[1])
    assert any(c == torch.cuda.current_stream() for c in calls)
    assert any(c != torch.cuda.current_stream() for c in calls)


def test_stepper_graph_replay_matches_eager(setup):
    mesh, ref, disc, q0, dt = setup
    want = single(setup, 3)
    st = HeviStepper(disc, ref, dt)
    st.set_state(q0, lattice=True)
    st.capture()          # records (and runs) one step
    st.step(2)
    assert torch.equal(st.state(lattice=True), want)


def test_stepper_graph_replay_matches_eager_set2c(setup):
    """set2c launches its domain-end kernel as a programmatic dependent of
    the sweep: captured in a CUDA graph and replayed it gives the eager bits."""
    mesh, ref, disc, _, _ = setup
    q0 = cases.bubble_lattice(mesh, ref, 0.5, (16_000.0, 12_000.0, 150.0), (6000.0, 6000.0, 100.0),
                              set_name="set2c")
    dt = cases.dt_for_courant(mesh, ref, q0, 15.0, "set2c")
    eager = HeviStepper(disc, ref, dt, set_name="set2c")
    eager.set_state(q0, lattice=True)
    eager.step(3)
    st = HeviStepper(disc, ref, dt, set_name="set2c")
    st.set_state(q0, lattice=True)
    st.capture()          # records (and runs) one step
    st.step(2)
    assert torch.equal(st.state(lattice=True), eager.state(lattice=True))


def test_resident_stepper_matches_drop_in_step(setup):
    mesh, ref, disc, q0, dt = setup
    plan = disc.plan_for(ref)
    E = plan.l2e(q0)
    prob = imexcore.ImplicitProblem(disc=disc, ref=ref, set_name="set2nc", dim="1d",
                                    solver=imexcore.SolverSpec(method="direct"))
    out = imexcore.ark_imex_step(E, dt, imexcore.ark2_tableau(), prob,
                                 euler.make_rhs(ref, disc, "set2nc"))
    want = single(setup, 1)
    assert torch.equal(plan.e2l(out)[..., :mesh.X], want)


@pytest.mark.parametrize("world", [2, 4])
def test_partitioned_set2c_step_is_bitwise_single_gpu(setup, world):
    """Same gate for the conservative set (flux-form kernel, set2c column solve)."""
    mesh, ref, disc, _, _ = setup
    q0 = cases.bubble_lattice(mesh, ref, 0.5, (16_000.0, 12_000.0, 150.0), (6000.0, 6000.0, 100.0),
                              set_name="set2c")
    dt = cases.dt_for_courant(mesh, ref, q0, 15.0, "set2c")
    st = HeviStepper(disc, ref, dt, set_name="set2c")
    st.set_state(q0, lattice=True)
    st.step(2)
    want = st.state(lattice=True).clone()
    px, py = dd.grid_for(world)
    ex = dd.LocalExchange(mesh, px, py)
    steppers = [dd.DistributedStepper(mesh, ref, disc, dt, px, py, r, exchange=ex, set_name="set2c")
                for r in range(world)]
    for s in steppers:
        s.load_global(q0)
    dd.run_local_partitioned(steppers, ex, nsteps=2)
    torch.cuda.synchronize()
    for s in steppers:
        s.plan.check_flags()
        x0, x1, y0, y1 = s.owned_region()
        assert torch.equal(s.owned()[..., :x1 - x0], want[:, :, y0:y1, x0:x1]), (world, s.block.rank)


def test_halo_pack_unpack_kernels_match_strided_copies(setup):
    """hevi_halo_pack / unpack move exactly the region torch slicing selects."""
    mesh, ref, disc, q0, dt = setup
    px, py = dd.grid_for(4)
    s = dd.DistributedStepper(mesh, ref, disc, dt, px, py, 3)
    s.load_global(q0)
    w = s.block.window
    _, phases = dd.halo_plan(mesh, px, py, 3)
    for phase in phases:
        for peer, sreg, rreg in phase:
            buf = dd.pack(s.plan, s.Q, sreg)
            assert torch.equal(buf, dd._view(s.Q, sreg, w).contiguous())
            t = s.Q.clone()
            src = torch.randn_like(dd._view(t, rreg, w).contiguous())
            dd.unpack(s.plan, t, rreg, src)
            assert torch.equal(dd._view(t, rreg, w), src)
            mask = torch.ones_like(t, dtype=torch.bool)
            dd._view(mask, rreg, w).fill_(False)
            assert torch.equal(t[mask], s.Q[mask])        # nothing outside the region moved
