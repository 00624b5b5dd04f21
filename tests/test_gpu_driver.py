"""Device simulation driver against the unmodified reference driver
(cli.run_simulation) on its 2D slab bubble / rest state: step counts, dt,
solve counts, the time-series CSV (mass, max |rho'|, max |theta'|, probe)
and the final snapshot table (goldens: tests/golden/make_driver_golden.py)."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

from paper_1702_04316_b200 import driver  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def load(name):
    return np.load(os.path.join(HERE, "golden", f"driver_{name}.npz"))


@pytest.mark.parametrize("name", ["ark2", "rk35", "bdf2_c", "ark2_rest", "ark2_3d", "bdf2_3d_bicg",
                                  "acoustic_ark2", "acoustic_rk35", "acoustic_bdf2_c", "acoustic_ark2_3d"])
def test_run_matches_reference_driver(name, tmp_path):
    g = load(name)
    cfg = driver.parse_config(None, list(g["overrides"]) + [f"--output_dir={tmp_path}"])
    res = driver.run_simulation(cfg, quiet=True)
    assert res.exit_code == int(g["exit_code"]) == 0
    assert res.steps == int(g["steps"])
    assert res.dt == pytest.approx(float(g["dt"]), rel=1e-13)
    assert res.stats.solves == int(g["solves"])
    # Krylov iteration totals: within one per two solves.  The balanced
    # acoustic pulse's momentum R is a near-cancellation, so the reference's
    # P' = P - P0f rounding (|P| eps ~ 1e-11 Pa) seeds noise the reference's
    # GMRES spends iterations on (per solve 6, 6, 4, 4 against 5, 4, 4, 4
    # here); its states still agree below (CSV, snapshot)
    slack = 3 if name == "acoustic_ark2_3d" else max(1, res.stats.solves // 2)
    assert abs(res.stats.iterations - int(g["iterations"])) <= slack
    ts = np.genfromtxt(tmp_path / "timeseries.csv", delimiter=",", names=True)
    mine = np.array([list(r) for r in ts])
    want = g["ts"]
    assert mine.shape == want.shape
    assert open(tmp_path / "timeseries.csv").readline() == str(g["csv"]).splitlines()[0] + "\n"
    np.testing.assert_allclose(mine[:, 0], want[:, 0], rtol=1e-13)            # time
    np.testing.assert_allclose(mine[:, 1], want[:, 1], rtol=1e-13)            # mass
    # max |rho'|, max |theta'|, probe P': relative 1e-8 with absolute floors for
    # states that are round-off noise in the reference (rest state)
    floor = np.array([1e-6, 1e-4, 1e-2])     # P' floor: ulp(P0) ~ 1.5e-11 Pa
    if name == "acoustic_ark2_3d":
        # the acoustic pulse (100 Pa) solved by GMRES to 1e-10: the probe, far
        # from the pulse (~1e-5 Pa), agrees to the solver's ~1e-8 Pa
        floor[2] = 1.0
    scale = np.maximum(np.abs(want[:, 2:]).max(axis=0), floor)
    assert (np.abs(mine[:, 2:] - want[:, 2:]).max(axis=0) <= 1e-8 * scale).all()
    snaps = [f for f in os.listdir(tmp_path) if f.startswith("snapshot_")]
    assert snaps == [str(g["snapshot_name"])]
    snap = np.loadtxt(tmp_path / snaps[0])
    ref = g["snapshot"]
    assert snap.shape == ref.shape
    np.testing.assert_allclose(snap[:, :3], ref[:, :3], rtol=1e-9, atol=1e-9)   # coords
    # rho_p, (u v w) as a vector (v in the slab is reference round-off), theta_p;
    # 10 significant digits in the file
    for cols, fl in (((3,), 1e-6), ((4, 5, 6), 1e-4), ((7,), 1e-4)):
        s = max(np.abs(ref[:, list(cols)]).max(), fl)
        err = np.abs(snap[:, list(cols)] - ref[:, list(cols)]).max()
        assert err <= 1e-8 * s, (cols, err, s)


@pytest.mark.parametrize("integrator", ["ark2", "rk35"])
def test_aborted_run_writes_the_last_good_state(integrator, tmp_path, monkeypatch):
    """A step that fails inside the fused (in-place) kernels leaves the
    last good state in the snapshot, as the reference driver does
    (cli.py:224-250): exit code 4, snapshot = the state after the good steps."""
    from paper_1702_04316_b200.plan import HeviPlan
    over = list(load("ark2")["overrides"])
    over = [o for o in over if not o.startswith(("--integrator", "--end_time"))]
    dt = float(load("ark2")["dt"])      # approximately this run's dt (the Courant rule)
    name = "rk35" if integrator == "rk35" else "step"
    orig = getattr(HeviPlan, name)
    calls = {"n": 0}

    def poisoned(self, *args, **kw):
        calls["n"] += 1
        if calls["n"] == 3:       # the third step starts from a corrupted state
            args[-2 if name == "rk35" else 2][3].view(-1)[7] = float("nan")
        return orig(self, *args, **kw)
    monkeypatch.setattr(HeviPlan, name, poisoned)
    bad = driver.run_simulation(driver.parse_config(None, over + [
        f"--integrator={integrator}", f"--end_time={10 * dt}", f"--output_dir={tmp_path / 'bad'}"]), quiet=True)
    monkeypatch.setattr(HeviPlan, name, orig)
    good = driver.run_simulation(driver.parse_config(None, over + [
        f"--integrator={integrator}", f"--end_time={2 * bad.dt!r}", f"--output_dir={tmp_path / 'good'}"]),
        quiet=True)
    assert good.exit_code == 0 and good.steps == 2
    assert bad.exit_code == 4 and bad.steps == 2, (bad.exit_code, bad.steps, bad.message)
    b, g = torch.as_tensor(bad.final_q), torch.as_tensor(good.final_q)
    assert torch.equal(b, g), float((b - g).abs().max())
