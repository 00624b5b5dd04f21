"""CPU tests of the simulation driver (drop-in for dycore.cli run mode and
dycore.bench diagnostics): config parsing and validation, CSV and snapshot
formats, mass weights.  Reference-backed checks are skipped where
/root/reference is absent."""
import os
import sys

import numpy as np
import pytest

from paper_1702_04316_b200 import driver, euler, specgrid

REF = "/root/reference/pkg/src"
needs_reference = pytest.mark.skipif(not os.path.isdir(REF), reason="reference not mounted")


@pytest.fixture(scope="module")
def dyc():
    sys.path.insert(0, REF)
    import dycore
    import dycore.cli
    import dycore.bench
    return dycore


def test_parse_config_defaults_overrides_and_errors(tmp_path):
    p = tmp_path / "run.cfg"
    p.write_text("# comment\nintegrator = ark2\nimex = 1d\nsolver = direct\nnx = 6 # trailing\n")
    cfg = driver.parse_config(str(p), ["--end_time=2.5", "--equation_set=set2c"])
    assert (cfg.integrator, cfg.imex, cfg.solver, cfg.nx, cfg.end_time, cfg.equation_set) == \
        ("ark2", "1d", "direct", 6, 2.5, "set2c")
    assert driver.parse_config(None, ["--integrator=ark2"]).imex == "3d"
    for bad in (["--nope=1"], ["--nx=abc"], ["--solver=lu"], ["--solver=direct"], ["nx=3"],
                ["--disc=dg"], ["--disc=dg", "--equation_set=set2c", "--imex=3d"]):
        with pytest.raises(driver.ConfigError):
            driver.parse_config(None, bad)
    p.write_text("bogus line\n")
    with pytest.raises(driver.ConfigError):
        driver.parse_config(str(p))


def test_unsupported_paths_raise():
    # dG and the standard (5-variable) form are outside the device path
    for ov in (["--disc=dg", "--equation_set=set2c"], ["--integrator=ark2", "--form=standard"]):
        with pytest.raises(NotImplementedError):
            driver._check_supported(driver.parse_config(None, ov))


def test_main_reports_config_errors_with_exit_code_2(tmp_path):
    assert driver.main(["run", str(tmp_path / "missing.cfg")]) == 2
    assert driver.main(["bogus"]) == 2


@needs_reference
def test_csv_format_matches_reference(dyc, tmp_path):
    mine, theirs = driver.Diagnostics(), dyc.bench.Diagnostics()
    for t, m, a, b, p in ((0.0, 1.2345678901234567e6, 1e-3, 0.5, (3.25,)),
                          (0.25, 1.2345678901234e6, 2e-3, 0.4999, (-1e-9,))):
        mine.record_values(t, m, a, b, p)
        theirs.times.append(t); theirs.mass.append(m); theirs.max_rho_p.append(a)
        theirs.max_theta_p.append(b); theirs.probes.append(p)
    mine.write_csv(tmp_path / "a.csv")
    theirs.write_csv(tmp_path / "b.csv")
    assert (tmp_path / "a.csv").read_text() == (tmp_path / "b.csv").read_text()
    with pytest.raises(ValueError):
        mine.record_values(0.1, 1.0, 0.0, 0.0)


@needs_reference
@pytest.mark.parametrize("slab", [True, False])
def test_axis_mass_weights_reproduce_reference_total_mass(dyc, slab):
    if slab:
        rmesh = dyc.specgrid.build_box_mesh(5, 4, 1000.0, 1000.0, 4)
        mesh = specgrid.build_box_mesh(5, 4, 1000.0, 1000.0, 4)
    else:
        pytest.importorskip("oracle.hevi_oracle")
        from oracle.hevi_oracle import BoxOracle
        o = BoxOracle(3, 2, 3, 3000.0, 2000.0, 600.0, 3)
        mesh = specgrid.build_box_mesh_3d(3, 2, 3, 3000.0, 2000.0, 600.0, 3)
    Wx, Wy, Wz = driver.axis_mass_weights(mesh)
    rng = np.random.default_rng(0)
    f = rng.standard_normal((mesh.Z, mesh.Y, mesh.X))
    mine = float(np.einsum("z,y,x,zyx->", Wz, Wy, Wx, f))
    if slab:
        disc = dyc.euler.build_discretization(rmesh)
        x, y, z = mesh.lattice_coords()
        c = rmesh.coords
        gx = np.searchsorted(x, c[..., 0]); gz = np.searchsorted(z, c[..., 2])
        gy = (c[..., 1] > 0).astype(int)
        want = float(np.sum(disc.metrics.wJ * f[gz, gy, gx]))
    else:
        want = float(np.sum(o.wJ * o.from_lattice(np.broadcast_to(f, (5,) + f.shape))[0]))
    assert mine == pytest.approx(want, rel=1e-13)
