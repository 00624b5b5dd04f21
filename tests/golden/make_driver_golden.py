"""Golden runs of the UNMODIFIED reference driver (``dycore.cli.run_simulation``)
for the device driver's parity tests (tests/test_gpu_driver.py).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_driver_golden.py

Each case runs the reference's own config path on its 2D slab bubble and
stores the time-series CSV columns, the final snapshot table, dt, the step
count and the solve count in ``tests/golden/driver_<case>.npz``."""
from __future__ import annotations

import os
import sys
import tempfile

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
sys.dont_write_bytecode = True

from dycore import cli  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

CASES = {
    "ark2": ["--integrator=ark2", "--imex=1d", "--solver=direct", "--nx=4", "--nz=4",
             "--courant=2", "--end_time=1.0"],
    "rk35": ["--integrator=rk35", "--nx=4", "--nz=4", "--courant=0.5", "--end_time=0.3"],
    "bdf2_c": ["--integrator=bdf2", "--imex=1d", "--solver=direct", "--equation_set=set2c",
               "--nx=4", "--nz=4", "--courant=2", "--end_time=1.0"],
    "ark2_rest": ["--case=rest-state", "--integrator=ark2", "--imex=1d", "--solver=direct",
                  "--nx=3", "--nz=3", "--courant=3", "--end_time=0.5", "--diag_interval=0.2"],
    "ark2_3d": ["--integrator=ark2", "--imex=3d", "--solver=gmres", "--tolerance=1e-10",
                "--nx=4", "--nz=4", "--courant=2", "--end_time=0.6"],
    "bdf2_3d_bicg": ["--integrator=bdf2", "--imex=3d", "--solver=bicgstab", "--precon_order=3",
                     "--tolerance=1e-10", "--nx=4", "--nz=4", "--courant=2", "--end_time=0.8"],
    # the cubed-sphere acoustic case (cli.py:131-141)
    "acoustic_ark2": ["--case=acoustic", "--integrator=ark2", "--imex=1d", "--solver=direct",
                      "--ne_panel=2", "--ne_vert=2", "--order=3", "--courant=4", "--end_time=60"],
    "acoustic_rk35": ["--case=acoustic", "--integrator=rk35", "--ne_panel=2", "--ne_vert=1",
                      "--order=3", "--courant=0.5", "--end_time=4"],
    "acoustic_ark2_3d": ["--case=acoustic", "--integrator=ark2", "--imex=3d", "--solver=gmres",
                         "--tolerance=1e-10", "--ne_panel=2", "--ne_vert=1", "--order=3", "--courant=4",
                         "--end_time=40"],
    "acoustic_bdf2_c": ["--case=acoustic", "--integrator=bdf2", "--imex=1d", "--solver=direct",
                        "--equation_set=set2c", "--ne_panel=2", "--ne_vert=2", "--order=3",
                        "--courant=4", "--end_time=60"],
}


def main():
    only = set(sys.argv[1:])
    for name, ov in CASES.items():
        if only and name not in only:
            continue
        with tempfile.TemporaryDirectory() as d:
            cfg = cli.parse_config(None, ov + [f"--output_dir={d}"])
            res = cli.run_simulation(cfg, quiet=True)
            ts = np.genfromtxt(os.path.join(d, "timeseries.csv"), delimiter=",", names=True)
            snaps = [f for f in os.listdir(d) if f.startswith("snapshot_")]
            snap = np.loadtxt(os.path.join(d, snaps[0]))
            csv_text = open(os.path.join(d, "timeseries.csv")).read()
        np.savez_compressed(os.path.join(HERE, f"driver_{name}.npz"), overrides=np.array(ov),
                            ts=np.array([list(r) for r in ts]), csv=np.array(csv_text),
                            snapshot=snap, snapshot_name=np.array(snaps[0]), dt=res.dt,
                            steps=res.steps, solves=res.stats.solves, exit_code=res.exit_code,
                            iterations=res.stats.iterations)
        print(name, res.steps, res.dt, res.exit_code, res.stats.solves, res.stats.iterations)


if __name__ == "__main__":
    main()
