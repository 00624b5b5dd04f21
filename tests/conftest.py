"""Shared fixtures and markers.

``gpu`` marks tests that need a B200 (run with ``-m gpu`` on the GPU box);
everything else must pass on a CPU-only host with ``-m "not gpu"``.
"""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")

# golden cases: constructor arguments shared by the oracle and the package
CASES = {
    "slab_aniso": dict(nx=5, ny=1, nz=4, Lx=20_000.0, Ly=None, Lz=1000.0, N=4,
                       slab=True, courant=15.0),
    "box3d_n4": dict(nx=4, ny=4, nz=4, Lx=16_000.0, Ly=16_000.0, Lz=400.0, N=4,
                     courant=15.0),
    "box3d_n3_iso": dict(nx=3, ny=2, nz=3, Lx=12_000.0, Ly=8_000.0, Lz=300.0, N=3,
                         background="isothermal", courant=15.0),
    "straka_n7": dict(nx=32, ny=1, nz=4, Lx=51_200.0, Ly=None, Lz=6_400.0, N=7,
                      slab=True, courant=0.7),
    # conservative equation set (set2c, flux form)
    "slab_aniso_c": dict(nx=5, ny=1, nz=4, Lx=20_000.0, Ly=None, Lz=1000.0, N=4,
                         slab=True, courant=15.0, set_name="set2c"),
    "box3d_n4_c": dict(nx=4, ny=4, nz=4, Lx=16_000.0, Ly=16_000.0, Lz=400.0, N=4,
                       courant=15.0, set_name="set2c"),
    # further orders (make_golden.py --extra)
    "box3d_n5": dict(nx=3, ny=3, nz=3, Lx=15_000.0, Ly=15_000.0, Lz=600.0, N=5, courant=15.0),
    "box3d_n6_c": dict(nx=3, ny=2, nz=2, Lx=12_000.0, Ly=8_000.0, Lz=400.0, N=6,
                       courant=15.0, set_name="set2c"),
    "slab_n2": dict(nx=8, ny=1, nz=6, Lx=16_000.0, Ly=None, Lz=600.0, N=2, slab=True,
                    courant=15.0),
    "box3d_n2_iso": dict(nx=4, ny=4, nz=5, Lx=8_000.0, Ly=8_000.0, Lz=500.0, N=2,
                         background="isothermal", courant=15.0),
}


def set_of(name):
    return CASES[name].get("set_name", "set2nc")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


def load_golden(name):
    return np.load(os.path.join(GOLDEN, f"{name}.npz"))


def oracle_for(name, pprime="reference"):
    from oracle.hevi_oracle import BoxOracle
    kw = dict(CASES[name])
    kw.pop("courant")
    return BoxOracle(**kw, pprime=pprime)   # set_name passes through


def rel_scalar(a, b):
    n = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (n if n > 0 else 1.0))


def rel_fields(a, b, floor=1e-30):
    """(rho', |vel| vector, theta') relative L2 errors of 5-field states.

    Velocity is compared as a vector (SURVEY 8(c) gate B): single velocity
    components can be pure reference round-off noise (v in the 2D slab)."""
    a = np.asarray(a)
    b = np.asarray(b)
    nv = np.linalg.norm(b[1:4])
    return (rel_scalar(a[0], b[0]),
            float(np.linalg.norm(a[1:4] - b[1:4]) / max(nv, floor)),
            rel_scalar(a[4], b[4]))
