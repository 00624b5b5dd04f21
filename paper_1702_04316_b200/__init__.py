"""B200-native HEVI 1D-IMEX ARK2 step (drop-in for the reference ``dycore``
stepper/operator entry points along that path).  See DESIGN.md."""
from . import specgrid, euler, imexcore, columnsolve  # noqa: F401

__version__ = "0.1.0"
