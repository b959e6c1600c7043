"""B200-native per-time-step Newton-Krylov-Schwarz solver for the coupled
Allen-Cahn / Cahn-Hilliard system with logarithmic free energy
(arXiv 2007.04560), with the reference package ``acch``'s solver API.

Modules mirror the reference: grid, physics, scheme, linalg, newton,
timestep, drivers (simulate).  All numerics run in hand-written sm_100a
kernels in libacch_b200.so (C ABI: include/acch_b200.h) loaded via ctypes.
"""

from .grid import BoundaryCondition, Grid
from .physics import Field, Params, State

__all__ = ["BoundaryCondition", "Field", "Grid", "Params", "State"]
__version__ = "0.1.0"
