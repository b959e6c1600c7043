"""Structured uniform cell-centred grid (API of the reference's acch/grid.py:23-100).

On the device a field is stored without ghost layers: periodic wrap and the
Neumann mirror are index arithmetic inside the kernels (the reference fills
an explicit ghost layer, grid.py:177-194).  Storage order is the reference's:
axes reversed, x fastest, so flat cell id = i + Nx (j + Ny k).
"""

from __future__ import annotations

import enum
from dataclasses import dataclass

import numpy as np


class BoundaryCondition(enum.Enum):
    PERIODIC = "periodic"
    NEUMANN = "neumann"


@dataclass(frozen=True)
class Grid:
    """Uniform cell-centred mesh on a 2D or 3D box (grid.py:29-60)."""

    counts: tuple
    lengths: tuple
    bc: BoundaryCondition

    def __post_init__(self):
        if len(self.counts) not in (2, 3):
            raise ValueError(f"grid must be 2D or 3D, got {len(self.counts)} axes")
        if len(self.lengths) != len(self.counts):
            raise ValueError("counts and lengths must have the same number of axes")
        if any(int(n) < 4 for n in self.counts):
            raise ValueError(f"need at least 4 cells per axis, got {self.counts}")
        if any(not (float(L) > 0.0) for L in self.lengths):
            raise ValueError(f"box extents must be positive, got {self.lengths}")
        object.__setattr__(self, "counts", tuple(int(n) for n in self.counts))
        object.__setattr__(self, "lengths", tuple(float(L) for L in self.lengths))
        if not isinstance(self.bc, BoundaryCondition):
            object.__setattr__(self, "bc", BoundaryCondition(self.bc))

    @property
    def dim(self) -> int:
        return len(self.counts)

    @property
    def periodic(self) -> bool:
        return self.bc is BoundaryCondition.PERIODIC

    @property
    def spacing(self) -> tuple:
        return tuple(L / n for L, n in zip(self.lengths, self.counts))

    @property
    def cell_volume(self) -> float:
        return float(np.prod(self.spacing))

    @property
    def domain_volume(self) -> float:
        return float(np.prod(self.lengths))

    @property
    def n_cells(self) -> int:
        return int(np.prod(self.counts))

    @property
    def n_store(self) -> int:
        """Cells stored per field on this device (a slab adds ghost planes)."""
        return self.n_cells

    @property
    def array_shape(self) -> tuple:
        """Interior array shape, axis order reversed (x fastest)."""
        return tuple(reversed(self.counts))

    def numpy_axis(self, axis: int) -> int:
        if not 0 <= axis < self.dim:
            raise ValueError(f"axis {axis} out of range for {self.dim}D grid")
        return self.dim - 1 - axis

    def cell_centers(self, axis: int) -> np.ndarray:
        d = self.spacing[axis]
        return (np.arange(self.counts[axis]) + 0.5) * d

    def center_mesh(self) -> tuple:
        coords = [self.cell_centers(a) for a in range(self.dim)]
        mesh = np.meshgrid(*reversed(coords), indexing="ij")
        return tuple(reversed(mesh))
