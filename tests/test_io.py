"""History CSV / VTK writers (io.py) against the bytes the reference's
cli/io.py:19-198 writes (golden io.npz) -- host code, no GPU."""

import numpy as np

from conftest import golden

from paper_2007_04560_b200.drivers import HistoryRow
from paper_2007_04560_b200.grid import BoundaryCondition, Grid
from paper_2007_04560_b200.io import (HISTORY_HEADER, read_history, read_vtk, write_history, write_vtk,
                                      write_xy)


class HostState:
    """Stand-in with the State surface write_vtk uses (grid, to_numpy)."""

    def __init__(self, grid, u, v):
        self.grid, self.u_, self.v_ = grid, u, v

    def to_numpy(self):
        return self.u_.copy(), self.v_.copy()


def _rows(z):
    return [HistoryRow(int(r[0]), r[1], r[2], r[3], r[4], r[5], int(r[6]), int(r[7]), r[8]) for r in z["rows"]]


def test_history_csv_bytes_match_reference(tmp_path):
    z = golden("io.npz")
    path = tmp_path / "sub" / "history.csv"
    write_history(_rows(z), str(path))
    assert path.read_text() == str(z["csv"])
    assert path.read_text().splitlines()[0] == HISTORY_HEADER
    back = read_history(str(path))
    assert [(r.step, r.time, r.energy, r.gmres) for r in back] == [(r.step, r.time, r.energy, r.gmres)
                                                                      for r in _rows(z)]


def test_vtk_bytes_match_reference_and_round_trip(tmp_path):
    z = golden("io.npz")
    for tag in ("2d", "3d"):
        counts = tuple(int(c) for c in z[f"counts_{tag}"])
        g = Grid(counts, tuple(float(x) for x in z[f"lengths_{tag}"]), BoundaryCondition.PERIODIC)
        path = tmp_path / f"{tag}.vtk"
        write_vtk(HostState(g, z[f"u_{tag}"], z[f"v_{tag}"]), str(path), title=f"snapshot {tag}")
        assert path.read_text() == str(z[f"vtk_{tag}"])
        meta = read_vtk(str(path))
        np.testing.assert_array_equal(meta["arrays"]["u"], z[f"u_{tag}"].ravel())
        np.testing.assert_array_equal(meta["arrays"]["v"], z[f"v_{tag}"].ravel())
        assert meta["dimensions"][:len(counts)] == counts


def test_write_xy(tmp_path):
    write_xy(str(tmp_path / "a.dat"), [1.0, 0.1], [3.0, 1e-17])
    assert (tmp_path / "a.dat").read_text() == "1 3\n0.10000000000000001 1.0000000000000001e-17\n"
