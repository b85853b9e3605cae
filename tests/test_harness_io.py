"""Host-side file formats of the harness integration (no GPU)."""

import numpy as np
import pytest

from paper_1903_07884_b200.errors import ConfigError
from paper_1903_07884_b200.grid import VoxelGrid
from paper_1903_07884_b200.harness import (homog_internal, read_field, read_residuals, write_field,
                                           write_residuals)


def test_field_roundtrip(tmp_path, rng):
    grid = VoxelGrid(4, 3, 2, 0.05)
    f = rng.normal(size=grid.n_unknowns) + 1j * rng.normal(size=grid.n_unknowns)
    write_field(tmp_path / "field.bin", grid, f, wavelength=1.55e-6)
    g, side = read_field(tmp_path / "field.bin")
    assert np.array_equal(g, f) and side["dims"] == [4, 3, 2]
    with pytest.raises(ValueError):
        write_field(tmp_path / "bad.bin", grid, f[:5])


def test_residuals_roundtrip(tmp_path):
    res = [1.0, 0.5, 1e-3, 2e-6]
    write_residuals(tmp_path / "r.csv", res, 0.01)
    assert read_residuals(tmp_path / "r.csv") == res


def test_homog_names():
    assert homog_internal("real-mean-x") == "real_mean_x"
    with pytest.raises(ConfigError):
        homog_internal("median")
