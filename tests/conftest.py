import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = Path(__file__).resolve().parent / "golden"
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU and the built libtacsl_b200.so")


@pytest.fixture(scope="session")
def golden():
    def load(name):
        return np.load(GOLDEN / f"{name}.npz")
    return load


@pytest.fixture(scope="session")
def golden_grid():
    """The reference-built (gelsim build_sdf) 16x16x32 peg grid, float64."""
    from paper_2408_06506_b200.geometry import SdfGrid

    z = np.load(GOLDEN / "sdf.npz")
    return SdfGrid(origin=z["origin"], spacing=float(z["spacing"]), dims=tuple(int(v) for v in z["dims"]),
                   values=z["values"], gradients=z["gradients"])


def sdf_tuple(grid):
    return (grid.origin, grid.spacing, grid.dims, grid.values, grid.gradients)


def vec_close(got, ref, rtol=1e-5, atol=1e-12):
    """Per-vector ||got - ref|| <= rtol ||ref|| + atol (the 1e-5 relative
    force-field contract of BASELINE.json, with an absolute floor for
    zero vectors).  Returns (ok, worst relative excess)."""
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    err = np.linalg.norm(got - ref, axis=-1)
    bound = rtol * np.linalg.norm(ref, axis=-1) + atol
    return bool(np.all(err <= bound)), float(np.max(err / bound)) if err.size else 0.0
