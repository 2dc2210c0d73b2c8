import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(Path(__file__).resolve().parent))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture
def rng():
    return np.random.default_rng(1234)


def random_coordinate_set(rng, n_atoms, num_types=14, extent=8.0, index_mode=True):
    """Same draws as the reference fixture (pkg/tests/conftest.py:63-71)."""
    from paper_1912_04822_b200.coordsets import CoordinateSet

    coords = rng.uniform(-extent, extent, size=(n_atoms, 3)).astype(np.float32)
    radii = rng.uniform(1.0, 2.2, size=n_atoms).astype(np.float32)
    if index_mode:
        return CoordinateSet(coords=coords, radii=radii, num_types=num_types,
                             type_index=rng.integers(0, num_types, size=n_atoms))
    vec = rng.uniform(0.0, 1.0, size=(n_atoms, num_types)).astype(np.float32)
    return CoordinateSet(coords=coords, radii=radii, num_types=num_types, type_vector=vec)
