import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the sm_100a library")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture
def rng():
    return np.random.default_rng(1234)


@pytest.fixture
def desk_geometry():
    """Table-1 distances with a small detector (reference tests/conftest.py:12-23)."""
    from paper_2005_11976_b200 import ScanGeometry, make_circular_trajectory
    return ScanGeometry(sdd=791.0, sod=679.0, det_cols=65, det_rows=33, pixel_pitch=0.748,
                        principal_point=(32.0, 16.0),
                        stage_angles=make_circular_trajectory(8, np.radians(200.0)))


def load_golden(name):
    path = GOLDEN / name
    if not path.exists():
        pytest.skip(f"golden fixture {name} missing (run tests/golden/make_golden.py)")
    return dict(np.load(path))


@pytest.fixture(scope="session")
def golden_small():
    return load_golden("golden_small.npz")


@pytest.fixture(scope="session")
def golden_sart():
    return load_golden("golden_sart.npz")


@pytest.fixture(scope="session")
def golden_c1():
    return load_golden("golden_c1.npz")


@pytest.fixture(scope="session")
def golden_c2():
    return load_golden("golden_c2.npz")


@pytest.fixture(scope="session")
def oracle():
    sys.path.insert(0, str(ROOT / "oracle"))
    import oracle as orc
    orc.build()
    return orc
