"""Shared fixtures.  GPU tests carry @pytest.mark.gpu and run on the B200 box
(`pytest -m gpu`); everything else runs on CPU (`pytest -m "not gpu"`)."""

import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
for p in (ROOT, ROOT / "tests"):
    if str(p) not in sys.path:
        sys.path.insert(0, str(p))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running CPU oracle checks")


def golden_npz(name):
    return np.load(GOLDEN / name)


def golden_json(name):
    return json.loads((GOLDEN / name).read_text())


@pytest.fixture(scope="session")
def vehicle():
    from paper_2104_01284_b200 import make_vehicle
    return make_vehicle()


@pytest.fixture(scope="session")
def short_route():
    from paper_2104_01284_b200 import load_fixture_route
    return load_fixture_route("short", seed=2)


@pytest.fixture(scope="session")
def urban_route():
    from paper_2104_01284_b200 import load_fixture_route
    return load_fixture_route("urban", seed=0)
