import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session")
def golden():
    arrs = np.load(os.path.join(GOLDEN_DIR, "ref_golden.npz"))
    with open(os.path.join(GOLDEN_DIR, "ref_golden.json")) as f:
        meta = json.load(f)
    return arrs, meta


@pytest.fixture(scope="session")
def ds():
    from paper_2202_05048_b200.dataset import make_dataset
    return make_dataset(seed=0)


@pytest.fixture(scope="session")
def toys():
    from paper_2202_05048_b200.fixtures import generate_fixture
    return {r: generate_fixture(r, 1) for r in ("lenet-ish", "resnet-toy", "mobile-toy")}
