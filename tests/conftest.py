import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (CUDA) — run on the GPU box")
    config.addinivalue_line("markers", "slow: long-running (full-size oracle runs)")


def golden(name):
    with open(os.path.join(GOLDEN, name)) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def worked():
    return golden("worked_examples.json")


@pytest.fixture(scope="session")
def paper_params():
    return golden("paper_parameters.json")
