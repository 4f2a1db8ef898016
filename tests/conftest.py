import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) and the built CUDA library")


def load_golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


STREAMS = sorted(f[:-5] for f in os.listdir(GOLDEN) if f.startswith("stream_") and f.endswith(".json"))


@pytest.fixture(scope="session")
def kat():
    return load_golden("kat.json")


@pytest.fixture(scope="session")
def verifier():
    from paper_2506_08781_b200 import Verifier
    v = Verifier(0)
    yield v
    v.close()
