import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through libuwbnli.so on cuda:0)")


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(ROOT, "tests", "golden", "golden.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def golden_cfm():
    with open(os.path.join(ROOT, "tests", "golden", "golden_cfm.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def golden_stress():
    with open(os.path.join(ROOT, "tests", "golden", "golden_stress.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def oracle():
    from pyoracle import Oracle, build_oracle

    build_oracle()
    return Oracle()


@pytest.fixture(scope="session")
def engine():
    import paper_2401_18022_b200 as uwb

    eng = uwb.Engine(0)
    yield eng
    eng.close()
