"""Shared fixtures.  `-m gpu` tests need a CUDA device; everything else runs
on CPU (the driver runs `pytest -m "not gpu"` in a GPU-less container)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (runs the B200 path)")
    config.addinivalue_line("markers", "slow: long-running parity sweep")


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(ROOT, "tests", "golden", "golden.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def orc():
    """The C restatement (oracle/scls_oracle.c) — the checker."""
    from oracle import pyoracle
    if not os.path.exists(pyoracle.ORACLE_SO):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle")], check=True,
                       capture_output=True)
    return pyoracle.oracle_lib()


@pytest.fixture(scope="session")
def ref():
    """The unmodified reference compiled from /root/reference (oracle/_ref)."""
    from oracle import pyoracle
    lib = pyoracle.ref_lib()
    if lib is None:
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    return lib


@pytest.fixture(scope="session")
def ctx():
    from paper_2406_13511_b200 import lib
    with lib.Context(0) as c:
        yield c
