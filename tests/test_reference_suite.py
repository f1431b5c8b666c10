"""The reference's OWN test files (batcher, offloader, sim_engine,
sched_policies, metrics, and the 11-criterion acceptance gate), compiled
unchanged by tests/refsuite/Makefile:

  *_ref   against the unmodified reference core — proves the gtest shim
          harness (CPU, runs here);
  *_b200  against the B200 drop-in (batch_requests / offload /
          Simulator::run / sweep on the GPU via libscls_b200.so) — the
          reference's own parity suite passing on the new implementation.

The binaries are built where /root/reference exists (build()) and travel to
the GPU box with the repository snapshot."""
import os
import subprocess

import pytest

from tests.conftest import ROOT

SUITE = ["batcher_test", "offloader_test", "sim_engine_test", "sched_policies_test", "metrics_test",
         "acceptance_test"]
BIN = os.path.join(ROOT, "build", "refsuite")


def _run(path):
    p = subprocess.run([path], capture_output=True, text=True, timeout=900)
    return p.returncode, p.stdout + p.stderr


def _require(path):
    if not os.path.exists(path):
        if os.path.isdir("/root/reference/proj/tests"):
            subprocess.run(["make", "-C", os.path.join(ROOT, "tests", "refsuite"), "-j8"], check=True,
                           capture_output=True)
        else:
            pytest.skip(f"{path} not built and /root/reference (its sources) unavailable here")


@pytest.mark.parametrize("name", SUITE)
def test_reference_suite_on_reference(name):
    path = os.path.join(BIN, name + "_ref")
    _require(path)
    rc, out = _run(path)
    assert rc == 0, out[-3000:]
    assert "0 failed" in out


@pytest.mark.gpu
@pytest.mark.parametrize("name", SUITE)
def test_reference_suite_on_b200(name):
    path = os.path.join(BIN, name + "_b200")
    _require(path)
    rc, out = _run(path)
    assert rc == 0, out[-3000:]
    assert "0 failed" in out
    if name == "acceptance_test":
        assert out.count("PASS") == 11, out


def _post_run_state(kind):
    path = os.path.join(BIN, "post_run_state_" + kind)
    _require(path)
    p = subprocess.run([path], capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stderr[-2000:]
    return p.stdout


def test_post_run_state_reference_harness():
    out = _post_run_state("ref")
    assert out.count("horizon: simulated clock reached horizon") == 9, out[-2000:]


@pytest.mark.gpu
def test_post_run_state_b200_matches_reference():
    """clock(), request(id) progress, workers() loads / busy_until and the
    NonTermination message after Simulator::run, drop-in vs reference
    (sim_engine.h:64-79, sim_engine.cpp:159-163)."""
    want = _post_run_state("ref").splitlines()
    got = _post_run_state("b200").splitlines()
    assert len(got) == len(want)
    for a, b in zip(got, want):
        assert a == b, (a, b)
