"""The reference's OWN doctest suites (/root/reference/proj/tests/test_{coefficients,graph,
cpaa,power,metrics}.cpp), compiled unchanged against the C++ drop-in layer
(include/chebpr/*.hpp + libchebpr_dropin.so over the C-ABI) by `make reftests` where the
reference sources exist; the binaries travel with the repo to the GPU box.  The
coefficient suite is host-only; the others run their solves on the B200."""
import os
import subprocess

import pytest

from conftest import ROOT

BIN = os.path.join(ROOT, "build", "reftests")


def run_suite(name):
    path = os.path.join(BIN, name)
    if not os.path.exists(path):
        pytest.skip(f"{path} not built (needs /root/reference at build time)")
    p = subprocess.run([path], capture_output=True, text=True, timeout=900)
    summary = p.stdout.strip().splitlines()[-1] if p.stdout.strip() else ""
    assert p.returncode == 0, f"{name} failed:\n{p.stderr[-4000:]}\n{summary}"
    assert "| 0 failed |" in summary, summary
    return summary


def test_reference_coefficient_suite_host():
    run_suite("test_coefficients")


@pytest.mark.gpu
@pytest.mark.parametrize("suite", ["test_graph", "test_cpaa", "test_power", "test_metrics"])
def test_reference_suite_on_b200(suite):
    run_suite(suite)
