"""The reference's own unit tests (proj/tests/test_{cost_model,distribution,
distribution_spec,cache_planner,trace,simulator}.cpp), compiled unchanged
against include/embcomm/*.hpp and linked to libembcomm_gpu.so (SURVEY §8(b):
the drop-in boundary).  tests/cpp/Makefile builds them where /root/reference
exists (__graft_entry__.build()); the binary travels to the GPU box.

CPU: every case that needs no device passes; the GPU ones (sampler,
simulator, skew table, hot/normal partition) report a DeviceError and are
skipped.  GPU: all 63 cases pass, including the reference's statistical
checks, since every SimResult field is bit-identical to the reference's."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "_bin", "ref_unit_tests")
N_CASES = 63


def _run(*args):
    if not os.path.exists(BIN):
        pytest.skip("tests/cpp/_bin/ref_unit_tests not built (needs /root/reference once)")
    r = subprocess.run([BIN, *args], capture_output=True, text=True, timeout=900)
    m = re.search(r"test cases: (\d+) \| (\d+) passed \| (\d+) failed \| (\d+) skipped", r.stdout)
    assert m, r.stdout[-3000:] + r.stderr[-2000:]
    return r, [int(x) for x in m.groups()]


def test_reference_unit_tests_host_cases():
    r, (cases, passed, failed, skipped) = _run("--skip-device")
    assert r.returncode == 0 and failed == 0, r.stdout[-4000:]
    assert cases == N_CASES
    assert passed + skipped == cases and passed >= 40  # cost model, planner, distributions, specs, trace text I/O


@pytest.mark.gpu
def test_reference_unit_tests_all_cases_on_gpu():
    r, (cases, passed, failed, skipped) = _run()
    assert r.returncode == 0 and failed == 0, r.stdout[-4000:]
    assert (cases, passed, skipped) == (N_CASES, N_CASES, 0)
