"""GPU: run the C++ drop-in API test driver (tests/cpp/test_host_api.cpp),
which calls splatsim::project_all / bin_tiles / tile_load_histogram /
render_reference / run_kernel / checkpoint like the reference's C++ callers and
checks every result against the CPU oracle."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "paper_2412_17378_b200", "build", "test_host_api")


def test_cpp_api_driver():
    if not os.path.exists(BIN):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "paper_2412_17378_b200"), "test-bin"], check=True)
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "OK: 0 failure(s)" in r.stdout
