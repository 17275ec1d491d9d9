"""CPU: the product's host-side bookkeeping (C++ drop-in API: make_task_specs,
trace_from_work/trace_csv, warp_steps_*, the image_io writers, compare_outputs,
binning_csv, scene JSON) against the reference's own code (oracle/_ref), via
the C++ driver tests/cpp/test_ref_host.cpp.  No GPU needed: none of these
functions launch kernels."""
import os
import subprocess

import pytest

import ref_lib as R

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "paper_2412_17378_b200", "build", "test_ref_host")

pytestmark = pytest.mark.skipif(not R.available(), reason="oracle/_ref not built and /root/reference absent")


def test_host_bookkeeping_matches_reference(tmp_path):
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "paper_2412_17378_b200"), "test-ref-bin"], check=True)
    r = subprocess.run([BIN, R.REF_LIB, str(tmp_path)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "OK:" in r.stdout and " 0 failure(s)" in r.stdout
