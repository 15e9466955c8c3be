"""The reference's own C++ call sites (build_input_periodic, evaluate,
descriptors, switch_value, ForceFunction in velocity_verlet_step) with the B200
path swapped in through include/hmdp_halomd.hpp; the program links the
reference compiled from its sources (oracle/Makefile `dropin`)."""
import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu
BIN = os.path.join(ROOT, "oracle", "_ref", "dropin_test")


@pytest.mark.skipif(not os.path.exists(BIN), reason="dropin_test not built (needs /root/reference at build time)")
def test_reference_call_sites_with_b200_path():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "DROPIN PASS" in r.stdout, r.stdout + r.stderr
