"""The reference's OWN unit tests on the B200 drop-in (VERDICT
r1 next-round item 6): /root/reference/proj/tests/test_batch_sizer.cpp,
test_predictor.cpp, test_coordination.cpp and test_sgd.cpp are compiled
unchanged -- their `#include "lbbsp/..."` resolve to include/lbbsp/*.hpp (the
reference types over the C-ABI of liblbbsp_b200.so) and <doctest.h> to the
minimal harness in tests/cpp/doctest/ -- by tests/cpp/Makefile at build time
(the binary travels with the repo; /root/reference is not read here)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

BIN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp", "_refbin", "ref_unit_tests")


def test_reference_unit_tests_pass_on_the_b200_shim():
    if not os.path.exists(BIN):
        pytest.skip("tests/cpp/_refbin/ref_unit_tests not built (needs /root/reference at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    tail = r.stdout[-3000:] + r.stderr[-3000:]
    assert r.returncode == 0, tail
    assert "| 0 failed" in r.stdout, tail
