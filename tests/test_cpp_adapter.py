"""The C++ drop-in (include/ndgx_ndg.hpp) replayed on the reference's own test
scenarios against the unmodified reference library (tests/cpp/test_adapter.cpp)."""
import os
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
BIN = os.path.join(HERE, "cpp", "_build", "test_adapter")


@pytest.mark.gpu
def test_cpp_dropin_matches_reference_library():
    if not os.path.exists(BIN):
        pytest.skip("tests/cpp/_build/test_adapter not built (needs /root/reference at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "FAIL" not in r.stdout
