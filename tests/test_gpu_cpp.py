"""C++ drop-in parity: the reference's own dynpr:: types and engines vs the
same calls through include/dynpr_b200.hpp (tests/cpp/shim_parity.cpp, built
by oracle/Makefile next to the reference library)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
BIN = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref", "shim_parity")


@pytest.mark.skipif(not os.path.exists(BIN), reason="shim_parity not built (needs /root/reference at build time)")
def test_cpp_shim_matches_reference(dp):
    out = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "0 failure(s)" in out.stdout
