"""The reference's own C++ API driven through include/bandmatch_b200.hpp on the
B200, compared inside one process with the unmodified reference
(tests/cpp/test_reference_binding.cpp, built by tests/cpp/Makefile)."""
import subprocess
from pathlib import Path

import pytest

BIN = Path(__file__).resolve().parent / "cpp" / "_bin" / "test_reference_binding"


@pytest.mark.gpu
def test_reference_api_through_the_binding():
    if not BIN.exists():
        pytest.skip("binding test binary not built (needs /root/reference at build time)")
    r = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "FAIL" not in r.stdout and r.stdout.count("PASS") >= 11
