"""GPU: the C++ drop-in headers (include/pmagraph/*.hpp) used the way the
reference's own tests use the reference API (tests/cpp/test_dropin.cpp),
linked against libpmagraph_cuda.so."""
import os
import subprocess

import pytest

from paper_1709_05061_b200 import build as b

pytestmark = pytest.mark.gpu


def test_cpp_dropin_program():
    exe = b.build_cpp_tests()
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "ok: 0 failure(s)" in r.stdout
