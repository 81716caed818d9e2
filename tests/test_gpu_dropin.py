"""The reference's own test cases compiled against the C++ drop-in headers
(tests/cxx/test_dropin.cpp -> include/ngram/*.hpp -> libngram.so -> the C-ABI -> CUDA)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def test_reference_cases_through_cpp_dropin(cuda):
    exe = os.path.join(ROOT, "tests", "cxx", "test_dropin")
    if not os.path.exists(exe):
        from paper_2601_21204_b200 import build
        build.build_cxx()
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout
