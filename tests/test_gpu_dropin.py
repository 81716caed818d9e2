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


@pytest.mark.parametrize("name", ["hashing", "cache", "embedding", "ple"])
def test_reference_test_files_unmodified(cuda, name):
    """The reference's own proj/tests/test_{hashing,cache,embedding,ple}.cpp, compiled unmodified
    against include/ngram (tests/cxx/Makefile, doctest / cpp_int shims) and run on the B200: the
    float cases on the device float path, the double gradient checks on the device fp64 path."""
    exe = os.path.join(ROOT, "tests", "cxx", "_ref_tests", f"test_{name}")
    assert os.path.exists(exe), "build() compiles tests/cxx/_ref_tests from /root/reference (make -C tests/cxx)"
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout[-4000:])
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "| 0 failed |" in r.stdout
