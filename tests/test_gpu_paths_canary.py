"""tests/sanitize_paths.py as a GPU test: every kernel family at small sizes with canary-guarded
outputs (no write outside a declared output) and per-step invariants -- the pool refuses
compute-sanitizer, so this is the out-of-bounds evidence that runs with the suite."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_every_kernel_family_canary_clean(cuda):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "sanitize_paths.py")], capture_output=True,
                       text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "all paths ran" in r.stdout
