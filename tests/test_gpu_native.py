"""GPU: the C++ drop-in adapter (include/diffmpm/mpm_batch.hpp) driven from a
native program linked against libdiffmpm.so."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cpp_adapter_smoke():
    exe = os.path.join(ROOT, "tests", "native", "cpp_adapter_smoke")
    assert os.path.exists(exe), "built by __graft_entry__.build()"
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(out.stdout, out.stderr)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "cpp adapter ok" in out.stdout
