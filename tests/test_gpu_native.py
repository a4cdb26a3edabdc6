"""GPU: the C++ drop-in adapter (include/diffmpm/mpm_batch.hpp) driven from a
native program linked against libdiffmpm.so."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cpp_adapter_smoke():
    import hostcheck
    exe = hostcheck.build_cpp_smoke()  # rebuilt when the ABI headers changed
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(out.stdout, out.stderr)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "cpp adapter ok" in out.stdout
